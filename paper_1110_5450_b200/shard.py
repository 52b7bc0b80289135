"""Sharded compacting clip across the GPUs of one node.

Segments are independent, so the array is partitioned contiguously: rank r owns global
indices [floor(r n / P), floor((r+1) n / P)).  Each rank runs the one-pass compacting
kernel on its shard; the only exchange is an NCCL allgather of the P int64 visible
counts (8 bytes per rank, over NVLink/NVSwitch), after which the K4 kernel turns them
into this rank's global output offset and the total.  No segment data crosses GPUs: the
output stays sharded, rank r owning global compacted rows [offset_r, offset_r + c_r);
out_index is already global through index_base = shard start.

torch.distributed is plumbing here (process group, allgather); all compute is in
libclipseg.so.  The local clip and offset functions are parameters so the host logic
can be exercised on CPU ranks (gloo) in tests.
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_range(n: int, world: int, rank: int):
    """Contiguous shard [start, stop) of n segments for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    return n * rank // world, n * (rank + 1) // world


@dataclass
class ShardResult:
    start: int          # global index of this rank's first segment
    count: object       # local visible count (device int64[1])
    offsets: object     # device int64[2]: (global output offset of this rank, total)
    counts: object      # allgathered counts (device int64[world])


def nccl_exchange(count, world, group=None):
    """All-gather of the per-rank visible counts (int64[1] device tensors) over NCCL."""
    import torch  # noqa: PLC0415
    import torch.distributed as dist  # noqa: PLC0415

    counts = torch.empty(world, dtype=torch.int64, device=count.device)
    dist.all_gather_into_tensor(counts, count, group=group)
    return counts


def host_exchange(count, world, group=None):
    """The same exchange through host memory, for process groups whose backend cannot gather
    device tensors (gloo): count -> host, all_gather, counts -> the count's device."""
    import torch  # noqa: PLC0415
    import torch.distributed as dist  # noqa: PLC0415

    parts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, count.cpu(), group=group)
    return torch.cat(parts).to(count.device)


def sharded_compact(local_planes, n_local, lo, hi, start, group=None, bufs=None, stream=None,
                    compact_fn=None, offsets_fn=None, exchange_fn=None):
    """Compact this rank's shard and fix its global output offset.

    compact_fn(planes, n, lo, hi, bufs, index_base) -> bufs with .count (int64[1] tensor);
    offsets_fn(counts, rank) -> int64[2] tensor (offset, total);
    exchange_fn(count, world, group) -> int64[world] counts (default: nccl_exchange).
    Defaults: the CUDA path.  Every step is issued on `stream` (torch's current stream when
    None): the compaction, the allgather (NCCL orders against the current stream, which is
    `stream` inside the block) and the offsets kernel, so none reads a count before it is
    written."""
    import contextlib  # noqa: PLC0415

    import torch  # noqa: PLC0415
    import torch.distributed as dist  # noqa: PLC0415

    if compact_fn is None or offsets_fn is None:
        from . import clipseg  # noqa: PLC0415

        def _cf(p, n, lo_, hi_, b, base):
            return clipseg.clip_compact(p, n, lo_, hi_, bufs=b, with_index=True, index_base=base, stream=stream)

        compact_fn = compact_fn or _cf
        offsets_fn = offsets_fn or (lambda c, r: clipseg.shard_offsets(c, r, stream=stream))
    exchange_fn = exchange_fn or nccl_exchange
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        bufs = compact_fn(local_planes, n_local, lo, hi, bufs, start)
        counts = exchange_fn(bufs.count, world, group)
        offsets = offsets_fn(counts, rank)
    return ShardResult(start=start, count=bufs.count, offsets=offsets, counts=counts), bufs
