"""Sharded mode host logic on CPU ranks (gloo, world_size 2): contiguous partition,
count allgather, global offsets; the concatenation of the per-rank compacted slices at
their offsets equals the single-rank result.  The local compaction is the
oracle here (test infrastructure); on GPUs it is the CUDA kernel (tests/test_gpu_*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1110_5450_b200.shard import shard_range, sharded_compact

N = 50021
LO, HI = [0.0, 0.0], [1.0, 1.0]


class _Bufs:
    pass


def _oracle_compact(planes, n, lo, hi, bufs, base):
    out, idx, cnt = oracle.compact(planes, n, lo, hi, 2, index_base=base)
    b = _Bufs()
    b.out, b.index, b.count = out, idx, torch.tensor([cnt], dtype=torch.int64)
    return b


def _offsets(counts, rank):
    c = counts.tolist()
    return torch.tensor([sum(c[:rank]), sum(c)], dtype=torch.int64)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N, world, rank)
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(5), b - a, i0=a)
    res, bufs = sharded_compact(planes, b - a, LO, HI, a, compact_fn=_oracle_compact, offsets_fn=_offsets)
    c = int(res.count.item())
    q.put((rank, int(res.offsets[0]), int(res.offsets[1]), res.counts.tolist(),
           bufs.out[:, :c].copy(), bufs.index[:c].copy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 10**9):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_sharded_compaction_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=120) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(5), N)
    want, widx, wcnt = oracle.compact(planes, N, LO, HI, 2)
    total = got[0][2]
    assert total == wcnt == got[1][2]
    assert got[0][3] == got[1][3]                       # same allgathered counts
    assert got[0][1] == 0 and got[1][1] == got[0][3][0]  # offsets = exclusive prefix
    cat = np.concatenate([g[4] for g in got], axis=1)
    idx = np.concatenate([g[5] for g in got])
    assert np.array_equal(cat.view(np.uint32), want[:, :wcnt].view(np.uint32))
    assert np.array_equal(idx, widx)                    # global indices via index_base
