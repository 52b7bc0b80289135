"""Sharded mode with P >= 2 ranks on the real CUDA path (BASELINE configs[4]).

Each rank is a process on cuda:0 running the production pieces — the seeded generator,
the compacting kernel on its contiguous shard (index_base = shard start), the count
exchange and the K4 offsets kernel — with the 8-byte count exchange carried by a gloo
group through host memory (one GPU on the test box; NCCL needs one GPU per rank).  The
per-rank compacted slices placed at their offsets must equal the single-rank oracle
output bit for bit, indices included.  The ranks' kernels never wait on one another: the
only cross-rank step is the host-side exchange."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

LO, HI = [0.0, 0.0], [1.0, 1.0]


def _worker(rank, world, port, n, fam, q):
    import torch
    import torch.distributed as dist

    from paper_1110_5450_b200 import clipseg
    from paper_1110_5450_b200.shard import host_exchange, shard_range, sharded_compact

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        a, b = shard_range(n, world, rank)
        planes = clipseg.empty_planes(max(b - a, 1), 2, torch.float32)
        synth.fill_device(planes, fam, 2, synth.seed_for(5), b - a, i0=a)
        stream = torch.cuda.Stream()  # a non-current stream: every step must be ordered on it
        stream.wait_stream(torch.cuda.current_stream())
        res, bufs = sharded_compact(planes, b - a, LO, HI, a, stream=stream, exchange_fn=host_exchange)
        torch.cuda.synchronize()
        c = int(res.count.item())
        q.put((rank, res.offsets.tolist(), res.counts.tolist(), bufs.out[:, :c].cpu().numpy(),
               bufs.index[:c].cpu().numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n,fam", [(2, 1_000_003, synth.UNIFORM), (3, 777_777, synth.UNIFORM),
                                         (2, 200_003, synth.ADVERSARIAL), (4, 5, synth.UNIFORM)])
def test_multi_rank_sharded_compaction_matches_single_rank(world, n, fam):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, fam, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    planes, _ = synth.fill_host(fam, 2, synth.seed_for(5), n)
    want, widx, wcnt = oracle.compact(planes, n, LO, HI, 2)
    counts = got[0][2]
    assert all(g[2] == counts for g in got)                 # every rank holds the same counts
    assert sum(counts) == wcnt
    for r, g in enumerate(got):
        assert g[1] == [sum(counts[:r]), wcnt]              # offset = exclusive prefix, total
    cat = np.concatenate([g[3] for g in got], axis=1)
    idx = np.concatenate([g[4] for g in got])
    assert np.array_equal(cat.view(np.uint32), want[:, :wcnt].view(np.uint32))
    assert np.array_equal(idx, widx)                        # global indices via index_base
