"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element,
on the same seeded inputs.  Bar: bit-exact flags, compaction order, counts AND endpoints
(the kernel executes the same IEEE operations the rules prescribe), which implies the
north-star tolerances (1e-6 x extent fp32, 1e-14 fp64)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

UNIT = {2: ([0.0, 0.0], [1.0, 1.0]), 3: ([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])}
# sizes spanning several compacting tiles with exact and ragged ends (round-1 tiles: fp32 2D
# 4096, fp32 3D 2816, fp64 2D 2048, fp64 3D 1024 segments; packed-kernel tiles: PACKED_TILES)
SIZES = [1, 3, 4, 5, 31, 1023, 1024, 1025, 2815, 2816, 2817, 4097, 8448, 10007, 100003, 1 << 20]
# packed compacting kernel block tiles (compute warps x batch, clip_kernels.cuh knobs)
PACKED_TILES = {(2, np.float32): 15 * 256, (3, np.float32): 10 * 256, (2, np.float64): 11 * 128}


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def to_dev(torch, planes):
    return torch.from_numpy(np.ascontiguousarray(planes)).cuda()


def gen(family, dim, seed, n, dtype, mix=(1 / 3, 1 / 3)):
    pin, pc = synth.mix_thresholds(*mix)
    planes, tag = synth.fill_host(family, dim, seed, n, dtype=dtype, p_in=pin, p_cross=pc)
    return planes, tag


def check_dense(torch, cs, planes, n, lo, hi, dim):
    want, wflags = oracle.clip(planes, n, lo, hi, dim, nthreads=8)
    d_in = to_dev(torch, planes)
    out, flags = cs.clip(d_in, n, lo, hi)
    torch.cuda.synchronize()
    got, gflags = out.cpu().numpy(), flags.cpu().numpy()[:n]
    assert np.array_equal(gflags, wflags), np.nonzero(gflags != wflags)[0][:10]
    diff = np.nonzero(np.any(bits(got[:, :n]) != bits(want[:, :n]), axis=0))[0]
    assert len(diff) == 0, (diff[:5], planes[:, diff[:3]], got[:, diff[:3]], want[:, diff[:3]])
    return wflags


def check_compact(torch, cs, planes, n, lo, hi, dim, index_base=0):
    want, widx, wcnt, wflags = oracle.compact(planes, n, lo, hi, dim, index_base=index_base, with_flags=True)
    d_in = to_dev(torch, planes)
    b = cs.clip_compact(d_in, n, lo, hi, with_index=True, with_flags=True, index_base=index_base)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert cnt == wcnt
    assert np.array_equal(b.flags.cpu().numpy()[:n], wflags)
    assert np.array_equal(b.index.cpu().numpy()[:cnt], widx)
    got = b.out.cpu().numpy()
    assert np.array_equal(bits(got[:, :cnt]), bits(want[:, :cnt]))


@pytest.mark.parametrize("n", SIZES)
def test_dense_2d_f32_uniform_sizes(torch, cs, n):
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(1), n, np.float32)
    check_dense(torch, cs, planes, n, *UNIT[2], 2)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("family", [synth.UNIFORM, synth.MIX, synth.ADVERSARIAL])
def test_dense_families(torch, cs, dim, dtype, family):
    n = 300007
    planes, _ = gen(family, dim, synth.seed_for(2, family), n, dtype)
    check_dense(torch, cs, planes, n, *UNIT[dim], dim)


@pytest.mark.parametrize("mix", [(0.10, 0.80), (1 / 3, 1 / 3), (0.90, 0.05)])
def test_dense_mix_sweep_ground_truth(torch, cs, mix):
    n = 1 << 20
    planes, tag = gen(synth.MIX, 2, synth.seed_for(2), n, np.float32, mix)
    flags = check_dense(torch, cs, planes, n, *UNIT[2], 2)
    assert np.array_equal(flags, (tag != synth.CAT_OUTSIDE).astype(np.uint8))


@pytest.mark.parametrize("lo,hi", [([0.25, -0.5], [0.75, 1.25]), ([0.5, 0.5], [0.5, 0.5]), ([-1, -1], [1, 1])])
def test_dense_other_windows(torch, cs, lo, hi):
    n = 100003
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(1, 9), n, np.float32)
    check_dense(torch, cs, planes, n, lo, hi, 2)
    check_compact(torch, cs, planes, n, lo, hi, 2)


def test_dense_nonfinite_inputs(torch, cs):
    n = 4096
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(1, 10), n, np.float32)
    rng = np.random.default_rng(0)
    for v in (np.nan, np.inf, -np.inf):
        idx = rng.integers(0, n, 50)
        planes[rng.integers(0, 4, 50), idx] = v
    check_dense(torch, cs, planes, n, *UNIT[2], 2)


def test_dense_in_place(torch, cs):
    n = 50001
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(1, 11), n, np.float32)
    want, wflags = oracle.clip(planes, n, *UNIT[2], 2)
    d = to_dev(torch, planes)
    out, flags = cs.clip(d, n, *UNIT[2], out=d)
    torch.cuda.synchronize()
    assert np.array_equal(bits(d.cpu().numpy()[:, :n]), bits(want[:, :n]))


@pytest.mark.parametrize("n", SIZES)
def test_compact_2d_f32_sizes(torch, cs, n):
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(5), n, np.float32)
    check_compact(torch, cs, planes, n, *UNIT[2], 2, index_base=12345)


@pytest.mark.parametrize("key", list(PACKED_TILES))
@pytest.mark.parametrize("m", [(1, -1), (1, 0), (1, 1), (2, 1), (3, -1), (7, 13)])
def test_compact_packed_tile_edges(torch, cs, key, m):
    dim, dtype = key
    n = m[0] * PACKED_TILES[key] + m[1]
    planes, _ = gen(synth.ADVERSARIAL if m[0] == 7 else synth.UNIFORM, dim, synth.seed_for(5, n), n, dtype)
    check_compact(torch, cs, planes, n, *UNIT[dim], dim, index_base=777)
    # the bench's instantiation: flags, no index
    want, _, wcnt, wflags = oracle.compact(planes, n, *UNIT[dim], dim, with_flags=True)
    b = cs.clip_compact(to_dev(torch, planes), n, *UNIT[dim], with_flags=True)
    torch.cuda.synchronize()
    assert int(b.count.item()) == wcnt
    assert np.array_equal(b.flags.cpu().numpy()[:n], wflags)
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :wcnt]), bits(want[:, :wcnt]))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("family", [synth.UNIFORM, synth.MIX, synth.ADVERSARIAL])
def test_compact_families(torch, cs, dim, dtype, family):
    n = 300007
    planes, _ = gen(family, dim, synth.seed_for(5, family), n, dtype)
    check_compact(torch, cs, planes, n, *UNIT[dim], dim)


def test_compact_all_and_none_visible(torch, cs):
    n = 70001
    pin, pc = synth.mix_thresholds(1.0 - 2**-32, 0.0)
    planes, _ = synth.fill_host(synth.MIX, 2, 3, n, p_in=pin, p_cross=pc)      # all inside
    check_compact(torch, cs, planes, n, *UNIT[2], 2)
    planes, _ = synth.fill_host(synth.MIX, 2, 3, n, p_in=0, p_cross=0)          # all outside
    check_compact(torch, cs, planes, n, *UNIT[2], 2)


def test_compact_zero_n(torch, cs):
    d = torch.zeros((4, 32), dtype=torch.float32, device="cuda")
    b = cs.clip_compact(d, 0, *UNIT[2])
    torch.cuda.synchronize()
    assert int(b.count.item()) == 0


def test_compact_repeat_reuses_workspace(torch, cs):
    n = 200003
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(5, 3), n, np.float32)
    d = to_dev(torch, planes)
    b = cs.clip_compact(d, n, *UNIT[2], with_index=True)
    first = b.out.clone()
    for _ in range(3):
        cs.clip_compact(d, n, *UNIT[2], bufs=b)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert torch.equal(first[:, :cnt], b.out[:, :cnt])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_host_pipeline(torch, cs, dtype):
    n = 1000003
    planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(5, 4), n, dtype)
    want, _, wcnt, wflags = oracle.compact(planes, n, *UNIT[2], 2, with_flags=True)
    h_in = torch.from_numpy(planes).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_flags = torch.empty(n, dtype=torch.uint8).pin_memory()
    cnt, staging = cs.clip_compact_host(h_in, n, *UNIT[2], h_out, h_flags=h_flags, chunk=300000)
    assert cnt == wcnt
    assert np.array_equal(h_flags.numpy(), wflags)
    assert np.array_equal(bits(h_out.numpy()[:, :cnt]), bits(want[:, :cnt]))
    # again on the same thread (the pipeline's streams and events are reused), a shorter input
    m = 77777
    want2, _, wcnt2, wflags2 = oracle.compact(planes[:, :synth.plane_stride(m)].copy(), m, *UNIT[2], 2,
                                              with_flags=True)
    h_out.zero_()
    cnt2, _ = cs.clip_compact_host(h_in[:, :synth.plane_stride(m)].contiguous(), m, *UNIT[2], h_out, h_flags=h_flags,
                                   chunk=30000, staging=None)
    assert cnt2 == wcnt2
    assert np.array_equal(h_flags.numpy()[:m], wflags2)
    assert np.array_equal(bits(h_out.numpy()[:, :cnt2]), bits(want2[:, :cnt2]))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("family", [synth.UNIFORM, synth.MIX, synth.ADVERSARIAL])
def test_generator_device_twin(torch, family, dtype):
    n = 200003
    pin, pc = synth.mix_thresholds(0.1, 0.8)
    host, htag = synth.fill_host(family, 3 if family != synth.ADVERSARIAL else 2, 99, n, dtype=dtype, i0=777,
                                 p_in=pin, p_cross=pc)
    d = torch.zeros(host.shape, dtype=torch.float32 if dtype == np.float32 else torch.float64, device="cuda")
    tag = torch.zeros(n, dtype=torch.uint8, device="cuda")
    synth.fill_device(d, family, host.shape[0] // 2, 99, n, i0=777, p_in=pin, p_cross=pc, tag_t=tag)
    torch.cuda.synchronize()
    assert np.array_equal(bits(d.cpu().numpy()[:, :n]), bits(host[:, :n]))
    assert np.array_equal(tag.cpu().numpy(), htag)


def test_shard_offsets_kernel(torch, cs):
    counts = torch.tensor([5, 0, 7, 11, 3], dtype=torch.int64, device="cuda")
    for r in range(5):
        off = cs.shard_offsets(counts, r)
        torch.cuda.synchronize()
        assert off.tolist() == [int(counts[:r].sum()), 26]


def test_sharded_compact_single_rank_nccl(torch, cs):
    """The sharded entry (CUDA compaction + NCCL allgather + offset kernel) at world size 1."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1110_5450_b200.shard import sharded_compact
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        n = 300007
        planes, _ = gen(synth.UNIFORM, 2, synth.seed_for(5), n, np.float32)
        want, widx, wcnt = oracle.compact(planes, n, *UNIT[2], 2, index_base=1000)
        res, b = sharded_compact(to_dev(torch, planes), n, *UNIT[2], 1000)
        torch.cuda.synchronize()
        assert res.offsets.tolist() == [0, wcnt] and res.counts.tolist() == [wcnt]
        assert np.array_equal(bits(b.out.cpu().numpy()[:, :wcnt]), bits(want[:, :wcnt]))
        assert np.array_equal(b.index.cpu().numpy()[:wcnt], widx)
    finally:
        dist.destroy_process_group()


def test_negative_zero_window_takes_the_exact_path(torch, cs):
    """A -0 window edge disables the fast path (clip_math.cuh): every group runs the rules
    select by select; results stay bit-identical (signed zeros included)."""
    n = 100003
    planes, _ = gen(synth.ADVERSARIAL, 2, synth.seed_for(3, 7), n, np.float32)
    lo, hi = [-0.0, 0.0], [1.0, 1.0]
    check_dense(torch, cs, planes, n, lo, hi, 2)
    check_compact(torch, cs, planes, n, lo, hi, 2)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_padded_strides(torch, cs, dtype):
    """Input and output planes with different, padded strides (ld > n, ld_in != ld_out; the ABI
    requires 16-byte aligned planes, checked in test_abi)."""
    n = 50007
    planes, _ = gen(synth.MIX, 3, synth.seed_for(2, 8), n, dtype)
    want, wflags = oracle.clip(planes, n, *UNIT[3], 3)
    wc, widx, wcnt, wcf = oracle.compact(planes, n, *UNIT[3], 3, with_flags=True)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    ld = synth.plane_stride(n)
    d_in = torch.zeros((6, ld + 96), dtype=tdt, device="cuda")
    d_in[:, :n] = torch.from_numpy(planes[:, :n]).cuda()
    out = torch.zeros((6, ld + 160), dtype=tdt, device="cuda")
    out, flags = cs.clip(d_in, n, *UNIT[3], out=out)
    b = cs.CompactBuffers(n, 3, tdt, with_flags=True, with_index=True)
    b.out = torch.zeros((6, ld + 224), dtype=tdt, device="cuda")
    cs.clip_compact(d_in, n, *UNIT[3], bufs=b)
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()[:, :n]), bits(want[:, :n]))
    assert int(b.count.item()) == wcnt
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :wcnt]), bits(wc[:, :wcnt]))
    assert np.array_equal(b.index.cpu().numpy()[:wcnt], widx)
