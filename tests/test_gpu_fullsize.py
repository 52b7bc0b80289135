"""Full-size parity at BASELINE.json's sizes, in bench.py's launch configuration:
sampled outputs recomputed one by one by the oracle, plus properties that hold at any
size (count == sum of flags, compacted rows in input order)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def sample_oracle(family, dim, seed, idx, dtype, p_in=0, p_cross=0, lo=None, hi=None):
    """Regenerate the sampled segments on the host and clip them with the oracle."""
    m = len(idx)
    P = np.zeros((2 * dim, synth.plane_stride(m)), dtype=dtype)
    for j, i in enumerate(idx):
        p, _ = synth.fill_host(family, dim, seed, 1, dtype=dtype, i0=int(i), p_in=p_in, p_cross=p_cross,
                               nthreads=1, with_tag=False)
        P[:, j] = p[:, 0]
    out, flags = oracle.clip(P, m, lo, hi, dim)
    return P, out, flags


@pytest.mark.parametrize("mix", [None, (0.10, 0.80), (1 / 3, 1 / 3), (0.90, 0.05)])
def test_dense_1e8_sampled(torch, cs, mix):
    n, dim = 10**8, 2
    fam = synth.UNIFORM if mix is None else synth.MIX
    pin, pc = synth.mix_thresholds(*mix) if mix else (0, 0)
    seed = synth.seed_for(2)
    planes = cs.empty_planes(n, dim, torch.float32)
    synth.fill_device(planes, fam, dim, seed, n, p_in=pin, p_cross=pc)
    out, flags = cs.clip(planes, n, [0, 0], [1, 1])
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([rng.integers(0, n, 4000), np.arange(8), np.arange(n - 8, n)]))
    P, want, wflags = sample_oracle(fam, dim, seed, idx, np.float32, pin, pc, [0, 0], [1, 1])
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(bits(planes[:, ti].cpu().numpy()), bits(P[:, :len(idx)]))
    assert np.array_equal(flags[ti].cpu().numpy(), wflags)
    assert np.array_equal(bits(out[:, ti].cpu().numpy()), bits(want[:, :len(idx)]))
    del planes, out, flags
    torch.cuda.empty_cache()


def test_compact_1e9_sampled(torch, cs):
    """The bench workload: 10^9 2D fp32 C1-uniform segments, compacting clip with flags."""
    n, dim = 10**9, 2
    seed = synth.seed_for(5)
    planes = cs.empty_planes(n, dim, torch.float32)
    synth.fill_device(planes, synth.UNIFORM, dim, seed, n)
    b = cs.clip_compact(planes, n, [0, 0], [1, 1], with_flags=True)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    fl = b.flags[:n]
    assert cnt == int(fl.sum(dtype=torch.int64).item())
    assert abs(cnt / n - 0.521) < 0.001
    pos = torch.cumsum(fl, 0, dtype=torch.int32) - 1            # compacted row of each visible segment
    rng = np.random.default_rng(2)
    idx = np.unique(np.concatenate([rng.integers(0, n, 3000), np.arange(8), np.arange(n - 8, n)]))
    P, want, wflags = sample_oracle(synth.UNIFORM, dim, seed, idx, np.float32, lo=[0, 0], hi=[1, 1])
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(fl[ti].cpu().numpy(), wflags)
    vis = np.nonzero(wflags)[0]
    rows = pos[ti[torch.from_numpy(vis).cuda()]].long()
    got = b.out[:, rows].cpu().numpy()
    assert np.array_equal(bits(got), bits(want[:, vis]))
    del planes, b, pos, fl
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_adversarial_1e7(torch, cs, dtype):
    """configs[2]: 10^7 adversarial cases, full element-by-element comparison."""
    n, dim = 10**7, 2
    dt = np.float32 if dtype == "f32" else np.float64
    planes, tag = synth.fill_host(synth.ADVERSARIAL, dim, synth.seed_for(3), n, dtype=dt)
    want, wflags = oracle.clip(planes, n, [0, 0], [1, 1], dim, nthreads=8)
    d = torch.from_numpy(planes).cuda()
    out, flags = cs.clip(d, n, [0, 0], [1, 1])
    torch.cuda.synchronize()
    assert np.array_equal(flags.cpu().numpy()[:n], wflags)
    assert np.array_equal(bits(out.cpu().numpy()[:, :n]), bits(want[:, :n]))


def test_3d_1e8_sampled(torch, cs):
    """configs[3]: 10^8 3D fp32 segments against the unit cube."""
    n, dim = 10**8, 3
    seed = synth.seed_for(4)
    planes = cs.empty_planes(n, dim, torch.float32)
    synth.fill_device(planes, synth.UNIFORM, dim, seed, n)
    b = cs.clip_compact(planes, n, [0, 0, 0], [1, 1, 1], with_flags=True, with_index=True)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert abs(cnt / n - 0.3274) < 0.002
    rng = np.random.default_rng(3)
    idx = np.unique(rng.integers(0, n, 3000))
    P, want, wflags = sample_oracle(synth.UNIFORM, dim, seed, idx, np.float32, lo=[0, 0, 0], hi=[1, 1, 1])
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(b.flags[ti].cpu().numpy(), wflags)
    # out_index is sorted, so the compacted row of segment i is found by binary search
    oi = b.index[:cnt]
    vis = np.nonzero(wflags)[0]
    rows = torch.searchsorted(oi, ti[torch.from_numpy(vis).cuda()])
    assert torch.equal(oi[rows], ti[torch.from_numpy(vis).cuda()])
    assert np.array_equal(bits(b.out[:, rows].cpu().numpy()), bits(want[:, vis]))
