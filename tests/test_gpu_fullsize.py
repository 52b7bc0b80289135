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


@pytest.mark.parametrize("ndc", [False, True])
def test_homog_1e8_sampled(torch, cs, ndc):
    """NEXT-1 at bench.py's size: 10^8 fp32 HOMOG segments, compacting clip with flags and
    index; sampled flags and compacted rows bit-exact vs the oracle, count == sum of flags,
    indices strictly increasing."""
    n = 10**8
    seed = synth.seed_for(6)
    planes = torch.empty((8, cs.clip_plane_stride(n)), dtype=torch.float32, device="cuda")
    synth.fill_device(planes, synth.HOMOG, 4, seed, n)
    b = cs.clip_homog_compact(planes, n, ndc=ndc, with_flags=True, with_index=True)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    fl = b.flags[:n]
    assert cnt == int(fl.sum(dtype=torch.int64).item())
    oi = b.index[:cnt]
    assert bool((oi[1:] > oi[:-1]).all())
    rng = np.random.default_rng(11)
    idx = np.unique(np.concatenate([rng.integers(0, n, 3000), np.arange(8), np.arange(n - 8, n)]))
    P = np.zeros((8, synth.plane_stride(len(idx))), np.float32)
    for j, i in enumerate(idx):
        p, _ = synth.fill_host(synth.HOMOG, 4, seed, 1, i0=int(i), nthreads=1, with_tag=False)
        P[:, j] = p[:, 0]
    want, wfl = oracle.homog_clip(P, len(idx), ndc=ndc)
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(bits(planes[:, ti].cpu().numpy()), bits(P[:, :len(idx)]))
    assert np.array_equal(fl[ti].cpu().numpy(), wfl)
    vis = torch.from_numpy(np.nonzero(wfl)[0]).cuda()
    rows = torch.searchsorted(oi, ti[vis])
    assert torch.equal(oi[rows], ti[vis])
    assert np.array_equal(bits(b.out[:, rows].cpu().numpy()), bits(want[:, vis.cpu().numpy()]))
    del planes, b, fl, oi
    torch.cuda.empty_cache()


def test_tof_8192_frames_sampled(torch, cs):
    """NEXT-2 at bench.py's size: 8192 ToF frames of 204 x 204; sampled frames (first, a
    middle one, last) exact in codes and counts, phi within 1e-6 rad; every count in range."""
    from oracle import tof_oracle  # noqa: PLC0415
    nframes, ppf = 8192, synth.TOF_PPF
    n = nframes * ppf
    seed = synth.seed_for(7)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    I = torch.empty_like(d)
    r = torch.from_numpy(synth.tof_device(d, I, seed, nframes)).cuda()
    phi, code, kept = cs.tof_range_phi(d, I, ppf, r)
    torch.cuda.synchronize()
    assert int(kept.sum().item()) == int((code == 0).sum().item())
    for f in (0, 4097, nframes - 1):
        hd, hI, hr = synth.tof_host(seed, 1, f0=f)
        s = slice(f * ppf, (f + 1) * ppf)
        assert np.array_equal(bits(d[s].cpu().numpy()), bits(hd))
        wc, wp, wk = tof_oracle.tof_range_phi(hd, hI, ppf, hr)
        assert np.array_equal(code[s].cpu().numpy(), wc)
        assert int(kept[f]) == int(wk[0])
        k = wc == 0
        got = phi[s].cpu().numpy()
        assert np.abs(got[k].astype(np.float64) - wp[k]).max() <= 1e-6
        assert np.isnan(got[~k]).all()
    del d, I, phi, code
    torch.cuda.empty_cache()


def test_cluster_296_frames_sampled(torch, cs):
    """NEXT-3 at bench.py's size: a batch of 296 fused 204 x 204 frames in one call (the
    one-block-per-frame schedule); the first and last frames' labels and region counts
    identical to the oracle's; every frame's labels are region ids of valid pixels."""
    from oracle import cluster_oracle  # noqa: PLC0415
    from synth import scenes  # noqa: PLC0415
    z, ph, v, _ = scenes.batch(296, 204, 204, seed=14)
    dz, dph, dv = (torch.from_numpy(a).cuda() for a in (z, ph, v.astype(np.uint8)))
    lab, nreg, rounds, _ = cs.cluster_frames(dz, dph, dv)
    torch.cuda.synchronize()
    L = lab.cpu().numpy()
    assert np.array_equal(L == 0, ~v)
    for f in (0, 295):
        wl, wr, _, _ = cluster_oracle.cluster(z[f], ph[f], v[f])
        assert np.array_equal(L[f], wl)
        assert int(nreg[f]) == len(wr)
