"""GPU parity of NEXT-1 (homogeneous clip space): the CUDA path through the C ABI vs the
CPU oracle (oracle/clip_homog_impl.h), element by element and bit for bit — flags,
homogeneous or NDC endpoints (NaN patterns, signed zeros), compaction order, indices and
counts — on the seeded HOMOG inputs, at sizes spanning several tiles and ragged tails."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

SIZES = [1, 3, 5, 31, 1023, 1025, 1920, 1921, 2049, 2944, 2945, 5888, 10007, 300007]  # incl. the fp32 compacting tile edges (1920; 2944 with NDC output)


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


def gen(n, seed, dtype):
    return synth.fill_host(synth.HOMOG, 4, synth.seed_for(6, seed), n, dtype=dtype)[0]


def check_dense(torch, cs, planes, n, ndc):
    want, wflags = oracle.homog_clip(planes, n, ndc=ndc, nthreads=8)
    out, flags = cs.clip_homog(torch.from_numpy(planes).cuda(), n, ndc=ndc)
    torch.cuda.synchronize()
    got, gflags = out.cpu().numpy(), flags.cpu().numpy()[:n]
    assert np.array_equal(gflags, wflags), np.nonzero(gflags != wflags)[0][:10]
    diff = np.nonzero(np.any(bits(got[:, :n]) != bits(want[:, :n]), axis=0))[0]
    assert len(diff) == 0, (diff[:5], planes[:, diff[:2]], got[:, diff[:2]], want[:, diff[:2]])
    return wflags


def check_compact(torch, cs, planes, n, ndc, index_base=0):
    want, widx, wcnt, wflags = oracle.homog_compact(planes, n, index_base=index_base, with_flags=True, ndc=ndc)
    b = cs.clip_homog_compact(torch.from_numpy(planes).cuda(), n, ndc=ndc, with_index=True, with_flags=True,
                              index_base=index_base)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert cnt == wcnt
    assert np.array_equal(b.flags.cpu().numpy()[:n], wflags)
    assert np.array_equal(b.index.cpu().numpy()[:cnt], widx)
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :cnt]), bits(want[:, :cnt]))


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("ndc", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_dense(torch, cs, n, ndc, dtype):
    check_dense(torch, cs, gen(n, 1, dtype), n, ndc)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("ndc", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_compact(torch, cs, n, ndc, dtype):
    check_compact(torch, cs, gen(n, 2, dtype), n, ndc, index_base=99)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_w1_matches_cuboid_kernel(torch, cs, dtype):
    """At w = 1 the homogeneous kernel and the 3D cuboid kernel ([-1,1]^3) agree bit for bit."""
    n = 200003
    planes = gen(n, 3, dtype)
    planes[3, :] = 1
    planes[7, :] = 1
    out, flags = cs.clip_homog(torch.from_numpy(planes).cuda(), n)
    cub = torch.from_numpy(np.ascontiguousarray(planes[[0, 1, 2, 4, 5, 6]])).cuda()
    cout, cflags = cs.clip(cub, n, [-1.0] * 3, [1.0] * 3)
    torch.cuda.synchronize()
    assert torch.equal(flags[:n], cflags[:n])
    o, c = out.cpu().numpy(), cout.cpu().numpy()
    assert np.array_equal(bits(o[[0, 1, 2, 4, 5, 6], :n]), bits(c[:, :n]))


def test_nonfinite_inputs(torch, cs):
    n = 4099
    planes = gen(n, 4, np.float32)
    rng = np.random.default_rng(1)
    for v in (np.nan, np.inf, -np.inf):
        planes[rng.integers(0, 8, 60), rng.integers(0, n, 60)] = v
    for ndc in (False, True):
        flags = check_dense(torch, cs, planes, n, ndc)
        check_compact(torch, cs, planes, n, ndc)
    assert flags.sum() > 0


def test_large_sampled(torch, cs):
    """10^7 fp32 segments, compacting with NDC, every element against the oracle."""
    n = 10**7
    planes = gen(n, 5, np.float32)
    check_compact(torch, cs, planes, n, True)


@pytest.mark.parametrize("ndc", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_on_plane_grazing(torch, cs, ndc, dtype):
    """P0 exactly on a clip plane (boundary coordinate +0: w0 = 1, x0 = -1 or +1) and P1 outside
    that plane by a boundary coordinate of subnormal or tiny magnitude: the exiting alpha is
    +0 / |b1|, the exact +0 — a fast path must not divide by a flushed subnormal.  Mixed into
    the seeded HOMOG rows so every warp holds some."""
    n = 20011
    planes = gen(n, 7, dtype)
    rng = np.random.default_rng(77)
    emin = 149 if dtype == np.float32 else 1074
    rows = np.nonzero(rng.random(n) < 0.2)[0]
    for i in rows:
        k = int(rng.integers(0, 3))
        s = dtype(rng.choice([-1.0, 1.0]))  # the plane x_k = s w
        planes[3, i] = dtype(1)
        planes[k, i] = s
        for c in range(3):
            if c != k:
                planes[c, i] = dtype(rng.uniform(-0.9, 0.9))
        if rng.random() < 0.7:  # subnormal boundary coordinate of P1: w1 = 2^-(emin-22), |x1| = w1 + 2^-e
            w1 = np.ldexp(dtype(1), -(emin - 22)).astype(dtype)
            t = np.ldexp(dtype(1), -int(rng.integers(emin - 20, emin + 1))).astype(dtype)
        else:  # tiny normal one
            w1 = np.ldexp(dtype(1), -80).astype(dtype)
            t = np.ldexp(dtype(1), -int(rng.integers(81, 100))).astype(dtype)
        planes[7, i] = w1
        planes[4 + k, i] = s * (w1 + t)  # boundary coordinate w1 - |x1| = -t exactly
        for c in range(3):
            if c != k:
                planes[4 + c, i] = dtype(rng.uniform(-0.4, 0.4))
    check_dense(torch, cs, planes, n, ndc)
    check_compact(torch, cs, planes, n, ndc)
