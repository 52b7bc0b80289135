"""GPU parity across the fast path's whole claimed operand range (clip_math.cuh file comment):
the fast path divides with MUFU.RCP + Newton + residual correction and clamps with FMNMX,
claimed bit-identical to the rules for every group with |p| <= 2^58 and |WEC(P0)| >= 2^-60
(fp32; 2^500 / 2^-500 fp64).  These families put the operands across that range and across
its borders, so groups straddle the fast/exact range test, and compare the dense and the
compacting kernels (2D, 3D, fp32, fp64) with the oracle bit for bit:

  * scaled:    the standard workload scaled by 2^k (exact), windows [0, 2^k]^D and
               [-2^k, 2^k]^D, k in {-40, -20, 20, 40, 57} (fp32; fp64 adds +-300, 497);
  * near-edge: P0 at +-2^-e from a zero window edge, e spanning 2^-35 .. 2^-75 (fp32) /
               2^-480 .. 2^-520 (fp64), so some WECs sit below kTiny and some just above;
  * huge:      one coordinate of +-2^e, e spanning 2^50 .. 2^64 (fp32) / 2^490 .. 2^510
               (fp64), across kBig, with the rest of the segment crossing the window.

Inputs are seeded (numpy PCG64); every value is exactly representable in the dtype."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

N = 40009  # several compacting tiles and a ragged end


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


def check_both(torch, cs, planes, n, lo, hi, dim):
    d_in = torch.from_numpy(np.ascontiguousarray(planes)).cuda()
    want, wflags = oracle.clip(planes, n, lo, hi, dim, nthreads=8)
    out, flags = cs.clip(d_in, n, lo, hi)
    torch.cuda.synchronize()
    assert np.array_equal(flags.cpu().numpy()[:n], wflags)
    got = out.cpu().numpy()
    diff = np.nonzero(np.any(bits(got[:, :n]) != bits(want[:, :n]), axis=0))[0]
    assert len(diff) == 0, (diff[:5], planes[:, diff[:3]], got[:, diff[:3]], want[:, diff[:3]])
    cw, cidx, ccnt, cflags = oracle.compact(planes, n, lo, hi, dim, with_flags=True)
    b = cs.clip_compact(d_in, n, lo, hi, with_index=True, with_flags=True)
    torch.cuda.synchronize()
    cnt = int(b.count.item())
    assert cnt == ccnt
    assert np.array_equal(b.flags.cpu().numpy()[:n], cflags)
    assert np.array_equal(b.index.cpu().numpy()[:cnt], cidx)
    assert np.array_equal(bits(b.out.cpu().numpy()[:, :cnt]), bits(cw[:, :cnt]))
    return int(wflags.sum())


def planes_for(dim, dt, n):
    ld = synth.plane_stride(n)
    return np.zeros((2 * dim, ld), dtype=dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("sym", [False, True])
def test_scaled_windows(torch, cs, dt, dim, sym):
    ks = [-40, -20, 20, 40, 57] + ([-300, 300, 497] if dt == np.float64 else [])
    base, _ = synth.fill_host(synth.UNIFORM, dim, synth.seed_for(2, 91), N, dtype=dt)
    if sym:
        base = base * dt(2) - dt(1)  # [-3, 3) on the same grid: window [-1, 1]^D
    for k in ks:
        s = dt(2.0 ** k)
        lo = [float(-s) if sym else 0.0] * dim
        hi = [float(s)] * dim
        assert check_both(torch, cs, base * s, N, lo, hi, dim) > 0


def near_edge(dim, dt, n, seed):
    rng = np.random.default_rng(seed)
    P = planes_for(dim, dt, n)
    P[:, :n] = rng.uniform(-1.0, 2.0, size=(2 * dim, n)).astype(dt)
    lo_e, hi_e = (35, 75) if dt == np.float32 else (480, 520)
    e = rng.integers(lo_e, hi_e + 1, size=n)
    sign = rng.choice([-1.0, 1.0], size=n)
    off = (sign * np.ldexp(1.0, -e)).astype(dt)
    axis = rng.integers(0, dim, size=n)
    for k in range(dim):  # P0 just inside / outside the zero edge of one axis
        m = axis == k
        P[k, :n][m] = off[m]
    exact = rng.random(n) < 0.02  # a few P0 exactly on the edge
    P[0, :n][exact] = dt(0)
    return P


def huge(dim, dt, n, seed):
    rng = np.random.default_rng(seed)
    P = planes_for(dim, dt, n)
    P[:, :n] = rng.uniform(-1.0, 2.0, size=(2 * dim, n)).astype(dt)
    lo_e, hi_e = (50, 64) if dt == np.float32 else (490, 510)
    e = rng.integers(lo_e, hi_e + 1, size=n)
    sign = rng.choice([-1.0, 1.0], size=n)
    big = (sign * np.ldexp(1.0, e)).astype(dt)
    plane = rng.integers(0, 2 * dim, size=n)  # any coordinate of either endpoint
    for c in range(2 * dim):
        m = (plane == c) & (rng.random(n) < 0.5)
        P[c, :n][m] = big[m]
    return P


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("dim", [2, 3])
def test_near_edge_wecs(torch, cs, dt, dim):
    P = near_edge(dim, dt, N, 1000 + dim)
    assert check_both(torch, cs, P, N, [0.0] * dim, [1.0] * dim, dim) > 0


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("dim", [2, 3])
def test_huge_coordinates(torch, cs, dt, dim):
    P = huge(dim, dt, N, 2000 + dim)
    assert check_both(torch, cs, P, N, [0.0] * dim, [1.0] * dim, dim) > 0


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_huge_window_edges(torch, cs, dt):
    """Window edges at +-2^57 (fp32, inside the fast bound) and +-2^60 (outside: the host
    disables the fast path for the whole call)."""
    P = huge(2, dt, N, 3000)
    for e in (57, 60) if dt == np.float32 else (499, 502):
        s = float(2.0 ** e)
        assert check_both(torch, cs, P, N, [-s, -s], [s, s], 2) > 0
