"""Pins of the CPU oracle (oracle/) against things other than itself (CPU only).

Each test names what fixes the expected value: a hand-derived worked example
(tests/golden/worked_examples.json), exact rational geometry (tests/exact.py), an
exact int64 classifier, brute-force sampling, the textbook iterative Cohen–Sutherland
clipper, generator ground truth (categories built inside/outside by construction),
closed forms (reflection construction, corner grazes) or a bit-exact metamorphic
relation.  A plausible slip in the oracle (dropped term, wrong sign, wrong edge or
index, swapped operands, missing snap/clamp) fails at least one of them.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

import oracle
import synth
from exact import brute_force_visible, classic_cohen_sutherland, exact_clip, grid_visible

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")
TOL32 = 1e-6   # BASELINE.json north_star: fp32 endpoints within 1e-6 x window extent
TOL64 = 1e-14  # fp64 within 1e-14
UNIT2 = ([0.0, 0.0], [1.0, 1.0])
UNIT3 = ([0.0, 0.0, 0.0], [1.0, 1.0, 1.0])


def _num(s):
    return float.fromhex(s) if "p" in s or s.startswith(("0x", "-0x")) else float(s)


def _bits32(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def _bits_arr(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: c["id"])
def test_worked_example_f32(case):
    dim = case["dim"]
    lo, hi = (UNIT2 if dim == 2 else UNIT3)
    p = [_num(s) for s in case["p"]]
    q, vis, tr = oracle.clip_one(p, lo, hi, dim, np.float32)
    assert vis == case["visible"], case["why"]
    assert tr["c0"] == case["c0"] and tr["c1"] == case["c1"]
    if "t_in_bits" in case:
        assert _bits32(tr["t_in"]) == int(case["t_in_bits"], 16)
    if "t_out_bits" in case:
        assert _bits32(tr["t_out"]) == int(case["t_out_bits"], 16)
    if not vis:
        assert all(_bits32(v) == 0x7FC00000 for v in q)  # R8 canonical NaN
    if "q" in case:
        assert [_bits32(v) for v in q] == [_bits32(np.float32(_num(s))) for s in case["q"]]
    if "q_bits" in case:
        assert [_bits32(v) for v in q] == [int(s, 16) for s in case["q_bits"]]
    if "exact_visible" in case:  # W16: the fp32-ambiguous residue, reported against geometry
        assert (exact_clip(p[:dim], p[dim:], lo, hi) is not None) == case["exact_visible"]


@pytest.mark.parametrize("case", _golden()["f64"], ids=lambda c: c["id"])
def test_worked_example_f64(case):
    p = [_num(s) for s in case["p"]]
    q, vis, tr = oracle.clip_one(p, *UNIT2, 2, np.float64)
    assert vis == case["visible"]
    if "t_in_hex" in case:
        assert float(tr["t_in"]) == float.fromhex(case["t_in_hex"])
        assert float(tr["t_out"]) == float.fromhex(case["t_out_hex"])
    if "q" in case:
        assert [float(v) for v in q] == [_num(s) for s in case["q"]]
    if "q_hex" in case:
        assert [float(v) for v in q] == [float.fromhex(s) for s in case["q_hex"]]


# ---------------------------------------------------------------- exact geometry
def _check_against_exact(planes, n, dim, lo, hi, tol, dt):
    out, flags = oracle.clip(planes, n, lo, hi, dim)
    ambiguous = 0
    for i in range(n):
        p = [float(planes[c, i]) for c in range(2 * dim)]
        ex = exact_clip(p[:dim], p[dim:], lo, hi)
        if (ex is not None) != bool(flags[i]):
            # only the fp-ambiguous band may disagree: the exact parameter gap is tiny
            if ex is not None:
                gap = float(ex[3] - ex[2])
            else:
                gap = _exact_gap(p, dim, lo, hi)
            assert abs(gap) < 64 * np.finfo(dt).eps, (i, p, gap)
            ambiguous += 1
            continue
        if ex is None:
            assert np.all(np.isnan(out[:, i]))
            continue
        q = [float(out[c, i]) for c in range(2 * dim)]
        want = [float(v) for v in ex[0]] + [float(v) for v in ex[1]]
        err = max(abs(a - b) for a, b in zip(q, want))
        assert err <= tol * max(h - l for l, h in zip(lo, hi)), (i, p, q, want, err)
    return ambiguous


def _exact_gap(p, dim, lo, hi):
    from fractions import Fraction as F
    t_in, t_out = F(0), F(1)
    for k in range(dim):
        a, b = F(p[k]), F(p[dim + k])
        d = b - a
        if d == 0:
            continue
        ta, tb = (F(lo[k]) - a) / d, (F(hi[k]) - a) / d
        t_in = max(t_in, min(ta, tb))
        t_out = min(t_out, max(ta, tb))
    return float(t_out - t_in)


def test_exact_rational_2d_f32_uniform():
    n = 20000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1), n)
    amb = _check_against_exact(planes, n, 2, *UNIT2, TOL32, np.float32)
    assert amb <= 2


def test_exact_rational_2d_f32_mix():
    n = 6000
    for mix in [(0.10, 0.80), (1 / 3, 1 / 3), (0.90, 0.05)]:
        planes, _ = synth.fill_host(synth.MIX, 2, synth.seed_for(2), n, p_in=synth.mix_thresholds(*mix)[0],
                                    p_cross=synth.mix_thresholds(*mix)[1])
        assert _check_against_exact(planes, n, 2, *UNIT2, TOL32, np.float32) == 0


def test_exact_rational_3d_f32():
    n = 10000
    planes, _ = synth.fill_host(synth.UNIFORM, 3, synth.seed_for(4), n)
    assert _check_against_exact(planes, n, 3, *UNIT3, TOL32, np.float32) <= 2


def test_exact_rational_2d_f64():
    n = 8000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(3), n, dtype=np.float64)
    assert _check_against_exact(planes, n, 2, *UNIT2, TOL64, np.float64) == 0


def test_exact_rational_3d_f64():
    n = 4000
    planes, _ = synth.fill_host(synth.UNIFORM, 3, synth.seed_for(4, 1), n, dtype=np.float64)
    assert _check_against_exact(planes, n, 3, *UNIT3, TOL64, np.float64) == 0


def test_exact_rational_offset_window():
    """A window that is not the unit square (catches lo/hi or axis mix-ups)."""
    n = 8000
    lo, hi = [0.25, -0.5], [0.75, 1.25]
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 7), n)
    assert _check_against_exact(planes, n, 2, lo, hi, TOL32, np.float32) <= 2


def test_exact_grid_classifier_1e6():
    """Flags vs the exact int64 classifier on 10^6 C1 segments (grid 2^-22)."""
    n = 10**6
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 1), n)
    _, flags = oracle.clip(planes, n, *UNIT2, 2, nthreads=8)
    g = np.rint(planes[:, :n].astype(np.float64) * 2**22).astype(np.int64)
    vis, gap = grid_visible(g, [0, 0], [2**22, 2**22], 2)
    bad = np.nonzero(vis != flags.astype(bool))[0]
    assert len(bad) <= 5
    assert np.all(np.abs(gap[bad]) < 1e-6)
    # C1 shape: visible ~52.1 %
    assert abs(flags.mean() - 0.521) < 0.003


# ---------------------------------------------------------------- brute force
def test_brute_force_tiny():
    n = 400
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 2), n)
    _, flags = oracle.clip(planes, n, *UNIT2, 2)
    K = 1 << 14
    for i in range(n):
        p = planes[:, i].astype(np.float64)
        any_in, _ = brute_force_visible(p[:2], p[2:], [0, 0], [1, 1], K)
        if any_in:
            assert flags[i] == 1, (i, p)
        elif flags[i]:
            # visible but no sample inside: the visible part is shorter than 1/K
            ex = exact_clip(p[:2], p[2:], [0, 0], [1, 1])
            assert ex is None or float(ex[3] - ex[2]) < 2.0 / K


# ---------------------------------------------------------------- independent algorithm
def test_classic_cohen_sutherland():
    n = 20000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 3), n)
    out, flags = oracle.clip(planes, n, *UNIT2, 2)
    disagree = 0
    for i in range(n):
        p = planes[:, i].astype(np.float64)
        vis, q = classic_cohen_sutherland(p[:2], p[2:], (0.0, 0.0), (1.0, 1.0))
        if vis != bool(flags[i]):
            disagree += 1
            assert abs(_exact_gap(list(p), 2, [0, 0], [1, 1])) < 1e-6
            continue
        if vis:
            assert np.max(np.abs(np.array(q) - out[:, i].astype(np.float64))) <= TOL32
    assert disagree <= 2


# ---------------------------------------------------------------- invariants / ground truth
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_invariants_and_categories(dim, dtype):
    n = 200000
    lo, hi = UNIT2 if dim == 2 else UNIT3
    for mix in [(0.10, 0.80), (1 / 3, 1 / 3), (0.90, 0.05)]:
        pin, pc = synth.mix_thresholds(*mix)
        planes, tag = synth.fill_host(synth.MIX, dim, synth.seed_for(2), n, dtype=dtype, p_in=pin, p_cross=pc)
        out, flags = oracle.clip(planes, n, lo, hi, dim)
        P, Q = planes[:, :n], out[:, :n]
        # generator ground truth (exact by construction)
        assert np.all(flags[tag == synth.CAT_OUTSIDE] == 0)
        assert np.all(flags[tag != synth.CAT_OUTSIDE] == 1)
        ins = tag == synth.CAT_INSIDE
        assert np.array_equal(_bits_arr(Q[:, ins]), _bits_arr(P[:, ins]))  # unchanged, bit for bit
        _geom_invariants(P, Q, flags, dim, lo, hi, dtype)
    planes, _ = synth.fill_host(synth.UNIFORM, dim, synth.seed_for(1 if dim == 2 else 4), n, dtype=dtype)
    out, flags = oracle.clip(planes, n, lo, hi, dim)
    _geom_invariants(planes[:, :n], out[:, :n], flags, dim, lo, hi, dtype)
    # the adversarial families exercise the clamp (corner grazes, near-edge endpoints)
    planes, _ = synth.fill_host(synth.ADVERSARIAL, dim, synth.seed_for(3), n, dtype=dtype)
    out, flags = oracle.clip(planes, n, lo, hi, dim)
    _geom_invariants(planes[:, :n], out[:, :n], flags, dim, lo, hi, dtype, on_line=False)


def _geom_invariants(P, Q, flags, dim, lo, hi, dtype, on_line=True):
    vis = flags.astype(bool)
    tol = TOL32 if dtype == np.float32 else TOL64
    # invisible rows are canonical NaN (R8)
    nanbits = 0x7FC00000 if dtype == np.float32 else 0x7FF8000000000000
    assert np.all(_bits_arr(Q[:, ~vis]) == nanbits)
    Qv, Pv = Q[:, vis].astype(np.float64), P[:, vis].astype(np.float64)
    for e in range(2):
        for k in range(dim):
            assert np.all(Qv[e * dim + k] >= lo[k]) and np.all(Qv[e * dim + k] <= hi[k])
    # Q lies on the line P0P1 (distance within tolerance, relative to |P| for far inputs)
    d = Pv[dim:] - Pv[:dim]
    L = np.sqrt((d ** 2).sum(0))
    nz = L > 0
    for e in range(2):
        r = Qv[e * dim:(e + 1) * dim] - Pv[:dim]
        t = (r * d).sum(0) / np.where(nz, L ** 2, 1)
        perp = r - t * d
        dist = np.sqrt((perp ** 2).sum(0))
        if on_line:
            assert np.all(dist[nz] <= tol * 2)
    # every crossed endpoint sits exactly on an edge value of an axis it was outside on
    for e in range(2):
        pe = Pv[e * dim:(e + 1) * dim]
        qe = Qv[e * dim:(e + 1) * dim]
        crossed = np.zeros(pe.shape[1], bool)
        on_edge = np.zeros(pe.shape[1], bool)
        for k in range(dim):
            out_lo, out_hi = pe[k] < lo[k], pe[k] > hi[k]
            crossed |= out_lo | out_hi
            on_edge |= (out_lo & (qe[k] == lo[k])) | (out_hi & (qe[k] == hi[k]))
        assert np.all(on_edge[crossed])


# ---------------------------------------------------------------- metamorphic relations (bit-exact)
def test_idempotence():
    n = 100000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 4), n)
    out, flags = oracle.clip(planes, n, *UNIT2, 2)
    vis = np.nonzero(flags)[0]
    again = np.ascontiguousarray(out[:, vis])
    out2, flags2 = oracle.clip(again, len(vis), *UNIT2, 2)
    assert np.all(flags2 == 1)
    assert np.array_equal(_bits_arr(out2), _bits_arr(again))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("k", [-40, -20, -7, 5, 20, 40, 57])
def test_power_of_two_scaling(k, dim, dt):
    """Scaling inputs and window by 2^k scales every result by 2^k exactly: each rule is a
    correctly rounded operation, and RN(2^k x) = 2^k RN(x) while nothing under- or
    overflows (operands stay within [2^-62, 2^59] for fp32).  The range spans the GPU fast
    path's whole claimed operand range (tests/test_gpu_wide.py runs the same windows)."""
    n = 20000
    planes, _ = synth.fill_host(synth.UNIFORM, dim, synth.seed_for(1, 5), n, dtype=dt)
    lo, hi = [0.0] * dim, [1.0] * dim
    out, flags = oracle.clip(planes, n, lo, hi, dim)
    s = dt(2.0 ** k)
    out_s, flags_s = oracle.clip(planes * s, n, lo, [float(s)] * dim, dim)
    assert np.array_equal(flags, flags_s)
    v = flags.astype(bool)
    assert v.sum() > 0
    assert np.array_equal(_bits_arr(out_s[:, :n][:, v]), _bits_arr(out[:, :n][:, v] * s))
    # the symmetric window [-2^k, 2^k]^D against [-1, 1]^D
    sym = planes * dt(2) - dt(1)
    out1, fl1 = oracle.clip(sym, n, [-1.0] * dim, [1.0] * dim, dim)
    out2, fl2 = oracle.clip(sym * s, n, [float(-s)] * dim, [float(s)] * dim, dim)
    assert np.array_equal(fl1, fl2)
    v = fl1.astype(bool)
    assert np.array_equal(_bits_arr(out2[:, :n][:, v]), _bits_arr(out1[:, :n][:, v] * s))


def test_mirror_and_transpose():
    """On the window [-1,1]^2: x -> -x mirroring and x <-> y transposition are exact."""
    n = 100000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(1, 6), n)
    planes = planes * np.float32(2.0) - np.float32(1.0)   # [-3, 3), still exact
    lo, hi = [-1.0, -1.0], [1.0, 1.0]
    out, flags = oracle.clip(planes, n, lo, hi, 2)
    v = flags.astype(bool)
    mir = planes.copy(); mir[0] = -mir[0]; mir[2] = -mir[2]
    out_m, flags_m = oracle.clip(mir, n, lo, hi, 2)
    assert np.array_equal(flags, flags_m)
    exp = out.copy(); exp[0] = -exp[0]; exp[2] = -exp[2]
    assert np.array_equal(_bits_arr(out_m[:, :n][:, v]), _bits_arr(exp[:, :n][:, v]))
    tr = planes[[1, 0, 3, 2]].copy()
    out_t, flags_t = oracle.clip(tr, n, lo, hi, 2)
    assert np.array_equal(flags, flags_t)
    assert np.array_equal(_bits_arr(out_t[:, :n][:, v]), _bits_arr(out[[1, 0, 3, 2]][:, :n][:, v]))


# ---------------------------------------------------------------- adversarial closed forms
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_adversarial_closed_forms(dtype):
    n = 100000
    planes, tag = synth.fill_host(synth.ADVERSARIAL, 2, synth.seed_for(3), n, dtype=dtype)
    out, flags = oracle.clip(planes, n, *UNIT2, 2)
    fam = tag & 0x7F
    P, Q = planes[:, :n], out[:, :n]
    # F8 reflection: always visible and the crossed endpoint equals E = (P0+P1)/2 exactly
    r = fam == 7
    assert np.all(flags[r] == 1)
    E = (P[0:2, r] + P[2:4, r]) * dtype(0.5)
    p0_in = (P[0, r] >= 0) & (P[0, r] <= 1) & (P[1, r] >= 0) & (P[1, r] <= 1)
    got = np.where(p0_in, Q[2:4, r], Q[0:2, r])
    assert np.array_equal(got, E)
    # F5 corner grazes: visible, both endpoints clip to the corner C
    c = fam == 4
    assert np.all(flags[c] == 1)
    # the corner C: P0 = C + u*t, P1 = C - v*t with t = (+-1, +-1), u, v in [0,1)
    corner = np.stack([np.maximum(P[0, c], P[2, c]) > 1, np.maximum(P[1, c], P[3, c]) > 1])

    def _inside(x, y):
        return (x >= 0) & (x <= 1) & (y >= 0) & (y <= 1)
    both_out = ~_inside(P[0, c], P[1, c]) & ~_inside(P[2, c], P[3, c])
    # both alphas are RN(u / RN(u+v)), so t_in == t_out exactly (visible); the endpoints
    # snap on their deciding axis and land within tolerance of C on the other
    tol = TOL32 if dtype == np.float32 else TOL64
    C = corner[:, both_out].astype(np.float64)
    assert np.max(np.abs(Q[0:2, c][:, both_out] - C)) <= tol
    assert np.max(np.abs(Q[2:4, c][:, both_out] - C)) <= tol
    # every non-near case agrees with exact geometry on visibility
    idx = np.nonzero((tag & synth.TAG_NEAR) == 0)[0][:3000]
    for i in idx:
        p = [float(x) for x in P[:, i]]
        ex = exact_clip(p[:2], p[2:], [0, 0], [1, 1])
        if (ex is not None) != bool(flags[i]):
            assert abs(_exact_gap(p, 2, [0, 0], [1, 1])) < 1e-6


def test_nonfinite_inputs_invisible():
    nan, inf = float("nan"), float("inf")
    for p in [(nan, .5, .5, .5), (.5, .5, inf, .5), (-inf, .5, .5, .5), (.5, nan, .5, .5)]:
        q, vis, _ = oracle.clip_one(p, *UNIT2, 2)
        assert not vis and all(_bits32(v) == 0x7FC00000 for v in q)


def test_degenerate_window():
    """lo == hi: the window is a point; only segments through it are visible."""
    lo = hi = [0.5, 0.5]
    q, vis, _ = oracle.clip_one((0, 0, 1, 1), lo, hi, 2)
    assert vis and list(q) == [0.5, 0.5, 0.5, 0.5]
    q, vis, _ = oracle.clip_one((0, 0, 1, 0.9), lo, hi, 2)
    assert not vis


def test_compact_is_stable_filter():
    n = 50000
    planes, _ = synth.fill_host(synth.UNIFORM, 2, synth.seed_for(5), n)
    out, flags = oracle.clip(planes, n, *UNIT2, 2)
    cout, idx, cnt, cflags = oracle.compact(planes, n, *UNIT2, 2, index_base=1000, with_flags=True)
    vis = np.nonzero(flags)[0]
    assert cnt == len(vis) == int(flags.sum())
    assert np.array_equal(idx, vis + 1000)
    assert np.array_equal(cflags, flags)
    assert np.array_equal(_bits_arr(cout[:, :cnt]), _bits_arr(out[:, vis]))


def test_invalid_window_rejected():
    planes, _ = synth.fill_host(synth.UNIFORM, 2, 1, 10)
    with pytest.raises(AssertionError):
        oracle.clip(planes, 10, [1, 0], [0, 1], 2)  # lo > hi -> status -1
