"""Pins of the NEXT-1 oracle (homogeneous clip space, oracle/clip_homog_impl.h) against
things other than itself (CPU only):

* hand-derived worked examples (tests/golden/homog_examples.json);
* its reduction, bit for bit, to the (separately pinned) 3D cuboid oracle at w = 1 with the
  window [-1, 1]^3 (SURVEY.md §8(f) NEXT-1 pin);
* exact rational geometry (tests/exact.py exact_homog_clip): visibility exact up to the
  fp-ambiguous band, endpoints within tolerance;
* an independent algorithm: for w > 0 the divided (NDC) result equals the exact 3D clip
  of the projected segment against [-1, 1]^3 (tests/exact.py exact_clip);
* bit-exact metamorphic relations: scaling both endpoints by 2^k scales the homogeneous
  result by 2^k and leaves NDC and flags unchanged;
* invariants: visible results lie in the closed volume, crossed endpoints lie on a plane.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

import oracle
import synth
from exact import exact_clip, exact_homog_clip

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "homog_examples.json")
CUBE = ([-1.0, -1.0, -1.0], [1.0, 1.0, 1.0])


def _b32(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _gen(n, seed=11, dtype=np.float32):
    return synth.fill_host(synth.HOMOG, 4, synth.seed_for(6, seed), n, dtype=dtype)


@pytest.mark.parametrize("case", json.load(open(GOLDEN))["cases"], ids=lambda c: c["id"])
def test_worked_example(case):
    p = [float(s) for s in case["p"]]
    q, vis, tr = oracle.homog_one(p, np.float32)
    assert vis == case["visible"], case["why"]
    assert tr["c0"] == case["c0"] and tr["c1"] == case["c1"]
    if "t_in_bits" in case:
        assert _b32(tr["t_in"]) == int(case["t_in_bits"], 16)
        assert _b32(tr["t_out"]) == int(case["t_out_bits"], 16)
    if not vis:
        assert all(_b32(v) == 0x7FC00000 for v in q)
    if "q" in case:
        assert [_b32(v) for v in q] == [_b32(float(s)) for s in case["q"]]
    if "q_bits" in case:
        assert [_b32(v) for v in q] == [int(s, 16) for s in case["q_bits"]]
    if "ndc" in case or "ndc_bits" in case:
        planes = np.asarray(p, np.float32).reshape(8, 1).repeat(32, axis=1)
        out, flags = oracle.homog_clip(planes, 1, ndc=True)
        got = [_b32(v) for v in out[:, 0]]
        want = [int(s, 16) for s in case["ndc_bits"]] if "ndc_bits" in case else [_b32(float(s)) for s in case["ndc"]]
        assert got == want


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_reduces_to_cuboid_at_w1(dtype):
    """w0 = w1 = 1: every rule is the cuboid rule with lo = -1, hi = 1 (bit for bit)."""
    n = 60000
    planes, _ = _gen(n, 1, dtype)
    planes[3, :] = 1
    planes[7, :] = 1
    out, flags = oracle.homog_clip(planes, n)
    ndc, nflags = oracle.homog_clip(planes, n, ndc=True)
    cub = np.ascontiguousarray(planes[[0, 1, 2, 4, 5, 6]])
    want, wflags = oracle.clip(cub, n, *CUBE, 3)
    assert np.array_equal(flags, wflags) and np.array_equal(nflags, wflags)
    assert np.array_equal(_bits(out[[0, 1, 2, 4, 5, 6], :n]), _bits(want[:, :n]))
    vis = wflags.astype(bool)
    assert np.all(out[[3, 7]][:, vis] == 1)
    assert np.array_equal(_bits(ndc[:, :n]), _bits(want[:, :n]))  # q / 1 = q, NaN stays canonical
    assert 0.05 < vis.mean() < 0.95


@pytest.mark.parametrize("dtype,tol", [(np.float32, 4e-6), (np.float64, 1e-14)])
def test_exact_rational(dtype, tol):
    n = 8000
    planes, tag = _gen(n, 2, dtype)
    out, flags = oracle.homog_clip(planes, n)
    eps = np.finfo(dtype).eps
    amb = 0
    for i in range(n):
        p = [float(v) for v in planes[:, i]]
        ex = exact_homog_clip(p[:4], p[4:])
        if (ex is not None) != bool(flags[i]):
            amb += 1
            continue
        if ex is None:
            assert np.all(np.isnan(out[:, i]))
            continue
        want = [float(v) for v in ex[0]] + [float(v) for v in ex[1]]
        err = max(abs(float(a) - b) for a, b in zip(out[:, i], want))
        assert err <= tol * 4, (i, p, list(out[:, i]), want)  # coordinates are O(4)
    assert amb <= 2, amb
    assert 0.1 < flags.mean() < 0.9


@pytest.mark.parametrize("dtype,tol", [(np.float32, 2e-5), (np.float64, 1e-13)])
def test_ndc_equals_clip_of_projection(dtype, tol):
    """Independent algorithm: project (w > 0) then clip in 3D, exactly."""
    n = 6000
    planes, tag = _gen(n, 3, dtype)
    keep = (planes[3, :n] > 0) & (planes[7, :n] > 0)
    ndc, flags = oracle.homog_clip(planes, n, ndc=True)
    checked = amb = 0
    for i in np.nonzero(keep)[0]:
        p = [float(v) for v in planes[:, i]]
        from fractions import Fraction as F
        a = [F(p[k]) / F(p[3]) for k in range(3)]
        b = [F(p[4 + k]) / F(p[7]) for k in range(3)]
        ex = exact_clip(a, b, *CUBE)
        if (ex is not None) != bool(flags[i]):
            amb += 1
            continue
        checked += 1
        if ex is None:
            continue
        want = [float(v) for v in ex[0]] + [float(v) for v in ex[1]]
        err = max(abs(float(x) - y) for x, y in zip(ndc[:, i], want))
        assert err <= tol, (i, p, list(ndc[:, i]), want)
    assert amb <= 2 and checked > 0.8 * keep.sum()


@pytest.mark.parametrize("k", [-3, 5])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_scaling_metamorphic(k, dtype):
    n = 40000
    planes, _ = _gen(n, 4, dtype)
    s = dtype(2.0 ** k)
    out, flags = oracle.homog_clip(planes, n)
    out2, flags2 = oracle.homog_clip(planes * s, n)
    assert np.array_equal(flags, flags2)
    assert np.array_equal(_bits(out2[:, :n]), _bits(out[:, :n] * s))
    ndc, _ = oracle.homog_clip(planes, n, ndc=True)
    ndc2, _ = oracle.homog_clip(planes * s, n, ndc=True)
    assert np.array_equal(_bits(ndc[:, :n]), _bits(ndc2[:, :n]))


def test_invariants_and_modes():
    n = 50000
    planes, tag = _gen(n, 5)
    out, flags = oracle.homog_clip(planes, n)
    vis = flags.astype(bool)
    for e in range(2):
        q = out[4 * e:4 * e + 4, :n][:, vis].astype(np.float64)
        qw = q[3]
        ok = qw >= 0
        assert np.all(np.abs(q[:3][:, ok]) <= qw[ok])                   # inside the closed volume
        p = planes[4 * e:4 * e + 4, :n][:, vis]
        crossed = ~np.all(p == out[4 * e:4 * e + 4, :n][:, vis], axis=0)
        on_plane = np.any(np.abs(q[:3]) == np.abs(qw), axis=0)
        assert np.all(on_plane[crossed])                                 # a crossed endpoint is on a plane
    # every mode of the generator occurs and behaves as built
    assert set(np.unique(tag)) == {0, 1, 2, 3, 4}
    zero_len = (tag == synth.H_DEGENERATE) & np.all(planes[:4, :n] == planes[4:, :n], axis=0)
    inside0 = np.all(np.abs(planes[:3, :n]) <= planes[3, :n], axis=0)
    assert np.array_equal(vis[zero_len], inside0[zero_len])             # a point: visible iff inside
    both_behind = (planes[3, :n] < 0) & (planes[7, :n] < 0)
    assert not vis[both_behind].any()


def test_compact_matches_dense():
    n = 30011
    planes, _ = _gen(n, 6)
    for ndc in (False, True):
        out, flags = oracle.homog_clip(planes, n, ndc=ndc)
        cout, idx, cnt, cflags = oracle.homog_compact(planes, n, index_base=7, with_flags=True, ndc=ndc)
        assert np.array_equal(cflags, flags) and cnt == int(flags.sum())
        assert np.array_equal(idx, np.nonzero(flags)[0] + 7)
        assert np.array_equal(_bits(cout[:, :cnt]), _bits(out[:, np.nonzero(flags)[0]]))
