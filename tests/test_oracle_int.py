"""Pins of the NEXT-4 oracle (oracle/int_oracle.py): integer segments, exact rational
clipping, round-half-up endpoints.  CPU only.

Expected values never come from the oracle's own formula: hand-worked examples
(tests/golden/int_examples.json, each derived in its 'why'), a brute force that finds the
visible parameter interval by testing every candidate t = j / D (the interval's ends are
0, 1 or (c - p_k) / d_k, all multiples of 1 / (|d_x| |d_y|)), and invariants (containment,
identity for inside segments, exact snap onto the crossed edge, reversal symmetry of the
visible set, symmetry under reflection)."""
import json
import math
import os
import random
from fractions import Fraction

import numpy as np

from oracle import int_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def test_golden_examples():
    cases = json.load(open(os.path.join(HERE, "golden", "int_examples.json")))["cases"]
    assert len(cases) >= 10
    for c in cases:
        p, w = c["p"], c["win"]
        f, q0, q1 = O.clip_one(p[:2], p[2:], w[:2], w[2:])
        assert f == c["flag"], c["id"]
        if f == 1:
            assert [*q0, *q1] == c["q"], c["id"]


def _brute(p0, p1, lo, hi):
    d = (p1[0] - p0[0], p1[1] - p0[1])
    D = max(abs(d[0]), 1) * max(abs(d[1]), 1)
    inside = []
    for j in range(D + 1):
        t = Fraction(j, D)
        pt = (p0[0] + d[0] * t, p0[1] + d[1] * t)
        if all(lo[k] <= pt[k] <= hi[k] for k in range(2)):
            inside.append(t)
    if not inside:
        return 0, None, None
    rnd = lambda x: math.floor(x + Fraction(1, 2))  # noqa: E731  (I4, stated independently)
    q = lambda t: (p0[0] + rnd(d[0] * t), p0[1] + rnd(d[1] * t))  # noqa: E731
    return 1, q(min(inside)), q(max(inside))


def test_brute_force_tiny():
    rng = random.Random(11)
    for _ in range(4000):
        lo = [rng.randint(-4, 3), rng.randint(-4, 3)]
        hi = [lo[0] + rng.randint(0, 5), lo[1] + rng.randint(0, 5)]
        p0 = (rng.randint(-9, 9), rng.randint(-9, 9))
        p1 = (rng.randint(-9, 9), rng.randint(-9, 9))
        assert O.clip_one(p0, p1, lo, hi) == _brute(p0, p1, lo, hi), (p0, p1, lo, hi)


def test_invariants_large():
    rng = random.Random(5)
    B = 1 << 30
    for _ in range(3000):
        lo = [rng.randint(-B, B // 2), rng.randint(-B, B // 2)]
        hi = [rng.randint(lo[0], B), rng.randint(lo[1], B)]
        p0 = (rng.randint(-B, B), rng.randint(-B, B))
        p1 = (rng.randint(-B, B), rng.randint(-B, B))
        f, q0, q1 = O.clip_one(p0, p1, lo, hi)
        fr, r0, r1 = O.clip_one(p1, p0, lo, hi)
        assert f == fr  # the visible set does not depend on the direction
        fm, m0, m1 = O.clip_one((-p0[0], p0[1]), (-p1[0], p1[1]), [-hi[0], lo[1]], [-lo[0], hi[1]])
        assert fm == f  # reflection x -> -x maps the window onto itself
        if f != 1:
            continue
        for q in (q0, q1, r0, r1):
            assert all(lo[k] <= q[k] <= hi[k] for k in range(2))
        inside0 = all(lo[k] <= p0[k] <= hi[k] for k in range(2))
        inside1 = all(lo[k] <= p1[k] <= hi[k] for k in range(2))
        if inside0:
            assert q0 == p0
        else:  # P0 outside: Q0 lies exactly on an edge of the window
            assert q0[0] in (lo[0], hi[0]) or q0[1] in (lo[1], hi[1])
        if inside1:
            assert q1 == p1
        else:
            assert q1[0] in (lo[0], hi[0]) or q1[1] in (lo[1], hi[1])


def test_out_of_range_and_fill():
    B = 1 << 30
    assert O.clip_one((B, -B), (-B, B), [-B, -B], [B, B]) == (1, (B, -B), (-B, B))
    assert O.clip_one((B + 1, 0), (0, 0), [-1, -1], [1, 1])[0] == 2
    planes = np.array([[5, 0], [5, 0], [9, 1], [7, 1]], dtype=np.int32)
    out, flags = O.clip_segments_i32(planes, 2, [0, 0], [4, 4])
    assert flags.tolist() == [0, 1]
    assert (out[:, 0] == np.iinfo(np.int32).min).all() and out[:, 1].tolist() == [0, 0, 1, 1]
