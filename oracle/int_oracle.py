"""CPU oracle of NEXT-4: integer / pixel-coordinate segment clipping with
exact rational intersections (rules I1-I6).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg may import this module.  It shares no code with the CUDA path.

The paper defines no integer variant ("no paper pin"; BJ:5 only
mentions one), so the arithmetic is the float rule set's WEC formulation carried out in
exact rationals (``fractions.Fraction``): for each window edge the window-edge coordinate
WEC (\\wec / \\WEC) of both endpoints, trivial reject when both are
negative, and alpha = WEC(P0) / (WEC(P0) - WEC(P1)) for a straddled edge, entering edges
raising t_in and leaving edges lowering t_out (DESIGN.md §3 R4-R5).  The only inexact step
is the final conversion of each clipped endpoint to integers, which DESIGN.md §15 I4 fixes
as round-half-up: round(x) = floor(x + 1/2).

Pins (tests/test_oracle_int.py): brute force over every candidate parameter j / D on tiny
segments, hand-worked examples (tests/golden/int_examples.txt), invariants.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

COORD_MAX = 1 << 30  # I1: |coordinate| <= 2^30 (window and endpoints)
FILL = -(1 << 31)    # I5: INT32_MIN in every plane of an invisible / out-of-range row


def round_half_up(x: Fraction) -> int:
    """I4: floor(x + 1/2)."""
    return math.floor(x + Fraction(1, 2))


def clip_one(p0, p1, lo, hi):
    """Clip one segment P0P1 (2 ints each) against the closed window [lo, hi] (2 ints each).
    Returns (flag, q0, q1): flag 1 visible, 0 invisible, 2 a coordinate outside [-2^30, 2^30]
    (I1); q0 / q1 are the clipped integer endpoints (None unless flag == 1)."""
    if any(abs(int(v)) > COORD_MAX for v in (*p0, *p1)):
        return 2, None, None
    t_in, t_out = Fraction(0), Fraction(1)
    for k in range(2):
        # the two edges of axis k: x_k >= lo_k (WEC = x_k - lo_k) and x_k <= hi_k (WEC = hi_k - x_k)
        for w0, w1 in ((p0[k] - lo[k], p1[k] - lo[k]), (hi[k] - p0[k], hi[k] - p1[k])):
            if w0 < 0 and w1 < 0:
                return 0, None, None          # trivial reject for this edge
            if w0 < 0:                        # entering: P0 outside, P1 inside this half-plane
                t_in = max(t_in, Fraction(w0, w0 - w1))
            elif w1 < 0:                      # leaving
                t_out = min(t_out, Fraction(w0, w0 - w1))
    if t_in > t_out:
        return 0, None, None
    d = (p1[0] - p0[0], p1[1] - p0[1])
    q0 = tuple(int(p0[k]) + round_half_up(d[k] * t_in) for k in range(2))
    q1 = tuple(int(p0[k]) + round_half_up(d[k] * t_out) for k in range(2))
    return 1, q0, q1


def clip_segments_i32(planes, n, lo, hi, idx=None):
    """planes: int array (4, ld) x0, y0, x1, y1.  Returns (out int32 (4, n), flags uint8 (n,)),
    invisible rows filled with INT32_MIN (I5).  idx: optional subset of row indices (the
    returned arrays then follow idx's order)."""
    rows = range(n) if idx is None else [int(i) for i in idx]
    m = len(rows)
    out = np.full((4, m), FILL, dtype=np.int32)
    flags = np.zeros(m, dtype=np.uint8)
    P = np.asarray(planes, dtype=np.int64)
    for j, i in enumerate(rows):
        f, q0, q1 = clip_one((int(P[0, i]), int(P[1, i])), (int(P[2, i]), int(P[3, i])), lo, hi)
        flags[j] = f
        if f == 1:
            out[:, j] = (q0[0], q0[1], q1[0], q1[1])
    return out, flags
