"""Independent exact references used to PIN the oracle (never to produce expected values
for the CUDA path).  None of this imports or re-types the oracle's arithmetic:

* ``exact_clip`` — parametric (Liang–Barsky) clipping in exact rational arithmetic
  (``fractions.Fraction``): the geometric truth for the closed window.
* ``grid_visible`` — the same parametric test vectorised over int64 numerators for
  inputs on a dyadic grid (exact cross-multiplied fraction comparisons).
* ``brute_force_visible`` — dense sampling P(k/K) of the segment, exact on grid inputs.
* ``classic_cohen_sutherland`` — the textbook iterative Cohen–Sutherland clipper
  (edge order T, B, R, L), float64, an independent algorithm at tolerance.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def exact_clip(p0, p1, lo, hi):
    """Exact clip of P0P1 against the closed box [lo, hi].  Inputs are floats (converted
    exactly) or Fractions.  Returns (Q0, Q1, t_in, t_out) as Fractions, or None if the
    segment misses the box."""
    P0 = [Fraction(x) for x in p0]
    P1 = [Fraction(x) for x in p1]
    LO = [Fraction(x) for x in lo]
    HI = [Fraction(x) for x in hi]
    t_in, t_out = Fraction(0), Fraction(1)
    for k in range(len(P0)):
        d = P1[k] - P0[k]
        if d == 0:
            if P0[k] < LO[k] or P0[k] > HI[k]:
                return None
            continue
        ta = (LO[k] - P0[k]) / d
        tb = (HI[k] - P0[k]) / d
        enter, leave = (ta, tb) if d > 0 else (tb, ta)
        t_in = max(t_in, enter)
        t_out = min(t_out, leave)
    if t_in > t_out:
        return None
    Q0 = [P0[k] + t_in * (P1[k] - P0[k]) for k in range(len(P0))]
    Q1 = [P0[k] + t_out * (P1[k] - P0[k]) for k in range(len(P0))]
    return Q0, Q1, t_in, t_out


def grid_visible(g, lo, hi, dim):
    """Exact visibility for integer (grid-unit) coordinates.
    g: int64 array (2*dim, n); lo, hi: ints per axis (window in grid units).
    Returns (visible bool[n], gap) where gap = t_out - t_in as float64 (for ambiguity bands)."""
    n = g.shape[1]
    # current t_in = a_num/a_den, t_out = b_num/b_den with positive denominators
    a_num = np.zeros(n, np.int64); a_den = np.ones(n, np.int64)
    b_num = np.ones(n, np.int64); b_den = np.ones(n, np.int64)
    dead = np.zeros(n, bool)
    for k in range(dim):
        p0 = g[k].astype(np.int64); p1 = g[dim + k].astype(np.int64)
        d = p1 - p0
        zero = d == 0
        dead |= zero & ((p0 < lo[k]) | (p0 > hi[k]))
        sgn = np.where(d < 0, -1, 1)
        den = np.where(zero, 1, np.abs(d))
        n_lo = (lo[k] - p0) * sgn
        n_hi = (hi[k] - p0) * sgn
        en = np.where(d > 0, n_lo, n_hi)   # entering numerator
        le = np.where(d > 0, n_hi, n_lo)   # leaving numerator
        # t_in = max(t_in, en/den) where d != 0
        upd = (~zero) & (en * a_den > a_num * den)
        a_num = np.where(upd, en, a_num); a_den = np.where(upd, den, a_den)
        upd = (~zero) & (le * b_den < b_num * den)
        b_num = np.where(upd, le, b_num); b_den = np.where(upd, den, b_den)
    vis = (~dead) & (a_num * b_den <= b_num * a_den)
    gap = b_num / b_den - a_num / a_den
    return vis, gap


def brute_force_visible(p0, p1, lo, hi, K=1 << 16):
    """Some sample P(k/K), k = 0..K, inside the closed box?  Exact for dyadic inputs whose
    products with k/K fit in float64 (2^-22 grid coordinates in [-2, 2])."""
    p0 = np.asarray(p0, np.float64); p1 = np.asarray(p1, np.float64)
    t = np.arange(K + 1, dtype=np.float64) / K
    pts = p0[None, :] + t[:, None] * (p1 - p0)[None, :]
    inside = np.all((pts >= np.asarray(lo)[None, :]) & (pts <= np.asarray(hi)[None, :]), axis=1)
    return bool(inside.any()), inside


def classic_cohen_sutherland(p0, p1, lo, hi):
    """Textbook iterative Cohen–Sutherland in float64 (2D), edges tested T, B, R, L.
    Returns (visible, (x0, y0, x1, y1))."""
    INSIDE, LEFT, RIGHT, BOTTOM, TOP = 0, 1, 2, 4, 8
    xmin, ymin = lo
    xmax, ymax = hi

    def code(x, y):
        c = INSIDE
        if x < xmin:
            c |= LEFT
        elif x > xmax:
            c |= RIGHT
        if y < ymin:
            c |= BOTTOM
        elif y > ymax:
            c |= TOP
        return c

    x0, y0 = float(p0[0]), float(p0[1])
    x1, y1 = float(p1[0]), float(p1[1])
    c0, c1 = code(x0, y0), code(x1, y1)
    for _ in range(8):
        if not (c0 | c1):
            return True, (x0, y0, x1, y1)
        if c0 & c1:
            return False, None
        c = c0 if c0 else c1
        if c & TOP:
            x = x0 + (x1 - x0) * (ymax - y0) / (y1 - y0); y = ymax
        elif c & BOTTOM:
            x = x0 + (x1 - x0) * (ymin - y0) / (y1 - y0); y = ymin
        elif c & RIGHT:
            y = y0 + (y1 - y0) * (xmax - x0) / (x1 - x0); x = xmax
        else:
            y = y0 + (y1 - y0) * (xmin - x0) / (x1 - x0); x = xmin
        if c == c0:
            x0, y0 = x, y; c0 = code(x0, y0)
        else:
            x1, y1 = x, y; c1 = code(x1, y1)
    return False, None


def exact_homog_clip(p0, p1):
    """Exact clip of the homogeneous segment P0P1 (x, y, z, w) against the closed volume
    -w <= x, y, z <= w (Blinn & Newell), by the parametric (Liang–Barsky) method in exact
    rationals: each plane's boundary coordinate B(t) = B0 + t (B1 - B0) must stay >= 0.
    Returns (Q0, Q1, t_in, t_out) as Fractions (4 components each), or None."""
    P0 = [Fraction(x) for x in p0]
    P1 = [Fraction(x) for x in p1]
    t_in, t_out = Fraction(0), Fraction(1)
    for k in range(3):
        for s in (1, -1):  # w + x_k >= 0 and w - x_k >= 0
            b0 = P0[3] + s * P0[k]
            b1 = P1[3] + s * P1[k]
            if b0 < 0 and b1 < 0:
                return None
            if b0 < 0 <= b1:
                t_in = max(t_in, b0 / (b0 - b1))
            elif b1 < 0 <= b0:
                t_out = min(t_out, b0 / (b0 - b1))
    if t_in > t_out:
        return None
    Q0 = [P0[c] + t_in * (P1[c] - P0[c]) for c in range(4)]
    Q1 = [P0[c] + t_out * (P1[c] - P0[c]) for c in range(4)]
    return Q0, Q1, t_in, t_out
