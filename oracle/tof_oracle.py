"""NEXT-2 oracle: the paper's own per-pixel step — range clip + fused measure phi.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/: only tests/, smoke() and
bench.py's baseline legs may use it).  Plain numpy, fp64 for the arithmetic.

PAPER.md §5.2: "pixels outside the range [r_min, r_max] will be ignored for
clustering" — a closed interval, recomputed per frame.  PAPER.md §4.2, Eq. (5)
(P:565): phi = arctan(d sqrt(I)), from the inverse-square law I ~ 1/d^2.
DESIGN.md §13 states the readings:
  * code (uint8) per pixel: 4 if the pixel is invalid (d <= 0, the SPEC's dropout sentinel
    d = 0, or d / I non-finite, or I < 0), else bit 0 = [d < r_min], bit 1 = [d > r_max]
    (binary32 comparisons of the inputs, as given);
  * phi = arctan(d sqrt(I)) for kept pixels (code 0), NaN otherwise;
  * kept[f] = number of kept pixels of frame f (pixel i belongs to frame i // ppf).
"""
from __future__ import annotations

import numpy as np


def phi(d, I):
    """Eq. (5): arctan(d sqrt(I)) in fp64."""
    return np.arctan(np.asarray(d, np.float64) * np.sqrt(np.asarray(I, np.float64)))


def range_code(d, I, r_min, r_max):
    """The per-pixel 2-bit range outcode (+ the invalid code 4), decided in binary32."""
    d = np.asarray(d, np.float32)
    I = np.asarray(I, np.float32)
    r_min = np.asarray(r_min, np.float32)
    r_max = np.asarray(r_max, np.float32)
    invalid = ~(d > 0) | ~np.isfinite(d) | ~(I >= 0) | ~np.isfinite(I)
    below = d < r_min
    above = d > r_max
    code = below.astype(np.uint8) | (above.astype(np.uint8) << 1)
    return np.where(invalid, np.uint8(4), code).astype(np.uint8)


def tof_range_phi(d, I, ppf, ranges):
    """Batched frames: d, I float32[n] (n = F * ppf, or a ragged last frame), ranges
    float32[F, 2] = (r_min, r_max) per frame.  Returns (code uint8[n], phi float64[n],
    kept int64[F])."""
    d = np.asarray(d, np.float32)
    I = np.asarray(I, np.float32)
    n = d.shape[0]
    f = np.arange(n, dtype=np.int64) // ppf
    ranges = np.asarray(ranges, np.float32)
    code = range_code(d, I, ranges[f, 0], ranges[f, 1])
    keep = code == 0
    with np.errstate(invalid="ignore"):
        ph = np.where(keep, phi(d, np.where(keep, I, 0)), np.nan)
    kept = np.bincount(f[keep], minlength=ranges.shape[0]).astype(np.int64)
    return code, ph, kept
