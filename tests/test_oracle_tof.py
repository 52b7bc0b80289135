"""Pins of the NEXT-2 oracle (oracle/tof_oracle.py): range clip + phi (CPU only).

Expected values come from the paper's formulas and SPEC.md's worked values, not from the
oracle: phi(0, I) = 0, phi(1, 1) = pi/4, phi(2, 0.25) = pi/4; the
inverse-square invariance phi(d, rho/d^2) = arctan(sqrt(rho)) (PAPER.md P:557-565,
SPEC.md:143); monotonicity; the closed clip interval [r_min, r_max]
 at its exact boundaries; the paper's per-frame range formulas
 for the generated ranges."""
import math

import numpy as np
import pytest

import synth
from oracle import tof_oracle as T


def test_spec_values():
    assert T.phi(0.0, 5.0) == 0.0
    assert T.phi(1.0, 1.0) == math.pi / 4
    assert T.phi(2.0, 0.25) == math.pi / 4


def test_inverse_square_invariance():
    d = np.linspace(0.3, 7.5, 10001)
    for rho in (0.2, 0.5, 1.0, 3.0):
        v = T.phi(d, rho / d ** 2)
        assert np.max(np.abs(v - math.atan(math.sqrt(rho)))) < 1e-9


def test_monotone():
    d = np.linspace(0.3, 7.5, 5001)
    assert np.all(np.diff(T.phi(d, 0.7)) > 0)
    I = np.linspace(0.01, 10, 5001)
    assert np.all(np.diff(T.phi(1.3, I)) > 0)
    assert np.all((T.phi(d, 0.7) >= 0) & (T.phi(d, 0.7) < math.pi / 2))


def test_closed_interval_and_invalid():
    r0, r1 = np.float32(0.7), np.float32(1.1)
    below = np.nextafter(r0, np.float32(0))
    above = np.nextafter(r1, np.float32(np.inf))
    d = np.array([r0, r1, below, above, 0.9, 0.0, -1.0, np.nan, np.inf, 0.9, 0.9, 0.9], np.float32)
    I = np.array([1, 1, 1, 1, 1, 1, 1, 1, 1, -0.5, np.nan, np.inf], np.float32)
    code = T.range_code(d, I, r0, r1)
    assert list(code) == [0, 0, 1, 2, 0, 4, 4, 4, 4, 4, 4, 4]


def test_batched_frames_and_counts():
    ppf = 37  # ragged: frames do not align with vector widths
    rng = np.random.default_rng(3)
    F = 11
    d = rng.uniform(0.0, 3.0, F * ppf).astype(np.float32)
    I = rng.uniform(0.0, 2.0, F * ppf).astype(np.float32)
    d[::13] = 0
    ranges = np.stack([rng.uniform(0.2, 1.0, F), rng.uniform(1.0, 2.5, F)], 1).astype(np.float32)
    code, ph, kept = T.tof_range_phi(d, I, ppf, ranges)
    for f in range(F):
        s = slice(f * ppf, (f + 1) * ppf)
        want = (d[s] > 0) & (d[s] >= ranges[f, 0]) & (d[s] <= ranges[f, 1])
        assert np.array_equal(code[s] == 0, want)
        assert kept[f] == want.sum()
    k = code == 0
    assert np.all(np.isnan(ph[~k]))
    assert np.allclose(ph[k], np.arctan(d[k].astype(np.float64) * np.sqrt(I[k].astype(np.float64))), rtol=0,
                       atol=0)


def test_generator_ranges_follow_the_paper():
    """r_min = max(eps, min(d1, d2) - r_th), r_max = max(d1, d2) + r_th, r_th = 0.1 m."""
    d, I, r = synth.tof_host(17, 50)
    assert np.all(r[:, 0] >= np.float32(1e-3)) and np.all(r[:, 1] > r[:, 0])
    assert np.all(r[:, 1] - r[:, 0] >= np.float32(0.2) - np.float32(1e-6))
    n = d.shape[0]
    assert abs((d == 0).mean() - 0.02) < 0.003
    ok = d > 0
    rho = I[ok].astype(np.float64) * d[ok].astype(np.float64) ** 2
    assert rho.min() >= 0.2 - 1e-6 and rho.max() < 1.0 + 1e-6              # I = rho / d^2
    code, ph, kept = T.tof_range_phi(d, I, synth.TOF_PPF, r)
    assert 0.15 < (code == 0).mean() < 0.6 and kept.sum() == (code == 0).sum() and n == 50 * synth.TOF_PPF
