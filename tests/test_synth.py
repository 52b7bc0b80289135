"""The seeded input generator (CPU): determinism, shard invariance, value recipe."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("family", [synth.UNIFORM, synth.MIX, synth.ADVERSARIAL])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_shard_invariance(family, dtype):
    """Segment i depends only on (seed, i): any contiguous shard regenerates the same rows."""
    pin, pc = synth.mix_thresholds(1 / 3, 1 / 3)
    full, tf = synth.fill_host(family, 2, 77, 5000, dtype=dtype, p_in=pin, p_cross=pc, nthreads=4)
    part, tp = synth.fill_host(family, 2, 77, 1234, dtype=dtype, i0=3000, p_in=pin, p_cross=pc, nthreads=1)
    assert np.array_equal(full[:, 3000:4234].view(np.uint8), part[:, :1234].view(np.uint8))
    assert np.array_equal(tf[3000:4234], tp)


def test_uniform_grid_recipe():
    p, _ = synth.fill_host(synth.UNIFORM, 3, synth.seed_for(4), 200000)
    v = p[:, :200000].astype(np.float64)
    assert v.min() >= -1 and v.max() < 2
    g = v * 2**22
    assert np.array_equal(g, np.rint(g))              # on the 2^-22 grid
    assert abs(v.mean() - 0.5) < 0.01                  # uniform on [-1, 2)
    p64, _ = synth.fill_host(synth.UNIFORM, 2, 5, 1000, dtype=np.float64)
    assert np.array_equal(p64[:, :1000] * 2**50, np.rint(p64[:, :1000] * 2**50))


@pytest.mark.parametrize("dim", [2, 3])
def test_mix_categories(dim):
    n = 300000
    pin, pc = synth.mix_thresholds(0.10, 0.80)
    p, tag = synth.fill_host(synth.MIX, dim, 9, n, p_in=pin, p_cross=pc)
    frac = np.bincount(tag, minlength=3) / n
    assert np.allclose(frac, [0.10, 0.80, 0.10], atol=0.005)
    P = p[:, :n]
    inside = lambda e: np.all((P[e * dim:(e + 1) * dim] >= 0) & (P[e * dim:(e + 1) * dim] < 1), axis=0)  # noqa: E731
    i0, i1 = inside(0), inside(1)
    assert np.all(i0[tag == 0] & i1[tag == 0])
    assert np.all((i0 ^ i1)[tag == 1])                 # exactly one endpoint inside
    out = tag == 2
    beyond = np.zeros(n, bool)
    for k in range(dim):
        a, b = P[k], P[dim + k]
        beyond |= ((a < 0) & (b < 0)) | ((a > 1) & (b > 1))
    assert np.all(beyond[out])


def test_adversarial_families_present():
    p, tag = synth.fill_host(synth.ADVERSARIAL, 2, 3, 10000)
    fam = tag & 0x7F
    assert np.array_equal(fam, np.arange(10000) % 10)
    assert np.all((tag & synth.TAG_NEAR)[fam == 5] != 0)
    assert np.all((tag & synth.TAG_NEAR)[fam != 5] == 0)
    zl = fam == 0
    assert np.array_equal(p[0:2, :10000][:, zl], p[2:4, :10000][:, zl])  # zero-length
    bits = p[:, :10000][:, fam == 6].view(np.uint32)
    assert np.any(bits == 0x80000000) and np.any(bits == 1) and np.any(bits == 0x80000001)


def test_bad_arguments():
    with pytest.raises(ValueError):
        synth.fill_host(5, 2, 1, 10)
    with pytest.raises(ValueError):
        synth.fill_host(0, 4, 1, 10)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_homog_recipe(dtype):
    """NEXT-1 inputs (dim 4): shard invariance, exact grid values, every mode as built."""
    full, tf = synth.fill_host(synth.HOMOG, 4, 91, 60000, dtype=dtype, nthreads=4)
    part, tp = synth.fill_host(synth.HOMOG, 4, 91, 777, dtype=dtype, i0=5000, nthreads=1)
    assert np.array_equal(full[:, 5000:5777].view(np.uint8), part[:, :777].view(np.uint8))
    assert np.array_equal(tf[5000:5777], tp)
    n = 60000
    p = full[:, :n].astype(np.float64)
    frac = np.bincount(tf, minlength=5) / n
    assert abs(frac[0] - 0.6) < 0.02 and np.all(np.abs(frac[1:] - 0.1) < 0.01)
    pers = tf == synth.H_PERSPECTIVE
    for e in range(2):
        w = p[4 * e + 3, pers]
        assert w.min() >= 0.5 and w.max() < 2
        assert np.abs(p[4 * e:4 * e + 3, pers]).max() <= 3
    aff = tf == synth.H_AFFINE
    assert np.all(p[[3, 7]][:, aff] == 1)
    beh = tf == synth.H_BEHIND
    assert np.all((p[3, beh] < 0) ^ (p[7, beh] < 0))
    onp = tf == synth.H_ON_PLANE
    on_any = np.zeros(onp.sum(), bool)
    for e in range(2):
        on_any |= np.any(np.abs(p[4 * e:4 * e + 3, onp]) == p[4 * e + 3, onp], axis=0)
    assert on_any.all()
    scale = 2**21 if dtype == np.float32 else 2**49
    xyz = p[[0, 1, 2, 4, 5, 6]][:, pers] * scale
    assert np.array_equal(xyz, np.rint(xyz))                        # x, y, z on the grid (exact)
