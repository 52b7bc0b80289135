"""GPU parity of the packed kernel's deferred passes (clip_compact.cu phase 2, CLIPSEG_PK_DEFER;
clip_math.cuh box_fast_ok2): batches whose rounds meet a row outside the fast path's cheap
range test finish in passes A (finer test + fast path, in place), B (the rules, queued rows)
and C (compaction).  The rows here sit exactly where the finer test's reasoning is delicate:

  * on-edge:   an endpoint exactly on an edge line (a WEC of exactly +0);
  * grazing:   P0 on the low edge 0 and P1 outside it by 2^-e, e up to 149 (fp32: tiny and
               subnormal denominators behind a +0 numerator);
  * neg-zero:  a -0 coordinate against the +0 low edge (a WEC of -0: the clamp's hazard);
  * subnormal: coordinates of subnormal magnitude (WECs below kTiny);
  * collinear: both endpoints on one edge line;

mixed into uniform rows at two densities, so batches switch to the deferred passes at varied
list positions (and some never do).  Dense and compacting results are compared with the oracle
bit for bit (2D and 3D, fp32 and fp64).  Inputs are seeded (numpy PCG64)."""
from __future__ import annotations

import numpy as np
import pytest

from test_gpu_wide import check_both, planes_for

pytestmark = pytest.mark.gpu

N = 50021


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def special_rows(dim, dt, n, rate, seed):
    rng = np.random.default_rng(seed)
    P = planes_for(dim, dt, n)
    P[:, :n] = rng.uniform(-1.0, 2.0, size=(2 * dim, n)).astype(dt)
    kind = np.where(rng.random(n) < rate, rng.integers(0, 5, size=n), -1)
    axis = rng.integers(0, dim, size=n)
    emax = 149 if dt == np.float32 else 1074
    for i in np.nonzero(kind >= 0)[0]:
        k, a = kind[i], axis[i]
        if k == 0:  # on-edge: one endpoint coordinate exactly 0 or 1
            P[rng.integers(0, 2) * dim + a, i] = dt(rng.integers(0, 2))
        elif k == 1:  # grazing: P0 on the low edge, P1 just outside it
            P[a, i] = dt(0)
            P[dim + a, i] = -np.ldexp(dt(1), -int(rng.integers(20, emax + 1))).astype(dt)
        elif k == 2:  # neg-zero: a -0 coordinate (the low edge is +0)
            P[rng.integers(0, 2) * dim + a, i] = dt(-0.0)
            if rng.random() < 0.5:
                P[dim + a, i] = dt(rng.uniform(-1.0, -0.1))  # the other endpoint outside that edge
        elif k == 3:  # subnormal coordinates
            tiny = np.ldexp(dt(1), -int(rng.integers(emax - 20, emax + 1))).astype(dt)
            P[rng.integers(0, 2) * dim + a, i] = tiny * dt(rng.choice([-1, 1]))
        else:  # collinear with an edge line
            e = dt(rng.integers(0, 2))
            P[a, i] = e
            P[dim + a, i] = e
    return P


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("rate", [0.002, 0.3])
def test_deferred_passes(torch, cs, dt, dim, rate):
    P = special_rows(dim, dt, N, rate, 4000 + dim + int(rate * 1000))
    assert check_both(torch, cs, P, N, [0.0] * dim, [1.0] * dim, dim) > 0
