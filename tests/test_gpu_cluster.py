"""GPU parity of NEXT-3 (mutual-best region merging) through the C ABI vs
the plain-Python oracle (oracle/cluster_oracle.py): label maps (surviving ids), region counts
and round counts identical, on batched frames of seeded scenes and the SPEC examples."""
import numpy as np
import pytest

from oracle import cluster_oracle as C
from synth import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t  # noqa: PLC0415
    assert t.cuda.is_available()
    return t


@pytest.fixture(scope="module")
def cs():
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def run(torch, cs, z, ph, v, params=None):
    lab, nreg, rounds, _ = cs.cluster_frames(torch.from_numpy(np.ascontiguousarray(z)).cuda(),
                                             torch.from_numpy(np.ascontiguousarray(ph)).cuda(),
                                             torch.from_numpy(np.ascontiguousarray(v).astype(np.uint8)).cuda(),
                                             params)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), nreg.cpu().numpy(), int(rounds.item())


def check(torch, cs, z, ph, v, params=None):
    lab, nreg, rounds = run(torch, cs, z, ph, v, params)
    want_rounds = 0
    for f in range(z.shape[0]):
        wl, wr, wrounds, _ = C.cluster(z[f], ph[f], v[f], params)
        assert np.array_equal(lab[f], wl), (f, np.argwhere(lab[f] != wl)[:5])
        assert nreg[f] == len(wr)
        want_rounds = max(want_rounds, wrounds)
    assert rounds == want_rounds
    return lab


def test_chain_example(torch, cs):
    z = np.zeros((1, 1, 4), np.float32)
    ph = np.array([[[10, 30, 55, 95]]], np.float32)
    lab = check(torch, cs, z, ph, np.ones((1, 1, 4), bool), dict(t_z=1.0, t_phi=40.0, alpha_z=0.0, alpha_phi=1.0))
    assert lab.tolist() == [[[3, 3, 3, 4]]]


def test_uniform_checkerboard_and_plates(torch, cs):
    H = W = 16
    v = np.ones((3, H, W), bool)
    z = np.ones((3, H, W), np.float32)
    ph = np.full((3, H, W), 0.5, np.float32)
    ph[1] += 0.02 * ((np.arange(H)[:, None] + np.arange(W)[None, :]) % 2)
    z[2, :, W // 2:] = 1.5
    lab = check(torch, cs, z, ph, v)
    assert len(np.unique(lab[0])) == 1 and len(np.unique(lab[1])) == H * W and len(np.unique(lab[2])) == 2


@pytest.mark.parametrize("shape", [(1, 24, 32), (4, 40, 48), (2, 33, 17)])
def test_scenes(torch, cs, shape):
    F, H, W = shape
    z, ph, v, gt = scenes.batch(F, H, W, seed=H * W + F)
    check(torch, cs, z, ph, v)


def test_invalid_heavy(torch, cs):
    z, ph, v, gt = scenes.batch(2, 32, 32, seed=5, invalid=0.4)
    check(torch, cs, z, ph, v)


def test_all_invalid_and_tiny(torch, cs):
    z = np.ones((2, 3, 3), np.float32)
    v = np.zeros((2, 3, 3), bool)
    v[1, 1, 1] = True
    lab, nreg, rounds = run(torch, cs, z, z, v)
    assert lab[0].sum() == 0 and nreg.tolist() == [0, 1] and lab[1, 1, 1] == 5 and rounds == 1


def test_full_size_frames(torch, cs):
    """Two 204 x 204 frames (the paper's sensor): ~1000 rounds each, labels identical."""
    z, ph, v, gt = scenes.batch(2, 204, 204, seed=11)
    lab = check(torch, cs, z, ph, v)
    assert 2 <= len(np.unique(lab[0])) <= 50


@pytest.mark.parametrize("nframes,h,w", [(63, 12, 14), (67, 12, 14), (593, 8, 9)])
def test_batch_schedules(torch, cs, nframes, h, w):
    """Both schedules (grid-wide rounds below 64 frames, one block per frame from 64) and
    batches split into several launches (more than 592 frames): per-frame labels and counts
    identical to the oracle, rounds = the maximum over all frames."""
    z, ph, v, gt = scenes.batch(nframes, h, w, seed=21 + nframes)
    check(torch, cs, z, ph, v)
