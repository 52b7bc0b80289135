"""Pins of the NEXT-3 oracle (oracle/cluster_oracle.py): round-synchronous mutual-best
merging (§4.1, Eqs. (1)-(3)), against SPEC.md's worked examples and the
properties the paper's procedure guarantees (CPU only)."""
import math
from collections import deque

import numpy as np
import pytest

from oracle import cluster_oracle as C
from synth import scenes

P = C.TABLE1


def test_chain_example():
    """phi-like values (10, 30, 55, 95), z equal, t = 40: round 1 merges {1,2} -> id 2
    (value 20), 3 and 4 wait; round 2 merges {2,3} -> id 3 ((10+30+55)/3); then no merge."""
    z = np.zeros((1, 4), np.float32)
    ph = np.array([[10, 30, 55, 95]], np.float32)
    p = dict(t_z=1.0, t_phi=40.0, alpha_z=0.0, alpha_phi=1.0)
    regions, nbrs = C.init_regions(z, ph, np.ones((1, 4), bool))
    pp = dict(P, **p)
    assert C.merge_round(regions, nbrs, pp) == 1
    assert sorted(regions) == [2, 3, 4] and C.mean(regions[2])[1] == 20
    assert C.merge_round(regions, nbrs, pp) == 1
    assert sorted(regions) == [3, 4] and C.mean(regions[3])[1] == (10 + 30 + 55) / 3
    assert C.merge_round(regions, nbrs, pp) == 0
    lab, reg, rounds, per = C.cluster(z, ph, np.ones((1, 4), bool), p)
    assert lab.tolist() == [[3, 3, 3, 4]] and rounds == 3 and per == [1, 1, 0]


def test_init_examples():
    """S:187-189."""
    r, n = C.init_regions(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32), np.ones((2, 2), bool))
    assert len(r) == 4 and sum(len(v) for v in n.values()) // 2 == 4
    v = np.ones((2, 2), bool)
    v[1, 1] = False
    r, n = C.init_regions(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32), v)
    assert len(r) == 3 and sum(len(s) for s in n.values()) // 2 == 2
    r, n = C.init_regions(np.ones((1, 1), np.float32), np.ones((1, 1), np.float32), np.ones((1, 1), bool))
    assert len(r) == 1 and n[1] == set()


def test_criterion_examples():
    """Eq. (1) and Eq. (2) with Table 1 parameters."""
    assert C.allowed((1.00, 0.800), (1.03, 0.805), P)
    assert not C.allowed((1.00, 0.800), (1.05, 0.805), P)
    assert C.allowed((1.0, 0.8), (1.0, 0.8), P)
    assert C.dist((1.0, 0.8), (1.0, 0.8), P) == 0
    assert abs(C.dist((1.0, 0.8), (1.04, 0.8), P) - 0.10186) < 1e-5
    assert C.dist((1.0, 0.8), (1.04, 0.7), P) == C.dist((1.04, 0.7), (1.0, 0.8), P)


def test_best_neighbor_examples():
    """argmin, ties to the larger id, none if nothing passes Eq. (1)."""
    p = dict(P, t_z=10.0, t_phi=10.0, alpha_z=1.0, alpha_phi=0.0)
    regions = {1: [1, 0.0, 0.0], 2: [1, 0.3, 0.0], 3: [1, 0.1, 0.0], 4: [1, 0.2, 0.0]}
    nbrs = {1: {2, 3, 4}, 2: {1}, 3: {1}, 4: {1}}
    means = {r: C.mean(v) for r, v in regions.items()}
    assert C.best_neighbor(1, regions, nbrs, means, p) == 3
    regions = {1: [1, 0.0, 0.0], 7: [1, 0.1, 0.0], 9: [1, 0.1, 0.0]}
    nbrs = {1: {7, 9}, 7: {1}, 9: {1}}
    means = {r: C.mean(v) for r, v in regions.items()}
    assert C.best_neighbor(1, regions, nbrs, means, p) == 9
    p2 = dict(p, t_z=0.01)
    assert C.best_neighbor(1, regions, nbrs, means, p2) is None


def test_cluster_examples():
    """uniform frame -> 1 region; two plates 0.5 m apart -> 2; checkerboard of
    two phi values |dphi| > t_phi -> no merge."""
    H = W = 12
    v = np.ones((H, W), bool)
    lab, reg, _, _ = C.cluster(np.full((H, W), 1.0, np.float32), np.full((H, W), 0.5, np.float32), v)
    assert len(reg) == 1 and np.all(lab == lab[0, 0])
    z = np.where(np.arange(W)[None, :] < 6, 1.0, 1.5).repeat(H, 0).astype(np.float32)
    lab, reg, _, _ = C.cluster(z, np.full((H, W), 0.5, np.float32), v)
    assert len(reg) == 2 and len(set(lab[:, :6].ravel())) == 1 and len(set(lab[:, 6:].ravel())) == 1
    cb = ((np.arange(H)[:, None] + np.arange(W)[None, :]) % 2).astype(np.float32)
    lab, reg, rounds, per = C.cluster(np.ones((H, W), np.float32), 0.5 + 0.02 * cb, v)
    assert len(reg) == H * W and per == [0]


def _regions_of(lab):
    return {int(r) for r in np.unique(lab) if r != 0}


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_properties_on_scenes(seed):
    """Convergence post-condition: no 4-adjacent pair of distinct regions satisfies
    Eq. (1); conservation; every region 4-connected; ids are the max pixel id
    of their region (the larger id survives every merge); objects separated by more than
    t_z never share a region."""
    H, W = 40, 48
    z, ph, v, gt = scenes.scene(H, W, seed)
    lab, reg, rounds, per = C.cluster(z, ph, v)
    assert per[-1] == 0 and all(k > 0 for k in per[:-1])
    assert np.all((lab == 0) == ~v) and _regions_of(lab) == set(reg)
    means = {r: C.mean(x) for r, x in reg.items()}
    for dy, dx in ((0, 1), (1, 0)):
        a = lab[: H - dy, : W - dx]
        b = lab[dy:, dx:]
        m = (a != 0) & (b != 0) & (a != b)
        for r, s in zip(a[m], b[m]):
            assert not C.allowed(means[int(r)], means[int(s)], P)
    assert sum(x[0] for x in reg.values()) == v.sum()
    zs = sum(x[1] for x in reg.values())
    assert math.isclose(zs, float(z[v].astype(np.float64).sum()), rel_tol=1e-12)
    for r in reg:
        pix = np.argwhere(lab == r)
        assert r == int((pix[:, 0] * W + pix[:, 1]).max()) + 1
        seen = {tuple(pix[0])}
        q = deque([tuple(pix[0])])
        members = {tuple(x) for x in pix}
        while q:
            y, x = q.popleft()
            for yy, xx in ((y - 1, x), (y + 1, x), (y, x - 1), (y, x + 1)):
                if (yy, xx) in members and (yy, xx) not in seen:
                    seen.add((yy, xx))
                    q.append((yy, xx))
        assert len(seen) == len(members)
    # plates (0.5-1.5 m) never merge with the wall (2.5-3.5 m): every region is one depth layer
    for r in reg:
        zz = z[lab == r]
        assert zz.max() - zz.min() < 1.0


def test_waiting_region_and_closed_threshold():
    """Rule 3 (Fig. 3 caption "have to wait"): values (0, 10, 12), t = 40: best(1) = 2
    but best(2) = 3, so only {2, 3} merges in round 1 (id 3, value 11) and region 1 waits;
    round 2 merges {1, 3} (value 22/3).  Eq. (1) is the closed |dw| <= t: a
    difference of exactly t merges, one just above it does not."""
    p = dict(t_z=1.0, t_phi=40.0, alpha_z=0.0, alpha_phi=1.0)
    pp = dict(P, **p)
    regions, nbrs = C.init_regions(np.zeros((1, 3), np.float32), np.array([[0, 10, 12]], np.float32),
                                   np.ones((1, 3), bool))
    assert C.merge_round(regions, nbrs, pp) == 1
    assert sorted(regions) == [1, 3] and C.mean(regions[3])[1] == 11 and C.mean(regions[1])[1] == 0
    assert C.merge_round(regions, nbrs, pp) == 1 and sorted(regions) == [3]
    assert C.mean(regions[3])[1] == 22 / 3
    z = np.zeros((1, 2), np.float32)
    lab, reg, _, _ = C.cluster(z, np.array([[0, 40]], np.float32), np.ones((1, 2), bool), p)
    assert len(reg) == 1
    lab, reg, _, _ = C.cluster(z, np.array([[0, np.nextafter(np.float32(40), np.float32(50))]], np.float32),
                               np.ones((1, 2), bool), p)
    assert len(reg) == 2
    pz = dict(t_z=1.0, t_phi=1.0, alpha_z=1.0, alpha_phi=0.0)     # the same on the z component
    lab, reg, _, _ = C.cluster(np.array([[0, 1]], np.float32), np.zeros((1, 2), np.float32), np.ones((1, 2), bool),
                               pz)
    assert len(reg) == 1


@pytest.mark.parametrize("seed", [4, 5])
def test_round_is_the_mutual_best_matching(seed):
    """Every round, checked from a snapshot of the frozen state with an independent argmin
    (sorted by (distance, -id)): the merged pairs are exactly the mutual best choices, each
    region is in at most one pair, and the survivor is the larger id with summed count/sums."""
    import copy
    z, ph, v, _ = scenes.scene(24, 24, seed)
    regions, nbrs = C.init_regions(z, ph, v)
    for _ in range(60):
        before_r, before_n = copy.deepcopy(regions), copy.deepcopy(nbrs)
        means = {r: (x[1] / x[0], x[2] / x[0]) for r, x in before_r.items()}
        choice = {}
        for r, ns in before_n.items():
            ok = [s for s in ns if abs(means[r][0] - means[s][0]) <= P["t_z"]
                  and abs(means[r][1] - means[s][1]) <= P["t_phi"]]
            key = lambda s, r=r: (P["alpha_z"] * abs(means[r][0] - means[s][0])  # noqa: E731
                                  + P["alpha_phi"] * abs(means[r][1] - means[s][1]), -s)
            choice[r] = sorted(ok, key=key)[0] if ok else None
        want = {(min(r, s), max(r, s)) for r, s in choice.items() if s is not None and choice[s] == r}
        k = C.merge_round(regions, nbrs, P)
        assert k == len(want)
        assert set(before_r) - set(regions) == {a for a, b in want}
        for a, b in want:
            assert regions[b] == [before_r[a][0] + before_r[b][0], before_r[a][1] + before_r[b][1],
                                  before_r[a][2] + before_r[b][2]]
        if k == 0:
            break
