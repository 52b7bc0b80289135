"""NEXT-3 oracle: the paper's GPU hot path — round-synchronous mutual-best merging of the
4-neighbourhood region graph of a frame (§4.1; merge criterion §4.2,
Eqs. (1)-(3)).

TEST INFRASTRUCTURE ONLY (only tests/, smoke() and bench.py's baseline legs may use it).
Plain Python following SPEC.md's cluster_oracle: every decision of a round is a
function of the frozen state at the start of the round.  DESIGN.md §14 states the readings:

  * regions: one per valid pixel, id = row-major pixel index + 1; descriptor
    w = (z, phi) (Eq. 3) held as fp64 SUMS over the region's pixels of the binary32 inputs,
    mean = sum / count (fp64) — the merged descriptor is the pixel-count-weighted mean
    (S:202);
  * Eq. (1) allowed(R, S) iff |z_R - z_S| <= t_z and |phi_R - phi_S| <= t_phi;
  * Eq. (2) f(R, S) = alpha_z |z_R - z_S| + alpha_phi |phi_R - phi_S| (fp64, two products then
    one sum, no fused operation);
  * best(R) = the allowed neighbour minimising f, ties to the larger id (§4.1 rule 2), none if
    no neighbour is allowed;
  * R and S merge iff best(R) = S and best(S) = R (rule 3); the merged region keeps the
    larger id, count and sums added, neighbour sets united minus self;
  * rounds repeat until a round merges nothing (convergence).
"""
from __future__ import annotations

import numpy as np

TABLE1 = dict(t_z=0.04, t_phi=0.009, alpha_z=8 / np.pi, alpha_phi=4 / 3)  # PAPER Table 1 via S:102


def init_regions(z, phi, valid):
    """One region per valid pixel of an H x W frame.  Returns (regions, nbrs):
    regions[id] = [count, sum_z, sum_phi]; nbrs[id] = set of 4-adjacent valid pixel ids."""
    H, W = valid.shape
    regions, nbrs = {}, {}
    for y in range(H):
        for x in range(W):
            if not valid[y, x]:
                continue
            rid = y * W + x + 1
            regions[rid] = [1, float(np.float32(z[y, x])), float(np.float32(phi[y, x]))]
            s = set()
            for yy, xx in ((y - 1, x), (y + 1, x), (y, x - 1), (y, x + 1)):
                if 0 <= yy < H and 0 <= xx < W and valid[yy, xx]:
                    s.add(yy * W + xx + 1)
            nbrs[rid] = s
    return regions, nbrs


def mean(reg):
    c, sz, sp = reg
    return sz / c, sp / c


def allowed(mr, ms, p):
    return abs(mr[0] - ms[0]) <= p["t_z"] and abs(mr[1] - ms[1]) <= p["t_phi"]


def dist(mr, ms, p):
    return p["alpha_z"] * abs(mr[0] - ms[0]) + p["alpha_phi"] * abs(mr[1] - ms[1])


def best_neighbor(rid, regions, nbrs, means, p):
    best, bd = None, None
    for s in nbrs[rid]:
        if not allowed(means[rid], means[s], p):
            continue
        d = dist(means[rid], means[s], p)
        if best is None or d < bd or (d == bd and s > best):
            best, bd = s, d
    return best


def merge_round(regions, nbrs, p, members=None):
    """One round from the frozen state; returns the number of merged pairs.
    `members` (optional) maps each surviving id to its original pixel ids."""
    means = {r: mean(v) for r, v in regions.items()}
    best = {r: best_neighbor(r, regions, nbrs, means, p) for r in regions}
    pairs = [(r, s) for r, s in best.items() if s is not None and r < s and best.get(s) == r]
    for r, s in pairs:                                  # r is absorbed into s, the larger id
        cr, zr, pr = regions[r]
        cs, zs, ps = regions[s]
        regions[s] = [cs + cr, zs + zr, ps + pr]
        del regions[r]
        if members is not None:
            members[s].extend(members.pop(r))
        ns = (nbrs[s] | nbrs.pop(r)) - {r, s}
        nbrs[s] = ns
        for t in ns:                                    # t's neighbour r becomes s
            if r in nbrs[t]:
                nbrs[t].discard(r)
                nbrs[t].add(s)
    return len(pairs)


def cluster(z, phi, valid, p=None, max_rounds=None):
    """Rounds until a round merges nothing.  Returns (labels int32[H, W] — the
    surviving id of each pixel's region, 0 = invalid —, regions {id: [count, sum_z, sum_phi]},
    rounds run, merges per round)."""
    p = dict(TABLE1, **(p or {}))
    regions, nbrs = init_regions(z, phi, valid)
    members = {r: [r] for r in regions}
    per_round = []
    while True:
        k = merge_round(regions, nbrs, p, members)
        per_round.append(k)
        if k == 0 or (max_rounds is not None and len(per_round) >= max_rounds):
            break
    H, W = valid.shape
    labels = np.zeros(H * W, np.int32)
    for s, ms in members.items():
        labels[np.asarray(ms) - 1] = s
    return labels.reshape(H, W), regions, len(per_round), per_round
