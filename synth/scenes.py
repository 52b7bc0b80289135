"""NEXT-3 inputs: seeded synthetic fused frames (z, phi, valid) for the region-merging
clustering — INPUT GENERATOR ONLY (no clustering arithmetic).  numpy, deterministic in the
seed.  Shape and value ranges follow SPEC.md's synthetic ToF scenes at desk scale:
a background wall at 2.5-3.5 m, a few fronto-parallel plates ("hands") at 0.5-1.5 m, each
object with its own reflectivity so phi = arctan(sqrt(rho)) differs (inverse-square law,
P:557-565), small Gaussian noise (depth sigma 2 mm, phi sigma 0.5 mrad; SPEC.md:400 uses
5 mm / 1 %), and 2 % invalid pixels (the d = 0 sentinel)."""
from __future__ import annotations

import numpy as np


def scene(H, W, seed, n_plates=3, z_sigma=0.002, phi_sigma=0.0005, invalid=0.02):
    """Returns (z float32[H, W], phi float32[H, W], valid bool[H, W], gt int32[H, W]) where gt
    labels the object each pixel was drawn from (0 = wall, k = plate k)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W]
    z = 3.0 + 0.0005 * (xx - W / 2) + 0.0003 * (yy - H / 2)          # slightly slanted wall
    rho = np.full((H, W), 0.3)
    gt = np.zeros((H, W), np.int32)
    for k in range(1, n_plates + 1):
        h, w = rng.integers(H // 6, H // 2 + 1), rng.integers(W // 6, W // 2 + 1)
        y0, x0 = rng.integers(0, H - h + 1), rng.integers(0, W - w + 1)
        zk = rng.uniform(0.5, 1.5)
        rk = rng.uniform(0.4, 1.0)
        z[y0:y0 + h, x0:x0 + w] = zk
        rho[y0:y0 + h, x0:x0 + w] = rk
        gt[y0:y0 + h, x0:x0 + w] = k
    phi = np.arctan(np.sqrt(rho))
    z = (z + z_sigma * rng.standard_normal((H, W))).astype(np.float32)
    phi = (phi + phi_sigma * rng.standard_normal((H, W))).astype(np.float32)
    valid = rng.random((H, W)) >= invalid
    return z, phi, valid, gt


def batch(F, H, W, seed, **kw):
    """F independent scenes stacked: (z[F, H, W], phi[F, H, W], valid[F, H, W], gt[F, H, W])."""
    out = [scene(H, W, seed * 1000003 + f, **kw) for f in range(F)]
    return tuple(np.stack([o[i] for o in out]) for i in range(4))
