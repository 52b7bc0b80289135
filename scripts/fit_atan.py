"""Fit the degree-8 polynomial p(z) with atan(r) ~ r p(r^2) on r in [0, 1] (Lawson's
iteratively reweighted least squares -> near-minimax absolute error) used by
paper_1110_5450_b200/csrc/tof_range.cu, and report its error, alone and through a binary32
FMA evaluation with the kernel's range reduction (reciprocal for x > 1).

  python scripts/fit_atan.py"""
import numpy as np


def fit(D=8, N=4000, iters=200):
    t = np.cos(np.pi * (np.arange(N) + 0.5) / N)
    r = (t + 1) / 2
    A = np.stack([r * (r * r) ** k for k in range(D + 1)], 1)
    f = np.arctan(r)
    w = np.ones(N)
    for _ in range(iters):
        W = np.sqrt(w)
        c, *_ = np.linalg.lstsq(A * W[:, None], f * W, rcond=None)
        w = w * np.abs(A @ c - f)
        w /= w.sum()
    return c


def fp32_chain(x, c):
    c32 = [np.float32(v) for v in c]
    big = x > 1
    r = np.where(big, (1 / np.maximum(x.astype(np.float64), 1e-300)).astype(np.float32), x)
    z = (r.astype(np.float64) ** 2).astype(np.float32)
    p = np.full_like(z, c32[-1])
    for k in range(len(c) - 2, -1, -1):
        p = (p.astype(np.float64) * z.astype(np.float64) + np.float64(c32[k])).astype(np.float32)
    a = (r.astype(np.float64) * p).astype(np.float32)
    return np.where(big, (np.float64(np.float32(np.pi / 2)) - a).astype(np.float32), a)


if __name__ == "__main__":
    c = fit()
    rr = np.linspace(0, 1, 200001)
    print("coefficients (z^0 .. z^8):", [float(v) for v in c])
    print("approximation error on [0,1]:", np.abs(rr * np.polyval(c[::-1], rr * rr) - np.arctan(rr)).max())
    x = np.concatenate([np.linspace(0, 50, 800001), np.logspace(1, 20, 20001)]).astype(np.float32)
    print("binary32 chain error:", np.abs(fp32_chain(x, c).astype(np.float64) - np.arctan(x.astype(np.float64))).max())
