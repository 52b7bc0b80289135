"""ctypes front of the seeded segment generator (include/synth.h, synth/synth_core.h).

Input generator only — it holds none of the clipping arithmetic, so both the oracle
tests and the CUDA path may use it.  The host and device twins are bit-identical.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None
_lock = threading.Lock()

UNIFORM, MIX, ADVERSARIAL, HOMOG = 0, 1, 2, 3
# HOMOG (dim 4: planes x0,y0,z0,w0,x1,y1,z1,w1) tags
H_PERSPECTIVE, H_AFFINE, H_BEHIND, H_ON_PLANE, H_DEGENERATE = 0, 1, 2, 3, 4
CAT_INSIDE, CAT_CROSSING, CAT_OUTSIDE = 0, 1, 2
TAG_NEAR = 0x80

# seed_C = 0x11105450 + config number
SEED_BASE = 0x11105450


def seed_for(config_no: int, extra: int = 0) -> int:
    return SEED_BASE + config_no + (extra << 8)


def mix_thresholds(p_in: float, p_cross: float):
    """Probabilities -> the uint32 thresholds floor(p * 2^32) of the MIX family."""
    return int(p_in * 2**32) & 0xFFFFFFFF, int(p_cross * 2**32) & 0xFFFFFFFF


def plane_stride(n: int) -> int:
    """ld for n segments: n rounded up to a multiple of 32 elements (>= 32)."""
    return max(32, (n + 31) // 32 * 32)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                import build_all  # noqa: PLC0415
                build_all.build_synth()
            L = ctypes.CDLL(_SO)
            P, I64, U64, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32
            for s in ("f32", "f64"):
                f = getattr(L, "synth_fill_host_" + s)
                f.argtypes = [ctypes.c_int, ctypes.c_int, U64, I64, I64, P, I64, P, U32, U32, ctypes.c_int]
                f.restype = ctypes.c_int
                f = getattr(L, "synth_fill_device_" + s)
                f.argtypes = [ctypes.c_int, ctypes.c_int, U64, I64, I64, P, I64, P, U32, U32, P]
                f.restype = ctypes.c_int
            L.synth_tof_host.argtypes = [U64, I64, I64, I64, P, P, ctypes.c_int]
            L.synth_tof_host.restype = ctypes.c_int
            L.synth_tof_device.argtypes = [U64, I64, I64, I64, P, P, P]
            L.synth_tof_device.restype = ctypes.c_int
            L.synth_tof_ranges.argtypes = [U64, I64, I64, P]
            L.synth_tof_ranges.restype = ctypes.c_int
            _lib = L
    return _lib


def fill_host(family, dim, seed, n, dtype=np.float32, i0=0, ld=None, p_in=0, p_cross=0, nthreads=None,
              with_tag=True):
    """Generate n segments (global indices i0..i0+n-1) on the host.
    Returns (planes (2*dim, ld), tag uint8[n] or None)."""
    dt = np.dtype(dtype)
    ld = plane_stride(n) if ld is None else ld
    planes = np.zeros((2 * dim, ld), dtype=dt)
    tag = np.empty(max(n, 1), dtype=np.uint8) if with_tag else None
    nthreads = nthreads or min(8, os.cpu_count() or 1)
    f = lib().synth_fill_host_f32 if dt == np.float32 else lib().synth_fill_host_f64
    st = f(family, dim, seed, i0, n, planes.ctypes.data, ld, tag.ctypes.data if tag is not None else None,
           p_in, p_cross, nthreads)
    if st != 0:
        raise ValueError(f"synth_fill_host: status {st}")
    return planes, (tag[:n] if tag is not None else None)


def fill_device(planes_t, family, dim, seed, n, i0=0, p_in=0, p_cross=0, tag_t=None, stream=None):
    """Generate into an existing CUDA tensor of shape (2*dim, ld) (torch), asynchronously."""
    import torch  # noqa: PLC0415
    ld = planes_t.shape[1]
    f = lib().synth_fill_device_f32 if planes_t.dtype == torch.float32 else lib().synth_fill_device_f64
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    st = f(family, dim, seed, i0, n, planes_t.data_ptr(), ld, tag_t.data_ptr() if tag_t is not None else None,
           p_in, p_cross, stream)
    if st != 0:
        raise RuntimeError(f"synth_fill_device: status {st}")


# ---- NEXT-2: batched ToF frames -------------------------------------------
TOF_W = TOF_H = 204            # 204^2 pixel frames
TOF_PPF = TOF_W * TOF_H


def tof_host(seed, nframes, ppf=TOF_PPF, f0=0, nthreads=None):
    """Frames f0 .. f0+nframes-1 on the host: (d float32[n], I float32[n], ranges float32[nframes, 2])."""
    n = nframes * ppf
    d = np.empty(max(n, 1), np.float32)
    I = np.empty(max(n, 1), np.float32)
    r = np.empty((max(nframes, 1), 2), np.float32)
    nthreads = nthreads or min(8, os.cpu_count() or 1)
    assert lib().synth_tof_host(seed, f0 * ppf, n, ppf, d.ctypes.data, I.ctypes.data, nthreads) == 0
    assert lib().synth_tof_ranges(seed, f0, nframes, r.ctypes.data) == 0
    return d[:n], I[:n], r[:nframes]


def tof_device(d_t, I_t, seed, nframes, ppf=TOF_PPF, f0=0, stream=None):
    """Fill CUDA float32 tensors d_t, I_t (>= nframes*ppf elements) asynchronously; returns the
    per-frame ranges as a host float32 array (nframes, 2)."""
    import torch  # noqa: PLC0415
    n = nframes * ppf
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    st = lib().synth_tof_device(seed, f0 * ppf, n, ppf, d_t.data_ptr(), I_t.data_ptr(), stream)
    if st != 0:
        raise RuntimeError(f"synth_tof_device: status {st}")
    r = np.empty((max(nframes, 1), 2), np.float32)
    assert lib().synth_tof_ranges(seed, f0, nframes, r.ctypes.data) == 0
    return r[:nframes]


# ---- NEXT-4 inputs: int32 pixel-coordinate segments (DESIGN.md §15 recipe) ----------------
INT_SCREEN = 4096  # window [0, 4095]^2: a 4K-class raster


def int_segments_host(seed, n, mix="screen", ld=None):
    """Seeded int32 planes (4, ld) x0, y0, x1, y1 (ld = plane_stride(n) by default).
    mix "screen": endpoints uniform on [-S/2, 3S/2)^2, S = INT_SCREEN (about 1/4 of each
    endpoint inside); "wide": uniform on [-2^30, 2^30]; "edge": small coordinates around
    the window so endpoints hit edges, corners and ties; "range": "wide" with 1 % of the
    coordinates pushed outside [-2^30, 2^30] (flag 2); "mixed": each segment "screen" or
    "wide" with probability 1/2, and 1 % "edge" endpoints beyond +-2^14 (both kernel paths
    inside one warp).  No clipping arithmetic here."""
    ld = plane_stride(n) if ld is None else ld
    rng = np.random.default_rng(seed)
    out = np.zeros((4, ld), dtype=np.int32)
    if mix == "screen":
        v = rng.integers(-INT_SCREEN // 2, 3 * INT_SCREEN // 2, size=(4, n))
    elif mix == "mixed":
        B = 1 << 30
        v = np.where(rng.random(n) < 0.5, rng.integers(-INT_SCREEN // 2, 3 * INT_SCREEN // 2, size=(4, n)),
                     rng.integers(-B, B + 1, size=(4, n)))
        k = 1 << 14
        v = np.where(rng.random((4, n)) < 0.01, rng.choice(np.array([k, k + 1, -k, -k - 1]), size=(4, n)), v)
    elif mix == "edge":
        v = rng.integers(-3, INT_SCREEN // 512 + 3, size=(4, n)) * 512 + rng.integers(-2, 3, size=(4, n))
    else:
        B = 1 << 30
        v = rng.integers(-B, B + 1, size=(4, n))
        if mix == "range":
            bad = rng.random((4, n)) < 0.01
            v = np.where(bad, rng.choice(np.array([-(1 << 31), B + 1, -B - 1, (1 << 31) - 1]), size=(4, n)), v)
    out[:, :n] = v.astype(np.int32)
    return out
