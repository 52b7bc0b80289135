"""Thin Python binding of libclipseg.so (include/clipseg.h).

Argument marshalling only: every step of the clipping path runs in the library's
sm_100a kernels.  The low-level functions carry the C names and take raw pointers;
the helpers at the bottom take torch tensors (PyTorch provides device memory, streams
and process groups — nothing else).  There is no fallback: if the shared library is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CLIPSEG_LIB selects an experimental build of the same library (scripts/sweep_*.py)
LIB_PATH = os.environ.get("CLIPSEG_LIB") or os.path.join(_HERE, "lib", "libclipseg.so")

CLIP_OK, CLIP_EINVAL, CLIP_EALIGN, CLIP_ENOSPACE, CLIP_ECUDA = 0, -1, -2, -3, -4


class clip_window_f32(ctypes.Structure):  # noqa: N801  (C name)
    _fields_ = [("lo", ctypes.c_float * 3), ("hi", ctypes.c_float * 3), ("dim", ctypes.c_int)]


class clip_window_f64(ctypes.Structure):  # noqa: N801
    _fields_ = [("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3), ("dim", ctypes.c_int)]


class clip_merge_params(ctypes.Structure):  # noqa: N801
    _fields_ = [("t_z", ctypes.c_double), ("t_phi", ctypes.c_double), ("alpha_z", ctypes.c_double),
                ("alpha_phi", ctypes.c_double)]


class clip_window_i32(ctypes.Structure):  # noqa: N801
    _fields_ = [("lo", ctypes.c_int32 * 2), ("hi", ctypes.c_int32 * 2)]


TABLE1 = dict(t_z=0.04, t_phi=0.009, alpha_z=8 / 3.141592653589793, alpha_phi=4 / 3)  # PAPER Table 1


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libclipseg.so not built at {LIB_PATH}: run `python build_all.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, U8P, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    L.clip_plane_stride.argtypes = [I64]
    L.clip_plane_stride.restype = I64
    L.clip_status_string.argtypes = [ctypes.c_int]
    L.clip_status_string.restype = ctypes.c_char_p
    for s, W in (("f32", clip_window_f32), ("f64", clip_window_f64)):
        f = getattr(L, "clip_segments_" + s)
        f.argtypes = [P, I64, I64, ctypes.POINTER(W), P, I64, U8P, P]
        f.restype = ctypes.c_int
        f = getattr(L, "clip_segments_compact_" + s)
        f.argtypes = [P, I64, I64, ctypes.POINTER(W), P, I64, P, I64, U8P, P, P, SZ, P]
        f.restype = ctypes.c_int
        f = getattr(L, "clip_segments_compact_host_" + s)
        f.argtypes = [P, I64, I64, ctypes.POINTER(W), P, I64, U8P, ctypes.POINTER(I64), I64, P, SZ]
        f.restype = ctypes.c_int
        f = getattr(L, "clip_homog_segments_" + s)
        f.argtypes = [P, I64, I64, ctypes.c_int, P, I64, U8P, P]
        f.restype = ctypes.c_int
        f = getattr(L, "clip_homog_segments_compact_" + s)
        f.argtypes = [P, I64, I64, ctypes.c_int, P, I64, P, I64, U8P, P, P, SZ, P]
        f.restype = ctypes.c_int
    L.clip_segments_i32.argtypes = [P, I64, I64, ctypes.POINTER(clip_window_i32), P, I64, U8P, P]
    L.clip_segments_i32.restype = ctypes.c_int
    L.clip_segments_compact_i32.argtypes = [P, I64, I64, ctypes.POINTER(clip_window_i32), P, I64, P, I64, U8P, P, P,
                                            SZ, P]
    L.clip_segments_compact_i32.restype = ctypes.c_int
    L.clip_tof_range_phi_f32.argtypes = [P, P, I64, I64, P, P, U8P, P, P]
    L.clip_tof_range_phi_f32.restype = ctypes.c_int
    L.clip_cluster_workspace_bytes.argtypes = [I64, ctypes.c_int, ctypes.c_int]
    L.clip_cluster_workspace_bytes.restype = SZ
    L.clip_cluster_frames.argtypes = [P, P, P, I64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(clip_merge_params),
                                      ctypes.c_int, P, P, P, P, SZ, P]
    L.clip_cluster_frames.restype = ctypes.c_int
    L.clip_compact_workspace_bytes.argtypes = [I64]
    L.clip_compact_workspace_bytes.restype = SZ
    L.clip_host_staging_bytes.argtypes = [ctypes.c_int, ctypes.c_int, I64]
    L.clip_host_staging_bytes.restype = SZ
    L.clip_shard_offsets.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P, P]
    L.clip_shard_offsets.restype = ctypes.c_int
    return L


_lib = _load()

# ---- the C entry points, same names ------------------------------------------------------
clip_plane_stride = _lib.clip_plane_stride
clip_status_string = _lib.clip_status_string
clip_segments_f32 = _lib.clip_segments_f32
clip_segments_f64 = _lib.clip_segments_f64
clip_compact_workspace_bytes = _lib.clip_compact_workspace_bytes
clip_segments_compact_f32 = _lib.clip_segments_compact_f32
clip_segments_compact_f64 = _lib.clip_segments_compact_f64
clip_shard_offsets = _lib.clip_shard_offsets
clip_host_staging_bytes = _lib.clip_host_staging_bytes
clip_segments_compact_host_f32 = _lib.clip_segments_compact_host_f32
clip_segments_compact_host_f64 = _lib.clip_segments_compact_host_f64
clip_tof_range_phi_f32 = _lib.clip_tof_range_phi_f32
clip_segments_i32 = _lib.clip_segments_i32
clip_segments_compact_i32 = _lib.clip_segments_compact_i32
clip_cluster_workspace_bytes = _lib.clip_cluster_workspace_bytes
clip_cluster_frames = _lib.clip_cluster_frames
clip_homog_segments_f32 = _lib.clip_homog_segments_f32
clip_homog_segments_f64 = _lib.clip_homog_segments_f64
clip_homog_segments_compact_f32 = _lib.clip_homog_segments_compact_f32
clip_homog_segments_compact_f64 = _lib.clip_homog_segments_compact_f64

EXPORTED = ["clip_plane_stride", "clip_status_string", "clip_segments_f32", "clip_segments_f64",
            "clip_compact_workspace_bytes", "clip_segments_compact_f32", "clip_segments_compact_f64",
            "clip_shard_offsets", "clip_host_staging_bytes", "clip_segments_compact_host_f32",
            "clip_segments_compact_host_f64", "clip_homog_segments_f32", "clip_homog_segments_f64",
            "clip_homog_segments_compact_f32", "clip_homog_segments_compact_f64", "clip_tof_range_phi_f32",
            "clip_cluster_workspace_bytes", "clip_cluster_frames", "clip_segments_i32", "clip_segments_compact_i32"]


class ClipError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: {clip_status_string(status).decode()} ({status})")
        self.status = status


def _check(status, what):
    if status != CLIP_OK:
        raise ClipError(status, what)


def make_window(lo, hi, dtype="f32"):
    dim = len(lo)
    W = clip_window_f32 if dtype == "f32" else clip_window_f64
    w = W()
    for k in range(dim):
        w.lo[k] = lo[k]
        w.hi[k] = hi[k]
    w.dim = dim
    return w


# ---- torch-level helpers (allocation + marshalling) --------------------------------------
def _torch():
    import torch  # noqa: PLC0415
    return torch


def _sfx(t):
    torch = _torch()
    if t.dtype == torch.float32:
        return "f32"
    if t.dtype == torch.float64:
        return "f64"
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream):
    torch = _torch()
    return (stream if stream is not None else torch.cuda.current_stream()).cuda_stream


def empty_planes(n, dim, dtype, device="cuda"):
    """A (2*dim, clip_plane_stride(n)) planar buffer."""
    torch = _torch()
    return torch.empty((2 * dim, clip_plane_stride(n)), dtype=dtype, device=device)


def clip(planes, n, lo, hi, out=None, flags=None, want_flags=True, stream=None):
    """Dense clip of n segments held in `planes` (2*dim, ld) -> (out, flags)."""
    torch = _torch()
    dim = planes.shape[0] // 2
    sfx = _sfx(planes)
    if out is None:
        out = torch.empty_like(planes)
    if flags is None and want_flags:
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=planes.device)
    w = make_window(lo, hi, sfx)
    f = clip_segments_f32 if sfx == "f32" else clip_segments_f64
    _check(f(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w), out.data_ptr(), out.stride(0),
             flags.data_ptr() if flags is not None else None, _stream(stream)), "clip_segments_" + sfx)
    return out, flags


class CompactBuffers:
    """Reusable outputs + workspace for the compacting clip of up to n segments."""

    def __init__(self, n, dim, dtype, device="cuda", with_index=False, with_flags=False):
        torch = _torch()
        self.n, self.dim = n, dim
        self.out = empty_planes(n, dim, dtype, device)
        self.count = torch.zeros(1, dtype=torch.int64, device=device)
        # zero-filled once; every call leaves it zero-filled again (include/clipseg.h)
        self.ws = torch.zeros(max(int(clip_compact_workspace_bytes(n)), 128), dtype=torch.uint8, device=device)
        self.index = torch.empty(max(n, 1), dtype=torch.int64, device=device) if with_index else None
        self.flags = torch.empty(max(n, 1), dtype=torch.uint8, device=device) if with_flags else None


def clip_compact(planes, n, lo, hi, bufs: CompactBuffers | None = None, with_index=False, with_flags=False,
                 index_base=0, stream=None):
    """Stable compacting clip -> CompactBuffers (out rows [0, count) valid; count on device)."""
    dim = planes.shape[0] // 2
    sfx = _sfx(planes)
    if bufs is None:
        bufs = CompactBuffers(n, dim, planes.dtype, planes.device, with_index, with_flags)
    w = make_window(lo, hi, sfx)
    f = clip_segments_compact_f32 if sfx == "f32" else clip_segments_compact_f64
    _check(f(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w), bufs.out.data_ptr(), bufs.out.stride(0),
             bufs.index.data_ptr() if bufs.index is not None else None, index_base,
             bufs.flags.data_ptr() if bufs.flags is not None else None, bufs.count.data_ptr(),
             bufs.ws.data_ptr(), bufs.ws.numel(), _stream(stream)), "clip_segments_compact_" + sfx)
    return bufs


def clip_compact_host(h_planes, n, lo, hi, h_out, h_flags=None, chunk=1 << 24, staging=None):
    """End-to-end compacting clip of HOST planes (numpy or CPU torch, ideally pinned) through
    the device; returns the visible count.  `staging` (a CUDA uint8 tensor) is reused if given."""
    torch = _torch()
    import numpy as np  # noqa: PLC0415

    def ptr_ld(a):
        if isinstance(a, np.ndarray):
            return a.ctypes.data, a.strides[0] // a.itemsize, a.dtype
        return a.data_ptr(), a.stride(0), a.dtype

    pin, ld_in, dt = ptr_ld(h_planes)
    pout, ld_out, _ = ptr_ld(h_out)
    dim = h_planes.shape[0] // 2
    f64 = dt in (np.float64, torch.float64)
    esz = 8 if f64 else 4
    chunk = max(1, min(chunk, n)) if n > 0 else 1
    need = int(clip_host_staging_bytes(dim, esz, chunk))
    if staging is None or staging.numel() < need:
        staging = torch.empty(need, dtype=torch.uint8, device="cuda")
    w = make_window(lo, hi, "f64" if f64 else "f32")
    cnt = ctypes.c_int64(0)
    fl = None
    if h_flags is not None:
        fl = h_flags.ctypes.data if isinstance(h_flags, np.ndarray) else h_flags.data_ptr()
    f = clip_segments_compact_host_f64 if f64 else clip_segments_compact_host_f32
    _check(f(pin, ld_in, n, ctypes.byref(w), pout, ld_out, fl, ctypes.byref(cnt), chunk, staging.data_ptr(),
             staging.numel()), "clip_segments_compact_host")
    return cnt.value, staging


# ---- NEXT-1: homogeneous clip space (planes x0, y0, z0, w0, x1, y1, z1, w1) --------------
def clip_homog(planes, n, ndc=False, out=None, flags=None, want_flags=True, stream=None):
    """Dense homogeneous clip of n segments in `planes` (8, ld) -> (out (8 or 6 with ndc, ld), flags)."""
    torch = _torch()
    assert planes.shape[0] == 8
    sfx = _sfx(planes)
    if out is None:
        out = torch.empty((6 if ndc else 8, planes.shape[1]), dtype=planes.dtype, device=planes.device)
    if flags is None and want_flags:
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=planes.device)
    f = clip_homog_segments_f32 if sfx == "f32" else clip_homog_segments_f64
    _check(f(planes.data_ptr(), planes.stride(0), n, int(ndc), out.data_ptr(), out.stride(0),
             flags.data_ptr() if flags is not None else None, _stream(stream)), "clip_homog_segments_" + sfx)
    return out, flags


class HomogBuffers(CompactBuffers):
    """Reusable outputs + workspace for the compacting homogeneous clip (8 or 6 output planes)."""

    def __init__(self, n, dtype, ndc=False, device="cuda", with_index=False, with_flags=False):
        torch = _torch()
        super().__init__(n, 3, dtype, device, with_index, with_flags)
        self.ndc = ndc
        self.out = torch.empty((6 if ndc else 8, clip_plane_stride(n)), dtype=dtype, device=device)


def clip_homog_compact(planes, n, ndc=False, bufs: HomogBuffers | None = None, with_index=False,
                       with_flags=False, index_base=0, stream=None):
    """Stable compacting homogeneous clip -> HomogBuffers (out rows [0, count) valid)."""
    sfx = _sfx(planes)
    if bufs is None:
        bufs = HomogBuffers(n, planes.dtype, ndc, planes.device, with_index, with_flags)
    f = clip_homog_segments_compact_f32 if sfx == "f32" else clip_homog_segments_compact_f64
    _check(f(planes.data_ptr(), planes.stride(0), n, int(ndc), bufs.out.data_ptr(), bufs.out.stride(0),
             bufs.index.data_ptr() if bufs.index is not None else None, index_base,
             bufs.flags.data_ptr() if bufs.flags is not None else None, bufs.count.data_ptr(),
             bufs.ws.data_ptr(), bufs.ws.numel(), _stream(stream)), "clip_homog_segments_compact_" + sfx)
    return bufs


# ---- NEXT-4: int32 segments, exact clipping ---------------------------------------------------
def clip_int(planes, n, lo, hi, out=None, flags=None, want_flags=True, stream=None):
    """planes: CUDA int32 (4, ld) x0, y0, x1, y1 (ld a multiple of 4, >= n); lo, hi: 2 ints.
    Returns (out int32 (4, ld_out), flags uint8[n] or None)."""
    torch = _torch()
    if out is None:
        out = torch.empty_like(planes)
    for name, t in (("planes", planes), ("out", out)):
        if t.dtype != torch.int32:
            raise TypeError(f"clip_int: {name} must be int32, got {t.dtype}")
        if t.dim() != 2 or t.shape[0] != 4 or t.stride(1) != 1:
            raise ValueError(f"clip_int: {name} must be a (4, ld) row-major plane view with unit inner stride")
    if flags is None and want_flags:
        flags = torch.empty(max(n, 4), dtype=torch.uint8, device=planes.device)
    win = clip_window_i32((ctypes.c_int32 * 2)(*lo), (ctypes.c_int32 * 2)(*hi))
    # the plane strides are the views' row strides (a column slice big[:, :m] keeps big's ld)
    _check(clip_segments_i32(planes.data_ptr(), planes.stride(0), n, ctypes.byref(win), out.data_ptr(), out.stride(0),
                             flags.data_ptr() if flags is not None else None, _stream(stream)),
           "clip_segments_i32")
    return out, flags


def clip_int_compact(planes, n, lo, hi, bufs: CompactBuffers | None = None, with_index=False, with_flags=False,
                     index_base=0, stream=None):
    """Stable compacting int32 clip (NEXT-4 rules) -> CompactBuffers with int32 out rows [0, count)."""
    torch = _torch()
    if planes.dtype != torch.int32 or planes.dim() != 2 or planes.shape[0] != 4 or planes.stride(1) != 1:
        raise ValueError("clip_int_compact: planes must be an int32 (4, ld) row-major plane view")
    if bufs is None:
        bufs = CompactBuffers(n, 2, torch.int32, planes.device, with_index, with_flags)
    win = clip_window_i32((ctypes.c_int32 * 2)(*lo), (ctypes.c_int32 * 2)(*hi))
    _check(clip_segments_compact_i32(planes.data_ptr(), planes.stride(0), n, ctypes.byref(win), bufs.out.data_ptr(),
                                     bufs.out.stride(0), bufs.index.data_ptr() if bufs.index is not None else None,
                                     index_base, bufs.flags.data_ptr() if bufs.flags is not None else None,
                                     bufs.count.data_ptr(), bufs.ws.data_ptr(), bufs.ws.numel(), _stream(stream)),
           "clip_segments_compact_i32")
    return bufs


# ---- NEXT-2: range clip + phi over batched ToF frames ----------------------------------------
def tof_range_phi(d, I, ppf, ranges, phi=None, code=None, kept=None, want_code=True, want_kept=True, stream=None):
    """d, I: CUDA float32[n]; ranges: CUDA float32[F, 2] (r_min, r_max per frame).
    Returns (phi float32[n], code uint8[n] or None, kept int32[F] or None)."""
    torch = _torch()
    n = d.numel()
    nf = (n + ppf - 1) // ppf
    if phi is None:
        phi = torch.empty(max(n, 4), dtype=torch.float32, device=d.device)
    if code is None and want_code:
        code = torch.empty(max(n, 4), dtype=torch.uint8, device=d.device)
    if kept is None and want_kept:
        kept = torch.empty(max(nf, 1), dtype=torch.int32, device=d.device)
    _check(clip_tof_range_phi_f32(d.data_ptr(), I.data_ptr(), n, ppf, ranges.data_ptr(), phi.data_ptr(),
                                  code.data_ptr() if code is not None else None,
                                  kept.data_ptr() if kept is not None else None, _stream(stream)),
           "clip_tof_range_phi_f32")
    return phi, code, kept


# ---- NEXT-3: mutual-best region merging of batched frames -----------------------------------
def cluster_frames(z, phi, valid, params=None, max_rounds=1 << 30, labels=None, workspace=None, stream=None):
    """z, phi: CUDA float32[F, H, W]; valid: CUDA uint8/bool[F, H, W].  Returns (labels int32[F, H, W],
    nregions int32[F], rounds (device int32[1]), workspace)."""
    torch = _torch()
    F, H, W = z.shape
    p = dict(TABLE1, **(params or {}))
    prm = clip_merge_params(p["t_z"], p["t_phi"], p["alpha_z"], p["alpha_phi"])
    if valid.dtype == torch.bool:
        valid = valid.to(torch.uint8)
    if labels is None:
        labels = torch.empty((F, H, W), dtype=torch.int32, device=z.device)
    nregions = torch.empty(max(F, 1), dtype=torch.int32, device=z.device)
    rounds = torch.zeros(1, dtype=torch.int32, device=z.device)
    need = int(clip_cluster_workspace_bytes(F, H, W))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=z.device)
    _check(clip_cluster_frames(z.data_ptr(), phi.data_ptr(), valid.data_ptr(), F, H, W, ctypes.byref(prm),
                               min(max_rounds, 2**31 - 1), labels.data_ptr(), nregions.data_ptr(), rounds.data_ptr(),
                               workspace.data_ptr(), workspace.numel(), _stream(stream)), "clip_cluster_frames")
    return labels, nregions[:F], rounds, workspace


def shard_offsets(counts_t, rank, stream=None):
    """Exclusive prefix (offset of `rank`) and total of allgathered int64 counts (device)."""
    torch = _torch()
    off = torch.empty(2, dtype=torch.int64, device=counts_t.device)
    _check(clip_shard_offsets(counts_t.data_ptr(), counts_t.numel(), rank, off.data_ptr(), off.data_ptr() + 8,
                              _stream(stream)), "clip_shard_offsets")
    return off
