"""ctypes front of the CPU oracle (oracle/clip_oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg / ``--impl reference`` arm may import this package.  The product
path (``paper_1110_5450_b200``) never imports it, and it never imports the product.

Arrays use the planar layout of DESIGN.md §4: a C-contiguous ``(2*dim, ld)`` array whose
row ``c = e*dim + k`` holds coordinate ``k`` of endpoint ``e``.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CLIP_ORACLE_LIB: a mutated build of the same oracle (scripts/mutate_oracle.py only)
_SO = os.environ.get("CLIP_ORACLE_LIB") or os.path.join(_HERE, "libclip_oracle.so")
_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def _trace_type(real):
    class Trace(ctypes.Structure):
        _fields_ = [("c0", ctypes.c_uint), ("c1", ctypes.c_uint), ("visible", ctypes.c_int),
                    ("t_in", real), ("t_out", real), ("a_in", real * 3), ("a_out", real * 3),
                    ("has_in", ctypes.c_int * 3), ("has_out", ctypes.c_int * 3)]
    return Trace


_TRACE = {np.float32: _trace_type(ctypes.c_float), np.float64: _trace_type(ctypes.c_double)}


def _htrace_type(real):
    class HTrace(ctypes.Structure):
        _fields_ = [("c0", ctypes.c_uint), ("c1", ctypes.c_uint), ("visible", ctypes.c_int),
                    ("t_in", real), ("t_out", real), ("a_in", real * 6), ("a_out", real * 6),
                    ("has_in", ctypes.c_int * 6), ("has_out", ctypes.c_int * 6)]
    return HTrace


_HTRACE = {np.float32: _htrace_type(ctypes.c_float), np.float64: _htrace_type(ctypes.c_double)}
_SFX = {np.float32: "f32", np.float64: "f64"}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                import build_all  # noqa: PLC0415  (repo root on sys.path in tests/bench)
                build_all.build_oracle()
            L = ctypes.CDLL(_SO)
            for s in ("f32", "f64"):
                f = getattr(L, "oracle_clip_" + s)
                f.argtypes = [ctypes.c_int, _P, _P, _P, _I64, _I64, _P, _I64, _P]
                f.restype = ctypes.c_int
                f = getattr(L, "oracle_compact_" + s)
                f.argtypes = [ctypes.c_int, _P, _P, _P, _I64, _I64, _P, _I64, _P, _I64, _P]
                f.restype = ctypes.c_int64
                f = getattr(L, "oracle_clip_one_" + s)
                f.argtypes = [ctypes.c_int, _P, _P, _P, _P, _P]
                f.restype = ctypes.c_int
                f = getattr(L, "oracle_homog_clip_" + s)
                f.argtypes = [_P, _I64, _I64, _P, _I64, _P, ctypes.c_int]
                f.restype = ctypes.c_int
                f = getattr(L, "oracle_homog_compact_" + s)
                f.argtypes = [_P, _I64, _I64, _P, _I64, _P, _I64, _P, ctypes.c_int]
                f.restype = ctypes.c_int64
                f = getattr(L, "oracle_homog_one_" + s)
                f.argtypes = [_P, _P, _P]
                f.restype = ctypes.c_int
            _lib = L
    return _lib


def _dt(x):
    return np.float32 if np.dtype(x) == np.float32 else np.float64


def _win(lo, hi, dim, dt):
    lo3 = np.zeros(3, dtype=dt)
    hi3 = np.zeros(3, dtype=dt)
    lo3[:dim] = np.asarray(lo, dtype=dt)[:dim]
    hi3[:dim] = np.asarray(hi, dtype=dt)[:dim]
    return lo3, hi3


def _ptr(a):
    return a.ctypes.data if a is not None else None


def clip(planes, n, lo, hi, dim, nthreads=1):
    """Dense oracle: returns (out planes (2*dim, ld), flags uint8[n])."""
    dt = _dt(planes.dtype)
    planes = np.ascontiguousarray(planes)
    ld = planes.shape[1]
    assert planes.shape[0] == 2 * dim and n <= ld
    lo3, hi3 = _win(lo, hi, dim, dt)
    out = np.empty_like(planes)
    flags = np.empty(n, dtype=np.uint8)
    f = getattr(lib(), "oracle_clip_" + _SFX[dt])
    rows = planes.dtype.itemsize

    def run(a, b):
        # rows stay strided by ld; offset the base pointers by a elements
        st = f(dim, _ptr(lo3), _ptr(hi3), planes.ctypes.data + a * rows, ld, b - a,
               out.ctypes.data + a * rows, ld, flags.ctypes.data + a)
        assert st == 0, st

    _parallel(run, n, nthreads)
    return out, flags


def compact(planes, n, lo, hi, dim, index_base=0, with_flags=False):
    """Compacting oracle: returns (out planes (2*dim, ld) with the first `count` rows valid,
    out_index int64[count], count[, flags])."""
    dt = _dt(planes.dtype)
    planes = np.ascontiguousarray(planes)
    ld = planes.shape[1]
    lo3, hi3 = _win(lo, hi, dim, dt)
    out = np.full_like(planes, np.nan)
    idx = np.empty(max(n, 1), dtype=np.int64)
    flags = np.empty(max(n, 1), dtype=np.uint8)
    f = getattr(lib(), "oracle_compact_" + _SFX[dt])
    cnt = f(dim, _ptr(lo3), _ptr(hi3), _ptr(planes), ld, n, _ptr(out), ld, _ptr(idx), index_base, _ptr(flags))
    assert cnt >= 0, cnt
    if with_flags:
        return out, idx[:cnt], int(cnt), flags[:n]
    return out, idx[:cnt], int(cnt)


def clip_one(p, lo, hi, dim, dtype=np.float32):
    """One segment p = (x0, y0, [z0], x1, y1, [z1]); returns (q, visible, trace dict)."""
    dt = _dt(dtype)
    pa = np.zeros(6, dtype=dt)
    pa[:2 * dim] = np.asarray(p, dtype=dt)
    q = np.zeros(6, dtype=dt)
    lo3, hi3 = _win(lo, hi, dim, dt)
    tr = _TRACE[dt]()
    vis = getattr(lib(), "oracle_clip_one_" + _SFX[dt])(dim, _ptr(lo3), _ptr(hi3), _ptr(pa), _ptr(q),
                                                       ctypes.addressof(tr))
    assert vis in (0, 1)
    trace = dict(c0=tr.c0, c1=tr.c1, visible=tr.visible, t_in=dt(tr.t_in), t_out=dt(tr.t_out),
                 a_in=np.array(tr.a_in[:dim], dtype=dt), a_out=np.array(tr.a_out[:dim], dtype=dt),
                 has_in=list(tr.has_in[:dim]), has_out=list(tr.has_out[:dim]))
    return q[:2 * dim], bool(vis), trace


# ---- NEXT-1: homogeneous clip space (oracle/clip_homog_impl.h, rules H1..H10) ----------
# Input planes (8, ld): x0, y0, z0, w0, x1, y1, z1, w1.  Output: the same 8 homogeneous
# planes, or with ndc=True the 6 divided ones x0/w0, y0/w0, z0/w0, x1/w1, y1/w1, z1/w1.

def homog_clip(planes, n, ndc=False, nthreads=1):
    """Dense homogeneous oracle: returns (out planes (8 or 6, ld), flags uint8[n])."""
    dt = _dt(planes.dtype)
    planes = np.ascontiguousarray(planes)
    ld = planes.shape[1]
    assert planes.shape[0] == 8 and n <= ld
    out = np.empty((6 if ndc else 8, ld), dtype=dt)
    flags = np.empty(n, dtype=np.uint8)
    f = getattr(lib(), "oracle_homog_clip_" + _SFX[dt])
    rows = planes.dtype.itemsize

    def run(a, b):
        st = f(planes.ctypes.data + a * rows, ld, b - a, out.ctypes.data + a * rows, ld, flags.ctypes.data + a,
               int(ndc))
        assert st == 0, st

    _parallel(run, n, nthreads)
    return out, flags


def homog_compact(planes, n, index_base=0, with_flags=False, ndc=False):
    """Compacting homogeneous oracle: (out (8 or 6, ld) first `count` rows valid, index, count[, flags])."""
    dt = _dt(planes.dtype)
    planes = np.ascontiguousarray(planes)
    ld = planes.shape[1]
    out = np.full((6 if ndc else 8, ld), np.nan, dtype=dt)
    idx = np.empty(max(n, 1), dtype=np.int64)
    flags = np.empty(max(n, 1), dtype=np.uint8)
    f = getattr(lib(), "oracle_homog_compact_" + _SFX[dt])
    cnt = f(_ptr(planes), ld, n, _ptr(out), ld, _ptr(idx), index_base, _ptr(flags), int(ndc))
    assert cnt >= 0, cnt
    if with_flags:
        return out, idx[:cnt], int(cnt), flags[:n]
    return out, idx[:cnt], int(cnt)


def homog_one(p, dtype=np.float32):
    """One segment p = (x0,y0,z0,w0,x1,y1,z1,w1); returns (q[8], visible, trace dict); the
    trace's alphas are per plane j = 2k (w + x_k) / 2k + 1 (w - x_k)."""
    dt = _dt(dtype)
    pa = np.asarray(p, dtype=dt).copy()
    assert pa.shape == (8,)
    q = np.zeros(8, dtype=dt)
    tr = _HTRACE[dt]()
    vis = getattr(lib(), "oracle_homog_one_" + _SFX[dt])(_ptr(pa), _ptr(q), ctypes.addressof(tr))
    assert vis in (0, 1)
    trace = dict(c0=tr.c0, c1=tr.c1, visible=tr.visible, t_in=dt(tr.t_in), t_out=dt(tr.t_out),
                 a_in=np.array(tr.a_in[:], dtype=dt), a_out=np.array(tr.a_out[:], dtype=dt),
                 has_in=list(tr.has_in[:]), has_out=list(tr.has_out[:]))
    return q, bool(vis), trace


def _parallel(run, n, nthreads):
    if nthreads <= 1 or n < 4096:
        run(0, n)
        return
    ths = []
    for t in range(nthreads):
        a, b = n * t // nthreads, n * (t + 1) // nthreads
        th = threading.Thread(target=run, args=(a, b))
        th.start()
        ths.append(th)
    for th in ths:
        th.join()
