"""The C-ABI library loads, exports every symbol include/clipseg.h declares, and validates
its arguments (CPU only: no call here reaches a kernel launch)."""
import ctypes
import os
import re

import pytest

import build_all

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cs():
    build_all.build_clipseg()
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    return clipseg


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\**\s+\**(\w+)\s*\(", src, flags=re.M)))


def test_every_declared_symbol_is_exported(cs):
    names = _declared("clipseg.h")
    assert len(names) >= 11
    lib = ctypes.CDLL(cs.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
        assert nm in cs.EXPORTED, nm


def test_synth_symbols_exported():
    import synth  # noqa: PLC0415
    lib = synth.lib()
    for nm in _declared("synth.h"):
        assert hasattr(lib, nm), nm


def test_stride_and_sizes(cs):
    assert cs.clip_plane_stride(0) == 32
    assert cs.clip_plane_stride(1) == 32
    assert cs.clip_plane_stride(33) == 64
    assert cs.clip_plane_stride(10**9) == 10**9  # already a multiple of 32
    assert cs.clip_compact_workspace_bytes(0) == 128
    assert cs.clip_compact_workspace_bytes(10**9) == 128 + 8 * ((10**9 + 1023) // 1024)
    assert cs.clip_host_staging_bytes(2, 4, 1 << 20) > 2 * 2 * 4 * 4 * (1 << 20)
    assert cs.clip_host_staging_bytes(4, 4, 10) == 0
    for s in (0, -1, -2, -3, -4, 7):
        assert isinstance(cs.clip_status_string(s), bytes)


FAKE = 0x10000  # aligned, never dereferenced: validation fails before any launch


def test_dense_validation(cs):
    w = cs.make_window([0, 0], [1, 1])
    f = cs.clip_segments_f32
    assert f(FAKE, 32, -1, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_EINVAL
    assert f(FAKE, 32, 0, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_OK      # n == 0: no launch
    assert f(None, 32, 10, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_EINVAL
    assert f(FAKE, 8, 10, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_EINVAL   # ld < n
    assert f(FAKE + 4, 32, 10, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_EALIGN
    assert f(FAKE, 33, 10, ctypes.byref(w), FAKE, 32, None, None) == cs.CLIP_EALIGN  # ld*4 % 16
    assert f(FAKE, 32, 10, ctypes.byref(w), FAKE, 32, FAKE + 1, None) == cs.CLIP_EALIGN
    bad = cs.make_window([1, 0], [0, 1])
    assert f(FAKE, 32, 10, ctypes.byref(bad), FAKE, 32, None, None) == cs.CLIP_EINVAL
    nanw = cs.make_window([float("nan"), 0], [1, 1])
    assert f(FAKE, 32, 10, ctypes.byref(nanw), FAKE, 32, None, None) == cs.CLIP_EINVAL
    w4 = cs.make_window([0, 0], [1, 1]); w4.dim = 4
    assert f(FAKE, 32, 10, ctypes.byref(w4), FAKE, 32, None, None) == cs.CLIP_EINVAL
    w64 = cs.make_window([0, 0], [1, 1], "f64")
    assert cs.clip_segments_f64(FAKE, 33, 10, ctypes.byref(w64), FAKE, 32, None, None) == cs.CLIP_EALIGN  # 33*8 % 16


def test_compact_validation(cs):
    w = cs.make_window([0, 0], [1, 1])
    f = cs.clip_segments_compact_f32
    big = 1 << 30
    args = lambda **k: dict(dict(inp=FAKE, ld_in=1024, n=1000, out=FAKE + big, ld_out=1024, idx=None, base=0,  # noqa: E731
                                 flags=None, cnt=FAKE + 2 * big, ws=FAKE + 3 * big, wsb=1 << 20), **k)

    def call(a):
        return f(a["inp"], a["ld_in"], a["n"], ctypes.byref(w), a["out"], a["ld_out"], a["idx"], a["base"],
                 a["flags"], a["cnt"], a["ws"], a["wsb"], None)
    assert call(args(cnt=None)) == cs.CLIP_EINVAL
    assert call(args(n=-5)) == cs.CLIP_EINVAL
    assert call(args(wsb=100)) == cs.CLIP_ENOSPACE
    assert call(args(ws=None)) == cs.CLIP_EINVAL
    assert call(args(ws=FAKE + 3 * big + 8)) == cs.CLIP_EALIGN
    assert call(args(idx=FAKE + 4)) == cs.CLIP_EALIGN
    assert call(args(cnt=FAKE + 2 * big + 4)) == cs.CLIP_EALIGN
    assert call(args(out=FAKE + 64)) == cs.CLIP_EINVAL            # out overlaps in
    assert call(args(inp=FAKE + 8)) == cs.CLIP_EALIGN


def test_homog_validation(cs):
    big = 1 << 30
    f = cs.clip_homog_segments_f32
    assert f(FAKE, 32, -1, 0, FAKE, 32, None, None) == cs.CLIP_EINVAL
    assert f(FAKE, 32, 10, 2, FAKE, 32, None, None) == cs.CLIP_EINVAL            # ndc must be 0 / 1
    assert f(FAKE, 32, 0, 1, FAKE, 32, None, None) == cs.CLIP_OK                 # n == 0: no launch
    assert f(FAKE, 8, 10, 0, FAKE, 32, None, None) == cs.CLIP_EINVAL             # ld < n
    assert f(FAKE + 4, 32, 10, 0, FAKE, 32, None, None) == cs.CLIP_EALIGN
    assert f(FAKE, 32, 10, 0, FAKE, 32, FAKE + 2, None) == cs.CLIP_EALIGN
    assert cs.clip_homog_segments_f64(FAKE, 33, 10, 0, FAKE, 32, None, None) == cs.CLIP_EALIGN
    g = cs.clip_homog_segments_compact_f32
    ok = dict(inp=FAKE, ldi=1024, n=1000, ndc=0, out=FAKE + big, ldo=1024, idx=None, base=0, fl=None,
              cnt=FAKE + 2 * big, ws=FAKE + 3 * big, wsb=1 << 20)

    def call(**k):
        a = dict(ok, **k)
        return g(a["inp"], a["ldi"], a["n"], a["ndc"], a["out"], a["ldo"], a["idx"], a["base"], a["fl"], a["cnt"],
                 a["ws"], a["wsb"], None)
    assert call(cnt=None) == cs.CLIP_EINVAL
    assert call(ndc=-1) == cs.CLIP_EINVAL
    assert call(wsb=64) == cs.CLIP_ENOSPACE
    assert call(ws=FAKE + 3 * big + 8) == cs.CLIP_EALIGN
    assert call(out=FAKE + 7 * 1024 * 4) == cs.CLIP_EINVAL                     # overlaps in's last plane


def test_tof_validation(cs):
    f = cs.clip_tof_range_phi_f32
    assert f(FAKE, FAKE, -1, 10, FAKE, FAKE, None, None, None) == cs.CLIP_EINVAL
    assert f(FAKE, FAKE, 10, 0, FAKE, FAKE, None, None, None) == cs.CLIP_EINVAL      # ppf < 1
    assert f(FAKE, FAKE, 0, 10, FAKE, FAKE, None, None, None) == cs.CLIP_OK          # n == 0: no launch
    assert f(None, FAKE, 10, 10, FAKE, FAKE, None, None, None) == cs.CLIP_EINVAL
    assert f(FAKE, FAKE, 10, 10, None, FAKE, None, None, None) == cs.CLIP_EINVAL
    assert f(FAKE + 4, FAKE, 10, 10, FAKE, FAKE, None, None, None) == cs.CLIP_EALIGN
    assert f(FAKE, FAKE, 10, 10, FAKE, FAKE + 8, None, None, None) == cs.CLIP_EALIGN
    assert f(FAKE, FAKE, 10, 10, FAKE, FAKE, FAKE + 2, None, None) == cs.CLIP_EALIGN
    assert f(FAKE, FAKE, 10, 10, FAKE, FAKE, None, FAKE + 2, None) == cs.CLIP_EALIGN


def test_cluster_validation(cs):
    prm = cs.clip_merge_params(0.04, 0.009, 8 / 3.141592653589793, 4 / 3)
    ws = 1 << 32
    need = cs.clip_cluster_workspace_bytes(2, 8, 8)
    assert need > 0 and cs.clip_cluster_workspace_bytes(-1, 8, 8) == 0 and cs.clip_cluster_workspace_bytes(1, 0, 8) == 0
    # batches run in parts: the workspace of a huge batch is that of one part
    assert cs.clip_cluster_workspace_bytes(10**5, 204, 204) == cs.clip_cluster_workspace_bytes(592, 204, 204)
    f = cs.clip_cluster_frames

    def call(F=2, H=8, W=8, p=prm, rounds=100, z=FAKE, ph=FAKE, v=FAKE, lab=FAKE, nreg=None, d_r=None, w=ws,
             wb=None):
        return f(z, ph, v, F, H, W, ctypes.byref(p) if p is not None else None, rounds, lab, nreg, d_r, w,
                 need if wb is None else wb, None)
    assert call(F=-1) == cs.CLIP_EINVAL
    assert call(H=0) == cs.CLIP_EINVAL
    assert call(p=None) == cs.CLIP_EINVAL
    assert call(rounds=0) == cs.CLIP_EINVAL
    assert call(p=cs.clip_merge_params(-1.0, 0.009, 1.0, 1.0)) == cs.CLIP_EINVAL
    assert call(p=cs.clip_merge_params(float("nan"), 0.009, 1.0, 1.0)) == cs.CLIP_EINVAL
    assert call(F=0) == cs.CLIP_OK                                   # nothing to do, no launch
    assert call(z=None) == cs.CLIP_EINVAL
    assert call(w=ws + 16) == cs.CLIP_EALIGN                         # workspace 256-byte aligned
    assert call(lab=FAKE + 2) == cs.CLIP_EALIGN
    assert call(wb=need - 1) == cs.CLIP_ENOSPACE
    assert call(F=1 << 20, H=1 << 10, W=1 << 10) == cs.CLIP_EINVAL  # more than 2^30 pixels


def test_shard_offsets_validation(cs):
    assert cs.clip_shard_offsets(FAKE, 0, 0, FAKE, FAKE, None) == cs.CLIP_EINVAL
    assert cs.clip_shard_offsets(FAKE, 2, 2, FAKE, FAKE, None) == cs.CLIP_EINVAL
    assert cs.clip_shard_offsets(None, 2, 0, FAKE, FAKE, None) == cs.CLIP_EINVAL


def test_host_pipeline_validation(cs):
    w = cs.make_window([0, 0], [1, 1])
    cnt = ctypes.c_int64(5)
    f = cs.clip_segments_compact_host_f32
    assert f(FAKE, 32, 10, ctypes.byref(w), FAKE, 32, None, ctypes.byref(cnt), 0, FAKE, 1 << 20) == cs.CLIP_EINVAL
    assert f(FAKE, 32, 10, ctypes.byref(w), FAKE, 32, None, ctypes.byref(cnt), 16, FAKE, 10) == cs.CLIP_ENOSPACE
    assert f(FAKE, 32, 10, ctypes.byref(w), FAKE, 32, None, ctypes.byref(cnt), 16, FAKE + 16, 1 << 20) == cs.CLIP_EALIGN
    assert f(FAKE, 32, 0, ctypes.byref(w), FAKE, 32, None, ctypes.byref(cnt), 16, FAKE, 1 << 20) == cs.CLIP_OK
    assert cnt.value == 0


def test_product_path_does_not_import_oracle():
    """The product package never references oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1110_5450_b200")
    for dp, _, fs in os.walk(pkg):
        for fn in fs:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, fn)).read()
                assert "import oracle" not in src and "clip_oracle" not in src, fn


def test_int_validation(cs):
    f = cs.clip_segments_i32
    W = cs.clip_window_i32
    ok = W((ctypes.c_int32 * 2)(0, 0), (ctypes.c_int32 * 2)(4, 4))
    assert f(None, 32, 0, ctypes.byref(ok), None, 32, None, None) == cs.CLIP_OK  # n == 0
    assert f(None, 32, -1, ctypes.byref(ok), None, 32, None, None) == cs.CLIP_EINVAL
    assert f(None, 32, 1, None, None, 32, None, None) == cs.CLIP_EINVAL
    bad = W((ctypes.c_int32 * 2)(5, 0), (ctypes.c_int32 * 2)(4, 4))
    assert f(None, 32, 0, ctypes.byref(bad), None, 32, None, None) == cs.CLIP_EINVAL
    big = W((ctypes.c_int32 * 2)(0, 0), (ctypes.c_int32 * 2)((1 << 30) + 1, 4))
    assert f(None, 32, 0, ctypes.byref(big), None, 32, None, None) == cs.CLIP_EINVAL
    assert f(None, 32, 1, ctypes.byref(ok), None, 32, None, None) == cs.CLIP_EINVAL  # null planes
    assert f(16, 30, 1, ctypes.byref(ok), 16, 32, None, None) == cs.CLIP_EALIGN  # ld*4 % 16 != 0
    assert f(16, 32, 1, ctypes.byref(ok), 16, 32, 2, None) == cs.CLIP_EALIGN  # flags misaligned
