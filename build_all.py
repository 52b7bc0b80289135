"""Build every native artefact of the repo in-tree (no JIT cache, so the .so files travel
with the gpurun snapshot).

  synth/libsynth.so                       seeded input generator (host + device twins)
  oracle/libclip_oracle.so                the CPU oracle (test infrastructure; gcc)
  paper_1110_5450_b200/lib/libclipseg.so  the product: C-ABI + sm_100a kernels

Run ``python build_all.py`` or call :func:`build` (``__graft_entry__.build`` does).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE semantics on every path: no FTZ, correctly rounded div/sqrt, no mul+add contraction.
NVCC_FP = ["-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=false"]
NVCC_COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
               "-shared", "-cudart", "static"]

SYNTH_SO = os.path.join(ROOT, "synth", "libsynth.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "libclip_oracle.so")
CLIPSEG_SO = os.path.join(ROOT, "paper_1110_5450_b200", "lib", "libclipseg.so")

SYNTH_SRC = [os.path.join(ROOT, "synth", f) for f in ("synth.cu", "synth_core.h")] + [
    os.path.join(ROOT, "include", "synth.h")]
ORACLE_SRC = [os.path.join(ROOT, "oracle", f) for f in ("clip_oracle.c", "clip_oracle_impl.h", "clip_homog_impl.h")]
CSRC = os.path.join(ROOT, "paper_1110_5450_b200", "csrc")


def _clipseg_sources():
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".h"))]
    return srcs + [os.path.join(ROOT, "include", "clipseg.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources if os.path.exists(s))


def _run(cmd):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def build_synth(force=False):
    if force or _stale(SYNTH_SO, SYNTH_SRC):
        _run([NVCC, *ARCH, *NVCC_FP, *NVCC_COMMON, "synth/synth.cu", "-o", SYNTH_SO])
    return SYNTH_SO


def build_oracle(force=False):
    if force or _stale(ORACLE_SO, ORACLE_SRC):
        _run(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-ffp-contract=off", "-fno-fast-math",
              "-fexcess-precision=standard", "-fPIC", "-shared", "oracle/clip_oracle.c", "-o", ORACLE_SO, "-lm"])
    return ORACLE_SO


def build_clipseg(force=False, verbose=False):
    srcs = _clipseg_sources()
    if force or _stale(CLIPSEG_SO, srcs):
        os.makedirs(os.path.dirname(CLIPSEG_SO), exist_ok=True)
        cus = [os.path.relpath(s, ROOT) for s in srcs if s.endswith(".cu")]
        extra = ["-Xptxas", "-v"] if verbose else []
        out = _run([NVCC, *ARCH, *NVCC_FP, *NVCC_COMMON, *extra, "-Iinclude", *cus, "-o", CLIPSEG_SO])
        if verbose:
            sys.stdout.write(out)
    return CLIPSEG_SO


def build_trace():
    """Debug build of the library with per-tile timeline tracing (scripts/trace_compact.py)."""
    srcs = _clipseg_sources()
    out = os.path.join(ROOT, "build", "libclipseg_trace.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cus = [os.path.relpath(s, ROOT) for s in srcs if s.endswith(".cu")]
    _run([NVCC, *ARCH, *NVCC_FP, *NVCC_COMMON, "-DCLIPSEG_TRACE", "-Iinclude", *cus, "-o", out])
    return out


def build_variant(name, defines, verbose=False):
    """Experimental build with -D tuning knobs into build/libclipseg_<name>.so."""
    srcs = _clipseg_sources()
    out = os.path.join(ROOT, "build", f"libclipseg_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cus = [os.path.relpath(s, ROOT) for s in srcs if s.endswith(".cu")]
    extra = ["-Xptxas", "-v"] if verbose else []
    log = _run([NVCC, *ARCH, *NVCC_FP, *NVCC_COMMON, *extra, *[f"-D{d}" for d in defines], "-Iinclude", *cus,
                "-o", out])
    return out, log


def build(force=False, verbose=False):
    build_synth(force)
    build_oracle(force)
    if os.path.isdir(CSRC) and any(f.endswith(".cu") for f in os.listdir(CSRC)):
        build_clipseg(force, verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built:", SYNTH_SO, ORACLE_SO, CLIPSEG_SO)
