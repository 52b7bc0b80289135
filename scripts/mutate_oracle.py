"""Mutation check of the oracle's pins: apply one plausible slip at a time to the oracle
sources (a temporary copy), rebuild it, and run the CPU pin tests against the mutant.
Every mutant must be killed (some pin test fails), except those listed as equivalent.

  python scripts/mutate_oracle.py [--only cuboid|homog]

Test infrastructure: touches only a temporary copy of oracle/ (never the tree)."""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (id, file, original text, mutated text, expected: "killed" | "equivalent")
MUTANTS = [
    ("M0 unmutated (harness check)", "clip_homog_impl.h", "#define HCAT_(a, b) a##b", "#define HCAT_(a, b) a##b",
     "equivalent"),
    ("M0 unmutated (harness check)", "clip_oracle_impl.h", "#define CAT_(a, b) a##b", "#define CAT_(a, b) a##b",
     "equivalent"),
    ("C1 WEC sign", "clip_oracle_impl.h", "wl0[k] = P0[k] - lo[k];", "wl0[k] = lo[k] - P0[k];", "killed"),
    ("C2 max as min", "clip_oracle_impl.h", "if (has_in[k] && a_in[k] > t_in)", "if (has_in[k] && a_in[k] < t_in)",
     "killed"),
    ("C3 snap edge swapped", "clip_oracle_impl.h", "Q0[k] = (wl0[k] < 0) ? lo[k] : hi[k];",
     "Q0[k] = (wl0[k] < 0) ? hi[k] : lo[k];", "killed"),
    ("C4 fma from P1", "clip_oracle_impl.h", "q = FMA(t_in, d, P0[k]);", "q = FMA(t_in, d, P1[k]);", "killed"),
    ("C5 clamp dropped", "clip_oracle_impl.h",
     "      q = FMA(t_out, d, P0[k]);\n      Q1[k] = (q < lo[k]) ? lo[k] : (q > hi[k]) ? hi[k] : q;",
     "      q = FMA(t_out, d, P0[k]);\n      Q1[k] = q;", "killed"),
    ("C6 outcode <=", "clip_oracle_impl.h", "if (wl0[k] < 0) c0 |= 1u << (2 * k);",
     "if (wl0[k] <= 0) c0 |= 1u << (2 * k);", "killed"),
    ("C7 inside copy dropped", "clip_oracle_impl.h", "if (c0 == 0) Q0[k] = P0[k];\n    else if",
     "if (0) Q0[k] = P0[k];\n    else if", "killed"),
    ("C8 open window", "clip_oracle_impl.h", "if (!(t_in <= t_out)) goto invisible;",
     "if (!(t_in < t_out)) goto invisible;", "killed"),
    ("C9 no finiteness test", "clip_oracle_impl.h",
     "if (!isfinite(P0[k]) || !isfinite(P1[k])) goto invisible;", "(void)0;", "killed"),
    ("C10 alpha operands swapped", "clip_oracle_impl.h", "      a_in[k] = w0 / (w0 - w1);",
     "      a_in[k] = w1 / (w1 - w0);", "killed"),
    ("C11 trivial accept removed", "clip_oracle_impl.h", "if ((c0 | c1) == 0) {", "if (0) {", "equivalent"),
    ("H1 planes swapped", "clip_homog_impl.h", "bl0[k] = P0[3] + P0[k];", "bl0[k] = P0[3] - P0[k];", "killed"),
    ("H2 one plane dropped", "clip_homog_impl.h", "  for (k = 0; k < 6; ++k) {\n    const REAL b0",
     "  for (k = 0; k < 5; ++k) {\n    const REAL b0", "killed"),
    ("H3 w not interpolated", "clip_homog_impl.h", "qw0 = FMA(t_in, dw, P0[3]);", "qw0 = P0[3];", "killed"),
    ("H4 snap sign", "clip_homog_impl.h", "          Q0[k] = -qw0;", "          Q0[k] = qw0;", "killed"),
    ("H5 clamp to 0", "clip_homog_impl.h", "Q1[k] = (q < -qw1) ? -qw1 : (q > qw1) ? qw1 : q;",
     "Q1[k] = (q < 0) ? 0 : (q > qw1) ? qw1 : q;", "killed"),
    ("H6 NDC wrong w", "clip_homog_impl.h", "Q0[3] == 0 ? HNAME(canonical_nan_)() : Q0[k] / Q0[3];",
     "Q0[3] == 0 ? HNAME(canonical_nan_)() : Q0[k] / Q1[3];", "killed"),
    ("H7 NDC zero rule dropped", "clip_homog_impl.h", "Q1[3] == 0 ? HNAME(canonical_nan_)() : Q1[k] / Q1[3];",
     "Q1[k] / Q1[3];", "killed"),
    ("H8 dw reversed", "clip_homog_impl.h", "const REAL dw = P1[3] - P0[3];", "const REAL dw = P0[3] - P1[3];",
     "killed"),
    ("H9 exiting max", "clip_homog_impl.h", "if (has_out[k] && a_out[k] < t_out)",
     "if (has_out[k] && a_out[k] > t_out)", "killed"),
    ("H10 high snap before low", "clip_homog_impl.h",
     "        if (has_out[2 * k] && a_out[2 * k] == t_out) {\n          Q1[k] = -qw1;",
     "        if (0) {\n          Q1[k] = -qw1;", "killed"),
]

# NEXT-2 / NEXT-3 oracles (Python): mutated in a temporary copy of the repository
MUTANTS += [
    ("M0 unmutated (harness check)", "tof_oracle.py", "import numpy as np", "import numpy as np", "equivalent"),
    ("M0 unmutated (harness check)", "cluster_oracle.py", "import numpy as np", "import numpy as np", "equivalent"),
    ("T1 open interval", "tof_oracle.py", "below = d < r_min", "below = d <= r_min", "killed"),
    ("T2 sqrt dropped", "tof_oracle.py", "np.asarray(d, np.float64) * np.sqrt(np.asarray(I, np.float64))",
     "np.asarray(d, np.float64) * np.asarray(I, np.float64)", "killed"),
    ("T3 d = 0 accepted", "tof_oracle.py", "invalid = ~(d > 0)", "invalid = ~(d >= 0)", "killed"),
    ("T4 I < 0 accepted", "tof_oracle.py", "| ~(I >= 0)", "| ~(I >= -1)", "killed"),
    ("T5 wrong frame of a pixel", "tof_oracle.py", "f = np.arange(n, dtype=np.int64) // ppf",
     "f = (np.arange(n, dtype=np.int64) + 1) // ppf", "killed"),
    ("K1 ties to the smaller id", "cluster_oracle.py", "(d == bd and s > best)", "(d == bd and s < best)",
     "killed"),
    ("K2 merges need not be mutual", "cluster_oracle.py", "and r < s and best.get(s) == r]",
     "and r < s and best.get(s) is not None]", "killed"),
    ("K3 unweighted mean", "cluster_oracle.py", "regions[s] = [cs + cr, zs + zr, ps + pr]",
     "regions[s] = [cs + cr, (zs / cs + zr / cr) / 2 * (cs + cr), (ps / cs + pr / cr) / 2 * (cs + cr)]", "killed"),
    ("K4 strict Eq. (1)", "cluster_oracle.py", "abs(mr[0] - ms[0]) <= p[\"t_z\"]", "abs(mr[0] - ms[0]) < p[\"t_z\"]",
     "killed"),
    ("K5 Eq. (2) without phi", "cluster_oracle.py", " + p[\"alpha_phi\"] * abs(mr[1] - ms[1])", "", "killed"),
    ("K6 survivor keeps the smaller id", "cluster_oracle.py",
     "pairs = [(r, s) for r, s in best.items() if s is not None and r < s and best.get(s) == r]",
     "pairs = [(s, r) for r, s in best.items() if s is not None and r < s and best.get(s) == r]", "killed"),
    ("M0 unmutated (harness check)", "int_oracle.py", "import numpy as np", "import numpy as np", "equivalent"),
    ("I1 round half down", "int_oracle.py", "math.floor(x + Fraction(1, 2))", "math.ceil(x - Fraction(1, 2))", "killed"),
    ("I2 truncate instead of round", "int_oracle.py", "math.floor(x + Fraction(1, 2))", "int(x)", "killed"),
    ("I3 WEC sign on the lo edge", "int_oracle.py", "(p0[k] - lo[k], p1[k] - lo[k])", "(lo[k] - p0[k], lo[k] - p1[k])",
     "killed"),
    ("I4 max as min for t_in", "int_oracle.py", "t_in = max(t_in, Fraction(w0, w0 - w1))",
     "t_in = min(t_in, Fraction(w0, w0 - w1))", "killed"),
    ("I5 open window", "int_oracle.py", "if t_in > t_out:", "if t_in >= t_out:", "killed"),
    ("I6 Q1 from t_in", "int_oracle.py", "q1 = tuple(int(p0[k]) + round_half_up(d[k] * t_out)",
     "q1 = tuple(int(p0[k]) + round_half_up(d[k] * t_in)", "killed"),
    ("I7 range bound 2^31", "int_oracle.py", "COORD_MAX = 1 << 30", "COORD_MAX = 1 << 31", "killed"),
    ("I8 swapped axes in d", "int_oracle.py", "d = (p1[0] - p0[0], p1[1] - p0[1])", "d = (p1[1] - p0[1], p1[0] - p0[0])",
     "killed"),
]

TESTS = {"clip_oracle_impl.h": ["tests/test_oracle_pins.py", "tests/test_oracle_homog.py"],
         "clip_homog_impl.h": ["tests/test_oracle_homog.py"],
         "tof_oracle.py": ["tests/test_oracle_tof.py"],
         "cluster_oracle.py": ["tests/test_oracle_cluster.py"],
         "int_oracle.py": ["tests/test_oracle_int.py"]}


def run_python_mutant(fname, orig, mut):
    """Mutate a Python oracle in a temporary copy of the repository and run its pins there."""
    with tempfile.TemporaryDirectory() as td:
        repo = os.path.join(td, "repo")
        shutil.copytree(ROOT, repo, ignore=shutil.ignore_patterns(".git", "build", "gpurun_out", "__pycache__",
                                                                  ".pytest_cache", "profiles"))
        path = os.path.join(repo, "oracle", fname)
        text = open(path).read()
        assert text.count(orig) >= 1, (fname, orig)
        open(path, "w").write(text.replace(orig, mut, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            *TESTS[fname]], cwd=repo, capture_output=True, text=True)
        return r.returncode != 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["cuboid", "homog", "python", "int"])
    a = ap.parse_args()
    rows, bad = [], 0
    for mid, fname, orig, mut, expect in MUTANTS:
        if (a.only == "cuboid" and fname != "clip_oracle_impl.h" or a.only == "homog" and fname != "clip_homog_impl.h"
                or a.only == "python" and not fname.endswith(".py") or a.only == "int" and fname != "int_oracle.py"):
            continue
        if fname.endswith(".py"):
            got = "killed" if run_python_mutant(fname, orig, mut) else "survived"
            ok = (got == "killed") == (expect == "killed")
            bad += not ok
            rows.append((mid, got, expect, "ok" if ok else "UNEXPECTED"))
            print(f"{mid:30s} {got:9s} (expected {expect}) {'' if ok else '<-- UNEXPECTED'}", flush=True)
            continue
        with tempfile.TemporaryDirectory() as td:
            src = os.path.join(td, "oracle")
            shutil.copytree(os.path.join(ROOT, "oracle"), src, ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            path = os.path.join(src, fname)
            text = open(path).read()
            assert text.count(orig) >= 1, (mid, orig)
            open(path, "w").write(text.replace(orig, mut, 1))
            so = os.path.join(td, "libmut.so")
            subprocess.run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                            "-fexcess-precision=standard", "-fPIC", "-shared", os.path.join(src, "clip_oracle.c"),
                            "-o", so, "-lm"], check=True, capture_output=True)
            env = dict(os.environ, CLIP_ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", *TESTS[fname]],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            got = "killed" if r.returncode != 0 else "survived"
            ok = (got == "killed") == (expect == "killed")
            bad += not ok
            rows.append((mid, got, expect, "ok" if ok else "UNEXPECTED"))
            print(f"{mid:30s} {got:9s} (expected {expect}) {'' if ok else '<-- UNEXPECTED'}", flush=True)
    print(f"{len(rows)} mutants, {bad} unexpected")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
