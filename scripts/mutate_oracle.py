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

TESTS = {"clip_oracle_impl.h": ["tests/test_oracle_pins.py", "tests/test_oracle_homog.py"],
         "clip_homog_impl.h": ["tests/test_oracle_homog.py"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["cuboid", "homog"])
    a = ap.parse_args()
    rows, bad = [], 0
    for mid, fname, orig, mut, expect in MUTANTS:
        if a.only == "cuboid" and fname != "clip_oracle_impl.h" or a.only == "homog" and fname != "clip_homog_impl.h":
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
