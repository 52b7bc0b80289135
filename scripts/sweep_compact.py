"""Build tuning variants of the compacting kernel (here) and time them (on the GPU box).
  python scripts/sweep_compact.py build        # CPU: nvcc variants into build/
  python scripts/sweep_compact.py run [n]      # GPU: time each variant with kernel_probe
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {
    "s16b3m2": ["CLIPSEG_NSUB_F32_2D=16", "CLIPSEG_NBUF_F32_2D=3", "CLIPSEG_MINB_F32_2D=2"],
    "s8b6m2": ["CLIPSEG_NSUB_F32_2D=8", "CLIPSEG_NBUF_F32_2D=6", "CLIPSEG_MINB_F32_2D=2"],
    "s8b4m2": ["CLIPSEG_NSUB_F32_2D=8", "CLIPSEG_NBUF_F32_2D=4", "CLIPSEG_MINB_F32_2D=2"],
    "s16b2m2": ["CLIPSEG_NSUB_F32_2D=16", "CLIPSEG_NBUF_F32_2D=2", "CLIPSEG_MINB_F32_2D=2"],
}


def main():
    if sys.argv[1] == "build":
        import build_all
        for name, defs in VARIANTS.items():
            out, log = build_all.build_variant(name, defs, verbose=True)
            regs = [ln for ln in log.splitlines() if "compact_kernelIfLi2" in ln]
            i = log.find("compact_kernelIfLi2")
            print(name, log[i:i + 400].splitlines()[1:3])
    else:
        n = sys.argv[2] if len(sys.argv) > 2 else "1000000000"
        for name in VARIANTS:
            env = dict(os.environ, CLIPSEG_LIB=os.path.join(ROOT, "build", f"libclipseg_{name}.so"))
            r = subprocess.run(["timeout", "120", sys.executable, os.path.join(ROOT, "scripts", "kernel_probe.py"), "--n", n,
                                "--kernel", "compact", "--reps", "5"], env=env, capture_output=True, text=True)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])["compact"]
                print(name, f"{d['ms']:.3f} ms  {d['GBps']:.0f} GB/s", flush=True)
            except Exception:
                print(name, "FAILED", r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
