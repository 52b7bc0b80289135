"""Time individual kernels with CUDA events (and give ncu a short, fixed launch sequence).

  python scripts/kernel_probe.py --kernel compact --n 100000000 --reps 5 [--dim 2] [--dtype f32] [--mix uniform]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", choices=["dense", "compact", "both"], default="both")
    ap.add_argument("--n", type=int, default=10**8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--family", choices=["uniform", "mix10", "mix33", "mix90", "adv", "homog"], default="uniform")
    ap.add_argument("--ndc", type=int, default=0, help="homog family: perspective-divided output")
    ap.add_argument("--persp", type=float, default=0.0, help="homog family: perspective share (0: recipe default)")
    ap.add_argument("--flags", type=int, default=1)
    ap.add_argument("--index", type=int, default=0)
    a = ap.parse_args()

    import torch
    import synth
    from paper_1110_5450_b200 import clipseg

    dt = torch.float32 if a.dtype == "f32" else torch.float64
    esz = 4 if a.dtype == "f32" else 8
    fam = {"uniform": synth.UNIFORM, "adv": synth.ADVERSARIAL, "homog": synth.HOMOG}.get(a.family, synth.MIX)
    homog = fam == synth.HOMOG
    mix = {"mix10": (0.10, 0.80), "mix33": (1 / 3, 1 / 3), "mix90": (0.90, 0.05)}.get(a.family, (0, 0))
    pin, pc = synth.mix_thresholds(*mix)
    if a.family == "homog" and a.persp > 0:
        pin = synth.mix_thresholds(a.persp, 0)[0]
    n, D = a.n, (4 if homog else a.dim)
    planes = clipseg.empty_planes(n, D, dt)
    synth.fill_device(planes, fam, D, synth.seed_for(5), n, p_in=pin, p_cross=pc)
    lo, hi = [0.0] * D, [1.0] * D
    res = {"n": n, "dim": D, "dtype": a.dtype, "family": a.family, "persp": a.persp, "ndc": a.ndc}
    IN = 2 * D
    OUT = (6 if a.ndc else 8) if homog else 2 * D
    s = torch.cuda.current_stream()

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), min(ts)

    if a.kernel in ("dense", "both"):
        out = torch.empty((OUT, planes.shape[1]), dtype=dt, device="cuda")
        flags = torch.empty(n, dtype=torch.uint8, device="cuda") if a.flags else None
        if homog:
            med, best = timeit(lambda: clipseg.clip_homog(planes, n, ndc=bool(a.ndc), out=out, flags=flags,
                                                          want_flags=bool(a.flags)))
        else:
            med, best = timeit(lambda: clipseg.clip(planes, n, lo, hi, out=out, flags=flags, want_flags=bool(a.flags)))
        b = n * ((IN + OUT) * esz + (1 if a.flags else 0))
        res["dense"] = {"ms": med, "best_ms": best, "GBps": b / med / 1e6, "seg_per_s": n / med * 1e3}
        del out
    if a.kernel in ("compact", "both"):
        if homog:
            bufs = clipseg.HomogBuffers(n, dt, bool(a.ndc), with_index=bool(a.index), with_flags=bool(a.flags))
            med, best = timeit(lambda: clipseg.clip_homog_compact(planes, n, ndc=bool(a.ndc), bufs=bufs))
        else:
            bufs = clipseg.CompactBuffers(n, D, dt, with_index=bool(a.index), with_flags=bool(a.flags))
            med, best = timeit(lambda: clipseg.clip_compact(planes, n, lo, hi, bufs=bufs))
        cnt = int(bufs.count.item())
        b = n * (IN * esz + (1 if a.flags else 0)) + cnt * (OUT * esz + (8 if a.index else 0))
        res["compact"] = {"ms": med, "best_ms": best, "GBps": b / med / 1e6, "seg_per_s": n / med * 1e3,
                          "visible": cnt / n}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
