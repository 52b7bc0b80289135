"""Time the NEXT-4 compacting int32 clip (bench.py run_next4's recipe) for A/B of library
variants: CLIPSEG_LIB=build/libclipseg_<v>.so python scripts/int_probe.py [--n N] [--reps R]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import synth
    from paper_1110_5450_b200 import clipseg
    dev = torch.device("cuda", 0)
    S = synth.INT_SCREEN
    g = torch.Generator(device=dev)
    g.manual_seed(synth.seed_for(9))
    planes = torch.randint(-S // 2, 3 * S // 2, (4, a.n), generator=g, device=dev, dtype=torch.int32)
    bufs = clipseg.CompactBuffers(a.n, 2, torch.int32, dev, with_flags=True)
    s = torch.cuda.current_stream()
    for _ in range(3):
        clipseg.clip_int_compact(planes, a.n, [0, 0], [S - 1, S - 1], bufs=bufs, stream=s)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
    for x, y in ev:
        x.record(s)
        clipseg.clip_int_compact(planes, a.n, [0, 0], [S - 1, S - 1], bufs=bufs, stream=s)
        y.record(s)
    torch.cuda.synchronize()
    print(json.dumps({"int_compact": {"ms": statistics.median(x.elapsed_time(y) for x, y in ev)}}))


if __name__ == "__main__":
    main()
