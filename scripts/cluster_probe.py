"""Time the NEXT-3 cluster kernel on batches of 204 x 204 scene frames.
  python scripts/cluster_probe.py [F ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1110_5450_b200 import clipseg
    from synth import scenes
    for F in [int(a) for a in sys.argv[1:]] or [1, 16, 64, 256]:
        z, ph, v, _ = scenes.batch(F, 204, 204, seed=14)
        dz, dph, dv = (torch.from_numpy(a).cuda() for a in (z, ph, v.astype(np.uint8)))
        lab, nreg, rounds, ws = clipseg.cluster_frames(dz, dph, dv)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            clipseg.cluster_frames(dz, dph, dv, labels=lab, workspace=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        nr = int(rounds.item())
        print(json.dumps({"frames": F, "ms": ms, "ms_per_frame": ms / F, "rounds": nr, "us_per_round": 1e3 * ms / nr,
                          "mean_regions": float(nreg.float().mean())}), flush=True)


if __name__ == "__main__":
    main()
