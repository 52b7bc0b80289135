"""Per-tile timeline of the compacting kernel (debug build with -DCLIPSEG_TRACE).
  python scripts/trace_compact.py [--n 100000000]
Prints percentiles of: claim->compute start, compute time, A publish -> P publish,
look-back duration, P -> copy start, and the copy wait of each tile."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10**8)
    ap.add_argument("--family", choices=["uniform", "adv"], default="uniform")
    a = ap.parse_args()
    import torch
    import synth
    from paper_1110_5450_b200 import clipseg
    L = ctypes.CDLL(os.path.join(ROOT, "build", "libclipseg_trace.so"))
    P, I64 = ctypes.c_void_p, ctypes.c_int64
    f = L.clip_segments_compact_f32
    f.argtypes = [P, I64, I64, ctypes.POINTER(clipseg.clip_window_f32), P, I64, P, I64, P, P, P, ctypes.c_size_t, P]
    L.clip_trace_read.argtypes = [P, ctypes.c_size_t]
    L.clip_trace_read.restype = ctypes.c_int
    L.clip_trace_clear.restype = ctypes.c_int
    n = a.n
    planes = clipseg.empty_planes(n, 2, torch.float32)
    fam = synth.UNIFORM if a.family == "uniform" else synth.ADVERSARIAL
    synth.fill_device(planes, fam, 2, synth.seed_for(5), n)
    b = clipseg.CompactBuffers(n, 2, torch.float32, with_flags=True)
    w = clipseg.make_window([0, 0], [1, 1])
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        L.clip_trace_clear()
        st = f(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w), b.out.data_ptr(), b.out.stride(0), None, 0,
               b.flags.data_ptr(), b.count.data_ptr(), b.ws.data_ptr(), b.ws.numel(), s)
        assert st == 0
        torch.cuda.synchronize()
    ntiles = (n + int(os.environ.get("BT", "4096")) - 1) // int(os.environ.get("BT", "4096"))
    buf = np.zeros(min(ntiles, 1 << 19) * 8, dtype=np.uint64)
    assert L.clip_trace_read(buf.ctypes.data, buf.nbytes) == 0
    t = buf.reshape(-1, 8).astype(np.int64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    tr = t.copy()
    tr[:, :7] -= t0
    ok = (t[:, 1] > 0) & (t[:, 2] > 0) & (t[:, 5] > 0) & (t[:, 6] > 0)
    tr = tr[ok]
    pct = lambda x: {p: round(float(np.percentile(x, p)) / 1000, 2) for p in (10, 50, 90, 99)}  # noqa: E731
    res = {
        "tiles": int(ok.sum()),
        "span_us": float(tr[:, 6].max()) / 1000,
        "claim_to_start_us": pct(tr[:, 1] - tr[:, 0]),
        "compute_us (start->A)": pct(tr[:, 2] - tr[:, 1]),
        "lookback_us": pct(tr[:, 4] - tr[:, 3]),
        "lookback_end_minus_A_us": pct(tr[:, 4] - tr[:, 2]),
        "A_to_P_us (scanner publish)": pct(tr[:, 5] - tr[:, 2]),
        "P_published_to_seen_us": pct(tr[:, 4] - tr[:, 5]),
        "poll_start_minus_A_us": pct(tr[:, 3] - tr[:, 2]),
        "P_seen_to_copy_us": pct(tr[:, 6] - tr[:, 4]),
        "claim_order_vs_A_order_inversions": float(np.mean(np.diff(tr[:, 2]) < 0)),
    }
    # per block: busy time (sum of start->A over its tiles) against the launch span
    blk = t[ok][:, 7]
    comp = (tr[:, 2] - tr[:, 1]).astype(np.float64)
    busy = np.array([comp[blk == bb].sum() for bb in np.unique(blk)]) / 1000
    ntl = np.array([(blk == bb).sum() for bb in np.unique(blk)])
    res["block_busy_us"] = {p: round(float(np.percentile(busy, p)), 2) for p in (10, 50, 90)}
    res["block_tiles"] = {p: int(np.percentile(ntl, p)) for p in (10, 50, 90)}
    # copy-out waits: a block copies tile t_i out right after publishing t_{i+2}'s aggregate;
    # the wait is max(0, copy start of t_i - A of t_{i+2}) (warp 0's view)
    tiles_ok = np.nonzero(ok)[0]
    waits, spans = [], []
    for bb in np.unique(blk):
        tl = tiles_ok[blk == bb]
        tl = tl[np.argsort(t[tl, 0])]  # claim order
        for i in range(len(tl) - 2):
            waits.append(max(0, int(t[tl[i], 6]) - int(t[tl[i + 2], 2])))
        spans.append(float(t[tl, 6].max() - t[tl, 1].min()))
    waits = np.array(waits, dtype=np.float64) / 1000
    res["copy_wait_us"] = {p: round(float(np.percentile(waits, p)), 3) for p in (50, 75, 90, 99)}
    res["copy_wait_share_of_block_span"] = round(float(waits.sum() / (np.sum(spans) / 1000)), 4)
    res["first_start_us"] = float(tr[:, 1].min()) / 1000
    res["last_A_us"] = float(tr[:, 2].max()) / 1000
    # lateness of predecessor: A time of t-1 minus A time of t
    res["pred_A_later_than_mine_us"] = pct(np.maximum(tr[:-1, 2] - tr[1:, 2], 0))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
