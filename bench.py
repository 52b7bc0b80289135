"""bench.py — throughput of the B200 segment-clipping hot path (BASELINE.json metric:
clipped segments/sec and achieved HBM GB/s, % of peak, at 1/2/4/8 B200).

Workload (BASELINE.json configs[4], the metric's multi-GPU config):
10^9 2D fp32 segments, endpoints on the 2^-22 grid uniform in [-1,2)^2, window [0,1]^2,
one step = the whole hot path over the batch: the one-pass compacting clip (outcodes,
trivial accept/reject, WEC intersection, clipped endpoints + flags, stable compaction +
count) and, for N > 1, the NCCL allgather of the per-shard counts plus the offset kernel.
Strong scaling: the 10^9 segments are split contiguously across the N ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (oracle/) on the
host cores over a bounded sample of the same workload (there is no reference code base:
the paper is the reference).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOTAL = 10**9
DIM = 2
WORKLOAD = "C5: 2D fp32 compacting clip, 1e9 segments, endpoints uniform on the 2^-22 grid in [-1,2)^2, window [0,1]^2"
METRIC = "clipped segments/sec"
SEED = 0x11105450 + 5          # synth.seed_for(5)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=N_TOTAL, help="total segments (default 1e9)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=40_000_000)
    ap.add_argument("--no-next1", action="store_true", help="skip the secondary NEXT-1 (homogeneous) measurement")
    ap.add_argument("--no-next2", action="store_true", help="skip the secondary NEXT-2 (range clip + phi) measurement")
    ap.add_argument("--no-next3", action="store_true", help="skip the secondary NEXT-3 (region merging) measurement")
    ap.add_argument("--no-next4", action="store_true", help="skip the secondary NEXT-4 (int32 exact clip) measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE.json configs[0..3] sweep")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.2)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        rows = []
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                rows.append((float(f[0]), float(f[1]), f[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def cpu_oracle_rate(n_sample, nthreads, min_seconds=10.0):
    """The oracle as it stands (oracle/libclip_oracle.so, plain scalar C) on host cores.
    Bounded sample: the first n_sample segments of the workload (regenerated on the host by
    the same seeded generator), clipped repeatedly until min_seconds of wall time have
    passed, statically split over nthreads threads.  Returns (seg/s, seconds, threads, passes)."""
    import numpy as np  # noqa: PLC0415
    import oracle  # noqa: PLC0415  (cpu_baseline leg: the one place bench.py runs oracle/)
    import synth  # noqa: PLC0415
    planes, _ = synth.fill_host(synth.UNIFORM, DIM, SEED, n_sample, dtype=np.float32, with_tag=False)
    ld = planes.shape[1]
    out = np.empty_like(planes)
    flags = np.empty(n_sample, dtype=np.uint8)
    lo3 = np.zeros(3, np.float32)
    hi3 = np.array([1, 1, 0], np.float32)
    f = oracle.lib().oracle_clip_f32

    def run(a, b):
        f(DIM, lo3.ctypes.data, hi3.ctypes.data, planes.ctypes.data + 4 * a, ld, b - a, out.ctypes.data + 4 * a,
          ld, flags.ctypes.data + a)

    passes = 0
    t0 = time.perf_counter()
    while True:
        ths = [threading.Thread(target=run, args=(n_sample * t // nthreads, n_sample * (t + 1) // nthreads))
               for t in range(nthreads)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return passes * n_sample / dt, dt, nthreads, passes


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank, world):
    """`--impl reference`: the oracle timed on the host cores, rank 0 only."""
    if rank != 0:
        return
    nth = min(host_threads(), 64)
    n_s = args.cpu_sample
    cpu_oracle_rate(min(n_s, 1_000_000), nth, 0.0)   # warm-up (page-in, thread start)
    rates = []
    total_t = 0.0
    for _ in range(args.steps):
        r, dt, _, passes = cpu_oracle_rate(n_s, nth, 0.0)
        rates.append(r)
        total_t += dt
        if total_t > 120:
            break
    v = statistics.median(rates)
    sample = f"first {n_s} segments of the workload per step, {len(rates)} steps, {nth} threads (static split)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "segments/s", "n_gpus": world,
            "steps": len(rates), "warmup": args.warmup, "ms_per_step": 1e3 * n_s / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_total": args.n, "sample": n_s, "parallelism": "host threads"},
            "cpu_baseline": {"value": v, "unit": "segments/s", "cores": nth, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch  # noqa: PLC0415
    import torch.distributed as dist  # noqa: PLC0415
    import synth  # noqa: PLC0415
    from paper_1110_5450_b200 import clipseg  # noqa: PLC0415
    from paper_1110_5450_b200.shard import shard_range  # noqa: PLC0415

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    start, stop = shard_range(args.n, world, rank)
    n = stop - start

    # inputs resident in HBM (generated on device by the seeded generator; not timed)
    planes = clipseg.empty_planes(n, DIM, torch.float32, dev)
    synth.fill_device(planes, synth.UNIFORM, DIM, SEED, n, i0=start)
    bufs = clipseg.CompactBuffers(n, DIM, torch.float32, dev, with_index=False, with_flags=True)
    counts = torch.zeros(world, dtype=torch.int64, device=dev)
    offs = torch.zeros(2, dtype=torch.int64, device=dev)
    w = clipseg.make_window([0.0, 0.0], [1.0, 1.0])
    sp = stream.cuda_stream
    launches_per_step = 1 + (1 if world > 1 else 0)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        st = clipseg.clip_segments_compact_f32(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w),
                                               bufs.out.data_ptr(), bufs.out.stride(0), None, start,
                                               bufs.flags.data_ptr(), bufs.count.data_ptr(), bufs.ws.data_ptr(),
                                               bufs.ws.numel(), sp)
        if ev is not None:
            ev[1].record(stream)
        if st != 0:
            raise RuntimeError(clipseg.clip_status_string(st))
        if world > 1:
            dist.all_gather_into_tensor(counts, bufs.count)
            clipseg.clip_shard_offsets(counts.data_ptr(), world, rank, offs.data_ptr(), offs.data_ptr() + 8, sp)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = t0.elapsed_time(t1)
    kts = [a.elapsed_time(b) for a, b in kev]
    kern_ms = statistics.mean(kts)
    kern_med, kern_best = statistics.median(kts), min(kts)
    cnt = int(bufs.count.item())
    if world > 1:
        t = torch.tensor([ms, kern_ms, kern_med, kern_best], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms, kern_med, kern_best = float(t[0]), float(t[1]), float(t[2]), float(t[3])
        total = torch.tensor([cnt], dtype=torch.int64, device=dev)
        dist.all_reduce(total)
        visible_total = int(total.item())
    else:
        visible_total = cnt
    ms_per_step = ms / args.steps
    value = args.n / (ms_per_step / 1e3)

    # algorithmic bytes of the dominant kernel, per launch on this rank
    alg_bytes = n * (2 * DIM * 4 + 1) + cnt * (2 * DIM * 4)
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if tj.get("n") == n:
            traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass

    # sampled parity of this run's output against the oracle (outside the timed region)
    parity = sampled_parity(torch, bufs, n, start, rank)

    # secondary: the NEXT-1 row (homogeneous clip space), rank 0 at N = 1 only
    next1 = None
    if rank == 0 and world == 1 and not args.no_next1:
        next1 = run_next1(torch, clipseg, synth, dev, stream)
    next2 = None
    if rank == 0 and world == 1 and not args.no_next2:
        next2 = run_next2(torch, clipseg, synth, dev, stream)
    next4 = None
    if rank == 0 and world == 1 and not args.no_next4:
        next4 = run_next4(torch, clipseg, synth, dev, stream)
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = run_config_sweep(torch, clipseg, synth, dev, stream)
    # secondary C5 mix row at full size (same buffers, regenerated) and the per-step fixed
    # cost of the sharded step at the N=8 per-rank size
    mix_row = None
    if rank == 0 and world == 1 and not args.no_configs:
        mix_row = run_c5_mix(torch, clipseg, synth, planes, bufs, n, stream)
    fixed = None
    if world == 1 and not args.no_configs:
        fixed = run_fixed_cost(torch, dist, clipseg, synth, dev, stream)
    next3 = None
    if rank == 0 and world == 1 and not args.no_next3:
        next3 = run_next3(torch, clipseg, dev, stream)

    # end to end through the public host-buffer API (pinned host memory, H2D + D2H timed)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(torch, dist, clipseg, synth, args, world, rank, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = min(host_threads(), 64)
        r, dt, nth, passes = cpu_oracle_rate(args.cpu_sample, nth, 10.0)
        s1 = max(args.cpu_sample // 16, 1_000_000)
        r1, dt1, _, passes1 = cpu_oracle_rate(s1, 1, 4.0)
        cpu = {"value": r, "unit": "segments/s", "cores": nth, "kind": "oracle",
               "sample": f"first {args.cpu_sample} segments of the workload, {passes} passes in {dt:.1f} s "
                         f"wall on {nth} threads (static split)",
               "value_1_thread": r1,
               "sample_1_thread": f"first {s1} segments, {passes1} passes in {dt1:.1f} s on 1 thread",
               "cpu_model": cpu_model(), "nproc": os.cpu_count()}

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_total": args.n, "n_per_gpu": n, "dim": DIM, "flags": True,
                   "out_index": False, "visible_fraction": visible_total / args.n,
                   "l2": f"no flush: inputs {16 * n / 1e9:.1f} GB per GPU >> 126 MB L2",
                   "parallelism": f"shard{world} (contiguous; NCCL allgather of counts)"},
        "hbm_gbs_step": alg_bytes / (ms_per_step / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "frac_vs_measured": achieved / peak, "frac_vs_8tbs": achieved / 8000.0,
                     "traffic": traffic, "kernel": "clip_compact_packed_kernel<float,BoxOp<float,2>,1,0>",
                     "kernel_ms": kern_ms, "kernel_ms_median": kern_med, "kernel_ms_best": kern_best,
                     "kernel_ms_stat": f"mean (median, best) over {args.steps} steps",
                     "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src},
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "configs": configs,
        "c5_mix_33": mix_row,
        "fixed_cost": fixed,
        "next1": next1,
        "next2": next2,
        "next4": next4,
        "next3": next3,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sampled_parity(torch, bufs, n, start, rank, m=2000):
    import numpy as np  # noqa: PLC0415
    import oracle  # noqa: PLC0415
    import synth  # noqa: PLC0415
    rng = np.random.default_rng(rank)
    idx = np.unique(np.concatenate([rng.integers(0, n, m), [0, n - 1]]))
    P = np.zeros((2 * DIM, synth.plane_stride(len(idx))), np.float32)
    for j, i in enumerate(idx):
        p, _ = synth.fill_host(synth.UNIFORM, DIM, SEED, 1, i0=start + int(i), nthreads=1, with_tag=False)
        P[:, j] = p[:, 0]
    want, wfl = oracle.clip(P, len(idx), [0, 0], [1, 1], DIM)
    fl = bufs.flags[:n]
    ti = torch.from_numpy(idx).to(fl.device)
    ok = np.array_equal(fl[ti].cpu().numpy(), wfl)
    pos = torch.cumsum(fl, 0, dtype=torch.int32) - 1
    vis = np.nonzero(wfl)[0]
    rows = pos[ti[torch.from_numpy(vis).to(fl.device)]].long()
    got = bufs.out[:, rows].cpu().numpy()
    ok = ok and np.array_equal(got.view(np.uint32), want[:, vis].view(np.uint32))
    del pos
    return f"{'ok' if ok else 'MISMATCH'}: {len(idx)} sampled segments bit-exact vs oracle"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_c5_mix(torch, clipseg, synth, planes, bufs, n, stream, steps=10):
    """C5's secondary row: the same 1e9-segment compacting clip on the MIX
    family with a 1/3 inside, 1/3 crossing, 1/3 outside mix, regenerated into the headline's
    buffers after the headline was timed."""
    pin, pc = synth.mix_thresholds(1 / 3, 1 / 3)
    synth.fill_device(planes, synth.MIX, DIM, synth.seed_for(5, 33), n, p_in=pin, p_cross=pc)
    w = clipseg.make_window([0.0, 0.0], [1.0, 1.0])
    sp = stream.cuda_stream

    def one():
        st = clipseg.clip_segments_compact_f32(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w),
                                               bufs.out.data_ptr(), bufs.out.stride(0), None, 0,
                                               bufs.flags.data_ptr(), bufs.count.data_ptr(), bufs.ws.data_ptr(),
                                               bufs.ws.numel(), sp)
        if st != 0:
            raise RuntimeError(clipseg.clip_status_string(st))

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        one()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    cnt = int(bufs.count.item())
    ms = statistics.median(ts)
    alg = n * (2 * DIM * 4 + 1) + cnt * 2 * DIM * 4
    peak, _ = measured_peak()
    return {"workload": "C5 mix: 1e9 2D fp32 segments, MIX family 1/3 inside, 1/3 crossing, 1/3 outside, "
                        "window [0,1]^2, compacting clip + flags",
            "value": n / (ms / 1e3), "unit": "segments/s", "ms": ms, "ms_best": min(ts),
            "visible_fraction": cnt / n, "GBps": alg / ms / 1e6, "frac": alg / ms / 1e6 / peak,
            "frac_vs_8tbs": alg / ms / 1e6 / 8000.0}


def run_fixed_cost(torch, dist, clipseg, synth, dev, stream, n=125_000_000, steps=30):
    """Per-step fixed cost of the sharded step at the per-rank size of N = 8 (1.25e8): the
    compacting kernel + the NCCL count allgather + the offsets kernel, on a 1-rank NCCL
    group; fixed = median(step) - median(kernel), CUDA events on the launching stream."""
    import socket  # noqa: PLC0415
    made = False
    if not dist.is_initialized():
        with socket.socket() as s_:
            s_.bind(("127.0.0.1", 0))
            port = s_.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        made = True
    try:
        planes = clipseg.empty_planes(n, DIM, torch.float32, dev)
        synth.fill_device(planes, synth.UNIFORM, DIM, SEED, n)
        bufs = clipseg.CompactBuffers(n, DIM, torch.float32, dev, with_flags=True)
        counts = torch.zeros(1, dtype=torch.int64, device=dev)
        offs = torch.zeros(2, dtype=torch.int64, device=dev)
        w = clipseg.make_window([0.0, 0.0], [1.0, 1.0])
        sp = stream.cuda_stream

        def step(ev):
            ev[0].record(stream)
            st = clipseg.clip_segments_compact_f32(planes.data_ptr(), planes.stride(0), n, ctypes.byref(w),
                                                   bufs.out.data_ptr(), bufs.out.stride(0), None, 0,
                                                   bufs.flags.data_ptr(), bufs.count.data_ptr(), bufs.ws.data_ptr(),
                                                   bufs.ws.numel(), sp)
            ev[1].record(stream)
            if st != 0:
                raise RuntimeError(clipseg.clip_status_string(st))
            dist.all_gather_into_tensor(counts, bufs.count)
            clipseg.clip_shard_offsets(counts.data_ptr(), 1, 0, offs.data_ptr(), offs.data_ptr() + 8, sp)
            ev[2].record(stream)

        mk = lambda: tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))  # noqa: E731
        for _ in range(3):
            step(mk())
        torch.cuda.synchronize()
        evs = [mk() for _ in range(steps)]
        for e in evs:
            step(e)
        torch.cuda.synchronize()
        kern = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
        whole = statistics.median(e[0].elapsed_time(e[2]) for e in evs)
        del planes, bufs
        return {"n_per_rank": n, "step_ms": whole, "kernel_ms": kern, "fixed_us": 1e3 * (whole - kern),
                "budget_us": 60, "what": "median(compact + NCCL allgather of 8 B + offsets kernel) - median(compact),"
                                         " 1-rank NCCL group, per-rank size of the N=8 run"}
    finally:
        if made:
            dist.destroy_process_group()


def run_config_sweep(torch, clipseg, synth, dev, stream, steps=10):
    """BASELINE.json configs[0..3] at one GPU, beside the C5 headline:
    the compacting (flags on) and dense kernels, CUDA events, algorithmic bytes / HBM peak."""
    peak, _ = measured_peak()
    rows = []

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    cases = [("C1 2D fp32 1e4 uniform", synth.UNIFORM, 2, torch.float32, 10**4, (0, 0)),
             ("C2 2D fp32 1e8 mix 10/80/10", synth.MIX, 2, torch.float32, 10**8, (0.10, 0.80)),
             ("C2 2D fp32 1e8 mix 33/33/33", synth.MIX, 2, torch.float32, 10**8, (1 / 3, 1 / 3)),
             ("C2 2D fp32 1e8 mix 90/5/5", synth.MIX, 2, torch.float32, 10**8, (0.90, 0.05)),
             ("C2 2D fp32 1e8 uniform", synth.UNIFORM, 2, torch.float32, 10**8, (0, 0)),
             ("C3 2D fp32 1e7 adversarial", synth.ADVERSARIAL, 2, torch.float32, 10**7, (0, 0)),
             ("C3 2D fp64 1e7 adversarial", synth.ADVERSARIAL, 2, torch.float64, 10**7, (0, 0)),
             ("C4 3D fp32 1e8 uniform", synth.UNIFORM, 3, torch.float32, 10**8, (0, 0))]
    for name, fam, D, dt, n, mix in cases:
        esz = 4 if dt == torch.float32 else 8
        pin, pc = synth.mix_thresholds(*mix)
        planes = clipseg.empty_planes(n, D, dt, dev)
        synth.fill_device(planes, fam, D, synth.seed_for(2), n, p_in=pin, p_cross=pc)
        lo, hi = [0.0] * D, [1.0] * D
        bufs = clipseg.CompactBuffers(n, D, dt, dev, with_flags=True)
        ms_c = timed(lambda: clipseg.clip_compact(planes, n, lo, hi, bufs=bufs, stream=stream))
        cnt = int(bufs.count.item())
        del bufs
        out = torch.empty_like(planes)
        flags = torch.empty(n, dtype=torch.uint8, device=dev)
        ms_d = timed(lambda: clipseg.clip(planes, n, lo, hi, out=out, flags=flags, stream=stream))
        near = None
        if fam == synth.ADVERSARIAL:
            # the generator's near-boundary segments (tag bit 0x80: an endpoint within tolerance
            # of an edge), reported separately as north_star asks; for fp32 also the flags that
            # differ from the same inputs clipped in fp64 (upcast exactly) — fp32-ambiguous cases
            tag = torch.empty(n, dtype=torch.uint8, device=dev)
            synth.fill_device(planes, fam, D, synth.seed_for(2), n, p_in=pin, p_cross=pc, tag_t=tag)
            isnear = (tag & 0x80) != 0
            near = {"near_tagged": int(isnear.sum())}
            if dt == torch.float32:
                _, f64 = clipseg.clip(planes.double(), n, lo, hi, stream=stream)
                dis = flags[:n] != f64[:n]
                near["flag_disagree_fp64_near"] = int((dis & isnear).sum())
                near["flag_disagree_fp64_other"] = int((dis & ~isnear).sum())
                del f64, dis
            del tag, isnear
        del out, flags, planes
        bc = n * (2 * D * esz + 1) + cnt * 2 * D * esz
        bd = n * (4 * D * esz + 1)
        rows.append({"config": name, "visible_fraction": cnt / n, "near_boundary": near,
                     "compact": {"ms": ms_c, "segments_per_s": n / ms_c * 1e3, "GBps": bc / ms_c / 1e6,
                                 "frac": bc / ms_c / 1e6 / peak},
                     "dense": {"ms": ms_d, "segments_per_s": n / ms_d * 1e3, "GBps": bd / ms_d / 1e6,
                               "frac": bd / ms_d / 1e6 / peak}})
    return rows


def run_next1(torch, clipseg, synth, dev, stream, n=10**8, steps=20):
    """NEXT-1: the compacting clip in homogeneous clip space, 1e8 fp32
    segments of the HOMOG recipe, homogeneous output + flags; CUDA events on the launching
    stream; roofline against the same measured HBM peak; sampled parity vs the oracle."""
    import numpy as np  # noqa: PLC0415
    import oracle  # noqa: PLC0415
    seed = synth.seed_for(6)
    planes = torch.empty((8, clipseg.clip_plane_stride(n)), dtype=torch.float32, device=dev)
    synth.fill_device(planes, synth.HOMOG, 4, seed, n)
    bufs = clipseg.HomogBuffers(n, torch.float32, False, dev, with_flags=True)
    for _ in range(3):
        clipseg.clip_homog_compact(planes, n, bufs=bufs, stream=stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record(stream)
        clipseg.clip_homog_compact(planes, n, bufs=bufs, stream=stream)
        b.record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    cnt = int(bufs.count.item())
    alg = n * (8 * 4 + 1) + cnt * 8 * 4
    peak, _ = measured_peak()
    # sampled parity: flags and compacted rows of 2000 segments vs the oracle
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.integers(0, n, 2000), [0, n - 1]]))
    P = np.zeros((8, synth.plane_stride(len(idx))), np.float32)
    for j, i in enumerate(idx):
        p, _ = synth.fill_host(synth.HOMOG, 4, seed, 1, i0=int(i), nthreads=1, with_tag=False)
        P[:, j] = p[:, 0]
    want, wfl = oracle.homog_clip(P, len(idx))
    fl = bufs.flags[:n]
    ti = torch.from_numpy(idx).to(dev)
    ok = np.array_equal(fl[ti].cpu().numpy(), wfl)
    pos = torch.cumsum(fl, 0, dtype=torch.int32) - 1
    vis = np.nonzero(wfl)[0]
    got = bufs.out[:, pos[ti[torch.from_numpy(vis).to(dev)]].long()].cpu().numpy()
    ok = ok and np.array_equal(got.view(np.uint32), want[:, vis].view(np.uint32))
    del planes, bufs, pos
    return {"workload": "NEXT-1: homogeneous clip space (-w <= x,y,z <= w), compacting clip, 1e8 fp32 segments "
                        "(HOMOG recipe: 60% perspective, 10% each affine / behind / on-plane / degenerate), "
                        "homogeneous output + flags",
            "value": n / (ms / 1e3), "unit": "segments/s", "ms": ms, "visible_fraction": cnt / n,
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "kernel": "clip_compact_kernel<float,HomogOp>",
                         "alg_bytes_per_launch": alg},
            "parity": f"{'ok' if ok else 'MISMATCH'}: {len(idx)} sampled segments bit-exact vs oracle"}


def run_next2(torch, clipseg, synth, dev, stream, nframes=8192, steps=20):
    """NEXT-2: the paper's per-pixel step — range clip [r_min, r_max] + phi =
    arctan(d sqrt I) with codes and per-frame kept counts — over 8192 frames of 204 x 204;
    CUDA events on the launching stream; sampled frames checked against the oracle."""
    import numpy as np  # noqa: PLC0415
    from oracle import tof_oracle  # noqa: PLC0415
    ppf = synth.TOF_PPF
    n = nframes * ppf
    seed = synth.seed_for(7)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    I = torch.empty_like(d)
    r = torch.from_numpy(synth.tof_device(d, I, seed, nframes)).to(dev)
    phi = torch.empty_like(d)
    code = torch.empty(n, dtype=torch.uint8, device=dev)
    kept = torch.empty(nframes, dtype=torch.int32, device=dev)
    for _ in range(3):
        clipseg.tof_range_phi(d, I, ppf, r, phi=phi, code=code, kept=kept, stream=stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record(stream)
        clipseg.tof_range_phi(d, I, ppf, r, phi=phi, code=code, kept=kept, stream=stream)
        b.record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    alg = n * (4 + 4 + 4 + 1) + nframes * 4
    peak, _ = measured_peak()
    ok = True
    for f in (0, nframes // 3, nframes - 1):
        hd, hI, hr = synth.tof_host(seed, 1, f0=f)
        s = slice(f * ppf, (f + 1) * ppf)
        wc, wp, wk = tof_oracle.tof_range_phi(hd, hI, ppf, hr)
        k = wc == 0
        ok &= bool(np.array_equal(code[s].cpu().numpy(), wc)) and int(kept[f]) == int(wk[0])
        ok &= bool(np.abs(phi[s].cpu().numpy()[k].astype(np.float64) - wp[k]).max() <= 1e-6)
    kept_frac = float(kept.sum().item()) / n
    del d, I, phi, code
    return {"workload": f"NEXT-2: range clip [r_min, r_max] + phi = arctan(d sqrt I), {nframes} ToF frames of "
                        "204x204 (SURVEY §8(f); per-frame ranges, 2% dropouts), codes + per-frame counts",
            "value": n / (ms / 1e3), "unit": "pixels/s", "ms": ms, "kept_fraction": kept_frac,
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "kernel": "tof_range_phi_kernel",
                         "alg_bytes_per_launch": alg},
            "parity": f"{'ok' if ok else 'MISMATCH'}: 3 sampled frames, codes/counts exact, phi within 1e-6"}


def run_next4(torch, clipseg, synth, dev, stream, n=1 << 28, steps=20):
    """NEXT-4: int32 pixel-coordinate segments, exact rational clipping with
    round-half-up endpoints, against the 4096^2 screen window; endpoints uniform on
    [-2048, 6144)^2 drawn on the device by a seeded torch generator (no clipping arithmetic);
    CUDA events on the launching stream; 2048 sampled rows checked against the oracle."""
    import numpy as np  # noqa: PLC0415
    from oracle import int_oracle  # noqa: PLC0415
    S = synth.INT_SCREEN
    lo, hi = [0, 0], [S - 1, S - 1]
    g = torch.Generator(device=dev)
    g.manual_seed(synth.seed_for(9))
    planes = torch.randint(-S // 2, 3 * S // 2, (4, n), generator=g, device=dev, dtype=torch.int32)
    out = torch.empty_like(planes)
    flags = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        clipseg.clip_int(planes, n, lo, hi, out=out, flags=flags, stream=stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record(stream)
        clipseg.clip_int(planes, n, lo, hi, out=out, flags=flags, stream=stream)
        b.record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    alg = n * (16 + 16 + 1)
    peak, _ = measured_peak()
    idx = np.concatenate([np.random.default_rng(2).choice(n, 2048, replace=False), [0, n - 1]])
    ti = torch.from_numpy(idx).to(dev)
    hp = planes[:, ti].cpu().numpy()
    wout, wflags = int_oracle.clip_segments_i32(hp, len(idx), lo, hi)
    ok = bool(np.array_equal(flags[ti].cpu().numpy(), wflags)) and bool(np.array_equal(out[:, ti].cpu().numpy(), wout))
    vis = float((flags == 1).sum().item()) / n
    # the compacting variant (same rules): visible rows in input order, flags 0/1/2
    del out
    bufs = clipseg.CompactBuffers(n, 2, torch.int32, dev, with_flags=True)
    for _ in range(3):
        clipseg.clip_int_compact(planes, n, lo, hi, bufs=bufs, stream=stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record(stream)
        clipseg.clip_int_compact(planes, n, lo, hi, bufs=bufs, stream=stream)
        b.record(stream)
    torch.cuda.synchronize()
    ms_c = statistics.median(a.elapsed_time(b) for a, b in ev)
    cnt = int(bufs.count.item())
    alg_c = n * (16 + 1) + cnt * 16
    # parity of the compacted rows: sampled visible rows found through the flags' prefix sum
    cfl = bufs.flags[:n]
    okc = bool(np.array_equal(cfl[ti].cpu().numpy(), wflags)) and cnt == int((flags == 1).sum().item())
    pos = torch.cumsum(cfl == 1, 0, dtype=torch.int64) - 1
    vrows = np.nonzero(wflags == 1)[0]
    got = bufs.out[:, pos[ti[torch.from_numpy(vrows).to(dev)]]].cpu().numpy()
    okc = okc and bool(np.array_equal(got, wout[:, vrows]))
    del planes, flags, bufs, pos, cfl
    return {"workload": f"NEXT-4: int32 2D segments, exact clip, {n} segments, endpoints uniform on [-{S // 2}, "
                        f"{3 * S // 2})^2, window [0, {S - 1}]^2 (SURVEY §8(f))",
            "value": n / (ms / 1e3), "unit": "segments/s", "ms": ms, "visible_fraction": vis,
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "kernel": "clip_int_kernel",
                         "alg_bytes_per_launch": alg},
            "parity": f"{'ok' if ok else 'MISMATCH'}: {len(idx)} sampled rows bit-exact vs the exact-rational oracle",
            "compact": {"value": n / (ms_c / 1e3), "unit": "segments/s", "ms": ms_c,
                        "roofline": {"bound": "hbm", "achieved": alg_c / (ms_c / 1e3) / 1e9, "peak": peak,
                                     "unit": "GB/s", "frac": alg_c / (ms_c / 1e3) / 1e9 / peak,
                                     "kernel": "clip_compact_packed_kernel<int,IntOp>", "alg_bytes_per_launch": alg_c},
                        "parity": f"{'ok' if okc else 'MISMATCH'}: flags of {len(idx)} sampled rows and their "
                                  "compacted rows bit-exact vs the oracle, count = visible flags"}}


def run_next3(torch, clipseg, dev, stream, nframes=296, steps=3):
    """NEXT-3: the paper's GPU hot path, round-synchronous mutual-best region
    merging to convergence, on a batch of 204 x 204 fused frames (synth/scenes.py) — one
    cooperative launch per batch, timed with CUDA events; one frame checked against the oracle."""
    import numpy as np  # noqa: PLC0415
    from oracle import cluster_oracle  # noqa: PLC0415
    from synth import scenes  # noqa: PLC0415
    z, ph, v, _ = scenes.batch(nframes, 204, 204, seed=14)
    dz, dph, dv = (torch.from_numpy(a).to(dev) for a in (z, ph, v.astype(np.uint8)))
    lab, nreg, rounds, ws = clipseg.cluster_frames(dz, dph, dv, stream=stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        clipseg.cluster_frames(dz, dph, dv, labels=lab, workspace=ws, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    nr = int(rounds.item())
    wl, wr, wrounds, _ = cluster_oracle.cluster(z[0], ph[0], v[0])
    ok = bool(np.array_equal(lab[0].cpu().numpy(), wl)) and int(nreg[0]) == len(wr)
    pix = nframes * 204 * 204
    io_bytes = pix * (4 + 4 + 1 + 4)   # one pass: z, phi, valid in, labels out
    peak, _ = measured_peak()
    return {"workload": f"NEXT-3: mutual-best region merging to convergence (PAPER §4.1, Table 1 params), "
                        f"{nframes} fused frames of 204x204 (synth/scenes.py), one block per frame",
            "value": nframes / (ms / 1e3), "unit": "frames/s", "ms_per_batch": ms, "ms_per_frame": ms / nframes,
            "rounds": nr, "us_per_round": ms * 1e3 / max(nr, 1),
            "mean_regions_per_frame": float(nreg.float().mean().item()),
            "roofline": {"bound": "latency (dependent gathers and 3 block barriers per round, ~1900 rounds)",
                         "achieved": io_bytes / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": io_bytes / (ms / 1e3) / 1e9 / peak, "kernel": "cluster_kernel",
                         "alg_bytes_per_launch": io_bytes},
            "paper_context": "27-29 ms Find Mergepartner, 59-67 ms per frame in total on a GTX 480 (Table 2)",
            "parity": f"{'ok' if ok else 'MISMATCH'}: frame 0 labels identical to the oracle ({wrounds} rounds)"}


def run_e2e(torch, dist, clipseg, synth, args, world, rank, dev):
    """Same metric through the public C-ABI host-buffer entry (clip_segments_compact_host_f32):
    pinned host planes in, compacted planes + flags + count out; copies inside the timed region."""
    import numpy as np  # noqa: PLC0415
    from paper_1110_5450_b200.shard import shard_range  # noqa: PLC0415
    start, stop = shard_range(args.n, world, rank)
    n = stop - start
    try:
        h_in = torch.empty((2 * DIM, clipseg.clip_plane_stride(n)), dtype=torch.float32, pin_memory=True)
        h_out = torch.empty_like(h_in, pin_memory=True)
        h_flags = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    except Exception as e:  # host memory too small for the full workload
        return {"value": None, "unit": "segments/s", "error": f"pinned alloc failed: {e}"[:200]}
    d_tmp = clipseg.empty_planes(min(n, 1 << 26), DIM, torch.float32, dev)
    for a in range(0, n, 1 << 26):   # fill host input from the device generator, chunk by chunk (not timed)
        m = min(1 << 26, n - a)
        synth.fill_device(d_tmp, synth.UNIFORM, DIM, SEED, m, i0=start + a)
        h_in[:, a:a + m].copy_(d_tmp[:, :m])
    del d_tmp
    chunk = 1 << 25
    staging = torch.empty(int(clipseg.clip_host_staging_bytes(DIM, 4, min(chunk, n))), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    cnt, staging = clipseg.clip_compact_host(h_in, n, [0, 0], [1, 1], h_out, h_flags=h_flags, chunk=chunk,
                                             staging=staging)  # warm-up
    times = []
    for _ in range(max(args.e2e_steps, 1)):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        cnt, _ = clipseg.clip_compact_host(h_in, n, [0, 0], [1, 1], h_out, h_flags=h_flags, chunk=chunk,
                                           staging=staging)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    return {"value": args.n / t, "unit": "segments/s", "h2d_bytes_per_step": 2 * DIM * 4 * n,
            "d2h_bytes_per_step": 2 * DIM * 4 * cnt + n + 8, "api": "clip_segments_compact_host_f32",
            "chunk": chunk, "s_per_step": t, "timer": "host wall clock around the blocking call, max over ranks"}


if __name__ == "__main__":
    main()
