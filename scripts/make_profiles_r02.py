"""Round-2 profile set -> tracked profiles/ (replaces scripts/make_profiles.py's .ncu-rep input
with the raw-page CSVs gpurun brings back).

  python scripts/make_profiles_r02.py <gpurun_out dir> <tag>

Writes, from <dir>/<tag>p_*:
  profiles/<tag>_launches.csv + <tag>_launch_shares.txt   launch list of `bench.py --steps 3 --warmup 3`
  profiles/<tag>_ncu_<kernel>.csv                          key counters of each ncu --set full capture
  profiles/<tag>_ncu_summary.txt                            one block per kernel (time, DRAM, issue, stalls)
  profiles/traffic.json                                     DRAM bytes per launch of the headline kernel
"""
import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct", "sm__warps_active.avg.pct", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "gpu__dram_throughput.avg.pct", "lts__t_bytes.sum", "smsp__average_warps_issue_stalled",
        "launch__shared_mem_per_block", "sm__inst_executed_pipe_", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
# capture -> (segments or units per launch, what)
UNITS = {"headline": (10**9, "C5 1e9 2D fp32 compacting (bench.py context)"),
         "dense2d": (10**8, "C2 1e8 2D fp32 dense"), "compact3d": (10**8, "C4 1e8 3D fp32 compacting"),
         "homog": (10**8, "NEXT-1 1e8 homogeneous compacting"), "homogndc": (10**8, "NEXT-1 1e8 NDC compacting"),
         "adv2d": (10**7, "C3 1e7 2D fp32 adversarial compacting"),
         "adv2d64": (10**7, "C3 1e7 2D fp64 adversarial compacting"),
         "mix33": (10**8, "C2 1e8 mix 1/3 compacting"),
         "tof_range_phi_kernel": (8192 * 204 * 204, "NEXT-2 range clip + phi, 8192 frames"),
         "clip_int_kernel": (1 << 28, "NEXT-4 int32 exact clip, 2^28")}


def load_raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None, None
    return dict(zip(rows[0], rows[1])), dict(zip(rows[0], rows[2]))


def main():
    d, tag = sys.argv[1:3]
    os.makedirs(P, exist_ok=True)
    # launch list + shares
    lsrc = os.path.join(d, f"{tag}p_launches.csv")
    shutil.copy(lsrc, os.path.join(P, f"{tag}_launches.csv"))
    rows = [r for r in csv.reader(open(lsrc)) if r and not r[0].startswith("==")]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) == len(h) and r[ix["Metric Name"]] == "gpu__time_duration.sum":
            agg[r[ix["Kernel Name"]].split("(")[0][:100]].append(
                float(r[ix["Metric Value"]]) * TSCALE.get(r[ix["Metric Unit"]], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(P, f"{tag}_launch_shares.txt"), "w") as f:
        f.write(f"# {lsrc}: ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
                "--steps 3 --warmup 3 (cold-cache, serialised launches: compare shares, not absolute times)\n")
        f.write("launches  total_ms  share  kernel\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{len(v):8d} {sum(v):9.3f} {100 * sum(v) / tot:5.1f}%  {k}\n")
    # per-kernel captures
    summary = []
    for name, (units, what) in UNITS.items():
        path = os.path.join(d, f"{tag}p_{name}_raw.csv")
        if not os.path.exists(path):
            continue
        u, v = load_raw(path)
        if v is None:
            continue
        with open(os.path.join(P, f"{tag}_ncu_{name}.csv"), "w") as f:
            w = csv.writer(f)
            w.writerow(["metric", "unit", "value"])
            w.writerow(["Kernel Name", "", v.get("Kernel Name", "")])
            for k in u:
                if any(k.startswith(p) for p in KEEP) and v.get(k) not in ("", "n/a", None):
                    w.writerow([k, u.get(k, ""), v[k]])
        ms = float(v["gpu__time_duration.sum"]) * TSCALE.get(u["gpu__time_duration.sum"], 1e-3)
        rd = float(v["dram__bytes_read.sum"]) * SCALE.get(u["dram__bytes_read.sum"], 1)
        wr = float(v["dram__bytes_write.sum"]) * SCALE.get(u["dram__bytes_write.sum"], 1)
        inst = float(v["smsp__inst_executed.sum"])
        st = sorted(((k, float(x)) for k, x in v.items() if k.startswith("smsp__average_warps_issue_stalled")
                     and k.endswith("per_issue_active.ratio") and x not in ("", "n/a")), key=lambda t: -t[1])[:6]
        pipes = sorted(((k.split("pipe_")[1].split(".")[0], float(x)) for k, x in v.items()
                        if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active")
                        and x not in ("", "n/a")), key=lambda t: -t[1])[:4]
        summary.append(
            f"== {name}: {what}\n   kernel {v.get('Kernel Name', '')[:110]}\n"
            f"   {ms:.3f} ms, DRAM {rd / 1e9:.3f} GB read + {wr / 1e9:.3f} GB written = {(rd + wr) / ms / 1e6:.0f} GB/s, "
            f"{32 * inst / units:.1f} thread-instructions per unit, issue active "
            f"{float(v['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} %, warps active "
            f"{float(v['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} %, "
            f"{v.get('launch__registers_per_thread')} registers, grid {v.get('launch__grid_size')} x "
            f"{v.get('launch__block_size')}\n"
            "   busiest pipes (% of peak): " + ", ".join(f"{p} {x:.1f}" for p, x in pipes) + "\n"
            "   stalls per issue: " + ", ".join(
                f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
                f"{x:.2f}" for k, x in st) + "\n")
        if name == "headline":
            json.dump({"kernel": v.get("Kernel Name", "")[:120], "n": units, "dram_bytes_per_launch": rd + wr,
                       "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "source": f"profiles/{tag}_ncu_headline.csv (ncu --set full on bench.py --steps 1 "
                                 "--warmup 3 --no-e2e --no-cpu-baseline --no-next1..4 --no-configs, 4th launch)"},
                      open(os.path.join(P, "traffic.json"), "w"), indent=1)
    with open(os.path.join(P, f"{tag}_ncu_summary.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none captures (gpurun, B200), summarised by "
                "scripts/make_profiles_r02.py\n\n" + "\n".join(summary))
    print(open(os.path.join(P, f"{tag}_launch_shares.txt")).read())
    print("\n".join(summary))


if __name__ == "__main__":
    main()
