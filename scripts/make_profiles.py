"""Turn a round's raw gpurun captures into the tracked profiles/ summaries.

  python scripts/make_profiles.py <tag> <bench.json> <launches.csv> <full.ncu-rep> [n]

writes profiles/<tag>_bench.json, profiles/<tag>_launches.csv (+ a share table in
profiles/<tag>_launch_shares.txt), profiles/<tag>_ncu_compact_full.csv and
profiles/traffic.json (DRAM bytes per launch of the compacting kernel, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct", "sm__warps_active.avg.pct", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "gpu__dram_throughput.avg.pct", "lts__t_bytes.sum", "smsp__average_warps_issue_stalled",
        "launch__shared_mem_per_block"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    tag, bench, launches, rep = sys.argv[1:5]
    n = int(sys.argv[5]) if len(sys.argv) > 5 else 10**9
    os.makedirs(P, exist_ok=True)
    shutil.copy(bench, os.path.join(P, f"{tag}_bench.json"))
    shutil.copy(launches, os.path.join(P, f"{tag}_launches.csv"))
    rows = [r for r in csv.reader(open(launches)) if r and not r[0].startswith("==")]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) == len(h) and r[ix["Metric Name"]] == "gpu__time_duration.sum":
            agg[r[ix["Kernel Name"]].split("(")[0][:90]].append(float(r[ix["Metric Value"]]))
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(P, f"{tag}_launch_shares.txt"), "w") as f:
        f.write("launches  total_us  share  kernel\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{len(v):8d} {sum(v) / 1e3:9.1f} {100 * sum(v) / tot:5.1f}%  {k}\n")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    h, u, d = rr[0], dict(zip(rr[0], rr[1])), dict(zip(rr[0], rr[2]))
    with open(os.path.join(P, f"{tag}_ncu_compact_full.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        for k in h:
            if any(k.startswith(p) for p in KEEP):
                w.writerow([k, u.get(k, ""), d[k]])
    rd = float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
    json.dump({"kernel": d.get("Kernel Name", "clip_compact_kernel")[:120], "n": n, "dram_bytes_per_launch": rd + wr,
               "dram_read_bytes": rd, "dram_write_bytes": wr,
               "source": f"profiles/{tag}_ncu_compact_full.csv (ncu --set full on bench.py --steps 3 --warmup 3 "
                         "--no-e2e --no-cpu-baseline, 4th compacting launch)"},
              open(os.path.join(P, "traffic.json"), "w"), indent=1)
    print(open(os.path.join(P, f"{tag}_launch_shares.txt")).read())
    print("traffic", rd + wr)


if __name__ == "__main__":
    main()
