"""Summarise an .ncu-rep (run here): per kernel launch, time, DRAM bytes, instructions,
issue activity, occupancy and the top warp-stall reasons.
  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [n_segments]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("smsp__inst_executed.sum", "warp_inst"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("sm__cycles_elapsed.avg.per_second", "sm_clk"), ("launch__grid_size", "grid"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%")]


def main():
    rep = sys.argv[1]
    nseg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print("==", d.get("Kernel Name", "?")[:90])
        for k, nm in KEYS:
            print(f"   {nm:10s} {d.get(k)} {u.get(k, '')}")
        if nseg and d.get("smsp__inst_executed.sum"):
            print(f"   thread-inst/segment {32 * float(d['smsp__inst_executed.sum']) / nseg:.1f}")
        st = [(k, float(v or 0)) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
        st.sort(key=lambda kv: -kv[1])
        print("   stalls:", ", ".join(f"{k[34:-29]}={v:.2f}" for k, v in st[:7]))


if __name__ == "__main__":
    main()
