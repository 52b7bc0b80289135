"""Key counters of an ncu raw-page CSV (one kernel): python scripts/raw_summary.py raw.csv [n_segments]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nseg = float(sys.argv[2]) if len(sys.argv) > 2 else 1e9
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("==", d.get("Kernel Name", "?")[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    for k in keys:
        print(f"   {k:70s} {d.get(k)}")
    if d.get("smsp__inst_executed.sum"):
        print(f"   thread-inst/segment {32 * float(d['smsp__inst_executed.sum']) / nseg:.1f}")
    st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled")
          and k.endswith("per_issue_active.ratio") and v not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    for k, v in st[:9]:
        print(f"   {v:7.3f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
