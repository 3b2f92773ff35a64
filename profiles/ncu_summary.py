"""Summarise an ncu --set full report (exported with `ncu -i X.ncu-rep --page raw --csv`)
into the handful of counters the design notes cite.  Usage: ncu_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
keys = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("==", r[col["Kernel Name"]][:80])
    for k in keys:
        if k in col:
            print(f"   {k:66s} {r[col[k]]:>16s} {units[col[k]]}")
    top = sorted(((float(r[col[s]] or 0), s) for s in stalls), reverse=True)[:6]
    print("   stalls (warps per issue):", ", ".join(
        f"{s.split('stalled_')[1].replace('_per_issue_active.ratio', '')}={v:.2f}" for v, s in top))
