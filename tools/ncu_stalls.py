"""Per-launch summary of an ncu raw CSV: time, warp instructions, issue %,
occupancy, pipe utilisation and the top stall reasons (per issue-active).
Usage: python tools/ncu_stalls.py RAW.csv [kernel-regex]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[0], rows[2:]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
want = {"ms": "gpu__time_duration.sum", "inst": "smsp__inst_executed.sum",
        "thr": "smsp__thread_inst_executed_per_inst_executed.ratio",
        "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "alu%": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma%": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread", "dramMB": "dram__bytes_read.sum"}
stall = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
ki = h.index("Kernel Name")
for r in data:
    if pat and not pat.search(r[ki]):
        continue
    vals = {k: r[h.index(v)] for k, v in want.items() if v in h}
    vals["ms"] = "%.4f" % (float(vals["ms"]) * 1e-6)
    top = sorted(((float(r[h.index(n)] or 0), n[34:-23]) for n in stall), reverse=True)[:5]
    print(r[ki][:44], " ".join(f"{k}={v}" for k, v in vals.items()))
    print("    stalls:", ", ".join(f"{b} {a:.2f}" for a, b in top))
