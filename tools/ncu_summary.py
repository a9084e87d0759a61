"""Summarise an `ncu --set full` report of tools/frame.py into the per-kernel
CSV kept under profiles/ (one row per launch of the LAST frame):

    python tools/ncu_summary.py REPORT.ncu-rep|RAW.csv [first_kernel] > profiles/rNN_frame_kernels_summary.csv

(first_kernel: rows start at its LAST launch, default vox_ranges_kernel = the
start of the last frame)

Columns: time, warp instructions, threads per instruction (SIMD efficiency),
issue-active %, ALU / FMA / FP64 pipe %, DRAM MB read / written, achieved
occupancy %, registers, L2 hit rate."""
import csv
import io
import subprocess
import sys

COLS = [
    ("time[ms]", "gpu__time_duration.sum", 1e-6),  # ns -> ms
    ("inst", "smsp__inst_executed.sum", 1.0),
    ("thr/inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
    ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("alu%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    ("fma%", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1.0),
    ("fp64%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    ("dram_rd[MB]", "dram__bytes_read.sum", 1e-6),
    ("dram_wr[MB]", "dram__bytes_write.sum", 1e-6),
    ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("l2hit%", "lts__t_sector_hit_rate.pct", 1.0),
]
UNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
        "second": 1e9, "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep = sys.argv[1]
    first = sys.argv[2] if len(sys.argv) > 2 else "vox_ranges_kernel"
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    ki = head.index("Kernel Name")
    idx = {name: head.index(name) for _, name, _ in COLS if name in head}
    starts = [i for i, r in enumerate(data) if first in r[ki]]
    last = data[starts[-1]:] if starts else data
    out = csv.writer(sys.stdout)
    out.writerow(["kernel"] + [c for c, _, _ in COLS])
    for r in last:
        vals = []
        for col, name, scale in COLS:
            if name not in idx:
                vals.append("")
                continue
            v = r[idx[name]].replace(",", "")
            try:
                x = float(v) * UNIT.get(units[idx[name]], 1.0) * scale
            except ValueError:
                vals.append(v)
                continue
            vals.append(f"{x:.4f}" if abs(x) < 1e5 else f"{x:.0f}")
        name = r[ki].split("(")[0].replace("void ", "").replace("rtsdf::", "")
        out.writerow([name] + vals)


if __name__ == "__main__":
    main()
