"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
the kernels of the last frame (second half of the list) with their times."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
out = [(r[ki].split("(")[0][:60], float(r[vi].replace(",", "")) * scale[r[ui]]) for r in rows[1:]]
half = out[len(out) // 2:] if len(sys.argv) < 3 else out
for n, t in half:
    print(f"{t:8.4f} ms  {n}")
print(f"total {sum(t for _, t in half):.3f} ms over {len(half)} launches")
