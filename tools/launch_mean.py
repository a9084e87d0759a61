"""Mean duration (us) per kernel name of an ncu --metrics gpu__time_duration.sum --csv log."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
k, u, v = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
acc = collections.defaultdict(list)
for r in rows[1:]:
    acc[r[k].split("(")[0]].append(float(r[v].replace(",", "")) * scale.get(r[u], 1.0))
tag = sys.argv[2] if len(sys.argv) > 2 else ""
for name, xs in acc.items():
    tail = xs[len(xs) // 3:]  # skip the first frame
    print(f"{tag:10s} {name[:60]:60s} n={len(xs):3d} mean_us={sum(tail) / len(tail):9.2f}")
