"""Per-source-line totals of an `ncu --page source --print-source sass,cuda --csv`
export: thread instructions executed and stall samples, top N lines.
Usage: python tools/ncu_lines.py SRC.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
fname = None
head = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        head = r
        continue
    if head is None or len(r) != len(head) or not r[0].isdigit():
        continue
    ti = head.index("Thread Instructions Executed")
    ie = head.index("Instructions Executed")
    sm = head.index("Warp Stall Sampling (All Samples)")
    try:
        out.append((int(r[ti] or 0), int(r[ie] or 0), int(r[sm] or 0), fname, int(r[0]), r[1].strip()[:70]))
    except ValueError:
        pass
tot_t = sum(o[0] for o in out) or 1
tot_s = sum(o[2] for o in out) or 1
print(f"total thread instr {tot_t:.4g}, samples {tot_s}")
for t, i, s, f, ln, src in sorted(out, key=lambda o: -o[2])[:n_top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*t/tot_t:5.1f}% thr  thr/inst {t/max(i,1):5.1f}  {f}:{ln}  {src}")
