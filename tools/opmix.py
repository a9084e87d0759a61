"""Opcode mix of one kernel launch from `ncu --page source --print-source sass --csv`:
executed thread instructions per output cell by opcode, and the split over the
ALU / FMA(IMAD) pipes.  Usage: python tools/opmix.py SASS.csv N_CELLS [title]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cells = float(sys.argv[2])
title = sys.argv[3] if len(sys.argv) > 3 else ""
head = None
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "Address":
        head = r
        continue
    if head is None or len(r) != len(head):
        continue
    src = r[head.index("Source")].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    t = r[head.index("Thread Instructions Executed")]
    if t and t.isdigit():
        cnt[op.split(".")[0]] += int(t)
tot = sum(cnt.values())
ALU = {"ISETP", "VIMNMX", "IMNMX", "LOP3", "SHF", "IADD3", "SEL", "LEA", "VIADD", "PLOP3", "P2R", "R2P",
       "FMNMX", "PRMT", "VIADDMNMX", "FSEL", "MOV"}
FMA = {"IMAD", "IMUL", "FFMA", "FADD", "FMUL"}
alu = sum(v for k, v in cnt.items() if k in ALU)
fma = sum(v for k, v in cnt.items() if k in FMA)
print(f"{title}\nthread instructions per cell: {tot / cells:.1f}  (ALU pipe {alu / cells:.1f}, "
      f"FMA pipe {fma / cells:.1f}, other {(tot - alu - fma) / cells:.1f})")
for op, v in cnt.most_common(25):
    print(f"  {op:12s} {v / cells:8.2f} per cell  {100.0 * v / tot:5.1f} %")
