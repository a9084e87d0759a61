#!/bin/bash
# Round profile on the GPU box (writes only small files under gpurun_out/):
#   1. launch list of 3 C3 frames (ncu gpu__time_duration, cold/serialised)
#   2. ncu --set full of the LAST of 2 frames, exported as per-kernel raw CSV
#      + SASS source CSVs of the JFA dense pass and the sampler passes
# usage: bash tools/profile_round.sh TAG
set -e
TAG=${1:-r2}
OUT=gpurun_out
python tools/frame.py --frames 3 > $OUT/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches_raw.csv python tools/frame.py --frames 3 > /dev/null 2>&1
# launches of the first frame = where the second vox_ranges_kernel starts (of a 2-frame run)
SKIP=$(python - "$OUT/${TAG}_launches_raw.csv" <<'PY'
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
ki = rows[0].index("Kernel Name")
names = [r[ki] for r in rows[1:]]
firsts = [i for i, n in enumerate(names) if n.startswith("vox_ranges_kernel")]
print(firsts[1] if len(firsts) > 1 else 0)
PY
)
echo "skip $SKIP" > $OUT/${TAG}_skip.txt
ncu --set full --clock-control none --import-source on -s $SKIP -o /tmp/${TAG}_frame \
    python tools/frame.py --frames 2 > $OUT/${TAG}_ncu_full.log 2>&1
ncu -i /tmp/${TAG}_frame.ncu-rep --page raw --csv > $OUT/${TAG}_frame_raw.csv
for K in jfa_pass2_kernel wf_pass1_kernel wf_pass2_kernel; do
  ncu -i /tmp/${TAG}_frame.ncu-rep --page source --csv --print-source sass --kernel-name regex:$K \
      --launch-skip 0 --launch-count 1 > $OUT/${TAG}_${K}_sass.csv 2>/dev/null || true
done
ls -la $OUT
