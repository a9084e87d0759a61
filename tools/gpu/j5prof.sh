mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"jfa_pass|jfa_fixup" -o /tmp/j5 python tools/jfa_once.py > gpurun_out/j5prof_ncu.log 2>&1
ncu -i /tmp/j5.ncu-rep --page raw --csv > gpurun_out/j5prof_raw.csv
ncu -i /tmp/j5.ncu-rep --page details --csv > gpurun_out/j5prof_details.csv
ncu -i /tmp/j5.ncu-rep --page source --csv --print-source sass --kernel-name regex:jfa_pass5 --launch-skip 7 --launch-count 1 > gpurun_out/j5prof_sass.csv 2>/dev/null
ls -la gpurun_out
