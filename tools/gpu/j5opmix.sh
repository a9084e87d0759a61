mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"jfa_pass5" --launch-skip 5 --launch-count 1 -o /tmp/p5 python tools/jfa_once.py > gpurun_out/p5_ncu.log 2>&1
ncu -i /tmp/p5.ncu-rep --page raw --csv > gpurun_out/p5_raw.csv
ncu -i /tmp/p5.ncu-rep --page source --csv --print-source sass > gpurun_out/p5_sass.csv 2>/dev/null
ls -la gpurun_out/p5*
