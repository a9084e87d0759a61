mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"wf_pass" --launch-skip 2 --launch-count 2 -o /tmp/rt python tools/frame.py --frames 2 > gpurun_out/rtprof_ncu.log 2>&1
ncu -i /tmp/rt.ncu-rep --page raw --csv > gpurun_out/rtprof_raw.csv
ncu -i /tmp/rt.ncu-rep --page source --csv --print-source sass,cuda --kernel-name regex:wf_pass1 > gpurun_out/rtprof_p1.csv 2>/dev/null
ncu -i /tmp/rt.ncu-rep --page source --csv --print-source sass,cuda --kernel-name regex:wf_pass2 > gpurun_out/rtprof_p2.csv 2>/dev/null
ls -la gpurun_out/rtprof*
