mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -k "jfa or flood or golden or frame" > gpurun_out/j5_test.log 2>&1; echo "rc=$?" >> gpurun_out/j5_test.log
for v in default $VARIANTS; do
  if [ $v = default ]; then timeout 120 python tools/jfa_time.py; else RTSDF_LIB=$PWD/variants/$v.so timeout 120 python tools/jfa_time.py; fi
done > gpurun_out/j5_time.log 2>&1
tail -3 gpurun_out/j5_test.log; cat gpurun_out/j5_time.log
