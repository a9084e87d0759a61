# per-kernel launch means of 3 C3 frames + bench line for each library variant
# usage: VARIANTS="a b" KREGEX="wf_pass|fixup" bash tools/gpu/varq.sh
mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then L="X=1"; else L="RTSDF_LIB=$PWD/variants/$v.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_$v.csv python tools/frame.py --frames 3 > /dev/null 2>&1
  python tools/launch_mean.py gpurun_out/v_$v.csv $v | grep -iE "${KREGEX:-wf_pass}"
done
bash tools/gpu/benchvar.sh
