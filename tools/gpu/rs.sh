mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then L="X=1"; else L="RTSDF_LIB=$PWD/variants/$v.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KREGEX" --csv --log-file /tmp/l_$v.csv python tools/frame.py --frames 3 > /tmp/o_$v.log 2>&1 || tail -3 /tmp/o_$v.log
  python tools/launch_mean.py /tmp/l_$v.csv $v || true
done
