# usage: KREGEX=... ENVS="A=1 A=2" bash tools/gpu/envsweep.sh
mkdir -p gpurun_out
for e in $ENVS; do
  env $e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KREGEX" --csv --log-file /tmp/l_$e.csv python tools/frame.py --frames 3 > /tmp/o_$e.log 2>&1 || tail -3 /tmp/o_$e.log
  python tools/launch_mean.py /tmp/l_$e.csv $e || true
done
