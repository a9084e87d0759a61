mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ $v = default ]; then L="X=1"; else L="RTSDF_LIB=$PWD/variants/$v.so"; fi
  env $L timeout 300 python tools/jfa_time.py 512,512,512 big_sphere
  env $L timeout 300 python tools/jfa_time.py 1024,1024,1024 box_spheres
done
