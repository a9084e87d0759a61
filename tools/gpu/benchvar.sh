for v in default $VARIANTS; do
  if [ $v = default ]; then L="X=1"; else L="RTSDF_LIB=$PWD/variants/$v.so"; fi
  env $L timeout 300 python bench.py --no-cpu --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'], d['frame_stages_ms'])"
done
