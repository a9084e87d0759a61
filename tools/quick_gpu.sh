mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "jfa or frame or pipeline" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --steps 10 > gpurun_out/bench2.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1]);print(d['value'],d['frame_stages_ms'],d['jfa']['per_pass_ms'],d['jfa']['ms'])"
