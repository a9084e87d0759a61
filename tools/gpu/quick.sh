# bench line + per-kernel launch times of 2 C3 frames + the ray / sampler GPU tests
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/q_bench.log 2>&1
tail -1 gpurun_out/q_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['e2e']['value'], d['frame_stages_ms'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python tools/frame.py --frames 3 > /dev/null 2>&1
python tools/launch_mean.py gpurun_out/q_launches.csv 2>/dev/null | grep -i "wf_pass\|jfa_pass5\|occlusion"
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-bvh or ray or sampl or frame or rng}" > gpurun_out/q_tests.log 2>&1; tail -2 gpurun_out/q_tests.log
