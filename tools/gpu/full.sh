mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python bench.py --no-cpu --steps 20 > gpurun_out/bench_head.log 2>&1
tail -3 gpurun_out/gputest.log
tail -1 gpurun_out/bench_head.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['frame_stages_ms'], d['jfa']['ms'], d['jfa']['per_pass_ms'])"
