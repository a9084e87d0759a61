# Round-end evidence on one B200: GPU test suite, bench lines (ours + the
# reference arm), launch list + full ncu capture of a C3 frame.
# usage: bash tools/gpu/final.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
tail -2 gpurun_out/${TAG}_gputest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.jsonl
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1; tail -1 gpurun_out/${TAG}_bench_ref.log > gpurun_out/${TAG}_bench_reference.jsonl
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench.jsonl').read()); print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'])"
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_reference.jsonl').read()); print('ref', d['value'])"
timeout 1200 bash tools/profile_round.sh $TAG > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"
python tools/ncu_summary.py gpurun_out/${TAG}_frame_raw.csv > gpurun_out/${TAG}_frame_kernels_summary.csv 2>gpurun_out/${TAG}_summary.err; echo "summary rc=$?"
