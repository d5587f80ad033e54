# tests + bench (extended, mixed) + launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_gpu.log | tail -4; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -8
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], json.dumps(d['kernel_stats']))"
timeout 600 python bench.py --steps 5 --warmup 3 --precision mixed --no-cpu-baseline > gpurun_out/bench_mixed.json 2> gpurun_out/bench_mixed.err; echo mixed_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_mixed.json')); print('MIX', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu1_rc=$?
