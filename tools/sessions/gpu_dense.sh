mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -s -k "dense or sparse_state or default or cgemm" > gpurun_out/pytest_dense.log 2>&1; echo pytest_rc=$?
grep -E "sub-network|passed|failed" gpurun_out/pytest_dense.log | tail -4; grep -E "^FAILED|^E  " gpurun_out/pytest_dense.log | head -10
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step'], json.dumps(d['kernel_stats'])); [print(t) for t in d['top_steps'][:8]]"
