mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -s -k "simt or sparse_state or default" > gpurun_out/pytest_wd.log 2>&1; echo pytest_rc=$?
grep -E "sub-network|passed|failed" gpurun_out/pytest_wd.log | tail -4; grep -E "^FAILED|^E  " gpurun_out/pytest_wd.log | head -6
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step']); [print(t) for t in d['top_steps'][:6]]"
