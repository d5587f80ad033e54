mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider -s -k "simt or sparse_state or default or c2" > gpurun_out/pytest_bsk.log 2>&1; echo pytest_rc=$?
grep -E "sub-network|passed|failed" gpurun_out/pytest_bsk.log | tail -4; grep -E "^FAILED|^E  " gpurun_out/pytest_bsk.log | head -6
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step']); [print(t) for t in d['top_steps'][:5]]"
timeout 600 python bench.py --workload c3 --peak 30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('C3', d['value'], d['ms_per_step'])"
