mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_all.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_all.log | tail -5; grep -E "^FAILED|^E  " gpurun_out/pytest_all.log | head -6
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step']); [print(t) for t in d['top_steps'][:5]]"
