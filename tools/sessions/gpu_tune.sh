mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > gpurun_out/pytest_tune.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_tune.log | tail -1; grep -E "^FAILED|^E  " gpurun_out/pytest_tune.log | head -10
AB_ENV_B=TN_AUTOTUNE=0 bash tools/gpu_ab.sh
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
