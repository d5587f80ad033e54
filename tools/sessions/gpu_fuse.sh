mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -s > gpurun_out/pytest_w.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_w.log | tail -3; grep -E "^FAILED|^E  " gpurun_out/pytest_w.log | head -10
AB_ENV_B=TN_WAVE_SYNC=0 bash tools/gpu_ab.sh
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'], d['cuda_graph']['ms_per_step'])"
