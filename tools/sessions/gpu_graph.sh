mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > gpurun_out/pytest_graph.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_graph.log | tail -1; grep -E "^FAILED|^E  " gpurun_out/pytest_graph.log | head -10
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('C2', d['value'], d['ms_per_step'], d['cuda_graph'], d['gpu_launches'])"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'], d['cuda_graph'])"
tail -3 gpurun_out/bench.err
