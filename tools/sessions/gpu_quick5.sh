# grouped sparse merges: targeted tests, C3 bench, full GPU suite, C4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout=800 -p no:cacheprovider -s -k "grouped or c3" > gpurun_out/pytest_grouped.log 2>&1; echo grouped_rc=$?
grep -E "sub-network|passed|failed" gpurun_out/pytest_grouped.log | tail -3; grep -E "^FAILED|^E  " gpurun_out/pytest_grouped.log | head -8
timeout 600 python bench.py --workload c3 --peak 30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('C3', d['value'], d['ms_per_step'], json.dumps(d['kernel_stats']))"
tail -3 gpurun_out/bench_c3.err
bash tools/gpu_quick.sh
