# one GPU session: parity tests, bench (extended + mixed + C2 + C3 + C4-sparse), launch list, ncu of the top GEMM
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_gpu.log | tail -5; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -8
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'], d['cuda_graph']['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --steps 5 --warmup 3 --precision mixed --no-cpu-baseline > gpurun_out/bench_mixed.json 2> gpurun_out/bench_mixed.err; echo mixed_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_mixed.json')); print('MIX', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('C2', d['value'], d['ms_per_step'], d['cuda_graph']['ms_per_step'])"
timeout 600 python bench.py --workload c3 --peak 30 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('C3', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo c4s_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph-pass > gpurun_out/ncu_bench.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm -s ${TOPGEMM:-74} -c 1 -o gpurun_out/prof_gemm_top python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph-pass > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
