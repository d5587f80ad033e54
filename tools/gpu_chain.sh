# chain session: tests of the fused skinny chains, same-box A/B (TN_CHAIN=0 as B), headline bench
KSEL="chains or sparse_state or c4_bench or default" AB_ENV_B="TN_CHAIN=0" bash tools/gpu_ab.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
