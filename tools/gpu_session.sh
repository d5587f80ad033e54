mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "C4 sub-slice|passed|failed" gpurun_out/pytest_gpu.log | tail -3; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -8
rm -f gpurun_out/gemm_sweep.jsonl
for kc in 1 2 4 0; do TN_KCHUNK3=$kc timeout 120 python tools/gemm_bench.py 8192 8192 16384 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1; done
for gr in 1 8 32; do TN_GEMM_GROUP=$gr timeout 120 python tools/gemm_bench.py 8192 8192 16384 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1; done
timeout 120 python tools/gemm_bench.py 8192 8192 16384 --passes 1 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1
timeout 120 python tools/gemm_bench.py 32768 16384 16384 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1
cat gpurun_out/gemm_sweep.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', d['value'], d['ms_per_step'], d['roofline']['achieved'], json.dumps(d['kernel_stats']))"
tail -2 gpurun_out/bench.err
