mkdir -p gpurun_out
bash tools/gpu_quick.sh
rm -f gpurun_out/gemm_sweep.jsonl
for ew in 8 16; do TN_GEMM_EPI=$ew timeout 120 python tools/gemm_bench.py 8192 8192 16384 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1; TN_GEMM_EPI=$ew timeout 120 python tools/gemm_bench.py 32768 16384 16384 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1; done
cat gpurun_out/gemm_sweep.jsonl
