# CTA-pair GEMM: unit tests (bounded), GEMM sweep pair vs single, C4 bench
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x --timeout=120 -p no:cacheprovider -k "cgemm" > gpurun_out/pytest_pair.log 2>&1; echo cgemm_rc=$?
grep -E "passed|failed" gpurun_out/pytest_pair.log | tail -2; grep -E "^FAILED|^E  " gpurun_out/pytest_pair.log | head -10
rm -f gpurun_out/gemm_pair.jsonl
for pm in 0 1; do
  for shp in "8192 8192 16384" "32768 16384 16384" "2048 8192 16384"; do
    TN_GEMM_PAIR_MIN_M=$pm timeout 120 python tools/gemm_bench.py $shp --out gpurun_out/gemm_pair.jsonl > /dev/null 2>&1; echo "pm=$pm $shp rc=$?"
  done
  TN_GEMM_PAIR_MIN_M=$pm timeout 120 python tools/gemm_bench.py 8192 8192 16384 --passes 1 --out gpurun_out/gemm_pair.jsonl > /dev/null 2>&1
done
cat gpurun_out/gemm_pair.jsonl
