mkdir -p gpurun_out; rm -f gpurun_out/kchunk2.jsonl
timeout 300 python -m pytest tests -m gpu -q -x --timeout=200 -p no:cacheprovider -k "cgemm" > gpurun_out/pytest_cg.log 2>&1; echo cgemm_rc=$?; tail -1 gpurun_out/pytest_cg.log
for kc in 1 2 0; do
  TN_KCHUNK3=$kc timeout 120 python tools/gemm_bench.py 16384 16384 16384 --out gpurun_out/kchunk2.jsonl > /dev/null 2>&1
done
TN_GEMM_PAIR_MIN_M=0 timeout 120 python tools/gemm_bench.py 16384 16384 16384 --out gpurun_out/kchunk2.jsonl > /dev/null 2>&1
timeout 120 python tools/gemm_bench.py 16384 16384 16384 --passes 1 --out gpurun_out/kchunk2.jsonl > /dev/null 2>&1
cut -c1-200 gpurun_out/kchunk2.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cgemm -s 1 -c 1 -o gpurun_out/prof_gemm_pair2 python tools/gemm_bench.py 16384 16384 16384 --reps 1 > gpurun_out/ncu_pair2.log 2>&1; echo ncu_rc=$?
