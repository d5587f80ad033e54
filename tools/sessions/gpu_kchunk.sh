# GEMM drain study: pair kernel, 3-pass, kchunk sweep (TMEM drain vs MMA pacing), EW=16
mkdir -p gpurun_out; rm -f gpurun_out/kchunk.jsonl
for kc in 1 2 4 0; do
  TN_KCHUNK3=$kc timeout 120 python tools/gemm_bench.py 16384 16384 16384 --out gpurun_out/kchunk.jsonl > /dev/null 2>&1; echo "kc=$kc rc=$?"
done
TN_GEMM_EPI=16 TN_GEMM_PAIR_MIN_M=0 timeout 120 python tools/gemm_bench.py 16384 16384 16384 --out gpurun_out/kchunk.jsonl > /dev/null 2>&1
TN_GEMM_PAIR_MIN_M=0 timeout 120 python tools/gemm_bench.py 16384 16384 16384 --out gpurun_out/kchunk.jsonl > /dev/null 2>&1
timeout 120 python tools/gemm_bench.py 16384 16384 16384 --passes 1 --out gpurun_out/kchunk.jsonl > /dev/null 2>&1
cat gpurun_out/kchunk.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cgemm -s 1 -c 1 -o gpurun_out/prof_gemm_pair python tools/gemm_bench.py 16384 16384 16384 --reps 1 > gpurun_out/ncu_pair.log 2>&1; echo ncu_rc=$?
