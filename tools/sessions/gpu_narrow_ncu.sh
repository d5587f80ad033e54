# ncu capture of the C4 step-356 GEMM (m = 2^25, n = 128, k = 128; HBM-bound) + standalone timing
mkdir -p gpurun_out
timeout 600 python tools/gemm_bench.py 33554432 128 128 --reps 3 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm -s 42 -c 1 -o gpurun_out/prof_g356 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph-pass > gpurun_out/ncu_g356.log 2>&1; echo ncu_rc=$?
