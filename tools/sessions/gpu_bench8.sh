mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b8.json 2> gpurun_out/b8.err; echo bench_rc=$?
timeout 900 python bench.py --precision mixed --no-cpu-baseline > gpurun_out/b8_mixed.json 2>> gpurun_out/b8.err; echo mixed_rc=$?
