# round-2 checkpoint: full GPU suite, smoke, bench lines (headline C4-sparse16, C4 single, mixed, C5),
# ncu launch list of one steady headline slice, ncu --set full of its dominant GEMM (step 131)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_final.log; grep -E "^FAILED|^E  " gpurun_out/pytest_final.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?; tail -2 gpurun_out/bench_final.err
timeout 900 python bench.py --boundary single --no-cpu-baseline > gpurun_out/bench_final_single.json 2>/dev/null; echo rc=$?
timeout 900 python bench.py --precision mixed --no-cpu-baseline > gpurun_out/bench_final_mixed.json 2>/dev/null; echo rc=$?
timeout 900 python bench.py --workload c5 --boundary single --steps 5 --no-cpu-baseline > gpurun_out/bench_final_c5.json 2>/dev/null; echo rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_final_reference.json 2>/dev/null; echo rc=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/ncu_step.py --boundary sparse16 --peak 32 > gpurun_out/ncu_launch_final.log 2>&1; echo ncul_rc=$?
timeout 900 ncu --profile-from-start off -k regex:cgemm --launch-skip 12 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_gemm131 python tools/ncu_step.py --boundary sparse16 --peak 32 --step 131 > gpurun_out/ncu_gemm131.log 2>&1; echo ncu_rc=$?
