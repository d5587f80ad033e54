# session t: bench lines of the balanced (App. A.2) order and the peak-2^30 order on the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python bench.py --order-tag a64b1 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_b1.json 2>/dev/null; echo rc=$?
timeout 900 python bench.py --peak 30 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_p30.json 2>/dev/null; echo rc=$?
timeout 900 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_a64.json 2>/dev/null; echo rc=$?
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_t.json > gpurun_out/steps_t.txt 2>&1; head -1 gpurun_out/steps_t.txt
