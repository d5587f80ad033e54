# round-2 validation: build, full GPU suite, smoke, default bench and the sparse16 p30 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
timeout 900 python bench.py --boundary sparse16 --peak 30 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s16p30.json 2> gpurun_out/bench_s16p30.err; echo rc=$?; tail -c 1500 gpurun_out/bench_s16p30.json; tail -5 gpurun_out/bench_s16p30.err
