# round-2 session b: build, full GPU suite (12-warp setmaxnreg GEMM, reorder routes),
# sparse16 p32 bench + step profile, ncu of step 217's GEMM and the slice launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -30
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s16p32.json 2> gpurun_out/bench_s16p32.err; echo bench_rc=$?; tail -5 gpurun_out/bench_s16p32.err
timeout 900 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_s16p32.json > gpurun_out/steps_s16p32.txt 2>&1; echo sp_rc=$?; head -30 gpurun_out/steps_s16p32.txt
timeout 900 ncu --profile-from-start off -k regex:cgemm --launch-skip 20 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_s16_step217 python tools/ncu_step.py --boundary sparse16 --peak 32 --step 217 > gpurun_out/ncu217.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu217.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s16p32.csv python tools/ncu_step.py --boundary sparse16 --peak 32 > gpurun_out/ncu_launch.log 2>&1; echo ncul_rc=$?
