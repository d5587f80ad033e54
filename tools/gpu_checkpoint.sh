# checkpoint session: build, full GPU suite, smoke, bench (headline + secondary lines), launch list of one
# steady headline slice, ncu --set full of the jobs in $NCU_JOBS (see tools/gpu_ncu.sh)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu.log; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>/dev/null; echo "bench reference rc=$?"
for extra in "--boundary single" "--precision mixed" "--workload c5 --boundary single --steps 5" "--order-tag a64b1 --steps 5"; do
  tag=$(echo $extra | tr -d ' -' | cut -c1-24)
  timeout 900 python bench.py $extra --no-cpu-baseline > gpurun_out/bench_$tag.json 2>/dev/null; echo "bench $tag rc=$?"
done
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps.json > gpurun_out/steps.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/ncu_step.py --boundary sparse16 --peak 32 > gpurun_out/ncu_launch.log 2>&1; echo ncul_rc=$?
[ -n "$NCU_JOBS" ] && bash tools/gpu_ncu.sh
