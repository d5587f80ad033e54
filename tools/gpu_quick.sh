mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_s16.json 2> gpurun_out/b_s16.err; echo rc=$?
timeout 900 python tools/step_profile.py --workload c4 --boundary sparse16 --slices 2 --out gpurun_out/steps_s16.json > gpurun_out/steps_s16.txt 2>&1; echo rc=$?
head -45 gpurun_out/steps_s16.txt
