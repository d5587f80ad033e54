# launch list of the final code (same command as tools/gpu_session.sh)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v8.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph-pass > gpurun_out/ncu_bench_v8.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/launches_v8.csv > gpurun_out/launches_v8_summary.txt 2>&1; head -30 gpurun_out/launches_v8_summary.txt
