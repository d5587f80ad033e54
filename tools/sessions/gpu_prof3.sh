mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prep_gt -s 69 -c 1 -o gpurun_out/prof_gt3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gt3.log 2>&1; echo gt_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny2 -s 77 -c 1 -o gpurun_out/prof_sk3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sk3.log 2>&1; echo sk_rc=$?
timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('C3', d['value'], d['ms_per_step'], json.dumps(d['kernel_stats']))"
tail -2 gpurun_out/bench_c3.err
