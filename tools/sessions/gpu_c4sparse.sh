mkdir -p gpurun_out
timeout 900 python bench.py --boundary sparse16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4s16.json 2> gpurun_out/bench_c4s16.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c4s16.json')); print('C4s16', d['value'], d['ms_per_step'], json.dumps(d['kernel_stats'])); [print(t) for t in d['top_steps'][:8]]"
tail -3 gpurun_out/bench_c4s16.err
