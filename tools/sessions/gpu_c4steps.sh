mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print('C4', d['value'], d['ms_per_step'], json.dumps(d['kernel_stats']))
for s in d['top_steps']: print(s)"
tail -3 gpurun_out/bench_c4.err
