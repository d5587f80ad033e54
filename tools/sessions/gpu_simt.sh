# SIMT kernel rework: SIMT parity routes, full parity suite, per-step profile, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > gpurun_out/pytest_simt.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_simt.log | tail -2; grep -E "^FAILED|^E  " gpurun_out/pytest_simt.log | head -10
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_c4_simt.json > gpurun_out/steps_c4_simt.txt 2>&1; echo steps_rc=$?
head -1 gpurun_out/steps_c4_simt.txt; grep simt gpurun_out/steps_c4_simt.txt | head -16
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('EXT', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
