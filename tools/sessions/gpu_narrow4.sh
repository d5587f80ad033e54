mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout=300 -p no:cacheprovider -k "cgemm or tc" > gpurun_out/pn4.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pn4.log; grep -E "^FAILED" gpurun_out/pn4.log | head -5
rm -f gpurun_out/narrow.jsonl
for nm in 1 0; do for shp in "33554432 64 32" "16777216 64 256" "2097152 64 1024" "8388608 32 256"; do
  TN_NARROW_MMA=$nm timeout 120 python tools/gemm_bench.py $shp --reps 3 --out gpurun_out/narrow.jsonl > /dev/null 2>&1
done; done
python - <<'PY'
import json
for l in open('gpurun_out/narrow.jsonl'):
    d=json.loads(l); print(d['m'],d['n'],d['k'], "ms=%.2f"%d['ms_per_launch'], "TF=%.1f"%d['tflops_useful'], "err=%.1e"%d['rel_l2_block'])
PY
for i in 1; do timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_nm.json > gpurun_out/steps_nm.txt 2>&1; head -1 gpurun_out/steps_nm.txt; done
