mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -q -x --timeout=300 -p no:cacheprovider -k "cgemm or tc" > gpurun_out/pyt_n.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pyt_n.log
rm -f gpurun_out/narrow.jsonl
for shp in "33554432 64 32" "16777216 64 256" "33554432 128 128" "8388608 256 32"; do
  timeout 120 python tools/gemm_bench.py $shp --reps 3 --out gpurun_out/narrow.jsonl > /dev/null 2>&1
done
python - <<'PY'
import json
for l in open('gpurun_out/narrow.jsonl'):
    d=json.loads(l); m,n,k=d['m'],d['n'],d['k']
    by=8*(m*k+n*k+m*n); t=d['ms_per_launch']/1e3
    print(m,n,k, "ms=%.2f"%(t*1e3), "GB/s=%.0f"%(by/t/1e9), "TF=%.1f"%d['tflops_useful'], "err=%.1e"%d['rel_l2_block'])
PY
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_N.json > gpurun_out/steps_N.txt 2>&1; head -1 gpurun_out/steps_N.txt
