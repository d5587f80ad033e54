# narrow (HBM-bound) GEMM shapes: achieved bytes/s of operands (planes) + output
mkdir -p gpurun_out; rm -f gpurun_out/narrow.jsonl
for shp in "33554432 64 32" "16777216 64 256" "33554432 128 128" "8388608 256 32" "16777216 128 32"; do
  timeout 120 python tools/gemm_bench.py $shp --reps 3 --out gpurun_out/narrow.jsonl > /dev/null 2>&1; echo "$shp rc=$?"
done
python - <<'PY'
import json
for l in open('gpurun_out/narrow.jsonl'):
    d=json.loads(l); m,n,k=d['m'],d['n'],d['k']
    by=8*(m*k+n*k+m*n); t=d['ms_per_launch']/1e3
    print(m,n,k, "ms=%.2f"%(t*1e3), "GB/s=%.0f"%(by/t/1e9), "TF=%.1f"%d['tflops_useful'])
PY
