# A/B: HBM-bound GEMMs on single-CTA 16-epilogue-warp tiles (TN_GEMM_EPI16_MAXK)
mkdir -p gpurun_out
TN_GEMM_EPI16_MAXK=256 timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -k "cgemm or tc or default or c4" > gpurun_out/pe16.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pe16.log; grep -E "^FAILED" gpurun_out/pe16.log | head -3
for mk in 0 256; do for shp in "33554432 128 128" "33554432 64 32" "1024 2097152 128" "2097152 64 1024"; do
  TN_GEMM_EPI16_MAXK=$mk timeout 120 python tools/gemm_bench.py $shp --reps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('maxk=$mk', d['m'],d['n'],d['k'],'ms=%.2f'%d['ms_per_launch'],'err=%.1e'%d['rel_l2_block'])"
done; done
for mk in 0 256 0 256; do TN_GEMM_EPI16_MAXK=$mk timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_e16_$mk.json > gpurun_out/steps_e16_$mk.txt 2>&1; echo maxk=$mk; head -1 gpurun_out/steps_e16_$mk.txt; done
