# A/B: promotion interval (TN_KCHUNK3) on the HBM-bound narrow GEMMs + whole slice
mkdir -p gpurun_out
for kc in 1 2 4; do for shp in "33554432 128 128" "1024 2097152 128" "8192 8192 4096"; do
  TN_KCHUNK3=$kc timeout 120 python tools/gemm_bench.py $shp --reps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('kc=$kc', d['m'],d['n'],d['k'],'ms=%.2f'%d['ms_per_launch'],'err=%.2e'%d['rel_l2_block'])"
done; done
for kc in 1 4; do TN_KCHUNK3=$kc timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_kc_$kc.json > gpurun_out/steps_kc_$kc.txt 2>&1; echo kc=$kc; head -1 gpurun_out/steps_kc_$kc.txt; done
