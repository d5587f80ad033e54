# end-to-end parity error vs promotion interval (TN_KCHUNK3)
mkdir -p gpurun_out
for kc in 1 2 4; do
  TN_KCHUNK3=$kc timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s --timeout=800 -p no:cacheprovider -k "c4_bench or c2_sampled or c3_sparse or c4_sparse or c1_vs" > gpurun_out/kc2_$kc.log 2>&1; echo kc=$kc rc=$?; grep -iE "rel_l2|passed|failed|error" gpurun_out/kc2_$kc.log | head -12
done
