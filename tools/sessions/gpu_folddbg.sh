for env in "TN_FOLD_GATES=0" "TN_FOLD_GATES=0 TN_FUSE_PLANES=0" "TN_FOLD_GATES=0 TN_SIMT_VARIANT=1" "TN_FOLD_GATES=0 TN_SKINNY_VEC2=0" "TN_FOLD_GATES=0 TN_GRAPHS=0" "TN_FOLD_GATES=0 TN_PREP_FORCE=2"; do
  env $env timeout 300 python -m pytest tests -m gpu -q --timeout=200 -p no:cacheprovider -k "tc_folded" > gpurun_out/pf.log 2>&1
  echo "[$env] rc=$? $(tail -1 gpurun_out/pf.log) $(grep -o 'tc_folded-[a-z]*' gpurun_out/pf.log | sort -u | tr '\n' ' ')"
done
