mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -s -k "tc_folded or default or c4_bench or c2" > gpurun_out/pf4.log 2>&1; echo rc=$?; grep -E "sub-slice|passed|failed" gpurun_out/pf4.log | tail -2
AB_ENV_B=TN_FOLD_GATES=0 bash tools/gpu_ab.sh
