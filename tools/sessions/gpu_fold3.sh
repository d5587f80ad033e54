mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout=300 -p no:cacheprovider -k "tc_folded or default" > gpurun_out/pf3.log 2>&1; echo rc=$?; tail -1 gpurun_out/pf3.log
AB_ENV_B=TN_FOLD_GATES=1 bash tools/gpu_ab.sh
