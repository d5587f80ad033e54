mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -s > gpurun_out/pytest_fold.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_fold.log | tail -5; grep -E "^FAILED|^E  " gpurun_out/pytest_fold.log | head -10
AB_ENV_B=TN_FOLD_GATES=0 bash tools/gpu_ab.sh
