mkdir -p gpurun_out
python tools/fuse_check.py
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -s > gpurun_out/pytest_fuse.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_fuse.log | tail -3; grep -E "^FAILED|^E  " gpurun_out/pytest_fuse.log | head -10
AB_ENV_B=TN_FUSE_PLANES=0 bash tools/gpu_ab.sh
