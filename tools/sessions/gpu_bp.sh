mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -k "prep or default or c4 or c2" > gpurun_out/pytest_bp.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed" gpurun_out/pytest_bp.log | tail -2; grep -E "^FAILED|^E  " gpurun_out/pytest_bp.log | head -10
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_c4_bp.json > gpurun_out/steps_c4_bp.txt 2>&1; echo steps_rc=$?
head -30 gpurun_out/steps_c4_bp.txt
