mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -s -k "prep or default or c4 or c2 or tc" > gpurun_out/pytest_bp2.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_bp2.log | tail -3; grep -E "^FAILED|^E  " gpurun_out/pytest_bp2.log | head -5
for i in 1 2; do timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_bp2_$i.json > gpurun_out/steps_bp2_$i.txt 2>&1; head -1 gpurun_out/steps_bp2_$i.txt; done
