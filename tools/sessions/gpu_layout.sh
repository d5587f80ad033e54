mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_gpu.log | tail -4; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -10
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_c4.json > gpurun_out/steps_c4.txt 2>&1; echo c4_rc=$?
head -30 gpurun_out/steps_c4.txt
timeout 600 python tools/step_profile.py --workload c3 --slices 2 --out gpurun_out/steps_c3.json > gpurun_out/steps_c3.txt 2>&1; echo c3_rc=$?
head -12 gpurun_out/steps_c3.txt
