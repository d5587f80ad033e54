mkdir -p gpurun_out
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_c4.json > gpurun_out/steps_c4.txt 2>&1; echo c4_rc=$?
timeout 600 python tools/step_profile.py --workload c3 --slices 2 --out gpurun_out/steps_c3.json > gpurun_out/steps_c3.txt 2>&1; echo c3_rc=$?
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --precision mixed --out gpurun_out/steps_c4_mixed.json > gpurun_out/steps_c4_mixed.txt 2>&1; echo c4m_rc=$?
head -45 gpurun_out/steps_c4.txt
