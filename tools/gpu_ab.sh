# same-box A/B of per-step times: $AB_ENV_B (variant B) vs default (A)
mkdir -p gpurun_out
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_A.json > gpurun_out/steps_A.txt 2>&1
env ${AB_ENV_B:-TN_SIMT_OLD=1} timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_B.json > gpurun_out/steps_B.txt 2>&1
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_A2.json > gpurun_out/steps_A2.txt 2>&1
head -1 gpurun_out/steps_A.txt gpurun_out/steps_B.txt gpurun_out/steps_A2.txt
