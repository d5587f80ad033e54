mkdir -p gpurun_out
python tools/fold_debug.py 2>&1 | cat
TN_FOLD_GATES=1 timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_A.json > gpurun_out/steps_A.txt 2>&1
timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_B.json > gpurun_out/steps_B.txt 2>&1
TN_FOLD_GATES=1 timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_A2.json > gpurun_out/steps_A2.txt 2>&1
head -1 gpurun_out/steps_A.txt gpurun_out/steps_B.txt gpurun_out/steps_A2.txt
