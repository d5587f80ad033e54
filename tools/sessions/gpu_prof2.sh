mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prep_gt -s 32 -c 1 -o gpurun_out/prof_gt python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gt.log 2>&1; echo gt_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny -s 104 -c 1 -o gpurun_out/prof_skinny2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_skinny2.log 2>&1; echo skinny_rc=$?
