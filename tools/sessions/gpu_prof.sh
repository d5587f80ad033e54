# focused ncu captures of one prep launch and one skinny launch of the bench workload
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prep -s 86 -c 1 -o gpurun_out/prof_prep python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_prep.log 2>&1; echo prep_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny -s 107 -c 1 -o gpurun_out/prof_skinny python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_skinny.log 2>&1; echo skinny_rc=$?
