# ncu sections for the SIMT einsum kernels of one C4 slice
mkdir -p gpurun_out
timeout 1200 ncu --clock-control none --section SpeedOfLight --section Occupancy --section WarpStateStats --section LaunchStats --section MemoryWorkloadAnalysis -k regex:einsum_ -o gpurun_out/prof_simt python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_simt.log 2>&1; echo ncu_rc=$?
