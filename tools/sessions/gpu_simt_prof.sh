mkdir -p gpurun_out
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:einsum_wide -c 12 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph-pass > gpurun_out/wide_list.csv 2>&1; echo rc=$?
grep -E "gpu__time_duration|dram__bytes_write" gpurun_out/wide_list.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160
