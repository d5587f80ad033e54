# DRAM traffic of the top GEMM shape vs tile-rasterization group (ncu metrics, one launch each)
mkdir -p gpurun_out; rm -f gpurun_out/dram_group.txt
for g in 1 2 4 8 16 64; do
  TN_GEMM_GROUP=$g timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second -k regex:cgemm -s 1 -c 1 --csv python tools/gemm_bench.py 32768 16384 16384 --reps 1 > gpurun_out/dram_g$g.csv 2>&1
  echo "group $g" >> gpurun_out/dram_group.txt; grep -E "dram__bytes_read|time_duration|hit_rate|per_second" gpurun_out/dram_g$g.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/dram_group.txt
done
cat gpurun_out/dram_group.txt
