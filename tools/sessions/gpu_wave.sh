mkdir -p gpurun_out; rm -f gpurun_out/wave.jsonl gpurun_out/dram_wave.txt
timeout 300 python -m pytest tests -m gpu -q -x --timeout=200 -p no:cacheprovider -k "cgemm" > gpurun_out/pyt_w.log 2>&1; echo cgemm_rc=$?; tail -1 gpurun_out/pyt_w.log
for ws in 1 0; do for g in 8 1; do
  TN_WAVE_SYNC=$ws TN_GEMM_GROUP=$g timeout 120 python tools/gemm_bench.py 32768 16384 16384 --reps 3 --out gpurun_out/wave.jsonl > /dev/null 2>&1
  TN_WAVE_SYNC=$ws TN_GEMM_GROUP=$g timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second -k regex:cgemm -s 1 -c 1 --csv python tools/gemm_bench.py 32768 16384 16384 --reps 1 > gpurun_out/dw.csv 2>&1
  echo "ws=$ws g=$g" >> gpurun_out/dram_wave.txt; grep -E "dram__bytes_read|time_duration|per_second" gpurun_out/dw.csv | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/dram_wave.txt
done; done
cut -c1-150 gpurun_out/wave.jsonl; cat gpurun_out/dram_wave.txt
