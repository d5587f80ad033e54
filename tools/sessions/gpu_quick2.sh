mkdir -p gpurun_out
bash tools/gpu_quick.sh
timeout 900 python tools/topk_sweep.py gpurun_out/topk_sweep.json > gpurun_out/topk.log 2>&1; echo topk_rc=$?; tail -3 gpurun_out/topk.log
