mkdir -p gpurun_out
bash tools/gpu_quick.sh
timeout 900 python tools/topk_sweep.py gpurun_out/topk_sweep.json > gpurun_out/topk.log 2>&1; echo topk_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/topk_sweep.json'))
for r in d['rows']: print('k=%3d ratio %.3f rel_time %.3f ms %.1f rel_l2 %.2e eps %.2e' % (r['k'], r['tcc_ratio'], r['relative_time'], r['ms_per_slice'], r['rel_l2'], r['eps_l2sq']))"
rm -f gpurun_out/gemm_sweep.jsonl
timeout 120 python tools/gemm_bench.py 8192 8192 16384 --passes 1 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1
TN_KCHUNK1=0 timeout 120 python tools/gemm_bench.py 8192 8192 16384 --passes 1 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1
TN_KCHUNK1=8 timeout 120 python tools/gemm_bench.py 8192 8192 16384 --passes 1 --out gpurun_out/gemm_sweep.jsonl > /dev/null 2>&1
cat gpurun_out/gemm_sweep.jsonl
