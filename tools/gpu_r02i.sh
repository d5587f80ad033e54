# session i: tensor throughput of N=64 (narrow, CTA pair) vs N=128 MMAs at large K (3M feasibility)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for shp in "65536 128 16384" "65536 64 16384" "131072 64 8192" "65536 128 8192"; do
  for p in 3 1; do timeout 300 python tools/gemm_bench.py $shp --passes $p --reps 5 --out gpurun_out/gemm_n64.jsonl; done
done
cat gpurun_out/gemm_n64.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=900 -p no:cacheprovider -k "c5 or c3 or c4_sparse or c2 or lxeb or c4_bench" -s > gpurun_out/pytest_i.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed|^E  " gpurun_out/pytest_i.log | head -20
