# session p: L2 evict_last operand loads + streaming row stores: parity + A/B step profiles (same box)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:cacheprovider -x -k "cgemm or default or tc_pair or tc_grouped" > gpurun_out/pytest_p.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_p.log
for v in 1 0 1 0; do
  TN_GEMM_L2HINT=$v timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_p$v.json > gpurun_out/steps_p$v.txt 2>&1; echo "l2hint=$v"; head -1 gpurun_out/steps_p$v.txt; grep -E "^ *(131|217|218|321|233) " gpurun_out/steps_p$v.txt
done
