# session f: parity of the small-K tensor-core route; reorder ablation (TN_REORDER 0/1/2) step profiles; bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:cacheprovider -k "small_k or reorder or default" > gpurun_out/pytest_f.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_f.log; grep -E "^FAILED|^E  " gpurun_out/pytest_f.log | head -20
for r in 2 1 0; do
  TN_REORDER=$r timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_reorder$r.json > gpurun_out/steps_reorder$r.txt 2>&1; echo "reorder $r rc=$?"; head -1 gpurun_out/steps_reorder$r.txt
done
for r in 2 1 0; do
  TN_REORDER=$r timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_single_reorder$r.json > gpurun_out/steps_single_reorder$r.txt 2>&1; echo "single reorder $r rc=$?"; head -1 gpurun_out/steps_single_reorder$r.txt
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo bench_rc=$?; tail -3 gpurun_out/bench_f.err
