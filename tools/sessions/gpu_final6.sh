# full GPU suite + smoke + default bench on the final code
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/final6_pytest.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/final6_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo bench_rc=$?
timeout 900 python bench.py --precision mixed --no-cpu-baseline > gpurun_out/final6_bench_mixed.json 2>> gpurun_out/final6_bench.err; echo mixed_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final6_ref.json 2>> gpurun_out/final6_bench.err; echo ref_rc=$?
