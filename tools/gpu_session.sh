# one GPU session: build, the GPU test files given in $TESTS (default all), bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout ${PYT_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q --timeout=900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_gpu.log | tail -5; grep -E "^FAILED|^E  " gpurun_out/pytest_gpu.log | head -20
