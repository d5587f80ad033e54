# session g: staged row stores + cached column tables in the GEMM epilogue: parity + step profile
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -m gpu -q --timeout=600 -p no:cacheprovider -x > gpurun_out/pytest_g.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_g.log; grep -E "^FAILED|^E  " gpurun_out/pytest_g.log | head -20
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_g.json > gpurun_out/steps_g.txt 2>&1; echo sp_rc=$?; head -16 gpurun_out/steps_g.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_g_single.json > gpurun_out/steps_g_single.txt 2>&1; echo sp_rc=$?; head -16 gpurun_out/steps_g_single.txt
