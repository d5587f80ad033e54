# session j: epilogue exponent split + smem address space fix: C5 diagnosis, parity, profiles
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for e in "TAG=default" "TAG=simt TN_DISABLE_TC=1" "TAG=unfused TN_FUSE_PLANES=0 TN_FOLD_GATES=0"; do env $e timeout 600 python tools/c5_debug.py 2>&1 | tail -1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py tests/test_gpu_runtime.py tests/test_gpu_precision.py -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/pytest_j.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_j.log; grep -E "^FAILED|^E  " gpurun_out/pytest_j.log | head -20
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_j.json > gpurun_out/steps_j.txt 2>&1; echo sp_rc=$?; head -14 gpurun_out/steps_j.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_j_single.json > gpurun_out/steps_j_single.txt 2>&1; echo sp_rc=$?; head -1 gpurun_out/steps_j_single.txt
