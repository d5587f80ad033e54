# session n: staged plane (cols mode) stores: parity + step profiles
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -m gpu -q --timeout=900 -p no:cacheprovider -k "not c5" > gpurun_out/pytest_n.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_n.log; grep -E "^FAILED|^E  " gpurun_out/pytest_n.log | head -10
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_n.json > gpurun_out/steps_n.txt 2>&1; echo sp_rc=$?; head -10 gpurun_out/steps_n.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_n_single.json > gpurun_out/steps_n_single.txt 2>&1; echo sp_rc=$?; head -10 gpurun_out/steps_n_single.txt
