# session d: parity of the changed SIMT/gate kernels, step profile C4 sparse16 p32, gate-prep ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py -m gpu -q --timeout=600 -p no:cacheprovider -x > gpurun_out/pytest_d.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_d.log; grep -E "^FAILED|^E  " gpurun_out/pytest_d.log | head -20
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_d.json > gpurun_out/steps_d.txt 2>&1; echo sp_rc=$?; head -25 gpurun_out/steps_d.txt
timeout 600 ncu --profile-from-start off -k regex:prep_gate --launch-skip 10 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_gate217 python tools/ncu_step.py --boundary sparse16 --peak 32 --step 217 > gpurun_out/ncu_gate.log 2>&1; echo ncu_rc=$?; tail -2 gpurun_out/ncu_gate.log
