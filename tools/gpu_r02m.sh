# session m: tensor-core gate prep parity + timing; C5 precision diagnosis
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:cacheprovider -x -k "fold or c4_bench or c4_sparse or c3 or default or tc" > gpurun_out/pytest_m.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_m.log; grep -E "^FAILED|^E  " gpurun_out/pytest_m.log | head -10
for e in "TAG=default" "TAG=simt TN_DISABLE_TC=1" "TAG=gate_ffma TN_GATE_MMA=0" "TAG=nofold TN_FOLD_GATES=0 TN_FUSE_PLANES=0"; do env $e timeout 600 python tools/c5_debug.py 2>&1 | tail -2; done
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_m.json > gpurun_out/steps_m.txt 2>&1; echo sp_rc=$?; head -8 gpurun_out/steps_m.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_m_single.json > gpurun_out/steps_m_single.txt 2>&1; echo sp_rc=$?; head -8 gpurun_out/steps_m_single.txt
