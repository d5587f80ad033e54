# session r: B-slab-ordered final merge, swizzled gate-prep output tile: parity + step profiles (+ ncu of the gate prep)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:cacheprovider -x -k "fold or wdot or default or c4_sparse or c3" > gpurun_out/pytest_r.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_r.log; grep -E "^FAILED|^E  " gpurun_out/pytest_r.log | head
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_r.json > gpurun_out/steps_r.txt 2>&1; echo sp_rc=$?; head -1 gpurun_out/steps_r.txt; grep -E "^ *(217|235|384|207) " gpurun_out/steps_r.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_r_single.json > gpurun_out/steps_r_single.txt 2>&1; echo sp_rc=$?; head -1 gpurun_out/steps_r_single.txt; grep -E "^ *(356|358|338) " gpurun_out/steps_r_single.txt
