# session k: ncu of the gate-folded prep of C4-single step 356 (A side, 2^32 elements, N=K=8)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 600 ncu --profile-from-start off -k regex:prep_gate --launch-skip 37 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_gate356 python tools/ncu_step.py --boundary single --peak 32 --step 356 > gpurun_out/ncu_gate356.log 2>&1; echo ncu_rc=$?; head -2 gpurun_out/ncu_gate356.log
