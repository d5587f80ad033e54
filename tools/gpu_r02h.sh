# session h: narrow GEMMs with split epilogue halves (4 TMEM buffers): parity + step profiles + narrow ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -m gpu -q --timeout=600 -p no:cacheprovider -x > gpurun_out/pytest_h.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_h.log; grep -E "^FAILED|^E  " gpurun_out/pytest_h.log | head -20
timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_h.json > gpurun_out/steps_h.txt 2>&1; echo sp_rc=$?; head -1 gpurun_out/steps_h.txt; grep -E "^ *(269|207|208|201|130) " gpurun_out/steps_h.txt
timeout 600 python tools/step_profile.py --workload c4 --boundary single --peak 32 --slices 2 --out gpurun_out/steps_h_single.json > gpurun_out/steps_h_single.txt 2>&1; echo sp_rc=$?; head -1 gpurun_out/steps_h_single.txt; grep -E "^ *(356|188|368|184|187) " gpurun_out/steps_h_single.txt
timeout 600 ncu --profile-from-start off -k regex:cgemm --launch-skip 29 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_h269 python tools/ncu_step.py --boundary sparse16 --peak 32 --step 269 > gpurun_out/ncu_h269.log 2>&1; echo ncu_rc=$?
