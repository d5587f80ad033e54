# session o: ncu of the headline's dominant GEMM (step 131) for roofline traffic; skinny SIMT steps 346/348 (C4 single)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 ncu --profile-from-start off -k regex:cgemm --launch-skip 13 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_gemm131 python tools/ncu_step.py --boundary sparse16 --peak 32 --step 131 > gpurun_out/ncu_gemm131.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --profile-from-start off -k regex:einsum_skinny --launch-skip 65 --launch-count 2 --set full --import-source on -o gpurun_out/ncu_skinny346 python tools/ncu_step.py --boundary single --peak 32 --step 346 > gpurun_out/ncu_skinny.log 2>&1; echo ncu2_rc=$?
