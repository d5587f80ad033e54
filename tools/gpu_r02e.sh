# session e: ncu full of the output-heavy / narrow GEMMs of C4 sparse16 p32 (steps 321, 218, 269)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for sk in "321 38" "218 21" "269 29"; do set -- $sk
  timeout 600 ncu --profile-from-start off -k regex:cgemm --launch-skip $2 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_gemm$1 python tools/ncu_step.py --boundary sparse16 --peak 32 --step $1 > gpurun_out/ncu_gemm$1.log 2>&1; echo "ncu $1 rc=$?"; head -1 gpurun_out/ncu_gemm$1.log
done
