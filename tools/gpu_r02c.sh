# session c: new wdotj + precision formats parity; A/B step profiles on C4 sparse16 p32
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests/test_gpu_precision.py tests/test_gpu_parity.py -m gpu -q --timeout=600 -p no:cacheprovider -k "precision or fig4 or scaled or wdot or cgemm or gemm" > gpurun_out/pytest_c.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_c.log; grep -E "^FAILED|^E  " gpurun_out/pytest_c.log | head -30
timeout 600 python tools/precision_study.py --k 16384 --out gpurun_out/precision_study.json > gpurun_out/precision.txt 2>&1; echo prec_rc=$?; cat gpurun_out/precision.txt
for v in default fold0 wave256; do
  case $v in default) E="";; fold0) E="TN_FOLD_GATES=0";; wave256) E="TN_WAVE_MIN_K=256";; esac
  env $E timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_$v.json > gpurun_out/steps_$v.txt 2>&1; echo "$v rc=$?"; head -12 gpurun_out/steps_$v.txt
done
