# session q: short-K promotion interval A/B (TN_KCHUNK3_SHORT 1 vs 2 vs 4) on time and C4 / C5 sub-slice error
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for v in 1 2 4 1 2; do
  TN_KCHUNK3_SHORT=$v timeout 600 python tools/step_profile.py --workload c4 --boundary sparse16 --peak 32 --slices 2 --out gpurun_out/steps_q$v.json > gpurun_out/steps_q$v.txt 2>&1; echo "kchunk_short=$v"; head -1 gpurun_out/steps_q$v.txt; grep -E "^ *(217|218|321|383) " gpurun_out/steps_q$v.txt
done
for v in 1 2; do TN_KCHUNK3_SHORT=$v TAG=k$v timeout 600 python tools/c5_debug.py 2>&1 | tail -1; done
for v in 1 2; do TN_KCHUNK3_SHORT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=900 -p no:cacheprovider -k "c4_bench or c4_sparse" -s 2>&1 | grep -E "sub-slice|sub-network"; done
