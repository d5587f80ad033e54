# parity after the register-free prep loads; A/B gate-folded prep at 3 vs 4 blocks per SM
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -k "bitperm or prep or fold or gate or c4_bench or c3_sparse or c4_sparse or c2_sampled or default or upload" > gpurun_out/gbps.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/gbps.log; grep -E "^FAILED" gpurun_out/gbps.log | head -3
for v in 3 4 3 4; do TN_GATE_BPS=$v timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_gbps_$v.json > gpurun_out/steps_gbps_$v.txt 2>&1; echo bps=$v; head -1 gpurun_out/steps_gbps_$v.txt; done
