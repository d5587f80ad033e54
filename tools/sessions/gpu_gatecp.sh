# A/B: gate-folded prep loads through cp.async (TN_GATE_CPASYNC) vs register rounds
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -k "fold or gate or c4_bench or c3_sparse or c2_sampled or default" > gpurun_out/gcp.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/gcp.log; grep -E "^FAILED" gpurun_out/gcp.log | head -3
for v in 0 1 0 1; do TN_GATE_CPASYNC=$v timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_gcp_$v.json > gpurun_out/steps_gcp_$v.txt 2>&1; echo cpa=$v; head -1 gpurun_out/steps_gcp_$v.txt; done
