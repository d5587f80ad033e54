# A/B: evict-first (st.global.cs) GEMM output stores (TN_CS_STORE)
mkdir -p gpurun_out
TN_CS_STORE=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout=800 -p no:cacheprovider -k "cgemm or c4_bench or default" > gpurun_out/cs.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/cs.log
for v in 0 1 0 1; do TN_CS_STORE=$v timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_cs_$v.json > gpurun_out/steps_cs_$v.txt 2>&1; echo cs=$v; head -1 gpurun_out/steps_cs_$v.txt; done
