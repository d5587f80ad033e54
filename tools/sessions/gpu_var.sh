mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider -k "simt or default" > gpurun_out/pv.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pv.log
for i in 1 2; do timeout 600 python tools/step_profile.py --workload c4 --slices 2 --out gpurun_out/steps_var_$i.json > gpurun_out/steps_var_$i.txt 2>&1; head -1 gpurun_out/steps_var_$i.txt; done
