# one GPU session: build, a subset of the GPU tests ($TESTS, -k $KSEL), then same-box A/B step
# profiles of the headline slice: default (A) vs $AB_ENV_B (B), alternating A B A
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
if [ -n "$KSEL" ]; then
  timeout ${PYT_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -m gpu -q --timeout=900 -p no:cacheprovider -s -k "$KSEL" > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$?
  grep -E "sub-network|sub-slice|passed|failed" gpurun_out/pytest_ab.log | tail -6; grep -E "^FAILED|^E  " gpurun_out/pytest_ab.log | head -20
fi
P="tools/step_profile.py --workload c4 --boundary ${BOUNDARY:-sparse16} --peak 32 --slices 2"
timeout 600 python $P --out gpurun_out/steps_A.json > gpurun_out/steps_A.txt 2>&1
env $AB_ENV_B timeout 600 python $P --out gpurun_out/steps_B.json > gpurun_out/steps_B.txt 2>&1
timeout 600 python $P --out gpurun_out/steps_A2.json > gpurun_out/steps_A2.txt 2>&1
env $AB_ENV_B timeout 600 python $P --out gpurun_out/steps_B2.json > gpurun_out/steps_B2.txt 2>&1
head -1 gpurun_out/steps_A.txt gpurun_out/steps_B.txt gpurun_out/steps_A2.txt gpurun_out/steps_B2.txt
python tools/ab_compare.py ms 2>/dev/null | head -30
