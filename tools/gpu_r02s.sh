# session s: ncu (source-level) of the short-K output-heavy GEMMs 218 and 217 on the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for sk in "218 22" "217 21"; do set -- $sk
  timeout 600 ncu --profile-from-start off -k regex:cgemm --launch-skip $2 --launch-count 1 --set full --import-source on -o gpurun_out/ncu_s$1 python tools/ncu_step.py --boundary sparse16 --peak 32 --step $1 > gpurun_out/ncu_s$1.log 2>&1; echo "ncu $1 rc=$?"; grep "launches before" gpurun_out/ncu_s$1.log
done
