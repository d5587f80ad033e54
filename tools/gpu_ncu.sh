# ncu --set full of one kernel launch of a steady headline slice: $NCU_JOBS = "name:kernel_regex:step ..."
# (launch-skip from tools/ncu_step.py's count of that kernel family's launches before the step)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
for job in $NCU_JOBS; do
  name=${job%%:*}; rest=${job#*:}; kre=${rest%%:*}; step=${rest#*:}
  skip=$(TN_GRAPHS=0 timeout 600 python tools/ncu_step.py --boundary ${BOUNDARY:-sparse16} --step $step 2>/dev/null | \
         sed -n "s/.*${kre%%_*} launches before it: \([0-9]*\).*/\1/p" | head -1)
  [ -z "$skip" ] && skip=0
  if [ "$kre" = "prep_gate" ]; then skip=$(TN_GRAPHS=0 timeout 600 python tools/ncu_step.py --boundary ${BOUNDARY:-sparse16} --step $step 2>/dev/null | sed -n "s/.*prep_gate launches before it: \([0-9]*\).*/\1/p" | head -1); fi
  echo "job $name: kernel $kre step $step skip $skip"
  timeout 900 ncu --profile-from-start off -k regex:$kre --launch-skip $skip --launch-count 1 --set full \
      --import-source on --clock-control none -o gpurun_out/ncu_$name -f \
      python tools/ncu_step.py --boundary ${BOUNDARY:-sparse16} --step $step > gpurun_out/ncu_$name.log 2>&1; echo ncu_rc=$?
  # summaries travel back (gpurun_out is capped at 64 MiB): raw metrics + per-line stalls
  ncu -i gpurun_out/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/ncu_$name.ncu-rep 40 > gpurun_out/ncu_${name}_lines.txt 2>&1
  [ -z "$KEEP_REP" ] && rm -f gpurun_out/ncu_$name.ncu-rep
done
