mkdir -p gpurun_out
for dbg in 0 1 2 4 3 7; do
  DASMC_CONV_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$dbg.csv python tools/conv_prof.py c4 > /dev/null 2>&1
  echo "== dbg $dbg"; python tools/launch_summary.py gpurun_out/ab_$dbg.csv 4
done
