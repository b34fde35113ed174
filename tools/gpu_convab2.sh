mkdir -p gpurun_out
for v in main nospin; do
  lib=""; [ $v = nospin ] && lib="DASMC_GPU_LIB=_exp/nospin.so"
  for dbg in 0 7; do
    env $lib DASMC_CONV_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab2_${v}_$dbg.csv python tools/conv_prof.py c4 > /dev/null 2>&1
    echo "== $v dbg $dbg"; python tools/launch_summary.py gpurun_out/ab2_${v}_$dbg.csv 4
  done
done
