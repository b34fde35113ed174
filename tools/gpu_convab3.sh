mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "not full_batch and not long_window" > gpurun_out/t_ab3.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_ab3.log; grep -E "^E " gpurun_out/t_ab3.log | head
for dbg in 0 7; do
  DASMC_CONV_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab3_$dbg.csv python tools/conv_prof.py c4 > /dev/null 2>&1
  echo "== dbg $dbg"; python tools/launch_summary.py gpurun_out/ab3_$dbg.csv 5
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab3_c3.csv python tools/conv_prof.py c3 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/ab3_c3.csv 5
