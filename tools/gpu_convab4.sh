mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "not full_batch and not long_window" > gpurun_out/t_ab4.log 2>&1; echo tests=$?; tail -1 gpurun_out/t_ab4.log
for v in main pw4; do
  lib=""; [ $v = pw4 ] && lib="DASMC_GPU_LIB=_exp/pw4.so"
  env $lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab4_$v.csv python tools/conv_prof.py c4 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/ab4_$v.csv 5
done
