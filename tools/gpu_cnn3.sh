mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "not long_window and not full_batch" > gpurun_out/cnn_tc3.log 2>&1; echo cnn=$?; tail -2 gpurun_out/cnn_tc3.log
REPS=4 python tools/conv_prof.py c4 2>&1 | tail -2
REPS=4 DASMC_GPU_LIB=_exp/minb1.so python tools/conv_prof.py c4 2>&1 | tail -2
REPS=4 python tools/conv_prof.py c3 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4b.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 11 --launch-count 11 -o gpurun_out/conv_c4 -f python tools/conv_prof.py c4 > gpurun_out/ncu_conv.log 2>&1; echo ncu2=$?; tail -3 gpurun_out/ncu_conv.log
