mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cnn_tc.py -q -x -s -k "value_and_grad" > gpurun_out/t_dir.log 2>&1; echo tests_main=$?; grep -E "tc cnn|passed|failed" gpurun_out/t_dir.log | head; grep -E "^E " gpurun_out/t_dir.log | head -5
DASMC_GPU_LIB=_exp/nobase.so timeout 600 python -m pytest tests/test_gpu_cnn_tc.py -q -x -s -k "value_and_grad" > gpurun_out/t_dir_nb.log 2>&1; echo tests_nobase=$?; grep -E "tc cnn|passed|failed" gpurun_out/t_dir_nb.log | head
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dir_c4.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/dir_c4.csv 6
DASMC_GPU_LIB=_exp/nobase.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dir_c4nb.csv python tools/conv_prof.py c4 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/dir_c4nb.csv 6
