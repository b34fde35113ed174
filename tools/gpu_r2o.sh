mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "batching_tail" > gpurun_out/t_tail.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_tail.log; grep -E "^E " gpurun_out/t_tail.log | head -8
