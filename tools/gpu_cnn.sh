mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -x -q -s -k "value_and_grad" > gpurun_out/cnn_tc1.log 2>&1; echo cnn1=$?; grep -E "tc cnn|passed|failed|Error|error" gpurun_out/cnn_tc1.log | head -30
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py tests/test_gpu_cnn.py -q -s > gpurun_out/cnn_tc2.log 2>&1; echo cnn2=$?; grep -E "passed|failed|Error|assert" gpurun_out/cnn_tc2.log | head -30
