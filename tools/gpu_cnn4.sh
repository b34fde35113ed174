mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x -s -k "not full_batch" > gpurun_out/cnn_tc4.log 2>&1; echo cnn=$?; grep -E "tc cnn|M=2100|passed|failed|^E " gpurun_out/cnn_tc4.log | head -20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4c.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3c.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -c 900 gpurun_out/bench_c4.log
