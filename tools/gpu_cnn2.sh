mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -s > gpurun_out/cnn_tc2.log 2>&1; echo cnn2=$?; grep -E "M=2100|passed|failed|^E " gpurun_out/cnn_tc2.log | head -20
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -c 1500 gpurun_out/bench_c4.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3=$?; tail -c 1500 gpurun_out/bench_c3.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1; echo ncu=$?
timeout 900 python bench.py --config c4fb --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/bench_c4fb.log 2>&1; echo c4fb=$?; tail -c 1500 gpurun_out/bench_c4fb.log
