mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_dist.py tests/test_gpu_cnn_tc.py tests/test_gpu_parity.py -q -x > gpurun_out/t_r2c.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_r2c.log; grep -E "^E |Error" gpurun_out/t_r2c.log | head -10
python tools/membench.py --config c2 > gpurun_out/membench_c2.json 2>&1; tail -1 gpurun_out/membench_c2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 11 --launch-count 11 -o gpurun_out/conv_c4d -f python tools/conv_prof.py c4 > gpurun_out/ncu_conv.log 2>&1; echo ncu2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -c 300 gpurun_out/bench_c4.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo c1=$?; tail -c 300 gpurun_out/bench_c1.log
