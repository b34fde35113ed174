mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py tests/test_gpu_cnn.py tests/test_gpu_parity.py -q -x > gpurun_out/t_r2b.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_r2b.log
python tools/membench.py --config c2 > gpurun_out/membench_c2.json 2>&1; tail -1 gpurun_out/membench_c2.json
python tools/membench.py --config c5 > gpurun_out/membench_c5.json 2>&1; tail -1 gpurun_out/membench_c5.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4c.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3c.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -c 700 gpurun_out/bench_c4.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3=$?; tail -c 700 gpurun_out/bench_c3.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo c1=$?; tail -c 400 gpurun_out/bench_c1.log
