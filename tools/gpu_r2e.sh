mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x > gpurun_out/t_r2e.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_r2e.log; grep -E "^E " gpurun_out/t_r2e.log | head -10
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4f.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3f.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c1 --precision fp32 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1fp32.log 2>&1; echo c1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --no-graphs --e2e-steps 1 > /dev/null 2>&1; echo ncu3=$?
for f in bench_c4 bench_c3 bench_c1fp32; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['ms_per_step'], d['value'], d['config']['window_rows'])"; done
