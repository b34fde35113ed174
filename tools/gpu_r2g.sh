# round-2 re-entry check: CNN TC tests first (latest conv_tc commits), then full suite, C2 + C4 bench, C4/C3 launch lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x > gpurun_out/t_cnn.log 2>&1; echo cnn_tests=$?; tail -1 gpurun_out/t_cnn.log; grep -E "^E " gpurun_out/t_cnn.log | head -8
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?
for f in bench_c2 bench_c4; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac', d['roofline']['frac'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c4.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/l_c4.csv 10
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3.csv python tools/conv_prof.py c3 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/l_c3.csv 10
