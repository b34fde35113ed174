mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_cnn_tc.py -q -x > gpurun_out/t_r2d.log 2>&1; echo tests=$?; tail -3 gpurun_out/t_r2d.log; grep -E "^E " gpurun_out/t_r2d.log | head -10
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4e.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3e.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-graphs > gpurun_out/bench_c1ng.log 2>&1; echo c1ng=$?
for f in bench_c4 bench_c1 bench_c1ng; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['ms_per_step'], d['value'], d['gpu_launches'])"; done
