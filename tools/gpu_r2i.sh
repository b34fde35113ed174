# round-2 re-entry baseline: full GPU suite, smoke, benches of every config, launch lists
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1; echo c5=$?
for f in bench_c2 bench_c4 bench_c3 bench_c1 bench_c5; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac', d['roofline']['frac'], d['config'].get('window_rows'))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c4.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/l_c4.csv 12
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/l_c3.csv 12
