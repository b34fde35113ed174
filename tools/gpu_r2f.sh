# round-2 checkpoint: full GPU suite, smoke, default bench (driver command), reference arm, per-config benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_c2.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-graphs > gpurun_out/bench_c1ng.log 2>&1; echo c1ng=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo c3=$?
python tools/membench.py --config c2 > gpurun_out/membench_c2.json 2>&1
python tools/membench.py --config c5 > gpurun_out/membench_c5.json 2>&1
for f in bench_c2 bench_c1 bench_c1ng bench_c5 bench_c4 bench_c3; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); cb=d.get('cpu_baseline') or {}; print('$f', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac', d['roofline']['frac'], 'cpu', cb.get('value'), d['config']['window_rows'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1; echo ncu=$?
