# every BASELINE config through bench.py (1 GPU) + the GPU test suite
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | cut -c1-300; done
