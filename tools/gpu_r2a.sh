# round 2, first check: build state, bench-window parity, smoke, GPU tests, bench (f16x2 default, tf32h), reference arm
set -x
mkdir -p gpurun_out
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python -m pytest tests/test_gpu_bench_window.py -x -q -s > gpurun_out/pytest_window.log 2>&1; echo window=$?; tail -15 gpurun_out/pytest_window.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --precision tf32h --no-cpu > gpurun_out/bench_tf32h.log 2>&1; tail -1 gpurun_out/bench_tf32h.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
