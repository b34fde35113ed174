# round-end style check: smoke, GPU tests, default bench, f16 bench line, reference arm, launch list
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --precision f16 --no-cpu > gpurun_out/bench_f16.log 2>&1; tail -1 gpurun_out/bench_f16.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_torchrun.log 2>&1; echo torchrun=$?; tail -1 gpurun_out/bench_torchrun.log
