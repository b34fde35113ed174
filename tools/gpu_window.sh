mkdir -p gpurun_out
DASMC_REPORT_ONLY=1 timeout 1200 python -m pytest tests/test_gpu_bench_window.py -q -s > gpurun_out/pytest_window.log 2>&1; echo window=$?; grep -E "^(f16x2|tf32h|3xtf32|tf32|f16|fp32) " gpurun_out/pytest_window.log; tail -2 gpurun_out/pytest_window.log
