mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_bench_window.py tests/test_gpu_graphs.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/t_l2.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_l2.log; grep -E "^E " gpurun_out/t_l2.log | head -5
python tools/tune_fwd.py --precision f16x2 --rounds 3 --steps 3 "LIB=_exp/oldsplit.so" "DASMC_X=1" "DASMC_DEBUG_EPI=3" "DASMC_DEBUG_EPI=1" "PREC=f16" "PREC=f16 LIB=_exp/oldsplit.so" "PREC=tf32h" "PREC=tf32h LIB=_exp/oldsplit.so" > gpurun_out/ab_l2.log 2>&1; tail -9 gpurun_out/ab_l2.log
