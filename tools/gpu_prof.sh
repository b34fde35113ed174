# launch list + ncu --set full captures of the top kernels of the default bench (run on the GPU box)
set -x
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:'tc_kernel<(int)[01],' -s 3 -c 3 -o gpurun_out/tc_full -f $B > gpurun_out/ncu_tc.log 2>&1; echo tcfull=$?
ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel|split_w1' -s 6 -c 8 -o gpurun_out/mem_full -f $B > gpurun_out/ncu_mem.log 2>&1; echo memfull=$?
ls -la gpurun_out
