mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu --config c1"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c1.csv $B > gpurun_out/ncu_l_c1.log 2>&1; echo l_c1=$?; python tools/launch_summary.py gpurun_out/launches_c1.csv 30
