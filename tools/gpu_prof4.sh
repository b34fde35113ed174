# final-build launch list (default bench) + ncu --set full of the f16-mode forward, summarised on the box
set -x
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
mkdir -p /tmp/prof
ncu --set full --clock-control none -k regex:tc_kernel -s 6 -c 1 -o /tmp/prof/f16 -f $B --precision f16 > gpurun_out/ncu_f16.log 2>&1; echo f16=$?
python tools/ncu_summary.py full /tmp/prof/f16.ncu-rep gpurun_out/ncu_f16.json "ncu --set full --clock-control none -k regex:tc_kernel -s 6 -c 1 $B --precision f16"
