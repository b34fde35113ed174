set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python tools/membench.py --config c2 > gpurun_out/membench_c2.json 2>&1; cat gpurun_out/membench_c2.json
python tools/membench.py --config c5 > gpurun_out/membench_c5.json 2>&1; cat gpurun_out/membench_c5.json
python tools/membench.py --config c2 --J 16384 > gpurun_out/membench_c2_16k.json 2>&1; cat gpurun_out/membench_c2_16k.json
ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel' -c 4 -o gpurun_out/membench_full -f python tools/membench.py --config c2 --reps 1 > gpurun_out/ncu_membench.log 2>&1; echo ncumem=$?
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu"
ncu --set full --import-source on --clock-control none -k regex:tc_kernel -s 6 -c 3 -o gpurun_out/tc_full -f $B > gpurun_out/ncu_tc.log 2>&1; echo tcfull=$?
