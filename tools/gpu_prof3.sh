# GPU tests, memory-kernel microbench, and ncu captures summarised ON the box
# (reports are large; only the JSON/CSV summaries come back)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for a in "--config c2" "--config c5" "--config c2 --J 16384"; do python tools/membench.py $a; done > gpurun_out/membench.jsonl 2>&1; cat gpurun_out/membench.jsonl
mkdir -p /tmp/prof
ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel|slot_sum' -c 6 -o /tmp/prof/mem -f python tools/membench.py --config c2 --reps 1 > gpurun_out/ncu_membench.log 2>&1; echo ncumem=$?
python tools/ncu_summary.py full /tmp/prof/mem.ncu-rep gpurun_out/ncu_mem.json "ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel|slot_sum' -c 6 python tools/membench.py --config c2 --reps 1"
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu"
ncu --set full --import-source on --clock-control none -k regex:tc_kernel -s 6 -c 3 -o /tmp/prof/tc -f $B > gpurun_out/ncu_tc.log 2>&1; echo tcfull=$?
python tools/ncu_summary.py full /tmp/prof/tc.ncu-rep gpurun_out/ncu_tc.json "ncu --set full --import-source on --clock-control none -k regex:tc_kernel -s 6 -c 3 $B"
ncu -i /tmp/prof/tc.ncu-rep --page source --csv --print-source sass > /tmp/prof/src.csv 2>/dev/null; echo src=$?
gzip -c /tmp/prof/src.csv > gpurun_out/tc_src.csv.gz; ls -la gpurun_out
