# round-2 evidence run: full GPU suite, smoke, every config's bench line, the reference arm, launch
# lists and ncu --set full summaries (summarised on the box; only JSON / CSV comes back)
mkdir -p gpurun_out /tmp/prof
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log; grep -E "^(FAILED|ERROR)" $O/pytest_gpu.log | head
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo ref=$?; tail -1 $O/bench_ref.log | cut -c1-400
timeout 600 python bench.py > $O/bench_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > $O/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 > $O/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > $O/bench_c4.log 2>&1; echo c4=$?
timeout 1500 python bench.py --config c4fb --steps 1 --warmup 1 --e2e-steps 1 --no-cpu > $O/bench_c4fb.log 2>&1; echo c4fb=$?; tail -1 $O/bench_c4fb.log | cut -c1-300
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > $O/bench_c5.log 2>&1; echo c5=$?
for f in bench_c2 bench_c1 bench_c3 bench_c4 bench_c5; do tail -1 $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac', round(d['roofline']['frac'],4), d['config'].get('window_rows'), 'cpu', d.get('cpu_baseline',{}).get('value'))"; done
for a in "--config c2" "--config c5"; do python tools/membench.py $a; done > $O/membench.jsonl 2>/dev/null; cat $O/membench.jsonl | cut -c1-300
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c2.csv $B > $O/ncu_l_c2.log 2>&1; echo l_c2=$?; python tools/launch_summary.py $O/launches_c2.csv 8
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_c5.csv $B --config c5 > $O/ncu_l_c5.log 2>&1; echo l_c5=$?; python tools/launch_summary.py $O/launches_c5.csv 10
for cfg in c3 c4; do ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$cfg.csv python tools/conv_prof.py $cfg > /dev/null 2>&1; echo l_$cfg=$?; python tools/launch_summary.py $O/launches_$cfg.csv 10; done
ncu --set full --import-source on --clock-control none -k regex:tc_kernel -s 6 -c 3 -o /tmp/prof/tc -f $B > $O/ncu_tc.log 2>&1; echo tcfull=$?
python tools/ncu_summary.py full /tmp/prof/tc.ncu-rep $O/ncu_tc_c2.json "ncu --set full --import-source on --clock-control none -k regex:tc_kernel -s 6 -c 3 $B"
ncu --set full --clock-control none -k regex:'conv_tc_kernel|pool_' -s 11 -c 11 -o /tmp/prof/conv -f python tools/conv_prof.py c4 > $O/ncu_conv.log 2>&1; echo convfull=$?
python tools/ncu_summary.py full /tmp/prof/conv.ncu-rep $O/ncu_conv_c4.json "ncu --set full --clock-control none -k regex:'conv_tc_kernel|pool_' -s 11 -c 11 python tools/conv_prof.py c4"
ncu --set full --clock-control none -k regex:'conv_tc_kernel|pool_' -s 7 -c 7 -o /tmp/prof/conv3 -f python tools/conv_prof.py c3 > $O/ncu_conv3.log 2>&1; echo conv3full=$?
python tools/ncu_summary.py full /tmp/prof/conv3.ncu-rep $O/ncu_conv_c3.json "ncu --set full --clock-control none -k regex:'conv_tc_kernel|pool_' -s 7 -c 7 python tools/conv_prof.py c3"
ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel|slot_sum' -c 6 -o /tmp/prof/mem -f python tools/membench.py --config c2 --reps 1 > $O/ncu_membench.log 2>&1; echo ncumem=$?
python tools/ncu_summary.py full /tmp/prof/mem.ncu-rep $O/ncu_mem_c2.json "ncu --set full --clock-control none -k regex:'gather_kernel|sumsq_kernel|normals_kernel|weights_kernel|slot_sum' -c 6 python tools/membench.py --config c2 --reps 1"
ls -la $O | tail -40
