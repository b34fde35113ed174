# CNN: argmax-coded pool backward, no stage-0 NHWC delta -- parity + C3/C4 benches + launch lists
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cnn_tc.py tests/test_gpu_cnn.py -q -x > gpurun_out/t_cnn.log 2>&1; echo tests=$?; tail -2 gpurun_out/t_cnn.log; grep -E "^E " gpurun_out/t_cnn.log | head -5
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo c3=$?
for f in bench_c4 bench_c3; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'frac', d['roofline']['frac'], d['config'].get('window_rows'))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c4.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/l_c4.csv 8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3.csv python tools/conv_prof.py c3 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/l_c3.csv 8
