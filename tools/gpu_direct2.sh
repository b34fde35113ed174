mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cnn_tc.py -q -x > gpurun_out/t_dir2.log 2>&1; echo tests=$?; tail -1 gpurun_out/t_dir2.log; grep -E "^E " gpurun_out/t_dir2.log | head -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dir2_c4.csv python tools/conv_prof.py c4 > /dev/null 2>&1; echo ncu=$?; python tools/launch_summary.py gpurun_out/dir2_c4.csv 7
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dir2_c3.csv python tools/conv_prof.py c3 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/dir2_c3.csv 6
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -1 gpurun_out/bench_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"
