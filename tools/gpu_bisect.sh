# which conv_tc commit broke the CNN tensor-core path; per-variant C4/C3 evaluation time
mkdir -p gpurun_out
for v in 9497ba5 41dc1e7 c53c787 92b9e92 9673f0f 41444ee HEAD; do
  lib=""; [ $v != HEAD ] && lib="DASMC_GPU_LIB=_exp/at_$v.so"
  env $lib timeout 300 python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "value_and_grad or chunked" > gpurun_out/bis_$v.log 2>&1; r=$?
  echo "== $v tests=$r $(tail -1 gpurun_out/bis_$v.log)"
  if [ $r = 0 ]; then
    env $lib REPS=3 timeout 300 python tools/conv_prof.py c4 2>&1 | tail -1
    env $lib REPS=3 timeout 300 python tools/conv_prof.py c3 2>&1 | tail -1
  fi
done
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_cnn_tc.py -q -x -k "value_and_grad" > gpurun_out/san.log 2>&1; echo san=$?; grep -m5 -A12 "=====" gpurun_out/san.log | head -60
