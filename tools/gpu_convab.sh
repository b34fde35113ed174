# C4 step time with library variants swapped in (conv weight-gradient block shapes)
L=paper_2601_21983_b200/libdasmc_gpu.so
cp $L /tmp/main.so
for v in /tmp/main.so _exp/ci1.so _exp/ci4.so; do cp $v $L; echo "$v $(timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; done
cp /tmp/main.so $L
timeout 600 python -m pytest tests/test_gpu_cnn.py -x -q 2>&1 | tail -1
