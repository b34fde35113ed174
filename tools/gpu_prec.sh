# precision modes: interleaved timing (tools/tune_fwd.py) + accuracy vs the fp64 oracle (tools/diag_prec.py)
set -x
python tools/tune_fwd.py "PREC=tf32h" "PREC=f16x2" "PREC=f16" "PREC=tf32" --rounds 3 > gpurun_out/prec_tune.log 2>&1; tail -8 gpurun_out/prec_tune.log
python tools/diag_prec.py > gpurun_out/prec_diag.jsonl 2>&1; cat gpurun_out/prec_diag.jsonl
