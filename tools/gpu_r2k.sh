mkdir -p gpurun_out
for d in 64 128 14; do echo DBG=$d; DASMC_CONV_DWT=1 DASMC_CONV_DBG=$d timeout 120 python tools/dwt_probe.py 5 16 32 2>&1 | tail -1 | cut -c1-200; done
