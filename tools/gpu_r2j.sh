# fused forward (f16x2): multicast cluster shapes, scheduling group size
mkdir -p gpurun_out
python tools/tune_fwd.py --precision f16x2 --rounds 2 --steps 3 "LIB=_exp/mc.so DASMC_TC_CLUSTER=1" "LIB=_exp/mc.so DASMC_TC_CLUSTER=3" "LIB=_exp/mc.so DASMC_TC_CLUSTER=2" "LIB=_exp/mc.so DASMC_TC_CLUSTER=4" "LIB=_exp/mc.so DASMC_TC_CLUSTER=3 DASMC_DEBUG_EPI=3" "LIB=_exp/mc.so DASMC_TC_CLUSTER=4 DASMC_DEBUG_EPI=3" "DASMC_TC_RG=63" "DASMC_TC_RG=8" "DASMC_TC_RG=4" "DASMC_TC_RG=63 DASMC_DEBUG_EPI=3" > gpurun_out/ab_fwd3.log 2>&1; tail -12 gpurun_out/ab_fwd3.log
