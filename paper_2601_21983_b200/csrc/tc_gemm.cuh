// tcgen05 / TMA / TMEM tensor-core path for the layer-1 contractions
// (see tc_gemm.cu).  The layer-1 forward Z1 = X W1^T and weight gradient
// dW1 = delta1^T X dominate the FLOPs of every BASELINE config.
#pragma once

#include "ctx.cuh"

namespace dasmc_b200 {

bool tc_layer1_eligible(const Ctx& c);
void tc_forward_layer1(Ctx& c, const float* theta_in, int64_t J, int64_t M);
void tc_delta_layer1(Ctx& c, const float* theta_in, int64_t J, int64_t M);
void tc_dw_layer1(Ctx& c, int64_t J, int64_t M, const EpiParams& epi);
void launch_p_sumsq(Ctx& c, int64_t J);

}  // namespace dasmc_b200
