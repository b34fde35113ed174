// tcgen05 / TMA / TMEM tensor-core path (tc_gemm.cu) for one-hidden-layer
// MLPs (every BASELINE MLP config except C5's two hidden layers):
//
//   fused forward  D[m, o] = X[m, :] . W1[o, :]   (128 x N tile in TMEM, kind::tf32)
//                  epilogue per window row m (one thread per TMEM lane):
//                  a1 = act(D + b1); z2 = W2 a1 + b2; log-softmax / ll;
//                  delta2 = w_m (onehot - softmax); delta1 = (W2^T delta2) . act'(a1)
//                  -> writes a1^T, delta1^T, delta2^T (m-contiguous) + ll partials
//   weight grads   dW1^T[i, o] = sum_m X^T[i, m] delta1^T[o, m]   (+ ones row -> db1)
//                  dW2^T[o, c] = sum_m a1^T[o, m] delta2^T[c, m]  (+ ones row -> db2)
//                  epilogue: the fused leapfrog (epi.cuh)
// Precision: kind::tf32 (1 MMA) or split-tf32 (hi/lo operands, 3 MMAs per
// k-step: hi.hi + hi.lo + lo.hi) for fp32-level accuracy.
#pragma once

#include "ctx.cuh"

namespace dasmc_b200 {

bool tc_layer1_eligible(const Ctx& c);
void tc_init(Ctx& c);  // allocates X^T (+ splits) once per context
void tc_refresh_data(Ctx& c);  // re-derive the operand copies of X after the active rows changed
void tc_free(Ctx& c);
void tc_ensure_rows(Ctx& c, int64_t Mcap);
// One gradient evaluation (or forward-only pass) of the whole network on the tensor cores.
void tc_eval(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
             const EpiParams* epi);
void launch_p_sumsq(Ctx& c, int64_t J);

}  // namespace dasmc_b200
