// The leapfrog move fused into every weight-gradient epilogue (SIMT and
// tcgen05 kernels share it).  For parameter idx of particle j with data
// gradient `acc` (unscaled window sum):
//   g = -theta/sigma^2 + scale * acc                 (target.hpp:147-173)
//   s = 0      : p += h/2 g ; theta_out = theta + h p (kernels.hpp:89-91)
//   0 < s < S  : p += h/2 g ; p += h/2 g ; theta_out = theta + h p
//                (the closing half kick of step s-1 and the opening half kick of step s)
//   s = S      : p += h/2 g                          (kernels.hpp:94)
// Non-finite g, p or theta_out sets the particle's divergence flag
// (kernels.hpp:87-95).
#pragma once

#include "ctx.cuh"

namespace dasmc_b200 {

__device__ __forceinline__ void leapfrog_update(const EpiParams& e, int j, int64_t idx, float acc) {
  const float th = e.theta_in[idx];
  const float g = fmaf(e.scale, acc, -th * e.inv_var);
  bool bad = !isfinite(g);
  if (e.mode == kEpiStoreGrad) {
    e.grad_out[idx] = g;
    return;
  }
  float p = e.p[idx];
  p = fmaf(e.hh, g, p);
  if (e.mode == kEpiMid) p = fmaf(e.hh, g, p);
  bad |= !isfinite(p);
  e.p[idx] = p;
  if (e.mode != kEpiLast) {
    const float tn = fmaf(e.h, p, th);
    bad |= !isfinite(tn);
    e.theta_out[idx] = tn;
  }
  if (bad) atomicOr(&e.flags[j], 1);
}

}  // namespace dasmc_b200
