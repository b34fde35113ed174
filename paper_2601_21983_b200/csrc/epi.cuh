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

// Chunked windows (EpiParams::acc_mode): true when `acc` now holds the whole window's sum.
__device__ __forceinline__ bool grad_accumulate(const EpiParams& e, int64_t idx, float& acc) {
  if (e.acc_mode == 0) return true;
  if (e.acc_mode == 1) {
    e.gacc[idx] = acc;
    return false;
  }
  if (e.acc_mode == 2) {
    e.gacc[idx] += acc;
    return false;
  }
  acc = e.gacc[idx] + acc;
  return true;
}

__device__ __forceinline__ void leapfrog_update(const EpiParams& e, int j, int64_t idx, float acc) {
  if (!grad_accumulate(e, idx, acc)) return;
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
  if (e.mode == kEpiLast && e.grad_cache) e.grad_cache[idx] = g;
  bad |= !isfinite(p);
  e.p[idx] = p;
  if (e.mode != kEpiLast) {
    const float tn = fmaf(e.h, p, th);
    bad |= !isfinite(tn);
    e.theta_out[idx] = tn;
  }
  if (bad) atomicOr(&e.flags[j], 1);
}

// N parameters at once (a 16-column chunk of a weight-gradient tile): every load is
// issued before any store, so the chunk's 2N loads are in flight together instead of
// one dependent round trip per parameter (short-K GEMMs are epilogue-latency bound).
template <int N>
__device__ __forceinline__ void leapfrog_update_n(const EpiParams& e, int j, const int64_t* idx, const float* acc_in,
                                                  int count) {
  float acc[N];
#pragma unroll
  for (int q = 0; q < N; ++q) acc[q] = acc_in[q];
  if (e.acc_mode != 0) {
    bool apply = true;
#pragma unroll
    for (int q = 0; q < N; ++q)
      if (q < count) apply = grad_accumulate(e, idx[q], acc[q]);
    if (!apply) return;
  }
  float th[N], p[N];
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (q < count) {
      th[q] = e.theta_in[idx[q]];
      if (e.mode != kEpiStoreGrad) p[q] = e.p[idx[q]];
    }
  bool bad = false;
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (q < count) {
      const float g = fmaf(e.scale, acc[q], -th[q] * e.inv_var);
      bad |= !isfinite(g);
      if (e.mode == kEpiStoreGrad) {
        e.grad_out[idx[q]] = g;
        continue;
      }
      float pq = fmaf(e.hh, g, p[q]);
      if (e.mode == kEpiMid) pq = fmaf(e.hh, g, pq);
      if (e.mode == kEpiLast && e.grad_cache) e.grad_cache[idx[q]] = g;
      bad |= !isfinite(pq);
      e.p[idx[q]] = pq;
      if (e.mode != kEpiLast) {
        const float tn = fmaf(e.h, pq, th[q]);
        bad |= !isfinite(tn);
        e.theta_out[idx[q]] = tn;
      }
    }
  if (bad && e.mode != kEpiStoreGrad) atomicOr(&e.flags[j], 1);
}

}  // namespace dasmc_b200
