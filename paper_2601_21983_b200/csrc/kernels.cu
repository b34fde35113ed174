// CUDA-core (SIMT, fp32) kernels of the SMC hot path for sm_100a: batched
// per-particle MLP forward / log-softmax / backward with the leapfrog move
// fused into the weight-gradient epilogue, the parallel xoshiro256++ momentum
// generator, the log-weight / normalise / ESS / resampling block and the
// particle gather.  The tcgen05 tensor-core GEMMs (tc_gemm.cu) replace the
// layer-1 contractions when the context's precision asks for them.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <cstdio>
#include <stdexcept>

#include "ctx.cuh"
#include "epi.cuh"
#include "host.h"
#include "tc_gemm.cuh"
#include "conv_tc.cuh"

namespace dasmc_b200 {

std::atomic<long long> g_launch_count{0};

KTimer::KTimer(Ctx& cc, int k) : c(cc), kind(cc.capturing ? -1 : k) {
  if (!c.ktime || kind < 0) return;
  auto& v = c.kev[kind];
  while ((int)v.size() < 2 * (c.kev_used[kind] + 1)) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    v.push_back(e);
  }
  CK(cudaEventRecord(v[2 * c.kev_used[kind]], c.stream));
}

KTimer::~KTimer() {
  if (!c.ktime || kind < 0) return;
  cudaEventRecord(c.kev[kind][2 * c.kev_used[kind] + 1], c.stream);
  ++c.kev_used[kind];
}

void harvest_timers(Ctx& c) {
  CK(cudaStreamSynchronize(c.stream));
  for (int k = 0; k < kTimerKinds; ++k) {
    for (int i = 0; i < c.kev_used[k]; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c.kev[k][2 * i], c.kev[k][2 * i + 1]));
      c.kms[k] += ms;
      ++c.kcount[k];
    }
    c.kev_used[k] = 0;
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError{std::string(what) + ": " + cudaGetErrorString(e)};
}

namespace {

constexpr double kLogTwoPi = 1.8378770664093455;

__device__ __forceinline__ bool finitef(float v) { return isfinite(v); }

// ---- reference <-> internal parameter index ------------------------------------------------
// Reference layout of layer l (network.hpp:55-62): W(r, c) at ref_off + r + c*out, then b.
// Internal: W row-major [out][in] at woff, b at boff.
__device__ __forceinline__ int64_t internal_index(const NetDev& net, int64_t i) {
  int l = 0;
#pragma unroll 1
  for (; l < net.nseg - 1; ++l)
    if (i < net.seg[l + 1].ref_off) break;
  const LayerDev& ly = net.seg[l];
  const int64_t t = i - ly.ref_off;
  const int64_t nw = (int64_t)ly.in * ly.out;
  if (t < nw) {
    const int64_t r = t % ly.out, c = t / ly.out;
    return ly.woff + r * ly.in + c;
  }
  return ly.boff + (t - nw);
}

template <typename S, typename T>
__global__ void ref_to_internal_kernel(NetDev net, const S* __restrict__ src, T* __restrict__ dst, int64_t J) {
  const int64_t total = J * net.D;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / net.D, i = g - j * net.D;
    dst[j * net.Dp + internal_index(net, i)] = (T)src[g];
  }
}

template <typename S, typename T>
__global__ void internal_to_ref_kernel(NetDev net, const S* __restrict__ src, T* __restrict__ dst, int64_t J) {
  const int64_t total = J * net.D;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / net.D, i = g - j * net.D;
    dst[g] = (T)src[j * net.Dp + internal_index(net, i)];
  }
}

// ---- deterministic block reductions -------------------------------------------------------
template <int NT>
__device__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) t += sh[i];
    sh[NT / 32] = t;
  }
  __syncthreads();
  t = sh[NT / 32];
  __syncthreads();
  return t;
}

template <int NT>
__device__ double block_max(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sh[0];
    for (int i = 1; i < NT / 32; ++i) t = fmax(t, sh[i]);
    sh[NT / 32] = t;
  }
  __syncthreads();
  const double t = sh[NT / 32];
  __syncthreads();
  return t;
}

// ---- batched SIMT SGEMM with fused epilogues --------------------------------------------------
// C(m, n) = sum_k A(m, k) B(n, k) for batch j = blockIdx.z.
//   AK: A(m,k) = A[m*lda + k] (K-major) else A[k*lda + m];  same for BK / B.
//   ones_col >= 0: B(ones_col, k) = 1 (bias-gradient column of the dW GEMM).
// 64x64 block tile, 16-deep k slices double-buffered through shared memory,
// 4x4 register micro-tile, two-level fp32 accumulation (partial sums are
// folded every 256 k) to bound the rounding of long data reductions.
constexpr int TB = 64, TK = 16;

template <bool AK, bool BK, class Epi>
__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda,
                                                    int64_t sA, const float* __restrict__ B, int64_t ldb,
                                                    int64_t sB, int ones_col, Epi epi) {
  __shared__ __align__(16) float As[2][TK][TB + 4];
  __shared__ __align__(16) float Bs[2][TK][TB + 4];
  const int j = blockIdx.z;
  const int m0 = blockIdx.y * TB, n0 = blockIdx.x * TB;
  A += (int64_t)j * sA;
  B += (int64_t)j * sB;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  float ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int m, k;
      if (AK) {
        m = tid >> 2;
        k = ((tid & 3) << 2) + q;
      } else {
        k = tid >> 4;
        m = ((tid & 15) << 2) + q;
      }
      const int gm = m0 + m, gk = k0 + k;
      ra[q] = (gm < M && gk < K) ? (AK ? A[(int64_t)gm * lda + gk] : A[(int64_t)gk * lda + gm]) : 0.f;
      int n, kb;
      if (BK) {
        n = tid >> 2;
        kb = ((tid & 3) << 2) + q;
      } else {
        kb = tid >> 4;
        n = ((tid & 15) << 2) + q;
      }
      const int gn = n0 + n, gkb = k0 + kb;
      float v = 0.f;
      if (gkb < K && gn < N) {
        if (gn == ones_col)
          v = 1.f;
        else
          v = BK ? B[(int64_t)gn * ldb + gkb] : B[(int64_t)gkb * ldb + gn];
      }
      rb[q] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (AK)
        As[buf][((tid & 3) << 2) + q][tid >> 2] = ra[q];
      else
        As[buf][tid >> 4][((tid & 15) << 2) + q] = ra[q];
      if (BK)
        Bs[buf][((tid & 3) << 2) + q][tid >> 2] = rb[q];
      else
        Bs[buf][tid >> 4][((tid & 15) << 2) + q] = rb[q];
    }
  };

  float acc[4][4], tot[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = tot[i][q] = 0.f;

  const int nk = (K + TK - 1) / TK;
  load(0);
  store(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load((t + 1) * TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
    }
    if ((t & 15) == 15) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tot[i][q] += acc[i][q];
          acc[i][q] = 0.f;
        }
    }
    if (t + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + q;
      if (m < M && n < N) epi(j, m, n, tot[i][q] + acc[i][q]);
    }
}

// Forward epilogue: out = act(acc + b) (network.hpp:92-95).
struct EpiFwd {
  float* C;
  int64_t ldc, sC;
  const float* theta;
  int64_t Dp, boff;
  int hidden, act;
  __device__ void operator()(int j, int m, int n, float v) const {
    v += theta[(int64_t)j * Dp + boff + n];
    if (hidden) v = act == DASMC_RELU ? fmaxf(v, 0.f) : tanhf(v);
    C[(int64_t)j * sC + (int64_t)m * ldc + n] = v;
  }
};

// Backward delta epilogue: delta_prev = acc * act'(a_prev), in place over a_prev
// (network.hpp:209-215; relu' from the post-activation, tanh' = 1 - a^2).
struct EpiDx {
  float* D;
  int64_t ldd, sD;
  int act;
  __device__ void operator()(int j, int m, int n, float v) const {
    float* p = D + (int64_t)j * sD + (int64_t)m * ldd + n;
    const float a = *p;
    // act < 0: no activation derivative (a pooled CNN stage output: the pool backward applies it)
    *p = act < 0 ? v : act == DASMC_RELU ? v * (a > 0.f ? 1.f : 0.f) : v * (1.f - a * a);
  }
};

// Weight-gradient epilogue with the leapfrog move fused (kernels.hpp:85-96).
// (o, i) = (m, n); i == in is the bias column.  g = -theta/sigma^2 + scale*acc.
struct EpiDw {
  EpiParams e;
  int64_t Dp, woff, boff;
  int in;
  __device__ void operator()(int j, int o, int i, float acc) const {
    const int64_t idx = (int64_t)j * Dp + (i < in ? woff + (int64_t)o * in + i : boff + o);
    leapfrog_update(e, j, idx, acc);
  }
};

template <bool AK, bool BK, class Epi>
void sgemm(cudaStream_t s, int M, int N, int K, const float* A, int64_t lda, int64_t sA, const float* B,
           int64_t ldb, int64_t sB, int ones_col, int64_t J, const Epi& epi) {
  if (M <= 0 || N <= 0 || J <= 0) return;
  dim3 grid((N + TB - 1) / TB, (M + TB - 1) / TB, (unsigned)J);
  sgemm_kernel<AK, BK, Epi><<<grid, 256, 0, s>>>(M, N, K, A, lda, sA, B, ldb, sB, ones_col, epi);
  LAUNCHED();
}

// ---- log-softmax likelihood and output residual (network.hpp:180-193) --------------------------
// One thread per window row; per-row arithmetic in fp64; per-block prefix and
// block partial sums of the unscaled log-likelihood.  delta = w_row*(onehot - softmax)
// with w_row = 1 on the prefix and beta_rows on the block (SDA tempering).
constexpr int kRowsPerBlock = 128;

__global__ void __launch_bounds__(kRowsPerBlock) softmax_kernel(float* __restrict__ logits, int64_t sL, int C,
                                                              const int32_t* __restrict__ y, int64_t M, int64_t P,
                                                              float beta_rows, int need_grad,
                                                              double* __restrict__ ll_part, int slots) {
  __shared__ double sh[kRowsPerBlock / 32 + 1];
  const int j = blockIdx.y;
  const int64_t m = (int64_t)blockIdx.x * kRowsPerBlock + threadIdx.x;
  double pre = 0.0, blk = 0.0;
  if (m < M) {
    float* z = logits + (int64_t)j * sL + m * C;
    const int yi = y[m];
    double mx = (double)z[0];
    for (int c = 1; c < C; ++c) mx = fmax(mx, (double)z[c]);
    double den = 0.0;
    for (int c = 0; c < C; ++c) den += exp((double)z[c] - mx);
    const double ll = (double)z[yi] - (mx + log(den));
    if (m < P)
      pre = ll;
    else
      blk = ll;
    if (need_grad) {
      const float wr = m < P ? 1.f : beta_rows;
      for (int c = 0; c < C; ++c) {
        const double pr = exp((double)z[c] - mx) / den;
        z[c] = wr * (float)((c == yi ? 1.0 : 0.0) - pr);
      }
    }
  }
  pre = block_sum<kRowsPerBlock>(pre, sh);
  blk = block_sum<kRowsPerBlock>(blk, sh);
  if (threadIdx.x == 0) {
    double* o = ll_part + ((int64_t)j * slots + blockIdx.x) * 2;
    o[0] = pre;
    o[1] = blk;
  }
}

// Sum of squares of a particle-major [J][Dp] fp32 array, per (particle, chunk).
constexpr int kSqChunk = 8192;
__global__ void __launch_bounds__(256) sumsq_kernel(const float* __restrict__ v, int64_t Dp, double* part,
                                                   int slots) {
  __shared__ double sh[256 / 32 + 1];
  const int j = blockIdx.y;
  const int64_t base = (int64_t)j * Dp + (int64_t)blockIdx.x * kSqChunk;
  const int64_t lim = min((int64_t)kSqChunk, Dp - (int64_t)blockIdx.x * kSqChunk);
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < lim; i += 256) {
    const double x = (double)v[base + i];
    s += x * x;
  }
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) part[(int64_t)j * slots + blockIdx.x] = s;
}

// Per-particle log target from the slots (target.hpp:131-173 arithmetic in fp64).
__global__ void eval_finalize_kernel(int64_t J, const double* __restrict__ ll_part, int ll_slots, int used_ll,
                                     const double* __restrict__ th_part, int th_slots, int used_th, double D,
                                     double var, int mode, double scale, double beta, double* values,
                                     double* pre_out, double* blk_out, int* flags) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= J) return;
  double llp = 0.0, llb = 0.0;
  for (int s = 0; s < used_ll; ++s) {
    llp += ll_part[(j * ll_slots + s) * 2];
    llb += ll_part[(j * ll_slots + s) * 2 + 1];
  }
  if (pre_out) pre_out[j] = llp;
  if (blk_out) blk_out[j] = llb;
  if (values) {
    double th2 = 0.0;
    for (int s = 0; s < used_th; ++s) th2 += th_part[j * th_slots + s];
    double v = -0.5 * D * (kLogTwoPi + log(var)) - th2 / (2.0 * var);  // network.hpp:221-227
    if (mode == DASMC_SCALED)
      v += scale * llp;
    else
      v += llp + beta * llb;
    values[j] = v;
    if (flags && !isfinite(v)) atomicOr(&flags[j], 1);
  }
}

// ---- parallel xoshiro256++ normals ------------------------------------------------------------
// normal() of rng.hpp:76-81 -- sqrt(-2 ln(1 - u1)) cos(2 pi u2), u = (x >> 11) 2^-53 -- in fp32
// from the exact integer draws (the device stores fp32 momenta):
//  * radius: ln(1 - u1) as log1p(-u1) for u1 < 1/2, else ln((2^53 - a) 2^-53) with the
//    integer complement, so both branches see a 24-bit-exact argument;
//  * angle: the quadrant comes from the top two bits of the 53-bit integer and the remainder
//    is folded to phi in [0, pi/4] (complemented in integers when past pi/4), so sin / cos
//    are evaluated on a relatively exact small angle -- including next to the zeros of cos.
// The stored value is within a few fp32 ulp of the fp64 normal rounded to fp32 (stated bound
// in tests/test_gpu_parity.py), at ~1/3 of the fp64 Box-Muller's instruction count.
__device__ __forceinline__ float normal_from_draws(uint64_t x1, uint64_t x2) {
  const uint64_t a = x1 >> 11;
  const float L = a < (1ULL << 52) ? log1pf(-__ull2float_rn(a) * 0x1p-53f)
                                   : logf(__ull2float_rn((1ULL << 53) - a) * 0x1p-53f);
  const float r = sqrtf(-2.f * L);
  const uint64_t b = x2 >> 11;
  const int q = (int)(b >> 51);
  const uint64_t f = b & ((1ULL << 51) - 1);
  const bool comp = f >= (1ULL << 50);
  const uint64_t g = comp ? (1ULL << 51) - f : f;
  float sp, cp;
  sincosf(__ull2float_rn(g) * (6.28318530717958647692f * 0x1p-53f), &sp, &cp);
  const float ct = comp ? sp : cp;  // cos / sin of the angle within its quadrant
  const float st = comp ? cp : sp;
  const float cs = q == 0 ? ct : q == 1 ? -st : q == 2 ? -ct : st;
  return r * cs;
}

// Thread (j, c) draws the c-th chunk of `chunk` normals of stream fork(a, b, c')
// by jumping c*2*chunk steps ahead (F2-linear jump with host-precomputed
// polynomials); each normal consumes two draws (rng.hpp:76-81) and is stored in fp32
// at its internal position.  With chunk = a layer's fan-out a chunk is one column of
// W, so a warp's stores are coalesced.
__global__ void normals_kernel(NetDev net, uint64_t root, uint64_t a, uint64_t b, int per_particle_c,
                               int64_t J, int64_t nchunks, int64_t chunk, const uint64_t* __restrict__ jump_tab,
                               float scale, float* __restrict__ dst, double* __restrict__ sq_part, int64_t j_offset,
                               const DevStep* __restrict__ ds) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= J * nchunks) return;
  const int64_t j = g / nchunks, c = g - j * nchunks;
  if (ds) b = (uint64_t)ds->k;  // the step's iteration, from device memory (graph replay)
  // fork(kProposal, k, j) -> (a, b, j); fork(kInit, j) -> (a, j, 0); j is the GLOBAL slot
  const uint64_t jg = (uint64_t)(j + j_offset);
  const uint64_t key = per_particle_c ? fork_key(root, a, b, jg) : fork_key(root, a, jg, 0);
  Xoshiro x;
  x.seed(key);
  if (c > 0) x.jump(jump_tab + 4 * c);
  const int64_t lo = c * chunk, hi = min(net.D, lo + chunk);
  double sq = 0.0;
  float* out = dst + j * net.Dp;
  // reference index i -> internal offset, walked incrementally (one division per chunk):
  // layer l, W(r, c) at ref_off + r + c*out -> woff + r*in + c; then the bias block.
  // The destination is walked as a pointer: + `in` per row of a column, back to the next column's top at
  // the end of one, then the bias run (no multiplication or 64-bit index arithmetic per normal; the loop is
  // integer-issue bound).
  int l = 0;
  while (l < net.nseg - 1 && lo >= net.seg[l + 1].ref_off) ++l;
  int64_t t = lo - net.seg[l].ref_off;
  int64_t nw = (int64_t)net.seg[l].in * net.seg[l].out;
  int r = t < nw ? (int)(t % net.seg[l].out) : 0;
  {
    const int64_t cc = t < nw ? t / net.seg[l].out : 0;
    out += t < nw ? net.seg[l].woff + (int64_t)r * net.seg[l].in + cc : net.seg[l].boff + (t - nw);
  }
  int rem = (int)min((int64_t)0x7fffffff, (t < nw ? nw : nw + net.seg[l].nb) - t);  // elements left in this run
  bool in_w = t < nw;
  for (int64_t i = lo; i < hi; ++i) {
    const uint64_t x1 = x.next();
    const uint64_t x2 = x.next();
    const float v = scale * normal_from_draws(x1, x2);
    *out = v;
    sq += (double)v * (double)v;
    // advance to i + 1
    const LayerDev& ly = net.seg[l];
    if (--rem > 0) {
      if (in_w) {
        if (++r == ly.out) {  // top of the next column
          r = 0;
          out -= (int64_t)(ly.out - 1) * ly.in - 1;
        } else {
          out += ly.in;
        }
      } else {
        ++out;
      }
    } else if (in_w) {  // the weights are done: this layer's bias run
      in_w = false;
      rem = ly.nb;
      out = dst + j * net.Dp + ly.boff;
      if (rem == 0 && l + 1 < net.nseg) {
        ++l;
        in_w = true;
        r = 0;
        rem = (int)min((int64_t)0x7fffffff, (int64_t)net.seg[l].in * net.seg[l].out);
        out = dst + j * net.Dp + net.seg[l].woff;
      }
    } else if (l + 1 < net.nseg) {  // next layer's weights
      ++l;
      in_w = true;
      r = 0;
      rem = (int)min((int64_t)0x7fffffff, (int64_t)net.seg[l].in * net.seg[l].out);
      out = dst + j * net.Dp + net.seg[l].woff;
    }
  }
  if (sq_part) sq_part[j * nchunks + c] = sq;
}

// `count` uniforms of one stream (resampling), chunked with the same jumps
// (a chunk of `chunk` normals = 2*chunk draws).
__global__ void uniforms_kernel(uint64_t key, int64_t count, int64_t chunk, const uint64_t* __restrict__ jump_tab,
                                double* __restrict__ dst, const DevStep* __restrict__ ds) {
  if (ds) key = ds->ukey;
  const int64_t per = 2 * chunk;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c * per >= count) return;
  Xoshiro x;
  x.seed(key);
  if (c > 0) x.jump(jump_tab + 4 * c);
  const int64_t hi = min(count, (c + 1) * per);
  for (int64_t i = c * per; i < hi; ++i) dst[i] = x.uniform();
}

// Fixed-order per-particle sum of `slots` fp64 partials, one warp per particle: lane l
// adds slots l, l+32, ... in order, then a fixed shuffle tree (lane 0's result).  Coalesced,
// so the single-block weights kernel reads one value per particle instead of walking
// every particle's slot row itself (J x 795 strided loads at C2).
__global__ void slot_sum_kernel(const double* __restrict__ part, int slots, int64_t J, double* __restrict__ out) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= J) return;
  double s = 0.0;
  for (int i = lane; i < slots; i += 32) s += part[j * slots + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[j] = s;
}

// ---- weights / normalise / ESS / resample (smc.hpp:127-156) ---------------------------------------
// Single 1024-thread block (J <= 65536).  Deterministic fixed-order reductions.
constexpr int kWT = 1024;
// Largest ensemble whose CDF is built in shared memory (128 KB of fp64).
constexpr int64_t kCdfSmemMax = 16384;

// Sequential fp64 CDF of the normalised weights with last = 1.0 (numeric.hpp:87-94),
// then upper_bound per particle (multinomial: sorted-or-not uniforms uni[j];
// systematic: (uni[0] + j) / J).  The running sum keeps the reference's strict
// left-to-right order (bit-exact cdf); one thread adds while its operands come
// from shared memory in batches, so the chain is DADD-latency bound, not a
// dependent global load per element.  cdf (global) receives the same values.
__device__ void cdf_and_search(int64_t J, const double* __restrict__ w, double* __restrict__ cdf,
                               const double* __restrict__ uni, int kind, int32_t* __restrict__ idx,
                               double* __restrict__ logw_reset, double lw_value) {
  extern __shared__ double cdf_s[];
  const bool sm = J <= kCdfSmemMax;
  double* cd = sm ? cdf_s : cdf;
  if (sm) {
    for (int64_t j = threadIdx.x; j < J; j += kWT) cdf_s[j] = w[j];
  } else {
    for (int64_t j = threadIdx.x; j < J; j += kWT) cdf[j] = w[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    int64_t j = 0;
    for (; j + 8 <= J; j += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = cd[j + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc += v[u];
        cd[j + u] = acc;
      }
    }
    for (; j < J; ++j) {
      acc += cd[j];
      cd[j] = acc;
    }
    cd[J - 1] = 1.0;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < J; j += kWT) {
    const double u = kind == DASMC_MULTINOMIAL ? uni[j] : (uni[0] + (double)j) / (double)J;
    int64_t lo = 0, hi = J;  // first index with cdf > u
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cd[mid] > u)
        hi = mid;
      else
        lo = mid + 1;
    }
    idx[j] = (int32_t)lo;
    if (sm) cdf[j] = cd[j];
    if (logw_reset) logw_reset[j] = lw_value;  // smc.hpp:100
  }
}

size_t cdf_smem_bytes(int64_t J) { return J <= kCdfSmemMax ? (size_t)J * sizeof(double) : 0; }
__global__ void __launch_bounds__(kWT) weights_kernel(int64_t J, double* __restrict__ logw,
                                                      const double* __restrict__ lt_old,
                                                      const double* __restrict__ lt_new,
                                                      const double* __restrict__ p0_part, int p0_slots,
                                                      const double* __restrict__ pS_part, int pS_slots,
                                                      const int* __restrict__ flags, double* __restrict__ w,
                                                      double* __restrict__ cdf, const double* __restrict__ uni,
                                                      int32_t* __restrict__ idx, double fraction, int always,
                                                      int kind, double* __restrict__ rec, int k, int compute_lw,
                                                      const DevStep* __restrict__ ds) {
  __shared__ double sh[kWT / 32 + 1];
  if (ds) {  // record slot and iteration from device memory (graph replay); rec = the ring base
    rec += (size_t)ds->slot * 8;
    k = ds->k;
  }
  __shared__ int s_res;
  // 1) new log-weights (kernels.hpp:153-163, smc.hpp:127-138); with compute_lw = 0
  //    logw already holds them (the gathered vector of a sharded ensemble)
  int ndiv = 0;
  for (int64_t j = threadIdx.x; j < J && !compute_lw; j += kWT) ndiv += logw[j] == -CUDART_INF ? 1 : 0;
  for (int64_t j = threadIdx.x; j < J && compute_lw; j += kWT) {
    double lw;
    if (flags[j]) {
      lw = -CUDART_INF;
      ++ndiv;
    } else {
      double p0 = 0.0, ps = 0.0;
      for (int s = 0; s < p0_slots; ++s) p0 += p0_part[j * p0_slots + s];
      for (int s = 0; s < pS_slots; ++s) ps += pS_part[j * pS_slots + s];
      const double a = lt_new[j], b = lt_old[j];
      const double inc = (isfinite(a) && isfinite(b) && isfinite(p0) && isfinite(ps))
                             ? (a - b) + 0.5 * (p0 - ps)
                             : -CUDART_INF;
      lw = logw[j] + inc;
    }
    logw[j] = lw;
  }
  const double nd = block_sum<kWT>((double)ndiv, sh);
  // 2) normalise (smc.hpp:57-64)
  double mx = -CUDART_INF;
  for (int64_t j = threadIdx.x; j < J; j += kWT) mx = fmax(mx, logw[j]);
  mx = block_max<kWT>(mx, sh);
  if (mx == -CUDART_INF) {  // all particles dead -> SamplerError
    if (threadIdx.x == 0) {
      rec[0] = k;
      rec[1] = 0.0;
      rec[2] = 0.0;
      rec[3] = 0.0;
      rec[4] = nd;
      rec[5] = 1.0;
    }
    return;
  }
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < J; j += kWT) {
    const double e = exp(logw[j] - mx);
    w[j] = e;
    s += e;
  }
  s = block_sum<kWT>(s, sh);
  double s2 = 0.0, mlt = 0.0;
  for (int64_t j = threadIdx.x; j < J; j += kWT) {
    const double v = w[j] / s;
    w[j] = v;
    s2 += v * v;
    if (v > 0.0) mlt += v * lt_new[j];  // smc.hpp:144-148
  }
  s2 = block_sum<kWT>(s2, sh);
  mlt = block_sum<kWT>(mlt, sh);
  const double ess = 1.0 / s2;  // smc.hpp:67-69
  if (threadIdx.x == 0) {
    s_res = (always || ess < fraction * (double)J) ? 1 : 0;  // smc.hpp:151
    rec[0] = k;
    rec[1] = ess;
    rec[2] = s_res;
    rec[3] = mlt;
    rec[4] = nd;
    rec[5] = 0.0;
  }
  __syncthreads();
  if (!s_res) {
    for (int64_t j = threadIdx.x; j < J; j += kWT) idx[j] = (int32_t)j;
    return;
  }
  // 3) sequential fp64 CDF with last = 1.0 (numeric.hpp:87-94), then upper_bound.
  cdf_and_search(J, w, cdf, uni, kind, idx, logw, -log((double)J));
}

// Sharded ensemble, step 1: new (unnormalised) log-weights of the local slots
// (kernels.hpp:153-163, smc.hpp:127-138) into out_lw; logw itself is untouched.
__global__ void local_weights_kernel(int64_t J, const double* __restrict__ logw, const double* __restrict__ lt_old,
                                     const double* __restrict__ lt_new, const double* __restrict__ p0_part,
                                     int p0_slots, const double* __restrict__ pS_part, int pS_slots,
                                     const int* __restrict__ flags, double* __restrict__ out_lw,
                                     double* __restrict__ out_lt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= J) return;
  double lw = -CUDART_INF;
  if (!flags[j]) {
    double p0 = 0.0, ps = 0.0;
    for (int s = 0; s < p0_slots; ++s) p0 += p0_part[j * p0_slots + s];
    for (int s = 0; s < pS_slots; ++s) ps += pS_part[j * pS_slots + s];
    const double a = lt_new[j], b = lt_old[j];
    const double inc =
        (isfinite(a) && isfinite(b) && isfinite(p0) && isfinite(ps)) ? (a - b) + 0.5 * (p0 - ps) : -CUDART_INF;
    lw = logw[j] + inc;
  }
  out_lw[j] = lw;
  out_lt[j] = lt_new[j];
}

// theta rows: dst[i] = src_buf[rows[i]] (pack) or dst_buf[rows[i]] = src[i] (unpack); float4 copies.
__global__ void __launch_bounds__(256) rows_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                                   int64_t Dp4, const int32_t* __restrict__ rows, int pack) {
  const int64_t i = blockIdx.y;
  const int64_t r = rows[i];
  const float4* s = src + (pack ? r : i) * Dp4;
  float4* d = dst + (pack ? i : r) * Dp4;
  for (int64_t q = blockIdx.x * 256 + threadIdx.x; q < Dp4; q += (int64_t)gridDim.x * 256) d[q] = s[q];
}

// Bit-exact resampling hook: caller-provided normalised weights and uniforms.
__global__ void __launch_bounds__(kWT) resample_hook_kernel(int64_t J, const double* __restrict__ w,
                                                            double* __restrict__ cdf,
                                                            const double* __restrict__ uni, int kind,
                                                            int32_t* __restrict__ idx) {
  cdf_and_search(J, w, cdf, uni, kind, idx, nullptr, 0.0);
}

// dst[j] = (flags[s] ? start : end)[s], s = idx[j]  (smc.hpp:97-99 + 129-131).
// Vectorised 16-byte copies; grid (chunks, J).
__global__ void __launch_bounds__(256) gather_kernel(const float4* __restrict__ start,
                                                     const float4* __restrict__ end, float4* __restrict__ dst,
                                                     int64_t Dp4, const int32_t* __restrict__ idx,
                                                     const int* __restrict__ flags) {
  const int64_t j = blockIdx.y;
  const int32_t s = idx[j];
  const float4* src = (flags[s] ? start : end) + (int64_t)s * Dp4;
  float4* d = dst + j * Dp4;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < Dp4; i += (int64_t)gridDim.x * 256) d[i] = src[i];
}

__global__ void gather_parts_kernel(int64_t J, const int32_t* __restrict__ idx, const int* __restrict__ flags,
                                    const double* __restrict__ pre0, const double* __restrict__ blk0,
                                    const double* __restrict__ pre, const double* __restrict__ blk,
                                    double* __restrict__ out_pre, double* __restrict__ out_blk) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int32_t s = idx[j];
  out_pre[j] = flags[s] ? pre0[s] : pre[s];
  out_blk[j] = flags[s] ? blk0[s] : blk[s];
}

__global__ void set_step_kernel(DevStep v, DevStep* d) { *d = v; }

__global__ void zero_ints_kernel(int* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

int grid_for(int64_t total, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + threads - 1) / threads, 148 * 32));
}

// dynamic shared memory of the weights / resampling kernels (the opt-in above 48 KB, once)
size_t cdf_smem(int64_t J) {
  static bool attr[kMaxDevices] = {};
  const int dv = current_device();
  if (!attr[dv]) {
    const int b = (int)(kCdfSmemMax * sizeof(double));
    CK(cudaFuncSetAttribute(weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CK(cudaFuncSetAttribute(resample_hook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    attr[dv] = true;
  }
  return cdf_smem_bytes(J);
}

}  // namespace

// ---- host launchers ----------------------------------------------------------------------------
void ensure_stage(Ctx& c, size_t bytes) {
  if (bytes <= c.stage_bytes) return;
  ++c.alloc_epoch;
  if (c.stage) CK(cudaFree(c.stage));
  c.stage = nullptr;
  CK(cudaMalloc(&c.stage, bytes));
  c.stage_bytes = bytes;
}

void ensure_host_stage(Ctx& c, size_t bytes) {
  if (bytes <= c.h_stage_bytes) return;
  if (c.h_stage) CK(cudaFreeHost(c.h_stage));
  c.h_stage = nullptr;
  CK(cudaMallocHost(&c.h_stage, bytes));
  c.h_stage_bytes = bytes;
}

// ---- [EXT] CNN stages (dasmc_gpu.h conv descriptor; oracle cnn_stages / cnn_stages_backward) ----
// One thread per output element, grid-stride.  Images are [c][h][w]; stage buffers are
// [Jmax][Mcap][per-image floats].  Stage 0 reads X (shared by every particle).
__device__ __forceinline__ float act_apply(float z, int act) { return act == DASMC_RELU ? fmaxf(z, 0.f) : tanhf(z); }
__device__ __forceinline__ float act_grad_post(float a, int act) {
  return act == DASMC_RELU ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a;
}

// Register-tiled direct convolution: a block owns one image of one particle and CT output
// channels; W for the tile sits in shared memory as [cin*k*k][CT] so one float4 load
// feeds four FMAs; each thread owns output pixels and keeps CT accumulators.
template <int K, int CT>
__global__ void __launch_bounds__(128) conv_fwd_kernel(ConvDev d, int act, const float* __restrict__ in,
                                                        int64_t in_ps, const float* __restrict__ theta, int64_t Dp,
                                                        float* __restrict__ A, int64_t a_ps) {
  extern __shared__ float4 cv_sh4[];
  float* Ws = reinterpret_cast<float*>(cv_sh4);
  __shared__ float bs[CT];
  const int64_t m = blockIdx.x, j = blockIdx.z;
  const int co0 = blockIdx.y * CT, KW = d.cin * K * K;
  const float* W = theta + j * Dp + d.woff;
  for (int i = threadIdx.x; i < KW * CT; i += blockDim.x) {
    const int kidx = i / CT, c = i - kidx * CT;
    Ws[i] = co0 + c < d.cout ? W[(int64_t)(co0 + c) * KW + kidx] : 0.f;
  }
  if (threadIdx.x < CT) bs[threadIdx.x] = co0 + (int)threadIdx.x < d.cout ? theta[j * Dp + d.boff + co0 + threadIdx.x] : 0.f;
  __syncthreads();
  const int64_t in_img = (int64_t)d.cin * d.hin * d.win, per = (int64_t)d.cout * d.ho * d.wo;
  const float* src = in + j * in_ps + m * in_img;
  float* dst = A + j * a_ps + m * per;
  const int npix = d.ho * d.wo;
  for (int p = threadIdx.x; p < npix; p += blockDim.x) {
    const int y = p / d.wo, x = p - y * d.wo;
    float acc[CT];
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[c] = bs[c];
    for (int ci = 0; ci < d.cin; ++ci)
#pragma unroll
      for (int ky = 0; ky < K; ++ky) {
        const float* srow = src + ((int64_t)ci * d.hin + y + ky) * d.win + x;
        const float4* wrow = cv_sh4 + (int64_t)((ci * K + ky) * K) * (CT / 4);
        float v[K];
#pragma unroll
        for (int kx = 0; kx < K; ++kx) v[kx] = srow[kx];
#pragma unroll
        for (int kx = 0; kx < K; ++kx)
#pragma unroll
          for (int u = 0; u < CT / 4; ++u) {
            const float4 w = wrow[kx * (CT / 4) + u];
            acc[4 * u] = fmaf(v[kx], w.x, acc[4 * u]);
            acc[4 * u + 1] = fmaf(v[kx], w.y, acc[4 * u + 1]);
            acc[4 * u + 2] = fmaf(v[kx], w.z, acc[4 * u + 2]);
            acc[4 * u + 3] = fmaf(v[kx], w.w, acc[4 * u + 3]);
          }
      }
#pragma unroll
    for (int c = 0; c < CT; ++c)
      if (co0 + c < d.cout) dst[(int64_t)(co0 + c) * npix + p] = act_apply(acc[c], act);
  }
}

__global__ void pool_fwd_kernel(ConvDev d, const float* __restrict__ A, int64_t a_ps, float* __restrict__ P,
                                int64_t p_ps, int64_t M, int64_t J) {
  const int64_t per_a = (int64_t)d.cout * d.ho * d.wo, per = (int64_t)d.cout * d.sh * d.sw;
  const int64_t total = J * M * per;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / (M * per), r = g - j * M * per, m = r / per, o = r - m * per;
    const int co = (int)(o / ((int64_t)d.sh * d.sw));
    const int yx = (int)(o - (int64_t)co * d.sh * d.sw), y = yx / d.sw, x = yx - y * d.sw;
    const float* a = A + j * a_ps + m * per_a + ((int64_t)co * d.ho + 2 * y) * d.wo + 2 * x;
    P[j * p_ps + m * per + o] = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[d.wo], a[d.wo + 1]));
  }
}

// dz = (first argmax of the window ? dP : 0) * act'(A); positions outside the pooled region get 0
// 2x2/2 max-pool backward: one thread per pooled output (2 index divisions, 32-bit inside an
// image) routes dP to the first maximum of its window in (dy, dx) order, times act'(max),
// and writes the window's four dz values.  Pre-pool rows / columns that no window covers
// (odd sizes, floor pooling) are zeroed by the caller.
__global__ void pool_bwd_kernel(ConvDev d, int act, const float* __restrict__ A, int64_t a_ps,
                                const float* __restrict__ dP, int64_t p_ps, float* __restrict__ dZ, int64_t M,
                                int64_t J) {
  const int64_t per_a = (int64_t)d.cout * d.ho * d.wo;
  const int npool = d.cout * d.sh * d.sw, nplane = d.sh * d.sw;
  const int64_t total = J * M * npool;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = g / npool;
    const int q = (int)(g - img * npool);
    const int64_t j = img / M, m = img - j * M;
    const int co = q / nplane, pyx = q - co * nplane, py = pyx / d.sw, px = pyx - py * d.sw;
    const int64_t off = j * a_ps + m * per_a + ((int64_t)co * d.ho + 2 * py) * d.wo + 2 * px;
    const float* a = A + off;
    const float a0 = a[0], a1 = a[1], a2 = a[d.wo], a3 = a[d.wo + 1];
    int best = 0;
    float mx = a0;
    if (a1 > mx) { mx = a1; best = 1; }
    if (a2 > mx) { mx = a2; best = 2; }
    if (a3 > mx) { mx = a3; best = 3; }
    const float v = dP[j * p_ps + m * (int64_t)npool + q] * act_grad_post(mx, act);
    float* z = dZ + off;
    z[0] = best == 0 ? v : 0.f;
    z[1] = best == 1 ? v : 0.f;
    z[d.wo] = best == 2 ? v : 0.f;
    z[d.wo + 1] = best == 3 ? v : 0.f;
  }
}

// Weight gradient of one stage, pass 1: a block owns (particle j, input channel ci, CT
// output channels, a chunk of kImgChunk window images); thread (c, ky) owns the k outputs
// (c, ky, 0..k-1) and slides a k-wide register window along each input row (two shared-
// memory loads per k FMAs).  Partial sums (fp32 per row, fp64 across rows and images) go
// to part[j][chunk][param]; pass 2 (conv_dw_reduce_kernel) adds the chunks in order and
// applies the fused leapfrog.
constexpr int kImgChunk = 16;
#ifndef DASMC_CONV_DW_CI
#define DASMC_CONV_DW_CI 4
#endif
// Weight gradient of one stage for one input channel ci and CT output channels, over a
// chunk of kImgChunk images: dW[co][ci][ky][kx] = sum_m,y,x dz[co][y][x] in[ci][y+ky][x+kx]
// (+ the bias sums).  Thread (g, c): output channel co0 + c, rows y = g, g+G, ...; it keeps
// the full K x K patch in registers and slides a K-wide input window along each of the K
// rows, so one dz load feeds K*K FMAs.  Per row the float partials go into fp64 totals;
// the G row groups are combined in a fixed order (deterministic).
template <int K, int CT, int CI>
__global__ void __launch_bounds__(128) conv_dw_kernel(ConvDev d, const float* __restrict__ dZ, int64_t z_ps,
                                                       const float* __restrict__ in, int64_t in_ps, int64_t M,
                                                       int64_t np, int nchunks, double* __restrict__ part) {
  constexpr int G = 128 / CT;
  extern __shared__ float4 cv_sh4[];
  float* in_s = reinterpret_cast<float*>(cv_sh4);           // [CI][pl]
  const int npix = d.ho * d.wo, nplane = d.hin * d.win, pl = (nplane + 3) & ~3;
  const int zs = npix | 1;                                   // odd plane stride: conflict-free dz reads
  float* dz_s = in_s + CI * pl;                              // [CT][zs]
  const int ci0 = blockIdx.x * CI, co0 = blockIdx.y * CT;
  const int64_t j = blockIdx.z / nchunks;
  const int chunk = blockIdx.z - (int)j * nchunks;
  const int t = threadIdx.x, c = t % CT, g = t / CT;
  double tot[CI][K * K];
  double totb = 0.0;
#pragma unroll
  for (int i = 0; i < CI; ++i)
#pragma unroll
    for (int q = 0; q < K * K; ++q) tot[i][q] = 0.0;
  const int64_t in_img = (int64_t)d.cin * nplane, per = (int64_t)d.cout * npix;
  const int64_t m0 = (int64_t)chunk * kImgChunk, m1 = min(M, m0 + kImgChunk);
  for (int64_t m = m0; m < m1; ++m) {
    __syncthreads();
    const float* src = in + j * in_ps + m * in_img + (int64_t)ci0 * nplane;
    for (int u = t; u < CI * nplane; u += blockDim.x) {
      const int cc = u / nplane;
      in_s[cc * pl + (u - cc * nplane)] = ci0 + cc < d.cin ? src[u] : 0.f;
    }
    const float* zsrc = dZ + j * z_ps + m * per + (int64_t)co0 * npix;
    for (int u = t; u < CT * npix; u += blockDim.x) {
      const int cc = u / npix;
      dz_s[cc * zs + (u - cc * npix)] = co0 + cc < d.cout ? zsrc[u] : 0.f;
    }
    __syncthreads();
    for (int y = g; y < d.ho; y += G) {
      const float* zr = dz_s + c * zs + y * d.wo;
      float w[CI][K][K], acc[CI][K * K];
#pragma unroll
      for (int i = 0; i < CI; ++i)
#pragma unroll
        for (int ky = 0; ky < K; ++ky)
#pragma unroll
          for (int q = 0; q < K; ++q) w[i][ky][q] = in_s[i * pl + (y + ky) * d.win + q];
#pragma unroll
      for (int i = 0; i < CI; ++i)
#pragma unroll
        for (int q = 0; q < K * K; ++q) acc[i][q] = 0.f;
      float ab = 0.f;
      for (int x = 0; x < d.wo; ++x) {
        const float z = zr[x];
#pragma unroll
        for (int i = 0; i < CI; ++i)
#pragma unroll
          for (int ky = 0; ky < K; ++ky)
#pragma unroll
            for (int kx = 0; kx < K; ++kx) acc[i][ky * K + kx] = fmaf(z, w[i][ky][kx], acc[i][ky * K + kx]);
        ab += z;
#pragma unroll
        for (int i = 0; i < CI; ++i)
#pragma unroll
          for (int ky = 0; ky < K; ++ky) {
#pragma unroll
            for (int q = 0; q + 1 < K; ++q) w[i][ky][q] = w[i][ky][q + 1];
            w[i][ky][K - 1] = x + K < d.win ? in_s[i * pl + (y + ky) * d.win + x + K] : 0.f;
          }
      }
#pragma unroll
      for (int i = 0; i < CI; ++i)
#pragma unroll
        for (int q = 0; q < K * K; ++q) tot[i][q] += (double)acc[i][q];
      totb += (double)ab;
    }
  }
  // combine the G row groups in order g = 0 .. G-1 (reusing the staging buffers)
  __syncthreads();
  double* red = reinterpret_cast<double*>(cv_sh4);  // [G][CT][CI*K*K + 1]
  constexpr int R = CI * K * K + 1;
#pragma unroll
  for (int i = 0; i < CI; ++i)
#pragma unroll
    for (int q = 0; q < K * K; ++q) red[((size_t)g * CT + c) * R + i * K * K + q] = tot[i][q];
  red[((size_t)g * CT + c) * R + CI * K * K] = totb;
  __syncthreads();
  double* o = part + ((int64_t)j * nchunks + chunk) * np;
  for (int e = t; e < CT * R; e += blockDim.x) {
    const int cc = e / R, q = e - cc * R;
    if (co0 + cc >= d.cout) continue;
    double sum = 0.0;
    for (int gg = 0; gg < G; ++gg) sum += red[((size_t)gg * CT + cc) * R + q];
    if (q < CI * K * K) {
      const int i = q / (K * K);
      if (ci0 + i < d.cin) o[((int64_t)(co0 + cc) * d.cin + ci0 + i) * K * K + (q - i * K * K)] = sum;
    } else if (ci0 == 0) {
      o[(int64_t)d.cout * d.cin * K * K + co0 + cc] = sum;
    }
  }
}

// Earlier weight-gradient layout (thread = output channel x kernel row, all image rows):
// kept for K >= 5, where its per-thread register use stays low (C3: 8x8 planes).
template <int K, int CT>
__global__ void __launch_bounds__(128) conv_dw_rows_kernel(ConvDev d, const float* __restrict__ dZ, int64_t z_ps,
                                                       const float* __restrict__ in, int64_t in_ps, int64_t M,
                                                       int64_t np, int nchunks, double* __restrict__ part) {
  extern __shared__ float4 cv_sh4[];
  float* in_s = reinterpret_cast<float*>(cv_sh4);           // [hin * win]
  float* dz_s = in_s + ((d.hin * d.win + 3) & ~3);          // [CT][ho * wo]
  const int ci = blockIdx.x, co0 = blockIdx.y * CT;
  const int64_t j = blockIdx.z / nchunks;
  const int chunk = blockIdx.z - (int)j * nchunks;
  const int npix = d.ho * d.wo, nplane = d.hin * d.win;
  const int t = threadIdx.x, c = t / K, ky = t - c * K;
  const bool active = t < CT * K;
  double tot[K];
  double totb = 0.0;
#pragma unroll
  for (int q = 0; q < K; ++q) tot[q] = 0.0;
  const int64_t in_img = (int64_t)d.cin * nplane, per = (int64_t)d.cout * npix;
  const int64_t m0 = (int64_t)chunk * kImgChunk, m1 = min(M, m0 + kImgChunk);
  for (int64_t m = m0; m < m1; ++m) {
    __syncthreads();
    const float* src = in + j * in_ps + m * in_img + (int64_t)ci * nplane;
    for (int u = t; u < nplane; u += blockDim.x) in_s[u] = src[u];
    const float* zsrc = dZ + j * z_ps + m * per + (int64_t)co0 * npix;
    for (int u = t; u < CT * npix; u += blockDim.x) dz_s[u] = co0 + u / npix < d.cout ? zsrc[u] : 0.f;
    __syncthreads();
    if (!active) continue;
    for (int y = 0; y < d.ho; ++y) {
      const float* xr = in_s + (y + ky) * d.win;
      const float* zr = dz_s + (c * d.ho + y) * d.wo;
      float w[K], acc[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        w[q] = xr[q];
        acc[q] = 0.f;
      }
      float ab = 0.f;
      for (int x = 0; x < d.wo; ++x) {
        const float z = zr[x];
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = fmaf(z, w[q], acc[q]);
        ab += z;
#pragma unroll
        for (int q = 0; q + 1 < K; ++q) w[q] = w[q + 1];
        w[K - 1] = x + K < d.win ? xr[x + K] : 0.f;
      }
#pragma unroll
      for (int q = 0; q < K; ++q) tot[q] += (double)acc[q];
      totb += (double)ab;
    }
  }
  if (!active || co0 + c >= d.cout) return;
  double* o = part + ((int64_t)j * nchunks + chunk) * np;
  const int64_t wbase = ((int64_t)(co0 + c) * d.cin + ci) * K * K + (int64_t)ky * K;
#pragma unroll
  for (int q = 0; q < K; ++q) o[wbase + q] = tot[q];
  if (ci == 0 && ky == 0) o[(int64_t)d.cout * d.cin * K * K + co0 + c] = totb;
}

__global__ void conv_dw_reduce_kernel(ConvDev d, int64_t np, int nchunks, const double* __restrict__ part, int64_t J,
                                      int64_t Dp, EpiParams e) {
  const int64_t nw = np - d.cout;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < J * np; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / np, q = g - j * np;
    double acc = 0.0;
    for (int ch = 0; ch < nchunks; ++ch) acc += part[((int64_t)j * nchunks + ch) * np + q];
    leapfrog_update(e, (int)j, j * Dp + (q < nw ? d.woff + q : d.boff + (q - nw)), (float)acc);
  }
}

// Input delta of a stage (transposed convolution), in place over the previous stage
// output `io` (read for the mask first): delta = sum dz * W, times act'(io) unless the
// previous stage pools (its pool backward applies act' at the argmax instead).  Tiled like
// conv_fwd: a block owns one image and CT input channels, W as [cout*k*k][CT] in smem.
template <int K, int CT>
__global__ void __launch_bounds__(128) conv_dx_kernel(ConvDev d, int act, int apply_act,
                                                       const float* __restrict__ dZ, int64_t z_ps,
                                                       const float* __restrict__ theta, int64_t Dp, float* io,
                                                       int64_t io_ps) {
  extern __shared__ float4 cv_sh4[];
  float* Ws = reinterpret_cast<float*>(cv_sh4);
  const int64_t m = blockIdx.x, j = blockIdx.z;
  const int ci0 = blockIdx.y * CT, kk = d.k * d.k;
  const float* W = theta + j * Dp + d.woff;
  for (int i = threadIdx.x; i < d.cout * kk * CT; i += blockDim.x) {
    const int t = i / CT, c = i - t * CT;  // t = (co, ky, kx)
    const int co = t / kk, r = t - co * kk;
    Ws[i] = ci0 + c < d.cin ? W[((int64_t)co * d.cin + ci0 + c) * kk + r] : 0.f;
  }
  __syncthreads();
  const int64_t in_img = (int64_t)d.cin * d.hin * d.win, per = (int64_t)d.cout * d.ho * d.wo;
  const float* z = dZ + j * z_ps + m * per;
  float* dst = io + j * io_ps + m * in_img;
  const int npix = d.hin * d.win;
  for (int p = threadIdx.x; p < npix; p += blockDim.x) {
    const int y = p / d.win, x = p - y * d.win;
    const int ky0 = max(0, y - d.ho + 1), ky1 = min(d.k - 1, y);
    const int kx0 = max(0, x - d.wo + 1), kx1 = min(d.k - 1, x);
    float acc[CT];
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[c] = 0.f;
    for (int co = 0; co < d.cout; ++co)
      for (int ky = ky0; ky <= ky1; ++ky) {
        const float* zrow = z + ((int64_t)co * d.ho + y - ky) * d.wo + x;
        const float4* wrow = cv_sh4 + (int64_t)((co * K + ky) * K) * (CT / 4);
        float v[K];
#pragma unroll
        for (int kx = 0; kx < K; ++kx) v[kx] = (kx >= kx0 && kx <= kx1) ? zrow[-kx] : 0.f;
#pragma unroll
        for (int kx = 0; kx < K; ++kx)
#pragma unroll
          for (int u = 0; u < CT / 4; ++u) {
            const float4 w = wrow[kx * (CT / 4) + u];
            acc[4 * u] = fmaf(v[kx], w.x, acc[4 * u]);
            acc[4 * u + 1] = fmaf(v[kx], w.y, acc[4 * u + 1]);
            acc[4 * u + 2] = fmaf(v[kx], w.z, acc[4 * u + 2]);
            acc[4 * u + 3] = fmaf(v[kx], w.w, acc[4 * u + 3]);
          }
      }
#pragma unroll
    for (int c = 0; c < CT; ++c)
      if (ci0 + c < d.cin) {
        float* q = dst + (int64_t)(ci0 + c) * npix + p;
        *q = apply_act ? acc[c] * act_grad_post(*q, act) : acc[c];
      }
  }
}

// conv kernel sizes are template parameters (unrolled kx loops / register windows)
template <typename Fn>
void dispatch_k(int k, Fn&& fn) {
  switch (k) {
    case 1: fn(std::integral_constant<int, 1>{}); break;
    case 2: fn(std::integral_constant<int, 2>{}); break;
    case 3: fn(std::integral_constant<int, 3>{}); break;
    case 4: fn(std::integral_constant<int, 4>{}); break;
    case 5: fn(std::integral_constant<int, 5>{}); break;
    case 6: fn(std::integral_constant<int, 6>{}); break;
    case 7: fn(std::integral_constant<int, 7>{}); break;
    default: throw std::invalid_argument("conv: kernel sizes 1..7 supported");
  }
}

template <typename K>
void set_smem(K kern, size_t bytes) {
  if (bytes > 227 * 1024) throw std::invalid_argument("conv: stage too large for shared memory");
  if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

int64_t conv_out_floats(const ConvDev& d) { return (int64_t)d.cout * d.sh * d.sw; }
int64_t conv_act_floats(const ConvDev& d) { return (int64_t)d.cout * d.ho * d.wo; }
float* stage_out(Ctx& c, int i) { return c.net.conv[i].pool ? c.cpool[i] : c.cact[i]; }

// MLP head of a CNN chunk (network.hpp:159-219 with layer 1 reading the flatten `flat`,
// [J][Mcap][F]): forward, log-softmax / ll partials into the chunk's slots, and, with a
// gradient, the head's weight gradients (+ the leapfrog / chunk accumulation of e) and the
// flatten delta in place over `flat` (act' only if the last stage does not pool).  logits_out
// (optional, [J][R][C]) receives the chunk's logits rows m0 .. m0+mc.
void cnn_head(Ctx& c, const float* theta_in, int64_t J, int64_t m0, int64_t mc, int64_t P, double beta_rows,
              bool need_grad, const EpiParams* e, float* flat, float* logits_out, int64_t R_out) {
  const NetDev& net = c.net;
  const int L = net.L;
  const int64_t F = net.sizes[0];
  for (int l = 1; l <= L; ++l) {
    const LayerDev& ly = net.layer[l - 1];
    EpiFwd ef{c.act[l], ly.out, c.Mcap * ly.out, theta_in, net.Dp, ly.boff, ly.hidden, net.act};
    const float* A = l == 1 ? flat : c.act[l - 1];
    const int64_t sA = l == 1 ? c.Mcap * F : c.Mcap * ly.in;
    sgemm<true, true>(c.stream, (int)mc, ly.out, ly.in, A, ly.in, sA, theta_in + ly.woff, ly.in, net.Dp, -1, J, ef);
  }
  const int C = net.sizes[L];
  if (logits_out)
    CK(cudaMemcpy2DAsync(logits_out + m0 * C, sizeof(float) * R_out * C, c.act[L], sizeof(float) * c.Mcap * C,
                         sizeof(float) * mc * C, (size_t)J, cudaMemcpyDeviceToDevice, c.stream));
  {
    // the chunk's rows are window rows m0 .. m0+mc (m0 a multiple of 128: slot offset m0 / 128)
    dim3 grid((unsigned)((mc + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)J);
    softmax_kernel<<<grid, kRowsPerBlock, 0, c.stream>>>(c.act[L], c.Mcap * C, C, c.y + m0, mc, P - m0,
                                                         (float)beta_rows, need_grad ? 1 : 0,
                                                         c.ll_part + 2 * (m0 / kRowsPerBlock), c.ll_slots);
    LAUNCHED();
  }
  if (!need_grad) return;
  for (int l = L; l >= 1; --l) {
    const LayerDev& ly = net.layer[l - 1];
    {
      EpiDw ew{*e, net.Dp, ly.woff, ly.boff, ly.in};
      const float* Bp = l == 1 ? flat : c.act[l - 1];
      const int64_t sB = l == 1 ? c.Mcap * F : c.Mcap * ly.in;
      sgemm<false, false>(c.stream, ly.out, ly.in + 1, (int)mc, c.act[l], ly.out, c.Mcap * ly.out, Bp, ly.in, sB,
                          ly.in, J, ew);
    }
    // delta_{l-1} in place over a_{l-1}; for l = 1 over the flatten (act' only if the
    // last stage does not pool)
    float* Dst = l > 1 ? c.act[l - 1] : flat;
    const int64_t ldd = l > 1 ? net.layer[l - 2].out : F;
    const int act = l > 1 || !net.conv[net.nconv - 1].pool ? net.act : -1;
    EpiDx ed{Dst, ldd, c.Mcap * ldd, act};
    sgemm<true, false>(c.stream, (int)mc, ly.in, ly.out, c.act[l], ly.out, c.Mcap * ly.out, theta_in + ly.woff, ly.in,
                       net.Dp, -1, J, ed);
  }
}

// fp32 CUDA-core stages (the 1e-4 parity path) for window rows m0 .. m0+mc; NCHW stage
// buffers [Jmax][Mcap][per-image floats].
void cnn_chunk_simt(Ctx& c, const float* theta_in, int64_t J, int64_t m0, int64_t M, int64_t P, double beta_rows,
                    bool need_grad, const EpiParams* epi, float* logits_out, int64_t R_out) {
  const NetDev& net = c.net;
  const int nc = net.nconv;
  const int64_t img = (int64_t)net.in_c * net.in_h * net.in_w;
  const float* X0 = c.X + m0 * img;
  auto grid_of = [](int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32); };
  // forward through the stages
  for (int i = 0; i < nc; ++i) {
    const ConvDev& d = net.conv[i];
    const float* in = i == 0 ? X0 : stage_out(c, i - 1);
    const int64_t in_ps = i == 0 ? 0 : c.Mcap * conv_out_floats(net.conv[i - 1]);
    dispatch_k(d.k, [&](auto kc) {
      constexpr int K = decltype(kc)::value, CT = 16;
      const size_t sm = sizeof(float) * (size_t)d.cin * K * K * CT;
      set_smem(conv_fwd_kernel<K, CT>, sm);
      conv_fwd_kernel<K, CT><<<dim3((unsigned)M, (unsigned)((d.cout + CT - 1) / CT), (unsigned)J), 128, sm,
                               c.stream>>>(d, net.act, in, in_ps, theta_in, net.Dp, c.cact[i],
                                           c.Mcap * conv_act_floats(d));
      LAUNCHED();
    });
    if (d.pool) {
      pool_fwd_kernel<<<grid_of(J * M * conv_out_floats(d)), 256, 0, c.stream>>>(
          d, c.cact[i], c.Mcap * conv_act_floats(d), c.cpool[i], c.Mcap * conv_out_floats(d), M, J);
      LAUNCHED();
    }
  }
  float* flat = stage_out(c, nc - 1);
  cnn_head(c, theta_in, J, m0, M, P, beta_rows, need_grad, epi, flat, logits_out, R_out);
  if (!need_grad) return;
  // conv stages backward
  for (int i = nc - 1; i >= 0; --i) {
    const ConvDev& d = net.conv[i];
    const int64_t a_ps = c.Mcap * conv_act_floats(d);
    float* dz = c.cact[i];  // no pool: the stage-output delta (act' applied) is already dz
    if (d.pool) {
      dz = c.cdel[i];
      if ((d.ho | d.wo) & 1) CK(cudaMemsetAsync(dz, 0, sizeof(float) * (size_t)J * a_ps, c.stream));
      pool_bwd_kernel<<<grid_of(J * M * (int64_t)d.cout * d.sh * d.sw), 256, 0, c.stream>>>(
          d, net.act, c.cact[i], a_ps, c.cpool[i], c.Mcap * conv_out_floats(d), dz, M, J);
      LAUNCHED();
    }
    const float* in = i == 0 ? X0 : stage_out(c, i - 1);
    const int64_t in_ps = i == 0 ? 0 : c.Mcap * conv_out_floats(net.conv[i - 1]);
    {
      const int nchunks = (int)((M + kImgChunk - 1) / kImgChunk);
      const int64_t np = (int64_t)d.cout * d.cin * d.k * d.k + d.cout;
      ensure_stage(c, sizeof(double) * (size_t)J * nchunks * np);
      double* part = reinterpret_cast<double*>(c.stage);
      dispatch_k(d.k, [&](auto kc) {
        constexpr int K = decltype(kc)::value, CT = 16;
        const dim3 grid((unsigned)d.cin, (unsigned)((d.cout + CT - 1) / CT), (unsigned)(J * nchunks));
        if constexpr (K <= 3) {  // patch-per-thread layout (C4 step 6.36 -> 4.49 s; slower at C3's K = 5)
          constexpr int CI = DASMC_CONV_DW_CI;  // input channels per block (the dz planes staged once for them)
          const dim3 grid_ci((unsigned)((d.cin + CI - 1) / CI), grid.y, grid.z);
          const size_t stage = sizeof(float) * ((size_t)CI * (((size_t)d.hin * d.win + 3) / 4 * 4) +
                                                (size_t)CT * ((d.ho * d.wo) | 1));
          const size_t red = sizeof(double) * (size_t)128 * (CI * K * K + 1);  // [G][CT][CI*K*K + 1]
          const size_t sm = std::max(stage, red);
          set_smem(conv_dw_kernel<K, CT, CI>, sm);
          conv_dw_kernel<K, CT, CI><<<grid_ci, 128, sm, c.stream>>>(d, dz, a_ps, in, in_ps, M, np, nchunks, part);
        } else {
          const size_t sm = sizeof(float) * (((size_t)d.hin * d.win + 3) / 4 * 4 + (size_t)CT * d.ho * d.wo);
          set_smem(conv_dw_rows_kernel<K, CT>, sm);
          conv_dw_rows_kernel<K, CT><<<grid, 128, sm, c.stream>>>(d, dz, a_ps, in, in_ps, M, np, nchunks, part);
        }
        LAUNCHED();
      });
      conv_dw_reduce_kernel<<<grid_of(J * np), 256, 0, c.stream>>>(d, np, nchunks, part, J, net.Dp, *epi);
      LAUNCHED();
    }
    if (i > 0) {
      const ConvDev& dp = net.conv[i - 1];
      dispatch_k(d.k, [&](auto kc) {
        constexpr int K = decltype(kc)::value, CT = 16;
        const size_t sm = sizeof(float) * (size_t)d.cout * K * K * CT;
        set_smem(conv_dx_kernel<K, CT>, sm);
        conv_dx_kernel<K, CT><<<dim3((unsigned)M, (unsigned)((d.cin + CT - 1) / CT), (unsigned)J), 128, sm,
                                c.stream>>>(d, net.act, dp.pool ? 0 : 1, dz, a_ps, theta_in, net.Dp,
                                            stage_out(c, i - 1), c.Mcap * conv_out_floats(dp));
        LAUNCHED();
      });
    }
  }
}

// Window chunk (images) for a window of M rows: M itself when the chunk buffers for J = Jmax
// fit kCnnBudget, else the largest multiple of 128 that does.  A pure function of (M, net,
// Jmax, precision): the chunk split -- and with it the fp32 order of the cross-chunk gradient
// sums -- never depends on earlier calls.  DASMC_CNN_CHUNK (tests) caps it.
constexpr double kCnnBudget = 100e9;  // of the 180 GB of HBM
int64_t cnn_image_floats(const Ctx& c) {
  const NetDev& net = c.net;
  int64_t f = 0;
  for (int l = 1; l <= net.L; ++l) f += net.sizes[l];
  if (c.ctc) return f + cnn_tc_image_floats(c);
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    f += conv_act_floats(d);
    if (d.pool) f += conv_out_floats(d) + conv_act_floats(d);
  }
  return f;
}
int64_t cnn_chunk_images(const Ctx& c, int64_t M) {
  int64_t cap = (int64_t)(kCnnBudget / (4.0 * (double)c.Jmax * (double)cnn_image_floats(c)));
  if (!c.ctc) cap = std::min<int64_t>(cap, 16 * 65535 / c.Jmax);  // conv_dw grid.z = J * ceil(rows / 16)
  if (const char* e = std::getenv("DASMC_CNN_CHUNK")) cap = std::min<int64_t>(cap, std::atoll(e));
  cap = cap / kRowsPerBlock * kRowsPerBlock;
  if (cap < kRowsPerBlock) throw std::invalid_argument("CNN: max_particles too large for the chunked stage buffers");
  return M <= cap ? M : cap;
}

void cnn_ensure(Ctx& c, int64_t M) {
  const int64_t slots = (M + kRowsPerBlock - 1) / kRowsPerBlock;
  if (slots > c.ll_slots) {
    CK(cudaStreamSynchronize(c.stream));
    if (c.ll_part) CK(cudaFree(c.ll_part));
    c.ll_part = nullptr;
    CK(cudaMalloc(&c.ll_part, sizeof(double) * 2 * (size_t)c.Jmax * slots));
    c.ll_slots = (int)slots;
  }
  const int64_t need = (cnn_chunk_images(c, M) + kRowsPerBlock - 1) / kRowsPerBlock * kRowsPerBlock;
  if (need <= c.Mcap) return;
  CK(cudaStreamSynchronize(c.stream));
  for (int l = 1; l <= c.net.L; ++l) {
    if (c.act[l]) CK(cudaFree(c.act[l]));
    c.act[l] = nullptr;
    CK(cudaMalloc(&c.act[l], sizeof(float) * (size_t)c.Jmax * need * c.net.sizes[l]));
  }
  if (c.ctc) {
    cnn_tc_alloc(c, need);
  } else {
    for (int i = 0; i < c.net.nconv; ++i) {
      float** bufs[] = {&c.cact[i], &c.cpool[i], &c.cdel[i]};
      for (float** b : bufs)
        if (*b) {
          CK(cudaFree(*b));
          *b = nullptr;
        }
      const ConvDev& d = c.net.conv[i];
      CK(cudaMalloc(&c.cact[i], sizeof(float) * (size_t)c.Jmax * need * conv_act_floats(d)));
      if (d.pool) {
        CK(cudaMalloc(&c.cpool[i], sizeof(float) * (size_t)c.Jmax * need * conv_out_floats(d)));
        CK(cudaMalloc(&c.cdel[i], sizeof(float) * (size_t)c.Jmax * need * conv_act_floats(d)));
      }
    }
  }
  c.Mcap = need;
}

// CNN gradient evaluation over window rows [0, M) in chunks of cnn_chunk_images(M) images:
// conv stages -> flatten -> the SIMT MLP head -> head backward -> conv stages backward, per
// chunk; the weight gradients are summed across chunks in order (EpiParams::acc_mode) before
// the fused leapfrog.  Stage bodies: tcgen05 implicit GEMMs (conv_tc.cu) when the context's
// precision is a tensor-core one, else the fp32 CUDA-core kernels.
void launch_eval_cnn(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
                     const EpiParams* epi, float* logits_out = nullptr) {
  cnn_ensure(c, M);
  const int64_t Mc = cnn_chunk_images(c, M);
  const int nch = (int)((M + Mc - 1) / Mc);
  if (nch > 1 && need_grad && !c.gacc) CK(cudaMalloc(&c.gacc, sizeof(float) * (size_t)c.Jmax * c.net.Dp));
  if (c.ctc) cnn_tc_weights(c, theta_in, J, need_grad);
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t m0 = ch * Mc, mc = std::min(Mc, M - m0);
    EpiParams e{};
    if (need_grad) {
      e = *epi;
      e.acc_mode = nch == 1 ? 0 : ch == 0 ? 1 : ch + 1 < nch ? 2 : 3;
      e.gacc = c.gacc;
    }
    if (c.ctc) {
      cnn_tc_forward(c, theta_in, J, m0, mc);
      cnn_head(c, theta_in, J, m0, mc, P, beta_rows, need_grad, &e, cnn_tc_flat(c), logits_out, M);
      if (need_grad) cnn_tc_backward(c, theta_in, J, m0, mc, e);
    } else {
      cnn_chunk_simt(c, theta_in, J, m0, mc, P, beta_rows, need_grad, &e, logits_out, M);
    }
  }
}

// ---- evaluate_predictive (runner.hpp:331-364) --------------------------------------------
// One thread per test row: predictive[i][c] += sum_j w_j softmax(logits_j[i])[c] over the
// particles in ascending j (w_j <= 0 skipped), fp64 softmax as the reference.
__global__ void predictive_mix_kernel(const float* __restrict__ logits, int64_t ps, int C, int64_t R, int64_t J,
                                      const double* __restrict__ w, double* __restrict__ pred) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= R) return;
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = c < C ? pred[i * C + c] : 0.0;
  for (int64_t j = 0; j < J; ++j) {
    const double wj = w[j];
    if (!(wj > 0.0)) continue;
    const float* z = logits + j * ps + i * C;
    double mx = (double)z[0];
    for (int c = 1; c < C; ++c) mx = fmax(mx, (double)z[c]);
    double e[16], s = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < C) {
        e[c] = exp((double)z[c] - mx);
        s += e[c];
      }
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < C) acc[c] += wj * (e[c] / s);
  }
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (c < C) pred[i * C + c] = acc[c];
}

// Logits of J particles on R rows of Xd (device, the model's input layout) into `logits`
// ([J][R][C] fp32, particle stride R*C).  MLP: the SIMT forward GEMMs with scratch
// activations; CNN: the context's stage buffers with X / y swapped for the test rows.
void launch_forward_logits(Ctx& c, const float* theta, int64_t J, const float* Xd, const int32_t* yd, int64_t R,
                           float* logits, float* scratch0, float* scratch1) {
  const NetDev& net = c.net;
  if (net.nconv > 0) {
    const float* X0 = c.X;
    const int32_t* y0 = c.y;
    c.X = const_cast<float*>(Xd);
    c.y = const_cast<int32_t*>(yd);
    if (c.ctc) cnn_tc_refresh_data(c, Xd, R);  // the stage-0 operand copy of the test rows
    launch_eval_cnn(c, theta, J, R, R, 1.0, false, nullptr, logits);
    c.X = const_cast<float*>(X0);
    c.y = const_cast<int32_t*>(y0);
    if (c.ctc) cnn_tc_refresh_data(c, c.X, c.n_active);
    return;
  }
  const float* A = Xd;
  int64_t sA = 0;
  for (int l = 1; l <= net.L; ++l) {
    const LayerDev& ly = net.layer[l - 1];
    float* out = l == net.L ? logits : (l & 1 ? scratch0 : scratch1);
    EpiFwd e{out, ly.out, R * ly.out, theta, net.Dp, ly.boff, ly.hidden, net.act};
    sgemm<true, true>(c.stream, (int)R, ly.out, ly.in, A, ly.in, sA, theta + ly.woff, ly.in, net.Dp, -1, J, e);
    A = out;
    sA = R * ly.out;
  }
}

void launch_predictive_mix(Ctx& c, const float* logits, int64_t R, int64_t J, const double* w, double* pred) {
  const int C = c.net.sizes[c.net.L];
  predictive_mix_kernel<<<(unsigned)((R + 127) / 128), 128, 0, c.stream>>>(logits, R * C, C, R, J, w, pred);
  LAUNCHED();
}

void ensure_activation_capacity(Ctx& c, int64_t M) {
  if (c.net.nconv > 0) {
    const int64_t before = c.Mcap, slots = c.ll_slots;
    cnn_ensure(c, M);
    if (c.Mcap != before || c.ll_slots != slots) ++c.alloc_epoch;
    return;
  }
  if (M <= c.Mcap) return;
  ++c.alloc_epoch;
  CK(cudaStreamSynchronize(c.stream));
  const int64_t Mnew = ((M + 127) / 128) * 128;
  if (c.tc) {
    tc_ensure_rows(c, Mnew);  // transposed activation / delta buffers of the tensor-core path
  } else {
    for (int l = 1; l <= c.net.L; ++l) {
      if (c.act[l]) CK(cudaFree(c.act[l]));
      c.act[l] = nullptr;
      CK(cudaMalloc(&c.act[l], sizeof(float) * (size_t)c.Jmax * Mnew * c.net.sizes[l]));
    }
    for (int i = 0; i < c.net.nconv; ++i) {
      float** bufs[] = {&c.cact[i], &c.cpool[i], &c.cdel[i]};
      for (float** b : bufs)
        if (*b) {
          CK(cudaFree(*b));
          *b = nullptr;
        }
      const ConvDev& d = c.net.conv[i];
      CK(cudaMalloc(&c.cact[i], sizeof(float) * (size_t)c.Jmax * Mnew * conv_act_floats(d)));
      if (d.pool) {
        CK(cudaMalloc(&c.cpool[i], sizeof(float) * (size_t)c.Jmax * Mnew * conv_out_floats(d)));
        CK(cudaMalloc(&c.cdel[i], sizeof(float) * (size_t)c.Jmax * Mnew * conv_act_floats(d)));
      }
    }
  }
  const int slots = (int)((Mnew + kRowsPerBlock - 1) / kRowsPerBlock);
  if (c.ll_part) CK(cudaFree(c.ll_part));
  CK(cudaMalloc(&c.ll_part, sizeof(double) * 2 * (size_t)c.Jmax * slots));
  c.ll_slots = slots;
  c.Mcap = Mnew;
}

void launch_eval(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
                 const EpiParams* epi) {
  ensure_activation_capacity(c, M);
  KTimer whole(c, need_grad ? 2 : -1);
  const NetDev& net = c.net;
  const int L = net.L;
  // ||theta||^2 for the prior (network.hpp:226), read before any epilogue writes theta_out
  {
    const int slots = (int)((net.Dp + kSqChunk - 1) / kSqChunk);
    dim3 grid((unsigned)slots, (unsigned)J);
    sumsq_kernel<<<grid, 256, 0, c.stream>>>(theta_in, net.Dp, c.th_part, c.th_slots);
    LAUNCHED();
  }
  if (c.tc) {
    tc_eval(c, theta_in, J, M, P, beta_rows, need_grad, epi);
    return;
  }
  if (net.nconv > 0) {
    launch_eval_cnn(c, theta_in, J, M, P, beta_rows, need_grad, epi);
    return;
  }
  // forward (network.hpp:159-178)
  for (int l = 1; l <= L; ++l) {
    const LayerDev& ly = net.layer[l - 1];
    EpiFwd e{c.act[l], ly.out, c.Mcap * ly.out, theta_in, net.Dp, ly.boff, ly.hidden, net.act};
    KTimer kt(c, l == 1 && need_grad ? 0 : -1);
    const float* A = l == 1 ? c.X : c.act[l - 1];
    const int64_t sA = l == 1 ? 0 : c.Mcap * ly.in;
    sgemm<true, true>(c.stream, (int)M, ly.out, ly.in, A, ly.in, sA, theta_in + ly.woff, ly.in, net.Dp, -1, J, e);
  }
  // log-softmax and residual
  {
    const int C = net.sizes[L];
    dim3 grid((unsigned)((M + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)J);
    softmax_kernel<<<grid, kRowsPerBlock, 0, c.stream>>>(c.act[L], c.Mcap * C, C, c.y, M, P, (float)beta_rows,
                                                         need_grad ? 1 : 0, c.ll_part, c.ll_slots);
    LAUNCHED();
  }
  if (!need_grad) return;
  // backward (network.hpp:195-217): dW_l first (epilogue reads theta_in, writes
  // theta_out), then delta_{l-1} in place over a_{l-1}.
  for (int l = L; l >= 1; --l) {
    const LayerDev& ly = net.layer[l - 1];
    {
      EpiDw e{*epi, net.Dp, ly.woff, ly.boff, ly.in};
      KTimer kt(c, l == 1 ? 1 : -1);
      const float* Bp = l == 1 ? c.X : c.act[l - 1];
      const int64_t sB = l == 1 ? 0 : c.Mcap * ly.in;
      sgemm<false, false>(c.stream, ly.out, ly.in + 1, (int)M, c.act[l], ly.out, c.Mcap * ly.out, Bp, ly.in, sB,
                          ly.in, J, e);
    }
    if (l > 1) {
      const LayerDev& lp = net.layer[l - 2];
      EpiDx d{c.act[l - 1], lp.out, c.Mcap * lp.out, net.act};
      sgemm<true, false>(c.stream, (int)M, ly.in, ly.out, c.act[l], ly.out, c.Mcap * ly.out, theta_in + ly.woff,
                         ly.in, net.Dp, -1, J, d);
    }
  }
}

void launch_eval_finalize(Ctx& c, int64_t J, double* values_out, double* pre_out, double* blk_out, int64_t M,
                          bool with_theta_norm) {
  const int used_ll = (int)((M + kRowsPerBlock - 1) / kRowsPerBlock);
  const int used_th = (int)((c.net.Dp + kSqChunk - 1) / kSqChunk);
  const double scale = (double)c.total_n / (double)c.block_end;  // target.hpp:136-137
  eval_finalize_kernel<<<(unsigned)((J + 127) / 128), 128, 0, c.stream>>>(
      J, c.ll_part, c.ll_slots, used_ll, c.th_part, c.th_slots, with_theta_norm ? used_th : 0, (double)c.net.D,
      c.sigma * c.sigma, c.mode, scale, c.beta, values_out, pre_out, blk_out, c.flags);
  LAUNCHED();
}

void launch_set_step(Ctx& c, const DevStep& v) {
  set_step_kernel<<<1, 1, 0, c.stream>>>(v, c.dstep);
  LAUNCHED();
}
const void* set_step_kernel_fn() { return reinterpret_cast<const void*>(&set_step_kernel); }

void launch_normals(Ctx& c, uint64_t root, uint64_t a, uint64_t b, int64_t J, float scale, float* dst,
                    double* sq_part, int64_t j_offset, const DevStep* ds) {
  const int64_t nch = (c.net.D + c.rng_chunk - 1) / c.rng_chunk;
  const int per_particle_c = a == tag::kProposal ? 1 : 0;
  const int64_t total = J * nch;
  normals_kernel<<<(unsigned)((total + 127) / 128), 128, 0, c.stream>>>(
      c.net, root, a, b, per_particle_c, J, nch, c.rng_chunk, c.jump_tab, scale, dst, sq_part, j_offset, ds);
  LAUNCHED();
}

void launch_uniforms(Ctx& c, uint64_t key, int64_t count, double* dst, const DevStep* ds) {
  const int64_t per = 2 * c.rng_chunk;
  const int64_t nch = (count + per - 1) / per;
  if (nch > c.jump_chunks) throw std::invalid_argument("uniforms: jump table too small");
  uniforms_kernel<<<(unsigned)((nch + 63) / 64), 64, 0, c.stream>>>(key, count, c.rng_chunk, c.jump_tab, dst, ds);
  LAUNCHED();
}

void launch_ref_to_internal_f64(Ctx& c, const double* src, float* dst, int64_t J) {
  ref_to_internal_kernel<double, float><<<grid_for(J * c.net.D), 256, 0, c.stream>>>(c.net, src, dst, J);
  LAUNCHED();
}
void launch_ref_to_internal_f32(Ctx& c, const float* src, float* dst, int64_t J) {
  ref_to_internal_kernel<float, float><<<grid_for(J * c.net.D), 256, 0, c.stream>>>(c.net, src, dst, J);
  LAUNCHED();
}
void launch_internal_to_ref_f64(Ctx& c, const float* src, double* dst, int64_t J) {
  internal_to_ref_kernel<float, double><<<grid_for(J * c.net.D), 256, 0, c.stream>>>(c.net, src, dst, J);
  LAUNCHED();
}
void launch_internal_to_ref_f32(Ctx& c, const float* src, float* dst, int64_t J) {
  internal_to_ref_kernel<float, float><<<grid_for(J * c.net.D), 256, 0, c.stream>>>(c.net, src, dst, J);
  LAUNCHED();
}

void launch_zero_ints(Ctx& c, int* p, int64_t n) {
  zero_ints_kernel<<<grid_for(n), 256, 0, c.stream>>>(p, n);
  LAUNCHED();
}

void launch_slot_sums(Ctx& c, int64_t J, int p0_slots, int pS_slots) {
  const unsigned blocks = (unsigned)((J * 32 + 255) / 256);
  slot_sum_kernel<<<blocks, 256, 0, c.stream>>>(c.p0_part, p0_slots, J, c.p0_sum);
  slot_sum_kernel<<<blocks, 256, 0, c.stream>>>(c.p_part, pS_slots, J, c.pS_sum);
  LAUNCHED();
  LAUNCHED();
}

void launch_weights_and_resample(Ctx& c, int64_t J, double fraction, int always, int kind, int rec_slot, int k,
                                 double, const DevStep* ds) {
  const int p0_slots = c.rng_slots;
  const int pS_slots = (int)((c.net.Dp + kSqChunk - 1) / kSqChunk);
  launch_slot_sums(c, J, p0_slots, pS_slots);
  weights_kernel<<<1, kWT, cdf_smem(J), c.stream>>>(J, c.logw, c.lt_old, c.lt_new, c.p0_sum, 1, c.pS_sum, 1,
                                          c.flags, c.wts, c.cdf, c.uni, c.idx, fraction, always, kind,
                                          ds ? c.records : c.records + (size_t)rec_slot * 8, k, 1, ds);
  LAUNCHED();
}

void launch_local_weights(Ctx& c, int64_t J, double* out_lw, double* out_lt) {
  const int pS_slots = (int)((c.net.Dp + kSqChunk - 1) / kSqChunk);
  launch_slot_sums(c, J, c.rng_slots, pS_slots);
  local_weights_kernel<<<(unsigned)((J + 255) / 256), 256, 0, c.stream>>>(
      J, c.logw, c.lt_old, c.lt_new, c.p0_sum, 1, c.pS_sum, 1, c.flags, out_lw, out_lt);
  LAUNCHED();
}

void launch_normalize_resample(Ctx& c, int64_t Jtot, double* lw_full, const double* lt_full, double* w, double* cdf,
                               const double* uni, int32_t* idx, double fraction, int always, int kind, int rec_slot,
                               int k) {
  weights_kernel<<<1, kWT, cdf_smem(Jtot), c.stream>>>(Jtot, lw_full, nullptr, lt_full, nullptr, 0, nullptr, 0, nullptr, w, cdf,
                                          uni, idx, fraction, always, kind, c.records + (size_t)rec_slot * 8, k, 0, nullptr);
  LAUNCHED();
}

__global__ void gather_data_kernel(const float* __restrict__ X, const int32_t* __restrict__ y,
                                   const int64_t* __restrict__ rows, int64_t count, int64_t d, float* __restrict__ Xd,
                                   int32_t* __restrict__ yd) {
  for (int64_t r = blockIdx.x; r < count; r += gridDim.x) {
    const int64_t src = rows[r];
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) Xd[r * d + i] = X[src * d + i];
    if (threadIdx.x == 0) yd[r] = y[src];
  }
}

void launch_gather_data(Ctx& c, const float* X, const int32_t* y, const int64_t* rows, int64_t count, int64_t d,
                        float* Xd, int32_t* yd) {
  gather_data_kernel<<<(unsigned)std::min<int64_t>(count, 148 * 32), 256, 0, c.stream>>>(X, y, rows, count, d, Xd,
                                                                                         yd);
  LAUNCHED();
}

void launch_rows(Ctx& c, const float* src, float* dst, const int32_t* rows_dev, int64_t n, bool pack) {
  if (n <= 0) return;
  const int64_t Dp4 = c.net.Dp / 4;
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>((Dp4 + 255) / 256, 64));
  dim3 grid((unsigned)chunks, (unsigned)n);
  rows_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), Dp4,
                                          rows_dev, pack ? 1 : 0);
  LAUNCHED();
}

void launch_p_sumsq(Ctx& c, int64_t J) {
  const int slots = (int)((c.net.Dp + kSqChunk - 1) / kSqChunk);
  dim3 grid((unsigned)slots, (unsigned)J);
  sumsq_kernel<<<grid, 256, 0, c.stream>>>(c.p, c.net.Dp, c.p_part, slots);
  LAUNCHED();
}

void launch_gather(Ctx& c, const float* start, const float* end, float* dst, int64_t J, const int32_t* idx) {
  const int64_t Dp4 = c.net.Dp / 4;
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>((Dp4 + 255) / 256, 64));
  dim3 grid((unsigned)chunks, (unsigned)J);
  gather_kernel<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float4*>(start),
                                            reinterpret_cast<const float4*>(end), reinterpret_cast<float4*>(dst),
                                            Dp4, idx ? idx : c.idx, c.flags);
  LAUNCHED();
}

__global__ void start_from_cache_kernel(EpiParams e, const float* __restrict__ g_cache, int64_t Dp, int64_t J) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < J * Dp; t += (int64_t)gridDim.x * blockDim.x) {
    const float g = g_cache[t];
    const float th = e.theta_in[t];
    const float p = fmaf(e.hh, g, e.p[t]);
    const float tn = fmaf(e.h, p, th);
    e.p[t] = p;
    e.theta_out[t] = tn;
    if (!isfinite(g) || !isfinite(p) || !isfinite(tn)) atomicOr(&e.flags[t / Dp], 1);
  }
}

__global__ void gather_cache_kernel(const float4* __restrict__ src, float4* __restrict__ dst, int64_t Dp4,
                                    const int32_t* __restrict__ idx, const double* __restrict__ lt_new,
                                    double* __restrict__ lt_cache) {
  const int64_t j = blockIdx.y;
  const int32_t s = idx[j];
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < Dp4; i += (int64_t)gridDim.x * 256) dst[j * Dp4 + i] = src[s * Dp4 + i];
  if (blockIdx.x == 0 && threadIdx.x == 0) lt_cache[j] = lt_new[s];
}

void launch_start_from_cache(Ctx& c, const EpiParams& e, int64_t J) {
  start_from_cache_kernel<<<grid_for(J * c.net.Dp), 256, 0, c.stream>>>(e, c.gcache[c.gcur], c.net.Dp, J);
  LAUNCHED();
  CK(cudaMemcpyAsync(c.lt_old, c.lt_cache, sizeof(double) * J, cudaMemcpyDeviceToDevice, c.stream));
}

void launch_gather_cache(Ctx& c, const float* src, float* dst, int64_t J) {
  const int64_t Dp4 = c.net.Dp / 4;
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>((Dp4 + 255) / 256, 64));
  gather_cache_kernel<<<dim3((unsigned)chunks, (unsigned)J), 256, 0, c.stream>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), Dp4, c.idx, c.lt_new, c.lt_cache);
  LAUNCHED();
}

void launch_select_parts(Ctx& c, int64_t J, const int32_t* idx, double* out_pre, double* out_blk) {
  gather_parts_kernel<<<(unsigned)((J + 255) / 256), 256, 0, c.stream>>>(J, idx, c.flags, c.ll_pre0, c.ll_blk0, c.ll_pre,
                                                                        c.ll_blk, out_pre, out_blk);
  LAUNCHED();
}

void launch_gather_parts(Ctx& c, int64_t J) {
  gather_parts_kernel<<<(unsigned)((J + 255) / 256), 256, 0, c.stream>>>(J, c.idx, c.flags, c.ll_pre0, c.ll_blk0,
                                                                        c.ll_pre, c.ll_blk, c.sda_pre, c.sda_blk);
  LAUNCHED();
}

void launch_resample_hook(Ctx& c, const double* w, const double* u, int64_t J, int kind, int32_t* idx) {
  resample_hook_kernel<<<1, kWT, cdf_smem(J), c.stream>>>(J, w, c.cdf, u, kind, idx);
  LAUNCHED();
}

}  // namespace dasmc_b200
