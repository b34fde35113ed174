// [EXT] CNN stages (BASELINE.json configs[2..3]) on the tcgen05 tensor cores: implicit-GEMM
// convolutions.  The reference is MLP-only; its contraction sites (network.hpp:171-173 forward,
// 203-209 dW and delta) are generalised to the convolution stages of dasmc_gpu.h's conv
// descriptor, with the oracle's semantics (oracle/dasmc_oracle.hpp CnnSpec: valid stride-1
// convolutions, activation, optional 2x2/2 max-pool with floor, first-max routing).
//
// One gather-GEMM kernel serves all three contractions of a stage, per particle j:
//   forward  Z[r, co]   = sum_q A[r, q] W[co, q]      r = output pixel (image, y, x), q = (ky, kx, ci)
//   delta    dI[r, ci]  = sum_q dZpad[r, q] W'[ci, q] r = input pixel, q = (ky, kx, co)
//   weights  dW[i, co]  = sum_r In[i, r] dZ[co, r]    i = (ky, kx, ci) (+ the bias row of ones)
// Operands are never materialised as im2col matrices in HBM: four producer warps gather each
// 128 x 32 tf32 k-block straight from the NHWC activation buffers into the 128B-swizzled
// K-major shared-memory layout the UMMA reads, with cp.async (16-byte chunks when four
// consecutive k are contiguous channels, else 4-byte elements), element offsets taken from
// small per-stage row / column tables (row part + column part), and zero fill past the edges.
// cp.async.mbarrier.arrive completes the stage's full barrier; one thread issues
// tcgen05.mma kind::tf32 (M = 128, N <= 256, K = 8) into double-buffered TMEM accumulators;
// four epilogue warps drain them (tcgen05.ld) with the fused epilogue:
//   forward: bias + activation, tf32-rounded NHWC store (the next stage's operand);
//   delta:   times act'(mask) (or identity before a max-pool), store into the previous stage's
//            zero-bordered delta buffer (so the next delta GEMM needs no bounds checks);
//   weights: the fused leapfrog (epi.cuh), with the chunked-window accumulation.
// Activations are stored tf32-rounded (round to nearest), so the MMA's operand truncation
// does not bias the long sums (same rule as tc_gemm.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <vector>

#include "conv_tc.cuh"
#include "epi.cuh"
#include "tc_ptx.cuh"

namespace dasmc_b200 {

namespace {

#ifndef DASMC_CONV_PW
#define DASMC_CONV_PW 8  // gather producer warps per CTA
#endif
#ifndef DASMC_CONV_GEW
#define DASMC_CONV_GEW 4  // epilogue warps of the gather kernels (4 or 8)
#endif
#ifndef DASMC_CONV_MINB
#define DASMC_CONV_MINB 1  // CTAs per SM the register budget is sized for
#endif
constexpr int kCBM = 128;              // UMMA M
constexpr int kCBK = 32;               // tf32 elements per 128-byte swizzle row (one k-block)
constexpr int kProdWarps = DASMC_CONV_PW;  // gather producers
// warps per CTA: gather mode = kProdWarps producers + MMA warp + 4 epilogue warps; direct mode =
// one TMA warp + MMA warp + 8 epilogue warps (two per TMEM lane group, splitting the columns:
// the direct tiles are epilogue-heavy)
// TMA weight gradient (direct + weights): one TMA warp + kShiftWarps shifter warps (they build the k
// kx-shifted B tiles of a k block from one unshifted staging tile in shared memory) + MMA warp + 8
// epilogue warps
constexpr int kShiftWarps = 8;
// FWDG (the gather-mode forward): 4 producers + 8 epilogue warps instead of 8 + 4 -- its tiles are one or a
// few k blocks feeding up to 256 output columns, and one epilogue warp per scheduler ran its long dependent
// instruction stream (TMEM load, bias, activation, rounding, 4 + 16 stores per 16 columns) at a fraction of
// the issue rate; the thread count and so the register budget stay the same
template <bool DIRECT, bool DWT = false, bool FWDG = false>
struct ConvWarps {
  static constexpr int P = DWT ? 1 + kShiftWarps : DIRECT ? 1 : FWDG ? kProdWarps / 2 : kProdWarps,
                       E = DIRECT && !DWT ? 8 : DIRECT ? 4 : FWDG ? 2 * DASMC_CONV_GEW : DASMC_CONV_GEW,
                       T = 32 * (P + 1 + E);
};
constexpr int kOnesRow = -2147483647;  // row table entry: a row of ones (the bias row of dW)
constexpr int kZeroRow = -2147483647 - 1;

struct GOperand {
  const float* base;
  int64_t ps;          // particle stride (floats); 0 = shared by all particles
  const int* rowoff;   // element offset of row i (nullptr: i * ld)
  int ld;
  int nrows;           // rows >= nrows are zero
  const int* coloff;   // element offset of column q (nullptr: q)
  int K;               // columns >= K are zero
  int vec;             // 1: coloff[4c .. 4c+3] are consecutive and 16-byte aligned (16-byte copies)
};

struct GParams {
  GOperand a, b;
  const float* ones;  // 16 bytes of 1.0f (the source of kOnesRow elements)
  int J, rtiles, nkb, nmma, tcols_half, stages;
  // TMEM accumulators in flight (2, 4 or 8; nacc * tcols_half <= 512 / CTAs per SM).  A tile's hand-offs
  // (commit -> epilogue wake-up -> tcgen05.ld -> stores -> arrive -> issuer wake-up) take a few thousand
  // cycles, and these short-K tiles spend less than that in their MMAs: with two accumulators the round trip,
  // not the work, set the time per tile
  int nacc;
  int nsub;  // 128B-swizzle k atoms (32 tf32 each) per pipeline stage: nkb stages cover nkb * nsub atoms
  // particle batching (gather kernels whose A operand is shared by every particle: the stage-0 forward
  // over the im2col of X and the stage-0 weight gradient over its transpose): a unit covers nb
  // consecutive particles, MMA N = nb * nmma_p, column n belongs to particle j0 + n / nmma_p.  The B rows
  // of consecutive particles are contiguous (b.ps = nmma_p rows), so the producers see one tall matrix.
  int nb, nmma_p;
  // direct convolution (DIRECT kernels, forward / delta with 32-channel blocks): each stage is one
  // TMA slab of bh + k - 1 input rows x win_w pixels x 32 channels plus the k*k weight atoms of
  // that channel block; the k*k shifted A operands are the same slab read through descriptors
  // offset by (ky * win_w + kx) rows -- every input pixel crosses L2 -> SM once per tile
  CUtensorMap mapA;  // 4-D {C, W, H, images}: the NHWC input (box {32, win_w, bh + k - 1, 1})
  CUtensorMap mapB;  // 3-D {Kp, nmma, J}: the weight copy (box {32, nmma, 1})
  int kk, cbn, flipB;        // kernel size, 32-channel blocks, weight atoms in flipped (ky, kx) order
  // kx fold (slab width divides 32, k * nmma <= 256): the k weight atoms of a kernel row are one B tile of
  // k * nmma rows, so a tile issues k instead of k * k MMA groups, D2[r][(kx, n)] = sum_(ky, c) slab[r + ky W][c]
  // B[(ky, kx)][n][c], and the epilogue forms out[r][n] = sum_kx D2[r + kx][(kx, n)] with warp shuffles (a
  // slab line never straddles a warp, and valid outputs have x + kx inside the line).  The MMAs at small N
  // are bound by their 128-row A reads, so this is k times fewer of them.
  int fold;
  int ksteps;  // MMA k-steps (8 channels each) per tap and channel block: < 4 when the block's upper channels are padding
  // resident weights (direct forward / delta): the k * k * cbn weight atoms of a particle stay in shared
  // memory while the CTA works through a contiguous range of that particle's tiles (they were re-loaded per
  // tile, most of the L2 -> SM bytes); the pipeline stages then hold input slabs only
  int persist;
  int win_w, bh, ybl;        // slab line pitch (pixels), output rows per tile, tiles per image
  // tma_w < win_w: the input is tma_w pixels wide and each slab line is loaded by its own TMA box into a
  // line pitch of win_w = 16 or 32 pixels (the pad pixels are never written and only feed dropped outputs).
  // A pitch that divides 32 makes the kx fold possible and keeps every A matrix start on an 8-row boundary:
  // at unaligned starts (row offset ky * W + kx) the same MMAs measured ~3x slower (C3 stage-1 forward,
  // N = 32: ~100 cycles per MMA against ~34 for the aligned N = 80 ones of the folded delta GEMM)
  int tma_w;
  int out_h, out_w, slab_rows, imgs_pp, mimg;
  // weight gradient from TMA (DIRECT + kEpiConvDw): K = (image, q) over flattened channel-major planes
  // of row stride win_p; A rows (ky, ci) are boxes of inT at q + ky * win_p (16-byte aligned: win_p is a
  // multiple of 4).  B rows (kx, co) are the unshifted delta at q - kx: a TMA box must start 16-byte
  // aligned, so one unswizzled staging tile [cout][halo + 32] starting at q - halo is loaded per k block
  // (TMA zero fill supplies the out-of-plane positions) and shifter warps copy its k shifted windows
  // into the swizzled B tile (shared memory to shared memory: no kx-shifted copies in HBM)
  int cin_rows, cout_rows, kpi, wpd, a_imgs_pp, halo, stg_bytes;
  int dbg;  // DASMC_CONV_DBG ablations (profiling only): 1 no operand copies, 2 no epilogue stores, 4 no MMAs
  // epilogue (forward / delta): out[j * out_ps + outoff[r] + n] for r < Rvalid, n < nvalid
  int Rvalid, nvalid;
  float* out;
  int64_t out_ps;
  const int* outoff;
  int out_ld;
  // second, channel-major copy of the output (the weight-gradient operands): value (r, n) also
  // goes to out2[j * out2_ps + out2off[r] + n * out2_cs + kx * (out2_ks + 1)] for kx < out2_k
  // (out2_k = 1: the next stage's input copy; k: the kx-shifted delta copies)
  float* out2;
  int64_t out2_ps, out2_cs, out2_ks;
  const int* out2off;
  int out2_k;
  const float* mask;  // delta: act'(mask[j * mask_ps + maskoff[r] + n]) (nullptr: identity)
  int64_t mask_ps;
  int mask_ld;
  const float* theta;  // forward: bias b[n] at theta[j * Dp + boff + n]
  int64_t Dp, boff;
  // weights: row i < nrows_w, column n is parameter woff + prow[i] + pcol[n]; the bias row
  // (prow[i] < 0) is boff + bcol[n] where bcol[n] >= 0 (other columns of that row are skipped)
  EpiParams e;
  int64_t woff;
  int nrows_w;
  const int* prow;
  const int* pcol;
  const int* bcol;
};

constexpr int kEpiConvFwd = 0, kEpiConvDx = 1, kEpiConvDw = 2;
#ifndef DASMC_CONV_BASEOFF
#define DASMC_CONV_BASEOFF 0  // 1: set the descriptor base-offset field for slab starts off the 1024-B atom
                              // (measured wrong on B200: the swizzle follows the absolute address)
#endif
// K-major SW128 descriptor of a matrix starting at any 128-B row of a swizzled slab
__device__ __forceinline__ uint64_t smem_desc_row(uint32_t addr) {
  const uint64_t a = (addr >> 4) & 0x3FFFULL;
  uint64_t d = a | (1ULL << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ULL << 46) | (2ULL << 61);
  if (DASMC_CONV_BASEOFF) d |= (uint64_t)((addr >> 7) & 7) << 49;
  return d;
}

// byte offset of element (row, k) of a 128B-swizzled K-major tile (8-row atoms of 1024 B)
__device__ __forceinline__ uint32_t swz(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ row) & 7) << 4) + ((k & 3) << 2));
}

// .ca: allocate in L1 -- an input pixel is re-read by up to k*k rows of the implicit im2col
// tile, which then hit L1 instead of crossing the L2 -> SM crossbar k*k times
__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ int row_off(const GOperand& o, int i) {
  if (i >= o.nrows) return kZeroRow;
  return o.rowoff ? o.rowoff[i] : i * o.ld;
}
__device__ __forceinline__ int col_off(const GOperand& o, int q) { return o.coloff ? o.coloff[q] : q; }

// Column (k) offsets of k-block kb that this lane's copies use: the vector path needs one
// (16-byte chunk lane % 8), the scalar path eight (element lane % 4 of chunks 0..7).
// kZeroRow marks columns past K.
template <bool VEC>
__device__ __forceinline__ void load_cols(const GOperand& o, int kb, int lane, int* co) {
  const int q0 = kb * kCBK;
  if (VEC) {
    const int q = q0 + 4 * (lane & 7);
    co[0] = q < o.K ? col_off(o, q) : kZeroRow;
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int q = q0 + 4 * c + (lane & 3);
      co[c] = q < o.K ? col_off(o, q) : kZeroRow;
    }
  }
}

// Row offsets of the tile rows this lane copies (pass p: vector rows (p*4 + warp)*4 + lane/8,
// scalar rows (p*4 + warp)*8 + lane/4); kZeroRow past the operand's rows or the tile.
template <int MAXP, int NPW = kProdWarps>
__device__ __forceinline__ void load_rows(const GOperand& o, int r0, int nrt, int pt, int lane, int* ro,
                                          int nlim = 0x7fffffff) {
#pragma unroll
  for (int p = 0; p < MAXP; ++p) {
    const int rl = o.vec ? (p * NPW + pt) * 4 + (lane >> 3) : (p * NPW + pt) * 8 + (lane >> 2);
    if (rl >= nlim) {  // rows of particles past the ensemble (a batched unit's tail): zeros
      ro[p] = kZeroRow;
      continue;
    }
    if (rl >= nrt) {  // past the tile: nothing to copy
      ro[p] = kZeroRow;
      continue;
    }
    ro[p] = row_off(o, r0 + rl);
  }
}

// One operand tile (k-block kb) into shared memory at `tile` from precomputed row / column
// offsets.  Vector path: lane -> (row lane / 8, 16-byte chunk lane % 8), a warp stores 4 full
// rows.  Scalar path: lane -> (row lane / 4, element lane % 4 of a chunk), 8 rows x 16 bytes
// per instruction; both are bank-conflict free under the 128B swizzle.
template <int MAXP, bool VEC, int NPW = kProdWarps>
__device__ __forceinline__ void gather_tile(const GOperand& o, const float* pbase, const float* ones, uint32_t tile,
                                            const int* roff, const int* coff, int nrt, int pt, int lane) {
  if (VEC) {
    const int c = lane & 7;
    const int co = coff[0];
#pragma unroll
    for (int p = 0; p < MAXP; ++p) {
      const int rl = (p * NPW + pt) * 4 + (lane >> 3);  // row within the tile
      if (rl >= nrt) break;
      const int ro = roff[p];
      const bool v = co != kZeroRow && ro != kZeroRow;
      const float* src = ro == kOnesRow ? ones : (v ? pbase + (int64_t)ro + co : pbase);
      cp_async16(tile + swz(rl, 4 * c), src, v);
    }
  } else {
    const int e = lane & 3;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int co = coff[VEC ? 0 : c];
#pragma unroll
      for (int p = 0; p < MAXP; ++p) {
        const int rl = (p * NPW + pt) * 8 + (lane >> 2);
        if (rl >= nrt) break;
        const int ro = roff[p];
        const bool v = co != kZeroRow && ro != kZeroRow;
        const float* src = ro == kOnesRow ? ones : (v ? pbase + (int64_t)ro + co : pbase);
        cp_async4(tile + swz(rl, 4 * c + e), src, v);
      }
    }
  }
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// mbarrier wait without a suspend-time hint: the convolution tiles are short (a few k-blocks),
// so the pipeline hand-offs are frequent and a parked warp's wake-up latency would dominate
// (DASMC_CONV_SPIN=0 restores the suspending wait for A/B)
#ifndef DASMC_CONV_SPIN
#define DASMC_CONV_SPIN 1
#endif
// epilogue warps back off between polls (8 spinning warps otherwise take issue slots from the lone
// MMA-issuing thread on their scheduler; DASMC_CONV_BACKOFF=0 for A/B)
#ifndef DASMC_CONV_BACKOFF
#define DASMC_CONV_BACKOFF 1
#endif
__device__ __forceinline__ void cwait_epi(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  for (uint32_t i = 0;; ++i) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.b32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
#if DASMC_CONV_BACKOFF
    __nanosleep(64);
#endif
    if ((i & 0xFFFFu) == 0xFFFFu && clock64() - t0 > 20000000000LL) __trap();  // watchdog (~10 s)
  }
}
__device__ __forceinline__ void cwait(uint64_t* bar, uint32_t parity) {
#if DASMC_CONV_SPIN
  uint32_t ok = 0;
  const long long t0 = clock64();
  for (uint32_t i = 0;; ++i) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.b32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((i & 0xFFFFu) == 0xFFFFu && clock64() - t0 > 20000000000LL) __trap();  // watchdog (~10 s)
  }
#else
  mbar_wait(bar, parity);
#endif
}

// EW8: the gather-mode forward with 4 producer + 8 epilogue warps (ConvWarps FWDG)
template <int EPI, int ACT, bool EW8, bool DIRECT>
__global__ void __launch_bounds__((ConvWarps<DIRECT, DIRECT && EPI == 2, EW8 && !DIRECT && EPI == 0>::T), DASMC_CONV_MINB)
    conv_tc_kernel(const __grid_constant__ GParams p) {
  using CW_ = ConvWarps<DIRECT, DIRECT && EPI == 2, EW8 && !DIRECT && EPI == 0>;
  constexpr int PW = CW_::P, EW = CW_::E;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_bytes = kCBM * 128, b_bytes = (uint32_t)p.nmma * 128;
  constexpr bool DWT = DIRECT && EPI == kEpiConvDw;  // weight gradient from TMA
  const uint32_t slab_bytes = DIRECT && !DWT ? (uint32_t)p.slab_rows * 128 : 0u;
  const uint32_t stage_bytes = DWT      ? a_bytes + b_bytes + (uint32_t)p.stg_bytes           // [A][B][staging]
                               : DIRECT ? slab_bytes + (p.persist ? 0u : (uint32_t)(p.kk * p.kk) * b_bytes)  // [slab][k*k B atoms]
                                        : (uint32_t)p.nsub * (a_bytes + b_bytes);             // [A atoms][B atoms]
  const bool PERS = DIRECT && !DWT && p.persist;
  uint8_t* wres = smem + (size_t)p.stages * stage_bytes;  // resident weight atoms [cb][ky * k + kx]
  const uint32_t wres_bytes = PERS ? (uint32_t)(p.cbn * p.kk * p.kk) * b_bytes : 0u;
  uint64_t* full = (uint64_t*)(wres + wres_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  constexpr int kMaxAcc = 8;
  uint64_t* tempty = tfull + kMaxAcc;
  uint64_t* sfull = tempty + kMaxAcc;  // DWT: the staging tile of a stage has landed
  uint32_t* tmem_holder = (uint32_t*)(sfull + p.stages);
  const int nb = DIRECT ? 1 : p.nb;  // particles per unit
  // resident weights: CTA b takes the contiguous tiles [u0, u1) (a particle's tiles are consecutive)
  const int pu = PERS ? p.J * p.mimg * p.ybl : 0;
  const int u0 = PERS ? (int)((int64_t)pu * blockIdx.x / gridDim.x) : 0;
  const int u1 = PERS ? (int)((int64_t)pu * (blockIdx.x + 1) / gridDim.x) : 0;
  const int units = DIRECT && !DWT ? p.J * p.mimg * p.ybl : p.rtiles * ((p.J + nb - 1) / nb);

  if (!DIRECT && p.rtiles == 1 && p.a.nrows < kCBM) {  // see the gather producers: A rows past the operand stay zero
    const uint32_t words = (uint32_t)p.stages * stage_bytes / 16;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      // TMA expect_tx (+ one arrival per shifter warp) / one cp.async arrival per producer thread
      mbar_init(&full[s], DWT ? 1 + kShiftWarps : DIRECT ? 1 : 32 * PW);
      mbar_init(&empty[s], 1);
      mbar_init(&sfull[s], 1);
    }
    for (int b = 0; b < kMaxAcc; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == PW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(p.nacc * p.tcols_half)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (DWT && warp < PW) {
    // ===================== TMA producer + shifter warps (weight gradient) =====================
    if (warp == 0) {
      if (lane == 0) {
        prefetch_map(&p.mapA);
        prefetch_map(&p.mapB);
        int s = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < units; t += gridDim.x) {
          const int rt = t % p.rtiles, j = t / p.rtiles;
          // this tile's ky blocks (cin_rows rows each); the ones row (bias) is stage memory, set below
          const int ky0 = rt * kCBM / p.cin_rows, ky1 = min(p.kk, (rt + 1) * kCBM / p.cin_rows);
          const uint32_t txa = (uint32_t)(ky1 - ky0) * p.cin_rows * 128;
          const uint32_t txs = (uint32_t)p.cout_rows * (uint32_t)(p.halo + kCBK) * 4;
          const int one_row = p.kk * p.cin_rows - rt * kCBM < kCBM ? p.kk * p.cin_rows - rt * kCBM : -1;
          for (int m = 0; m < p.mimg; ++m)
            for (int kb = 0; kb < p.kpi; ++kb) {
              cwait(&empty[s], ph ^ 1);
              uint8_t* st = smem + (size_t)s * stage_bytes;
              if (one_row >= 0 && !(p.dbg & 16)) {  // the bias row of ones (all 32 values equal: swizzle-invariant)
                float4* o = reinterpret_cast<float4*>(st + (one_row >> 3) * 1024 + (one_row & 7) * 128);
#pragma unroll
                for (int u = 0; u < 8; ++u) o[u] = make_float4(1.f, 1.f, 1.f, 1.f);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              }
              const int q0 = kb * kCBK;
              mbar_expect_tx(&sfull[s], txs);
              tma_3d(st + a_bytes + b_bytes, &p.mapB, &sfull[s], q0 - p.halo, 0, j * p.imgs_pp + m);
              mbar_expect_tx(&full[s], txa);
              for (int ky = ky0; ky < ky1; ++ky)
                tma_3d(st + (ky - ky0) * p.cin_rows * 128, &p.mapA, &full[s], q0 + ky * p.wpd, 0, j * p.a_imgs_pp + m);
              if (++s == p.stages) {
                s = 0;
                ph ^= 1;
              }
            }
        }
      }
    } else {
      // shifter warp: B tile row (kx, co) = staging row co shifted by kx; one row per instruction pair
      // (lane = k element: consecutive staging words, and a conflict-free swizzled row of the tile)
      // Warp sw takes rows co = sw, sw + 8, ... of every kx block (cout is a multiple of 8, so those
      // rows sit at the same position of consecutive 8-row swizzle atoms: 1024 bytes apart); four rows
      // are in flight per step
      const int sw = warp - 1;
      const int ldst = p.halo + kCBK, nco = p.cout_rows / kShiftWarps;
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < units; t += gridDim.x)
        for (int mk = 0; mk < p.mimg * p.kpi; ++mk) {
          cwait(&sfull[s], ph);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          const float* stg = reinterpret_cast<const float*>(st + a_bytes + b_bytes) + sw * ldst + p.halo + lane;
          const uint32_t tile = smem_u32(st + a_bytes);
          for (int kx = 0; kx < ((p.dbg & 8) ? 0 : p.kk); ++kx) {
            const int r0 = kx * p.cout_rows + sw;
            const uint32_t dst = tile + swz(r0, lane);
            const float* src = stg - kx;
            for (int u = 0; u < nco; u += 4) {
              float v[4];
#pragma unroll
              for (int w = 0; w < 4; ++w) v[w] = u + w < nco ? src[(u + w) * kShiftWarps * ldst] : 0.f;
#pragma unroll
              for (int w = 0; w < 4; ++w)
                if (u + w < nco)
                  asm volatile("st.shared.f32 [%0], %1;" ::"r"(dst + (uint32_t)(u + w) * 1024u), "f"(v[w]) : "memory");
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(smem_u32(&full[s]));
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
    }
  } else if (DIRECT && warp < PW) {
    // ===================== TMA producer (direct convolution) =====================
    if (warp == 0 && lane == 0) {
      prefetch_map(&p.mapA);
      prefetch_map(&p.mapB);
      const uint32_t txs = (uint32_t)(p.bh + p.kk - 1) * p.tma_w * 128;
      const uint32_t tx = txs + (PERS ? 0u : (uint32_t)(p.kk * p.kk) * b_bytes);
      int s = 0, jres = -1;
      uint32_t ph = 0;
      for (int t = PERS ? u0 : (int)blockIdx.x; t < (PERS ? u1 : units); t += PERS ? 1 : (int)gridDim.x) {
        const int yb = t % p.ybl, m = (t / p.ybl) % p.mimg, j = t / (p.ybl * p.mimg);
        if (PERS && j != jres) {
          // a new particle: every MMA issued so far has completed once each stage is free again; then its
          // weight atoms replace the previous particle's (sfull[0] completes when they have landed)
          if (jres >= 0) {
            int s2 = s;
            uint32_t ph2 = ph;
            for (int i = 0; i < p.stages; ++i) {
              cwait(&empty[s2], ph2 ^ 1);
              if (++s2 == p.stages) {
                s2 = 0;
                ph2 ^= 1;
              }
            }
          }
          jres = j;
          mbar_expect_tx(&sfull[0], wres_bytes);
          for (int cb = 0; cb < p.cbn; ++cb)
            for (int a = 0; a < p.kk * p.kk; ++a) {
              const int src = p.flipB ? p.kk * p.kk - 1 - a : a;
              tma_3d(wres + (size_t)(cb * p.kk * p.kk + a) * b_bytes, &p.mapB, &sfull[0], (src * p.cbn + cb) * kCBK, 0, j);
            }
        }
        for (int cb = 0; cb < p.cbn; ++cb) {
          cwait(&empty[s], ph ^ 1);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          mbar_expect_tx(&full[s], tx);
          if (p.tma_w == p.win_w) {
            tma_4d(st, &p.mapA, &full[s], cb * kCBK, 0, yb * p.bh, j * p.imgs_pp + m);
          } else {  // one box per slab line, into the padded line pitch
            for (int ln = 0; ln < p.bh + p.kk - 1; ++ln)
              tma_4d(st + (size_t)ln * p.win_w * 128, &p.mapA, &full[s], cb * kCBK, 0, yb * p.bh + ln, j * p.imgs_pp + m);
          }
          if (!PERS)
            for (int a = 0; a < p.kk * p.kk; ++a) {
              const int src = p.flipB ? p.kk * p.kk - 1 - a : a;  // delta: W'[ky'][kx'] = W[k-1-ky'][k-1-kx']
              tma_3d(st + slab_bytes + a * b_bytes, &p.mapB, &full[s], (src * p.cbn + cb) * kCBK, 0, j);
            }
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp < PW) {
    // ===================== gather producers =====================
    // Offsets are loaded one step ahead (next k-block's columns, next tile's rows) so the
    // table lookups overlap the copies instead of stalling every k-block on an L2 round trip;
    // the column tables are also L1-prefetched 8 k-blocks ahead.
    const uint32_t stages0 = smem_u32(smem);
    int s = 0;
    uint32_t ph = 0;
    int t = blockIdx.x;
    // a single row tile with few rows (the stage-0 weight gradient: 26-28 of 128): the rows past the operand
    // are zeroed once (below, before the first barrier) and never copied again
    const int a_rows = p.rtiles == 1 ? min(kCBM, (p.a.nrows + 7) & ~7) : kCBM;
    constexpr int MAXS = 4;  // atoms per stage
    int ra[8], rb[16], ran[8], rbn[16], ca[MAXS], cb[MAXS], can[MAXS], cbn[MAXS];
    // B rows a unit may read: its particles that exist (batched units; all rows otherwise)
    auto blim = [&](int tt) { return nb > 1 ? min(nb, p.J - (tt / p.rtiles) * nb) * p.nmma_p : 0x7fffffff; };
    if (t < units) {
      load_rows<8, PW>(p.a, (t % p.rtiles) * kCBM, kCBM, warp, lane, ra);
      load_rows<16, PW>(p.b, 0, p.nmma, warp, lane, rb, blim(t));
    }
#pragma unroll
    for (int u = 0; u < MAXS; ++u)
      if (u < p.nsub) {
        load_cols<true>(p.a, u, lane, ca + u);
        load_cols<true>(p.b, u, lane, cb + u);
      }
    while (t < units) {
      const int j = (t / p.rtiles) * nb;  // first particle of the unit
      const int tn = t + gridDim.x;
      if (tn < units) {
        load_rows<8, PW>(p.a, (tn % p.rtiles) * kCBM, kCBM, warp, lane, ran);
        load_rows<16, PW>(p.b, 0, p.nmma, warp, lane, rbn, blim(tn));
      }
      const float* abase = p.a.base + (int64_t)j * p.a.ps;
      const float* bbase = p.b.base + (int64_t)j * p.b.ps;
      for (int kb = 0; kb < p.nkb; ++kb) {
        const int kbn = kb + 1 < p.nkb ? kb + 1 : 0;  // the next tile starts again at stage 0
#pragma unroll
        for (int u = 0; u < MAXS; ++u)
          if (u < p.nsub) {
            load_cols<true>(p.a, kbn * p.nsub + u, lane, can + u);
            load_cols<true>(p.b, kbn * p.nsub + u, lane, cbn + u);
          }
        if (lane == 0 && kb + 4 < p.nkb) {
          if (p.a.coloff) prefetch_l1(p.a.coloff + (kb + 4) * p.nsub * kCBK);
          if (p.b.coloff) prefetch_l1(p.b.coloff + (kb + 4) * p.nsub * kCBK);
        }
        cwait(&empty[s], ph ^ 1);
        const uint32_t st = stages0 + (uint32_t)s * stage_bytes;
        if (!(p.dbg & 1)) {
#pragma unroll
          for (int u = 0; u < MAXS; ++u)
            if (u < p.nsub) {
              gather_tile<8, true, PW>(p.a, abase, p.ones, st + u * a_bytes, ra, ca + u, a_rows, warp, lane);
              gather_tile<16, true, PW>(p.b, bbase, p.ones, st + p.nsub * a_bytes + u * b_bytes, rb, cb + u, p.nmma, warp,
                                    lane);
            }
        }
        cp_async_arrive(&full[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
#pragma unroll
        for (int u = 0; u < MAXS; ++u) {
          ca[u] = can[u];
          cb[u] = cbn[u];
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) ra[q] = ran[q];
#pragma unroll
      for (int q = 0; q < 16; ++q) rb[q] = rbn[q];
      t = tn;
    }
    // drain: the CTA may not exit with copies in flight
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == PW) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(p.nmma, kCBM);
      int s = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      int jres = -1;
      uint32_t wph = 0;
      for (int t = PERS ? u0 : (int)blockIdx.x; t < (PERS ? u1 : units); t += PERS ? 1 : (int)gridDim.x) {
        cwait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * p.tcols_half);
        if (DIRECT && !DWT) {
          if (PERS) {
            const int j = t / (p.ybl * p.mimg);
            if (j != jres) {  // this particle's weight atoms have landed
              jres = j;
              cwait(&sfull[0], wph);
              wph ^= 1;
            }
          }
          for (int cb = 0; cb < p.cbn; ++cb) {
            cwait(&full[s], ph);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + (size_t)s * stage_bytes);
            // weight atoms of this channel block: resident, or behind the stage's slab
            const uint32_t wat = PERS ? smem_u32(wres) + (uint32_t)(cb * p.kk * p.kk) * b_bytes : st + slab_bytes;
            // The issuing thread's instruction count bounds these short-K tiles (25 taps x 4 MMAs per 128
            // pixels at C3), so the per-tap descriptors advance by precomputed increments (descriptor
            // address fields count 16-byte units; no divisions, no per-MMA predicates past the first)
            if (!(p.dbg & 4)) {
              uint64_t ad = smem_desc_row(st), bd = smem_desc_row(wat);
              const uint32_t idf = p.fold ? idesc_tf32(p.kk * p.nmma, kCBM) : idesc;
              const uint64_t bstep = (uint64_t)(b_bytes >> 4) * (p.fold ? (uint32_t)p.kk : 1u);
              const uint64_t ax = p.fold ? (uint64_t)p.win_w * 8 : 8, ay = (uint64_t)(p.win_w - p.kk + 1) * 8;
              auto group = [&](bool acc0) {
                tc_mma<0>(d, ad, bd, idf, acc0);
                if (p.ksteps == 4) {
                  tc_mma<0>(d, ad + 2, bd + 2, idf, 1);
                  tc_mma<0>(d, ad + 4, bd + 4, idf, 1);
                  tc_mma<0>(d, ad + 6, bd + 6, idf, 1);
                } else {
                  for (int k = 1; k < p.ksteps; ++k) tc_mma<0>(d, ad + 2 * k, bd + 2 * k, idf, 1);
                }
                bd += bstep;
              };
              if (p.fold) {
                for (int ky = 0; ky < p.kk; ++ky) {
                  group((cb | ky) != 0);
                  ad += ax;
                }
              } else {
                for (int ky = 0; ky < p.kk; ++ky) {
                  for (int kx = 0; kx < p.kk; ++kx) {
                    group((cb | ky | kx) != 0);
                    ad += ax;
                  }
                  ad += ay - ax;
                }
              }
            }
            tc_commit(&empty[s]);
            if (++s == p.stages) {
              s = 0;
              ph ^= 1;
            }
          }
          tc_commit(&tfull[acc]);
          if (++acc == p.nacc) {
            acc = 0;
            aph ^= 1;
          }
          continue;
        }
        for (int kb = 0; kb < p.nkb; ++kb) {
          cwait(&full[s], ph);
          // the stage was written through the generic proxy (cp.async); order it before the
          // tensor core's async-proxy reads
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_fence_after();
          uint8_t* st = smem + (size_t)s * stage_bytes;
          if (!(p.dbg & 4))
            for (int u = 0; u < p.nsub; ++u) {
              const uint64_t ad = smem_desc(st + u * a_bytes), bd = smem_desc(st + p.nsub * a_bytes + u * b_bytes);
#pragma unroll
              for (int k = 0; k < 4; ++k) tc_mma<0>(d, ad + 2 * k, bd + 2 * k, idesc, (kb | u | k) != 0);
            }
          tc_commit(&empty[s]);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == p.nacc) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue (4 warps, one TMEM lane group each) =====================
    const int lg = warp & 3;
    const int part = (warp - PW - 1) >> 2;  // column half (direct mode: two warps per lane group)
    const int nch = p.nmma / 16;
    const int ch_lo = EW == 8 ? (part * nch) / 2 : 0, ch_hi = EW == 8 ? ((part + 1) * nch) / 2 : nch;
    const int row_in_tile = lg * 32 + lane;
    int acc = 0;
    uint32_t aph = 0;
    for (int t = PERS ? u0 : (int)blockIdx.x; t < (PERS ? u1 : units); t += PERS ? 1 : (int)gridDim.x) {
      int j, r;
      bool rv = true;  // the row is an output of this tile
      if (DIRECT && !DWT) {  // slab row -> output pixel (y, x) of image m; wide rows (x >= out_w) are dropped
        const int yb = t % p.ybl, m = (t / p.ybl) % p.mimg;
        j = t / (p.ybl * p.mimg);
        const int yl = row_in_tile / p.win_w, x = row_in_tile - yl * p.win_w, y = yb * p.bh + yl;
        rv = yl < p.bh && y < p.out_h && x < p.out_w;
        r = (m * p.out_h + y) * p.out_w + x;
      } else {
        const int rt = t % p.rtiles;
        j = (t / p.rtiles) * nb;  // first particle of the unit
        r = rt * kCBM + row_in_tile;
      }
      const int j_unit = j;
      // Row offsets (table lookups) and the first chunk's act' mask are loaded BEFORE the accumulator wait:
      // their global-memory latency then overlaps the tile's MMAs instead of sitting between the TMEM load
      // and the stores (the delta epilogue was the longer half of its kernel, ncu / DASMC_CONV_DBG=2)
      int64_t off1 = 0;
      int off2 = 0;
      float4 mk[4];
      bool mk_ok = false;
      if ((EPI == kEpiConvFwd || EPI == kEpiConvDx) && rv && r < p.Rvalid) {
        off1 = p.outoff ? (int64_t)p.outoff[r] : (int64_t)r * p.out_ld;
        if (p.out2) off2 = p.out2off[r];
        if (EPI == kEpiConvDx && p.mask && ch_lo < ch_hi && (p.mask_ld & 3) == 0 && p.nvalid - ch_lo * 16 >= 16) {
          const float4* m4 =
              reinterpret_cast<const float4*>(p.mask + (int64_t)j * p.mask_ps + (int64_t)r * p.mask_ld + ch_lo * 16);
          if ((reinterpret_cast<uintptr_t>(m4) & 15) == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u) mk[u] = __ldg(m4 + u);
            mk_ok = true;
          }
        }
      }
      cwait_epi(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t)(acc * p.tcols_half) + ((uint32_t)(lg * 32) << 16);
      for (int ch = ch_lo; ch < ch_hi; ++ch) {
        float v[16];
        tmem_ld16(taddr + ch * 16, v);
        if (DIRECT && !DWT && p.fold) {  // out[r] = sum_kx D2[r + kx][(kx, .)]: every lane takes part in the shuffles
          for (int kx = 1; kx < p.kk; ++kx) {
            float u[16];
            tmem_ld16(taddr + (kx * nch + ch) * 16, u);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += __shfl_down_sync(0xffffffffu, u[q], kx);
          }
        }
        int n0 = ch * 16;
        if (!DIRECT && nb > 1) {  // batched unit: this chunk's particle and its column within the particle
          const int jb = n0 / p.nmma_p;
          j = j_unit + jb;
          n0 -= jb * p.nmma_p;
          if (j >= p.J) continue;
        }
        const int nq = min(16, p.nvalid - n0);  // warp-uniform
        if (nq <= 0) continue;
        if (p.dbg & 2) continue;
        if (EPI == kEpiConvFwd || EPI == kEpiConvDx) {
          if (!rv || r >= p.Rvalid) continue;
          float* dst = p.out + (int64_t)j * p.out_ps + off1 + n0;
          if (EPI == kEpiConvFwd) {
            const float* b = p.theta + (int64_t)j * p.Dp + p.boff + n0;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q < nq) {
                const float z = v[q] + b[q];
                v[q] = tf32_hi(ACT == DASMC_RELU ? fmaxf(z, 0.f) : tanhf(z));
              }
          } else {
            if (p.mask && mk_ok && ch == ch_lo) {
              const float* a16 = reinterpret_cast<const float*>(mk);
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                const float a = a16[q];
                v[q] *= ACT == DASMC_RELU ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a;
              }
            } else if (p.mask) {
              const float* m = p.mask + (int64_t)j * p.mask_ps + (int64_t)r * p.mask_ld + n0;
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (q < nq) {
                  const float a = m[q];
                  v[q] *= ACT == DASMC_RELU ? (a > 0.f ? 1.f : 0.f) : 1.f - a * a;
                }
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = tf32_hi(v[q]);
          }
          if (!p.out) {  // delta into stage 0: only the channel-major copy below is read
          } else if (nq == 16 && (((uintptr_t)dst) & 15) == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              reinterpret_cast<float4*>(dst)[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q < nq) dst[q] = v[q];
          }
          if (p.out2) {  // lanes are consecutive pixels: each (channel, kx) store is coalesced
            float* d2 = p.out2 + (int64_t)j * p.out2_ps + off2 + (int64_t)n0 * p.out2_cs;
            for (int kx = 0; kx < p.out2_k; ++kx) {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (q < nq) d2[(int64_t)q * p.out2_cs] = v[q];
              d2 += p.out2_ks + 1;
            }
          }
        } else {
          if (r >= p.nrows_w) continue;
          const int pr = p.prow[r];
          const int64_t base = (int64_t)j * p.Dp;
          if (pr >= 0) {
            int64_t idx[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) idx[q] = base + p.woff + pr + (q < nq ? p.pcol[n0 + q] : 0);
            leapfrog_update_n<16>(p.e, j, idx, v, nq);
          } else {  // the bias row: one column per output channel
            for (int q = 0; q < nq; ++q) {
              const int b = p.bcol[n0 + q];
              if (b >= 0) leapfrog_update(p.e, j, base + p.boff + b, v[q]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[acc]));
      if (++acc == p.nacc) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == PW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.nacc * p.tcols_half)
                 : "memory");
  }
}

// ---- stage helpers -------------------------------------------------------------------------
// W copies for the forward (Wf[j][n][kk], kk in the stage's k-order) and delta (Wd[j][ci][kk],
// kk = (ky, kx, co)) GEMMs, tf32-rounded, zero padded to [nrows][Kp].
__global__ void conv_wcopy_kernel(const float* __restrict__ theta, int64_t Dp, int64_t woff, int cin, int k, int cout,
                                  int mode, int korder, int nrows, int Kp, int64_t J, float* __restrict__ out,
                                  int cin_p) {
  const int kk2 = k * k;
  const int64_t per = (int64_t)nrows * Kp, total = J * per;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / per;
    const int rem = (int)(g - j * per), n = rem / Kp, q = rem - n * Kp;
    float v = 0.f;
    if (mode == 0) {  // forward: row co, column q over (ky, kx, ci) [korder 0] or (ci, ky, kx) [korder 1]
      // korder 0: q = (ky, kx, ci) with ci < cin_p (the input's channel pitch; zero columns past cin)
      const int ci = korder == 0 ? q % cin_p : 0, tap = korder == 0 ? q / cin_p : 0;
      if (n < cout && (korder == 0 ? (tap < kk2 && ci < cin) : q < cin * kk2)) {
        const int src = korder == 0 ? ci * kk2 + tap : q;
        v = theta[j * Dp + woff + (int64_t)n * cin * kk2 + src];
      }
    } else {  // delta: row ci, column q over (ky, kx, co)
      if (n < cin && q < cout * kk2) {
        const int kyx = q / cout, co = q - kyx * cout;
        v = theta[j * Dp + woff + ((int64_t)co * cin + n) * kk2 + kyx];
      }
    }
    out[g] = tf32_hi(v);
  }
}

// 2x2/2 max-pool forward of an NHWC stage output; flat != 0 writes the flatten order (c, y, x)
// of the head input instead of NHWC.
// code[j][m][py][px][c] (one byte per pooled element) = position 0..3 of the window's first maximum in
// (dy, dx) order, bit 2 = max > 0: the max-pool backward routes through it and (ReLU) never re-reads
// the pre-pool plane.
template <bool P2>
__global__ void __launch_bounds__(256) pool_fwd_nhwc_kernel(ConvDev d, const float* __restrict__ A, int64_t a_ps,
                                                            float* __restrict__ P, int64_t p_ps, int M, int flat,
                                                            float* __restrict__ T, int64_t t_ps, int t_wp,
                                                            uint8_t* __restrict__ code, int logC, int cp) {
  // cp: channel pitch of the pooled NHWC plane (>= C; padding channels are never written and stay zero)
  const int C = d.cout, per = d.sh * d.sw * C, shsw = d.sh * d.sw;
  const int m = (int)(blockIdx.x % (unsigned)M);  // one image of one particle per block: 32-bit index math inside
  const int64_t j = blockIdx.x / (unsigned)M;
  const float* aimg = A + j * a_ps + (int64_t)m * d.ho * d.wo * C;
  float* pimg = P + j * p_ps + (int64_t)m * (flat ? per : shsw * cp);
  uint8_t* cimg = code ? code + (j * M + m) * per : nullptr;
  float* timg = T ? T + j * t_ps + (int64_t)m * C * d.sh * t_wp : nullptr;
  const int rowC = d.wo * C;
  for (int py = 0; py < d.sh; ++py) {
    const float* arow = aimg + 2 * py * rowC;
    for (int i = threadIdx.x; i < d.sw * C; i += 256) {  // (px, c), c fastest
      const int px = P2 ? i >> logC : i / C, c = P2 ? i & (C - 1) : i - px * C;
      const float* a = arow + 2 * px * C + c;
      const float a0 = a[0], a1 = a[C], a2 = a[rowC], a3 = a[rowC + C];
      int best = 0;
      float v = a0;
      if (a1 > v) { v = a1; best = 1; }
      if (a2 > v) { v = a2; best = 2; }
      if (a3 > v) { v = a3; best = 3; }
      const int o = py * d.sw * C + i;
      pimg[flat ? c * shsw + py * d.sw + px : (py * d.sw + px) * cp + c] = v;
      if (cimg) cimg[o] = (uint8_t)(best | (v > 0.f ? 4 : 0));  // bit 2: relu'(max)
      // the next stage's channel-major, width-padded input copy (its weight-gradient operand)
      if (timg) timg[(c * d.sh + py) * t_wp + px] = v;
    }
  }
}

void launch_pool_fwd(Ctx& c, const ConvDev& d, const float* A, int64_t a_ps, float* P, int64_t p_ps, int64_t M,
                     int64_t J, int flat, float* T, int64_t t_ps, int t_wp, uint8_t* code, int cp) {
  const bool p2 = (d.cout & (d.cout - 1)) == 0;
  int logC = 0;
  while ((1 << logC) < d.cout) ++logC;
  if (p2)
    pool_fwd_nhwc_kernel<true><<<(unsigned)(J * M), 256, 0, c.stream>>>(d, A, a_ps, P, p_ps, (int)M, flat, T, t_ps, t_wp,
                                                                        code, logC, cp);
  else
    pool_fwd_nhwc_kernel<false><<<(unsigned)(J * M), 256, 0, c.stream>>>(d, A, a_ps, P, p_ps, (int)M, flat, T, t_ps,
                                                                         t_wp, code, logC, cp);
  LAUNCHED();
}

// Max-pool backward into the stage's zero-bordered delta buffer: the pooled delta (NHWC, or the
// head's flatten order) times act'(max) goes to the first maximum of the window in (dy, dx)
// order, zeros to the other three positions (network activation derivative from the
// post-activation value, network.hpp:211-214).  Pad = k - 1 on every side.  One block per
// (particle, image, pooled row): the two pre-pool rows are staged in shared memory, so both
// outputs -- the NHWC zero-bordered delta (the delta GEMM's operand) and the k kx-shifted
// channel-major copies (the weight-gradient operand) -- are written with coalesced rows.
// Rows / columns no window covers (odd sizes, floor pooling) are never written (zero from
// allocation).
// Layout of a stage's weight-gradient delta copies (ConvTcState::DzLayout): value (m, c, y, x)
// goes to S[kx * s_kx + c * s_c + m * s_m + y * s_y + x + kx] for kx < kc.
struct DzL {
  int kc, s_y;
  int64_t s_kx, s_m, s_c;
};

// code = pool_fwd_nhwc_kernel's argmax codes (ReLU: act' from the code; tanh: the maximum is read back from
// the pre-pool plane A at the coded position); dZ == nullptr (stage 0: no delta GEMM reads it) skips the
// NHWC output.
// The index arithmetic is shifts and masks when C is a power of two (P2; logC = log2 C): the kernel is
// issue-bound, and per-element integer divisions were most of its instructions.
template <bool P2>
__global__ void __launch_bounds__(256) pool_bwd_rows_kernel(ConvDev d, int act, const float* __restrict__ A,
                                                            int64_t a_ps, const uint8_t* __restrict__ code,
                                                            const float* __restrict__ dP, int64_t dp_ps,
                                                            int flat, float* __restrict__ dZ, int64_t dz_ps, int M,
                                                            float* __restrict__ S, int64_t s_ps, DzL L, int logC,
                                                            int PR) {
  extern __shared__ float pz[];  // [2 PR][wo][C + 1]: the window deltas of PR pooled rows (2 PR pre-pool rows)
  const int C = d.cout, pad = d.k - 1, W2 = d.wo + 2 * pad, H2 = d.ho + 2 * pad, CP = C + 1;
  const int m = (int)(blockIdx.x % (unsigned)M);  // (j, m): one image of one particle per block
  const int64_t j = blockIdx.x / (unsigned)M;
  const int wo2 = 2 * d.sw;  // pre-pool columns covered by windows
  const int per = d.sh * d.sw * C, shsw = d.sh * d.sw;
  const uint8_t* cimg = code + (j * M + m) * per;
  const float* dpimg = dP + j * dp_ps + (int64_t)m * per;
  const float* aimg = A + j * a_ps + (int64_t)m * d.ho * d.wo * C;
  float* z = dZ ? dZ + j * dz_ps + (int64_t)m * H2 * W2 * C : nullptr;
  float* sb = S + j * s_ps + m * L.s_m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int py0 = 0; py0 < d.sh; py0 += PR) {
    const int npr = min(PR, d.sh - py0);  // pooled rows of this pass
    __syncthreads();  // the previous pass's reads of pz are done
    for (int pyl = 0; pyl < npr; ++pyl) {
      const int py = py0 + pyl;
      float* prow = pz + 2 * pyl * d.wo * CP;
      for (int i = threadIdx.x; i < d.sw * C; i += 256) {  // (px, c), c fastest: coalesced NHWC reads
        const int px = P2 ? i >> logC : i / C, c = P2 ? i & (C - 1) : i - px * C;
        const int o = py * d.sw * C + i;
        const int po = flat ? c * shsw + py * d.sw + px : o;  // pooled-output layout
        const int cd = cimg[o], best = cd & 3;
        const float gp = dpimg[po];
        float dact;
        if (act == DASMC_RELU) {
          dact = (cd & 4) ? 1.f : 0.f;
        } else {
          const float mx = aimg[((2 * py + (best >> 1)) * d.wo + 2 * px + (best & 1)) * C + c];
          dact = 1.f - mx * mx;
        }
        const float v = tf32_hi(gp * dact);
        // all four window positions (the three non-maxima get 0): no separate zeroing pass
        float* w = prow + (2 * px) * CP + c;
        w[0] = best == 0 ? v : 0.f;
        w[CP] = best == 1 ? v : 0.f;
        w[d.wo * CP] = best == 2 ? v : 0.f;
        w[(d.wo + 1) * CP] = best == 3 ? v : 0.f;
      }
    }
    __syncthreads();
    // NHWC zero-bordered rows: (x, c) contiguous per row
    if (z)
      for (int yl = 0; yl < 2 * npr; ++yl) {
        float* zr = z + ((int64_t)(2 * py0 + yl + pad) * W2 + pad) * C;
        const float* src = pz + yl * d.wo * CP;
        for (int i = threadIdx.x; i < wo2 * C; i += 256) {
          const int x = P2 ? i >> logC : i / C, c = P2 ? i & (C - 1) : i - x * C;
          zr[i] = src[x * CP + c];
        }
      }
    // channel-major (kx-shifted) copies: one warp per (kx, c) pair, a run over x per pre-pool row
    for (int kcc = warp; kcc < L.kc * C; kcc += 8) {
      const int kx = P2 ? kcc >> logC : kcc / C, c = P2 ? kcc & (C - 1) : kcc - kx * C;
      float* dst = sb + kx * L.s_kx + c * L.s_c + (int64_t)(2 * py0) * L.s_y + kx;
      const float* src = pz + c;
      for (int yl = 0; yl < 2 * npr; ++yl, dst += L.s_y, src += d.wo * CP)
        for (int x = lane; x < wo2; x += 32) dst[x] = src[x * CP];
    }
  }
}

// Max-pool backward with one channel-major delta copy S (the TMA weight-gradient form / stage 0) and, for
// stages >= 1, the zero-bordered NHWC delta: two passes over the pooled elements instead of a transposition
// through shared memory.  One block per (particle, image).  NHWC pass: channel fastest.  Channel-major pass:
// thread -> (channel c, pooled column px) with px fastest, so a warp's stores per pooled row are contiguous runs
// of one channel-major row, and the strided code / delta reads of neighbouring channels share cache lines
// within the block.  ~4x fewer instructions than the staged kernel, which was issue-bound (ncu: 89-92 %).
__global__ void __launch_bounds__(256) pool_bwd_cm_kernel(ConvDev d, int act, const float* __restrict__ A, int64_t a_ps,
                                                          const uint8_t* __restrict__ code,
                                                          const float* __restrict__ dP, int64_t dp_ps, int flat, int M,
                                                          float* __restrict__ dZ, int64_t dz_ps,
                                                          float* __restrict__ S, int64_t s_ps, DzL L) {
  const int C = d.cout, per = d.sh * d.sw * C, shsw = d.sh * d.sw;
  const int m = (int)(blockIdx.x % (unsigned)M);
  const int64_t j = blockIdx.x / (unsigned)M;
  const uint8_t* cimg = code + (j * M + m) * per;
  const float* dpimg = dP + j * dp_ps + (int64_t)m * per;
  const float* aimg = A + j * a_ps + (int64_t)m * d.ho * d.wo * C;
  float* sb = S + j * s_ps + m * L.s_m;
  if (dZ) {
    // the zero-bordered NHWC delta (stages >= 1), channel fastest: every store of a warp is one run of
    // channels of a pixel row.  The codes and pooled deltas are read again below (cache hits).
    const int pad = d.k - 1, W2 = d.wo + 2 * pad, H2 = d.ho + 2 * pad;
    float* z = dZ + j * dz_ps + (int64_t)m * H2 * W2 * C;
    for (int o = threadIdx.x; o < per; o += 256) {
      const int pp = o / C, c = o - pp * C, py = pp / d.sw, px = pp - py * d.sw;
      const int po = flat ? c * shsw + pp : o;
      const int cd = cimg[o], best = cd & 3;
      const float gp = dpimg[po];
      float dact;
      if (act == DASMC_RELU) {
        dact = (cd & 4) ? 1.f : 0.f;
      } else {
        const float mx = aimg[((2 * py + (best >> 1)) * d.wo + 2 * px + (best & 1)) * C + c];
        dact = 1.f - mx * mx;
      }
      const float v = tf32_hi(gp * dact);
      float* z0 = z + ((int64_t)(2 * py + pad) * W2 + 2 * px + pad) * C + c;
      z0[0] = best == 0 ? v : 0.f;
      z0[C] = best == 1 ? v : 0.f;
      z0[(int64_t)W2 * C] = best == 2 ? v : 0.f;
      z0[(int64_t)W2 * C + C] = best == 3 ? v : 0.f;
    }
  }
  for (int i = threadIdx.x; i < C * d.sw; i += 256) {
    const int c = i / d.sw, px = i - c * d.sw;
    float* srow = sb + c * L.s_c + 2 * px;
    for (int py = 0; py < d.sh; ++py) {
      const int o = (py * d.sw + px) * C + c;
      const int po = flat ? c * shsw + py * d.sw + px : o;
      const int cd = cimg[o], best = cd & 3;
      const float gp = dpimg[po];
      float dact;
      if (act == DASMC_RELU) {
        dact = (cd & 4) ? 1.f : 0.f;
      } else {
        const float mx = aimg[((2 * py + (best >> 1)) * d.wo + 2 * px + (best & 1)) * C + c];
        dact = 1.f - mx * mx;
      }
      const float v = tf32_hi(gp * dact);
      float* r0 = srow + (int64_t)(2 * py) * L.s_y;
      float* r1 = r0 + L.s_y;
      r0[0] = best == 0 ? v : 0.f;
      r0[1] = best == 1 ? v : 0.f;
      r1[0] = best == 2 ? v : 0.f;
      r1[1] = best == 3 ? v : 0.f;
    }
  }
}

void launch_pool_bwd(Ctx& c, const ConvDev& d, int act, const float* A, int64_t a_ps, const uint8_t* code,
                     const float* dP, int64_t dp_ps, int flat, float* dZ, int64_t dz_ps, int64_t M, int64_t J, float* S,
                     int64_t s_ps, const DzL& L) {
  if (L.kc == 1) {  // one channel-major copy (+ the NHWC delta): no staging through shared memory needed
    pool_bwd_cm_kernel<<<(unsigned)(J * M), 256, 0, c.stream>>>(d, act, A, a_ps, code, dP, dp_ps, flat, (int)M, dZ, dz_ps, S,
                                                                s_ps, L);
    LAUNCHED();
    return;
  }
  // pooled rows per pass (fewer block-wide barriers per image): what ~kb KB of shared memory hold
  const size_t row_bytes = sizeof(float) * 2 * (size_t)d.wo * (d.cout + 1);
  static const int kb = [] {
    const char* e = std::getenv("DASMC_POOL_KB");
    return e ? std::atoi(e) : 24;
  }();
  const int PR = (int)std::max<size_t>(1, std::min<size_t>((size_t)d.sh, (size_t)kb * 1024 / row_bytes));
  const size_t sm = row_bytes * PR;
  const bool p2 = (d.cout & (d.cout - 1)) == 0;
  int logC = 0;
  while ((1 << logC) < d.cout) ++logC;
  auto go = [&](auto kern) {
    if (sm > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    kern<<<(unsigned)(J * M), 256, sm, c.stream>>>(d, act, A, a_ps, code, dP, dp_ps, flat, dZ, dz_ps, (int)M, S, s_ps, L,
                                                   logC, PR);
  };
  if (p2)
    go(pool_bwd_rows_kernel<true>);
  else
    go(pool_bwd_rows_kernel<false>);
  LAUNCHED();
}

// Last stage without a pool: NHWC output <-> the head's flatten order (c, y, x).
__global__ void nhwc_to_flat_kernel(ConvDev d, const float* __restrict__ A, int64_t a_ps, float* __restrict__ F,
                                    int64_t f_ps, int64_t M, int64_t J) {
  const int C = d.cout;
  const int64_t per = (int64_t)d.ho * d.wo * C, total = J * M * per;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / (M * per), rem = g - j * M * per, m = rem / per;
    const int o = (int)(rem - m * per), c = o % C, yx = o / C;
    F[j * f_ps + m * per + (int64_t)c * d.ho * d.wo + yx] = A[j * a_ps + m * per + o];
  }
}
__global__ void flat_to_dzpad_kernel(ConvDev d, const float* __restrict__ F, int64_t f_ps, float* __restrict__ dZ,
                                     int64_t dz_ps, int64_t M, int64_t J, float* __restrict__ S, int64_t s_ps, DzL L) {
  const int C = d.cout, pad = d.k - 1, W2 = d.wo + 2 * pad, H2 = d.ho + 2 * pad;
  const int64_t per = (int64_t)d.ho * d.wo * C, total = J * M * per;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / (M * per), rem = g - j * M * per, m = rem / per;
    const int o = (int)(rem - m * per), c = o % C, yx = o / C, y = yx / d.wo, x = yx - y * d.wo;
    const float v = tf32_hi(F[j * f_ps + m * per + (int64_t)c * d.ho * d.wo + yx]);
    if (dZ) dZ[j * dz_ps + m * (int64_t)H2 * W2 * C + ((int64_t)(y + pad) * W2 + x + pad) * C + c] = v;
    float* s0 = S + j * s_ps + m * L.s_m + c * L.s_c + (int64_t)y * L.s_y + x;
    for (int kx = 0; kx < L.kc; ++kx, s0 += L.s_kx + 1) *s0 = v;
  }
}

__global__ void im2col_x_kernel(ConvDev d, const float* __restrict__ X, int64_t rows, int Kp, float* __restrict__ out) {
  const int K = d.cin * d.k * d.k, npix = d.ho * d.wo;
  const int64_t total = rows * npix * Kp;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rp = g / Kp;
    const int q = (int)(g - rp * Kp);
    const int64_t m = rp / npix;
    const int p = (int)(rp - m * npix), y = p / d.wo, x = p - y * d.wo;
    float v = 0.f;
    if (q < K) {
      const int ci = q / (d.k * d.k), r = q - ci * d.k * d.k, ky = r / d.k, kx = r - ky * d.k;
      v = X[((m * d.cin + ci) * d.hin + y + ky) * d.win + x + kx];
    }
    out[g] = v;
  }
}

// XcolT[q][r] = Xcol[r][q] (q < K) and XcolT[K][r] = 1 (the bias row): the stage-0
// weight-gradient A operand, pixel-contiguous rows
__global__ void xcolT_kernel(const float* __restrict__ Xcol, int64_t R, int Kp, int K, int64_t ld,
                             float* __restrict__ XcolT) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R * (K + 1);
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = g / R, r = g - q * R;
    XcolT[q * ld + r] = q < K ? Xcol[r * Kp + q] : 1.f;
  }
}

__global__ void round_tf32_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = tf32_hi(src[i]);
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

int64_t pad_plane(const ConvDev& d) { return (int64_t)(d.ho + 2 * d.k - 2) * (d.wo + 2 * d.k - 2) * d.cout; }
int64_t act_plane(const ConvDev& d) { return (int64_t)d.ho * d.wo * d.cout; }
int64_t pool_plane(const ConvDev& d) { return (int64_t)d.sh * d.sw * d.cout; }
int round_up(int v, int a) { return (v + a - 1) / a * a; }

}  // namespace

// ---- per-context state ------------------------------------------------------------------------
// Weight-gradient layout (the "shifted rows" form): with K = (image, y, x') over the input
// width x' in [0, win_p) (win_p = win rounded up to 4),
//   dW[co, ci, ky, kx] = sum_K In[ci][y + ky][x'] * dZ[co][y][x' - kx],
// A rows (ky, ci) read the stage input in a channel-major, width-padded copy (inT: x'
// contiguous) and B rows (kx, co) read k copies of dZ shifted by kx (dZs), so both operands are
// 16-byte chunks of 4 consecutive x' -- no scalar im2col gathers -- and N = k * cout.
struct ConvTcState {
  float* Xr = nullptr;  // tf32-rounded copy of the active X rows (stage-0 operand)
  int64_t Xr_rows = 0;
  float* Xcol = nullptr;  // stage-0 im2col of Xr, [rows * ho * wo][KpF[0]], k = (ci, ky, kx): shared by
  int64_t Xcol_rows = 0;  // every particle, built once per data set (16-byte gathers for the stage-0 GEMM)
  float* ones = nullptr;
  int64_t mcap = 0;  // images per chunk the buffers hold
  int korder[kMaxConv] = {};   // forward k order: 0 = (ky, kx, ci) over NHWC input; 1 = (ci, ky, kx) over X
  int nmmaF[kMaxConv] = {}, KpF[kMaxConv] = {}, nmmaD[kMaxConv] = {}, KpD[kMaxConv] = {}, nmmaW[kMaxConv] = {};
  int winp[kMaxConv] = {};     // stage input width padded to a multiple of 4
  float* Wf[kMaxConv] = {};
  float* Wd[kMaxConv] = {};
  float* dP[kMaxConv] = {};    // delta of a pooled (non-last) stage output, NHWC
  uint8_t* pcode[kMaxConv] = {};  // pooled stages: argmax code of every window, [Jmax][mcap][sh][sw][cout]
  // weight-gradient operands, written by the producers of the stage input / delta (epilogue
  // second outputs, pool kernels): zero-initialised, so padding columns stay zero
  float* inT[kMaxConv] = {};   // stage input [mcap][cin][hin][win_p] per particle (stage 0: shared X copy)
  float* dZs[kMaxConv] = {};   // [k][mcap][cout][ho][win_p] per particle: dZ shifted right by kx
  DzL dzl[kMaxConv] = {};      // layout of dZs[i] (set with the chunk capacity)
  // stage 0 with pixels-per-image % 4 == 0: its weight gradient contracts the shared im2col of X
  // (transposed, XcolT[q][image * npix + p]) with the unshifted channel-major delta, instead of
  // k kx-shifted delta copies of the (largest) stage-0 plane
  bool xcol0 = false;
  float* XcolT = nullptr;
  int64_t XcolT_rows = 0;
  bool direct_ok = true;       // DASMC_CONV_DIRECT=0 forces the gather path (A/B, tests)
  bool batch0 = true;          // DASMC_CONV_BATCH0=0: one particle per unit in the stage-0 GEMMs (A/B)
  // channel pitch of stage i's pooled NHWC output: cout, or 32 when the next stage then qualifies for the
  // direct convolution (its input needs 32-channel blocks; the padding channels stay zero and the next
  // stage's weight copy has zero columns for them).  C3: the 16-channel 12x12 input of stage 1 -- gathered
  // as an implicit im2col, that forward was bound by the L1 gather rate (7.3 ms per launch)
  int cpd[kMaxConv] = {};
  bool dwt[kMaxConv] = {};     // weight gradient from TMA (flattened, unshifted delta copy: DzL kc = 1)
  int* c2o[kMaxConv] = {};     // input pixel of stage i -> its inT[i] offset (channel 0)
  int* dzo[kMaxConv] = {};     // output pixel of stage i -> its dZs[i] offset (channel 0, kx 0)
  // tables (device, int32)
  int* fa_row[kMaxConv] = {};  // output pixel -> input pixel base (forward A rows)
  int* fa_col[kMaxConv] = {};  // forward k -> offset
  int* zpix[kMaxConv] = {};    // output pixel -> zero-bordered delta buffer position
  int* da_row[kMaxConv] = {};  // delta A rows: input pixel -> dZpad base
  int* da_col[kMaxConv] = {};  // delta k = (ky, kx, co) -> offset
  int* wa_row[kMaxConv] = {};  // weight-gradient A rows (ky, ci) -> inT offset (+ the ones row)
  int* wa_col[kMaxConv] = {};  // weight-gradient K (m, y, x') -> inT offset
  int* wb_row[kMaxConv] = {};  // weight-gradient B rows (kx, co) -> dZs offset
  int* wb_col[kMaxConv] = {};  // weight-gradient K (m, y, x') -> dZs offset
  int* prow[kMaxConv] = {};    // weight-gradient row (ky, ci) -> ci*k*k + ky*k (-1: bias row)
  int* pcol[kMaxConv] = {};    // weight-gradient column (kx, co) -> co*cin*k*k + kx
  int* bcol[kMaxConv] = {};    // bias row column (kx, co) -> co if kx == 0 else -1
  int num_sms = 148;
};

namespace {

template <typename T>
T* upload_vec(const std::vector<T>& v) {
  T* d = nullptr;
  CK(cudaMalloc(&d, sizeof(T) * std::max<size_t>(v.size(), 1)));
  CK(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return d;
}

void free_tables(ConvTcState* s) {
  int** t[] = {s->fa_row, s->fa_col, s->zpix, s->da_row, s->da_col, s->wa_row, s->wa_col,
               s->wb_row, s->wb_col, s->prow, s->pcol, s->bcol, s->c2o, s->dzo};
  for (int** a : t)
    for (int i = 0; i < kMaxConv; ++i)
      if (a[i]) {
        cudaFree(a[i]);
        a[i] = nullptr;
      }
}

// Tables of every stage for chunks of up to `mc` images (host-built, geometry only).
void build_tables(Ctx& c, int64_t mc) {
  ConvTcState* s = c.ctc;
  free_tables(s);
  const NetDev& net = c.net;
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    const int k = d.k, kk2 = k * k, pad = k - 1, H2 = d.ho + 2 * pad, W2 = d.wo + 2 * pad, wp = s->winp[i];
    const int64_t npix = (int64_t)d.ho * d.wo, nin = (int64_t)d.hin * d.win;
    const bool x_nchw = i == 0;  // stage 0 reads X [c][h][w]; later stages NHWC activations
    const int64_t limit = (int64_t)1 << 31;
    const int64_t biggest = std::max({nin * d.cin, (int64_t)H2 * W2 * d.cout, (int64_t)d.cin * d.hin * wp,
                                      (int64_t)k * mc * d.cout * d.ho * wp / std::max<int64_t>(mc, 1)});
    if (mc * biggest >= limit || (int64_t)k * mc * d.cout * d.ho * wp >= limit)
      throw std::invalid_argument("conv: chunk too large for 32-bit operand tables");
    std::vector<int> fa_row((size_t)(mc * npix)), zpix((size_t)(mc * npix));
    for (int64_t m = 0; m < mc; ++m)
      for (int y = 0; y < d.ho; ++y)
        for (int x = 0; x < d.wo; ++x) {
          const int64_t r = m * npix + (int64_t)y * d.wo + x;
          fa_row[(size_t)r] = x_nchw ? (int)(m * d.cin * nin + (int64_t)y * d.win + x)
                                     : (int)(m * nin * d.cin + ((int64_t)y * d.win + x) * d.cin);
          zpix[(size_t)r] = (int)(m * (int64_t)H2 * W2 * d.cout + ((int64_t)(y + pad) * W2 + x + pad) * d.cout);
        }
    const int Kf = d.cin * kk2;
    std::vector<int> fa_col((size_t)Kf);
    for (int q = 0; q < Kf; ++q) {
      int ci, ky, kx;
      if (s->korder[i] == 0) {
        ci = q % d.cin;
        ky = (q / d.cin) / k;
        kx = (q / d.cin) % k;
      } else {
        ci = q / kk2;
        ky = (q % kk2) / k;
        kx = q % k;
      }
      fa_col[(size_t)q] = x_nchw ? (int)(ci * nin + (int64_t)ky * d.win + kx) : (int)(((int64_t)ky * d.win + kx) * d.cin + ci);
    }
    s->fa_row[i] = upload_vec(fa_row);
    s->zpix[i] = upload_vec(zpix);
    s->fa_col[i] = upload_vec(fa_col);
    // weight gradient: shifted-rows form, or (stage 0, xcol0) the shared im2col of X
    const int64_t planeA = (int64_t)d.cin * d.hin * wp;
    const DzL& L = s->dzl[i];
    const bool xc = i == 0 && s->xcol0;
    const int nA = xc ? Kf + 1 : k * d.cin + 1, nB = xc ? d.cout : k * d.cout;
    std::vector<int> wa_row((size_t)nA), prow((size_t)nA);
    if (xc) {
      for (int q = 0; q < Kf; ++q) prow[(size_t)q] = q;  // (ci, ky, kx): the internal W order
    } else {
      for (int ky = 0; ky < k; ++ky)
        for (int ci = 0; ci < d.cin; ++ci) {
          wa_row[(size_t)ky * d.cin + ci] = (int)((int64_t)ci * d.hin * wp + (int64_t)ky * wp);
          prow[(size_t)ky * d.cin + ci] = ci * kk2 + ky * k;
        }
      wa_row[(size_t)k * d.cin] = kOnesRow;
    }
    prow[(size_t)nA - 1] = -1;
    const int64_t kw = xc ? mc * npix : mc * d.ho * wp;  // K of the weight-gradient GEMM
    std::vector<int> wa_col(xc ? 0 : (size_t)kw), wb_col(xc ? 0 : (size_t)kw);
    if (!xc)
      for (int64_t m = 0; m < mc; ++m)
        for (int y = 0; y < d.ho; ++y)
          for (int x = 0; x < wp; ++x) {
            const int64_t q = (m * d.ho + y) * wp + x;
            wa_col[(size_t)q] = (int)(m * planeA + (int64_t)y * wp + x);
            wb_col[(size_t)q] = (int)(m * L.s_m + (int64_t)y * L.s_y + x);
          }
    std::vector<int> wb_row((size_t)nB), pcol((size_t)nB), bcol((size_t)nB);
    for (int kx = 0; kx < nB / d.cout; ++kx)
      for (int co = 0; co < d.cout; ++co) {
        const size_t n = (size_t)kx * d.cout + co;
        wb_row[n] = (int)(kx * L.s_kx + co * L.s_c);
        pcol[n] = co * Kf + kx;
        bcol[n] = kx == 0 ? co : -1;
      }
    std::vector<int> c2o((size_t)(mc * nin)), dzo((size_t)(mc * npix));
    for (int64_t m = 0; m < mc; ++m) {
      for (int y = 0; y < d.hin; ++y)
        for (int x = 0; x < d.win; ++x) c2o[(size_t)(m * nin + (int64_t)y * d.win + x)] = (int)(m * planeA + (int64_t)y * wp + x);
      for (int y = 0; y < d.ho; ++y)
        for (int x = 0; x < d.wo; ++x) dzo[(size_t)(m * npix + (int64_t)y * d.wo + x)] = (int)(m * L.s_m + (int64_t)y * L.s_y + x);
    }
    s->c2o[i] = upload_vec(c2o);
    s->dzo[i] = upload_vec(dzo);
    s->wa_row[i] = xc ? nullptr : upload_vec(wa_row);
    s->wa_col[i] = xc ? nullptr : upload_vec(wa_col);
    s->wb_row[i] = upload_vec(wb_row);
    s->wb_col[i] = xc ? nullptr : upload_vec(wb_col);
    s->prow[i] = upload_vec(prow);
    s->pcol[i] = upload_vec(pcol);
    s->bcol[i] = upload_vec(bcol);
    if (i > 0) {  // delta GEMM of stage i: rows = input pixels of stage i (= stage i-1 output or pool)
      std::vector<int> da_row((size_t)(mc * nin)), da_col((size_t)d.cout * kk2);
      for (int64_t m = 0; m < mc; ++m)
        for (int y = 0; y < d.hin; ++y)
          for (int x = 0; x < d.win; ++x)
            da_row[(size_t)(m * nin + (int64_t)y * d.win + x)] =
                (int)(m * (int64_t)H2 * W2 * d.cout + ((int64_t)(y + pad) * W2 + x + pad) * d.cout);
      for (int q = 0; q < d.cout * kk2; ++q) {
        const int kyx = q / d.cout, co = q % d.cout, ky = kyx / k, kx = kyx % k;
        da_col[(size_t)q] = -(ky * W2 + kx) * d.cout + co;
      }
      s->da_row[i] = upload_vec(da_row);
      s->da_col[i] = upload_vec(da_col);
    }
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn conv_encode_fn() {
  static EncodeTiledFn fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r));
    if (!q) throw CudaError{"cuTensorMapEncodeTiled unavailable"};
    return (EncodeTiledFn)q;
  }();
  return fn;
}
// fp32 tensor, innermost dim first; strides in bytes for dims >= 1; 128B-swizzled boxes
CUtensorMap conv_map(const float* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                     bool swizzle = true) {
  CUtensorMap m;
  const uint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = conv_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<float*>(base),
                                      dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled (conv) failed (" + std::to_string((int)r) + ")"};
  return m;
}

// Direct-convolution stage parameters (GParams::mapA ...) for an NHWC input [J][cap][H][W][C]
// convolved with k x k weights into out_h x out_w outputs; false when the slab ring does not fit.
bool setup_direct(GParams& p, const float* in, int64_t cap, int H, int W, int C, int k, int out_h, int out_w,
                  int64_t mc, const float* wcopy, int Kp, int J, bool flip, int c_real = 0) {
  if (C % kCBK != 0 || W > 128) return false;
  // channels that carry data (c_real < C: a channel-padded input of one block)
  p.ksteps = c_real > 0 && c_real < C && C == kCBK ? (c_real + 7) / 8 : 4;
  p.kk = k;
  p.cbn = C / kCBK;
  p.flipB = flip ? 1 : 0;
  const bool fold_ok = [] {  // read per call: the tests toggle it within one process
    const char* e = std::getenv("DASMC_CONV_FOLD");  // 0: one MMA group per tap, unpadded slab lines (A/B, tests)
    return !(e && e[0] == '0');
  }();
  // line pitch: the next of 16 / 32 when the fold applies (then also every A start is 8-row aligned)
  int Wp = W;
  if (fold_ok && k > 1 && W <= 32 && k * p.nmma <= 256 && 32 % W != 0) Wp = W <= 16 ? 16 : 32;
  p.tma_w = W;
  p.win_w = Wp;
  W = Wp;
  p.bh = std::max(1, kCBM / W);
  p.ybl = (out_h + p.bh - 1) / p.bh;
  p.out_h = out_h;
  p.out_w = out_w;
  const int rows = std::max((p.bh + k - 1) * W, (k - 1) * (W + 1) + kCBM);
  p.slab_rows = (rows + 7) / 8 * 8;
  p.imgs_pp = (int)cap;
  p.mimg = (int)mc;
  const size_t slabb = (size_t)p.slab_rows * 128, watoms = (size_t)k * k * p.nmma * 128;
  // two [slab | atoms] stages, or resident atoms + three slabs (launch_gemm picks the same way)
  if (2 * (slabb + watoms) + 2048 > 227 * 1024 && (size_t)p.cbn * watoms + 3 * slabb + 4096 > 227 * 1024) return false;
  p.fold = fold_ok && k > 1 && 32 % W == 0 && k * p.nmma <= 256 ? 1 : 0;
  const uint64_t Wr = (uint64_t)p.tma_w;  // the input's real width
  const uint64_t da[4] = {(uint64_t)C, Wr, (uint64_t)H, (uint64_t)J * cap};
  const uint64_t sa[3] = {(uint64_t)C * 4, Wr * C * 4, (uint64_t)H * Wr * C * 4};
  const uint32_t ba[4] = {(uint32_t)kCBK, (uint32_t)Wr, p.tma_w == p.win_w ? (uint32_t)(p.bh + k - 1) : 1u, 1};
  p.mapA = conv_map(in, 4, da, sa, ba);
  const uint64_t db[3] = {(uint64_t)Kp, (uint64_t)p.nmma, (uint64_t)J};
  const uint64_t sb[2] = {(uint64_t)Kp * 4, (uint64_t)p.nmma * Kp * 4};
  const uint32_t bb[3] = {(uint32_t)kCBK, (uint32_t)p.nmma, 1};
  p.mapB = conv_map(wcopy, 3, db, sb, bb);
  return true;
}

template <int EPI>
void launch_gemm(Ctx& c, GParams& p, int act, bool direct = false) {
  if (p.nb < 1) {
    p.nb = 1;
    p.nmma_p = p.nmma;
  }
  if (p.nmma > 256) throw std::invalid_argument("conv: MMA N > 256");
  if (!p.b.vec && !direct) throw std::invalid_argument("conv: B operands are 16-byte gathers");
  const size_t fixed = 1024 + 64 * 8 + 64;
  size_t stage_bytes, wres = 0;  // wres: resident weight atoms (direct kernels)
  int stages;
  if (direct && EPI == kEpiConvDw) {
    p.nsub = 1;
    stage_bytes = (size_t)kCBM * 128 + (size_t)p.nmma * 128 + (size_t)p.stg_bytes;
    stages = (int)std::min<size_t>(8, (227 * 1024 - fixed) / stage_bytes);
  } else if (direct) {
    p.nsub = 1;
    const size_t slab = (size_t)p.slab_rows * 128, watoms = (size_t)p.kk * p.kk * p.nmma * 128;
    const bool persist_ok = [] {  // read per call: the tests toggle it within one process
      const char* e = std::getenv("DASMC_CONV_PERSIST");  // 0: weight atoms re-loaded with every tile (A/B, tests)
      return !(e && e[0] == '0');
    }();
    wres = (persist_ok || 2 * (slab + watoms) + 2048 > 227 * 1024) && (size_t)p.cbn * watoms + 3 * slab + 4096 <= 227 * 1024
               ? (size_t)p.cbn * watoms
               : 0;
    p.persist = wres ? 1 : 0;
    stage_bytes = wres ? slab : slab + watoms;
    stages = (int)std::min<size_t>(wres ? 6 : 4, (227 * 1024 - fixed - wres) / stage_bytes);
  } else {
    // Atoms per stage: several 32-wide k atoms per pipeline hand-off (the producer -> MMA ->
    // producer round trip costs hundreds of cycles; conv tiles have few k atoms), a divisor of
    // the atom count when one exists
    const int natoms = p.nkb;  // callers pass the atom count
    const size_t atom_bytes = (size_t)kCBM * 128 + (size_t)p.nmma * 128;
    auto fits = [&](int ns) { return 2 * ns * atom_bytes + fixed <= 227 * 1024; };  // >= 2 stages
    int nsub = 1;
    for (int cand : {4, 3, 2})
      if (natoms % cand == 0 && fits(cand)) {
        nsub = cand;
        break;
      }
    if (nsub == 1 && natoms > 8)
      for (int cand : {4, 3, 2})
        if (fits(cand)) {  // padded last stage (zero-filled atoms)
          nsub = cand;
          break;
        }
    p.nsub = nsub;
    p.nkb = (natoms + nsub - 1) / nsub;
    stage_bytes = (size_t)nsub * atom_bytes;
    // two CTAs per SM when each gets >= 3 stages in ~110 KB, else one CTA with up to 6 stages
    stages = (int)std::min<size_t>(6, (110 * 1024 - fixed) / stage_bytes);
    if (stages < 3) stages = (int)std::min<size_t>(6, (227 * 1024 - fixed) / stage_bytes);
  }
  if (stages < 2) throw std::invalid_argument("conv: GEMM tile does not fit in shared memory");
  p.stages = stages;
  const size_t smem = 1024 + stages * stage_bytes + wres + (3 * stages + 16) * 8 + 16;
  int tc = 32;
  while (tc < (direct && EPI != kEpiConvDw && p.fold ? p.kk * p.nmma : p.nmma)) tc <<= 1;
  p.tcols_half = tc;
  static const int dbg = [] {
    const char* e = std::getenv("DASMC_CONV_DBG");
    return e ? std::atoi(e) : 0;
  }();
  p.dbg = dbg;
  const int units = direct && EPI != kEpiConvDw ? p.J * p.mimg * p.ybl : p.rtiles * ((p.J + p.nb - 1) / p.nb);
  // gather-mode forward without a second (channel-major) output: 4 producer + 8 epilogue warps (measured on
  // B200: C3 stage 0, pooled, 5.1 -> 3.5 ms; with the second output, C4 stage 0, 6.7 -> 8.0 ms, so 8 + 4 stays)
  const bool ew8 = EPI == kEpiConvFwd && !direct && !p.out2;
  auto go = [&](auto act_c, auto dir_c, auto ew_c) {
    constexpr int A_ = decltype(act_c)::value;
    constexpr bool DI = decltype(dir_c)::value;
    constexpr bool E8 = decltype(ew_c)::value && EPI == kEpiConvFwd && !DI;
    auto kern = conv_tc_kernel<EPI, A_, E8, DI>;
    static bool attr[kMaxDevices] = {};  // one flag per instantiation and device
    const int dv = current_device();
    if (!attr[dv]) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr[dv] = true;
    }
    // unified L1 / shared split: just the shared memory two CTAs need, the rest stays L1
    const int carve = (int)std::min<size_t>(100, (2 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    int per_sm = 1;
    constexpr int NT = ConvWarps<DI, DI && EPI == kEpiConvDw, E8>::T;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    per_sm = std::max(1, std::min(2, per_sm));
    if (2 * tc * per_sm > 512) per_sm = 1;  // TMEM: 512 columns per SM
    p.nacc = 2;
    while (p.nacc < 8 && 2 * p.nacc * tc * per_sm <= 512) p.nacc *= 2;
    if (const char* e = std::getenv("DASMC_CONV_NACC")) p.nacc = std::max(2, std::min(p.nacc, std::atoi(e)));  // A/B
    const int grid = std::max(1, std::min(units, c.ctc->num_sms * per_sm));
    kern<<<grid, NT, smem, c.stream>>>(p);
    LAUNCHED();
  };
  if (!p.a.vec && !direct) throw std::invalid_argument("conv: A operands are 16-byte gathers");
  auto go_av = [&](auto act_c) {
    if (direct)
      go(act_c, std::true_type{}, std::false_type{});
    else if (ew8)
      go(act_c, std::false_type{}, std::true_type{});
    else
      go(act_c, std::false_type{}, std::false_type{});
  };
  if (act == DASMC_RELU)
    go_av(std::integral_constant<int, DASMC_RELU>{});
  else
    go_av(std::integral_constant<int, DASMC_TANH>{});
}

// [m][c][h][w] (stage 0: X) or NHWC [m][h][w][c] -> [m][c][h][w_p], zeros at x' >= w (the
// buffer is a scratch shared by the stages, so the padding is rewritten every time)
__global__ void to_chw_pad_kernel(const float* __restrict__ src, int64_t src_ps, int nhwc, int C, int H, int W, int Wp,
                                  float* __restrict__ dst, int64_t dst_ps, int64_t M, int64_t J) {
  const int64_t per = (int64_t)C * H * Wp, total = J * M * per;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / (M * per), rem = g - j * M * per, m = rem / per;
    const int o = (int)(rem - m * per);  // (c, y, x') order of the destination
    const int c = o / (H * Wp), yx = o - c * H * Wp, y = yx / Wp, x = yx - y * Wp;
    float v = 0.f;
    if (x < W) {
      const int64_t s0 = j * src_ps + m * (int64_t)C * H * W;
      v = src[s0 + (nhwc ? ((int64_t)y * W + x) * C + c : ((int64_t)c * H + y) * W + x)];
    }
    dst[j * dst_ps + m * per + o] = v;
  }
}

}  // namespace

// ---- public entry points (conv_tc.cuh) ----------------------------------------------------------
bool cnn_tc_eligible(const Ctx& c) {
  const NetDev& n = c.net;
  if (n.nconv < 1) return false;
  for (int i = 0; i < n.nconv; ++i) {
    const ConvDev& d = n.conv[i];
    if (d.cout % 4 != 0 || d.cout > 64 || d.cin > 64 || d.k * d.cout > 256) return false;  // MMA N <= 256
    if (i > 0 && d.cin % 4 != 0) return false;
  }
  return true;
}

void cnn_tc_init(Ctx& c) {
  auto* s = new ConvTcState();
  c.ctc = s;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, dev));
  const NetDev& net = c.net;
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    s->korder[i] = (i > 0 && d.cin % 4 == 0) ? 0 : 1;
    s->nmmaF[i] = round_up(d.cout, 16);
    s->KpF[i] = round_up(d.cin * d.k * d.k, kCBK);
    s->cpd[i] = d.cout;
    if (i > 0 && net.conv[i - 1].pool && d.cin < kCBK && d.cin % 4 == 0 && s->korder[i] == 0 && d.win <= 32 &&
        !(std::getenv("DASMC_CONV_CPAD") && std::getenv("DASMC_CONV_CPAD")[0] == '0') &&
        !(std::getenv("DASMC_CONV_DIRECT") && std::getenv("DASMC_CONV_DIRECT")[0] == '0')) {
      // pad the pooled input of this stage to one 32-channel block if its direct convolution then fits
      const int bh = std::max(1, kCBM / d.win);
      const size_t slabb = (size_t)round_up(std::max((bh + d.k - 1) * d.win, (d.k - 1) * (d.win + 1) + kCBM), 8) * 128;
      const size_t watoms = (size_t)d.k * d.k * s->nmmaF[i] * 128;
      if (2 * (slabb + watoms) + 2048 <= 227 * 1024 || watoms + 3 * slabb + 4096 <= 227 * 1024) {
        s->cpd[i - 1] = kCBK;
        s->KpF[i] = d.k * d.k * kCBK;
      }
    }
    s->nmmaD[i] = round_up(d.cin, 16);
    s->KpD[i] = round_up(d.cout * d.k * d.k, kCBK);
    s->nmmaW[i] = round_up(d.k * d.cout, 16);
    if (i == 0 && (d.ho * d.wo) % 4 == 0) {
      s->xcol0 = true;
      s->nmmaW[0] = round_up(d.cout, 16);
    }
    s->dwt[i] = !(i == 0 && s->xcol0) && kCBM % d.cin == 0 && d.k * d.cout <= 256 && d.k * d.cin < 8 * kCBM &&
                d.cout % 8 == 0;
    s->winp[i] = round_up(d.win, 4);
    CK(cudaMalloc(&s->Wf[i], sizeof(float) * (size_t)c.Jmax * s->nmmaF[i] * s->KpF[i]));
    if (i > 0) CK(cudaMalloc(&s->Wd[i], sizeof(float) * (size_t)c.Jmax * s->nmmaD[i] * s->KpD[i]));
  }
  if (const char* e = std::getenv("DASMC_CONV_DIRECT")) s->direct_ok = e[0] != '0';
  if (const char* e = std::getenv("DASMC_CONV_BATCH0")) s->batch0 = e[0] != '0';
  // weight gradient from TMA + shared-memory shifts (DASMC_CONV_DWT=0: the gather form with k kx-shifted
  // delta copies in HBM)
  const char* dwt_env = std::getenv("DASMC_CONV_DWT");
  const bool dwt_on = !(dwt_env && dwt_env[0] == '0');
  for (int i = 0; i < net.nconv; ++i) s->dwt[i] = s->dwt[i] && s->direct_ok && dwt_on;
  const float ones[4] = {1.f, 1.f, 1.f, 1.f};
  CK(cudaMalloc(&s->ones, sizeof(ones)));
  CK(cudaMemcpy(s->ones, ones, sizeof(ones), cudaMemcpyHostToDevice));
  cnn_tc_refresh_data(c, c.X, c.n_active);
}

void cnn_tc_refresh_data(Ctx& c, const float* X, int64_t rows) {
  ConvTcState* s = c.ctc;
  const int64_t d = (int64_t)c.net.in_c * c.net.in_h * c.net.in_w;
  if (rows > s->Xr_rows) {
    CK(cudaStreamSynchronize(c.stream));
    if (s->Xr) CK(cudaFree(s->Xr));
    s->Xr = nullptr;
    const int64_t cap = std::max(rows, c.n);
    CK(cudaMalloc(&s->Xr, sizeof(float) * (size_t)cap * d));
    s->Xr_rows = cap;
  }
  round_tf32_kernel<<<grid_of(rows * d), 256, 0, c.stream>>>(X, s->Xr, rows * d);
  LAUNCHED();
  const ConvDev& d0 = c.net.conv[0];
  const int64_t per = (int64_t)d0.ho * d0.wo * s->KpF[0];
  if (rows > s->Xcol_rows) {
    CK(cudaStreamSynchronize(c.stream));
    if (s->Xcol) CK(cudaFree(s->Xcol));
    s->Xcol = nullptr;
    const int64_t cap = std::max(rows, c.n);
    CK(cudaMalloc(&s->Xcol, sizeof(float) * (size_t)cap * per));
    s->Xcol_rows = cap;
  }
  im2col_x_kernel<<<grid_of(rows * per), 256, 0, c.stream>>>(d0, s->Xr, rows, s->KpF[0], s->Xcol);
  LAUNCHED();
  if (s->xcol0) {
    const int K0 = d0.cin * d0.k * d0.k;
    const int64_t npix = (int64_t)d0.ho * d0.wo;
    if (rows > s->XcolT_rows) {
      CK(cudaStreamSynchronize(c.stream));
      if (s->XcolT) CK(cudaFree(s->XcolT));
      s->XcolT = nullptr;
      const int64_t cap = std::max(rows, c.n);
      if ((int64_t)(K0 + 1) * cap * npix >= ((int64_t)1 << 31)) throw std::invalid_argument("conv: X im2col too large");
      CK(cudaMalloc(&s->XcolT, sizeof(float) * (size_t)(K0 + 1) * cap * npix));
      s->XcolT_rows = cap;
    }
    xcolT_kernel<<<grid_of(rows * npix * (K0 + 1)), 256, 0, c.stream>>>(s->Xcol, rows * npix, s->KpF[0], K0,
                                                                  s->XcolT_rows * npix, s->XcolT);
    LAUNCHED();
  }
}

void cnn_tc_free(Ctx& c) {
  ConvTcState* s = c.ctc;
  if (!s) return;
  free_tables(s);
  for (int i = 0; i < kMaxConv; ++i) {
    float* p[] = {s->Wf[i], s->Wd[i], s->dP[i], s->inT[i], s->dZs[i]};
    for (float* q : p)
      if (q) cudaFree(q);
    if (s->pcode[i]) cudaFree(s->pcode[i]);
  }
  if (s->Xr) cudaFree(s->Xr);
  if (s->Xcol) cudaFree(s->Xcol);
  if (s->XcolT) cudaFree(s->XcolT);
  if (s->ones) cudaFree(s->ones);
  delete s;
  c.ctc = nullptr;
}

int64_t cnn_tc_image_floats(const Ctx& c) {
  const NetDev& net = c.net;
  int64_t f = 0;
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    const int64_t wp = round_up(d.win, 4);
    f += act_plane(d) + (i > 0 ? pad_plane(d) : 0);  // output, zero-bordered delta (stages > 0)
    if (d.pool) f += (pool_plane(d) + 3) / 4;        // argmax codes (bytes)
    const bool one_copy = c.ctc && (c.ctc->dwt[i] || (i == 0 && c.ctc->xcol0));
    f += (int64_t)(one_copy ? 1 : d.k) * d.cout * d.ho * wp;  // channel-major delta copy (k kx-shifted ones: gather form)
    if (i > 0) f += (int64_t)d.cin * d.hin * wp;     // channel-major input copy
    if (d.pool) f += (int64_t)d.sh * d.sw * (c.ctc ? c.ctc->cpd[i] : d.cout);
    else if (i == net.nconv - 1) f += act_plane(d);  // the flatten copy
    if (d.pool && i + 1 < net.nconv) f += pool_plane(d);
  }
  return f;
}

// Stage buffers for chunks of mc images: cact = NHWC stage output, cpool = pooled NHWC (or the
// head's flatten order for the last stage), cdel = zero-bordered NHWC delta, dP = delta of a
// pooled non-last stage output, inT / dZs = the weight-gradient operands.
void cnn_tc_alloc(Ctx& c, int64_t mc) {
  ConvTcState* s = c.ctc;
  const NetDev& net = c.net;
  const size_t J = (size_t)c.Jmax;
  for (int i = 0; i < net.nconv; ++i) {
    float** bufs[] = {&c.cact[i], &c.cpool[i], &c.cdel[i], &s->dP[i], &s->inT[i], &s->dZs[i]};
    for (float** b : bufs)
      if (*b) {
        CK(cudaFree(*b));
        *b = nullptr;
      }
    if (s->pcode[i]) {
      CK(cudaFree(s->pcode[i]));
      s->pcode[i] = nullptr;
    }
    const ConvDev& d = net.conv[i];
    const size_t wp = (size_t)s->winp[i];
    CK(cudaMalloc(&c.cact[i], sizeof(float) * J * mc * act_plane(d)));
    if (i > 0) {  // stage 0 has no delta GEMM: its zero-bordered NHWC delta is never read, so never written
      CK(cudaMalloc(&c.cdel[i], sizeof(float) * J * mc * pad_plane(d)));
      CK(cudaMemsetAsync(c.cdel[i], 0, sizeof(float) * J * mc * pad_plane(d), c.stream));
    }
    if (d.pool) CK(cudaMalloc(&s->pcode[i], J * mc * pool_plane(d)));
    const bool last = i == net.nconv - 1;
    if (d.pool || last) {
      const size_t pf = J * mc * (size_t)(d.pool ? (int64_t)d.sh * d.sw * s->cpd[i] : act_plane(d));
      CK(cudaMalloc(&c.cpool[i], sizeof(float) * pf));
      if (d.pool && s->cpd[i] != d.cout) CK(cudaMemsetAsync(c.cpool[i], 0, sizeof(float) * pf, c.stream));  // padding channels
    }
    if (d.pool && !last) CK(cudaMalloc(&s->dP[i], sizeof(float) * J * mc * pool_plane(d)));
    const size_t fa = (size_t)mc * d.cin * d.hin * wp * (i == 0 ? 1 : J);  // stage 0: shared by particles
    DzL& L = s->dzl[i];
    if (s->dwt[i]) {  // unshifted, flattened channel-major planes of row stride win_p: [m][c][y * win_p + x]
      L.kc = 1;
      L.s_y = (int)wp;
      L.s_c = (int64_t)d.ho * wp;
      L.s_m = d.cout * L.s_c;
      L.s_kx = 0;
    } else if (i == 0 && s->xcol0) {  // unshifted, channel-major [c][m][y*wo + x]
      L.kc = 1;
      L.s_y = d.wo;
      L.s_m = (int64_t)d.ho * d.wo;
      L.s_c = mc * L.s_m;
      L.s_kx = 0;
    } else {  // k copies [kx][m][c][y][x'], x' < win_p
      L.kc = d.k;
      L.s_y = (int)wp;
      L.s_c = (int64_t)d.ho * wp;
      L.s_m = d.cout * L.s_c;
      L.s_kx = mc * L.s_m;
    }
    const size_t fb = J * (L.kc > 1 ? (size_t)L.kc * L.s_kx : s->dwt[i] ? (size_t)mc * L.s_m : (size_t)d.cout * L.s_c);
    CK(cudaMalloc(&s->inT[i], sizeof(float) * fa));
    CK(cudaMemsetAsync(s->inT[i], 0, sizeof(float) * fa, c.stream));
    CK(cudaMalloc(&s->dZs[i], sizeof(float) * fb));
    CK(cudaMemsetAsync(s->dZs[i], 0, sizeof(float) * fb, c.stream));
  }
  build_tables(c, mc);
  s->mcap = mc;
}

// Flatten buffer the head reads (and its delta is written to): [Jmax][mcap][F].
float* cnn_tc_flat(Ctx& c) { return c.cpool[c.net.nconv - 1]; }

void cnn_tc_weights(Ctx& c, const float* theta, int64_t J, bool need_grad) {
  ConvTcState* s = c.ctc;
  const NetDev& net = c.net;
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    conv_wcopy_kernel<<<grid_of(J * s->nmmaF[i] * s->KpF[i]), 256, 0, c.stream>>>(
        theta, net.Dp, d.woff, d.cin, d.k, d.cout, 0, s->korder[i], s->nmmaF[i], s->KpF[i], J, s->Wf[i],
        i > 0 && net.conv[i - 1].pool ? s->cpd[i - 1] : d.cin);
    LAUNCHED();
    if (need_grad && i > 0) {
      conv_wcopy_kernel<<<grid_of(J * s->nmmaD[i] * s->KpD[i]), 256, 0, c.stream>>>(
          theta, net.Dp, d.woff, d.cin, d.k, d.cout, 1, 0, s->nmmaD[i], s->KpD[i], J, s->Wd[i], d.cin);
      LAUNCHED();
    }
  }
}

void cnn_tc_forward(Ctx& c, const float* theta, int64_t J, int64_t m0, int64_t mc) {
  ConvTcState* s = c.ctc;
  const NetDev& net = c.net;
  const int64_t img = (int64_t)net.in_c * net.in_h * net.in_w;
  const int64_t cap = s->mcap;
  for (int i = 0; i < net.nconv; ++i) {
    const ConvDev& d = net.conv[i];
    const int64_t R = mc * d.ho * d.wo;
    GParams p{};
    if (i == 0) {  // the shared im2col of X: dense 16-byte rows
      p.a.base = s->Xcol + m0 * d.ho * d.wo * s->KpF[0];
      p.a.ps = 0;
      p.a.ld = s->KpF[0];
      p.a.nrows = (int)R;
      p.a.K = s->KpF[0];
      p.a.vec = 1;
    } else {
      const ConvDev& dp = net.conv[i - 1];
      p.a.base = dp.pool ? c.cpool[i - 1] : c.cact[i - 1];
      p.a.ps = cap * (dp.pool ? (int64_t)dp.sh * dp.sw * s->cpd[i - 1] : act_plane(dp));
      p.a.rowoff = s->fa_row[i];
      p.a.nrows = (int)R;
      p.a.coloff = s->fa_col[i];
      p.a.K = d.cin * d.k * d.k;
      p.a.vec = s->korder[i] == 0 ? 1 : 0;
    }
    p.b.base = s->Wf[i];
    p.b.ps = (int64_t)s->nmmaF[i] * s->KpF[i];
    p.b.ld = s->KpF[i];
    p.b.nrows = s->nmmaF[i];
    p.b.K = s->KpF[i];
    p.b.vec = 1;
    p.ones = s->ones;
    p.J = (int)J;
    p.rtiles = (int)((R + kCBM - 1) / kCBM);
    p.nkb = s->KpF[i] / kCBK;
    p.nmma = s->nmmaF[i];
    if (i == 0 && s->batch0 && d.cout == s->nmmaF[0]) {
      // X's im2col is shared by every particle: nb particles per unit (MMA N = nb * cout, one A tile
      // read for nb particles); their weight copies are consecutive rows of Wf
      p.nb = std::max(1, std::min<int>(256 / s->nmmaF[0], (int)J));
      p.nmma_p = s->nmmaF[0];
      p.nmma = round_up(p.nb * p.nmma_p, 16);
      p.b.nrows = p.nb * p.nmma_p;
    }
    p.Rvalid = (int)R;
    p.nvalid = d.cout;
    p.out = c.cact[i];
    p.out_ps = cap * act_plane(d);
    p.out_ld = d.cout;
    p.theta = theta;
    p.Dp = net.Dp;
    p.boff = d.boff;
    const bool last = i == net.nconv - 1;
    int64_t nxt_ps = 0;  // per-particle floats of the next stage's channel-major input copy
    if (!last) {
      const ConvDev& dn = net.conv[i + 1];
      nxt_ps = cap * (int64_t)dn.cin * dn.hin * s->winp[i + 1];
      if (!d.pool) {  // the epilogue writes it (no pool in between)
        p.out2 = s->inT[i + 1];
        p.out2_ps = nxt_ps;
        p.out2off = s->c2o[i + 1];
        p.out2_cs = (int64_t)dn.hin * s->winp[i + 1];
        p.out2_k = 1;
      }
    }
    // direct convolution from TMA slabs when the input has 32-channel blocks (DASMC_CONV_DIRECT=0: gathers)
    bool direct = false;
    if (i > 0 && s->direct_ok) {
      const ConvDev& dp = net.conv[i - 1];
      direct = setup_direct(p, p.a.base, cap, d.hin, d.win, dp.pool ? s->cpd[i - 1] : d.cin, d.k, d.ho, d.wo, mc,
                            s->Wf[i], s->KpF[i], (int)J, false, d.cin);
      if (!direct && dp.pool && s->cpd[i - 1] != dp.cout)
        throw std::invalid_argument("conv: channel-padded input without a direct convolution");
      (void)dp;
    }
    launch_gemm<kEpiConvFwd>(c, p, net.act, direct);
    if (d.pool) {
      launch_pool_fwd(c, d, c.cact[i], cap * act_plane(d), c.cpool[i],
                      cap * (last ? pool_plane(d) : (int64_t)d.sh * d.sw * s->cpd[i]), mc, J, last ? 1 : 0,
                      last ? nullptr : s->inT[i + 1], nxt_ps, last ? 0 : s->winp[i + 1], s->pcode[i], last ? d.cout : s->cpd[i]);
    } else if (last) {
      nhwc_to_flat_kernel<<<grid_of(J * mc * act_plane(d)), 256, 0, c.stream>>>(d, c.cact[i], cap * act_plane(d),
                                                                                 c.cpool[i], cap * act_plane(d), mc, J);
      LAUNCHED();
    }
  }
}

// Backward through the stages, given the flatten delta (head backward, act' applied unless the
// last stage pools) in cnn_tc_flat(c); e carries the chunk's accumulation mode.
void cnn_tc_backward(Ctx& c, const float* theta, int64_t J, int64_t m0, int64_t mc, const EpiParams& e) {
  ConvTcState* s = c.ctc;
  const NetDev& net = c.net;
  const int64_t img = (int64_t)net.in_c * net.in_h * net.in_w;
  const int64_t cap = s->mcap;
  const int L = net.nconv - 1;
  // per-particle floats of dZs[i]
  auto dzs_ps = [&](int i) {
    const DzL& Lz = s->dzl[i];
    return Lz.kc > 1 ? (int64_t)Lz.kc * Lz.s_kx : s->dwt[i] ? cap * Lz.s_m : (int64_t)net.conv[i].cout * Lz.s_c;
  };
  {
    const ConvDev& d = net.conv[L];
    if (d.pool) {
      launch_pool_bwd(c, d, net.act, c.cact[L], cap * act_plane(d), s->pcode[L], c.cpool[L], cap * pool_plane(d), 1,
                      L > 0 ? c.cdel[L] : nullptr, cap * pad_plane(d), mc, J, s->dZs[L], dzs_ps(L), s->dzl[L]);
    } else {
      flat_to_dzpad_kernel<<<grid_of(J * mc * act_plane(d)), 256, 0, c.stream>>>(
          d, c.cpool[L], cap * act_plane(d), c.cdel[L], cap * pad_plane(d), mc, J, s->dZs[L], dzs_ps(L), s->dzl[L]);
      LAUNCHED();
    }
  }
  for (int i = L; i >= 0; --i) {
    const ConvDev& d = net.conv[i];
    const int wp = s->winp[i];
    // ---- weight gradient + fused leapfrog:
    //   shifted-rows form  D[(ky, ci) | ones, (kx, co)] = sum_(m, y, x') inT[ci][y + ky][x'] dZs[kx][co][y][x']
    //   stage 0 (xcol0)    D[(ci, ky, kx) | ones, co]  = sum_(m, p) XcolT[(ci, ky, kx)][m, p] dZ[co][m, p]
    {
      const bool xc = i == 0 && s->xcol0;
      const int64_t planeA = (int64_t)d.cin * d.hin * wp;
      GParams p{};
      if (s->dwt[i]) {  // TMA operands: inT rows (ky, ci) at q + ky * win_p, unshifted delta rows (kx, co) at q - kx
        if (i == 0) {
          to_chw_pad_kernel<<<grid_of(mc * planeA), 256, 0, c.stream>>>(s->Xr + m0 * img, 0, 0, d.cin, d.hin, d.win,
                                                                       wp, s->inT[0], 0, mc, 1);
          LAUNCHED();
        }
        const uint64_t imgsA = i == 0 ? (uint64_t)cap : (uint64_t)J * cap;
        const uint64_t da[3] = {(uint64_t)d.hin * wp, (uint64_t)d.cin, imgsA};
        const uint64_t sa[2] = {(uint64_t)d.hin * wp * 4, (uint64_t)planeA * 4};
        const uint32_t ba[3] = {(uint32_t)kCBK, (uint32_t)d.cin, 1};
        p.mapA = conv_map(s->inT[i], 3, da, sa, ba);
        // the unshifted delta: unswizzled staging boxes [cout][halo + 32] starting at q - halo
        p.halo = round_up(d.k - 1, 4);
        p.stg_bytes = round_up(d.cout * (p.halo + kCBK) * 4, 1024);
        const uint64_t db[3] = {(uint64_t)d.ho * wp, (uint64_t)d.cout, (uint64_t)J * cap};
        const uint64_t sb[2] = {(uint64_t)d.ho * wp * 4, (uint64_t)d.cout * d.ho * wp * 4};
        const uint32_t bb[3] = {(uint32_t)(p.halo + kCBK), (uint32_t)d.cout, 1};
        p.mapB = conv_map(s->dZs[i], 3, db, sb, bb, false);
        p.kk = d.k;
        p.cin_rows = d.cin;
        p.cout_rows = d.cout;
        p.wpd = wp;
        p.kpi = (int)((d.ho * wp + kCBK - 1) / kCBK);
        p.mimg = (int)mc;
        p.imgs_pp = (int)cap;
        p.a_imgs_pp = i == 0 ? 0 : (int)cap;
        p.J = (int)J;
        p.rtiles = (d.k * d.cin + 1 + kCBM - 1) / kCBM;
        p.nkb = (int)mc * p.kpi;
        p.nmma = s->nmmaW[i];
        p.nvalid = d.k * d.cout;
        p.Dp = net.Dp;
        p.boff = d.boff;
        p.e = e;
        p.woff = d.woff;
        p.nrows_w = d.k * d.cin + 1;
        p.prow = s->prow[i];
        p.pcol = s->pcol[i];
        p.bcol = s->bcol[i];
        p.ones = s->ones;
        launch_gemm<kEpiConvDw>(c, p, net.act, true);
      } else {
      if (xc) {
        const int64_t npix = (int64_t)d.ho * d.wo;
        p.a.base = s->XcolT + m0 * npix;
        p.a.ps = 0;
        p.a.ld = (int)(s->XcolT_rows * npix);
        p.a.nrows = d.cin * d.k * d.k + 1;
        p.a.K = (int)(mc * npix);
      } else {
        if (i == 0) {  // stage 0's input is X: its channel-major padded copy, shared by the particles
          to_chw_pad_kernel<<<grid_of(mc * planeA), 256, 0, c.stream>>>(s->Xr + m0 * img, 0, 0, d.cin, d.hin, d.win,
                                                                       wp, s->inT[0], 0, mc, 1);
          LAUNCHED();
        }
        p.a.base = s->inT[i];
        p.a.ps = i == 0 ? 0 : cap * planeA;
        p.a.rowoff = s->wa_row[i];
        p.a.nrows = d.k * d.cin + 1;
        p.a.coloff = s->wa_col[i];
        p.a.K = (int)(mc * d.ho * wp);
      }
      p.a.vec = 1;
      p.b.base = s->dZs[i];
      p.b.ps = dzs_ps(i);
      p.b.rowoff = s->wb_row[i];
      p.b.nrows = s->dzl[i].kc * d.cout;
      p.b.coloff = s->wb_col[i];
      p.b.K = p.a.K;
      p.b.vec = 1;
      p.ones = s->ones;
      p.J = (int)J;
      p.rtiles = (p.a.nrows + kCBM - 1) / kCBM;
      p.nkb = (p.a.K + kCBK - 1) / kCBK;
      p.nmma = s->nmmaW[i];
      p.nvalid = p.b.nrows;
      if (xc && s->batch0 && d.cout == s->nmmaW[0]) {
        // the transposed im2col of X is shared by every particle: nb particles per unit; the unshifted
        // channel-major deltas [c][m][pixel] of consecutive particles are consecutive rows of s_c floats
        // K is the whole chunk, so the grid is only rtiles * J / nb units: batch while ~80 % of the SMs keep
        // one (measured on B200: C3 J = 512 nb 1 / 2 / 4 / 16 = 6.4 / 3.5 / 2.1 / 4.7 ms, C4 J = 256
        // nb 1 / 2 / 4 / 8 = 2.8 / 1.6 / 2.3 / 3.7 ms per launch)
        int nbw = 1;
        while (2 * nbw * d.cout <= 256 && 5 * p.rtiles * (J / (2 * nbw)) >= 4 * s->num_sms) nbw *= 2;
        if (const char* e = std::getenv("DASMC_CONV_NBW")) nbw = std::max(1, std::min(256 / d.cout, std::atoi(e)));
        if ((int64_t)nbw * d.cout * s->dzl[0].s_c < ((int64_t)1 << 31)) {
          p.nb = nbw;
          p.nmma_p = d.cout;
          p.nmma = round_up(nbw * d.cout, 16);
          p.b.rowoff = nullptr;
          p.b.ld = (int)s->dzl[0].s_c;
          p.b.nrows = nbw * d.cout;
        }
      }
      p.Dp = net.Dp;
      p.boff = d.boff;
      p.e = e;
      p.woff = d.woff;
      p.nrows_w = p.a.nrows;
      p.prow = s->prow[i];
      p.pcol = s->pcol[i];
      p.bcol = s->bcol[i];
      launch_gemm<kEpiConvDw>(c, p, net.act);
      }
    }
    if (i == 0) break;
    // ---- delta of the stage input: dI[r_in, ci] = sum_(ky,kx,co) dZpad[.] W[co, ci, ky, kx]
    const ConvDev& dp = net.conv[i - 1];
    const int64_t Rin = mc * d.hin * d.win;
    GParams p{};
    p.a.base = c.cdel[i];
    p.a.ps = cap * pad_plane(d);
    p.a.rowoff = s->da_row[i];
    p.a.nrows = (int)Rin;
    p.a.coloff = s->da_col[i];
    p.a.K = d.cout * d.k * d.k;
    p.a.vec = 1;
    p.b.base = s->Wd[i];
    p.b.ps = (int64_t)s->nmmaD[i] * s->KpD[i];
    p.b.ld = s->KpD[i];
    p.b.nrows = s->nmmaD[i];
    p.b.K = s->KpD[i];
    p.b.vec = 1;
    p.ones = s->ones;
    p.J = (int)J;
    p.rtiles = (int)((Rin + kCBM - 1) / kCBM);
    p.nkb = s->KpD[i] / kCBK;
    p.nmma = s->nmmaD[i];
    p.Rvalid = (int)Rin;
    p.nvalid = d.cin;
    if (dp.pool) {  // delta of the pooled output (NHWC); its max-pool backward follows
      p.out = s->dP[i - 1];
      p.out_ps = cap * pool_plane(dp);
      p.out_ld = dp.cout;
    } else {  // pre-activation delta of stage i-1: act'(a_{i-1}), into its zero-bordered buffer
      p.out = c.cdel[i - 1];  // nullptr for stage 0 (no delta GEMM reads it)
      p.out_ps = cap * pad_plane(dp);
      p.outoff = s->zpix[i - 1];
      p.mask = c.cact[i - 1];
      p.mask_ps = cap * act_plane(dp);
      p.mask_ld = dp.cout;
      // and its channel-major (kx-shifted) copies (stage i-1's weight-gradient B operand)
      p.out2 = s->dZs[i - 1];
      p.out2_ps = dzs_ps(i - 1);
      p.out2off = s->dzo[i - 1];
      p.out2_cs = s->dzl[i - 1].s_c;
      p.out2_ks = s->dzl[i - 1].s_kx;
      p.out2_k = s->dzl[i - 1].kc;
    }
    const int H2 = d.ho + 2 * (d.k - 1), W2 = d.wo + 2 * (d.k - 1);
    const bool direct = s->direct_ok && setup_direct(p, c.cdel[i], cap, H2, W2, d.cout, d.k, d.hin, d.win, mc,
                                                     s->Wd[i], s->KpD[i], (int)J, true);
    launch_gemm<kEpiConvDx>(c, p, net.act, direct);
    if (dp.pool)
      launch_pool_bwd(c, dp, net.act, c.cact[i - 1], cap * act_plane(dp), s->pcode[i - 1], s->dP[i - 1],
                      cap * pool_plane(dp), 0, i - 1 > 0 ? c.cdel[i - 1] : nullptr, cap * pad_plane(dp), mc, J,
                      s->dZs[i - 1], dzs_ps(i - 1), s->dzl[i - 1]);
  }
}

}  // namespace dasmc_b200
