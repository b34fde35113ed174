// tcgen05 / TMA / TMEM tensor-core kernels for sm_100a (see tc_gemm.cuh).
//
// One persistent, warp-specialised kernel template runs both GEMM shapes:
//   warp 0      TMA producer: 128B-swizzled K-major tiles of A (128 x 32 fp32)
//               and B (N x 32 fp32) into a STAGES-deep shared-memory ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32,
//               M = 128, N <= 256, K = 8 per instruction), double-buffered
//               128 x 256 fp32 accumulators in TMEM
//   warps 2..9  epilogue: tcgen05.ld 32x32b rows -> registers -> fused math
//               (two warps per TMEM lane group, each taking half the columns)
// mbarriers: full/empty per stage (TMA <-> MMA), tmem_full/tmem_empty per
// accumulator (MMA <-> epilogue).  tcgen05.commit arrives on the mbarriers.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "ctx.cuh"
#include "epi.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"

namespace dasmc_b200 {

struct TcState {
  int n0 = 0, n1 = 0, C = 0;
  int64_t n_pad = 0;     // X^T row stride (floats)
  int64_t mcap = 0;      // row stride of the transposed activation buffers
  bool split = false;    // split-tf32 (3 MMAs)
  bool f16 = false;      // fp16 operands, kind::f16 (DASMC_PREC_F16): same 10-bit mantissa as tf32
  int esz = 4;           // forward operand (Xhi, W1hi) element bytes (2 when f16)
  bool f16x2 = false;    // f16x2 (DASMC_PREC_F16X2): f16 mode with W1 as fp16 hi + lo (two forward MMAs)
  bool hstore = false;   // tf32h (DASMC_PREC_TF32H): tf32 forward, weight-gradient GEMM operands in fp16
  int besz = 4;          // weight-gradient operand (Xt, a1T, d1T, d2T) element bytes
  int cluster = 1;       // fused-forward cluster shape (ClusterShape CL; 0 = single CTAs); DASMC_TC_CLUSTER
  float* Xt = nullptr;   // [(n0+1) x n_pad], row n0 = 1
  int64_t kx = 0;        // row stride of Xhi / W1hi: [x, 1] padded to 16 bytes (bias folded into K)
  float* Xhi = nullptr;  // [n x kx] [X, 1, 0..] rounded to tf32 (rna): the MMA truncates raw fp32
  float* Xlo = nullptr;  // [n x kx]   (split)
  float* Xtlo = nullptr; // [(n0+1) x n_pad] (split; ones row lo = 0)
  float* W1hi = nullptr; // [J x n1 x kx] [W1, b1, 0..] rounded to tf32
  float* W1lo = nullptr;
  float* a1T = nullptr;  // [J x (n1+1) x mcap], row n1 = 1
  float* d1T = nullptr;  // [J x n1 x mcap]
  float* d2T = nullptr;  // [J x C x mcap]
  float* a1Tlo = nullptr;
  float* d1Tlo = nullptr;
  float* d2Tlo = nullptr;
  int num_sms = 148;
  // deep MLP (>= 2 hidden layers; tc_eval_deep): per layer l (1-based)
  bool deep = false;
  int L = 0;
  int sz[kMaxLayers + 1] = {};
  int64_t kxl[kMaxLayers + 1] = {};   // a_l row-major stride with the ones column (kxl[0] = kx)
  int64_t ldd[kMaxLayers + 1] = {};   // delta_l row-major stride (round4(n_l))
  float* Whi[kMaxLayers + 1] = {};    // [J][n_l][kx_{l-1}] = [W_l, b_l, 0..] tf32, l < L
  float* WThi[kMaxLayers + 1] = {};   // [J][n_{l-1}][ldd_l] = W_l^T tf32, 2 <= l < L
  float* aRow[kMaxLayers + 1] = {};   // a_l [J][mcap][kx_l] (column n_l = 1), l < L
  float* aT[kMaxLayers + 1] = {};     // a_l^T row-blocked [J][nblk][n_l + 1][128] (row n_l = 1), l < L
  float* dRow[kMaxLayers + 1] = {};   // delta_l [J][mcap][ldd_l], 2 <= l < L (tf32 hi)
  float* dRowLo[kMaxLayers + 1] = {}; // its split-tf32 low part (the backward-delta GEMMs run 3xtf32)
  float* WTlo[kMaxLayers + 1] = {};   // low part of WThi
  float* dTl[kMaxLayers + 1] = {};    // delta_l^T row-blocked [J][nblk][n_l][128], l <= L
};

namespace {

constexpr int BM = 128;  // UMMA_M
constexpr int BK = 32;   // fp32 per 128-byte swizzle row
#ifndef DASMC_EPI_WARPS
#define DASMC_EPI_WARPS 12
#endif
constexpr int kEpiWarps = DASMC_EPI_WARPS;  // 3 warps per TMEM lane group (a multiple of 4)
constexpr int kParts = kEpiWarps / 4;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;  // TMA warp + MMA warp + epilogue warps
constexpr int kTmemCols = 512;  // 2 accumulators x 256 columns
constexpr int kEpiKindFwd = 0, kEpiKindDw = 1, kEpiKindHidden = 2, kEpiKindBackDelta = 3;
// Deep path: run the backward-delta GEMMs in split-tf32.  Off: measured on B200 it does not
// move the deep gradients' error (dominated by ReLU activation-pattern flips under the
// tf32 forward, not by the backward operands) and costs 19 % of the C5 step.
constexpr bool kDeepSplitBack = false;
// A operand addressing: 2-D shared by every particle; 4-D row-blocked per particle
// (weight-gradient GEMMs, K = window rows); 3-D row-major per particle
constexpr int kAShared = 0, kABlocked = 1, kARowMajor = 2;

// forward epilogue: accumulator columns per TMEM load (8 or 16) and how many columns
// ahead of their FFMA2s the W2^T rows are loaded from shared memory
#ifndef DASMC_CW
#define DASMC_CW 0  // 0: per precision mode (see the forward epilogue)
#endif
#ifndef DASMC_W2_AHEAD
#define DASMC_W2_AHEAD 0
#endif
// Pass 2 of the fused-forward epilogue, delta1 = (delta2 W2) . act'(z1), as one small tensor-core MMA
// per tile (ReLU nets, CTA pairs, fp16-stored operands): delta2 (fp16, [128][16]) and W2 (fp16,
// [nmma / 2][16] per CTA) are written to shared memory in the unswizzled K-major core-matrix layout,
// one epilogue thread of the pair leader issues a cta_group::2 kind::f16 MMA (M = 256, N = nmma, K = 16)
// that overwrites the tile's z1 accumulator once every warp has read it, and the CUDA cores only mask
// (ReLU' bits kept in registers from pass 1), round and store.
// Opt-in (-DDASMC_L2TC=1): parity-green, but measured on B200 it does not move the default mode
// (C2 forward, interleaved A/B: f16x2 26.4 vs 26.3 ms, tf32h 25.8 vs 26.9 ms, f16 20.7 vs 19.8 ms per launch):
// the forward is bound by its operand loads and activation stores, not by the epilogue's instruction count.
#ifndef DASMC_L2TC
#define DASMC_L2TC 0
#endif
// Epilogue activation stores (a1^T, delta1^T: streamed once, re-read by the
// weight-gradient GEMMs after ~25 GB of other traffic)
#ifndef DASMC_ST_POLICY
#define DASMC_ST_POLICY 0
#endif
__device__ __forceinline__ void st_act(float* p, float v, uint64_t pol) {
#if DASMC_ST_POLICY == 1
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
#elif DASMC_ST_POLICY == 2
  asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
#elif DASMC_ST_POLICY == 3
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
  (void)pol;
  *p = v;
#endif
}
// ---------------------------------------------------------------- parameters
struct TileParams {
  int rtiles;  // row tiles (of BM rows) per particle
  int J;
  int rg;      // row tiles per scheduling group
  int nkb;     // k blocks of BK
  int klast;   // MMA k-steps (a quarter k block each) the last k block needs (0 = all 4): K tails skip the
               // all-zero quarters
  int nmma;    // MMA N (multiple of 16, <= 256)
  int brows;   // TMA box rows of B (valid rows)
  int stages;
  uint32_t stage_bytes_tx;
  int bbox;    // clusters with QB = 2: B rows per multicast piece (pieces at 0 and half - bbox)
  int hint_a, hint_b;  // L2 policies of the A / B loads (pairs): 0 normal, 1 evict_last, 2 evict_first
  int prefetch;        // pairs: L2-prefetch the next unit's A / B boxes
  int ntn;             // N tiles per (row tile, particle) (single-CTA kernels; 0 = 1): B rows nt * nmma ...
};

struct FwdParams {
  const float* theta;  // theta_in
  int64_t Dp, woff2, boff2;
  int n1, C, act;
  const int32_t* y;
  int64_t M, P;
  int Jn;  // particles (clusters with QA = 2 may carry one padding particle)
  float beta_rows;
  int need_grad;
  int64_t ldm;  // row stride (floats) of the transposed buffers
  float *a1T, *d1T, *d2T, *a1Tlo, *d1Tlo, *d2Tlo;
  double* ll_part;
  int ll_slots;
  int dbg;  // DASMC_DEBUG_EPI: 1 = skip global stores, 2 = skip pass 2, 3 = skip the whole epilogue math,
            // 4 = stores into one L2-resident block, 5 = skip the a1^T stores, 6 = skip the delta1^T stores
  // EPI kHidden (a_l = act(acc)) / kBackDelta (delta_{l-1} = acc . act'(a_{l-1})) of the
  // deep-MLP path: outputs in row-major [J][Mcap][out_ld] (optional) and row-blocked
  // transposed [J][nblk = ldm][out_rows][128] form, tf32-rounded (GEMM operands)
  float* out_row;
  int64_t out_ld, Mcap;
  float* out_T;
  int out_rows, n_valid;
  const float* mask_src;  // kBackDelta: a_{l-1} row-major [J][Mcap][mask_ld]
  int64_t mask_ld;
  float* out_row_lo;      // split-tf32 low part of out_row (kBackDelta chains), optional
};

struct DwParams {
  EpiParams e;
  int64_t Dp, woff, boff;
  int in;        // layer fan-in (row index `in` is the bias row)
  int n_out;     // valid output columns
};

__device__ __forceinline__ void tile_coords(const TileParams& tp, int t, int& rt, int& j) {
  const int gsz = tp.rg * tp.J;
  const int g = t / gsz;
  const int loc = t - g * gsz;
  const int size_g = min(tp.rg, tp.rtiles - g * tp.rg);
  j = loc / size_g;
  rt = g * tp.rg + loc % size_g;
}

// ---------------------------------------------------------------- the kernel
// CL = 0: one CTA per tile.  CL >= 1 (forward only): clusters of CTA pairs.  A
// pair (CTA ranks 2p, 2p+1 on one TPC) computes two 128-row tiles of one
// particle: CTA r loads rows of A for its tile and half the B rows, the leader
// (r = 0) issues cta_group::2 MMAs (M = 256) reading both CTAs' shared memory,
// and each CTA's epilogue drains its own TMEM.  Per CTA this halves the B
// (per-particle W1) bytes streamed from L2.  The cluster holds QA x QB pairs:
// QA = 2 puts two particles on the same rows (the A tile -- X -- is multicast to
// both pairs, each CTA loading half of it), QB = 2 puts two row pairs on the
// same particle (B -- W1 -- multicast).  Multicast cuts L2 -> SM traffic, the
// forward GEMM's bound.
template <int CL>
struct ClusterShape {
  static constexpr bool kPair = CL > 0;
  static constexpr int QA = (CL == 2 || CL == 4) ? 2 : 1;
  static constexpr int QB = (CL == 3 || CL == 4) ? 2 : 1;
  static constexpr int kSize = kPair ? 2 * QA * QB : 1;
};

template <int EPI, bool SPLIT, int AM, int CP, int ACT, int CL, int PREC>
__global__ void __launch_bounds__(kThreads, 1)
    tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
              const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo, TileParams tp,
              const __grid_constant__ FwdParams fp, DwParams dp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms; keep the pointer derived
  // from smem_raw so the compiler emits shared-memory (LDS/STS) accesses.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using CS_ = ClusterShape<CL>;
  constexpr bool PAIR = CS_::kPair;
  constexpr int QA = CS_::QA, QB = CS_::QB, CSZ = CS_::kSize;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const uint32_t prank = crank & 1u;              // rank inside the pair
  const int pr = (int)(crank >> 1);               // pair inside the cluster
  const int qa = pr / QB, qb = pr % QB;           // particle slot, row slot
  const int unit0 = (int)blockIdx.x / CSZ;
  const int ustride = (int)gridDim.x / CSZ;
  const uint32_t b_rows = PAIR ? (uint32_t)tp.nmma / 2 : (uint32_t)tp.nmma;  // B rows held by this CTA
  // PREC 0: tf32 MMA, fp32 containers; 1: fp16 MMA and stores; 2 (forward only): tf32 MMA
  // with the epilogue's GEMM-operand stores (a1^T, delta1^T, delta2^T) in fp16 (tf32h);
  // 3 (forward only, f16x2): fp16 MMAs with B split into fp16 hi + lo parts, two MMAs per
  // k-step (A . B_hi + A . B_lo), fp16 stores
  constexpr int KP = PREC == 2 ? 0 : PREC == 3 ? 1 : PREC;  // MMA kind / operand loads
  constexpr int SP = PREC >= 2 ? 1 : PREC;                  // epilogue store type
  constexpr bool BSPL = SPLIT || PREC == 3;                 // B carries a lo part
  constexpr int BKE = KP == 1 ? 64 : 32;    // K elements per 128-byte swizzle row (= per k-block)
  using TS = OpT<SP>;
  const uint32_t a_bytes = BM * 128;
  const uint32_t b_bytes = b_rows * 128;
  const uint32_t sub = SPLIT ? 2 : 1, subb = BSPL ? 2 : 1;
  const uint32_t stage_bytes = sub * a_bytes + subb * b_bytes;
  uint8_t* stages = smem;
  uint64_t* bars = (uint64_t*)(smem + (size_t)tp.stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + tp.stages;
  uint64_t* tfull = bars + 2 * tp.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 2);
  float* epi_smem = (float*)(tmem_holder + 4);  // 16-byte aligned
  // tensor-core pass 2 (see DASMC_L2TC): two mbarriers and the two small operand tiles behind the
  // CUDA-core epilogue's buffers
  constexpr bool L2TC = DASMC_L2TC && EPI == kEpiKindFwd && CL == 1 && ACT == DASMC_RELU && !SPLIT && PREC >= 1;
  uint64_t* l2bar = nullptr;  // [0] ready (every epilogue warp of the pair, on the leader), [1] done (MMA commit)
  uint8_t* d2tile = nullptr;  // delta2 [128][16] fp16
  uint8_t* w2h = nullptr;     // W2 rows o = prank * b_rows ..: [b_rows][16] fp16
  if constexpr (L2TC) {
    constexpr int CS0 = (CP + 3) & ~3;
    uint8_t* q = reinterpret_cast<uint8_t*>(epi_smem + 2 * ((size_t)fp.n1 * CS0 + CS0) + (size_t)kParts * 128 * CP) +
                 8 * sizeof(double);
    l2bar = reinterpret_cast<uint64_t*>(q);
    uint8_t* t0 = q + 16;
    t0 += (128u - (smem_u32(t0) & 127u)) & 127u;
    d2tile = t0;
    w2h = t0 + 4096;
  }

  auto A_of = [&](int s, int lo) { return stages + (size_t)s * stage_bytes + (lo ? a_bytes : 0); };
  auto B_of = [&](int s, int lo) { return stages + (size_t)s * stage_bytes + sub * a_bytes + (lo ? b_bytes : 0); };

  // zero the stage ring once: rows of B beyond the TMA box stay zero
  for (uint32_t i = threadIdx.x; i < tp.stages * stage_bytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(stages)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    if (SPLIT) prefetch_map(&mapAlo);
    if (BSPL) prefetch_map(&mapBlo);
    for (int s = 0; s < tp.stages; ++s) {
      mbar_init(&full[s], 1);
      // a stage is free once every pair of the cluster consumed it (multicast writes
      // land in other pairs' stages): one commit per pair leader
      mbar_init(&empty[s], PAIR ? QA * QB : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      // one arrival per epilogue warp (of both CTAs of a pair: the leader's barrier)
      mbar_init(&tempty[b], (PAIR ? 2 : 1) * kEpiWarps);
    }
    if constexpr (L2TC) {
      mbar_init(&l2bar[0], 2 * kEpiWarps);
      mbar_init(&l2bar[1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / complete_tx
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int ntn = tp.ntn > 0 ? tp.ntn : 1;
  const int ntiles = tp.rtiles * tp.J * ntn;  // scheduling units (row-tile pairs x particles when PAIR)

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      // multicast groups: CTAs sharing this CTA's A tile (same row slot and pair rank,
      // every particle slot) and its B rows (same particle slot and pair rank)
      uint16_t amask = 0, bmask = 0;
      for (int a = 0; a < QA; ++a) amask |= (uint16_t)(1u << (prank + 2 * (qb + QB * a)));
      for (int b = 0; b < QB; ++b) bmask |= (uint16_t)(1u << (prank + 2 * (b + QB * qa)));
      const int arows = BM / QA;                                   // A rows this CTA issues
      const int boff = qb == 0 ? 0 : (int)b_rows - tp.bbox;        // B piece this CTA issues
      const uint64_t pol_a = l2_policy(tp.hint_a), pol_b = l2_policy(tp.hint_b);
      for (int t = unit0; t < ntiles; t += ustride) {
        int ru, j;
        const int nt = t % ntn;
        tile_coords(tp, t / ntn, ru, j);
        const int rt = PAIR ? 2 * (QB * ru + qb) + (int)prank : ru;
        const int bn0 = nt * tp.nmma;  // first B row of this N tile
        if (PAIR) j = QA * j + qa;
        // warm L2 with the next unit's operands while this unit streams (pairs, no multicast)
        int pf_rt = -1, pf_j = 0;
        if (PAIR && QA == 1 && QB == 1 && tp.prefetch && t + ustride < ntiles) {
          int pru;
          tile_coords(tp, t + ustride, pru, pf_j);
          pf_rt = 2 * pru + (int)prank;
        }
        for (int kb = 0; kb < tp.nkb; ++kb) {
          if (pf_rt >= 0) {
            tma_prefetch_2d(&mapA, kb * BKE, pf_rt * BM);
            tma_prefetch_3d(&mapB, kb * BKE, (int)(prank * b_rows), pf_j);
          }
          mbar_wait(&empty[s], ph ^ 1);
          const int k0 = kb * BKE;
          if (PAIR) {
            // the pair's bytes complete on its leader's full barrier (expect_tx covers the pair)
            const uint32_t fb = mapa_shared(smem_u32(&full[s]), crank & ~1u);
            if (prank == 0) mbar_expect_tx(&full[s], tp.stage_bytes_tx);
            if (QA == 1) {
              tma2_2d(A_of(s, 0), &mapA, fb, k0, rt * BM, pol_a);
              if (SPLIT) tma2_2d(A_of(s, 1), &mapAlo, fb, k0, rt * BM, pol_a);
            } else {
              const int r0 = qa * arows;
              tma2_2d_mc(A_of(s, 0) + r0 * 128, &mapA, fb, k0, rt * BM + r0, amask, pol_a);
              if (SPLIT) tma2_2d_mc(A_of(s, 1) + r0 * 128, &mapAlo, fb, k0, rt * BM + r0, amask, pol_a);
            }
            const int brow = (int)(prank * b_rows);
            if (QB == 1) {
              tma2_3d(B_of(s, 0), &mapB, fb, k0, brow, j, pol_b);
              if (BSPL) tma2_3d(B_of(s, 1), &mapBlo, fb, k0, brow, j, pol_b);
            } else {
              tma2_3d_mc(B_of(s, 0) + boff * 128, &mapB, fb, k0, brow + boff, j, bmask, pol_b);
              if (BSPL) tma2_3d_mc(B_of(s, 1) + boff * 128, &mapBlo, fb, k0, brow + boff, j, bmask, pol_b);
            }
          } else {
            mbar_expect_tx(&full[s], tp.stage_bytes_tx);
            // row-blocked operands [J][blk][rows][128] (K = window rows): 4-D coordinates
            // (k within block, row, block, particle); a 32-wide k block never straddles blocks
            if (AM == kABlocked) {
              tma_4d(A_of(s, 0), &mapA, &full[s], k0 & 127, rt * BM, k0 >> 7, j);
              if (SPLIT) tma_4d(A_of(s, 1), &mapAlo, &full[s], k0 & 127, rt * BM, k0 >> 7, j);
            } else if (AM == kARowMajor) {
              tma_3d(A_of(s, 0), &mapA, &full[s], k0, rt * BM, j);
              if (SPLIT) tma_3d(A_of(s, 1), &mapAlo, &full[s], k0, rt * BM, j);
            } else {
              tma_2d(A_of(s, 0), &mapA, &full[s], k0, rt * BM);
              if (SPLIT) tma_2d(A_of(s, 1), &mapAlo, &full[s], k0, rt * BM);
            }
            if (EPI == kEpiKindDw) {
              tma_4d(B_of(s, 0), &mapB, &full[s], k0 & 127, bn0, k0 >> 7, j);
              if (BSPL) tma_4d(B_of(s, 1), &mapBlo, &full[s], k0 & 127, bn0, k0 >> 7, j);
            } else {
              tma_3d(B_of(s, 0), &mapB, &full[s], k0, bn0, j);
              if (BSPL) tma_3d(B_of(s, 1), &mapBlo, &full[s], k0, bn0, j);
            }
          }
          if (++s == tp.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if (PAIR) {
        // drain: every stage this CTA filled has been released by the leader's MMAs
        // (their multicast commits land in this CTA's shared memory before it exits)
        for (int i = 0; i < tp.stages; ++i) {
          mbar_wait(&empty[s], ph ^ 1);
          if (++s == tp.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread; the leader's when PAIR) =====================
    if (lane == 0 && prank == 0) {
      const uint32_t idesc = KP == 1 ? idesc_f16(tp.nmma, PAIR ? 2 * BM : BM) : idesc_tf32(tp.nmma, PAIR ? 2 * BM : BM);
      const uint16_t all_mask = (uint16_t)((1u << CSZ) - 1u);
      const uint16_t pair_mask = (uint16_t)(3u << (2 * pr));
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int t = unit0; t < ntiles; t += ustride) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * 256);
        // one k block: NKS MMA k-steps (32 bytes of K each) per operand part, straight-line code (the
        // issuing thread's instruction count is on the critical path of the MMA-bound GEMMs)
        auto kblock = [&](int kb, auto nks_c) {
          constexpr int NKS = decltype(nks_c)::value;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = smem_desc(A_of(s, 0)), bd = smem_desc(B_of(s, 0));
          const uint64_t adl = smem_desc(A_of(s, 1)), bdl = smem_desc(B_of(s, 1));
#pragma unroll
          for (int k = 0; k < NKS; ++k) {
            const uint64_t off = (uint64_t)(k * 32) >> 4;  // 32 bytes per K=8 step inside the swizzle row
            if (PAIR) {
              tc_mma2<KP>(d, ad + off, bd + off, idesc, (kb | k) != 0);
              if (BSPL) tc_mma2<KP>(d, ad + off, bdl + off, idesc, 1);
              if (SPLIT) tc_mma2<KP>(d, adl + off, bd + off, idesc, 1);
            } else {
              tc_mma<KP>(d, ad + off, bd + off, idesc, (kb | k) != 0);
              if (BSPL) tc_mma<KP>(d, ad + off, bdl + off, idesc, 1);
              if (SPLIT) tc_mma<KP>(d, adl + off, bd + off, idesc, 1);
            }
          }
          if (PAIR)
            tc_commit2(&empty[s], all_mask);
          else
            tc_commit(&empty[s]);
          if (++s == tp.stages) {
            s = 0;
            ph ^= 1;
          }
        };
        for (int kb = 0; kb < tp.nkb - 1; ++kb) kblock(kb, std::integral_constant<int, 4>{});
        // the last k block: a K tail skips its all-zero quarters (tp.klast k-steps)
        switch (tp.klast) {
          case 1: kblock(tp.nkb - 1, std::integral_constant<int, 1>{}); break;
          case 2: kblock(tp.nkb - 1, std::integral_constant<int, 2>{}); break;
          case 3: kblock(tp.nkb - 1, std::integral_constant<int, 3>{}); break;
          default: kblock(tp.nkb - 1, std::integral_constant<int, 4>{}); break;
        }
        if (PAIR)
          tc_commit2(&tfull[acc], pair_mask);
        else
          tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else {
    // ===================== epilogue warps 2..13 =====================
    // kParts warps share each TMEM lane group (warp % 4); `part` selects a
    // contiguous range of 16-column accumulator chunks.
    const int et = threadIdx.x - 64;
    const int lg = warp & 3;
    const int part = (warp - 2) >> 2;
    const int row_in_tile = lg * 32 + lane;
    auto chunk_range = [&](int nch, int& lo, int& hi) {
      lo = nch * part / kParts;
      hi = nch * (part + 1) / kParts;
    };
    // the accumulator buffer is drained: one arrival per warp on the MMA issuer's barrier
    const uint32_t tempty_addr0 = PAIR ? mapa_shared(smem_u32(&tempty[0]), crank & ~1u) : smem_u32(&tempty[0]);
    auto release_acc = [&](int a) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_addr0 + (uint32_t)(a * 8));
    };
    int acc = 0;
    uint32_t aph = 0;
    const uint64_t st_pol = l2_policy(2);  // activation stores: evict first (DASMC_ST_POLICY 3)
    int it = 0;                     // forward tiles processed (W2^T buffer parity)
    uint32_t l2ph = 0;              // parity of the pass-2 MMA barriers (L2TC)
    double* ll_pending = nullptr;   // forward: ll slot of the previous tile, written by thread 0
    double* red = (double*)(epi_smem + 2 * ((size_t)fp.n1 * ((CP + 3) & ~3) + ((CP + 3) & ~3)) +
                            (size_t)kParts * 128 * CP);  // [4][2] lane-group partials
    auto flush_ll = [&]() {
      ll_pending[0] = red[0] + red[2] + red[4] + red[6];
      ll_pending[1] = red[1] + red[3] + red[5] + red[7];
      ll_pending = nullptr;
    };
    for (int t = unit0; t < ntiles; t += ustride) {
      int rt, j;
      const int nt = t % ntn;
      tile_coords(tp, t / ntn, rt, j);
      if (PAIR) {
        rt = 2 * (QB * rt + qb) + (int)prank;
        j = QA * j + qa;
      }
      if (EPI == kEpiKindFwd && PAIR && ((int64_t)rt * BM >= fp.M || j >= fp.Jn)) {
        // a tile of the cluster wholly past the window (or a padding particle): nothing to store
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        if constexpr (L2TC) {
          if (fp.need_grad && (fp.dbg == 0 || fp.dbg >= 5)) {
            // the peer's pass-2 MMA still reads this CTA's half of W2 and writes this CTA's accumulator
            const float* thp = fp.theta + (int64_t)j * fp.Dp;
            for (int i = et; i < (int)b_rows * 16; i += kEpiThreads) {
              const int r = i >> 4, k = i & 15, o = (int)(prank * b_rows) + r;
              const float x = (o < fp.n1 && k < fp.C) ? thp[fp.woff2 + (int64_t)k * fp.n1 + o] : 0.f;
              *reinterpret_cast<__half*>(w2h + (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2) =
                  __float2half_rn(x);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&l2bar[0]), crank & ~1u));
            mbar_wait(&l2bar[1], l2ph);
            tc_fence_after();
            l2ph ^= 1;
          }
        }
        release_acc(acc);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
        continue;
      }
      if (EPI == kEpiKindFwd) {
        // Fused forward epilogue.  The accumulator row already holds the full
        // pre-activation z1 = [x, 1] . [W1, b1]^T (bias folded into the GEMM as
        // an extra K column), and rows past the window are TMA zero-fill, so
        // act(z1) = 0 there and every row-blocked store below is unconditional.
        const int n1 = fp.n1, C = fp.C;
        // store / math ablations (DASMC_DEBUG_EPI, profiling only).  Kept as a runtime value:
        // folding it to a constant measured 5 % slower (B200, in-process A/B, tools/tune_fwd.py):
        // ptxas schedules the predicated store groups of the column loops better
        const int dbg = fp.dbg;
        constexpr int CS = (CP + 3) & ~3;       // W2^T row stride (float4 aligned)
        // W2^T / b2 double-buffered by tile parity: the buffer written here was last read
        // two tiles ago, before every thread passed the previous tile's barriers
        float* W2T = epi_smem + (size_t)(it & 1) * ((size_t)n1 * CS + CS);  // [n1][CS]  W2 transposed, zero-padded
        float* b2s = W2T + (size_t)n1 * CS;     // [CS]
        float* z2x = epi_smem + 2 * ((size_t)n1 * CS + CS);  // [kParts][128][CP] partial layer-2 logits
        ++it;
        const float* th = fp.theta + (int64_t)j * fp.Dp;
        // the row's label: load in flight across the accumulator wait and pass 1
        const int y_row = ((int64_t)rt * BM + row_in_tile < fp.M) ? __ldg(fp.y + (int64_t)rt * BM + row_in_tile) : 0;
        // per-particle layer-2 parameters: all global loads issued before any
        // shared-memory store (one L2 round trip per tile, not one per element)
        constexpr int kPer = (256 * CS + kEpiThreads - 1) / kEpiThreads;
        float wv[kPer];
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
          const int i = et + r * kEpiThreads;
          const int o = i / CS, c = i - o * CS;
          wv[r] = (i < n1 * CS && c < C) ? th[fp.woff2 + (int64_t)c * n1 + o] : 0.f;
        }
        const float b2v = et < C ? th[fp.boff2 + et] : 0.f;
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
          const int i = et + r * kEpiThreads;
          if (i < n1 * CS) W2T[i] = wv[r];
        }
        if (et < CS) b2s[et] = b2v;
        named_bar(1, kEpiThreads);
        if (et == 0 && ll_pending) flush_ll();
        const bool l2go = L2TC && fp.need_grad && (dbg == 0 || dbg >= 5);  // pass 2 on the tensor core
        if constexpr (L2TC) {
          if (l2go) {
            // this CTA's half of W2 as the MMA's B operand: rows o, k = class (zero past C)
            for (int i = et; i < (int)b_rows * 8; i += kEpiThreads) {
              const int r = i >> 3, kp = i & 7, o = (int)(prank * b_rows) + r;
              const float x0 = (o < n1 && 2 * kp < C) ? W2T[o * CS + 2 * kp] : 0.f;
              const float x1 = (o < n1 && 2 * kp + 1 < C) ? W2T[o * CS + 2 * kp + 1] : 0.f;
              *reinterpret_cast<__half2*>(w2h + (r >> 3) * 256 + (kp >> 2) * 128 + (r & 7) * 16 + (kp & 3) * 4) =
                  __floats2half2_rn(x0, x1);
            }
          }
        }
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int64_t m = (int64_t)rt * BM + row_in_tile;
        const bool valid = m < fp.M;
        const bool st_rows = fp.need_grad && dbg != 1 && dbg != 5;  // 5: no a1^T stores
        int c_lo, c_hi;
        // 16-column TMEM loads, except in the fp16 mode whose (epilogue-bound) forward
        // runs 9 % faster with 8 (B200 in-process A/B; tf32 / tf32h 4 % slower with 8)
        constexpr int CW = DASMC_CW > 0 ? DASMC_CW : (PREC == 1 ? 8 : 16);
        // whole CW-column chunks per part (C2: 64 / 64 / 72 of 200 columns).  An even 67 / 67 / 66 split was
        // measured slower on B200 (26.1 vs 25.6 ms per C2 launch: unaligned TMEM chunks and 2-3 column tails)
        chunk_range((n1 + CW - 1) / CW, c_lo, c_hi);
        constexpr int col_lo = 0;
        const int col_hi = n1;
        if (dbg == 3) c_hi = c_lo;
        // transposed buffers are row-blocked [J][nblk][rows][128]: a tile's rows are one
        // contiguous region; consecutive rows of a block are 128 floats apart
        const int64_t nblk = fp.ldm;
        constexpr int64_t kRow = 128;
        // class pairs in packed fp32x2 registers: the layer-2 FMAs issue as FFMA2 (two IEEE
        // fp32 FMAs per instruction, the same per-class accumulation order)
        static_assert(CP % 2 == 0, "class padding must be even");
        float2 z2p[CP / 2];
#pragma unroll
        for (int c = 0; c < CP / 2; ++c) z2p[c] = make_float2(0.f, 0.f);
        uint32_t mk0 = 0, mk1 = 0, mk2 = 0;  // L2TC: ReLU' bits of this thread's columns (a 96-bit stack)
        // DASMC_DEBUG_EPI=4 (profiling only): every tile stores into one L2-resident block
        const int64_t sblk = dbg == 4 ? (int64_t)(blockIdx.x & 1) : (int64_t)j * nblk + rt;
        TS* a1T = reinterpret_cast<TS*>(fp.a1T) + sblk * (n1 + 1) * kRow + row_in_tile;
        float* a1Tlo = SPLIT ? fp.a1Tlo + ((int64_t)j * nblk + rt) * (n1 + 1) * kRow + row_in_tile : nullptr;
        // row o of W2^T (CP classes) from shared memory as class pairs: float4 loads (+ one float2)
        auto w2row2 = [&](int o, float2* w) {
          const float* p = W2T + o * CS;
#pragma unroll
          for (int u = 0; u < CP / 4; ++u) {
            const float4 x = *reinterpret_cast<const float4*>(p + 4 * u);
            w[2 * u] = make_float2(x.x, x.y);
            w[2 * u + 1] = make_float2(x.z, x.w);
          }
          if (CP % 4) w[CP / 2 - 1] = *reinterpret_cast<const float2*>(p + 4 * (CP / 4));
        };
        // the CW columns of a chunk, each W2^T row loaded DASMC_W2_AHEAD columns before its
        // FFMA2s (0: loaded at the column, scheduled by ptxas)
        auto w2_pipeline = [&](int o0, int nq, auto&& body) {
          if constexpr (DASMC_W2_AHEAD == 0) {
#pragma unroll
            for (int q = 0; q < CW; ++q)
              if (q < nq) {
                float2 w[CP / 2];
                w2row2(o0 + q, w);
                body(q, w);
              }
          } else {  // one column ahead: the next row is in flight while this one is used
            float2 wc[CP / 2], wn[CP / 2];
            w2row2(o0, wc);
#pragma unroll
            for (int q = 0; q < CW; ++q) {
              if (q + 1 < nq) w2row2(o0 + q + 1, wn);
              if (q < nq) body(q, wc);
#pragma unroll
              for (int c = 0; c < CP / 2; ++c) wc[c] = wn[c];
            }
          }
        };
        auto act = [](float z) { return ACT == DASMC_RELU ? fmaxf(z, 0.f) : tanhf(z); };
        // pass 1: a1 = act(z1); partial z2 = W2 a1 over this warp's columns
        auto chunk1 = [&](auto store, int ch, const float* v) {
          const int o0 = col_lo + ch * CW;
          const int nq = min(CW, col_hi - o0);  // warp-uniform
          TS* pa = a1T + (int64_t)o0 * kRow;
          float* pal = SPLIT ? a1Tlo + (int64_t)o0 * kRow : nullptr;
          uint32_t mcur = 0;  // L2TC: ReLU' bits of this chunk's columns
          auto one = [&](int q, const float2* w) {
            const float a = act(v[q]);
            const float2 aa = make_float2(a, a);
            if constexpr (L2TC) mcur |= a > 0.f ? (1u << q) : 0u;
#pragma unroll
            for (int c = 0; c < CP / 2; ++c) z2p[c] = __ffma2_rn(aa, w[c], z2p[c]);
            if (decltype(store)::value) {
              const TS hi = to_op<SP>(a);
              pa[q * kRow] = hi;
              if (SPLIT) st_act(pal + q * kRow, a - (float)hi, st_pol);
            }
          };
          if (nq == CW)
            w2_pipeline(o0, CW, one);
          else  // tail chunk: still unrolled so v[] stays in registers
            w2_pipeline(o0, nq, one);
          if constexpr (L2TC) {  // push the chunk's bits (pass 2 pops them in reverse chunk order)
            mk2 = (mk2 << CW) | (mk1 >> (32 - CW));
            mk1 = (mk1 << CW) | (mk0 >> (32 - CW));
            mk0 = (mk0 << CW) | mcur;
          }
        };
        // TMEM loads double-buffered: chunk ch+1 is in flight while ch is processed
        auto run_chunks = [&](auto body) {
          float va[CW] = {}, vb[CW] = {};
          int ch = c_lo;
          const uint32_t tcol = taddr + (uint32_t)col_lo;
          if (ch < c_hi) tmem_ldw_async<CW>(tcol + ch * CW, va);
          tmem_waitw<CW>(va);
          while (ch < c_hi) {
            if (ch + 1 < c_hi) tmem_ldw_async<CW>(tcol + (ch + 1) * CW, vb);
            body(ch, va);
            tmem_waitw<CW>(vb);
            if (++ch >= c_hi) break;
            if (ch + 1 < c_hi) tmem_ldw_async<CW>(tcol + (ch + 1) * CW, va);
            body(ch, vb);
            tmem_waitw<CW>(va);
            ++ch;
          }
        };
        if (st_rows)
          run_chunks([&](int ch, const float* v) { chunk1(std::true_type{}, ch, v); });
        else
          run_chunks([&](int ch, const float* v) { chunk1(std::false_type{}, ch, v); });
        // combine the column parts in a fixed order
        float* zx = z2x + ((size_t)part * 128 + row_in_tile) * CP;
#pragma unroll
        for (int c = 0; c < CP / 2; ++c) reinterpret_cast<float2*>(zx)[c] = z2p[c];
        named_bar(1, kEpiThreads);
        // every part: softmax of the row (fp32 exponentials and normaliser) and delta2,
        // computed redundantly per part (no second barrier); part 0 alone forms the row's
        // log-likelihood with an fp64 log-normaliser (network.hpp:183-193) and stores delta2^T
        double ll = 0.0;
        float z2[CP];
        float d2[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) d2[c] = 0.f;
        {
#pragma unroll
          for (int c = 0; c < CP; ++c) {
            float s = z2x[(size_t)row_in_tile * CP + c];
#pragma unroll
            for (int p = 1; p < kParts; ++p) s += z2x[((size_t)p * 128 + row_in_tile) * CP + c];
            z2[c] = s + b2s[c];
          }
          TS* d2T = reinterpret_cast<TS*>(fp.d2T) + ((int64_t)j * nblk + rt) * C * kRow + row_in_tile;
          float* d2Tlo = SPLIT ? fp.d2Tlo + ((int64_t)j * nblk + rt) * C * kRow + row_in_tile : nullptr;
          if (valid) {
            const int yi = y_row;
            float mx = z2[0];
#pragma unroll
            for (int c = 1; c < CP; ++c)
              if (c < C) mx = fmaxf(mx, z2[c]);
            float e[CP];
            float den = 0.f;
            float zy = 0.f;
#pragma unroll
            for (int c = 0; c < CP; ++c) {
#ifdef DASMC_V_FASTEXP
              e[c] = c < C ? __expf(z2[c] - mx) : 0.f;
#else
              e[c] = c < C ? expf(z2[c] - mx) : 0.f;
#endif
              den += e[c];
              if (c == yi) zy = z2[c];
            }
            if (part == 0) {
              // the row's log-likelihood (network.hpp:183-193): fp64 log-normaliser, one part only
              double den64 = 0.0;
#pragma unroll
              for (int c = 0; c < CP; ++c) den64 += (double)e[c];
              ll = (double)zy - ((double)mx + log(den64));
            }
            if (fp.need_grad) {
              const float wrow = m < fp.P ? 1.f : fp.beta_rows;
              const float rden = 1.f / den;  // every part: the same fp32 normaliser for delta2
#pragma unroll
              for (int c = 0; c < CP; ++c)
                if (c < C) {
                  d2[c] = wrow * ((c == yi ? 1.f : 0.f) - e[c] * rden);
                  if (part == 0) {
                    const TS hi = to_op<SP>(d2[c]);
                    d2T[c * kRow] = hi;
                    if (SPLIT) d2Tlo[c * kRow] = d2[c] - (float)hi;
                  }
                }
            }
          } else if (fp.need_grad && part == 0) {  // rows past the window: zeros in the row-blocked delta2^T
            for (int c = 0; c < C; ++c) {
              d2T[c * kRow] = to_op<SP>(0.f);
              if (SPLIT) d2Tlo[c * kRow] = 0.f;
            }
          }
        }
        if (l2go) {
          if constexpr (L2TC) {
            // pass 2 on the tensor core: delta1 = (delta2 W2) . relu'(z1)  (network.hpp:209-215)
            if (part == 0) {  // this row's delta2 as the MMA's A operand (zeros past the window / past C)
              __half2 h[8];
#pragma unroll
              for (int c = 0; c < 8; ++c)
                h[c] = __floats2half2_rn(2 * c < CP ? d2[2 * c] : 0.f, 2 * c + 1 < CP ? d2[2 * c + 1] : 0.f);
              uint4* dst = reinterpret_cast<uint4*>(d2tile + (row_in_tile >> 3) * 256 + (row_in_tile & 7) * 16);
              dst[0] = *reinterpret_cast<const uint4*>(&h[0]);
              dst[8] = *reinterpret_cast<const uint4*>(&h[4]);  // + 128 bytes: k = 8..15
            }
            // operand tiles (generic-proxy writes) -> the MMA's async-proxy reads; this warp's z1 loads are
            // complete (tcgen05.wait::ld in run_chunks) before the MMA overwrites the accumulator
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&l2bar[0]), crank & ~1u));
            if (et == 0 && prank == 0) {
              mbar_wait(&l2bar[0], l2ph);
              tc_fence_after();
              // unswizzled K-major core matrices (8 rows x 16 bytes): LBO (k) = 128 B, SBO (rows) = 256 B
              auto desc0 = [](const void* p) {
                return (uint64_t)((smem_u32(p) >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
                       ((uint64_t)(256 >> 4) << 32) | (1ULL << 46);
              };
              tc_mma2<1>(tmem_base + (uint32_t)(acc * 256), desc0(d2tile), desc0(w2h), idesc_f16(tp.nmma, 2 * BM), 0);
              tc_commit2(&l2bar[1], (uint16_t)(3u << (2 * pr)));
            }
            mbar_wait(&l2bar[1], l2ph);
            tc_fence_after();
            l2ph ^= 1;
            TS* d1T = reinterpret_cast<TS*>(fp.d1T) + sblk * n1 * kRow + row_in_tile;
            // chunks in reverse order (the bit stack), TMEM loads double-buffered
            auto chunk2t = [&](int ch, const float* v) {
              const int o0 = col_lo + ch * CW;
              const int nq = min(CW, col_hi - o0);  // warp-uniform
              TS* pd = d1T + (int64_t)o0 * kRow;
              const uint32_t mcur = mk0;
              mk0 = (mk0 >> CW) | (mk1 << (32 - CW));
              mk1 = (mk1 >> CW) | (mk2 << (32 - CW));
              mk2 >>= CW;
#pragma unroll
              for (int q = 0; q < CW; ++q)
                if (q < nq) {
                  const TS hi = to_op<SP>((mcur >> q) & 1u ? v[q] : 0.f);
                  if (dbg != 6) pd[q * kRow] = hi;
                }
            };
            {
              float va[CW] = {}, vb[CW] = {};
              const uint32_t tcol = taddr + (uint32_t)col_lo;
              int ch = c_hi - 1;
              if (ch >= c_lo) tmem_ldw_async<CW>(tcol + ch * CW, va);
              tmem_waitw<CW>(va);
              while (ch >= c_lo) {
                if (ch - 1 >= c_lo) tmem_ldw_async<CW>(tcol + (ch - 1) * CW, vb);
                chunk2t(ch, va);
                tmem_waitw<CW>(vb);
                if (--ch < c_lo) break;
                if (ch - 1 >= c_lo) tmem_ldw_async<CW>(tcol + (ch - 1) * CW, va);
                chunk2t(ch, vb);
                tmem_waitw<CW>(va);
                --ch;
              }
            }
          }
        } else if (fp.need_grad && (dbg == 0 || dbg >= 5)) {  // 6: no delta1^T stores
          // pass 2: delta1 = (W2^T delta2) . act'(z1)  (network.hpp:209-215); zero past the window
          TS* d1T = reinterpret_cast<TS*>(fp.d1T) + sblk * n1 * kRow + row_in_tile;
          float* d1Tlo = SPLIT ? fp.d1Tlo + ((int64_t)j * nblk + rt) * n1 * kRow + row_in_tile : nullptr;
          float2 d2p[CP / 2];
#pragma unroll
          for (int c = 0; c < CP / 2; ++c) d2p[c] = make_float2(d2[2 * c], d2[2 * c + 1]);
          auto chunk2 = [&](int ch, const float* v) {
            const int o0 = col_lo + ch * CW;
            const int nq = min(CW, col_hi - o0);  // warp-uniform
            TS* pd = d1T + (int64_t)o0 * kRow;
            float* pdl = SPLIT ? d1Tlo + (int64_t)o0 * kRow : nullptr;
            auto one = [&](int q, const float2* w) {
#ifndef DASMC_V_ACC2
              float2 acc = make_float2(0.f, 0.f);  // even / odd classes: two chains in one FFMA2
#pragma unroll
              for (int c = 0; c < CP / 2; ++c) acc = __ffma2_rn(d2p[c], w[c], acc);
              const float dz = acc.x + acc.y;
#else
              // class pairs alternate between two packed accumulators (four fp32 chains)
              float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
              for (int c = 0; c < CP / 2; c += 2) {
                acc0 = __ffma2_rn(d2p[c], w[c], acc0);
                if (c + 1 < CP / 2) acc1 = __ffma2_rn(d2p[c + 1], w[c + 1], acc1);
              }
              const float dz = (acc0.x + acc1.x) + (acc0.y + acc1.y);
#endif
              float d1;
              if (ACT == DASMC_RELU) {
                d1 = v[q] > 0.f ? dz : 0.f;
              } else {
                const float a = tanhf(v[q]);
                d1 = dz * (1.f - a * a);
              }
              const TS hi = to_op<SP>(d1);
              if (dbg != 6) pd[q * kRow] = hi;
              if (SPLIT) st_act(pdl + q * kRow, d1 - (float)hi, st_pol);
            };
            if (nq == CW)
              w2_pipeline(o0, CW, one);
            else
              w2_pipeline(o0, nq, one);
          };
          run_chunks(chunk2);
        }
        release_acc(acc);
        // per-tile prefix / block log-likelihood partials (deterministic order): the
        // four lane groups' sums go to red[]; thread 0 writes the tile's slot after the
        // next tile's staging barrier (or after the loop), which orders it behind them
        double pre = (valid && m < fp.P) ? ll : 0.0, blk = (valid && m >= fp.P) ? ll : 0.0;
        if (part == 0) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            pre += __shfl_xor_sync(0xffffffffu, pre, o);
            blk += __shfl_xor_sync(0xffffffffu, blk, o);
          }
          if (lane == 0) {
            red[lg * 2] = pre;
            red[lg * 2 + 1] = blk;
          }
        }
        ll_pending = fp.ll_part + ((int64_t)j * fp.ll_slots + rt) * 2;
      } else if (EPI == kEpiKindHidden || EPI == kEpiKindBackDelta) {
        // deep-MLP epilogues (network.hpp:159-178, 208-216): row m of the tile, columns
        // o = nt * nmma + ...; rows past the window hold act(0) = 0 / masked zeros
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int64_t m = (int64_t)rt * BM + row_in_tile;
        const bool valid = m < fp.M;
        const int64_t nblk = fp.ldm;
        const int nb0 = nt * tp.nmma;
        int c_lo, c_hi;
        chunk_range(tp.nmma >> 4, c_lo, c_hi);
        for (int ch = c_lo; ch < c_hi; ++ch) {
          const int o0 = nb0 + ch * 16;
          const int nq = min(16, fp.n_valid - o0);  // warp-uniform
          float v[16];
          tmem_ld16(taddr + ch * 16, v);
          if (nq <= 0) continue;
          if (EPI == kEpiKindHidden) {
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = tf32_hi(ACT == DASMC_RELU ? fmaxf(v[q], 0.f) : tanhf(v[q]));
          } else {
            float a[16];
            const float* src = fp.mask_src + ((int64_t)j * fp.Mcap + m) * fp.mask_ld + o0;
            if (valid && nq == 16 && (fp.mask_ld & 3) == 0) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float4 x = reinterpret_cast<const float4*>(src)[u];
                a[4 * u] = x.x;
                a[4 * u + 1] = x.y;
                a[4 * u + 2] = x.z;
                a[4 * u + 3] = x.w;
              }
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q) a[q] = (valid && q < nq) ? src[q] : 0.f;
            }
            float lo[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float dv = valid ? v[q] * (ACT == DASMC_RELU ? (a[q] > 0.f ? 1.f : 0.f) : 1.f - a[q] * a[q]) : 0.f;
              v[q] = tf32_hi(dv);
              lo[q] = dv - v[q];
            }
            if (fp.out_row_lo && valid) {
              float* dst = fp.out_row_lo + ((int64_t)j * fp.Mcap + m) * fp.out_ld + o0;
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (q < nq) dst[q] = lo[q];
            }
          }
          if (fp.out_row && valid) {
            float* dst = fp.out_row + ((int64_t)j * fp.Mcap + m) * fp.out_ld + o0;
            if (nq == 16 && (fp.out_ld & 3) == 0) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                reinterpret_cast<float4*>(dst)[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (q < nq) dst[q] = v[q];
            }
          }
          if (fp.out_T) {
            float* dT = fp.out_T + (((int64_t)j * nblk + rt) * fp.out_rows + o0) * 128 + row_in_tile;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q < nq) dT[(int64_t)q * 128] = v[q];
          }
        }
        release_acc(acc);
      } else {
        // weight-gradient tile: row i of A (input index, `in` = bias row), columns o
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int i = rt * BM + row_in_tile;
        const bool valid = i <= dp.in;
        const int64_t base = (int64_t)j * dp.Dp;
        const int nb0 = nt * tp.nmma;
        int c_lo, c_hi;
        chunk_range(min(tp.nmma, dp.n_out - nb0 + 15) >> 4, c_lo, c_hi);
        for (int ch = c_lo; ch < c_hi; ++ch) {
          const int o0 = nb0 + ch * 16;
          float v[16];
          tmem_ld16(taddr + ch * 16, v);
          if (valid) {
            int64_t idx[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              idx[q] = base + (i < dp.in ? dp.woff + (int64_t)(o0 + q) * dp.in + i : dp.boff + o0 + q);
            leapfrog_update_n<16>(dp.e, j, idx, v, min(16, dp.n_out - o0));
          }
        }
        release_acc(acc);
      }
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if (EPI == kEpiKindFwd) {
      named_bar(1, kEpiThreads);  // the last tile's lane-group partials are in red[]
      if (et == 0 && ll_pending) flush_ll();
    }
  }
  __syncwarp();
  if (PAIR) {
    cluster_sync_all();  // no remote arrive / commit targets this CTA any more
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
    }
  } else {
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
    }
  }
}

// ---------------------------------------------------------------- helper kernels
// X^T with a ones row (and tf32 hi/lo splits): Xt[i][m] = X[m][i], Xt[n0][m] = 1.
// Also the forward operand Xhi[m] = [X[m], 1, 0 ...] (row stride kx) and its lo part.
// PT / PH: operand precision (0 tf32, 1 fp16) of Xt (weight-gradient A) and Xhi (forward A).
template <int PT, int PH>
__global__ void transpose_x_kernel(const float* __restrict__ X, int64_t n, int n0, int64_t n_pad, int64_t kx,
                                   OpT<PT>* Xt, float* Xtlo, OpT<PH>* Xhi, float* Xlo, int split) {
  __shared__ float tile[32][33];
  const int64_t m0 = (int64_t)blockIdx.x * 32;
  const int i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t m = m0 + r;
    const int i = i0 + threadIdx.x;
    float v = 0.f;
    if (m < n && i < n0) v = X[m * n0 + i];
    if (m < n && i == n0) v = 1.f;
    if (m < n && i < kx) Xhi[m * kx + i] = to_op<PH>(v);
    if (split && m < n && i < kx) Xlo[m * kx + i] = v - tf32_hi(v);
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r;
    const int64_t m = m0 + threadIdx.x;
    if (i <= n0 && m < n_pad) {
      const float v = m < n ? tile[threadIdx.x][r] : 0.f;
      const OpT<PT> hi = to_op<PT>(v);
      Xt[(int64_t)i * n_pad + m] = hi;
      if (split) Xtlo[(int64_t)i * n_pad + m] = v - (float)hi;
    }
  }
}

// W1hi[j][o] = [W1[o], b1[o], 0 ...] (row stride kx) rounded to tf32, + lo part.
// One thread per 4 consecutive outputs (grid-stride): 16-B loads of the W row when
// the internal layout is 16-B aligned, 16-B (tf32) / 8-B (fp16) stores.
template <int PREC>
__global__ void __launch_bounds__(256) split_w1_kernel(const float* __restrict__ theta, int64_t Dp, int64_t woff,
                                                       int64_t boff, int n0, int64_t kx, int64_t cnt, int64_t J,
                                                       OpT<PREC>* __restrict__ hi, OpT<PREC>* __restrict__ lo) {
  const int64_t n1 = cnt / kx;
  const int kq = (int)(kx >> 2);
  const int64_t total = J * n1 * kq;
  const bool vec = ((woff | (int64_t)n0 | Dp) & 3) == 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / kq;
    const int i0 = 4 * (int)(e - row * kq);
    const int64_t j = row / n1, o = row - j * n1;
    const float* th = theta + j * Dp;
    const float* src = th + woff + o * n0;
    float v[4];
    if (vec && i0 + 4 <= n0) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(src + i0));
      v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        v[u] = i < n0 ? src[i] : (i == n0 ? th[boff + o] : 0.f);
      }
    }
    OpT<PREC> h[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) h[u] = to_op<PREC>(v[u]);
    const int64_t off = row * kx + i0;
    if constexpr (PREC == 1) {
      __half2 p0 = __halves2half2(h[0], h[1]), p1 = __halves2half2(h[2], h[3]);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&p0);
      w.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(hi + off) = w;
      if (lo) {  // f16x2: fp16 residual, hi + lo carries ~22 significand bits
        __half2 q0 = __floats2half2_rn(v[0] - __half2float(h[0]), v[1] - __half2float(h[1]));
        __half2 q1 = __floats2half2_rn(v[2] - __half2float(h[2]), v[3] - __half2float(h[3]));
        w.x = *reinterpret_cast<uint32_t*>(&q0);
        w.y = *reinterpret_cast<uint32_t*>(&q1);
        *reinterpret_cast<uint2*>(lo + off) = w;
      }
    } else {
      *reinterpret_cast<float4*>(hi + off) = make_float4(h[0], h[1], h[2], h[3]);
      if (lo) *reinterpret_cast<float4*>(lo + off) = make_float4(v[0] - h[0], v[1] - h[1], v[2] - h[2], v[3] - h[3]);
    }
  }
}

// WT[j][i][o] = tf32(W_l[o][i]) (internal W row-major [out][in] at woff), row stride ldt.
__global__ void transpose_w_kernel(const float* __restrict__ theta, int64_t Dp, int64_t woff, int in, int out,
                                   int64_t ldt, int64_t J, float* __restrict__ WT, float* __restrict__ WTlo) {
  __shared__ float tile[32][33];
  const int64_t j = blockIdx.z;
  const int o0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const float* W = theta + j * Dp + woff;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int o = o0 + r, i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (o < out && i < in) ? W[(int64_t)o * in + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, o = o0 + threadIdx.x;
    if (i < in && o < out) {
      const float v = tile[threadIdx.x][r], h = tf32_hi(v);
      WT[(j * in + i) * ldt + o] = h;
      if (WTlo) WTlo[(j * in + i) * ldt + o] = v - h;
    }
  }
}

// Column `col` of a row-major [J*rows][ld] buffer set to v (the bias-folding ones column).
__global__ void fill_col_kernel(float* buf, int64_t nrows, int64_t ld, int64_t col, float v) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nrows; g += (int64_t)gridDim.x * blockDim.x)
    buf[g * ld + col] = v;
}

// Output layer of the deep MLP on CUDA cores (network.hpp:174-193, 208-216): one thread
// per window row of a 128-row tile of particle j.  z_L = W_L a_{L-1} + b_L from the
// row-blocked a_{L-1}^T (coalesced), fp64 log-softmax / ll partials (the fused
// forward's slot layout), delta_L = w_m (onehot - softmax), delta_{L-1} = (W_L^T delta_L)
// . act'(a_{L-1}); writes delta_L^T, delta_{L-1}^T (row-blocked) and delta_{L-1} row-major.
template <int CP>
__global__ void __launch_bounds__(128) head_kernel(
    const float* __restrict__ aT, int n_in, int C, int64_t nblk, const float* __restrict__ theta, int64_t Dp,
    int64_t woff, int64_t boff, int act, const int32_t* __restrict__ y, int64_t M, int64_t P, float beta_rows,
    int need_grad, double* __restrict__ ll_part, int ll_slots, float* __restrict__ dLT, float* __restrict__ dT,
    float* __restrict__ dRow, float* __restrict__ dRowLo, int64_t ldd, int64_t Mcap) {
  extern __shared__ float hs[];
  __shared__ float stg[4][32][9];    // per-warp staging of the row-major delta stores
  float* Ws = hs;                    // [n_in][CP] = W_L transposed
  float* bs = Ws + (size_t)n_in * CP;  // [CP]
  __shared__ double red[8];
  const int rt = blockIdx.x, r = threadIdx.x;
  const int64_t j = blockIdx.y;
  const float* th = theta + j * Dp;
  for (int i = r; i < n_in * CP; i += 128) {
    const int o = i / CP, c = i - o * CP;
    Ws[i] = c < C ? th[woff + (int64_t)c * n_in + o] : 0.f;
  }
  if (r < CP) bs[r] = r < C ? th[boff + r] : 0.f;
  __syncthreads();
  const int64_t m = (int64_t)rt * 128 + r;
  const bool valid = m < M;
  const float* a = aT + (j * nblk + rt) * (int64_t)(n_in + 1) * 128 + r;
  float z[CP];
#pragma unroll
  for (int c = 0; c < CP; ++c) z[c] = bs[c];
  const float4* W4 = reinterpret_cast<const float4*>(Ws);
  auto accum = [&](float v, int o) {
#pragma unroll
    for (int u = 0; u < CP / 4; ++u) {
      const float4 w = W4[o * (CP / 4) + u];
      z[4 * u] = fmaf(v, w.x, z[4 * u]);
      z[4 * u + 1] = fmaf(v, w.y, z[4 * u + 1]);
      z[4 * u + 2] = fmaf(v, w.z, z[4 * u + 2]);
      z[4 * u + 3] = fmaf(v, w.w, z[4 * u + 3]);
    }
  };
  int o = 0;
  for (; o + 8 <= n_in; o += 8) {  // 8 loads in flight per thread
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = a[(int64_t)(o + q) * 128];
#pragma unroll
    for (int q = 0; q < 8; ++q) accum(v[q], o + q);
  }
  for (; o < n_in; ++o) accum(a[(int64_t)o * 128], o);
  double ll = 0.0;
  float d[CP];
#pragma unroll
  for (int c = 0; c < CP; ++c) d[c] = 0.f;
  if (valid) {
    const int yi = y[m];
    float mx = z[0];
#pragma unroll
    for (int c = 1; c < CP; ++c)
      if (c < C) mx = fmaxf(mx, z[c]);
    float e[CP];
    double den = 0.0;
    float zy = 0.f;
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      e[c] = c < C ? expf(z[c] - mx) : 0.f;
      den += (double)e[c];
      if (c == yi) zy = z[c];
    }
    ll = (double)zy - ((double)mx + log(den));
    const float wrow = m < P ? 1.f : beta_rows;
    const float rden = (float)(1.0 / den);
#pragma unroll
    for (int c = 0; c < CP; ++c)
      if (c < C) d[c] = wrow * ((c == yi ? 1.f : 0.f) - e[c] * rden);
  }
  if (need_grad) {
    float* lt = dLT + (j * nblk + rt) * (int64_t)C * 128 + r;
    for (int c = 0; c < C; ++c) lt[(int64_t)c * 128] = tf32_hi(d[c]);
    float* dt = dT + (j * nblk + rt) * (int64_t)n_in * 128 + r;
    const bool dr = dRow != nullptr;
    float* drl = dRowLo ? dRowLo + (j * Mcap + m) * ldd : nullptr;
    for (int o0 = 0; o0 < n_in; o0 += 8) {
      float av[8], g[8];
      const int nq = min(8, n_in - o0);
#pragma unroll
      for (int q = 0; q < 8; ++q) av[q] = q < nq ? a[(int64_t)(o0 + q) * 128] : 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float sacc = 0.f;
#pragma unroll
        for (int u = 0; u < CP / 4; ++u) {
          const float4 w = W4[(o0 + q < n_in ? o0 + q : 0) * (CP / 4) + u];
          sacc = fmaf(d[4 * u], w.x, sacc);
          sacc = fmaf(d[4 * u + 1], w.y, sacc);
          sacc = fmaf(d[4 * u + 2], w.z, sacc);
          sacc = fmaf(d[4 * u + 3], w.w, sacc);
        }
        g[q] = sacc * (act == DASMC_RELU ? (av[q] > 0.f ? 1.f : 0.f) : 1.f - av[q] * av[q]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nq) {
          const float h = tf32_hi(g[q]);
          dt[(int64_t)(o0 + q) * 128] = h;
          stg[r >> 5][r & 31][q] = h;
          if (drl) drl[o0 + q] = g[q] - h;
        }
      if (dr) {
        // row-major delta (the next backward-delta GEMM's A operand): the warp's 32 rows x 8
        // columns go out through shared memory as 32-byte row segments, 4 rows per store
        // instruction, instead of one 4-byte store per row and column
        __syncwarp();
        const int lane = r & 31;
        float* drw = dRow + (j * Mcap + (int64_t)rt * 128 + (r & ~31)) * ldd + o0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = i * 4 + (lane >> 3), col = lane & 7;
          if (col < nq) drw[(int64_t)row * ldd + col] = stg[r >> 5][row][col];
        }
        __syncwarp();
      }
    }
  }
  // per-tile prefix / block partials in a fixed order
  double pre = (valid && m < P) ? ll : 0.0, blk = (valid && m >= P) ? ll : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pre += __shfl_xor_sync(0xffffffffu, pre, o);
    blk += __shfl_xor_sync(0xffffffffu, blk, o);
  }
  if ((r & 31) == 0) {
    red[(r >> 5) * 2] = pre;
    red[(r >> 5) * 2 + 1] = blk;
  }
  __syncthreads();
  if (r == 0) {
    double* o = ll_part + (j * ll_slots + rt) * 2;
    o[0] = red[0] + red[2] + red[4] + red[6];
    o[1] = red[1] + red[3] + red[5] + red[7];
  }
}

// Row `row` of a row-blocked [J][nblk][rows][128] buffer set to v (a1^T's ones row -> db2).
template <typename T>
__global__ void fill_ones_row_kernel(T* buf, int64_t J, int64_t rows, int64_t row, int64_t mcap, float v) {
  const int64_t total = J * mcap;
  const int64_t nblk = mcap / 128;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jb = g / 128, r = g - jb * 128;  // jb = j * nblk + block
    buf[(jb * rows + row) * 128 + r] = (T)v;
    (void)nblk;
  }
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Driver entry point through the runtime (no -lcuda link dependency).
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw CudaError{"cuTensorMapEncodeTiled unavailable"};
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// rank-2/3 fp32 tensor, innermost dim first; strides in bytes for dims >= 1.
// esz: operand element size (4 = fp32 / tf32 containers, 2 = fp16); boxes are one
// 128-byte swizzle row (128 / esz elements) wide.
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, int esz = 4) {
  CUtensorMap m;
  uint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 (cuuint32_t)rank, const_cast<void*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

// Row-blocked transposed buffer [J][nblk_alloc][rows][128] as a 4-D operand:
// dims {128, rows, nblk_used, J}, box {32 (k), box_rows, 1, 1}.
CUtensorMap map_blk(const void* base, uint64_t rows, uint64_t nblk_used, uint64_t nblk_alloc, uint64_t J,
                    uint32_t box_rows, int esz = 4) {
  const uint64_t dims[4] = {128, rows, nblk_used, J};
  const uint64_t strides[3] = {128 * (uint64_t)esz, rows * 128 * esz, nblk_alloc * rows * 128 * esz};
  const uint32_t box[4] = {128u / esz, box_rows, 1, 1};
  CUtensorMap m;
  uint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                 const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled (4d) failed (" + std::to_string((int)r) + ")"};
  return m;
}


CUtensorMap map2d(const void* base, uint64_t inner, uint64_t rows, uint64_t ld, uint32_t box_rows, int esz = 4) {
  const uint64_t dims[2] = {inner, rows};
  const uint64_t strides[1] = {ld * esz};
  const uint32_t box[2] = {128u / esz, box_rows};
  return make_map(base, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, esz);
}

CUtensorMap map3d(const void* base, uint64_t inner, uint64_t rows, uint64_t ld, uint64_t J, uint64_t pstride,
                  uint32_t box_rows, int esz = 4) {
  const uint64_t dims[3] = {inner, rows, J};
  const uint64_t strides[2] = {ld * esz, pstride * esz};
  const uint32_t box[3] = {128u / esz, box_rows, 1};
  return make_map(base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, esz);
}

int round16(int v) { return (v + 15) / 16 * 16; }

// CL >= 1: tp.rtiles counts row groups (2 QB tiles) and tp.J particle groups (QA
// particles); B's TMA box is tp.nmma / 2 rows per CTA (tp.bbox rows per piece
// when QB = 2; tp.brows is ignored) and the grid is launched as clusters.
template <int EPI, bool SPLIT, int AM, int CP = 4, int ACT = 0, int CL = 0, int PREC = 0>
void launch_tc(Ctx& c, const CUtensorMap& A, const CUtensorMap& Alo, const CUtensorMap& B, const CUtensorMap& Blo,
               TileParams tp, const FwdParams& fp, const DwParams& dp, size_t epi_smem_bytes) {
  using CS_ = ClusterShape<CL>;
  const size_t sub = SPLIT ? 2 : 1, subb = (SPLIT || PREC == 3) ? 2 : 1;
  const size_t b_rows = CS_::kPair ? (size_t)tp.nmma / 2 : (size_t)tp.nmma;
  const size_t stage_bytes = sub * (size_t)BM * BK * 4 + subb * b_rows * BK * 4;
  const size_t fixed = 1024 + 64 * 8 + 64 + epi_smem_bytes;
  const size_t budget = 227 * 1024;
  int stages = (int)std::min<size_t>(8, (budget - fixed) / stage_bytes);
  if (stages < 1) throw CudaError{"tensor-core tile does not fit in shared memory"};
  tp.stages = stages;
  if (CS_::kPair) {
    // bytes landing in the pair per stage (two overlapping B pieces when QB = 2)
    const size_t b_land = CS_::QB == 2 ? 2 * (size_t)tp.bbox : b_rows;
    tp.stage_bytes_tx = (uint32_t)(2 * (sub * (size_t)BM * BK * 4 + subb * b_land * BK * 4));
  } else {
    tp.stage_bytes_tx = (uint32_t)(sub * (size_t)BM * BK * 4 + subb * (size_t)tp.brows * BK * 4);
  }
  const size_t smem = 1024 + stages * stage_bytes + (2 * stages + 4) * 8 + 16 + epi_smem_bytes + 64;
  auto kern = tc_kernel<EPI, SPLIT, AM, CP, ACT, CL, PREC>;
  static bool attr_set_dev[kMaxDevices] = {};
  static int max_clusters_dev[kMaxDevices] = {};
  const int dv = current_device();
  bool& attr_set = attr_set_dev[dv];
  int& max_clusters = max_clusters_dev[dv];
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  if (CS_::kPair) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS_::kSize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (!attr_set) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget));
    if (CS_::kPair) {
      cfg.gridDim = dim3((unsigned)(CS_::kSize * (c.tc->num_sms / CS_::kSize)));
      CK(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
      if (max_clusters < 1) throw CudaError{"tensor-core cluster does not fit on the device"};
    }
    attr_set = true;
  }
  const int ntiles = tp.rtiles * tp.J * std::max(tp.ntn, 1);
  if (CS_::kPair) {
    const int nclusters = std::max(1, std::min(ntiles, max_clusters));
    cfg.gridDim = dim3((unsigned)(CS_::kSize * nclusters));
    CK(cudaLaunchKernelEx(&cfg, kern, A, SPLIT ? Alo : A, B, (SPLIT || PREC == 3) ? Blo : B, tp, fp, dp));
  } else {
    const int grid = std::max(1, std::min(ntiles, c.tc->num_sms));
    kern<<<grid, kThreads, smem, c.stream>>>(A, SPLIT ? Alo : A, B, (SPLIT || PREC == 3) ? Blo : B, tp, fp, dp);
  }
  LAUNCHED();
}

}  // namespace

bool tc_layer1_eligible(const Ctx& c) {
  const NetDev& n = c.net;
  if (n.nconv != 0) return false;
  if (n.L == 2) return n.sizes[0] % 4 == 0 && n.sizes[0] >= 4 && n.sizes[1] <= 256 && n.sizes[2] <= 16;
  if (c.precision == DASMC_PREC_F16 || c.precision == DASMC_PREC_F16X2) return false;  // one-hidden-layer only
  // deep path (tc_eval_deep): tf32, <= 16 classes, output layer weights in shared memory
  if ((c.precision != DASMC_PREC_TF32 && c.precision != DASMC_PREC_TF32H) || n.sizes[n.L] > 16 || (int64_t)n.sizes[n.L - 1] * 16 > 16384) return false;
  for (int l = 0; l < n.L; ++l)
    if (n.sizes[l] > 8192) return false;
  return true;
}

// Xt (weight-gradient A operand, fp16 in the f16 / tf32h modes) and Xhi (forward A
// operand, fp16 only in the f16 mode) from the first n rows of X.
static void transpose_x(Ctx& c, int64_t n) {
  TcState* s = c.tc;
  dim3 grid((unsigned)((s->n_pad + 31) / 32), (unsigned)((s->n0 + 1 + 31) / 32));
  if (s->f16)
    transpose_x_kernel<1, 1><<<grid, dim3(32, 8), 0, c.stream>>>(
        c.X, n, s->n0, s->n_pad, s->kx, reinterpret_cast<__half*>(s->Xt), nullptr, reinterpret_cast<__half*>(s->Xhi),
        nullptr, 0);
  else if (s->hstore)
    transpose_x_kernel<1, 0><<<grid, dim3(32, 8), 0, c.stream>>>(c.X, n, s->n0, s->n_pad, s->kx,
                                                                 reinterpret_cast<__half*>(s->Xt), nullptr, s->Xhi,
                                                                 nullptr, 0);
  else
    transpose_x_kernel<0, 0><<<grid, dim3(32, 8), 0, c.stream>>>(c.X, n, s->n0, s->n_pad, s->kx, s->Xt, s->Xtlo,
                                                                 s->Xhi, s->Xlo, s->split ? 1 : 0);
  LAUNCHED();
}

void tc_init(Ctx& c) {
  auto* s = new TcState();
  c.tc = s;
  s->deep = c.net.L >= 3;
  s->L = c.net.L;
  for (int l = 0; l <= c.net.L; ++l) s->sz[l] = c.net.sizes[l];
  s->n0 = c.net.sizes[0];
  s->n1 = c.net.sizes[1];
  s->C = c.net.sizes[2];
  s->split = c.precision == DASMC_PREC_3XTF32;
  s->f16x2 = c.precision == DASMC_PREC_F16X2;
  s->f16 = c.precision == DASMC_PREC_F16 || s->f16x2;
  s->hstore = c.precision == DASMC_PREC_TF32H && !s->deep;  // deep MLPs: plain tf32
  s->esz = s->f16 ? 2 : 4;
  s->besz = (s->f16 || s->hstore) ? 2 : 4;
  if (const char* e = std::getenv("DASMC_TC_CLUSTER")) s->cluster = std::max(0, std::min(4, std::atoi(e)));
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, dev));
  s->n_pad = (c.n + 31) / 32 * 32;
  const size_t xt = (size_t)(s->n0 + 1) * s->n_pad;
  CK(cudaMalloc(&s->Xt, (size_t)s->besz * xt));
  // [x, 1] padded so the row stride is a multiple of 16 bytes
  s->kx = s->f16 ? (s->n0 + 1 + 7) / 8 * 8 : (s->n0 + 1 + 3) / 4 * 4;
  const size_t w = (size_t)c.Jmax * s->n1 * s->kx;
  CK(cudaMalloc(&s->Xhi, (size_t)s->esz * c.n * s->kx));
  if (s->deep) {
    s->kxl[0] = s->kx;
    for (int l = 1; l <= s->L; ++l) {
      s->kxl[l] = (s->sz[l] + 1 + 3) / 4 * 4;
      s->ldd[l] = (s->sz[l] + 3) / 4 * 4;
    }
    for (int l = 1; l < s->L; ++l)
      CK(cudaMalloc(&s->Whi[l], sizeof(float) * (size_t)c.Jmax * s->sz[l] * s->kxl[l - 1]));
    for (int l = 2; l < s->L; ++l) {
      CK(cudaMalloc(&s->WThi[l], sizeof(float) * (size_t)c.Jmax * s->sz[l - 1] * s->ldd[l]));
      if (kDeepSplitBack) CK(cudaMalloc(&s->WTlo[l], sizeof(float) * (size_t)c.Jmax * s->sz[l - 1] * s->ldd[l]));
    }
    s->W1hi = s->Whi[1];
  } else {
    CK(cudaMalloc(&s->W1hi, (size_t)s->esz * w));
  }
  if (s->f16x2) CK(cudaMalloc(&s->W1lo, (size_t)s->esz * w));
  if (s->split) {
    CK(cudaMalloc(&s->Xtlo, sizeof(float) * xt));
    CK(cudaMalloc(&s->Xlo, sizeof(float) * (size_t)c.n * s->kx));
    CK(cudaMalloc(&s->W1lo, sizeof(float) * w));
  }
  transpose_x(c, c.n);
  CK(cudaStreamSynchronize(c.stream));
}

void tc_free(Ctx& c) {
  TcState* s = c.tc;
  if (!s) return;
  if (s->deep) s->W1hi = nullptr;  // owned through Whi[1]
  float* p[] = {s->Xt, s->Xhi, s->Xlo, s->Xtlo, s->W1hi, s->W1lo, s->a1T, s->d1T, s->d2T, s->a1Tlo, s->d1Tlo, s->d2Tlo};
  for (float* q : p)
    if (q) cudaFree(q);
  for (int l = 0; l <= kMaxLayers; ++l) {
    float* d[] = {s->Whi[l], s->WThi[l], s->WTlo[l], s->aRow[l], s->aT[l], s->dRow[l], s->dRowLo[l], s->dTl[l]};
    for (float* q : d)
      if (q) cudaFree(q);
  }
  delete s;
  c.tc = nullptr;
}

void tc_refresh_data(Ctx& c) {
  transpose_x(c, c.n_active);
}

void tc_ensure_rows(Ctx& c, int64_t Mcap) {
  TcState* s = c.tc;
  if (Mcap <= s->mcap) return;
  if (s->deep) {
    const size_t J = (size_t)c.Jmax;
    for (int l = 0; l <= kMaxLayers; ++l) {
      float** d[] = {&s->aRow[l], &s->aT[l], &s->dRow[l], &s->dRowLo[l], &s->dTl[l]};
      for (float** q : d)
        if (*q) {
          CK(cudaFree(*q));
          *q = nullptr;
        }
    }
    for (int l = 1; l <= s->L; ++l) {
      if (l < s->L) {
        CK(cudaMalloc(&s->aRow[l], sizeof(float) * J * Mcap * s->kxl[l]));
        CK(cudaMalloc(&s->aT[l], sizeof(float) * J * (s->sz[l] + 1) * Mcap));
        fill_col_kernel<<<(unsigned)std::min<int64_t>((J * Mcap + 255) / 256, 148 * 16), 256, 0, c.stream>>>(
            s->aRow[l], (int64_t)(J * Mcap), s->kxl[l], s->sz[l], 1.f);
        LAUNCHED();
        fill_ones_row_kernel<<<(unsigned)std::min<int64_t>((J * Mcap + 255) / 256, 148 * 16), 256, 0, c.stream>>>(
            s->aT[l], (int64_t)J, s->sz[l] + 1, s->sz[l], Mcap, 1.f);
        LAUNCHED();
      }
      if (l >= 2 && l < s->L) {
        CK(cudaMalloc(&s->dRow[l], sizeof(float) * J * Mcap * s->ldd[l]));
        if (kDeepSplitBack) CK(cudaMalloc(&s->dRowLo[l], sizeof(float) * J * Mcap * s->ldd[l]));
      }
      CK(cudaMalloc(&s->dTl[l], sizeof(float) * J * s->sz[l] * Mcap));
    }
    s->mcap = Mcap;
    return;
  }
  float** bufs[] = {&s->a1T, &s->d1T, &s->d2T, &s->a1Tlo, &s->d1Tlo, &s->d2Tlo};
  for (float** b : bufs)
    if (*b) {
      CK(cudaFree(*b));
      *b = nullptr;
    }
  const size_t J = (size_t)c.Jmax;
  CK(cudaMalloc(&s->a1T, (size_t)s->besz * J * (s->n1 + 1) * Mcap));
  CK(cudaMalloc(&s->d1T, (size_t)s->besz * J * s->n1 * Mcap));
  CK(cudaMalloc(&s->d2T, (size_t)s->besz * J * s->C * Mcap));
  if (s->split) {
    CK(cudaMalloc(&s->a1Tlo, sizeof(float) * J * (s->n1 + 1) * Mcap));
    CK(cudaMalloc(&s->d1Tlo, sizeof(float) * J * s->n1 * Mcap));
    CK(cudaMalloc(&s->d2Tlo, sizeof(float) * J * s->C * Mcap));
  }
  s->mcap = Mcap;
  const int g = (int)std::min<int64_t>((J * Mcap + 255) / 256, 148 * 16);
  if (s->besz == 2)
    fill_ones_row_kernel<<<g, 256, 0, c.stream>>>(reinterpret_cast<__half*>(s->a1T), (int64_t)J, s->n1 + 1, s->n1,
                                                  Mcap, 1.f);
  else
    fill_ones_row_kernel<<<g, 256, 0, c.stream>>>(s->a1T, (int64_t)J, s->n1 + 1, s->n1, Mcap, 1.f);
  LAUNCHED();
  if (s->split) {
    fill_ones_row_kernel<<<g, 256, 0, c.stream>>>(s->a1Tlo, (int64_t)J, s->n1 + 1, s->n1, Mcap, 0.f);
    LAUNCHED();
  }
}

// Deep MLP (>= 2 hidden layers) on the tensor cores: per hidden layer a GEMM with the
// bias folded into K and the activation epilogue (a_l row-major + transposed); the output
// layer + softmax + delta_L + delta_{L-1} on CUDA cores (head_kernel); backward deltas as
// GEMMs against W_l^T with the act' epilogue; weight gradients as K = window-row GEMMs
// with the fused leapfrog (the fused one-hidden-layer path's Dw kernel, N-tiled).
void tc_eval_deep(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
                  const EpiParams* epi) {
  TcState* s = c.tc;
  const NetDev& net = c.net;
  const int L = s->L;
  const int64_t Mcap = s->mcap, nba = Mcap / 128, nbu = (M + 127) / 128;
  const int rtiles = (int)((M + BM - 1) / BM);
  auto ntiles_n = [](int n) { return (n + 255) / 256; };
  auto nmma_of = [&](int n) { return round16((n + ntiles_n(n) - 1) / ntiles_n(n)); };
  DwParams dp0{};
  // per-evaluation operand copies: [W_l, b_l] (tf32, bias column) and W_l^T (tf32)
  for (int l = 1; l < L; ++l) {
    const LayerDev& ly = net.layer[l - 1];
    const int64_t cnt = (int64_t)s->sz[l] * s->kxl[l - 1];
    split_w1_kernel<0><<<148 * 8, 256, 0, c.stream>>>(
        theta_in, net.Dp, ly.woff, ly.boff, s->sz[l - 1], s->kxl[l - 1], cnt, J, s->Whi[l], nullptr);
    LAUNCHED();
  }
  if (need_grad)
    for (int l = 2; l < L; ++l) {
      dim3 grid((unsigned)((s->sz[l] + 31) / 32), (unsigned)((s->sz[l - 1] + 31) / 32), (unsigned)J);
      transpose_w_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(theta_in, net.Dp, net.layer[l - 1].woff, s->sz[l - 1],
                                                             s->sz[l], s->ldd[l], J, s->WThi[l], s->WTlo[l]);
      LAUNCHED();
    }
  auto act_go = [&](auto fn) {
    if (net.act == DASMC_RELU)
      fn(std::integral_constant<int, DASMC_RELU>{});
    else
      fn(std::integral_constant<int, DASMC_TANH>{});
  };
  // forward through the hidden layers
  for (int l = 1; l < L; ++l) {
    const int nin = s->sz[l - 1], nout = s->sz[l], ntn = ntiles_n(nout), nm = nmma_of(nout);
    const CUtensorMap A = l == 1 ? map2d(s->Xhi, nin + 1, M, s->kxl[0], BM)
                                 : map3d(s->aRow[l - 1], nin + 1, M, s->kxl[l - 1], J, Mcap * s->kxl[l - 1], BM);
    const CUtensorMap B = map3d(s->Whi[l], nin + 1, nout, s->kxl[l - 1], J, (uint64_t)nout * s->kxl[l - 1], nm);
    TileParams tp{};
    tp.rtiles = rtiles;
    tp.J = (int)J;
    tp.rg = 32;
    tp.nkb = (nin + 1 + BK - 1) / BK;
    tp.nmma = nm;
    tp.brows = nm;
    tp.ntn = ntn;
    FwdParams fp{};
    fp.M = M;
    fp.Mcap = Mcap;
    fp.ldm = nba;
    fp.out_row = s->aRow[l];
    fp.out_ld = s->kxl[l];
    fp.out_T = s->aT[l];
    fp.out_rows = nout + 1;
    fp.n_valid = nout;
    act_go([&](auto a) {
      constexpr int A_ = decltype(a)::value;
      if (l == 1)
        launch_tc<kEpiKindHidden, false, kAShared, 4, A_>(c, A, A, B, B, tp, fp, dp0, 0);
      else
        launch_tc<kEpiKindHidden, false, kARowMajor, 4, A_>(c, A, A, B, B, tp, fp, dp0, 0);
    });
  }
  // output layer, log-softmax, delta_L, delta_{L-1} (CUDA cores)
  {
    const int nin = s->sz[L - 1], C = s->sz[L];
    const LayerDev& ly = net.layer[L - 1];
    dim3 grid((unsigned)rtiles, (unsigned)J);
    auto go = [&](auto cp) {
      constexpr int CPv = decltype(cp)::value;
      const size_t sm = sizeof(float) * ((size_t)nin * CPv + CPv);
      auto kern = head_kernel<CPv>;
      static bool attr[kMaxDevices] = {};
      const int dv = current_device();
      if (!attr[dv]) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr[dv] = true;
      }
      kern<<<grid, 128, sm, c.stream>>>(s->aT[L - 1], nin, C, nba, theta_in, net.Dp, ly.woff, ly.boff, net.act, c.y,
                                        M, P, (float)beta_rows, need_grad ? 1 : 0, c.ll_part, c.ll_slots, s->dTl[L],
                                        s->dTl[L - 1], L - 1 >= 2 ? s->dRow[L - 1] : nullptr,
                                        L - 1 >= 2 ? s->dRowLo[L - 1] : nullptr, s->ldd[L - 1], Mcap);
      LAUNCHED();
    };
    if (C <= 4)
      go(std::integral_constant<int, 4>{});
    else if (C <= 12)
      go(std::integral_constant<int, 12>{});
    else
      go(std::integral_constant<int, 16>{});
  }
  if (!need_grad) return;
  // backward deltas: delta_{l-1} = (delta_l W_l) . act'(a_{l-1})
  for (int l = L - 1; l >= 2; --l) {
    const int nk = s->sz[l], nout = s->sz[l - 1], ntn = ntiles_n(nout), nm = nmma_of(nout);
    const CUtensorMap A = map3d(s->dRow[l], nk, M, s->ldd[l], J, Mcap * s->ldd[l], BM);
    const CUtensorMap Alo = kDeepSplitBack ? map3d(s->dRowLo[l], nk, M, s->ldd[l], J, Mcap * s->ldd[l], BM) : A;
    const CUtensorMap B = map3d(s->WThi[l], nk, nout, s->ldd[l], J, (uint64_t)nout * s->ldd[l], nm);
    const CUtensorMap Blo =
        kDeepSplitBack ? map3d(s->WTlo[l], nk, nout, s->ldd[l], J, (uint64_t)nout * s->ldd[l], nm) : B;
    TileParams tp{};
    tp.rtiles = rtiles;
    tp.J = (int)J;
    tp.rg = 32;
    tp.nkb = (nk + BK - 1) / BK;
    tp.nmma = nm;
    tp.brows = nm;
    tp.ntn = ntn;
    FwdParams fp{};
    fp.M = M;
    fp.Mcap = Mcap;
    fp.ldm = nba;
    fp.out_row = l - 1 >= 2 ? s->dRow[l - 1] : nullptr;
    fp.out_row_lo = l - 1 >= 2 ? s->dRowLo[l - 1] : nullptr;
    fp.out_ld = s->ldd[l - 1];
    fp.out_T = s->dTl[l - 1];
    fp.out_rows = nout;
    fp.n_valid = nout;
    fp.mask_src = s->aRow[l - 1];
    fp.mask_ld = s->kxl[l - 1];
    act_go([&](auto a) {
      constexpr int A_ = decltype(a)::value;
      launch_tc<kEpiKindBackDelta, kDeepSplitBack, kARowMajor, 4, A_>(c, A, Alo, B, Blo, tp, fp, dp0, 0);
    });
  }
  // weight gradients + fused leapfrog: dW_l^T[i, o] = sum_m a_{l-1}^T[i, m] delta_l^T[o, m]
  FwdParams fp0{};
  for (int l = L; l >= 1; --l) {
    KTimer kt(c, l == 1 ? 1 : -1);
    const int nin = s->sz[l - 1], nout = s->sz[l], ntn = ntiles_n(nout), nm = nmma_of(nout);
    const CUtensorMap B = map_blk(s->dTl[l], nout, nbu, nba, J, nm);
    TileParams tp{};
    tp.rtiles = (nin + 1 + BM - 1) / BM;
    tp.J = (int)J;
    tp.rg = tp.rtiles;
    tp.nkb = (int)((M + BK - 1) / BK);
    tp.nmma = nm;
    tp.brows = nm;
    tp.ntn = ntn;
    const LayerDev& ly = net.layer[l - 1];
    DwParams dp{*epi, net.Dp, ly.woff, ly.boff, nin, nout};
    if (l == 1) {
      const CUtensorMap A = map2d(s->Xt, M, nin + 1, s->n_pad, BM);
      launch_tc<kEpiKindDw, false, kAShared>(c, A, A, B, B, tp, fp0, dp, 0);
    } else {
      const CUtensorMap A = map_blk(s->aT[l - 1], nin + 1, nbu, nba, J, BM);
      launch_tc<kEpiKindDw, false, kABlocked>(c, A, A, B, B, tp, fp0, dp, 0);
    }
  }
}

// The one-hidden-layer path (fused forward + two weight-gradient GEMMs); PREC 0 = tf32 /
// split-tf32 operands in fp32 containers, PREC 1 = fp16 operands (kind::f16).
template <int PREC>
void tc_eval_fused(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
                   const EpiParams* epi) {
  TcState* s = c.tc;
  // PREC 2 (tf32h): tf32 forward (X, W1 tf32), fp16 weight-gradient operands (kind::f16)
  constexpr int FP = PREC == 1 ? 1 : 0, BP = PREC >= 1 ? 1 : 0;
  constexpr int BKE = FP == 1 ? 64 : 32, BKB = BP == 1 ? 64 : 32;
  const int esz = FP == 1 ? 2 : 4, besz = BP == 1 ? 2 : 4;
  const NetDev& net = c.net;
  const LayerDev& l1 = net.layer[0];
  const LayerDev& l2 = net.layer[1];
  const int n0 = s->n0, n1 = s->n1, C = s->C;
  const int64_t ldm = s->mcap;
  const int rtiles = (int)((M + BM - 1) / BM);

  // ---- fused forward: Z1 = X W1^T on tensor cores, layer 2 + loss + deltas in the epilogue
  {
    KTimer kt(c, need_grad ? 0 : -1);
    // [W1, b1] -> tf32 (rna) hi [+ lo]: the MMA would otherwise truncate the low mantissa
    // bits; the bias rides along as K column n0 against X's ones column
    const int64_t kx = s->kx, cnt = (int64_t)n1 * kx;
    split_w1_kernel<FP><<<148 * 8, 256, 0, c.stream>>>(
        theta_in, net.Dp, l1.woff, l1.boff, n0, kx, cnt, J, reinterpret_cast<OpT<FP>*>(s->W1hi),
        (PREC == 0 && s->split) || (PREC == 1 && s->f16x2) ? reinterpret_cast<OpT<FP>*>(s->W1lo) : nullptr);
    LAUNCHED();
    // rows >= M of X are TMA zero fill (ones column included): z1 = 0 there
    // cluster shape (see ClusterShape): CTA pairs stream half of W1's rows each (box
    // nmma / 2, rows >= n1 zero fill); QA = 2 multicasts X rows (box 64 rows per CTA),
    // QB = 2 multicasts W1 rows (two pieces of bbox rows, multiples of 8)
#ifdef DASMC_V_F16X2_MC
    const int cl = (s->split || (PREC != 0 && !s->f16x2)) ? std::min(s->cluster, 1) : s->cluster;
#else
    const int cl = (s->split || PREC != 0) ? std::min(s->cluster, 1) : s->cluster;
#endif
    const bool pair = cl > 0;
    const int QA = (cl == 2 || cl == 4) ? 2 : 1, QB = (cl == 3 || cl == 4) ? 2 : 1;
    const int half = round16(n1) / 2;
    const int bpiece = QB == 2 ? (half / 2 + 7) / 8 * 8 : half;
    const uint32_t bbox = pair ? (uint32_t)bpiece : (uint32_t)n1;
    const CUtensorMap A = map2d(s->Xhi, n0 + 1, M, kx, BM / QA, esz);
    const CUtensorMap Alo = s->split ? map2d(s->Xlo, n0 + 1, M, kx, BM / QA) : A;
    const CUtensorMap B = map3d(s->W1hi, n0 + 1, n1, kx, J, cnt, bbox, esz);
    const CUtensorMap Blo = s->split    ? map3d(s->W1lo, n0 + 1, n1, kx, J, cnt, bbox)
                            : s->f16x2 ? map3d(s->W1lo, n0 + 1, n1, kx, J, cnt, bbox, esz)
                                       : B;
    TileParams tp{};
    tp.rtiles = pair ? (rtiles + 2 * QB - 1) / (2 * QB) : rtiles;
    tp.J = pair ? (int)((J + QA - 1) / QA) : (int)J;
    tp.rg = pair ? 32 / (2 * QB) : 32;
    tp.bbox = bpiece;
    tp.hint_a = 1;  // X (shared by every particle): keep it in L2 against the activation-store stream
    if (const char* e = std::getenv("DASMC_TC_RG")) tp.rg = std::max(1, std::atoi(e));   // tuning only
    if (const char* e = std::getenv("DASMC_TC_HINTA")) tp.hint_a = std::atoi(e);        // tuning only
    if (const char* e = std::getenv("DASMC_TC_HINTB")) tp.hint_b = std::atoi(e);        // tuning only
    if (const char* e = std::getenv("DASMC_TC_PREFETCH")) tp.prefetch = std::atoi(e);   // tuning only
    tp.nkb = (n0 + 1 + BKE - 1) / BKE;
    tp.klast = (n0 + 1 - (tp.nkb - 1) * BKE + BKE / 4 - 1) / (BKE / 4);  // C2: 785 = 12 x 64 + 17 -> 2 of 4 k-steps
    if (const char* e = std::getenv("DASMC_TC_KLAST")) tp.klast = std::atoi(e);         // tuning only
    tp.nmma = round16(n1);
    tp.brows = n1;
    FwdParams fp{};
    fp.theta = theta_in;
    fp.Dp = net.Dp;
    fp.woff2 = l2.woff;
    fp.boff2 = l2.boff;
    fp.n1 = n1;
    fp.C = C;
    fp.act = net.act;
    fp.y = c.y;
    fp.M = M;
    fp.P = P;
    fp.Jn = (int)J;
    fp.beta_rows = (float)beta_rows;
    fp.need_grad = need_grad ? 1 : 0;
    fp.ldm = ldm / 128;  // number of 128-row blocks allocated per particle
    fp.a1T = s->a1T;
    fp.d1T = s->d1T;
    fp.d2T = s->d2T;
    fp.a1Tlo = s->a1Tlo;
    fp.d1Tlo = s->d1Tlo;
    fp.d2Tlo = s->d2Tlo;
    fp.ll_part = c.ll_part;
    fp.ll_slots = c.ll_slots;
    if (const char* e = std::getenv("DASMC_DEBUG_EPI")) fp.dbg = std::atoi(e);  // profiling only
    // classes padded to 4, 10 or 16 (W2^T rows float4-aligned in shared memory)
    const int CP = C <= 4 ? 4 : C <= 10 ? 10 : 16;
    const int CS = (CP + 3) & ~3;
    // + the tensor-core pass 2's barriers and operand tiles (DASMC_L2TC): 16 + alignment + 4096 + 128 rows x 32 B
    const size_t epi_bytes = sizeof(float) * (2 * ((size_t)n1 * CS + CS) + kParts * 128 * CP) + 8 * sizeof(double) + 16 +
                             (16 + 128 + 4096 + 128 * 32);
    DwParams dp{};
    auto go = [&](auto cp, auto act) {
      constexpr int K = decltype(cp)::value, A_ = decltype(act)::value;
      if constexpr (PREC == 1) {
        if (s->f16x2) {
#ifdef DASMC_V_F16X2_MC  // multicast cluster shapes for the f16x2 forward (tuning builds)
          if (cl == 3)
            launch_tc<kEpiKindFwd, false, kAShared, K, A_, 3, 3>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          else if (cl == 4)
            launch_tc<kEpiKindFwd, false, kAShared, K, A_, 4, 3>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          else if (cl == 2)
            launch_tc<kEpiKindFwd, false, kAShared, K, A_, 2, 3>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          else
#endif
          if (pair)
            launch_tc<kEpiKindFwd, false, kAShared, K, A_, 1, 3>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          else
            launch_tc<kEpiKindFwd, false, kAShared, K, A_, 0, 3>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          return;
        }
      }
      if constexpr (PREC == 0) {
        if (s->split) {
          if (pair)
            launch_tc<kEpiKindFwd, true, kAShared, K, A_, 1>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          else
            launch_tc<kEpiKindFwd, true, kAShared, K, A_, 0>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
          return;
        }
      }
      // the multicast cluster shapes (CL 2..4, measured slower than plain pairs) are built for
      // the tf32 path only; fp16-operand modes run single CTAs or pairs
      if constexpr (PREC == 0) {
        switch (cl) {
          case 0: launch_tc<kEpiKindFwd, false, kAShared, K, A_, 0, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes); break;
          case 1: launch_tc<kEpiKindFwd, false, kAShared, K, A_, 1, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes); break;
          case 2: launch_tc<kEpiKindFwd, false, kAShared, K, A_, 2, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes); break;
          case 3: launch_tc<kEpiKindFwd, false, kAShared, K, A_, 3, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes); break;
          default: launch_tc<kEpiKindFwd, false, kAShared, K, A_, 4, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes); break;
        }
      } else {
        if (cl == 0)
          launch_tc<kEpiKindFwd, false, kAShared, K, A_, 0, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
        else
          launch_tc<kEpiKindFwd, false, kAShared, K, A_, 1, PREC>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
      }
    };
    auto go_act = [&](auto cp) {
      if (net.act == DASMC_RELU)
        go(cp, std::integral_constant<int, DASMC_RELU>{});
      else
        go(cp, std::integral_constant<int, DASMC_TANH>{});
    };
    switch (CP) {
      case 4: go_act(std::integral_constant<int, 4>{}); break;
      case 10: go_act(std::integral_constant<int, 10>{}); break;
      default: go_act(std::integral_constant<int, 16>{}); break;
    }
  }
  if (!need_grad) return;
  FwdParams fp0{};
  // ---- layer 2: dW2^T[o, c] = sum_m a1^T[o, m] delta2^T[c, m]  (ones row o = n1 -> db2)
  {
    const uint64_t nbu = (uint64_t)(M + 127) / 128, nba = (uint64_t)ldm / 128;
    const CUtensorMap A = map_blk(s->a1T, n1 + 1, nbu, nba, J, BM, besz);
    const CUtensorMap Alo = s->split ? map_blk(s->a1Tlo, n1 + 1, nbu, nba, J, BM) : A;
    const CUtensorMap B = map_blk(s->d2T, C, nbu, nba, J, C, besz);
    const CUtensorMap Blo = s->split ? map_blk(s->d2Tlo, C, nbu, nba, J, C) : B;
    TileParams tp{};
    tp.rtiles = (n1 + 1 + BM - 1) / BM;
    tp.J = (int)J;
    tp.rg = tp.rtiles;
    tp.nkb = (int)((M + BKB - 1) / BKB);
    tp.nmma = round16(C);
    tp.brows = C;
    DwParams dp{*epi, net.Dp, l2.woff, l2.boff, n1, C};
    if (PREC == 0 && s->split)
      launch_tc<kEpiKindDw, PREC == 0, kABlocked>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
    else
      launch_tc<kEpiKindDw, false, kABlocked, 4, 0, 0, BP>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
  }
  // ---- layer 1: dW1^T[i, o] = sum_m X^T[i, m] delta1^T[o, m]  (ones row i = n0 -> db1)
  {
    KTimer kt(c, 1);
    const CUtensorMap A = map2d(s->Xt, M, n0 + 1, s->n_pad, BM, besz);
    const CUtensorMap Alo = s->split ? map2d(s->Xtlo, M, n0 + 1, s->n_pad, BM) : A;
    const uint64_t nbu = (uint64_t)(M + 127) / 128, nba = (uint64_t)ldm / 128;
    const CUtensorMap B = map_blk(s->d1T, n1, nbu, nba, J, n1, besz);
    const CUtensorMap Blo = s->split ? map_blk(s->d1Tlo, n1, nbu, nba, J, n1) : B;
    TileParams tp{};
    tp.rtiles = (n0 + 1 + BM - 1) / BM;
    tp.J = (int)J;
    tp.rg = tp.rtiles;
    tp.nkb = (int)((M + BKB - 1) / BKB);
    tp.nmma = round16(n1);
    tp.brows = n1;
    DwParams dp{*epi, net.Dp, l1.woff, l1.boff, n0, n1};
    if (PREC == 0 && s->split)
      launch_tc<kEpiKindDw, PREC == 0, kAShared>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
    else
      launch_tc<kEpiKindDw, false, kAShared, 4, 0, 0, BP>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
  }
}

void tc_eval(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
             const EpiParams* epi) {
  TcState* s = c.tc;
  if (s->deep)
    tc_eval_deep(c, theta_in, J, M, P, beta_rows, need_grad, epi);
  else if (s->f16)
    tc_eval_fused<1>(c, theta_in, J, M, P, beta_rows, need_grad, epi);
  else if (s->hstore)
    tc_eval_fused<2>(c, theta_in, J, M, P, beta_rows, need_grad, epi);
  else
    tc_eval_fused<0>(c, theta_in, J, M, P, beta_rows, need_grad, epi);
}

}  // namespace dasmc_b200
