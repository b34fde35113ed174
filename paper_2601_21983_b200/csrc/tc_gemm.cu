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

namespace dasmc_b200 {

struct TcState {
  int n0 = 0, n1 = 0, C = 0;
  int64_t n_pad = 0;     // X^T row stride (floats)
  int64_t mcap = 0;      // row stride of the transposed activation buffers
  bool split = false;    // split-tf32 (3 MMAs)
  bool mma_layer2 = true; // fused forward runs the layer-2 products on mma.sync (DASMC_MMA_LAYER2=0: CUDA-core FFMA)
  bool tc_layer2 = false; // fused forward runs layer 2 as TMEM-A MMAs (opt-in: DASMC_TC_LAYER2=1;
                          // measured slower on B200: the small MMAs queue behind the next tile's)
  float* Xt = nullptr;   // [(n0+1) x n_pad], row n0 = 1
  float* Xhi = nullptr;  // [n x n0] X rounded to tf32 (cvt.rna): the MMA truncates raw fp32
  float* Xlo = nullptr;  // [n x n0]   (split)
  float* Xtlo = nullptr; // [(n0+1) x n_pad] (split; ones row lo = 0)
  float* W1hi = nullptr; // [J x n1 x n0] W1 rounded to tf32
  float* W1lo = nullptr;
  float* a1T = nullptr;  // [J x (n1+1) x mcap], row n1 = 1
  float* d1T = nullptr;  // [J x n1 x mcap]
  float* d2T = nullptr;  // [J x C x mcap]
  float* a1Tlo = nullptr;
  float* d1Tlo = nullptr;
  float* d2Tlo = nullptr;
  int num_sms = 148;
};

namespace {

constexpr int BM = 128;  // UMMA_M
constexpr int BK = 32;   // fp32 per 128-byte swizzle row
constexpr int kEpiWarps = 12;            // 3 warps per TMEM lane group
constexpr int kParts = kEpiWarps / 4;
// Epilogue a1^T / delta1^T stores through TMA bulk tensor stores instead of
// st.global.  Correct (tested) but measured slower on B200 at C2 (38.8 vs
// 36.2 ms per forward: the 48 KB staging costs a pipeline stage), so off.
constexpr bool kUseTmaStore = false;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;  // TMA warp + MMA warp + epilogue warps
constexpr int kTmemCols = 512;  // 2 accumulators x 256 columns
constexpr int kEpiKindFwd = 0, kEpiKindDw = 1, kEpiKindFwdTc = 2, kEpiKindFwdMma = 3;

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp is parked by the
// hardware (up to ~0.5 ms) instead of spinning and stealing issue slots from
// the epilogue warps on the same SM sub-partition.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
      "selp.b32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(500000u)
      : "memory");
  return ok != 0;
}
// Watchdog: a barrier that never completes (a protocol bug) traps after ~10 s
// instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t i = 1;; ++i) {
    if (mbar_try(bar, parity)) return;
    if ((i & 0x3FFFu) == 0 && clock64() - t0 > 20000000000LL) __trap();
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// Bulk tensor store smem -> global (bulk async-group of the issuing thread).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]  (A: 128 lanes x K columns, K-major)
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Byte offset of element (row r, k) inside a K-major 128B-swizzled tile of
// 32-element k-blocks (8-row core groups of 1024 B; 16 B chunks XOR row % 8).
__device__ __forceinline__ uint32_t sw128_offset(int r, int k, int rows) {
  const int kb = k >> 5, e = k & 31;
  return (uint32_t)(kb * rows * 128 + r * 128 + ((((e >> 2) ^ (r & 7)) & 7) << 4) + (e & 3) * 4);
}

// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// Asynchronous variant: issue the load, wait later with tmem_wait16 on the
// same registers (the "+f" operands order every later use after the wait).
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait16(float* v) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]),
                 "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]),
                 "+f"(v[15])::"memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// K-major, 128B-swizzled UMMA shared-memory descriptor: 8-row core groups
// 1024 B apart (SBO), LBO unused (1), version 1 (sm100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t a = (smem_u32(p) >> 4) & 0x3FFFULL;
  return a | (1ULL << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ULL << 46) | (2ULL << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Warp-level D(16x8) += A(16x8) . B(8x8), tf32 inputs, fp32 accumulate, split
// into hi/lo parts (hi.hi + hi.lo + lo.hi) for fp32-level products.
// Fragment layouts (g = lane / 4, t = lane % 4):
//   A: a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
//   B: b0 (k = t, n = g), b1 (k = t+4, n = g)
//   D: d0 (g, 2t), d1 (g, 2t+1), d2 (g+8, 2t), d3 (g+8, 2t+1)
__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_3xtf32(float* d, const float* a, const float* b) {
  uint32_t ah[4], al[4], bh[2], bl[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float h = tf32_hi(a[i]);
    ah[i] = __float_as_uint(h);
    al[i] = __float_as_uint(tf32_hi(a[i] - h));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float h = tf32_hi(b[i]);
    bh[i] = __float_as_uint(h);
    bl[i] = __float_as_uint(tf32_hi(b[i] - h));
  }
  mma_tf32(d, al, bh);
  mma_tf32(d, ah, bl);
  mma_tf32(d, ah, bh);
}

// ---------------------------------------------------------------- parameters
struct TileParams {
  int rtiles;  // row tiles (of BM rows) per particle
  int J;
  int rg;      // row tiles per scheduling group
  int nkb;     // k blocks of BK
  int nmma;    // MMA N (multiple of 16, <= 256)
  int brows;   // TMA box rows of B (valid rows)
  int stages;
  uint32_t stage_bytes_tx;
};

struct FwdParams {
  CUtensorMap mapS1;   // a1^T store map  {M, n1, J}, box {32, 16, 1}
  CUtensorMap mapS2;   // delta1^T store map
  const float* theta;  // theta_in
  int64_t Dp, boff1, woff2, boff2;
  int n1, C, act;
  const int32_t* y;
  int64_t M, P;
  float beta_rows;
  int need_grad;
  int64_t ldm;  // row stride (floats) of the transposed buffers
  float *a1T, *d1T, *d2T, *a1Tlo, *d1Tlo, *d2Tlo;
  double* ll_part;
  int ll_slots;
  int dbg;  // DASMC_DEBUG_EPI: 1 = skip global stores, 2 = skip pass 2, 3 = skip the whole epilogue math
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
template <int EPI, bool SPLIT, bool A3D, int CP>
__global__ void __launch_bounds__(kThreads, 1)
    tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
              const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo, TileParams tp,
              const __grid_constant__ FwdParams fp, DwParams dp) {
  constexpr bool kTmaStore = kUseTmaStore && EPI == kEpiKindFwd && !SPLIT;
  const CUtensorMap& mapS1 = fp.mapS1;
  const CUtensorMap& mapS2 = fp.mapS2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms; keep the pointer derived
  // from smem_raw so the compiler emits shared-memory (LDS/STS) accesses.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_bytes = BM * BK * 4;
  const uint32_t b_bytes = (uint32_t)tp.nmma * BK * 4;
  const uint32_t sub = SPLIT ? 2 : 1;
  const uint32_t stage_bytes = sub * (a_bytes + b_bytes);
  uint8_t* stages = smem;
  uint64_t* bars = (uint64_t*)(smem + (size_t)tp.stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + tp.stages;
  uint64_t* tfull = bars + 2 * tp.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 2);
  float* epi_smem = (float*)(tmem_holder + 4);  // 16-byte aligned

  auto A_of = [&](int s, int lo) { return stages + (size_t)s * stage_bytes + (lo ? a_bytes : 0); };
  auto B_of = [&](int s, int lo) { return stages + (size_t)s * stage_bytes + sub * a_bytes + (lo ? b_bytes : 0); };

  // zero the stage ring once: rows of B beyond the TMA box stay zero
  for (uint32_t i = threadIdx.x; i < tp.stages * stage_bytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(stages)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    if (SPLIT) {
      prefetch_map(&mapAlo);
      prefetch_map(&mapBlo);
    }
    for (int s = 0; s < tp.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = tp.rtiles * tp.J;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int rt, j;
        tile_coords(tp, t, rt, j);
        for (int kb = 0; kb < tp.nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], tp.stage_bytes_tx);
          const int k0 = kb * BK;
          if (A3D) {
            tma_3d(A_of(s, 0), &mapA, &full[s], k0, rt * BM, j);
            if (SPLIT) tma_3d(A_of(s, 1), &mapAlo, &full[s], k0, rt * BM, j);
          } else {
            tma_2d(A_of(s, 0), &mapA, &full[s], k0, rt * BM);
            if (SPLIT) tma_2d(A_of(s, 1), &mapAlo, &full[s], k0, rt * BM);
          }
          tma_3d(B_of(s, 0), &mapB, &full[s], k0, 0, j);
          if (SPLIT) tma_3d(B_of(s, 1), &mapBlo, &full[s], k0, 0, j);
          if (++s == tp.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(tp.nmma);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * 256);
        for (int kb = 0; kb < tp.nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t ad = smem_desc(A_of(s, 0)), bd = smem_desc(B_of(s, 0));
          const uint64_t adl = smem_desc(A_of(s, 1)), bdl = smem_desc(B_of(s, 1));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const uint64_t off = (uint64_t)(k * 32) >> 4;  // 32 bytes per K=8 step inside the swizzle row
            tc_mma(d, ad + off, bd + off, idesc, (kb | k) != 0);
            if (SPLIT) {
              tc_mma(d, ad + off, bdl + off, idesc, 1);
              tc_mma(d, adl + off, bd + off, idesc, 1);
            }
          }
          tc_commit(&empty[s]);
          if (++s == tp.stages) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else {
    // ===================== epilogue warps 2..9 =====================
    // kParts warps share each TMEM lane group (warp % 4); `part` selects a
    // contiguous range of 16-column accumulator chunks.
    const int et = threadIdx.x - 64;
    const int lg = warp & 3;
    const int part = (warp - 2) >> 2;
    const int half = part;  // (kept for the opt-in TMEM-A layer-2 path, which needs kParts == 2)
    const int row_in_tile = lg * 32 + lane;
    auto chunk_range = [&](int nch, int& lo, int& hi) {
      lo = nch * part / kParts;
      hi = nch * (part + 1) / kParts;
    };
    int acc = 0;
    uint32_t aph = 0;
    uint32_t sph = 0;  // parity of the small-MMA barrier (fused forward, tensor-core layer 2)
    int nst = 0;       // TMA-store staging buffer counter (alternates the warp's two buffers)
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int rt, j;
      tile_coords(tp, t, rt, j);
      if (EPI == kEpiKindFwd) {
        const int n1 = fp.n1, C = fp.C;
        float* W2T = epi_smem;                  // [n1][CP]  W2 transposed, zero-padded
        float* b1s = W2T + (size_t)n1 * CP;     // [n1]
        float* b2s = b1s + ((n1 + 3) & ~3);     // [CP]
        float* z2x = b2s + CP;                  // [kParts][128][CP] partial layer-2 logits
        double* red = (double*)(z2x + kParts * 128 * CP);  // [4][2]
        float* stg_all = (float*)((uint8_t*)(red + 8) + ((128u - (smem_u32(red + 8) & 127u)) & 127u));
        float* stg = stg_all + (warp - 2) * 1024;  // 2 x [16][32] fp32 per warp
        const float* th = fp.theta + (int64_t)j * fp.Dp;
        // per-particle layer-2 parameters: all global loads issued before any
        // shared-memory store (one L2 round trip per tile, not one per element)
        constexpr int kPer = (256 * CP + kEpiThreads - 1) / kEpiThreads;
        float wv[kPer];
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
          const int i = et + r * kEpiThreads;
          const int o = i / CP, c = i - o * CP;
          wv[r] = (i < n1 * CP && c < C) ? th[fp.woff2 + (int64_t)c * n1 + o] : 0.f;
        }
        const float bv = et < n1 ? th[fp.boff1 + et] : 0.f;
        const float b2v = et < C ? th[fp.boff2 + et] : 0.f;
        named_bar(1, kEpiThreads);  // the previous tile is done with the shared parameters
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
          const int i = et + r * kEpiThreads;
          if (i < n1 * CP) W2T[i] = wv[r];
        }
        if (et < n1) b1s[et] = bv;
        if (et < CP) b2s[et] = b2v;
        named_bar(1, kEpiThreads);
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int64_t m = (int64_t)rt * BM + row_in_tile;
        const bool valid = m < fp.M;
        const bool relu = fp.act == DASMC_RELU;
        const bool wr_out = valid && fp.need_grad && fp.dbg != 1;
        int c_lo, c_hi;
        chunk_range((n1 + 15) >> 4, c_lo, c_hi);
        if (fp.dbg == 3) c_hi = c_lo;
        const int64_t ldm = fp.ldm;
        const float4* W2T4 = reinterpret_cast<const float4*>(W2T);
        float z2[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) z2[c] = 0.f;
        float* a1T = fp.a1T + (int64_t)j * (n1 + 1) * ldm + m;
        float* a1Tlo = SPLIT ? fp.a1Tlo + (int64_t)j * (n1 + 1) * ldm + m : nullptr;
        // pass 1: a1 = act(z1 + b1); partial z2 = W2 a1 over this warp's columns
        // TMA-store staging (non-split): the warp's 32 rows x 16 columns go to a
        // [16][32] smem tile, one bulk tensor store per chunk (clipped at m >= M, o >= n1)
        const bool st_any = kTmaStore && fp.need_grad && fp.dbg != 1;
        auto stage_begin = [&]() -> float* {
          float* buf = stg + (nst & 1) * 512;
          if (lane == 0) bulk_wait_read1();  // the store that last used this buffer has read it
          __syncwarp();
          return buf;
        };
        auto stage_end = [&](const CUtensorMap* map, float* buf, int o0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(map, buf, rt * BM + lg * 32, o0, j);
            bulk_commit();
          }
          ++nst;
        };
        auto pass1 = [&](const float* v, int q, const float4* w4, float b, float*& pa, float*& pal, float* sb) {
          float a = v[q] + b;
          a = relu ? fmaxf(a, 0.f) : tanhf(a);
#pragma unroll
          for (int u = 0; u < CP / 4; ++u) {
            const float4 w = w4[q * (CP / 4) + u];
            z2[4 * u] = fmaf(a, w.x, z2[4 * u]);
            z2[4 * u + 1] = fmaf(a, w.y, z2[4 * u + 1]);
            z2[4 * u + 2] = fmaf(a, w.z, z2[4 * u + 2]);
            z2[4 * u + 3] = fmaf(a, w.w, z2[4 * u + 3]);
          }
          if (kTmaStore) {
            if (st_any) sb[q * 32 + lane] = tf32_hi(a);
          } else {
            if (wr_out) {
              const float hi = tf32_hi(a);
              *pa = hi;
              if (SPLIT) *pal = a - hi;
            }
            pa += ldm;
            if (SPLIT) pal += ldm;
          }
        };
        auto chunk1 = [&](int ch, const float* v) {
          const int o0 = ch * 16;
          const int nq = min(16, n1 - o0);  // warp-uniform
          float* pa = a1T + (int64_t)o0 * ldm;
          float* pal = SPLIT ? a1Tlo + (int64_t)o0 * ldm : nullptr;
          const float4* w4 = W2T4 + o0 * (CP / 4);
          float* sb = st_any ? stage_begin() : nullptr;
          if (nq == 16) {
#pragma unroll
            for (int q = 0; q < 16; ++q) pass1(v, q, w4, b1s[o0 + q], pa, pal, sb);
          } else {  // tail chunk: still unrolled so v[] stays in registers
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q < nq) pass1(v, q, w4, b1s[o0 + q], pa, pal, sb);
          }
          if (st_any) stage_end(&mapS1, sb, o0);
        };
        {  // TMEM loads double-buffered: chunk ch+1 is in flight while ch is processed
          float va[16] = {}, vb[16] = {};
          int ch = c_lo;
          if (ch < c_hi) tmem_ld16_async(taddr + ch * 16, va);
          tmem_wait16(va);
          while (ch < c_hi) {
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, vb);
            chunk1(ch, va);
            tmem_wait16(vb);
            if (++ch >= c_hi) break;
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, va);
            chunk1(ch, vb);
            tmem_wait16(va);
            ++ch;
          }
        }
        // combine the column parts in a fixed order
        float* zx = z2x + ((size_t)part * 128 + row_in_tile) * CP;
#pragma unroll
        for (int c = 0; c < CP; ++c) zx[c] = z2[c];
        named_bar(1, kEpiThreads);
        // part 0 alone: log-softmax likelihood of the row (network.hpp:183-193) --
        // fp32 exponentials, fp64 log-normaliser and ll -- and delta2, shared via
        // its z2x slot with the other parts
        double ll = 0.0;
        float d2[CP];
#pragma unroll
        for (int c = 0; c < CP; ++c) d2[c] = 0.f;
        if (part == 0) {
#pragma unroll
          for (int c = 0; c < CP; ++c) {
            float s = z2x[(size_t)row_in_tile * CP + c];
#pragma unroll
            for (int p = 1; p < kParts; ++p) s += z2x[((size_t)p * 128 + row_in_tile) * CP + c];
            z2[c] = s + b2s[c];
          }
          if (valid) {
            const int yi = fp.y[m];
            float mx = z2[0];
#pragma unroll
            for (int c = 1; c < CP; ++c)
              if (c < C) mx = fmaxf(mx, z2[c]);
            float e[CP];
            double den = 0.0;
            float zy = 0.f;
#pragma unroll
            for (int c = 0; c < CP; ++c) {
              e[c] = c < C ? expf(z2[c] - mx) : 0.f;
              den += (double)e[c];
              if (c == yi) zy = z2[c];
            }
            ll = (double)zy - ((double)mx + log(den));
            if (fp.need_grad) {
              const float wrow = m < fp.P ? 1.f : fp.beta_rows;
              const float rden = (float)(1.0 / den);
#pragma unroll
              for (int c = 0; c < CP; ++c)
                if (c < C) {
                  d2[c] = wrow * ((c == yi ? 1.f : 0.f) - e[c] * rden);
                  const float hi = tf32_hi(d2[c]);
                  fp.d2T[((int64_t)j * C + c) * ldm + m] = hi;
                  if (SPLIT) fp.d2Tlo[((int64_t)j * C + c) * ldm + m] = d2[c] - hi;
                }
            }
          }
#pragma unroll
          for (int c = 0; c < CP; ++c) zx[c] = d2[c];
        }
        if (fp.need_grad && fp.dbg == 0) {
          named_bar(1, kEpiThreads);
          if (part != 0) {
#pragma unroll
            for (int c = 0; c < CP; ++c) d2[c] = z2x[(size_t)row_in_tile * CP + c];
          }
        }
        if (fp.need_grad && fp.dbg == 0) {
          // pass 2: delta1 = (W2^T delta2) . act'(a1)  (network.hpp:209-215)
          float* d1T = fp.d1T + (int64_t)j * n1 * ldm + m;
          float* d1Tlo = SPLIT ? fp.d1Tlo + (int64_t)j * n1 * ldm + m : nullptr;
          auto pass2 = [&](const float* v, int q, const float4* w4, float b, float*& pd, float*& pdl, float* sb) {
            float a = v[q] + b;
            a = relu ? fmaxf(a, 0.f) : tanhf(a);
            float dx = 0.f, dy = 0.f, dzz = 0.f, dw = 0.f;  // 4 independent chains
#pragma unroll
            for (int u = 0; u < CP / 4; ++u) {
              const float4 w = w4[q * (CP / 4) + u];
              dx = fmaf(d2[4 * u], w.x, dx);
              dy = fmaf(d2[4 * u + 1], w.y, dy);
              dzz = fmaf(d2[4 * u + 2], w.z, dzz);
              dw = fmaf(d2[4 * u + 3], w.w, dw);
            }
            const float dz = (dx + dy) + (dzz + dw);
            const float d1 = relu ? dz * (a > 0.f ? 1.f : 0.f) : dz * (1.f - a * a);
            const float hi = tf32_hi(d1);
            if (kTmaStore) {
              sb[q * 32 + lane] = hi;
            } else {
              if (valid) {
                *pd = hi;
                if (SPLIT) *pdl = d1 - hi;
              }
              pd += ldm;
              if (SPLIT) pdl += ldm;
            }
          };
          auto chunk2 = [&](int ch, const float* v) {
            const int o0 = ch * 16;
            const int nq = min(16, n1 - o0);  // warp-uniform
            float* pd = d1T + (int64_t)o0 * ldm;
            float* pdl = SPLIT ? d1Tlo + (int64_t)o0 * ldm : nullptr;
            const float4* w4 = W2T4 + o0 * (CP / 4);
            float* sb = kTmaStore ? stage_begin() : nullptr;
            if (nq == 16) {
#pragma unroll
              for (int q = 0; q < 16; ++q) pass2(v, q, w4, b1s[o0 + q], pd, pdl, sb);
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (q < nq) pass2(v, q, w4, b1s[o0 + q], pd, pdl, sb);
            }
            if (kTmaStore) stage_end(&mapS2, sb, o0);
          };
          float va[16] = {}, vb[16] = {};
          int ch = c_lo;
          if (ch < c_hi) tmem_ld16_async(taddr + ch * 16, va);
          tmem_wait16(va);
          while (ch < c_hi) {
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, vb);
            chunk2(ch, va);
            tmem_wait16(vb);
            if (++ch >= c_hi) break;
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, va);
            chunk2(ch, vb);
            tmem_wait16(va);
            ++ch;
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        // per-tile prefix / block log-likelihood partials (deterministic order)
        double pre = (valid && m < fp.P) ? ll : 0.0, blk = (valid && m >= fp.P) ? ll : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pre += __shfl_xor_sync(0xffffffffu, pre, o);
          blk += __shfl_xor_sync(0xffffffffu, blk, o);
        }
        if (lane == 0 && half == 0) {
          red[lg * 2] = pre;
          red[lg * 2 + 1] = blk;
        }
        named_bar(1, kEpiThreads);
        if (et == 0) {
          double* o = fp.ll_part + ((int64_t)j * fp.ll_slots + rt) * 2;
          o[0] = red[0] + red[2] + red[4] + red[6];
          o[1] = red[1] + red[3] + red[5] + red[7];
        }
      } else if (EPI == kEpiKindFwdMma) {
        // Fused forward with the layer-2 products on warp-level tensor cores:
        // per 16-column chunk a warp stages its 32 rows x 16 columns of A1 in
        // shared memory and runs z2 += A1 . W2^T (M 32, N 16, K 16) and, in
        // pass 2, dz = delta2 . W2 (M 32, N 16, K 16) as split-tf32 mma.sync.
        constexpr int WS = 24;  // W2T row stride (floats): conflict-free B loads in pass 1
        constexpr int ZS = 20;  // row stride of the per-warp staging / exchange tiles
        const int n1 = fp.n1, C = fp.C;
        const int NP = tp.nmma;
        float* W2T = epi_smem;                  // [NP][WS]  W2 transposed, zero-padded (c >= C, o >= n1)
        float* b1s = W2T + (size_t)NP * WS;     // [NP]
        float* b2s = b1s + NP;                  // [16]
        float* z2x = b2s + 16;                  // [kParts][128][ZS] z2 partials, then delta2 in part 0
        double* red = (double*)(z2x + kParts * 128 * ZS);  // [4][2]
        float* As = (float*)(red + 8) + (warp - 2) * 32 * ZS;  // per-warp [32][ZS] staging
        const float* th = fp.theta + (int64_t)j * fp.Dp;
        constexpr int kPerW = (256 * 16 + kEpiThreads - 1) / kEpiThreads;
        float wv[kPerW];
#pragma unroll
        for (int r = 0; r < kPerW; ++r) {  // element (o, c) -> W2[c][o]
          const int i = et + r * kEpiThreads;
          const int o = i >> 4, c = i & 15;
          wv[r] = (o < n1 && c < C) ? th[fp.woff2 + (int64_t)c * n1 + o] : 0.f;
        }
        const float bv = et < n1 ? th[fp.boff1 + et] : 0.f;
        const float b2v = et < C ? th[fp.boff2 + et] : 0.f;
        named_bar(1, kEpiThreads);
#pragma unroll
        for (int r = 0; r < kPerW; ++r) {
          const int i = et + r * kEpiThreads;
          if (i < NP * 16) W2T[(i >> 4) * WS + (i & 15)] = wv[r];
        }
        if (et < NP) b1s[et] = bv;
        if (et < 16) b2s[et] = b2v;
        named_bar(1, kEpiThreads);
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int64_t m = (int64_t)rt * BM + row_in_tile;
        const bool valid = m < fp.M;
        const bool relu = fp.act == DASMC_RELU;
        const bool wr_out = valid && fp.need_grad && fp.dbg != 1;
        int c_lo, c_hi;
        chunk_range(NP >> 4, c_lo, c_hi);
        if (fp.dbg == 3) c_hi = c_lo;
        const int64_t ldm = fp.ldm;
        const int g = lane >> 2, tq = lane & 3;
        float zacc[2][2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int q = 0; q < 4; ++q) zacc[a][b][q] = 0.f;
        float* a1T = fp.a1T + (int64_t)j * (n1 + 1) * ldm + m;
        float* a1Tlo = SPLIT ? fp.a1Tlo + (int64_t)j * (n1 + 1) * ldm + m : nullptr;
        // pass 1: a1 = act(z1 + b1) -> a1^T; z2 += A1 . W2^T on mma.sync
        auto chunk1 = [&](int ch, const float* v) {
          const int o0 = ch * 16;
          float* pa = a1T + (int64_t)o0 * ldm;
          float* pal = SPLIT ? a1Tlo + (int64_t)o0 * ldm : nullptr;
          float a[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            a[q] = v[q] + b1s[o0 + q];
            a[q] = relu ? fmaxf(a[q], 0.f) : tanhf(a[q]);
            if (o0 + q >= n1) a[q] = 0.f;
            if (wr_out && o0 + q < n1) {
              const float hi = tf32_hi(a[q]);
              *pa = hi;
              if (SPLIT) *pal = a[q] - hi;
            }
            pa += ldm;
            if (SPLIT) pal += ldm;
          }
          float4* as4 = reinterpret_cast<float4*>(As + lane * ZS);
#pragma unroll
          for (int q = 0; q < 4; ++q) as4[q] = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
          __syncwarp();
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            float bf[2][2];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              bf[nt][0] = W2T[(o0 + 8 * ks + tq) * WS + 8 * nt + g];
              bf[nt][1] = W2T[(o0 + 8 * ks + tq + 4) * WS + 8 * nt + g];
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const float* r0 = As + (16 * mt + g) * ZS + 8 * ks + tq;
              const float af[4] = {r0[0], r0[8 * ZS], r0[4], r0[8 * ZS + 4]};
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) mma_3xtf32(zacc[mt][nt], af, bf[nt]);
            }
          }
          __syncwarp();
        };
        {
          float va[16] = {}, vb[16] = {};
          int ch = c_lo;
          if (ch < c_hi) tmem_ld16_async(taddr + ch * 16, va);
          tmem_wait16(va);
          while (ch < c_hi) {
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, vb);
            chunk1(ch, va);
            tmem_wait16(vb);
            if (++ch >= c_hi) break;
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, va);
            chunk1(ch, vb);
            tmem_wait16(va);
            ++ch;
          }
        }
        // z2 partial fragments -> exchange tile rows of this part
        {
          float* zb = z2x + ((size_t)part * 128 + lg * 32) * ZS;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              float* p0 = zb + (16 * mt + g) * ZS + 8 * nt + 2 * tq;
              *reinterpret_cast<float2*>(p0) = make_float2(zacc[mt][nt][0], zacc[mt][nt][1]);
              *reinterpret_cast<float2*>(p0 + 8 * ZS) = make_float2(zacc[mt][nt][2], zacc[mt][nt][3]);
            }
        }
        named_bar(1, kEpiThreads);
        double ll = 0.0;
        if (part == 0) {
          float z2[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float s = z2x[(size_t)row_in_tile * ZS + c];
#pragma unroll
            for (int p = 1; p < kParts; ++p) s += z2x[((size_t)p * 128 + row_in_tile) * ZS + c];
            z2[c] = s + b2s[c];
          }
          float d2[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) d2[c] = 0.f;
          if (valid) {
            const int yi = fp.y[m];
            float mx = z2[0];
#pragma unroll
            for (int c = 1; c < 16; ++c)
              if (c < C) mx = fmaxf(mx, z2[c]);
            float e[16];
            double den = 0.0;
            float zy = 0.f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              e[c] = c < C ? expf(z2[c] - mx) : 0.f;
              den += (double)e[c];
              if (c == yi) zy = z2[c];
            }
            ll = (double)zy - ((double)mx + log(den));
            if (fp.need_grad) {
              const float wrow = m < fp.P ? 1.f : fp.beta_rows;
              const float rden = (float)(1.0 / den);
#pragma unroll
              for (int c = 0; c < 16; ++c)
                if (c < C) {
                  d2[c] = wrow * ((c == yi ? 1.f : 0.f) - e[c] * rden);
                  const float hi = tf32_hi(d2[c]);
                  fp.d2T[((int64_t)j * C + c) * ldm + m] = hi;
                  if (SPLIT) fp.d2Tlo[((int64_t)j * C + c) * ldm + m] = d2[c] - hi;
                }
            }
          }
          float* zx = z2x + (size_t)row_in_tile * ZS;
#pragma unroll
          for (int c = 0; c < 16; ++c) zx[c] = d2[c];
        }
        if (fp.need_grad && fp.dbg == 0) {
          named_bar(1, kEpiThreads);
          // delta2 A fragments of this warp's 32 rows (K = classes)
          float df[2][2][4];
          {
            const float* db = z2x + (size_t)(lg * 32) * ZS;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const float* r0 = db + (16 * mt + g) * ZS + 8 * ks + tq;
                df[mt][ks][0] = r0[0];
                df[mt][ks][1] = r0[8 * ZS];
                df[mt][ks][2] = r0[4];
                df[mt][ks][3] = r0[8 * ZS + 4];
              }
          }
          float* d1T = fp.d1T + (int64_t)j * n1 * ldm + m;
          float* d1Tlo = SPLIT ? fp.d1Tlo + (int64_t)j * n1 * ldm + m : nullptr;
          auto chunk2 = [&](int ch, const float* v) {
            const int o0 = ch * 16;
            float dz[2][2][4];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int q = 0; q < 4; ++q) dz[a][b][q] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              float bf[2][2];
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) {  // B(k = c, n = o) = W2[c][o]
                bf[nt][0] = W2T[(o0 + 8 * nt + g) * WS + 8 * ks + tq];
                bf[nt][1] = W2T[(o0 + 8 * nt + g) * WS + 8 * ks + tq + 4];
              }
#pragma unroll
              for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) mma_3xtf32(dz[mt][nt], df[mt][ks], bf[nt]);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int nt = 0; nt < 2; ++nt) {
                float* p0 = As + (16 * mt + g) * ZS + 8 * nt + 2 * tq;
                *reinterpret_cast<float2*>(p0) = make_float2(dz[mt][nt][0], dz[mt][nt][1]);
                *reinterpret_cast<float2*>(p0 + 8 * ZS) = make_float2(dz[mt][nt][2], dz[mt][nt][3]);
              }
            __syncwarp();
            float dr[16];
            const float4* as4 = reinterpret_cast<const float4*>(As + lane * ZS);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = as4[q];
              dr[4 * q] = f.x;
              dr[4 * q + 1] = f.y;
              dr[4 * q + 2] = f.z;
              dr[4 * q + 3] = f.w;
            }
            __syncwarp();
            if (!valid) return;
            float* pd = d1T + (int64_t)o0 * ldm;
            float* pdl = SPLIT ? d1Tlo + (int64_t)o0 * ldm : nullptr;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              if (o0 + q < n1) {
                float a = v[q] + b1s[o0 + q];
                a = relu ? fmaxf(a, 0.f) : tanhf(a);
                const float d1 = relu ? dr[q] * (a > 0.f ? 1.f : 0.f) : dr[q] * (1.f - a * a);
                const float hi = tf32_hi(d1);
                *pd = hi;
                if (SPLIT) *pdl = d1 - hi;
              }
              pd += ldm;
              if (SPLIT) pdl += ldm;
            }
          };
          float va[16] = {}, vb[16] = {};
          int ch = c_lo;
          if (ch < c_hi) tmem_ld16_async(taddr + ch * 16, va);
          tmem_wait16(va);
          while (ch < c_hi) {
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, vb);
            chunk2(ch, va);
            tmem_wait16(vb);
            if (++ch >= c_hi) break;
            if (ch + 1 < c_hi) tmem_ld16_async(taddr + (ch + 1) * 16, va);
            chunk2(ch, vb);
            tmem_wait16(va);
            ++ch;
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        double pre = (valid && m < fp.P) ? ll : 0.0, blk = (valid && m >= fp.P) ? ll : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pre += __shfl_xor_sync(0xffffffffu, pre, o);
          blk += __shfl_xor_sync(0xffffffffu, blk, o);
        }
        if (lane == 0 && part == 0) {
          red[lg * 2] = pre;
          red[lg * 2 + 1] = blk;
        }
        named_bar(1, kEpiThreads);
        if (et == 0) {
          double* o = fp.ll_part + ((int64_t)j * fp.ll_slots + rt) * 2;
          o[0] = red[0] + red[2] + red[4] + red[6];
          o[1] = red[1] + red[3] + red[5] + red[7];
        }
      } else if (EPI == kEpiKindFwdTc) {
        // Layer 2 on the tensor core: A1 = act(Z1 + b1) is written back into
        // the accumulator's TMEM columns and becomes the A operand of
        //   z2 = A1 . W2^T   (N = 16, K = NP)   and   dz = delta2 . W2   (N = NP, K = 16),
        // issued by one epilogue thread; the CUDA cores only do elementwise work.
        const int n1 = fp.n1, C = fp.C;
        const int NP = tp.nmma;                 // padded hidden width (TMEM columns of Z1)
        const int nkb2 = (NP + 31) >> 5;        // 32-wide k blocks of the z2 GEMM
        uint8_t* eb = (uint8_t*)epi_smem;
        eb += (1024u - (smem_u32(eb) & 1023u)) & 1023u;
        uint8_t* W2B = eb;                       // [nkb2][16 rows c][128 B]   B of z2 (K-major, SW128)
        uint8_t* W2TB = W2B + nkb2 * 2048;      // [NP rows o][128 B]         B of dz (K = c, padded to 32)
        float* b1s = (float*)(W2TB + NP * 128);  // [NP]
        float* b2s = b1s + NP;                  // [16]
        double* red = (double*)(b2s + 16);      // [4][2]
        uint64_t* sbar = (uint64_t*)(red + 8);  // small-MMA completion barrier
        if (et == 0 && t == (int)blockIdx.x) {
          mbar_init(sbar, 1);
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        named_bar(1, kEpiThreads);
        const float* th = fp.theta + (int64_t)j * fp.Dp;
        for (int i = et; i < 16 * NP; i += kEpiThreads) {  // W2 (c, o) into both B tiles
          const int c = i / NP, o = i - c * NP;
          const float w = (c < C && o < n1) ? tf32_hi(th[fp.woff2 + (int64_t)c * n1 + o]) : 0.f;
          *(float*)(W2B + sw128_offset(c, o, 16)) = w;
          *(float*)(W2TB + sw128_offset(o, c, NP)) = w;
        }
        for (int i = et; i < NP * 16; i += kEpiThreads) {  // zero the c in [16, 32) half of W2TB rows
          const int o = i >> 4, c = 16 + (i & 15);
          *(float*)(W2TB + sw128_offset(o, c, NP)) = 0.f;
        }
        for (int i = et; i < NP; i += kEpiThreads) b1s[i] = i < n1 ? th[fp.boff1 + i] : 0.f;
        for (int i = et; i < 16; i += kEpiThreads) b2s[i] = i < C ? th[fp.boff2 + i] : 0.f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> MMA reads
        named_bar(1, kEpiThreads);
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tcol = tmem_base + (uint32_t)(acc * 256);
        const uint32_t lane_off = (uint32_t)(lg * 32) << 16;
        const int64_t m = (int64_t)rt * BM + row_in_tile;
        const bool valid = m < fp.M;
        const bool relu = fp.act == DASMC_RELU;
        const bool wr_out = valid && fp.need_grad;
        int c_lo, c_hi;
        chunk_range(NP >> 4, c_lo, c_hi);
        const int64_t ldm = fp.ldm;
        float* a1T = fp.a1T + (int64_t)j * (n1 + 1) * ldm + m;
        float* a1Tlo = SPLIT ? fp.a1Tlo + (int64_t)j * (n1 + 1) * ldm + m : nullptr;
        // pass 1: A1 = act(Z1 + b1) -> TMEM (in place, tf32-rounded) and a1^T
        for (int ch = c_lo; ch < c_hi; ++ch) {
          const int o0 = ch * 16;
          float v[16];
          tmem_ld16(tcol + lane_off + o0, v);
          float* pa = a1T + (int64_t)o0 * ldm;
          float* pal = SPLIT ? a1Tlo + (int64_t)o0 * ldm : nullptr;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float a = v[q] + b1s[o0 + q];
            a = relu ? fmaxf(a, 0.f) : tanhf(a);
            const float hi = tf32_hi(a);
            v[q] = hi;
            if (wr_out && o0 + q < n1) {
              *pa = hi;
              if (SPLIT) *pal = a - hi;
            }
            pa += ldm;
            if (SPLIT) pal += ldm;
          }
          tmem_st16(tcol + lane_off + o0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        named_bar(1, kEpiThreads);
        if (et == 0) {  // z2 = A1 . W2^T into columns [NP, NP+16)
          tc_fence_after();
          const uint32_t id16 = idesc_tf32(16);
          for (int s = 0; s < NP / 8; ++s)
            tc_mma_ts(tcol + NP, tcol + 8 * s, smem_desc(W2B + (s >> 2) * 2048) + (uint64_t)((s & 3) * 2), id16,
                      s > 0);
          tc_commit(sbar);
        }
        mbar_wait(sbar, sph);
        sph ^= 1;
        tc_fence_after();
        float z2[16];
        tmem_ld16(tcol + lane_off + NP, z2);
        double ll = 0.0;
        float d2[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) d2[c] = 0.f;
        if (valid) {
          const int yi = fp.y[m];
#pragma unroll
          for (int c = 0; c < 16; ++c) z2[c] += b2s[c];
          double mx = (double)z2[0];
#pragma unroll
          for (int c = 1; c < 16; ++c)
            if (c < C) mx = fmax(mx, (double)z2[c]);
          double den = 0.0, zy = 0.0;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < C) {
              den += exp((double)z2[c] - mx);
              if (c == yi) zy = (double)z2[c];
            }
          ll = zy - (mx + log(den));
          if (fp.need_grad) {
            const float wrow = m < fp.P ? 1.f : fp.beta_rows;
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c < C) {
                const double pr = exp((double)z2[c] - mx) / den;
                d2[c] = wrow * (float)((c == yi ? 1.0 : 0.0) - pr);
                if (half == 0) {
                  const float hi = tf32_hi(d2[c]);
                  fp.d2T[((int64_t)j * C + c) * ldm + m] = hi;
                  if (SPLIT) fp.d2Tlo[((int64_t)j * C + c) * ldm + m] = d2[c] - hi;
                }
              }
          }
        }
        if (fp.need_grad) {
          if (half == 0) {
#pragma unroll
            for (int c = 0; c < 16; ++c) d2[c] = tf32_hi(d2[c]);
            tmem_st16(tcol + lane_off + NP + 16, d2);
            tmem_st_wait();
          }
          tc_fence_before();
          named_bar(1, kEpiThreads);
          if (et == 0) {  // dz = delta2 . W2 into columns [0, NP) (overwrites A1)
            tc_fence_after();
            const uint32_t idn = idesc_tf32(NP);
            tc_mma_ts(tcol, tcol + NP + 16, smem_desc(W2TB), idn, 0);
            tc_mma_ts(tcol, tcol + NP + 24, smem_desc(W2TB) + 2, idn, 1);
            tc_commit(sbar);
          }
          mbar_wait(sbar, sph);
          sph ^= 1;
          tc_fence_after();
          // pass 2: delta1 = dz . act'(a1), a1 re-read from the a1^T just written (L2)
          float* d1T = fp.d1T + (int64_t)j * n1 * ldm + m;
          float* d1Tlo = SPLIT ? fp.d1Tlo + (int64_t)j * n1 * ldm + m : nullptr;
          for (int ch = c_lo; ch < c_hi; ++ch) {
            const int o0 = ch * 16;
            float v[16];
            tmem_ld16(tcol + lane_off + o0, v);
            if (!valid) continue;
            const float* pa = a1T + (int64_t)o0 * ldm;
            const float* pal = SPLIT ? a1Tlo + (int64_t)o0 * ldm : nullptr;
            float* pd = d1T + (int64_t)o0 * ldm;
            float* pdl = SPLIT ? d1Tlo + (int64_t)o0 * ldm : nullptr;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              if (o0 + q < n1) {
                float a = *pa;
                if (SPLIT && !relu) a += *pal;
                const float d1 = relu ? v[q] * (a > 0.f ? 1.f : 0.f) : v[q] * (1.f - a * a);
                const float hi = tf32_hi(d1);
                *pd = hi;
                if (SPLIT) *pdl = d1 - hi;
              }
              pa += ldm;
              pd += ldm;
              if (SPLIT) {
                pal += ldm;
                pdl += ldm;
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        double pre = (valid && m < fp.P) ? ll : 0.0, blk = (valid && m >= fp.P) ? ll : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pre += __shfl_xor_sync(0xffffffffu, pre, o);
          blk += __shfl_xor_sync(0xffffffffu, blk, o);
        }
        if (lane == 0 && half == 0) {
          red[lg * 2] = pre;
          red[lg * 2 + 1] = blk;
        }
        named_bar(1, kEpiThreads);
        if (et == 0) {
          double* o = fp.ll_part + ((int64_t)j * fp.ll_slots + rt) * 2;
          o[0] = red[0] + red[2] + red[4] + red[6];
          o[1] = red[1] + red[3] + red[5] + red[7];
        }
      } else {
        // weight-gradient tile: row i of A (input index, `in` = bias row), columns o
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(lg * 32) << 16);
        const int i = rt * BM + row_in_tile;
        const bool valid = i <= dp.in;
        const int64_t base = (int64_t)j * dp.Dp;
        int c_lo, c_hi;
        chunk_range((dp.n_out + 15) >> 4, c_lo, c_hi);
        for (int ch = c_lo; ch < c_hi; ++ch) {
          const int o0 = ch * 16;
          float v[16];
          tmem_ld16(taddr + o0, v);
          if (valid) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int o = o0 + q;
              if (o < dp.n_out) {
                const int64_t idx = base + (i < dp.in ? dp.woff + (int64_t)o * dp.in + i : dp.boff + o);
                leapfrog_update(dp.e, j, idx, v[q]);
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if (kTmaStore && lane == 0) bulk_wait_all();  // outstanding epilogue stores done
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols) : "memory");
  }
}

// ---------------------------------------------------------------- helper kernels
// X^T with a ones row (and tf32 hi/lo splits): Xt[i][m] = X[m][i], Xt[n0][m] = 1.
__global__ void transpose_x_kernel(const float* __restrict__ X, int64_t n, int n0, int64_t n_pad, float* Xt, float* Xtlo,
                                   float* Xhi, float* Xlo, int split) {
  __shared__ float tile[32][33];
  const int64_t m0 = (int64_t)blockIdx.x * 32;
  const int i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t m = m0 + r;
    const int i = i0 + threadIdx.x;
    float v = 0.f;
    if (m < n && i < n0) v = X[m * n0 + i];
    if (m < n && i == n0) v = 1.f;
    if (m < n && i < n0) Xhi[m * n0 + i] = tf32_hi(v);
    if (split && m < n && i < n0) Xlo[m * n0 + i] = v - tf32_hi(v);
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r;
    const int64_t m = m0 + threadIdx.x;
    if (i <= n0 && m < n_pad) {
      const float v = m < n ? tile[threadIdx.x][r] : 0.f;
      const float hi = tf32_hi(v);
      Xt[(int64_t)i * n_pad + m] = hi;
      if (split) Xtlo[(int64_t)i * n_pad + m] = v - hi;
    }
  }
}

__global__ void split_w1_kernel(const float* __restrict__ theta, int64_t Dp, int64_t woff, int64_t cnt, int64_t J,
                                float* hi, float* lo) {
  const int64_t total = J * cnt;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / cnt, r = g - j * cnt;
    const float v = theta[j * Dp + woff + r];
    const float h = tf32_hi(v);
    hi[g] = h;
    if (lo) lo[g] = v - h;
  }
}

__global__ void fill_ones_row_kernel(float* buf, int64_t J, int64_t rows, int64_t row, int64_t ldm, float v) {
  const int64_t total = J * ldm;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = g / ldm, m = g - j * ldm;
    buf[(j * rows + row) * ldm + m] = v;
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
CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  uint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

// Store map of a transposed activation buffer [J][rows_alloc][ld]: valid extent
// {M, rows} (stores beyond are clipped), box = one warp's 32 rows x 16 columns.
CUtensorMap map_store(const float* base, uint64_t M, uint64_t rows, uint64_t ld, uint64_t J, uint64_t pstride) {
  const uint64_t dims[3] = {M, rows, J};
  const uint64_t strides[2] = {ld * 4, pstride * 4};
  const uint32_t box[3] = {32, 16, 1};
  return make_map(base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

CUtensorMap map2d(const float* base, uint64_t inner, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  const uint64_t dims[2] = {inner, rows};
  const uint64_t strides[1] = {ld * 4};
  const uint32_t box[2] = {BK, box_rows};
  return make_map(base, 2, dims, strides, box);
}

CUtensorMap map3d(const float* base, uint64_t inner, uint64_t rows, uint64_t ld, uint64_t J, uint64_t pstride,
                  uint32_t box_rows) {
  const uint64_t dims[3] = {inner, rows, J};
  const uint64_t strides[2] = {ld * 4, pstride * 4};
  const uint32_t box[3] = {BK, box_rows, 1};
  return make_map(base, 3, dims, strides, box);
}

int round16(int v) { return (v + 15) / 16 * 16; }

template <int EPI, bool SPLIT, bool A3D, int CP = 4>
void launch_tc(Ctx& c, const CUtensorMap& A, const CUtensorMap& Alo, const CUtensorMap& B, const CUtensorMap& Blo,
               TileParams tp, const FwdParams& fp, const DwParams& dp, size_t epi_smem_bytes) {
  const uint32_t sub = SPLIT ? 2 : 1;
  const size_t stage_bytes = sub * ((size_t)BM * BK * 4 + (size_t)tp.nmma * BK * 4);
  const size_t fixed = 1024 + 64 * 8 + 64 + epi_smem_bytes;
  const size_t budget = 227 * 1024;
  int stages = (int)std::min<size_t>(6, (budget - fixed) / stage_bytes);
  if (stages < 1) throw CudaError{"tensor-core tile does not fit in shared memory"};
  tp.stages = stages;
  tp.stage_bytes_tx = (uint32_t)(sub * ((size_t)BM * BK * 4 + (size_t)tp.brows * BK * 4));
  const size_t smem = 1024 + stages * stage_bytes + (2 * stages + 4) * 8 + 16 + epi_smem_bytes + 64;
  auto kern = tc_kernel<EPI, SPLIT, A3D, CP>;
  static bool attr_set = false;
  if (!attr_set) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget));
    attr_set = true;
  }
  const int ntiles = tp.rtiles * tp.J;
  const int grid = std::max(1, std::min(ntiles, c.tc->num_sms));
  kern<<<grid, kThreads, smem, c.stream>>>(A, SPLIT ? Alo : A, B, SPLIT ? Blo : B, tp, fp, dp);
  LAUNCHED();
}

}  // namespace

bool tc_layer1_eligible(const Ctx& c) {
  const NetDev& n = c.net;
  return n.L == 2 && n.sizes[0] % 4 == 0 && n.sizes[0] >= 4 && n.sizes[1] <= 256 && n.sizes[2] <= 16;
}

void tc_init(Ctx& c) {
  auto* s = new TcState();
  c.tc = s;
  s->n0 = c.net.sizes[0];
  s->n1 = c.net.sizes[1];
  s->C = c.net.sizes[2];
  s->split = c.precision == DASMC_PREC_3XTF32;
  if (const char* e = std::getenv("DASMC_TC_LAYER2")) s->tc_layer2 = e[0] != '0';
  if (const char* e = std::getenv("DASMC_MMA_LAYER2")) s->mma_layer2 = e[0] != '0';
  if (s->tc_layer2) s->mma_layer2 = false;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, dev));
  s->n_pad = (c.n + 31) / 32 * 32;
  const size_t xt = (size_t)(s->n0 + 1) * s->n_pad;
  CK(cudaMalloc(&s->Xt, sizeof(float) * xt));
  const size_t w = (size_t)c.Jmax * s->n1 * s->n0;
  CK(cudaMalloc(&s->Xhi, sizeof(float) * (size_t)c.n * s->n0));
  CK(cudaMalloc(&s->W1hi, sizeof(float) * w));
  if (s->split) {
    CK(cudaMalloc(&s->Xtlo, sizeof(float) * xt));
    CK(cudaMalloc(&s->Xlo, sizeof(float) * (size_t)c.n * s->n0));
    CK(cudaMalloc(&s->W1lo, sizeof(float) * w));
  }
  dim3 grid((unsigned)((s->n_pad + 31) / 32), (unsigned)((s->n0 + 1 + 31) / 32));
  transpose_x_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(c.X, c.n, s->n0, s->n_pad, s->Xt, s->Xtlo, s->Xhi, s->Xlo,
                                                         s->split ? 1 : 0);
  LAUNCHED();
  CK(cudaStreamSynchronize(c.stream));
}

void tc_free(Ctx& c) {
  TcState* s = c.tc;
  if (!s) return;
  float* p[] = {s->Xt, s->Xhi, s->Xlo, s->Xtlo, s->W1hi, s->W1lo, s->a1T, s->d1T, s->d2T, s->a1Tlo, s->d1Tlo, s->d2Tlo};
  for (float* q : p)
    if (q) cudaFree(q);
  delete s;
  c.tc = nullptr;
}

void tc_ensure_rows(Ctx& c, int64_t Mcap) {
  TcState* s = c.tc;
  if (Mcap <= s->mcap) return;
  float** bufs[] = {&s->a1T, &s->d1T, &s->d2T, &s->a1Tlo, &s->d1Tlo, &s->d2Tlo};
  for (float** b : bufs)
    if (*b) {
      CK(cudaFree(*b));
      *b = nullptr;
    }
  const size_t J = (size_t)c.Jmax;
  CK(cudaMalloc(&s->a1T, sizeof(float) * J * (s->n1 + 1) * Mcap));
  CK(cudaMalloc(&s->d1T, sizeof(float) * J * s->n1 * Mcap));
  CK(cudaMalloc(&s->d2T, sizeof(float) * J * s->C * Mcap));
  if (s->split) {
    CK(cudaMalloc(&s->a1Tlo, sizeof(float) * J * (s->n1 + 1) * Mcap));
    CK(cudaMalloc(&s->d1Tlo, sizeof(float) * J * s->n1 * Mcap));
    CK(cudaMalloc(&s->d2Tlo, sizeof(float) * J * s->C * Mcap));
  }
  s->mcap = Mcap;
  const int g = (int)std::min<int64_t>((J * Mcap + 255) / 256, 148 * 16);
  fill_ones_row_kernel<<<g, 256, 0, c.stream>>>(s->a1T, (int64_t)J, s->n1 + 1, s->n1, Mcap, 1.f);
  LAUNCHED();
  if (s->split) {
    fill_ones_row_kernel<<<g, 256, 0, c.stream>>>(s->a1Tlo, (int64_t)J, s->n1 + 1, s->n1, Mcap, 0.f);
    LAUNCHED();
  }
}

void tc_eval(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows, bool need_grad,
             const EpiParams* epi) {
  TcState* s = c.tc;
  const NetDev& net = c.net;
  const LayerDev& l1 = net.layer[0];
  const LayerDev& l2 = net.layer[1];
  const int n0 = s->n0, n1 = s->n1, C = s->C;
  const int64_t ldm = s->mcap;
  const int rtiles = (int)((M + BM - 1) / BM);

  // ---- fused forward: Z1 = X W1^T on tensor cores, layer 2 + loss + deltas in the epilogue
  {
    KTimer kt(c, need_grad ? 0 : -1);
    const float* W1 = theta_in + l1.woff;
    int64_t wstride = net.Dp;
    {  // W1 -> tf32 (rna) hi [+ lo]: the MMA would otherwise truncate the low mantissa bits
      const int64_t cnt = (int64_t)n1 * n0;
      split_w1_kernel<<<(int)std::min<int64_t>((J * cnt + 255) / 256, 148 * 16), 256, 0, c.stream>>>(
          theta_in, net.Dp, l1.woff, cnt, J, s->W1hi, s->split ? s->W1lo : nullptr);
      LAUNCHED();
      W1 = s->W1hi;
      wstride = cnt;
    }
    const CUtensorMap A = map2d(s->Xhi, n0, M, n0, BM);
    const CUtensorMap Alo = s->split ? map2d(s->Xlo, n0, M, n0, BM) : A;
    const CUtensorMap B = map3d(W1, n0, n1, n0, J, wstride, n1);
    const CUtensorMap Blo = s->split ? map3d(s->W1lo, n0, n1, n0, J, wstride, n1) : B;
    TileParams tp{};
    tp.rtiles = rtiles;
    tp.J = (int)J;
    tp.rg = 32;
    tp.nkb = (n0 + BK - 1) / BK;
    tp.nmma = round16(n1);
    tp.brows = n1;
    FwdParams fp{};
    fp.theta = theta_in;
    fp.Dp = net.Dp;
    fp.boff1 = l1.boff;
    fp.woff2 = l2.woff;
    fp.boff2 = l2.boff;
    fp.n1 = n1;
    fp.C = C;
    fp.act = net.act;
    fp.y = c.y;
    fp.M = M;
    fp.P = P;
    fp.beta_rows = (float)beta_rows;
    fp.need_grad = need_grad ? 1 : 0;
    fp.ldm = ldm;
    fp.a1T = s->a1T;
    fp.d1T = s->d1T;
    fp.d2T = s->d2T;
    fp.a1Tlo = s->a1Tlo;
    fp.d1Tlo = s->d1Tlo;
    fp.d2Tlo = s->d2Tlo;
    fp.ll_part = c.ll_part;
    fp.ll_slots = c.ll_slots;
    if (const char* e = std::getenv("DASMC_DEBUG_EPI")) fp.dbg = std::atoi(e);  // profiling only
    // classes padded to a multiple of 4 (float4 rows of W2^T in shared memory)
    const int CP = (C + 3) / 4 * 4;
    const size_t epi_bytes =
        sizeof(float) * ((size_t)n1 * CP + ((n1 + 3) & ~3) + CP + kParts * 128 * CP) + 8 * sizeof(double) + 16 +
        (s->split || !kUseTmaStore ? 0 : 128 + (size_t)kEpiWarps * 4096);  // TMA-store staging
    if (!s->split && kUseTmaStore) {
      fp.mapS1 = map_store(s->a1T, M, n1, ldm, J, (uint64_t)(n1 + 1) * ldm);
      fp.mapS2 = map_store(s->d1T, M, n1, ldm, J, (uint64_t)n1 * ldm);
    }
    DwParams dp{};
    const int NP = tp.nmma;
    if (s->mma_layer2) {
      // layer 2 on warp-level mma.sync (split-tf32) inside the epilogue
      const size_t mma_bytes = sizeof(float) * ((size_t)NP * 24 + NP + 16 + (size_t)kParts * 128 * 20 +
                                                (size_t)kEpiWarps * 32 * 20) +
                               8 * sizeof(double) + 64;
      if (s->split)
        launch_tc<kEpiKindFwdMma, true, false, 4>(c, A, Alo, B, Blo, tp, fp, dp, mma_bytes);
      else
        launch_tc<kEpiKindFwdMma, false, false, 4>(c, A, Alo, B, Blo, tp, fp, dp, mma_bytes);
    } else if (s->tc_layer2 && NP + 32 <= 256) {
      // layer 2 on the tensor core (A1 / delta2 as TMEM A operands)
      const size_t tc_bytes = 1024 + (size_t)((NP + 31) / 32) * 2048 + (size_t)NP * 128 + (size_t)NP * 4 + 64 +
                              8 * sizeof(double) + 16;
      if (s->split)
        launch_tc<kEpiKindFwdTc, true, false, 4>(c, A, Alo, B, Blo, tp, fp, dp, tc_bytes);
      else
        launch_tc<kEpiKindFwdTc, false, false, 4>(c, A, Alo, B, Blo, tp, fp, dp, tc_bytes);
    } else {
    auto go = [&](auto cp) {
      constexpr int K = decltype(cp)::value;
      if (s->split)
        launch_tc<kEpiKindFwd, true, false, K>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
      else
        launch_tc<kEpiKindFwd, false, false, K>(c, A, Alo, B, Blo, tp, fp, dp, epi_bytes);
    };
    switch (CP) {
      case 4: go(std::integral_constant<int, 4>{}); break;
      case 8: go(std::integral_constant<int, 8>{}); break;
      case 12: go(std::integral_constant<int, 12>{}); break;
      default: go(std::integral_constant<int, 16>{}); break;
    }
    }
  }
  if (!need_grad) return;
  FwdParams fp0{};
  // ---- layer 2: dW2^T[o, c] = sum_m a1^T[o, m] delta2^T[c, m]  (ones row o = n1 -> db2)
  {
    const CUtensorMap A = map3d(s->a1T, M, n1 + 1, ldm, J, (uint64_t)(n1 + 1) * ldm, BM);
    const CUtensorMap Alo = s->split ? map3d(s->a1Tlo, M, n1 + 1, ldm, J, (uint64_t)(n1 + 1) * ldm, BM) : A;
    const CUtensorMap B = map3d(s->d2T, M, C, ldm, J, (uint64_t)C * ldm, C);
    const CUtensorMap Blo = s->split ? map3d(s->d2Tlo, M, C, ldm, J, (uint64_t)C * ldm, C) : B;
    TileParams tp{};
    tp.rtiles = (n1 + 1 + BM - 1) / BM;
    tp.J = (int)J;
    tp.rg = tp.rtiles;
    tp.nkb = (int)((M + BK - 1) / BK);
    tp.nmma = round16(C);
    tp.brows = C;
    DwParams dp{*epi, net.Dp, l2.woff, l2.boff, n1, C};
    if (s->split)
      launch_tc<kEpiKindDw, true, true>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
    else
      launch_tc<kEpiKindDw, false, true>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
  }
  // ---- layer 1: dW1^T[i, o] = sum_m X^T[i, m] delta1^T[o, m]  (ones row i = n0 -> db1)
  {
    KTimer kt(c, 1);
    const CUtensorMap A = map2d(s->Xt, M, n0 + 1, s->n_pad, BM);
    const CUtensorMap Alo = s->split ? map2d(s->Xtlo, M, n0 + 1, s->n_pad, BM) : A;
    const CUtensorMap B = map3d(s->d1T, M, n1, ldm, J, (uint64_t)n1 * ldm, n1);
    const CUtensorMap Blo = s->split ? map3d(s->d1Tlo, M, n1, ldm, J, (uint64_t)n1 * ldm, n1) : B;
    TileParams tp{};
    tp.rtiles = (n0 + 1 + BM - 1) / BM;
    tp.J = (int)J;
    tp.rg = tp.rtiles;
    tp.nkb = (int)((M + BK - 1) / BK);
    tp.nmma = round16(n1);
    tp.brows = n1;
    DwParams dp{*epi, net.Dp, l1.woff, l1.boff, n0, n1};
    if (s->split)
      launch_tc<kEpiKindDw, true, false>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
    else
      launch_tc<kEpiKindDw, false, false>(c, A, Alo, B, Blo, tp, fp0, dp, 0);
  }
}

}  // namespace dasmc_b200
