// Device context of the B200 SMC hot path: HBM layout, buffers, launch helpers.
//
// HBM layout:
//  * X   [n x n0]            fp32 row-major, the run's shuffled order; window = rows [0, M)
//  * Xt  [(n0+1) x n_pad]    fp32, X transposed plus an all-ones row (tensor-core dW1 operand)
//  * y   [n]                 int32
//  * theta[3] [Jmax x Dp]    fp32 particle-major; per layer W_l row-major [out][in]
//                            (K-major for the forward GEMM) then b_l, each segment
//                            16-byte aligned; the reference layout (W column-major)
//                            is converted at the C-ABI boundary only.
//                            Buffers rotate: start / trajectory / spare.
//  * p   [Jmax x Dp]         fp32 momenta
//  * act[l] [Jmax x Mcap x n_l] fp32 hidden activations, overwritten in place by
//                            the backward deltas; act[L] holds logits -> delta_L
//  * per-particle fp64 partial-sum slots, reduced in a fixed order (deterministic)
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dasmc_gpu.h"

namespace dasmc_b200 {

struct CudaError {
  std::string msg;
};
void cuda_check(cudaError_t e, const char* what);
#define CK(x) ::dasmc_b200::cuda_check((x), #x)

// Every kernel launch of the library is counted (bench.py's gpu_launches claim).
extern std::atomic<long long> g_launch_count;
#define LAUNCHED()                             \
  do {                                         \
    CK(cudaGetLastError());                    \
    ::dasmc_b200::g_launch_count.fetch_add(1); \
  } while (0)

// Optional CUDA-event timing of kernel ranges on the context stream
// (bench.py's live roofline): kind 0 = layer-1 forward GEMM, 1 = layer-1
// weight-gradient GEMM (+ fused leapfrog), 2 = whole gradient evaluation.
constexpr int kTimerKinds = 3;

constexpr int kMaxLayers = 8;
// Function attributes (dynamic shared memory opt-in) are per device: kernels keep one
// "already set" flag per device ordinal (multi-GPU groups drive several devices).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : kMaxDevices - 1;
}
constexpr int kMaxConv = 6;

struct LayerDev {
  int in, out;
  int64_t woff, boff;  // internal offsets (floats) of W_l [out][in] and b_l
  int64_t ref_off;     // reference offset of layer l's block (W column-major, then b)
  int hidden;          // 1 if the activation applies after this layer
  int nb;              // biases in the block (= out; cout for a conv block)
};

// [EXT] CNN stage (dasmc_gpu.h): valid stride-1 convolution + activation (+ 2x2 pool).
struct ConvDev {
  int cin, hin, win, k, cout, ho, wo, sh, sw, pool;  // sh x sw: stage output (after the pool)
  int64_t woff, boff;  // W[cout][cin][k][k] (same order as the reference layout), b[cout]
};

struct NetDev {
  int L;  // number of (fully connected) weight layers
  int act;
  int sizes[kMaxLayers + 1];
  LayerDev layer[kMaxLayers];
  int nconv;  // CNN front stages (0 for an MLP); sizes[0] = flatten size
  int in_c, in_h, in_w;
  ConvDev conv[kMaxConv];
  // every parameter block in reference order, for the reference <-> internal index
  // walks: MLP layers map W column-major -> row-major; a conv block is described as
  // a 1 x (cout*cin*k*k) "layer" so the same walk is the identity on it
  int nseg;
  LayerDev seg[kMaxLayers + kMaxConv];
  int64_t D;   // reference parameter count
  int64_t Dp;  // internal padded particle stride (floats)
};

// Phases of the leapfrog epilogue fused into the gradient kernels
// (kernels.hpp:85-96).
enum EpiMode : int {
  kEpiStoreGrad = 0,  // write the log-target gradient (parity hook)
  kEpiFirst = 1,      // s = 0: p += h/2 g ; theta_out = theta + h p
  kEpiMid = 2,        // 0 < s < S: p += h/2 g ; p += h/2 g ; theta_out = theta + h p
  kEpiLast = 3,       // s = S: p += h/2 g
  kEpiFirstLast = 4,  // S = 0 never happens; reserved
};

// Per-step scalars the step's kernels read from device memory (written by the step's first
// kernel), so a captured CUDA graph of smc_step replays unchanged across iterations: only that
// first node's by-value argument is updated per launch.
struct DevStep {
  int k;          // ensemble iteration (RNG forks, the record)
  int slot;       // record ring slot
  uint64_t ukey;  // root.fork(kResample, k) (smc.hpp:152)
};

constexpr int kSigLen = 24;
struct GraphEntry {  // one instantiated smc_step graph (capi.cu smc_step_graphed)
  int64_t sig[kSigLen];
  cudaGraphExec_t exec;
  cudaGraphNode_t node;  // the set_step kernel node (its by-value DevStep is updated per launch)
  cudaKernelNodeParams params;
  int start_after;
  long long launches;
};

struct EpiParams {
  int mode;
  float h, hh;     // step size, half step
  float inv_var;   // 1 / sigma^2
  float scale;     // N/M (scaled) or 1 (sda)
  const float* theta_in;
  float* theta_out;
  float* p;
  float* grad_out;       // kEpiStoreGrad
  double* th_part;       // [J][slots] sum theta_in^2
  double* p_part;        // [J][slots] sum p_final^2 (kEpiLast only)
  int* flags;            // [J] divergence flags
  int slots;             // slots per particle
  float* grad_cache;     // kEpiLast: also store the final-position gradient (start-gradient cache)
  // window evaluated in row chunks (CNN stages, memory independent of M): the data gradient
  // is summed over the chunks in order in gacc[J][Dp] (fp32) before the move.
  // acc_mode 0: one chunk (apply directly); 1: first chunk (store); 2: middle (add);
  // 3: last chunk (add, then apply)
  int acc_mode;
  float* gacc;
};

struct Ctx {
  NetDev net;
  int device = 0;
  int precision = DASMC_PREC_FP32;
  int64_t n = 0;
  int Jmax = 0;
  int64_t n_pad = 0;
  cudaStream_t stream = nullptr;

  // target
  int64_t prefix_end = 0, block_end = 0, total_n = 0;
  int mode = DASMC_SCALED;
  double beta = 1.0, sigma = 1.0;

  // data: X / y are the ACTIVE rows the target reads (the resident set, or a gathered
  // redraw batch in Xg / yg -- runner.hpp:531-556)
  float* X = nullptr;
  float* Xt = nullptr;
  int32_t* y = nullptr;
  float* X_full = nullptr;
  int32_t* y_full = nullptr;
  float* Xg = nullptr;
  int32_t* yg = nullptr;
  int64_t* rows_dev = nullptr;
  int64_t n_active = 0;  // rows of the active data

  // ensemble
  float* theta[3] = {nullptr, nullptr, nullptr};
  int start = 0;  // index of the ensemble's current positions
  float* p = nullptr;
  float* grad = nullptr;  // parity hook only (lazy)
  double* logw = nullptr;
  int64_t J = 0;
  int iteration = 0;
  bool has_ensemble = false;

  // activations
  int64_t Mcap = 0;
  float* act[kMaxLayers + 1] = {};
  // [EXT] CNN stages: cact = post-activation (pre-pool) [Jmax][Mcap][cout*ho*wo]; cpool =
  // pooled stage output; cdel = pre-activation delta of a pooled stage.  Backward
  // deltas of the stage outputs overwrite the outputs in place (as act[] does).
  float* cact[kMaxConv] = {};
  float* cpool[kMaxConv] = {};
  float* cdel[kMaxConv] = {};
  float* dT = nullptr;  // delta_1 transposed [J][n1][Mcap] (tensor-core dW1 operand)

  // per-particle scratch
  int ll_slots = 0, th_slots = 0, rng_slots = 0;
  double* ll_part = nullptr;   // [J][ll_slots][2]
  double* th_part = nullptr;   // [J][th_slots]
  double* p_part = nullptr;    // [J][th_slots]
  double* p0_part = nullptr;   // [J][rng_slots]
  double* p0_sum = nullptr;    // [J] fixed-order sums of p0_part / p_part (slot_sum_kernel)
  double* pS_sum = nullptr;
  int* flags = nullptr;        // [J]
  double* lt_old = nullptr;    // [J]
  double* lt_new = nullptr;    // [J]
  double* ll_pre = nullptr;    // [J] (forward-only passes; the step's last evaluation)
  double* ll_blk = nullptr;    // [J]
  // SDA moments fused into the step: unscaled (prefix, block) ll of the
  // step's first evaluation (the kept positions of divergent particles) and of the
  // post-step, post-resample ensemble, valid for window (step_P, step_M) until the
  // ensemble changes another way
  double* ll_pre0 = nullptr;
  double* ll_blk0 = nullptr;
  double* sda_pre = nullptr;
  double* sda_blk = nullptr;
  bool step_parts_valid = false;
  bool force_moment_pass = false;  // DASMC_SDA_MOMENT_PASS=1: always recompute (tests / A-B)
  // start-gradient cache: with an unchanged target the next
  // step's start positions are this step's (gathered) final positions, whose log target and
  // gradient the last leapfrog evaluation already produced; opt-in (dasmc_gpu_set_cache_start)
  bool cache_start = false, cache_valid = false;
  float* gcache[2] = {nullptr, nullptr};
  int gcur = 0;
  double* lt_cache = nullptr;
  int64_t cache_sig[4] = {0, 0, 0, 0};
  double cache_sigd[3] = {0, 0, 0};
  const float* cache_X = nullptr;
  bool last_step_cached = false;
  int64_t step_P = -1, step_M = -1;
  double* wts = nullptr;       // [J] normalised weights of the last step
  double* cdf = nullptr;       // [J]
  double* uni = nullptr;       // [J] resample uniforms
  int32_t* idx = nullptr;      // [J]
  double* records = nullptr;   // [kRecRing][8] device-side iteration records
  double* h_records = nullptr; // pinned mirror
  int rec_head = 0;            // number of queued records
  uint64_t* jump_tab = nullptr;  // [nchunks][4]
  int64_t jump_chunks = 0;
  int64_t rng_chunk = 1024;  // normals per RNG thread (set in create_ctx)

  // staging
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void* h_stage = nullptr;  // pinned
  size_t h_stage_bytes = 0;

  // events for sampler_ms
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // host <-> device ensemble transfers: DMA on `copy` in kXferChunks particle chunks,
  // overlapped with the layout conversion of the neighbouring chunk on `stream`
  cudaStream_t copy = nullptr;
  cudaEvent_t xfer_ev[9] = {};  // one per chunk + the start of a transfer

  // sharded-ensemble scratch (full-J vectors + row lists)
  double* sh_buf = nullptr;  // [5][sh_cap]: log_w, log_target_new, w, cdf, uniforms
  int32_t* sh_idx = nullptr; // [sh_cap]
  int64_t sh_cap = 0;
  int32_t* sh_rows = nullptr;
  int64_t sh_rows_cap = 0;
  int32_t* iota = nullptr;   // [Jmax] identity indices

  // tensor-core path state (tc_gemm.cu), null on the fp32 CUDA-core path
  struct TcState* tc = nullptr;
  // [EXT] CNN stages on the tensor cores (conv_tc.cu), null on the fp32 CUDA-core path
  struct ConvTcState* ctc = nullptr;
  float* gacc = nullptr;  // [Jmax][Dp] data-gradient sums across window chunks (EpiParams::acc_mode)
  int64_t cnn_ll_slots = 0;

  // CUDA-graph replay of smc_step (dasmc_gpu_set_graphs): one instantiated graph per step
  // signature (buffer rotation, target, kernel config, allocations)
  DevStep* dstep = nullptr;
  bool use_graphs = false, capturing = false;
  long long alloc_epoch = 0;  // bumped by every reallocation a captured graph could reference
  struct GraphEntry* graphs = nullptr;
  int n_graphs = 0;
  int64_t seen_sig[kSigLen] = {};
  bool seen_valid = false;

  // kernel-range timers
  bool ktime = false;
  std::vector<cudaEvent_t> kev[kTimerKinds];
  int kev_used[kTimerKinds] = {};
  double kms[kTimerKinds] = {};
  long long kcount[kTimerKinds] = {};
};

// Brackets a range of launches with an event pair when c.ktime is set.
struct KTimer {
  Ctx& c;
  int kind;
  KTimer(Ctx& cc, int k);
  ~KTimer();
};
void harvest_timers(Ctx& c);

constexpr int kRecRing = 4096;
constexpr int kRngChunkNormals = 1024;  // normals per RNG thread (2048 xoshiro draws)

// ---- launchers (kernels.cu) --------------------------------------------------------------
void ensure_activation_capacity(Ctx& c, int64_t M);
void ensure_stage(Ctx& c, size_t bytes);
void launch_forward_logits(Ctx& c, const float* theta, int64_t J, const float* Xd, const int32_t* yd, int64_t R,
                           float* logits, float* scratch0, float* scratch1);
void launch_predictive_mix(Ctx& c, const float* logits, int64_t R, int64_t J, const double* w, double* pred);
void ensure_host_stage(Ctx& c, size_t bytes);

// One forward pass (+ optional backward with the fused epilogue) over window
// rows [0, M), P = prefix_end, for particles [0, J) read from theta_in.
void launch_eval(Ctx& c, const float* theta_in, int64_t J, int64_t M, int64_t P, double beta_rows,
                 bool need_grad, const EpiParams* epi);
// Reduce the per-particle slots of the last eval: values (fp64 log target),
// optionally the unscaled prefix/block log-likelihoods.
void launch_eval_finalize(Ctx& c, int64_t J, double* values_out, double* pre_out, double* blk_out, int64_t M,
                          bool with_theta_norm);
void launch_normals(Ctx& c, uint64_t key_root, uint64_t tag_a, uint64_t a2, int64_t J, float scale, float* dst,
                    double* sq_part, int64_t j_offset = 0, const DevStep* ds = nullptr);
void launch_set_step(Ctx& c, const DevStep& v);
const void* set_step_kernel_fn();  // the set_step kernel (graph node lookup)
void launch_ref_to_internal_f64(Ctx& c, const double* src, float* dst, int64_t J);
void launch_ref_to_internal_f32(Ctx& c, const float* src, float* dst, int64_t J);
void launch_internal_to_ref_f64(Ctx& c, const float* src, double* dst, int64_t J);
void launch_internal_to_ref_f32(Ctx& c, const float* src, float* dst, int64_t J);
void launch_zero_ints(Ctx& c, int* p, int64_t n);
void launch_p_sumsq(Ctx& c, int64_t J);
void launch_uniforms(Ctx& c, uint64_t key, int64_t count, double* dst, const DevStep* ds = nullptr);
void launch_weights_and_resample(Ctx& c, int64_t J, double fraction, int always, int kind, int rec_slot,
                                 int k, double log_target_const, const DevStep* ds = nullptr);
void launch_gather(Ctx& c, const float* start, const float* end, float* dst, int64_t J,
                   const int32_t* idx = nullptr);
// post-step (prefix, block) ll: (flags[s] ? first-evaluation : last-evaluation)[s], s = idx[j]
void launch_gather_parts(Ctx& c, int64_t J);
// out[j] = (flags[s] ? first-evaluation : last-evaluation) (prefix, block) ll, s = idx[j]
void launch_select_parts(Ctx& c, int64_t J, const int32_t* idx, double* out_pre, double* out_blk);
// start-gradient cache: p += h/2 g_cached, theta_out = theta + h p (kernels.hpp:89-91), flags
void launch_start_from_cache(Ctx& c, const EpiParams& e, int64_t J);
// rows dst[j] = src[idx[j]] of Dp floats, and lt_cache[j] = lt_new[idx[j]]
void launch_gather_cache(Ctx& c, const float* src, float* dst, int64_t J);
void launch_local_weights(Ctx& c, int64_t J, double* out_lw, double* out_lt);
void launch_normalize_resample(Ctx& c, int64_t Jtot, double* lw_full, const double* lt_full, double* w, double* cdf,
                               const double* uni, int32_t* idx, double fraction, int always, int kind, int rec_slot,
                               int k);
void launch_rows(Ctx& c, const float* src, float* dst, const int32_t* rows_dev, int64_t n, bool pack);
// dst rows i = src rows rows[i] (data rows of d floats + labels): the redraw gather
void launch_gather_data(Ctx& c, const float* X, const int32_t* y, const int64_t* rows, int64_t count, int64_t d,
                        float* Xd, int32_t* yd);
void launch_resample_hook(Ctx& c, const double* w, const double* u, int64_t J, int kind, int32_t* idx);

}  // namespace dasmc_b200
