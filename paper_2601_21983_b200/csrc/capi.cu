// C-ABI implementation and host driver of the B200 SMC hot path
// (include/dasmc_gpu.h).  The driver owns the SMC loop (runner.hpp:581-604),
// the annealing schedules and the SDA controller (annealing.hpp), and queues
// every per-iteration kernel on one CUDA stream without host synchronisation
// except where the reference's control flow needs a device result on the
// host (SDA moments; a record the caller asked for).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "host.h"
#include "tc_gemm.cuh"
#include "conv_tc.cuh"

namespace dasmc_b200 {
struct MultiState;
}
struct dasmc_ctx {
  dasmc_b200::Ctx c;
  dasmc_b200::MultiState* multi = nullptr;  // single-process multi-GPU group (dasmc_gpu_create_multi)
};

namespace dasmc_b200 {

namespace {
thread_local std::string g_err;
}
void set_last_error(const std::string& m) { g_err = m; }

namespace {

struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Dead : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return DASMC_OK;
  } catch (const Dead& e) {
    g_err = e.what();
    return DASMC_EDEAD;
  } catch (const CudaError& e) {
    g_err = e.msg;
    return DASMC_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DASMC_EINVAL;
  }
}

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

NetDev make_net(const dasmc_net_desc* d) {
  if (d == nullptr || d->layer_sizes == nullptr) throw InvalidArg("net: null descriptor");
  if (d->num_layers < 2) throw InvalidArg("NetSpec: need at least input and output layers");
  if (d->num_layers - 1 > kMaxLayers) throw InvalidArg("NetSpec: too many layers for this build");
  for (int i = 0; i < d->num_layers; ++i)
    if (d->layer_sizes[i] < 1) throw InvalidArg("NetSpec: layer sizes must be >= 1");
  if (d->activation != DASMC_RELU && d->activation != DASMC_TANH) throw InvalidArg("NetSpec: bad activation");
  NetDev n{};
  n.L = d->num_layers - 1;
  n.act = d->activation;
  for (int i = 0; i < d->num_layers; ++i) n.sizes[i] = d->layer_sizes[i];
  int64_t ref = 0, off = 0;
  if (d->conv != nullptr) {  // [EXT] CNN front (dasmc_gpu.h)
    const int* cv = d->conv;
    n.in_c = cv[0];
    n.in_h = cv[1];
    n.in_w = cv[2];
    n.nconv = cv[3];
    if (n.in_c < 1 || n.in_h < 1 || n.in_w < 1) throw InvalidArg("CnnSpec: bad input shape");
    if (n.nconv < 1 || n.nconv > kMaxConv) throw InvalidArg("CnnSpec: 1..6 convolution stages supported");
    int ch = n.in_c, h = n.in_h, w = n.in_w;
    for (int i = 0; i < n.nconv; ++i) {
      ConvDev& c = n.conv[i];
      c.cin = ch;
      c.hin = h;
      c.win = w;
      c.k = cv[4 + 3 * i];
      c.cout = cv[5 + 3 * i];
      c.pool = cv[6 + 3 * i] != 0 ? 1 : 0;
      c.ho = h - c.k + 1;
      c.wo = w - c.k + 1;
      c.sh = c.pool ? c.ho / 2 : c.ho;
      c.sw = c.pool ? c.wo / 2 : c.wo;
      if (c.k < 1 || c.cout < 1 || c.ho < 1 || c.wo < 1 || c.sh < 1 || c.sw < 1)
        throw InvalidArg("CnnSpec: convolution does not fit its input");
      // reference and internal layouts coincide on a conv block: W[cout][cin][k][k], b[cout]
      LayerDev& sg = n.seg[n.nseg++];
      sg.out = 1;
      sg.in = c.cout * c.cin * c.k * c.k;
      sg.nb = c.cout;
      sg.ref_off = ref;
      ref += (int64_t)sg.in + sg.nb;
      c.woff = sg.woff = off;
      off = align_up(off + sg.in, 32);
      c.boff = sg.boff = off;
      off = align_up(off + sg.nb, 32);
      ch = c.cout;
      h = c.sh;
      w = c.sw;
    }
    if ((int64_t)ch * h * w != n.sizes[0]) throw InvalidArg("CnnSpec: head input size must equal the flatten size");
  }
  for (int l = 0; l < n.L; ++l) {
    LayerDev& ly = n.layer[l];
    ly.in = n.sizes[l];
    ly.out = n.sizes[l + 1];
    ly.nb = ly.out;
    ly.ref_off = ref;
    ref += (int64_t)ly.in * ly.out + ly.out;
    ly.woff = off;
    off = align_up(off + (int64_t)ly.in * ly.out, 32);
    ly.boff = off;
    off = align_up(off + ly.out, 32);
    ly.hidden = l + 1 < n.L ? 1 : 0;
    n.seg[n.nseg++] = ly;
  }
  n.D = ref;
  n.Dp = align_up(off, 32);
  return n;
}

// floats per input row: the MLP input or the CNN image
int64_t input_floats(const NetDev& n) { return n.nconv > 0 ? (int64_t)n.in_c * n.in_h * n.in_w : n.sizes[0]; }

void graphs_free(Ctx& c);

void free_ctx(Ctx& c) {
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  graphs_free(c);
  tc_free(c);
  cnn_tc_free(c);
  if (c.gacc) cudaFree(c.gacc);
  void* ptrs[] = {c.X_full, c.Xt, c.y_full, c.Xg, c.yg, c.rows_dev, c.gcache[0], c.gcache[1], c.lt_cache, c.theta[0], c.theta[1], c.theta[2], c.p, c.grad, c.logw, c.dT, c.ll_part,
                  c.th_part, c.p_part, c.p0_part, c.p0_sum, c.pS_sum, c.flags, c.lt_old, c.lt_new, c.ll_pre, c.ll_blk, c.ll_pre0, c.ll_blk0,
                  c.sda_pre, c.sda_blk, c.wts, c.cdf,
                  c.uni, c.idx, c.records, c.jump_tab, c.stage, c.sh_buf, c.sh_idx, c.sh_rows, c.iota, c.dstep};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int l = 0; l <= kMaxLayers; ++l)
    if (c.act[l]) cudaFree(c.act[l]);
  for (int i = 0; i < kMaxConv; ++i) {
    if (c.cact[i]) cudaFree(c.cact[i]);
    if (c.cpool[i]) cudaFree(c.cpool[i]);
    if (c.cdel[i]) cudaFree(c.cdel[i]);
  }
  if (c.h_records) cudaFreeHost(c.h_records);
  if (c.h_stage) cudaFreeHost(c.h_stage);
  if (c.copy) {
    cudaStreamSynchronize(c.copy);
    cudaStreamDestroy(c.copy);
    for (cudaEvent_t e : c.xfer_ev)
      if (e) cudaEventDestroy(e);
  }
  if (c.ev0) cudaEventDestroy(c.ev0);
  if (c.ev1) cudaEventDestroy(c.ev1);
  if (c.stream) cudaStreamDestroy(c.stream);
}

template <typename T>
void dmalloc(T*& p, size_t count) {
  CK(cudaMalloc(reinterpret_cast<void**>(&p), sizeof(T) * std::max<size_t>(count, 1)));
}

void validate_target(const Ctx& c) {  // target.hpp:104-113
  if (!(c.sigma > 0.0)) throw InvalidArg("PriorSpec: sigma must be > 0");
  if (c.prefix_end < 0 || c.prefix_end > c.block_end || c.block_end > c.total_n)
    throw InvalidArg("SubsetWindow: need 0 <= prefix_end <= block_end <= total_n");
  if (c.block_end < 1) throw InvalidArg("TargetContext: empty subset");
  if (c.block_end > c.n_active) throw InvalidArg("TargetContext: window exceeds dataset");
  if (c.mode == DASMC_SDA && !(c.beta > 0.0 && c.beta <= 1.0))
    throw InvalidArg("TargetContext: sda mode needs beta in (0, 1]");
  if (c.mode != DASMC_SCALED && c.mode != DASMC_SDA) throw InvalidArg("TargetContext: bad mode");
}

void check_J(const Ctx& c, int64_t J) {
  if (J < 1 || J > c.Jmax) throw InvalidArg("particle count out of range for this context");
}

// Window rows and their tempering for the current target: scaled mode puts
// every row in the "prefix" with weight 1; SDA weights block rows by beta.
void target_rows(const Ctx& c, int64_t& M, int64_t& P, double& beta_rows) {
  M = c.block_end;
  if (c.mode == DASMC_SCALED) {
    P = M;
    beta_rows = 1.0;
  } else {
    P = c.prefix_end;
    beta_rows = c.beta;
  }
}

EpiParams make_epi(Ctx& c, int mode, double h, const float* th_in, float* th_out) {
  EpiParams e{};
  e.mode = mode;
  e.h = (float)h;
  e.hh = (float)(0.5 * h);
  e.inv_var = (float)(1.0 / (c.sigma * c.sigma));
  e.scale = c.mode == DASMC_SCALED ? (float)((double)c.total_n / (double)c.block_end) : 1.0f;
  e.theta_in = th_in;
  e.theta_out = th_out;
  e.p = c.p;
  e.grad_out = c.grad;
  e.flags = c.flags;
  return e;
}

void upload(Ctx& c, void* dst, const void* src, size_t bytes) {
  ensure_host_stage(c, bytes);
  std::memcpy(c.h_stage, src, bytes);
  CK(cudaMemcpyAsync(dst, c.h_stage, bytes, cudaMemcpyHostToDevice, c.stream));
  CK(cudaStreamSynchronize(c.stream));
}

void download(Ctx& c, void* dst, const void* src, size_t bytes) {
  ensure_host_stage(c, bytes);
  CK(cudaMemcpyAsync(c.h_stage, src, bytes, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  std::memcpy(dst, c.h_stage, bytes);
}

void check_kernel_cfg(const dasmc_kernel_cfg& kc) {  // kernels.hpp:42-48
  if (!(kc.step_size > 0.0)) throw InvalidArg("KernelConfig: step_size must be > 0");
  if (kc.leapfrog_steps < 1) throw InvalidArg("KernelConfig: leapfrog_steps must be >= 1");
  if (kc.kind == DASMC_LANGEVIN && kc.leapfrog_steps != 1)
    throw InvalidArg("KernelConfig: langevin requires leapfrog_steps == 1");
}

int64_t cache_sig_of(const Ctx& c, int i) {
  const int64_t v[4] = {c.mode, c.prefix_end, c.block_end, c.total_n};
  return v[i];
}
bool cache_signature_matches(const Ctx& c) {
  for (int i = 0; i < 4; ++i)
    if (c.cache_sig[i] != cache_sig_of(c, i)) return false;
  return c.cache_sigd[0] == c.beta && c.cache_sigd[1] == c.sigma && c.cache_X == c.X && c.cache_sigd[2] == (double)c.J;
}
void cache_signature_store(Ctx& c) {
  for (int i = 0; i < 4; ++i) c.cache_sig[i] = cache_sig_of(c, i);
  c.cache_sigd[0] = c.beta;
  c.cache_sigd[1] = c.sigma;
  c.cache_sigd[2] = (double)c.J;
  c.cache_X = c.X;
}

// Fresh momenta + S-step leapfrog + log targets of the context's particles
// (smc.hpp:118-122, kernels.hpp:75-99).  Global slot of local particle j is
// j_offset + j (RNG streams).  Returns the buffer index (relative to c.start)
// holding theta_S.
int propose_async(Ctx& c, const dasmc_kernel_cfg& kc, uint64_t seed, int64_t j_offset, const DevStep* ds = nullptr) {
  check_kernel_cfg(kc);
  if (!c.has_ensemble) throw InvalidArg("smc_step: no ensemble (call init_ensemble or set_ensemble)");
  validate_target(c);
  const int64_t J = c.J;
  const int k = c.iteration;
  const int S = kc.leapfrog_steps;
  int64_t M, P;
  double br;
  target_rows(c, M, P, br);
  launch_zero_ints(c, c.flags, J);
  // fresh momenta p0 ~ N(0, I) from root.fork(kProposal, k, j) (smc.hpp:119-120; kernels.hpp:131)
  launch_normals(c, seed, tag::kProposal, (uint64_t)k, J, 1.0f, c.p, c.p0_part, j_offset, ds);
  const int t0 = c.start, t1 = (c.start + 1) % 3, t2 = (c.start + 2) % 3;
  float* bufs[3] = {c.theta[t0], c.theta[t1], c.theta[t2]};
  int in_idx = 0;
  // start-gradient cache: same target as the step that produced the cached final positions
  const bool use_cache = c.cache_start && c.cache_valid && j_offset == 0 && cache_signature_matches(c);
  c.last_step_cached = use_cache;
  for (int s = 0; s <= S; ++s) {
    const int out_idx = (s % 2 == 0) ? 1 : 2;
    const int mode = s == 0 ? kEpiFirst : (s < S ? kEpiMid : kEpiLast);
    EpiParams e = make_epi(c, mode, kc.step_size, bufs[in_idx], s < S ? bufs[out_idx] : nullptr);
    if (s == 0 && use_cache) {  // p += h/2 g(theta_0), theta_1 = theta_0 + h p; lt_old = cached
      launch_start_from_cache(c, e, J);
      in_idx = out_idx;
      continue;
    }
    if (s == S && c.cache_start) e.grad_cache = c.gcache[c.gcur ^ 1];
    launch_eval(c, bufs[in_idx], J, M, P, br, true, &e);
    // unscaled (prefix, block) ll of the first and last evaluations feed the fused SDA moments
    launch_eval_finalize(c, J, s == 0 ? c.lt_old : c.lt_new, s == 0 ? c.ll_pre0 : (s == S ? c.ll_pre : nullptr),
                         s == 0 ? c.ll_blk0 : (s == S ? c.ll_blk : nullptr), M, true);
    if (s < S) in_idx = out_idx;
  }
  launch_p_sumsq(c, J);
  return in_idx;
}

// One proposal + reweight + (conditional) resample of the whole ensemble
// (smc.hpp:109-158).  Asynchronous: the record lands in c.records[slot].
void smc_step_async(Ctx& c, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction, int always,
                    int slot) {
  if (rkind != DASMC_MULTINOMIAL && rkind != DASMC_SYSTEMATIC) throw InvalidArg("bad resample kind");
  const int64_t J = c.J;
  const int k = c.iteration;
  const int t1 = (c.start + 1) % 3, t2 = (c.start + 2) % 3;
  float* bufs[3] = {c.theta[c.start], c.theta[t1], c.theta[t2]};
  // the step's scalars (iteration, record slot, resampling stream key) go to device memory
  // first, so a captured graph of this sequence replays with only that argument changed
  const DevStep ds{k, slot, fork_key(seed, tag::kResample, (uint64_t)k, 0)};
  launch_set_step(c, ds);
  const int end_idx = propose_async(c, kc, seed, 0, c.dstep);  // theta_S
  // resampling uniforms from root.fork(kResample, k) (smc.hpp:152)
  launch_uniforms(c, ds.ukey, rkind == DASMC_MULTINOMIAL ? J : 1, c.uni, c.dstep);
  launch_weights_and_resample(c, J, fraction, always, rkind, slot, k, 0.0, c.dstep);
  const int dst_idx = end_idx == 1 ? 2 : 1;  // the free trajectory buffer
  launch_gather(c, bufs[0], bufs[end_idx], bufs[dst_idx], J);
  launch_gather_parts(c, J);  // the post-step ensemble's (prefix, block) ll, for sda_advance
  if (c.cache_start) {  // next step's start gradients / log targets = this step's final ones, resampled
    launch_gather_cache(c, c.gcache[c.gcur ^ 1], c.gcache[c.gcur], J);
    cache_signature_store(c);
  }
  c.cache_valid = false;  // confirmed by the host once the record shows no divergence
  c.step_parts_valid = true;
  c.step_P = c.mode == DASMC_SDA ? c.prefix_end : c.block_end;
  c.step_M = c.block_end;
  c.start = dst_idx == 1 ? t1 : t2;
  c.iteration = k + 1;  // smc.hpp:150, 154
}

// ---- CUDA-graph replay of smc_step (launch-bound configs, SURVEY.md §7 hard part 7) --------------
// The step's launch sequence depends on the buffer rotation, the target, the kernel
// configuration and the allocations, never on the iteration (DevStep carries that), so one
// instantiated graph per signature replays every iteration with that signature.  The first
// occurrence of a signature runs eagerly (warming lazily created state), the second captures.
constexpr int kMaxGraphs = 16;

void graphs_free(Ctx& c) {
  for (int i = 0; i < c.n_graphs; ++i) cudaGraphExecDestroy(c.graphs[i].exec);
  delete[] c.graphs;
  c.graphs = nullptr;
  c.n_graphs = 0;
  c.seen_valid = false;
}

void step_signature(const Ctx& c, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction, int always,
                    int64_t* sig) {
  auto bits = [](double v) {
    int64_t b;
    std::memcpy(&b, &v, sizeof b);
    return b;
  };
  const int64_t v[kSigLen] = {c.start, c.J, c.mode, c.prefix_end, c.block_end, c.total_n, bits(c.beta), bits(c.sigma),
                              bits(kc.step_size), kc.leapfrog_steps, kc.kind, (int64_t)seed, rkind, bits(fraction),
                              always, (int64_t)(uintptr_t)c.X, c.alloc_epoch, c.Mcap, c.ll_slots,
                              c.tc ? 1 : 0, c.n_active, c.cache_start ? 1 : 0, 0, 0};
  std::memcpy(sig, v, sizeof v);
}

GraphEntry* find_graph(Ctx& c, const int64_t* sig) {
  for (int i = 0; i < c.n_graphs; ++i)
    if (std::memcmp(c.graphs[i].sig, sig, sizeof(int64_t) * kSigLen) == 0) return &c.graphs[i];
  return nullptr;
}

void smc_step_async(Ctx& c, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction, int always,
                    int slot);

// One smc_step through the graph cache (falls back to eager launches while a signature is new).
void smc_step_graphed(Ctx& c, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction, int always,
                      int slot) {
  check_kernel_cfg(kc);
  if (!c.has_ensemble) throw InvalidArg("smc_step: no ensemble (call init_ensemble or set_ensemble)");
  validate_target(c);
  ensure_activation_capacity(c, c.block_end);  // never inside a capture
  int64_t sig[kSigLen];
  step_signature(c, kc, seed, rkind, fraction, always, sig);
  GraphEntry* e = find_graph(c, sig);
  const int k = c.iteration;
  if (!e) {
    const bool seen = c.seen_valid && std::memcmp(c.seen_sig, sig, sizeof sig) == 0;
    if (!seen || c.n_graphs >= kMaxGraphs) {
      std::memcpy(c.seen_sig, sig, sizeof sig);
      c.seen_valid = true;
      smc_step_async(c, kc, seed, rkind, fraction, always, slot);
      return;
    }
    if (!c.graphs) c.graphs = new GraphEntry[kMaxGraphs];
    const int start0 = c.start;
    const long long n0 = g_launch_count.load();
    cudaGraph_t g = nullptr;
    c.capturing = true;
    CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      smc_step_async(c, kc, seed, rkind, fraction, always, slot);
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      c.capturing = false;
      throw;
    }
    CK(cudaStreamEndCapture(c.stream, &g));
    c.capturing = false;
    GraphEntry& ne = c.graphs[c.n_graphs];
    std::memcpy(ne.sig, sig, sizeof sig);
    ne.start_after = c.start;
    ne.launches = g_launch_count.load() - n0;
    g_launch_count.fetch_sub(ne.launches);  // captured, not launched
    ne.node = nullptr;
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (cudaGraphNode_t n : nodes) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(n, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      CK(cudaGraphKernelNodeGetParams(n, &kp));
      if (kp.func == set_step_kernel_fn()) {
        ne.node = n;
        ne.params = kp;
        break;
      }
    }
    if (!ne.node) {
      cudaGraphDestroy(g);
      throw CudaError{"graph capture: step-parameter node not found"};
    }
    CK(cudaGraphInstantiate(&ne.exec, g, 0));
    CK(cudaGraphDestroy(g));  // the exec keeps its own copy; node handles stay valid for updates
    ++c.n_graphs;
    e = &ne;
    c.start = start0;  // nothing ran yet: replay below
  }
  DevStep v{k, slot, fork_key(seed, tag::kResample, (uint64_t)k, 0)};
  DevStep* dptr = c.dstep;
  void* args[2] = {&v, &dptr};
  cudaKernelNodeParams kp = e->params;
  kp.kernelParams = args;
  kp.extra = nullptr;
  CK(cudaGraphExecKernelNodeSetParams(e->exec, e->node, &kp));
  CK(cudaGraphLaunch(e->exec, c.stream));
  g_launch_count.fetch_add(e->launches);
  // the host-side effects smc_step_async has on the context
  c.last_step_cached = false;
  c.cache_valid = false;
  c.step_parts_valid = true;
  c.step_P = c.mode == DASMC_SDA ? c.prefix_end : c.block_end;
  c.step_M = c.block_end;
  c.start = e->start_after;
  c.iteration = k + 1;
}

dasmc_iter_record read_record(Ctx& c, int slot) {
  const double* r = c.h_records + (size_t)slot * 8;
  dasmc_iter_record o{};
  o.k = (int)r[0];
  o.ess = r[1];
  o.resampled = (int)r[2];
  o.mean_log_target = r[3];
  o.n_divergent = (int)r[4];
  o.beta = 1.0;
  if (r[5] != 0.0) throw Dead("normalize: all particles dead (every log-weight is -inf)");
  return o;
}

void fetch_records(Ctx& c, int first, int count) {
  CK(cudaMemcpyAsync(c.h_records + (size_t)first * 8, c.records + (size_t)first * 8, sizeof(double) * 8 * count,
                     cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
}

// Unscaled prefix / block log-likelihoods of particles under window (P, M) (target.hpp:121-129).
void loglik_parts_dev(Ctx& c, const float* theta, int64_t J, int64_t P, int64_t M) {
  launch_eval(c, theta, J, M, P, 1.0, false, nullptr);
  launch_eval_finalize(c, J, nullptr, c.ll_pre, c.ll_blk, M, false);
}

void sda_moments_dev(Ctx& c, int64_t P, int64_t M, double* out6) {  // annealing.hpp:153-174
  if (P < 0 || P > M || M > c.n) throw InvalidArg("SubsetWindow: need 0 <= prefix_end <= block_end <= total_n");
  if (M <= P) throw InvalidArg("sda_moments: window has no new block");
  const int64_t J = c.J;
  std::vector<double> pre((size_t)J), blk((size_t)J), lw((size_t)J);
  // fused: right after an SDA step on this window, the step's own last
  // evaluation (first one for divergent particles), gathered through the resample, gives the
  // post-step ensemble's ll without another forward pass; identical values to the pass
  if (c.step_parts_valid && c.step_P == P && c.step_M == M && c.X == c.X_full && !c.force_moment_pass) {
    download(c, pre.data(), c.sda_pre, sizeof(double) * J);
    download(c, blk.data(), c.sda_blk, sizeof(double) * J);
  } else {
    loglik_parts_dev(c, c.theta[c.start], J, P, M);
    download(c, pre.data(), c.ll_pre, sizeof(double) * J);
    download(c, blk.data(), c.ll_blk, sizeof(double) * J);
  }
  download(c, lw.data(), c.logw, sizeof(double) * J);
  for (int64_t j = 0; j < J; ++j) {
    pre[(size_t)j] = -pre[(size_t)j];
    blk[(size_t)j] = -blk[(size_t)j];
  }
  sda_moments_from(pre.data(), blk.data(), lw.data(), J, out6);
}

void init_ensemble_dev(Ctx& c, int64_t J, uint64_t seed, int64_t j_offset = 0) {  // smc.hpp:73-89
  if (J < 2) throw InvalidArg("init_ensemble: need at least 2 particles");
  check_J(c, J);
  validate_target(c);
  float* th = c.theta[c.start];
  // theta_j = sigma * normal_vector(D) from root.fork(kInit, j) (network.hpp:235-239)
  launch_normals(c, seed, tag::kInit, 0, J, (float)c.sigma, th, nullptr, j_offset);
  int64_t M, P;
  double br;
  target_rows(c, M, P, br);
  loglik_parts_dev(c, th, J, P, M);
  std::vector<double> pre((size_t)J), blk((size_t)J), lw((size_t)J);
  download(c, pre.data(), c.ll_pre, sizeof(double) * J);
  download(c, blk.data(), c.ll_blk, sizeof(double) * J);
  const double scale = (double)c.total_n / (double)c.block_end;
  for (int64_t j = 0; j < J; ++j)  // log_target - prior_logpdf (smc.hpp:85)
    lw[(size_t)j] = c.mode == DASMC_SCALED ? scale * pre[(size_t)j] : pre[(size_t)j] + c.beta * blk[(size_t)j];
  upload(c, c.logw, lw.data(), sizeof(double) * J);
  c.J = J;
  c.iteration = 0;
  c.has_ensemble = true;
  c.step_parts_valid = false;
  c.cache_valid = false;
}

void create_ctx(Ctx& c, const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n, int Jmax,
                int device, int precision) {
  c.net = make_net(net);
  if (const char* e = std::getenv("DASMC_SDA_MOMENT_PASS")) c.force_moment_pass = e[0] == '1';
  if (n < 1) throw InvalidArg("dataset: n must be >= 1");
  if (X == nullptr || y == nullptr) throw InvalidArg("dataset: null X or y");
  if (Jmax < 2) throw InvalidArg("max_particles must be >= 2");
  // per context: the gather / row kernels index particles by gridDim.y and the single-block weights
  // kernel walks J in shared-memory batches; larger ensembles shard over a multi-GPU group
  if (Jmax > 65535) throw InvalidArg("max_particles must be <= 65535 per context");
  if (precision != DASMC_PREC_FP32 && precision != DASMC_PREC_TF32 && precision != DASMC_PREC_3XTF32 &&
      precision != DASMC_PREC_F16 && precision != DASMC_PREC_TF32H && precision != DASMC_PREC_F16X2)
    throw InvalidArg("bad precision");
  const int C = c.net.sizes[c.net.L];
  for (int64_t i = 0; i < n; ++i)
    if (y[i] < 0 || y[i] >= C) throw InvalidArg("loglik_batch: label out of range");
  c.device = device;
  c.precision = precision;
  c.n = n;
  c.Jmax = Jmax;
  c.total_n = n;
  c.block_end = n;
  c.prefix_end = 0;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&c.ev0));
  CK(cudaEventCreate(&c.ev1));
  const int64_t n0 = input_floats(c.net);
  dmalloc(c.X, (size_t)n * n0);
  dmalloc(c.y, (size_t)n);
  CK(cudaMemcpy(c.X, X, sizeof(float) * (size_t)n * n0, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c.y, y, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice));
  c.X_full = c.X;
  c.y_full = c.y;
  c.n_active = n;
  const size_t pe = (size_t)Jmax * c.net.Dp;
  for (auto& t : c.theta) {
    dmalloc(t, pe);
    CK(cudaMemset(t, 0, sizeof(float) * pe));
  }
  dmalloc(c.p, pe);
  CK(cudaMemset(c.p, 0, sizeof(float) * pe));
  dmalloc(c.logw, (size_t)Jmax);
  c.th_slots = (int)((c.net.Dp + 8191) / 8192);
  // RNG chunk = one column of the widest layer (the reference's column-major W order
  // walks a column's rows consecutively; internally those are `in` floats apart, so
  // threads owning consecutive columns store coalesced); small nets keep 1024
  {
    int64_t widest = 0;
    for (int l = 1; l <= c.net.L; ++l) widest = std::max<int64_t>(widest, c.net.sizes[l]);
    // a few whole columns per thread: the 256-step F2 jump-ahead is paid once per ~1024 normals
    // (warp stores stay within a few 32-byte sectors per row)
    c.rng_chunk = widest >= 128 ? widest * std::max<int64_t>(1, kRngChunkNormals / widest) : kRngChunkNormals;
    // small nets (e.g. C1, D = 2410): at least ~64 chunks per particle, so there are enough
    // independent streams to fill the GPU (per-thread work is a serial chain).  A function of D
    // only: the fixed-order sums of the chunk partials do not depend on J or on the sharding
    c.rng_chunk = std::min<int64_t>(c.rng_chunk, std::max<int64_t>(16, c.net.D / 64));
  }
  const int64_t nch_rng = (c.net.D + c.rng_chunk - 1) / c.rng_chunk;
  c.rng_slots = (int)nch_rng;
  dmalloc(c.th_part, (size_t)Jmax * c.th_slots);
  dmalloc(c.p_part, (size_t)Jmax * c.th_slots);
  dmalloc(c.p0_part, (size_t)Jmax * c.rng_slots);
  dmalloc(c.p0_sum, (size_t)Jmax);
  dmalloc(c.pS_sum, (size_t)Jmax);
  dmalloc(c.flags, (size_t)Jmax);
  CK(cudaMemset(c.flags, 0, sizeof(int) * Jmax));
  dmalloc(c.lt_old, (size_t)Jmax);
  dmalloc(c.lt_new, (size_t)Jmax);
  dmalloc(c.ll_pre, (size_t)Jmax);
  dmalloc(c.ll_blk, (size_t)Jmax);
  dmalloc(c.ll_pre0, (size_t)Jmax);
  dmalloc(c.ll_blk0, (size_t)Jmax);
  dmalloc(c.sda_pre, (size_t)Jmax);
  dmalloc(c.sda_blk, (size_t)Jmax);
  dmalloc(c.wts, (size_t)Jmax);
  dmalloc(c.cdf, (size_t)Jmax);
  dmalloc(c.uni, (size_t)Jmax);
  dmalloc(c.idx, (size_t)Jmax);
  dmalloc(c.records, (size_t)kRecRing * 8);
  dmalloc(c.dstep, 1);
  {
    std::vector<int32_t> io((size_t)Jmax);
    for (int i = 0; i < Jmax; ++i) io[(size_t)i] = i;
    dmalloc(c.iota, (size_t)Jmax);
    CK(cudaMemcpy(c.iota, io.data(), sizeof(int32_t) * Jmax, cudaMemcpyHostToDevice));
  }
  CK(cudaMallocHost(reinterpret_cast<void**>(&c.h_records), sizeof(double) * kRecRing * 8));
  const int64_t nch_uni = (Jmax + 2 * c.rng_chunk - 1) / (2 * c.rng_chunk);
  c.jump_chunks = std::max(nch_rng, nch_uni) + 1;
  const auto tab = jump_table(2 * (uint64_t)c.rng_chunk, c.jump_chunks);
  dmalloc(c.jump_tab, (size_t)c.jump_chunks * 4);
  CK(cudaMemcpy(c.jump_tab, tab.data(), sizeof(uint64_t) * 4 * tab.size(), cudaMemcpyHostToDevice));
  if (precision != DASMC_PREC_FP32 && c.net.nconv > 0) {
    // [EXT] CNN: convolution stages on tcgen05 (kind::tf32 implicit GEMMs), the MLP head on CUDA cores
    if (precision != DASMC_PREC_TF32 && precision != DASMC_PREC_TF32H)
      throw InvalidArg("CNN contexts: precision fp32 (CUDA cores) or tf32 (tensor-core convolutions)");
    if (!cnn_tc_eligible(c))
      throw InvalidArg(
          "tensor-core CNN stages need cout % 4 == 0 (and cin % 4 == 0 after stage 0), cin, cout <= 64 and "
          "k * cout <= 256 (the weight-gradient GEMM's N); use precision fp32 for other stages");
    cnn_tc_init(c);
  } else if (precision != DASMC_PREC_FP32) {
    if (!tc_layer1_eligible(c))
      throw InvalidArg("tensor-core precision needs a one-hidden-layer MLP (no conv stages) with input % 4 == 0, "
                       "hidden <= 256, classes <= 16 (use DASMC_PREC_FP32)");
    tc_init(c);
  }
}

}  // namespace
}  // namespace dasmc_b200

namespace dasmc_b200 {
struct MultiState;
void multi_destroy(MultiState* m);
dasmc_ctx* multi_shard_handle(MultiState* m, int r);
void multi_set_target_api(MultiState& m, int64_t P, int64_t M, int64_t N, int mode, double beta, double sigma);
void multi_init_api(MultiState& m, int64_t J, uint64_t seed);
void multi_set_ensemble_api(MultiState& m, const void* theta, bool f32, const double* lw, int64_t J, int it);
void multi_get_ensemble_api(MultiState& m, void* theta, bool f32, double* lw, int* it);
void multi_smc_step_api(MultiState& m, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction,
                        int always, dasmc_iter_record* record);
void multi_sync_records_api(MultiState& m, dasmc_iter_record* records, int count);
void multi_sda_moments_api(MultiState& m, int64_t P, int64_t M, double* out6);
Ctx& multi_lead(MultiState& m);
}  // namespace dasmc_b200

using namespace dasmc_b200;

extern "C" {

const char* dasmc_last_error(void) { return g_err.c_str(); }

int dasmc_gpu_create(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n, int max_particles,
                     int device, int precision, dasmc_ctx** out) {
  if (out == nullptr) {
    g_err = "null out";
    return DASMC_EINVAL;
  }
  *out = nullptr;
  auto* h = new dasmc_ctx();
  const int rc = guarded([&] { create_ctx(h->c, net, X, y, n, max_particles, device, precision); });
  if (rc != DASMC_OK) {
    free_ctx(h->c);
    delete h;
    return rc;
  }
  *out = h;
  return DASMC_OK;
}

int dasmc_gpu_destroy(dasmc_ctx* ctx) {
  if (!ctx) return DASMC_OK;
  if (ctx->multi) {
    multi_destroy(ctx->multi);
    delete ctx;
    return DASMC_OK;
  }
  free_ctx(ctx->c);
  delete ctx;
  return DASMC_OK;
}

int dasmc_gpu_param_count(const dasmc_ctx* ctx) { return ctx ? (int)ctx->c.net.D : -1; }

// The target's data rows: the resident set (rows == NULL) or train[rows[0..count)] gathered
// on the device (the constant-redraw batch, runner.hpp:531-556).
void set_rows_dev(Ctx& c, const int64_t* rows, int64_t count) {
  if (rows == nullptr || count <= 0) {
    if (c.X == c.X_full) return;
    c.X = c.X_full;
    c.y = c.y_full;
    c.n_active = c.n;
  } else {
    for (int64_t i = 0; i < count; ++i)
      if (rows[i] < 0 || rows[i] >= c.n) throw InvalidArg("set_rows: row out of range");
    if (count > c.n) throw InvalidArg("set_rows: more rows than the dataset");
    const int64_t d = input_floats(c.net);
    if (!c.Xg) {
      dmalloc(c.Xg, (size_t)c.n * d);
      dmalloc(c.yg, (size_t)c.n);
      dmalloc(c.rows_dev, (size_t)c.n);
    }
    CK(cudaMemcpyAsync(c.rows_dev, rows, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c.stream));
    launch_gather_data(c, c.X_full, c.y_full, c.rows_dev, count, d, c.Xg, c.yg);
    c.X = c.Xg;
    c.y = c.yg;
    c.n_active = count;
  }
  if (c.tc) tc_refresh_data(c);
  if (c.ctc) cnn_tc_refresh_data(c, c.X, c.n_active);
}

int dasmc_gpu_set_target(dasmc_ctx* ctx, int64_t prefix_end, int64_t block_end, int64_t total_n, int mode,
                         double beta, double sigma) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) {
      multi_set_target_api(*ctx->multi, prefix_end, block_end, total_n, mode, beta, sigma);
      return;
    }
    Ctx t = ctx->c;  // validate on a copy (no allocation happens)
    t.prefix_end = prefix_end;
    t.block_end = block_end;
    t.total_n = total_n;
    t.mode = mode;
    t.beta = beta;
    t.sigma = sigma;
    validate_target(t);
    Ctx& c = ctx->c;
    c.prefix_end = prefix_end;
    c.block_end = block_end;
    c.total_n = total_n;
    c.mode = mode;
    c.beta = beta;
    c.sigma = sigma;
  });
}

int dasmc_gpu_value_and_grad(dasmc_ctx* ctx, const double* theta, int64_t J, double* values, double* grads) {
  return guarded([&] {
    if (!ctx || !theta || !values) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    check_J(c, J);
    validate_target(c);
    CK(cudaSetDevice(c.device));
    const int spare = (c.start + 2) % 3;
    ensure_stage(c, sizeof(double) * (size_t)J * c.net.D);
    upload(c, c.stage, theta, sizeof(double) * (size_t)J * c.net.D);
    launch_ref_to_internal_f64(c, (const double*)c.stage, c.theta[spare], J);
    if (!c.grad) {
      dmalloc(c.grad, (size_t)c.Jmax * c.net.Dp);
      CK(cudaMemset(c.grad, 0, sizeof(float) * (size_t)c.Jmax * c.net.Dp));
    }
    int64_t M, P;
    double br;
    target_rows(c, M, P, br);
    launch_zero_ints(c, c.flags, J);
    EpiParams e = make_epi(c, kEpiStoreGrad, 1.0, c.theta[spare], nullptr);
    launch_eval(c, c.theta[spare], J, M, P, br, grads != nullptr, &e);
    launch_eval_finalize(c, J, c.lt_new, nullptr, nullptr, M, true);
    download(c, values, c.lt_new, sizeof(double) * J);
    if (grads) {
      launch_internal_to_ref_f64(c, c.grad, (double*)c.stage, J);
      download(c, grads, c.stage, sizeof(double) * (size_t)J * c.net.D);
    }
  });
}

int dasmc_gpu_loglik_parts(dasmc_ctx* ctx, const double* theta, int64_t J, double* prefix, double* block) {
  return guarded([&] {
    if (!ctx || !theta || !prefix || !block) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    check_J(c, J);
    if (c.prefix_end < 0 || c.prefix_end > c.block_end || c.block_end > c.n)
      throw InvalidArg("unscaled_loglik_parts: window exceeds dataset");
    if (c.block_end < 1) throw InvalidArg("loglik_batch: empty batch");
    CK(cudaSetDevice(c.device));
    const int spare = (c.start + 2) % 3;
    ensure_stage(c, sizeof(double) * (size_t)J * c.net.D);
    upload(c, c.stage, theta, sizeof(double) * (size_t)J * c.net.D);
    launch_ref_to_internal_f64(c, (const double*)c.stage, c.theta[spare], J);
    loglik_parts_dev(c, c.theta[spare], J, c.prefix_end, c.block_end);
    download(c, prefix, c.ll_pre, sizeof(double) * J);
    download(c, block, c.ll_blk, sizeof(double) * J);
  });
}

int dasmc_gpu_momentum(dasmc_ctx* ctx, uint64_t seed, int k, int64_t J, double* p0) {
  return guarded([&] {
    if (!ctx || !p0) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    check_J(c, J);
    CK(cudaSetDevice(c.device));
    launch_normals(c, seed, tag::kProposal, (uint64_t)k, J, 1.0f, c.p, c.p0_part);
    ensure_stage(c, sizeof(double) * (size_t)J * c.net.D);
    launch_internal_to_ref_f64(c, c.p, (double*)c.stage, J);
    download(c, p0, c.stage, sizeof(double) * (size_t)J * c.net.D);
  });
}

int dasmc_gpu_uniforms(dasmc_ctx* ctx, uint64_t seed, int k, int64_t count, double* u) {
  return guarded([&] {
    if (!ctx || !u || count < 1) throw InvalidArg("bad argument");
    Ctx& c = ctx->c;
    if (count > c.Jmax) throw InvalidArg("uniforms: count exceeds max_particles");
    CK(cudaSetDevice(c.device));
    launch_uniforms(c, fork_key(seed, tag::kResample, (uint64_t)k, 0), count, c.uni);
    download(c, u, c.uni, sizeof(double) * count);
  });
}

int dasmc_gpu_resample_indices(dasmc_ctx* ctx, const double* w, const double* u, int64_t J, int kind,
                               int32_t* idx) {
  return guarded([&] {
    if (!ctx || !w || !u || !idx) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    check_J(c, J);
    double s = 0.0;  // check_normalized_weights (numeric.hpp:38-47)
    for (int64_t j = 0; j < J; ++j) {
      if (!(w[j] >= 0.0)) throw InvalidArg("weights: entries must be >= 0");
      s += w[j];
    }
    if (std::abs(s - 1.0) > 1e-9) throw InvalidArg("weights: must sum to 1");
    CK(cudaSetDevice(c.device));
    upload(c, c.wts, w, sizeof(double) * J);
    upload(c, c.uni, u, sizeof(double) * (kind == DASMC_MULTINOMIAL ? J : 1));
    launch_resample_hook(c, c.wts, c.uni, J, kind, c.idx);
    download(c, idx, c.idx, sizeof(int32_t) * J);
  });
}

int dasmc_gpu_init_ensemble(dasmc_ctx* ctx, int64_t J, uint64_t seed) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) {
      multi_init_api(*ctx->multi, J, seed);
      return;
    }
    CK(cudaSetDevice(ctx->c.device));
    init_ensemble_dev(ctx->c, J, seed);
  });
}

int dasmc_gpu_set_ensemble(dasmc_ctx* ctx, const double* theta, const double* log_weights, int64_t J,
                           int iteration) {
  return guarded([&] {
    if (!ctx || !theta || !log_weights) throw InvalidArg("null argument");
    if (ctx->multi) {
      multi_set_ensemble_api(*ctx->multi, theta, false, log_weights, J, iteration);
      return;
    }
    Ctx& c = ctx->c;
    check_J(c, J);
    if (J < 2) throw InvalidArg("ensemble needs at least 2 particles");
    CK(cudaSetDevice(c.device));
    ensure_stage(c, sizeof(double) * (size_t)J * c.net.D);
    CK(cudaMemcpyAsync(c.stage, theta, sizeof(double) * (size_t)J * c.net.D, cudaMemcpyHostToDevice, c.stream));
    launch_ref_to_internal_f64(c, (const double*)c.stage, c.theta[c.start], J);
    CK(cudaMemcpyAsync(c.logw, log_weights, sizeof(double) * J, cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    c.J = J;
    c.iteration = iteration;
    c.has_ensemble = true;
  c.step_parts_valid = false;
  c.cache_valid = false;
  });
}

}  // extern "C"

namespace {
constexpr int kXferChunks = 8;
void ensure_copy_stream(Ctx& c) {
  if (c.copy) return;
  CK(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
  for (cudaEvent_t& e : c.xfer_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}
// particle chunk ch of kXferChunks: [j0, j1)
void xfer_chunk(int64_t J, int ch, int64_t& j0, int64_t& j1) {
  j0 = J * ch / kXferChunks;
  j1 = J * (ch + 1) / kXferChunks;
}
}  // namespace

extern "C" {

int dasmc_gpu_set_ensemble_f32(dasmc_ctx* ctx, const float* theta, const double* log_weights, int64_t J,
                               int iteration) {
  return guarded([&] {
    if (!ctx || !theta || !log_weights) throw InvalidArg("null argument");
    if (ctx->multi) {
      multi_set_ensemble_api(*ctx->multi, theta, true, log_weights, J, iteration);
      return;
    }
    Ctx& c = ctx->c;
    check_J(c, J);
    if (J < 2) throw InvalidArg("ensemble needs at least 2 particles");
    CK(cudaSetDevice(c.device));
    ensure_stage(c, sizeof(float) * (size_t)J * c.net.D);
    ensure_copy_stream(c);
    // the copy stream starts after everything already queued on the context's stream
    CK(cudaEventRecord(c.xfer_ev[kXferChunks], c.stream));
    CK(cudaStreamWaitEvent(c.copy, c.xfer_ev[kXferChunks], 0));
    const int64_t D = c.net.D;
    float* stage = (float*)c.stage;
    for (int ch = 0; ch < kXferChunks; ++ch) {  // H2D of chunk ch+1 overlaps the conversion of ch
      int64_t j0, j1;
      xfer_chunk(J, ch, j0, j1);
      if (j1 == j0) continue;
      CK(cudaMemcpyAsync(stage + j0 * D, theta + j0 * D, sizeof(float) * (size_t)(j1 - j0) * D,
                         cudaMemcpyHostToDevice, c.copy));
      CK(cudaEventRecord(c.xfer_ev[ch], c.copy));
      CK(cudaStreamWaitEvent(c.stream, c.xfer_ev[ch], 0));
      launch_ref_to_internal_f32(c, stage + j0 * D, c.theta[c.start] + j0 * c.net.Dp, j1 - j0);
    }
    CK(cudaMemcpyAsync(c.logw, log_weights, sizeof(double) * J, cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    c.J = J;
    c.iteration = iteration;
    c.has_ensemble = true;
  c.step_parts_valid = false;
  c.cache_valid = false;
  });
}

int dasmc_gpu_get_ensemble(dasmc_ctx* ctx, double* theta, double* log_weights, int* iteration) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) {
      multi_get_ensemble_api(*ctx->multi, theta, false, log_weights, iteration);
      return;
    }
    Ctx& c = ctx->c;
    if (!c.has_ensemble) throw InvalidArg("no ensemble");
    CK(cudaSetDevice(c.device));
    if (theta) {
      ensure_stage(c, sizeof(double) * (size_t)c.J * c.net.D);
      launch_internal_to_ref_f64(c, c.theta[c.start], (double*)c.stage, c.J);
      CK(cudaMemcpyAsync(theta, c.stage, sizeof(double) * (size_t)c.J * c.net.D, cudaMemcpyDeviceToHost, c.stream));
    }
    if (log_weights) CK(cudaMemcpyAsync(log_weights, c.logw, sizeof(double) * c.J, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (iteration) *iteration = c.iteration;
  });
}

int dasmc_gpu_get_ensemble_f32(dasmc_ctx* ctx, float* theta, double* log_weights, int* iteration) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) {
      multi_get_ensemble_api(*ctx->multi, theta, true, log_weights, iteration);
      return;
    }
    Ctx& c = ctx->c;
    if (!c.has_ensemble) throw InvalidArg("no ensemble");
    CK(cudaSetDevice(c.device));
    if (theta) {
      ensure_stage(c, sizeof(float) * (size_t)c.J * c.net.D);
      ensure_copy_stream(c);
      const int64_t D = c.net.D;
      float* stage = (float*)c.stage;
      for (int ch = 0; ch < kXferChunks; ++ch) {  // D2H of chunk ch overlaps the conversion of ch+1
        int64_t j0, j1;
        xfer_chunk(c.J, ch, j0, j1);
        if (j1 == j0) continue;
        launch_internal_to_ref_f32(c, c.theta[c.start] + j0 * c.net.Dp, stage + j0 * D, j1 - j0);
        CK(cudaEventRecord(c.xfer_ev[ch], c.stream));
        CK(cudaStreamWaitEvent(c.copy, c.xfer_ev[ch], 0));
        CK(cudaMemcpyAsync(theta + j0 * D, stage + j0 * D, sizeof(float) * (size_t)(j1 - j0) * D,
                           cudaMemcpyDeviceToHost, c.copy));
      }
    }
    if (log_weights) CK(cudaMemcpyAsync(log_weights, c.logw, sizeof(double) * c.J, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (c.copy) CK(cudaStreamSynchronize(c.copy));
    if (iteration) *iteration = c.iteration;
  });
}

int dasmc_gpu_smc_step(dasmc_ctx* ctx, const dasmc_kernel_cfg* cfg, uint64_t seed, int resample_kind,
                       double fraction, int resample_always, dasmc_iter_record* record) {
  return guarded([&] {
    if (!ctx || !cfg) throw InvalidArg("null argument");
    if (!(fraction >= 0.0 && fraction <= 1.0)) throw InvalidArg("resample_fraction: must be in [0, 1]");
    if (ctx->multi) {
      multi_smc_step_api(*ctx->multi, *cfg, seed, resample_kind, fraction, resample_always, record);
      return;
    }
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    const int slot = c.rec_head % kRecRing;
    CK(cudaEventRecord(c.ev0, c.stream));
    if (c.use_graphs && !c.cache_start)
      smc_step_graphed(c, *cfg, seed, resample_kind, fraction, resample_always, slot);
    else
      smc_step_async(c, *cfg, seed, resample_kind, fraction, resample_always, slot);
    CK(cudaEventRecord(c.ev1, c.stream));
    ++c.rec_head;
    if (record) {
      fetch_records(c, slot, 1);
      *record = read_record(c, slot);
      c.cache_valid = c.cache_start && record->n_divergent == 0;
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      record->sampler_ms = ms;
      record->batch = c.block_end;
      record->beta = c.mode == DASMC_SDA ? c.beta : 1.0;
    }
  });
}

int dasmc_gpu_sync_records(dasmc_ctx* ctx, dasmc_iter_record* records, int count) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) {
      multi_sync_records_api(*ctx->multi, records, count);
      return;
    }
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    if (count < 0 || count > c.rec_head || count > kRecRing) throw InvalidArg("record count out of range");
    CK(cudaStreamSynchronize(c.stream));
    if (count == 0 || records == nullptr) return;
    CK(cudaMemcpy(c.h_records, c.records, sizeof(double) * 8 * kRecRing, cudaMemcpyDeviceToHost));
    for (int i = 0; i < count; ++i) {
      const int slot = (c.rec_head - count + i) % kRecRing;
      records[i] = read_record(c, slot);
      records[i].batch = c.block_end;
      records[i].beta = c.mode == DASMC_SDA ? c.beta : 1.0;
    }
  });
}

int dasmc_gpu_last_proposals(dasmc_ctx* ctx, double* p_final, double* log_target_new, double* log_target_old,
                             int32_t* divergent, double* norm_weights, int32_t* indices) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    Ctx& c = ctx->c;
    const int64_t J = c.J;
    CK(cudaSetDevice(c.device));
    if (p_final) {
      ensure_stage(c, sizeof(double) * (size_t)J * c.net.D);
      launch_internal_to_ref_f64(c, c.p, (double*)c.stage, J);
      download(c, p_final, c.stage, sizeof(double) * (size_t)J * c.net.D);
    }
    if (log_target_new) download(c, log_target_new, c.lt_new, sizeof(double) * J);
    if (log_target_old) download(c, log_target_old, c.lt_old, sizeof(double) * J);
    if (divergent) download(c, divergent, c.flags, sizeof(int32_t) * J);
    if (norm_weights) download(c, norm_weights, c.wts, sizeof(double) * J);
    if (indices) download(c, indices, c.idx, sizeof(int32_t) * J);
  });
}

int dasmc_gpu_sda_moments(dasmc_ctx* ctx, int64_t prefix_end, int64_t block_end, double* out6) {
  return guarded([&] {
    if (!ctx || !out6) throw InvalidArg("null argument");
    if (ctx->multi) {
      multi_sda_moments_api(*ctx->multi, prefix_end, block_end, out6);
      return;
    }
    if (!ctx->c.has_ensemble) throw InvalidArg("no ensemble");
    CK(cudaSetDevice(ctx->c.device));
    sda_moments_dev(ctx->c, prefix_end, block_end, out6);
  });
}

int64_t dasmc_batch_size(const dasmc_schedule* cfg, int k) {
  int64_t out = -1;
  const int rc = guarded([&] {
    if (!cfg) throw InvalidArg("null schedule");
    out = batch_size(*cfg, k);
  });
  return rc == DASMC_OK ? out : -1;
}

int dasmc_sda_init(const dasmc_schedule* cfg, double beta0, double entropy_step, dasmc_sda_state* out) {
  return guarded([&] {
    if (!cfg || !out) throw InvalidArg("null argument");
    *out = sda_init(*cfg, beta0, entropy_step);
  });
}

double dasmc_sda_beta_step(double beta, double* entropy_step, double denom) {
  return sda_beta_step(beta, *entropy_step, denom);
}

int dasmc_sda_advance_with(const dasmc_schedule* cfg, dasmc_sda_state* state, const double* moments6) {
  return guarded([&] {
    if (!cfg || !state || !moments6) throw InvalidArg("null argument");
    validate_schedule(*cfg);
    *state = sda_advance_with(*cfg, *state, moments6);
  });
}

int dasmc_sda_moments_from(const double* prefix_nll, const double* block_nll, const double* log_weights, int64_t J,
                           double* out6) {
  return guarded([&] {
    if (!prefix_nll || !block_nll || !log_weights || !out6 || J < 1) throw InvalidArg("bad argument");
    sda_moments_from(prefix_nll, block_nll, log_weights, J, out6);
  });
}

int dasmc_make_teacher_data(const dasmc_net_desc* net, int64_t n, int feature_kind, uint64_t seed, uint64_t cfg_id,
                            int threads, float* X, int32_t* y) {
  return guarded([&] {
    const NetDev nd = make_net(net);
    if (n < 1 || !X || !y) throw InvalidArg("bad argument");
    std::vector<int> layers(net->layer_sizes, net->layer_sizes + net->num_layers);
    make_teacher_data(layers, nd.act, n, feature_kind, seed, cfg_id, threads, X, y, net->conv);
  });
}

int dasmc_shuffle_permutation(uint64_t seed, int64_t n, int64_t* perm) {
  return guarded([&] {
    if (n < 1 || !perm) throw InvalidArg("bad argument");
    const auto p = shuffle_permutation(seed, n);
    std::memcpy(perm, p.data(), sizeof(int64_t) * (size_t)n);
  });
}

int dasmc_gpu_init_ensemble_at(dasmc_ctx* ctx, int64_t J, uint64_t seed, int64_t j_offset) {
  return guarded([&] {
    if (!ctx || j_offset < 0) throw InvalidArg("bad argument");
    CK(cudaSetDevice(ctx->c.device));
    init_ensemble_dev(ctx->c, J, seed, j_offset);
  });
}

void dasmc_shard_range(int64_t J, int world, int rank, int64_t* lo, int64_t* hi) {
  // parallel.hpp:30-31 static contiguous partition
  *lo = J * rank / world;
  *hi = J * (rank + 1) / world;
}

int dasmc_shard_plan(const int32_t* idx, int64_t J, int world, int rank, int32_t* recv_src, int32_t* recv_row,
                     int64_t* send_cnt, int32_t* send_rows) {
  return guarded([&] {
    if (!idx || world < 1 || rank < 0 || rank >= world || J < world) throw InvalidArg("shard_plan: bad argument");
    std::vector<int64_t> lo((size_t)world + 1);
    for (int r = 0; r <= world; ++r) lo[(size_t)r] = J * r / world;
    auto owner = [&](int64_t g) {
      return (int)(std::upper_bound(lo.begin(), lo.end(), g) - lo.begin()) - 1;
    };
    for (int64_t j = lo[(size_t)rank]; j < lo[(size_t)rank + 1]; ++j) {
      const int64_t g = idx[j];
      if (g < 0 || g >= J) throw InvalidArg("shard_plan: index out of range");
      const int s = owner(g);
      recv_src[j - lo[(size_t)rank]] = s;
      recv_row[j - lo[(size_t)rank]] = (int32_t)(g - lo[(size_t)s]);
    }
    int64_t n = 0;
    for (int d = 0; d < world; ++d) {
      send_cnt[d] = 0;
      for (int64_t j = lo[(size_t)d]; j < lo[(size_t)d + 1]; ++j) {
        const int64_t g = idx[j];
        if (owner(g) == rank) {
          send_rows[n++] = (int32_t)(g - lo[(size_t)rank]);
          ++send_cnt[d];
        }
      }
    }
  });
}

int dasmc_gpu_shard_propose(dasmc_ctx* ctx, const dasmc_kernel_cfg* cfg, uint64_t seed, int64_t j_offset,
                            double* log_w_dev, double* log_target_new_dev) {
  return guarded([&] {
    if (ctx) ctx->c.step_parts_valid = ctx->c.cache_valid = false;
    if (!ctx || !cfg || !log_w_dev || !log_target_new_dev) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    const int t1 = (c.start + 1) % 3, t2 = (c.start + 2) % 3;
    float* bufs[3] = {c.theta[c.start], c.theta[t1], c.theta[t2]};
    const int end_idx = propose_async(c, *cfg, seed, j_offset);
    launch_local_weights(c, c.J, log_w_dev, log_target_new_dev);
    // finalise positions: divergent particles keep theta (smc.hpp:129-131)
    const int dst_idx = end_idx == 1 ? 2 : 1;
    launch_gather(c, bufs[0], bufs[end_idx], bufs[dst_idx], c.J, c.iota);
    c.start = dst_idx == 1 ? t1 : t2;
    CK(cudaStreamSynchronize(c.stream));
  });
}

int dasmc_gpu_shard_resample(dasmc_ctx* ctx, const double* log_w_full_dev, const double* log_target_new_full_dev,
                             int64_t J_total, int64_t j_offset, uint64_t seed, int resample_kind, double fraction,
                             int resample_always, int32_t* idx_dev, dasmc_iter_record* record) {
  return guarded([&] {
    if (ctx) ctx->c.step_parts_valid = ctx->c.cache_valid = false;
    if (!ctx || !log_w_full_dev || !log_target_new_full_dev || !idx_dev) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    if (j_offset < 0 || j_offset + c.J > J_total) throw InvalidArg("shard_resample: slice out of range");
    if (resample_kind != DASMC_MULTINOMIAL && resample_kind != DASMC_SYSTEMATIC) throw InvalidArg("bad resample kind");
    CK(cudaSetDevice(c.device));
    if (J_total > c.sh_cap) {
      if (c.sh_buf) CK(cudaFree(c.sh_buf));
      if (c.sh_idx) CK(cudaFree(c.sh_idx));
      c.sh_buf = nullptr;
      c.sh_idx = nullptr;
      dmalloc(c.sh_buf, (size_t)5 * J_total);
      dmalloc(c.sh_idx, (size_t)J_total);
      c.sh_cap = J_total;
    }
    const int64_t need = (J_total + 2 * c.rng_chunk - 1) / (2 * c.rng_chunk) + 1;
    if (need > c.jump_chunks) {
      CK(cudaStreamSynchronize(c.stream));
      CK(cudaFree(c.jump_tab));
      c.jump_tab = nullptr;
      const auto tab = jump_table(2 * (uint64_t)c.rng_chunk, need);
      dmalloc(c.jump_tab, (size_t)need * 4);
      CK(cudaMemcpy(c.jump_tab, tab.data(), sizeof(uint64_t) * 4 * tab.size(), cudaMemcpyHostToDevice));
      c.jump_chunks = need;
    }
    double* lw = c.sh_buf;
    double* lt = lw + c.sh_cap;
    double* w = lt + c.sh_cap;
    double* cdf = w + c.sh_cap;
    double* uni = cdf + c.sh_cap;
    const int k = c.iteration;
    CK(cudaMemcpyAsync(lw, log_w_full_dev, sizeof(double) * J_total, cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(lt, log_target_new_full_dev, sizeof(double) * J_total, cudaMemcpyDeviceToDevice, c.stream));
    launch_uniforms(c, fork_key(seed, tag::kResample, (uint64_t)k, 0),
                    resample_kind == DASMC_MULTINOMIAL ? J_total : 1, uni);
    const int slot = c.rec_head % kRecRing;
    launch_normalize_resample(c, J_total, lw, lt, w, cdf, uni, c.sh_idx, fraction, resample_always, resample_kind,
                              slot, k);
    ++c.rec_head;
    CK(cudaMemcpyAsync(c.logw, lw + j_offset, sizeof(double) * c.J, cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(idx_dev, c.sh_idx, sizeof(int32_t) * J_total, cudaMemcpyDeviceToDevice, c.stream));
    fetch_records(c, slot, 1);
    dasmc_iter_record r = read_record(c, slot);
    r.batch = c.block_end;
    r.beta = c.mode == DASMC_SDA ? c.beta : 1.0;
    if (record) *record = r;
    c.iteration = k + 1;
  });
}

int64_t dasmc_gpu_row_floats(const dasmc_ctx* ctx) { return ctx ? ctx->c.net.Dp : -1; }

static void upload_rows(Ctx& c, const int32_t* rows, int64_t n) {
  if (n > c.sh_rows_cap) {
    if (c.sh_rows) CK(cudaFree(c.sh_rows));
    c.sh_rows = nullptr;
    dmalloc(c.sh_rows, (size_t)n);
    c.sh_rows_cap = n;
  }
  CK(cudaMemcpyAsync(c.sh_rows, rows, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c.stream));
}

int dasmc_gpu_pack_rows(dasmc_ctx* ctx, const int32_t* rows, int64_t n, float* dst_dev) {
  return guarded([&] {
    if (!ctx || (n > 0 && (!rows || !dst_dev)) || n < 0) throw InvalidArg("bad argument");
    Ctx& c = ctx->c;
    for (int64_t i = 0; i < n; ++i)
      if (rows[i] < 0 || rows[i] >= c.J) throw InvalidArg("pack_rows: row out of range");
    CK(cudaSetDevice(c.device));
    if (n == 0) return;
    upload_rows(c, rows, n);
    launch_rows(c, c.theta[c.start], dst_dev, c.sh_rows, n, true);
    CK(cudaStreamSynchronize(c.stream));
  });
}

int dasmc_gpu_unpack_rows(dasmc_ctx* ctx, const float* src_dev, const int32_t* slots, int64_t n) {
  return guarded([&] {
    if (ctx) ctx->c.step_parts_valid = ctx->c.cache_valid = false;
    if (!ctx || !src_dev || !slots) throw InvalidArg("null argument");
    Ctx& c = ctx->c;
    if (n != c.J) throw InvalidArg("unpack_rows: every local slot must be written exactly once");
    std::vector<char> seen((size_t)c.J, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (slots[i] < 0 || slots[i] >= c.J || seen[(size_t)slots[i]]) throw InvalidArg("unpack_rows: bad slot list");
      seen[(size_t)slots[i]] = 1;
    }
    CK(cudaSetDevice(c.device));
    const int next = (c.start + 1) % 3;
    upload_rows(c, slots, n);
    launch_rows(c, src_dev, c.theta[next], c.sh_rows, n, false);
    c.start = next;
    CK(cudaStreamSynchronize(c.stream));
  });
}

int dasmc_gpu_reserve_rows(dasmc_ctx* ctx, int64_t M) {
  if (ctx && ctx->multi) {
    for (int r = 0; r < dasmc_gpu_multi_shards(ctx); ++r) {
      const int rc = dasmc_gpu_reserve_rows(multi_shard_handle(ctx->multi, r), M);
      if (rc != DASMC_OK) return rc;
    }
    return DASMC_OK;
  }
  return guarded([&] {
    if (!ctx || M < 1 || M > ctx->c.n) throw InvalidArg("reserve_rows: M out of range");
    CK(cudaSetDevice(ctx->c.device));
    ensure_activation_capacity(ctx->c, M);
  });
}

void* dasmc_gpu_stream(dasmc_ctx* ctx) {
  if (ctx && ctx->multi) return (void*)multi_lead(*ctx->multi).stream;
  return ctx ? (void*)ctx->c.stream : nullptr;
}

int64_t dasmc_launch_count(void) { return (int64_t)g_launch_count.load(); }

int dasmc_gpu_set_timing(dasmc_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    Ctx& c = ctx->multi ? multi_lead(*ctx->multi) : ctx->c;  // a group times its lead shard
    CK(cudaSetDevice(c.device));
    harvest_timers(c);
    for (int k = 0; k < kTimerKinds; ++k) {
      c.kms[k] = 0.0;
      c.kcount[k] = 0;
    }
    c.ktime = enable != 0;
  });
}

int dasmc_gpu_kernel_times(dasmc_ctx* ctx, double* ms3, int64_t* count3) {
  return guarded([&] {
    if (!ctx || !ms3 || !count3) throw InvalidArg("null argument");
    Ctx& c = ctx->multi ? multi_lead(*ctx->multi) : ctx->c;
    CK(cudaSetDevice(c.device));
    harvest_timers(c);
    for (int k = 0; k < kTimerKinds; ++k) {
      ms3[k] = c.kms[k];
      count3[k] = c.kcount[k];
      c.kms[k] = 0.0;
      c.kcount[k] = 0;
    }
  });
}

int dasmc_rng_skip(uint64_t key, uint64_t skip, int64_t count, uint64_t* out) {
  return guarded([&] {
    if (count < 0 || (count > 0 && !out)) throw InvalidArg("bad argument");
    Xoshiro x;
    x.seed(key);
    if (skip > 0) {
      const auto tab = jump_table(skip, 2);
      x.jump(tab[1].data());
    }
    for (int64_t i = 0; i < count; ++i) out[i] = x.next();
  });
}

// ---- evaluate_predictive (runner.hpp:331-364) -------------------------------------------
int dasmc_gpu_predictive_mix(dasmc_ctx* ctx, const float* X_test, const int32_t* y_test, int64_t n_test,
                             const double* w, int64_t J, double* pred) {
  return guarded([&] {
    if (!ctx || !X_test || !w || !pred || n_test < 1) throw InvalidArg("bad argument");
    Ctx& c = ctx->c;
    if (!c.has_ensemble) throw InvalidArg("no ensemble");
    check_J(c, J);
    const int C = c.net.sizes[c.net.L];
    if (C > 16) throw InvalidArg("evaluate_predictive: at most 16 classes");
    if (c.net.nconv > 0 && !y_test) throw InvalidArg("evaluate_predictive: CNN contexts need the labels");
    CK(cudaSetDevice(c.device));
    const int64_t d_in = input_floats(c.net);
    int64_t widest = 0;
    for (int l = 1; l <= c.net.L; ++l) widest = std::max<int64_t>(widest, c.net.sizes[l]);
    // rows per chunk: scratch activations of J x R x widest floats stay below ~4 GB
    const int64_t R = std::max<int64_t>(1, std::min<int64_t>(n_test, (int64_t)(1 << 30) / std::max<int64_t>(1, J * widest)));
    float *Xd = nullptr, *logits = nullptr, *s0 = nullptr, *s1 = nullptr;
    int32_t* yd = nullptr;
    double *wd = nullptr, *pd = nullptr;
    dmalloc(Xd, (size_t)R * d_in);
    dmalloc(logits, (size_t)J * R * C);
    dmalloc(s0, (size_t)J * R * widest);
    dmalloc(s1, (size_t)J * R * widest);
    dmalloc(yd, (size_t)R);
    dmalloc(wd, (size_t)J);
    dmalloc(pd, (size_t)R * C);
    CK(cudaMemcpyAsync(wd, w, sizeof(double) * J, cudaMemcpyHostToDevice, c.stream));
    const float* th = c.theta[c.start];
    for (int64_t r0 = 0; r0 < n_test; r0 += R) {
      const int64_t rows = std::min(R, n_test - r0);
      CK(cudaMemcpyAsync(Xd, X_test + r0 * d_in, sizeof(float) * rows * d_in, cudaMemcpyHostToDevice, c.stream));
      if (y_test) CK(cudaMemcpyAsync(yd, y_test + r0, sizeof(int32_t) * rows, cudaMemcpyHostToDevice, c.stream));
      CK(cudaMemcpyAsync(pd, pred + r0 * C, sizeof(double) * rows * C, cudaMemcpyHostToDevice, c.stream));
      launch_forward_logits(c, th, J, Xd, yd, rows, logits, s0, s1);
      launch_predictive_mix(c, logits, rows, J, wd, pd);
      CK(cudaMemcpyAsync(pred + r0 * C, pd, sizeof(double) * rows * C, cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
    }
    void* bufs[] = {Xd, logits, s0, s1, yd, wd, pd};
    for (void* p : bufs) cudaFree(p);
  });
}

int dasmc_predictive_metrics(const double* pred, const int32_t* y, int64_t n, int C, double* log_pred,
                             double* accuracy) {
  return guarded([&] {
    if (!pred || !y || n < 1 || C < 1) throw InvalidArg("bad argument");
    double lp = 0.0;
    int64_t correct = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double* row = pred + i * C;
      if (y[i] < 0 || y[i] >= C) throw InvalidArg("label out of range");
      lp += std::log(std::max(row[y[i]], 1e-300));
      int am = 0;
      for (int c = 1; c < C; ++c)
        if (row[c] > row[am]) am = c;
      if (am == y[i]) ++correct;
    }
    if (log_pred) *log_pred = lp / (double)n;
    if (accuracy) *accuracy = 100.0 * (double)correct / (double)n;
  });
}

int dasmc_gpu_evaluate_predictive(dasmc_ctx* ctx, const float* X_test, const int32_t* y_test, int64_t n_test,
                                  double* log_pred, double* accuracy) {
  return guarded([&] {
    if (!ctx || !y_test) throw InvalidArg("bad argument");
    Ctx& c = ctx->c;
    if (!c.has_ensemble) throw InvalidArg("no ensemble");
    const int64_t J = c.J;
    std::vector<double> lw((size_t)J), w((size_t)J);
    CK(cudaSetDevice(c.device));
    CK(cudaMemcpyAsync(lw.data(), c.logw, sizeof(double) * J, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    double m = lw[0];  // normalize (smc.hpp:57-64)
    for (double x : lw) m = std::max(m, x);
    if (m == -std::numeric_limits<double>::infinity()) throw Dead("normalize: all particles dead");
    double s = 0.0;
    for (int64_t j = 0; j < J; ++j) {
      w[(size_t)j] = std::exp(lw[(size_t)j] - m);
      s += w[(size_t)j];
    }
    for (auto& x : w) x /= s;
    const int C = c.net.sizes[c.net.L];
    std::vector<double> pred((size_t)n_test * C, 0.0);
    int rc = dasmc_gpu_predictive_mix(ctx, X_test, y_test, n_test, w.data(), J, pred.data());
    if (rc != DASMC_OK) throw std::runtime_error(g_err);
    rc = dasmc_predictive_metrics(pred.data(), y_test, n_test, C, log_pred, accuracy);
    if (rc != DASMC_OK) throw InvalidArg(g_err);
  });
}

int dasmc_gpu_set_cache_start(dasmc_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    c.cache_start = enable != 0;
    c.cache_valid = false;
    if (c.cache_start && !c.gcache[0]) {
      for (auto& g : c.gcache) {
        dmalloc(g, (size_t)c.Jmax * c.net.Dp);
        CK(cudaMemset(g, 0, sizeof(float) * (size_t)c.Jmax * c.net.Dp));
      }
      dmalloc(c.lt_cache, (size_t)c.Jmax);
    }
  });
}

int dasmc_gpu_last_step_cached(dasmc_ctx* ctx) { return ctx && ctx->c.last_step_cached ? 1 : 0; }

int dasmc_gpu_set_rows(dasmc_ctx* ctx, const int64_t* rows, int64_t count) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    set_rows_dev(c, rows, count);
  });
}

// load_idx / parse_idx (dataset.hpp:84-196).  With X == NULL only the sizes are returned.
static int idx_out(const IdxData& d, int64_t* n, int64_t* dim, int* classes, float* X, int32_t* y) {
  if (n) *n = d.n;
  if (dim) *dim = d.d;
  if (classes) *classes = d.num_classes;
  if (X) std::memcpy(X, d.X.data(), sizeof(float) * d.X.size());
  if (y) std::memcpy(y, d.y.data(), sizeof(int32_t) * d.y.size());
  return DASMC_OK;
}

int dasmc_parse_idx(const uint8_t* image_bytes, int64_t image_len, const uint8_t* label_bytes, int64_t label_len,
                    int64_t* n, int64_t* d, int* num_classes, float* X, int32_t* y) {
  return guarded([&] {
    if ((!image_bytes && image_len) || (!label_bytes && label_len)) throw InvalidArg("null buffer");
    const std::vector<unsigned char> im(image_bytes, image_bytes + image_len), lb(label_bytes, label_bytes + label_len);
    idx_out(parse_idx(im, lb), n, d, num_classes, X, y);
  });
}

int dasmc_load_idx(const char* image_path, const char* label_path, int64_t* n, int64_t* d, int* num_classes, float* X,
                   int32_t* y) {
  return guarded([&] {
    if (!image_path || !label_path) throw InvalidArg("null path");
    idx_out(parse_idx(read_file_bytes(image_path), read_file_bytes(label_path)), n, d, num_classes, X, y);
  });
}

int dasmc_make_synthetic(int kind, int64_t n, double noise, uint64_t seed, float* X, int32_t* y) {
  return guarded([&] {
    if (!X || !y) throw InvalidArg("null argument");
    make_synthetic(kind, n, noise, seed, X, y);
  });
}

int dasmc_redraw_rows(uint64_t seed, int k, int64_t n, int64_t count, int64_t* rows) {
  return guarded([&] {
    if (n < 1 || count < 1 || count > n || !rows) throw InvalidArg("bad argument");
    const auto r = redraw_rows(seed, k, n, count);
    std::memcpy(rows, r.data(), sizeof(int64_t) * (size_t)count);
  });
}

int dasmc_gpu_run(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n, const dasmc_run_cfg* cfg,
                  int device, int precision, dasmc_iter_record* records, dasmc_sda_state* sda_trace,
                  double* final_theta, double* final_log_weights) {
  dasmc_ctx* ctx = nullptr;
  int rc = guarded([&] {
    if (!net || !X || !y || !cfg || !records) throw InvalidArg("null argument");
    // shuffle once with root.fork(kPermutation) (runner.hpp:486-489)
    const auto perm = shuffle_permutation(cfg->seed, n);
    const int64_t d = input_floats(make_net(net));
    std::vector<float> Xs((size_t)n * d);
    std::vector<int32_t> ys((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      std::memcpy(Xs.data() + (size_t)i * d, X + (size_t)perm[(size_t)i] * d, sizeof(float) * d);
      ys[(size_t)i] = y[perm[(size_t)i]];
    }
    const int rc2 = dasmc_gpu_create(net, Xs.data(), ys.data(), n, cfg->particles, device, precision, &ctx);
    if (rc2 != DASMC_OK) throw std::runtime_error(g_err);
    Ctx& c = ctx->c;
    dasmc_schedule sched = cfg->schedule;  // runner.hpp:512-521
    sched.iterations = cfg->iterations;
    sched.dataset_size = n;
    if (sched.initial_batch <= 0) sched.initial_batch = n;
    sched.initial_batch = std::min<int64_t>(sched.initial_batch, n);
    sched.increment = sched.increment > 0 ? std::min<int64_t>(sched.increment, n) : sched.initial_batch;
    if (sched.period < 1) sched.period = 1;
    validate_schedule(sched);
    const bool sda = sched.kind == DASMC_SCHED_SDA;
    dasmc_sda_state st{};
    if (sda) st = sda_init(sched, cfg->beta0, cfg->entropy_step);
    auto context_for = [&](int k) {  // runner.hpp:544-564
      c.sigma = cfg->sigma;
      c.total_n = n;
      if (sda) {
        c.mode = DASMC_SDA;
        c.prefix_end = st.prefix_end;
        c.block_end = st.block_end;
        c.beta = st.beta;
      } else if (cfg->redraw_constant) {  // runner.hpp:548-557: a fresh batch per iteration
        const auto rows = redraw_rows(cfg->seed, k, n, sched.initial_batch);
        set_rows_dev(c, rows.data(), (int64_t)rows.size());
        c.mode = DASMC_SCALED;
        c.prefix_end = 0;
        c.block_end = sched.initial_batch;
        c.beta = 1.0;
      } else {
        c.mode = DASMC_SCALED;
        c.prefix_end = 0;
        c.block_end = batch_size(sched, k);
        c.beta = 1.0;
      }
    };
    context_for(0);
    init_ensemble_dev(c, cfg->particles, cfg->seed);
    for (int k = 0; k < cfg->iterations; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      context_for(k);
      const int slot = c.rec_head % kRecRing;
      smc_step_async(c, cfg->kernel, cfg->seed, cfg->resample_kind, cfg->resample_fraction, cfg->resample_always,
                     slot);
      ++c.rec_head;
      fetch_records(c, slot, 1);
      dasmc_iter_record r = read_record(c, slot);
      r.batch = c.block_end;
      r.beta = sda ? c.beta : 1.0;
      if (sda && !st.terminal) {  // sda_advance on the post-step ensemble (runner.hpp:592)
        double m6[6];
        sda_moments_dev(c, st.prefix_end, st.block_end, m6);
        st = sda_advance_with(sched, st, m6);
      }
      r.sampler_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      records[k] = r;
      if (sda_trace) sda_trace[k] = st;
    }
    if (final_theta || final_log_weights) {
      const int rc3 = dasmc_gpu_get_ensemble(ctx, final_theta, final_log_weights, nullptr);
      if (rc3 != DASMC_OK) throw std::runtime_error(g_err);
    }
  });
  if (ctx) dasmc_gpu_destroy(ctx);
  return rc;
}

int dasmc_gpu_bench_memory(dasmc_ctx* ctx, int64_t J, const int32_t* idx, int reps, double* ms4, double* bytes4) {
  return guarded([&] {
    if (!ctx || !idx || !ms4 || !bytes4 || reps < 1) throw InvalidArg("bad argument");
    Ctx& c = ctx->c;
    check_J(c, J);
    for (int64_t j = 0; j < J; ++j)
      if (idx[j] < 0 || idx[j] >= J) throw InvalidArg("idx out of range");
    CK(cudaSetDevice(c.device));
    upload(c, c.idx, idx, sizeof(int32_t) * J);
    launch_zero_ints(c, c.flags, J);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double Dp = (double)c.net.Dp, D = (double)c.net.D;
    for (int kind = 0; kind < 4; ++kind) {
      auto once = [&] {
        switch (kind) {
          case 0: launch_gather(c, c.theta[0], c.theta[1], c.theta[2], J, c.idx); break;
          case 1: launch_p_sumsq(c, J); break;
          case 2: launch_normals(c, 12345u, tag::kProposal, 7u, J, 1.0f, c.p, c.p0_part, 0); break;
          default: launch_weights_and_resample(c, J, 0.5, 1, DASMC_SYSTEMATIC, 0, 0, 0.0); break;
        }
      };
      once();  // warm-up
      CK(cudaEventRecord(e0, c.stream));
      for (int r = 0; r < reps; ++r) once();
      CK(cudaEventRecord(e1, c.stream));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ms4[kind] = ms / reps;
    }
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
    bytes4[0] = 8.0 * (double)J * Dp;  // read + write one row per particle
    bytes4[1] = 4.0 * (double)J * Dp;
    bytes4[2] = 4.0 * (double)J * D;
    bytes4[3] = 48.0 * (double)J;      // log-weights, targets, weights, cdf (fp64), idx, flags
  });
}

}  // extern "C"

// =====================================================================================
// Single-process multi-GPU group: one ensemble of J particles sharded over
// G shard contexts, shard r on devices[r] owning the contiguous global slots [lo_r, hi_r)
// (parallel.hpp:30-31).  The C++ driver owns the whole iteration (smc.hpp:109-158):
//   1. every shard proposes / reweights its own slots (RNG streams keyed by the GLOBAL slot);
//   2. all-gather of the (log_w, log_target_new) vectors: peer copies over NVLink into every
//      shard's full-J vectors (reference order);
//   3. every shard runs the same normalise / ESS / decision / CDF / search on the full
//      vectors (identical indices, no broadcast) and finalises its own rows (divergent
//      particles keep theta, smc.hpp:129-131);
//   4. migration: each shard's gather kernel pulls its new rows theta_new[j] =
//      fin[owner(idx[j])][idx[j] - lo_owner] straight from the owners' memory (peer loads
//      over NVLink; no host plan, no staging copies).
// Cross-shard ordering is stream / event based; the only host read per iteration is the
// record the caller asks for.  Shards may share a device (devices = {0, 0, 0}): the same
// code then runs as an in-process emulation, bit-identical to one context.
// SDA moments (annealing.hpp:153-174) come from an all-gather of the per-particle final
// (prefix, block) log-likelihood pairs, reduced on the host in reference order.
namespace dasmc_b200 {

constexpr int kMaxShards = 16;

struct PeerRows {
  const float4* p[kMaxShards];
  int64_t lo[kMaxShards + 1];
  int G;
};

namespace {

__global__ void __launch_bounds__(256) peer_gather_kernel(PeerRows src, float4* __restrict__ dst, int64_t Dp4,
                                                          const int32_t* __restrict__ idx) {
  const int64_t j = blockIdx.y;
  const int64_t g = idx[j];
  int r = 0;
  while (r + 1 < src.G && g >= src.lo[r + 1]) ++r;
  const float4* s = src.p[r] + (g - src.lo[r]) * Dp4;
  float4* d = dst + j * Dp4;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < Dp4; i += (int64_t)gridDim.x * 256) d[i] = s[i];
}

__global__ void pick_pairs_kernel(int64_t J, const int32_t* __restrict__ idx, const double* __restrict__ pre,
                                  const double* __restrict__ blk, double* __restrict__ out_pre,
                                  double* __restrict__ out_blk) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= J) return;
  out_pre[j] = pre[idx[j]];
  out_blk[j] = blk[idx[j]];
}

}  // namespace

struct MultiState {
  int G = 0;
  std::vector<dasmc_ctx*> sh;
  std::vector<int> dev;
  std::vector<int64_t> lo;  // G + 1 slot boundaries
  int64_t J = 0, Jcap = 0;
  bool has = false;
  int rec_head = 0;
  // per shard, on its device: full-J vectors (log_w, log_target_new, w, cdf, uniforms,
  // final prefix / block ll, post-resample prefix / block ll) and indices; local vectors
  std::vector<double*> full;   // [9][Jcap]
  std::vector<int32_t*> idx;   // [Jcap]
  std::vector<double*> loc;    // [4][Jcap / G + 1]: log_w, log_target_new, final prefix, final block
  std::vector<cudaEvent_t> ev_w, ev_f, ev_g;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool parts_valid = false;
  int64_t parts_P = -1, parts_M = -1;
};

namespace {

enum { kLw = 0, kLt, kW, kCdf, kUni, kFp, kFb, kSp, kSb, kNumFull };

Ctx& shard(MultiState& m, int r) { return m.sh[(size_t)r]->c; }

void multi_free(MultiState* m) {
  if (!m) return;
  for (int r = 0; r < m->G; ++r) {
    if (r < (int)m->dev.size()) cudaSetDevice(m->dev[(size_t)r]);
    if (r < (int)m->full.size() && m->full[(size_t)r]) cudaFree(m->full[(size_t)r]);
    if (r < (int)m->idx.size() && m->idx[(size_t)r]) cudaFree(m->idx[(size_t)r]);
    if (r < (int)m->loc.size() && m->loc[(size_t)r]) cudaFree(m->loc[(size_t)r]);
    for (auto* v : {&m->ev_w, &m->ev_f, &m->ev_g})
      if (r < (int)v->size() && (*v)[(size_t)r]) cudaEventDestroy((*v)[(size_t)r]);
    if (r < (int)m->sh.size() && m->sh[(size_t)r]) dasmc_gpu_destroy(m->sh[(size_t)r]);
  }
  if (m->e0) cudaEventDestroy(m->e0);
  if (m->e1) cudaEventDestroy(m->e1);
  delete m;
}

// (re)size the full-J vectors for an ensemble of J particles
void multi_reserve(MultiState& m, int64_t J) {
  if (J <= m.Jcap) return;
  for (int r = 0; r < m.G; ++r) {
    CK(cudaSetDevice(m.dev[(size_t)r]));
    CK(cudaStreamSynchronize(shard(m, r).stream));
    if (m.full[(size_t)r]) CK(cudaFree(m.full[(size_t)r]));
    if (m.idx[(size_t)r]) CK(cudaFree(m.idx[(size_t)r]));
    if (m.loc[(size_t)r]) CK(cudaFree(m.loc[(size_t)r]));
    m.full[(size_t)r] = nullptr;
    m.idx[(size_t)r] = nullptr;
    m.loc[(size_t)r] = nullptr;
    dmalloc(m.full[(size_t)r], (size_t)kNumFull * J);
    dmalloc(m.idx[(size_t)r], (size_t)J);
    dmalloc(m.loc[(size_t)r], (size_t)4 * (J / m.G + 1));
    Ctx& c = shard(m, r);
    // the resampling uniforms of J_total slots need jump polynomials for J_total draws
    const int64_t need = (J + 2 * c.rng_chunk - 1) / (2 * c.rng_chunk) + 1;
    if (need > c.jump_chunks) {
      CK(cudaFree(c.jump_tab));
      c.jump_tab = nullptr;
      const auto tab = jump_table(2 * (uint64_t)c.rng_chunk, need);
      dmalloc(c.jump_tab, (size_t)need * 4);
      CK(cudaMemcpy(c.jump_tab, tab.data(), sizeof(uint64_t) * 4 * tab.size(), cudaMemcpyHostToDevice));
      c.jump_chunks = need;
    }
  }
  m.Jcap = J;
}

void multi_ranges(MultiState& m, int64_t J) {
  m.lo.assign((size_t)m.G + 1, 0);
  for (int r = 0; r <= m.G; ++r) m.lo[(size_t)r] = J * r / m.G;  // parallel.hpp:30-31
  for (int r = 0; r < m.G; ++r)
    if (m.lo[(size_t)r + 1] - m.lo[(size_t)r] < 2) throw InvalidArg("multi-GPU group: need >= 2 particles per shard");
}

void multi_peer_copy(MultiState& m, int d, double* dst, int r, const double* src, int64_t count) {
  if (count <= 0) return;
  CK(cudaMemcpyPeerAsync(dst, m.dev[(size_t)d], src, m.dev[(size_t)r], sizeof(double) * count, shard(m, d).stream));
}

// One SMC iteration of the whole sharded ensemble.  Asynchronous; the record lands in shard
// 0's record ring at `slot`.
void multi_step(MultiState& m, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction, int always,
                int slot) {
  if (rkind != DASMC_MULTINOMIAL && rkind != DASMC_SYSTEMATIC) throw InvalidArg("bad resample kind");
  const int G = m.G;
  const int64_t J = m.J;
  const int k = shard(m, 0).iteration;
  const bool parts = shard(m, 0).mode == DASMC_SDA;
  std::vector<float*> fin((size_t)G);
  // 1. propose + local weights (+ final ll pairs for the SDA moments) on every shard
  for (int r = 0; r < G; ++r) {
    Ctx& c = shard(m, r);
    CK(cudaSetDevice(c.device));
    for (int q = 0; q < G; ++q) CK(cudaStreamWaitEvent(c.stream, m.ev_g[(size_t)q], 0));  // peers done reading
    const int t1 = (c.start + 1) % 3, t2 = (c.start + 2) % 3;
    float* bufs[3] = {c.theta[c.start], c.theta[t1], c.theta[t2]};
    const int end_idx = propose_async(c, kc, seed, m.lo[(size_t)r]);
    const int64_t Jr = c.J;
    const int64_t stride = m.Jcap / G + 1;
    double* loc = m.loc[(size_t)r];
    launch_local_weights(c, Jr, loc, loc + stride);
    if (parts) launch_select_parts(c, Jr, c.iota, loc + 2 * stride, loc + 3 * stride);
    // finalised rows: divergent particles keep theta (smc.hpp:129-131), into the free buffer
    const int dst_idx = end_idx == 1 ? 2 : 1;
    launch_gather(c, bufs[0], bufs[end_idx], bufs[dst_idx], Jr, c.iota);
    fin[(size_t)r] = bufs[dst_idx];
    CK(cudaEventRecord(m.ev_w[(size_t)r], c.stream));
  }
  // 2. all-gather into every shard's full vectors (reference slot order)
  for (int d = 0; d < G; ++d) {
    Ctx& c = shard(m, d);
    CK(cudaSetDevice(c.device));
    double* full = m.full[(size_t)d];
    for (int r = 0; r < G; ++r) {
      CK(cudaStreamWaitEvent(c.stream, m.ev_w[(size_t)r], 0));
      const int64_t lo = m.lo[(size_t)r], n = m.lo[(size_t)r + 1] - lo, stride = m.Jcap / G + 1;
      const double* loc = m.loc[(size_t)r];
      multi_peer_copy(m, d, full + kLw * m.Jcap + lo, r, loc, n);
      multi_peer_copy(m, d, full + kLt * m.Jcap + lo, r, loc + stride, n);
      if (parts && d == 0) {
        multi_peer_copy(m, d, full + kFp * m.Jcap + lo, r, loc + 2 * stride, n);
        multi_peer_copy(m, d, full + kFb * m.Jcap + lo, r, loc + 3 * stride, n);
      }
    }
    // 3. redundant normalise / ESS / decision / resampling indices (smc.hpp:127-156)
    double* lw = full + kLw * m.Jcap;
    launch_uniforms(c, fork_key(seed, tag::kResample, (uint64_t)k, 0), rkind == DASMC_MULTINOMIAL ? J : 1,
                    full + kUni * m.Jcap);
    launch_normalize_resample(c, J, lw, full + kLt * m.Jcap, full + kW * m.Jcap, full + kCdf * m.Jcap,
                              full + kUni * m.Jcap, m.idx[(size_t)d], fraction, always, rkind, slot, k);
    CK(cudaMemcpyAsync(c.logw, lw + m.lo[(size_t)d], sizeof(double) * c.J, cudaMemcpyDeviceToDevice, c.stream));
    if (parts && d == 0)
      pick_pairs_kernel<<<(unsigned)((J + 255) / 256), 256, 0, c.stream>>>(
          J, m.idx[0], full + kFp * m.Jcap, full + kFb * m.Jcap, full + kSp * m.Jcap, full + kSb * m.Jcap);
    if (parts && d == 0) LAUNCHED();
  }
  // 4. migration: every shard pulls its new rows from the owners' finalised buffers
  PeerRows src{};
  src.G = G;
  for (int r = 0; r < G; ++r) src.p[r] = reinterpret_cast<const float4*>(fin[(size_t)r]);
  for (int r = 0; r <= G; ++r) src.lo[r] = m.lo[(size_t)r];
  for (int d = 0; d < G; ++d) {
    Ctx& c = shard(m, d);
    CK(cudaSetDevice(c.device));
    for (int r = 0; r < G; ++r) CK(cudaStreamWaitEvent(c.stream, m.ev_w[(size_t)r], 0));  // rows finalised
    const int64_t Dp4 = c.net.Dp / 4;
    const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>((Dp4 + 255) / 256, 64));
    peer_gather_kernel<<<dim3((unsigned)chunks, (unsigned)c.J), 256, 0, c.stream>>>(
        src, reinterpret_cast<float4*>(c.theta[c.start]), Dp4, m.idx[(size_t)d] + m.lo[(size_t)d]);
    LAUNCHED();
    CK(cudaEventRecord(m.ev_g[(size_t)d], c.stream));
    c.iteration = k + 1;  // smc.hpp:150, 154
    c.step_parts_valid = false;
    c.cache_valid = false;
  }
  // shard 0's stream marks the end of the whole iteration (records, timing)
  CK(cudaSetDevice(shard(m, 0).device));
  for (int r = 1; r < G; ++r) CK(cudaStreamWaitEvent(shard(m, 0).stream, m.ev_g[(size_t)r], 0));
  m.parts_valid = parts;
  m.parts_P = shard(m, 0).prefix_end;
  m.parts_M = shard(m, 0).block_end;
}

MultiState* multi_of(dasmc_ctx* ctx) { return ctx ? ctx->multi : nullptr; }

}  // namespace
}  // namespace dasmc_b200

extern "C" {

int dasmc_gpu_create_multi(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n,
                           int max_particles, const int* devices, int ndev, int precision, dasmc_ctx** out) {
  if (out == nullptr) {
    g_err = "null out";
    return DASMC_EINVAL;
  }
  *out = nullptr;
  auto* m = new MultiState();
  const int rc = guarded([&] {
    if (!devices || ndev < 1 || ndev > kMaxShards) throw InvalidArg("multi-GPU group: 1..16 devices");
    if (max_particles < 2 * ndev) throw InvalidArg("multi-GPU group: max_particles must be >= 2 per shard");
    m->G = ndev;
    m->dev.assign(devices, devices + ndev);
    m->sh.assign((size_t)ndev, nullptr);
    m->full.assign((size_t)ndev, nullptr);
    m->idx.assign((size_t)ndev, nullptr);
    m->loc.assign((size_t)ndev, nullptr);
    m->ev_w.assign((size_t)ndev, nullptr);
    m->ev_f.assign((size_t)ndev, nullptr);
    m->ev_g.assign((size_t)ndev, nullptr);
    const int per = (max_particles + ndev - 1) / ndev + 1;
    for (int r = 0; r < ndev; ++r) {
      const int rc2 = dasmc_gpu_create(net, X, y, n, per, devices[r], precision, &m->sh[(size_t)r]);
      if (rc2 != DASMC_OK) throw std::runtime_error(g_err);
      CK(cudaSetDevice(devices[r]));
      for (auto* v : {&m->ev_w, &m->ev_f, &m->ev_g})
        CK(cudaEventCreateWithFlags(&(*v)[(size_t)r], cudaEventDisableTiming));
      // peer access to every other shard's device (NVLink loads / copies)
      for (int q = 0; q < ndev; ++q) {
        if (devices[q] == devices[r]) continue;
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, devices[r], devices[q]));
        if (!can) throw InvalidArg("multi-GPU group: devices without peer access");
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
    }
    CK(cudaSetDevice(devices[0]));
    CK(cudaEventCreate(&m->e0));
    CK(cudaEventCreate(&m->e1));
    multi_reserve(*m, max_particles);
  });
  if (rc != DASMC_OK) {
    multi_free(m);
    return rc;
  }
  auto* h = new dasmc_ctx();
  h->multi = m;
  h->c.net = m->sh[0]->c.net;  // param_count, layouts
  h->c.device = devices[0];
  *out = h;
  return DASMC_OK;
}

int dasmc_gpu_multi_shards(const dasmc_ctx* ctx) { return ctx && ctx->multi ? ctx->multi->G : 1; }

int dasmc_gpu_set_graphs(dasmc_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw InvalidArg("null ctx");
    if (ctx->multi) throw InvalidArg("set_graphs: single contexts only");
    Ctx& c = ctx->c;
    CK(cudaSetDevice(c.device));
    CK(cudaStreamSynchronize(c.stream));
    graphs_free(c);
    c.use_graphs = enable != 0;
  });
}

}  // extern "C"

namespace dasmc_b200 {
namespace {

// ---- group versions of the hot-path entry points (dispatched from the C-ABI) ----------------
void multi_set_target(MultiState& m, int64_t P, int64_t M, int64_t N, int mode, double beta, double sigma) {
  for (int r = 0; r < m.G; ++r) {
    const int rc = dasmc_gpu_set_target(m.sh[(size_t)r], P, M, N, mode, beta, sigma);
    if (rc != DASMC_OK) throw InvalidArg(g_err);
  }
  m.parts_valid = false;
}

void multi_init(MultiState& m, int64_t J, uint64_t seed) {
  multi_ranges(m, J);
  multi_reserve(m, J);
  for (int r = 0; r < m.G; ++r) {
    Ctx& c = shard(m, r);
    CK(cudaSetDevice(c.device));
    init_ensemble_dev(c, m.lo[(size_t)r + 1] - m.lo[(size_t)r], seed, m.lo[(size_t)r]);
  }
  m.J = J;
  m.has = true;
  m.parts_valid = false;
}

template <typename T>
void multi_set_ensemble(MultiState& m, const T* theta, const double* lw, int64_t J, int iteration) {
  multi_ranges(m, J);
  multi_reserve(m, J);
  const int64_t D = shard(m, 0).net.D;
  for (int r = 0; r < m.G; ++r) {
    const int64_t lo = m.lo[(size_t)r], n = m.lo[(size_t)r + 1] - lo;
    int rc;
    if constexpr (std::is_same<T, float>::value)
      rc = dasmc_gpu_set_ensemble_f32(m.sh[(size_t)r], theta + lo * D, lw + lo, n, iteration);
    else
      rc = dasmc_gpu_set_ensemble(m.sh[(size_t)r], theta + lo * D, lw + lo, n, iteration);
    if (rc != DASMC_OK) throw InvalidArg(g_err);
  }
  m.J = J;
  m.has = true;
  m.parts_valid = false;
}

template <typename T>
void multi_get_ensemble(MultiState& m, T* theta, double* lw, int* iteration) {
  if (!m.has) throw InvalidArg("no ensemble");
  const int64_t D = shard(m, 0).net.D;
  for (int r = 0; r < m.G; ++r) {
    const int64_t lo = m.lo[(size_t)r];
    int rc;
    if constexpr (std::is_same<T, float>::value)
      rc = dasmc_gpu_get_ensemble_f32(m.sh[(size_t)r], theta ? theta + lo * D : nullptr, lw ? lw + lo : nullptr,
                                      nullptr);
    else
      rc = dasmc_gpu_get_ensemble(m.sh[(size_t)r], theta ? theta + lo * D : nullptr, lw ? lw + lo : nullptr, nullptr);
    if (rc != DASMC_OK) throw std::runtime_error(g_err);
  }
  if (iteration) *iteration = shard(m, 0).iteration;
}

void multi_sda_moments(MultiState& m, int64_t P, int64_t M, double* out6) {
  if (!m.has) throw InvalidArg("no ensemble");
  if (P < 0 || P > M || M > shard(m, 0).n) throw InvalidArg("SubsetWindow: need 0 <= prefix_end <= block_end <= total_n");
  if (M <= P) throw InvalidArg("sda_moments: window has no new block");
  const int64_t J = m.J;
  std::vector<double> pre((size_t)J), blk((size_t)J), lw((size_t)J);
  Ctx& c0 = shard(m, 0);
  CK(cudaSetDevice(c0.device));
  if (m.parts_valid && m.parts_P == P && m.parts_M == M && !c0.force_moment_pass) {
    // the all-gathered (prefix, block) pairs of the step's own evaluations, resampled
    download(c0, pre.data(), m.full[0] + kSp * m.Jcap, sizeof(double) * J);
    download(c0, blk.data(), m.full[0] + kSb * m.Jcap, sizeof(double) * J);
  } else {
    for (int r = 0; r < m.G; ++r) {
      Ctx& c = shard(m, r);
      CK(cudaSetDevice(c.device));
      loglik_parts_dev(c, c.theta[c.start], c.J, P, M);
      download(c, pre.data() + m.lo[(size_t)r], c.ll_pre, sizeof(double) * c.J);
      download(c, blk.data() + m.lo[(size_t)r], c.ll_blk, sizeof(double) * c.J);
    }
  }
  for (int r = 0; r < m.G; ++r) {
    Ctx& c = shard(m, r);
    CK(cudaSetDevice(c.device));
    download(c, lw.data() + m.lo[(size_t)r], c.logw, sizeof(double) * c.J);
  }
  for (int64_t j = 0; j < J; ++j) {
    pre[(size_t)j] = -pre[(size_t)j];
    blk[(size_t)j] = -blk[(size_t)j];
  }
  sda_moments_from(pre.data(), blk.data(), lw.data(), J, out6);
}

}  // namespace
}  // namespace dasmc_b200

namespace dasmc_b200 {
void multi_destroy(MultiState* m) { multi_free(m); }
dasmc_ctx* multi_shard_handle(MultiState* m, int r) { return m->sh[(size_t)r]; }
Ctx& multi_lead(MultiState& m) { return shard(m, 0); }
void multi_set_target_api(MultiState& m, int64_t P, int64_t M, int64_t N, int mode, double beta, double sigma) {
  multi_set_target(m, P, M, N, mode, beta, sigma);
}
void multi_init_api(MultiState& m, int64_t J, uint64_t seed) { multi_init(m, J, seed); }
void multi_set_ensemble_api(MultiState& m, const void* theta, bool f32, const double* lw, int64_t J, int it) {
  if (f32)
    multi_set_ensemble(m, static_cast<const float*>(theta), lw, J, it);
  else
    multi_set_ensemble(m, static_cast<const double*>(theta), lw, J, it);
}
void multi_get_ensemble_api(MultiState& m, void* theta, bool f32, double* lw, int* it) {
  if (f32)
    multi_get_ensemble(m, static_cast<float*>(theta), lw, it);
  else
    multi_get_ensemble(m, static_cast<double*>(theta), lw, it);
}
void multi_smc_step_api(MultiState& m, const dasmc_kernel_cfg& kc, uint64_t seed, int rkind, double fraction,
                        int always, dasmc_iter_record* record) {
  if (!m.has) throw InvalidArg("smc_step: no ensemble (call init_ensemble or set_ensemble)");
  Ctx& c0 = shard(m, 0);
  CK(cudaSetDevice(c0.device));
  const int slot = m.rec_head % kRecRing;
  CK(cudaEventRecord(m.e0, c0.stream));
  multi_step(m, kc, seed, rkind, fraction, always, slot);
  CK(cudaSetDevice(c0.device));
  CK(cudaEventRecord(m.e1, c0.stream));
  ++m.rec_head;
  if (record) {
    fetch_records(c0, slot, 1);
    *record = read_record(c0, slot);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, m.e0, m.e1));
    record->sampler_ms = ms;
    record->batch = c0.block_end;
    record->beta = c0.mode == DASMC_SDA ? c0.beta : 1.0;
  }
}
void multi_sync_records_api(MultiState& m, dasmc_iter_record* records, int count) {
  Ctx& c0 = shard(m, 0);
  CK(cudaSetDevice(c0.device));
  if (count < 0 || count > m.rec_head || count > kRecRing) throw InvalidArg("record count out of range");
  for (int r = 0; r < m.G; ++r) {
    CK(cudaSetDevice(shard(m, r).device));
    CK(cudaStreamSynchronize(shard(m, r).stream));
  }
  CK(cudaSetDevice(c0.device));
  if (count == 0 || records == nullptr) return;
  CK(cudaMemcpy(c0.h_records, c0.records, sizeof(double) * 8 * kRecRing, cudaMemcpyDeviceToHost));
  for (int i = 0; i < count; ++i) {
    const int slot = (m.rec_head - count + i) % kRecRing;
    records[i] = read_record(c0, slot);
    records[i].batch = c0.block_end;
    records[i].beta = c0.mode == DASMC_SDA ? c0.beta : 1.0;
  }
}
void multi_sda_moments_api(MultiState& m, int64_t P, int64_t M, double* out6) { multi_sda_moments(m, P, M, out6); }
}  // namespace dasmc_b200
