// C-ABI over the CPU oracle (TEST INFRASTRUCTURE ONLY).  Loaded through ctypes
// by tests/, __graft_entry__.smoke() and bench.py's CPU legs; the product
// (paper_2601_21983_b200/) never links or calls it.
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "dasmc_oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const SamplerError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

NetSpec net_of(const int* layers, int nl, int act) {
  NetSpec s;
  s.layer_sizes.assign(layers, layers + nl);
  s.activation = act == 1 ? Activation::kTanh : Activation::kRelu;
  validate(s);
  return s;
}

// Model encoding of the `layers` array: an MLP is its layer sizes; a CNN
// ([EXT], dasmc_oracle.hpp) is [-1, in_c, in_h, in_w, nconv, (k, cout, pool) x
// nconv, head layer sizes...] with head[0] = the flatten size.
ModelSpec model_of(const int* layers, int nl, int act) {
  if (nl >= 1 && layers[0] == -1) {
    if (nl < 5) throw std::invalid_argument("cnn descriptor too short");
    CnnSpec c;
    c.in_c = layers[1];
    c.in_h = layers[2];
    c.in_w = layers[3];
    const int nconv = layers[4];
    int p = 5;
    for (int i = 0; i < nconv; ++i, p += 3) {
      if (p + 2 >= nl) throw std::invalid_argument("cnn descriptor too short");
      c.convs.push_back(ConvSpec{layers[p], layers[p + 1], layers[p + 2] != 0});
    }
    c.head = net_of(layers + p, nl - p, act);
    validate(c);
    return c;
  }
  return net_of(layers, nl, act);
}
int input_dim(const ModelSpec& m) {
  if (const auto* c = std::get_if<CnnSpec>(&m)) return c->in_c * c->in_h * c->in_w;
  return std::get<NetSpec>(m).layer_sizes.front();
}
int classes_of(const ModelSpec& m) {
  if (const auto* c = std::get_if<CnnSpec>(&m)) return c->head.layer_sizes.back();
  return std::get<NetSpec>(m).layer_sizes.back();
}

Dataset dataset_of(const double* X, const int* y, int64_t n, int d, int classes) {
  Dataset ds;
  ds.n = n;
  ds.d = d;
  ds.features.assign(X, X + (size_t)n * d);
  ds.labels.assign(y, y + n);
  ds.num_classes = classes;
  ds.perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) ds.perm[(size_t)i] = i;
  return ds;
}

// ---- OpenBLAS hook (numpy's scipy-openblas64, ILP64 cblas) -----------------
using cblas_dgemm_t = void (*)(int, int, int, long, long, long, double, const double*, long,
                               const double*, long, double, double*, long);
cblas_dgemm_t g_dgemm = nullptr;

void blas_dgemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                const double* B, int ldb, double beta, double* C, int ldc) {
  // CblasRowMajor=101, CblasNoTrans=111, CblasTrans=112
  g_dgemm(101, ta ? 112 : 111, tb ? 112 : 111, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// Route the oracle's GEMMs through an OpenBLAS shared object (single-threaded
// per call; particles run in parallel_for like the reference's Eigen build).
int oracle_use_blas(const char* path) {
  if (path == nullptr || path[0] == 0) {
    dgemm_hook() = nullptr;
    return 0;
  }
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    g_err = dlerror();
    return -1;
  }
  auto set_threads = (void (*)(int))dlsym(h, "scipy_openblas_set_num_threads64_");
  if (set_threads) set_threads(1);
  g_dgemm = (cblas_dgemm_t)dlsym(h, "scipy_cblas_dgemm64_");
  if (!g_dgemm) {
    g_err = "scipy_cblas_dgemm64_ not found";
    return -1;
  }
  dgemm_hook() = &blas_dgemm;
  return 0;
}

// ---- rng ---------------------------------------------------------------------
uint64_t oracle_fork_key(uint64_t key, uint64_t a, uint64_t b, uint64_t c) {
  return RngStream(key).fork(a, b, c).key();
}
void oracle_rng_u64(uint64_t key, int64_t n, uint64_t* out) {
  RngStream r(key);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void oracle_rng_normals(uint64_t key, int64_t n, double* out) {
  RngStream r(key);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}
void oracle_rng_uniforms(uint64_t key, int64_t n, double* out) {
  RngStream r(key);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
int oracle_rng_uniform_below(uint64_t key, uint64_t bound, int64_t n, uint64_t* out) {
  return guarded([&] {
    RngStream r(key);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform_below(bound);
  });
}

// ---- data --------------------------------------------------------------------
int oracle_make_teacher(const int* layers, int nl, int act, int64_t n, int feature_kind, uint64_t seed,
                        uint64_t cfg_id, int threads, double* X, int* y) {
  return guarded([&] {
    const ModelSpec m = model_of(layers, nl, act);
    const Dataset d = std::holds_alternative<CnnSpec>(m)
                          ? make_teacher_dataset(std::get<CnnSpec>(m), n, feature_kind, seed, cfg_id, threads)
                          : make_teacher_dataset(std::get<NetSpec>(m), n, feature_kind, seed, cfg_id, threads);
    std::memcpy(X, d.features.data(), sizeof(double) * d.features.size());
    std::memcpy(y, d.labels.data(), sizeof(int) * d.labels.size());
  });
}
int oracle_make_synthetic(int kind, int64_t n, double noise, uint64_t seed, int dim, double* X, int* y,
                          double* targets) {
  return guarded([&] {
    const SyntheticData s = make_synthetic((SyntheticKind)kind, n, noise, seed, dim);
    std::memcpy(X, s.data.features.data(), sizeof(double) * s.data.features.size());
    if (y && !s.data.labels.empty()) std::memcpy(y, s.data.labels.data(), sizeof(int) * (size_t)n);
    if (targets && !s.data.targets.empty()) std::memcpy(targets, s.data.targets.data(), sizeof(double) * (size_t)n);
  });
}
// Permutation applied by shuffled(fork(kPermutation)) (runner.hpp:486-489): perm[i] = source row.
int oracle_shuffle_perm(uint64_t seed, int64_t n, int64_t* perm) {
  return guarded([&] {
    Dataset d;
    d.n = n;
    d.d = 0;
    d.perm.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) d.perm[(size_t)i] = i;
    RngStream ps = RngStream(seed).fork(tag::kPermutation);
    const Dataset s = shuffled(d, ps);
    std::memcpy(perm, s.perm.data(), sizeof(int64_t) * (size_t)n);
  });
}

// ---- network / target ----------------------------------------------------------
int oracle_param_count(const int* layers, int nl) {
  try {
    return model_param_count(model_of(layers, nl, 0));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// values[J], grads[J*D] of log_target_with_grad (target.hpp:147-173) for each
// particle theta[j*D...].  mode 0 = scaled, 1 = sda.
int oracle_value_and_grad(const int* layers, int nl, int act, const double* X, const int* y, int64_t n,
                          int64_t prefix_end, int64_t block_end, int64_t total_n, int mode, double beta,
                          double sigma, const double* theta, int64_t J, int threads, double* values,
                          double* grads) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n, input_dim(net), classes_of(net));
    TargetContext c;
    c.data = &d;
    c.window = SubsetWindow{prefix_end, block_end, total_n};
    c.mode = (TargetMode)mode;
    c.beta = beta;
    c.prior.sigma = sigma;
    c.model = net;
    validate(c);
    const int64_t D = model_param_count(net);
    parallel_for(J, threads, [&](int64_t j) {
      const ValueGrad vg = log_target_with_grad(c, theta + j * D);
      values[j] = vg.value;
      if (grads) std::memcpy(grads + j * D, vg.grad.data(), sizeof(double) * (size_t)D);
    });
  });
}

int oracle_loglik_parts(const int* layers, int nl, int act, const double* X, const int* y, int64_t n,
                        int64_t prefix_end, int64_t block_end, const double* theta, int64_t J, int threads,
                        double* prefix, double* block) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n, input_dim(net), classes_of(net));
    const SubsetWindow w{prefix_end, block_end, n};
    const int64_t D = model_param_count(net);
    parallel_for(J, threads, [&](int64_t j) {
      const LoglikParts p = unscaled_loglik_parts(d, w, net, theta + j * D);
      prefix[j] = p.prefix;
      block[j] = p.block;
    });
  });
}

// ---- smc step ------------------------------------------------------------------
struct oracle_step_out {
  double ess;
  double mean_log_target;
  int resampled;
  int n_divergent;
};

// One smc_step (smc.hpp:109-158) on the given ensemble (thetas J*D, log_w J,
// iteration k).  Outputs the next ensemble in place plus the proposal dumps
// (any dump pointer may be null).
int oracle_smc_step(const int* layers, int nl, int act, const double* X, const int* y, int64_t n,
                    int64_t prefix_end, int64_t block_end, int64_t total_n, int mode, double beta, double sigma,
                    double step_size, int leapfrog_steps, int kernel_kind, uint64_t seed, double fraction,
                    int resample_kind, int resample_always, int threads, int64_t J, double* thetas,
                    double* log_w, int* iteration, oracle_step_out* out, double* p0_out, double* ps_out,
                    double* lt_new_out, double* lt_old_out, int* divergent_out, double* w_out, int* idx_out) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n, input_dim(net), classes_of(net));
    TargetContext c;
    c.data = &d;
    c.window = SubsetWindow{prefix_end, block_end, total_n};
    c.mode = (TargetMode)mode;
    c.beta = beta;
    c.prior.sigma = sigma;
    c.model = net;
    validate(c);
    const int64_t D = model_param_count(net);
    ParticleEnsemble e;
    e.dim = D;
    e.count = J;
    e.thetas.assign(thetas, thetas + D * J);
    e.log_weights.assign(log_w, log_w + J);
    e.iteration = *iteration;
    KernelConfig kc{step_size, leapfrog_steps, (KernelKind)kernel_kind};
    SmcOptions o{threads, fraction, (ResampleKind)resample_kind, resample_always != 0};
    StepDump dump;
    auto [next, rec] = smc_step(e, ContextTarget{&c}, kc, RngStream(seed), o, &dump);
    std::memcpy(thetas, next.thetas.data(), sizeof(double) * (size_t)(D * J));
    std::memcpy(log_w, next.log_weights.data(), sizeof(double) * (size_t)J);
    *iteration = next.iteration;
    out->ess = rec.ess;
    out->mean_log_target = rec.mean_log_target;
    out->resampled = rec.resampled ? 1 : 0;
    out->n_divergent = rec.n_divergent;
    for (int64_t j = 0; j < J; ++j) {
      const ProposalResult& p = dump.proposals[(size_t)j];
      if (p0_out) std::memcpy(p0_out + j * D, p.p_initial.data(), sizeof(double) * (size_t)D);
      if (ps_out) std::memcpy(ps_out + j * D, p.p_final.data(), sizeof(double) * (size_t)D);
      if (lt_new_out) lt_new_out[j] = p.log_target_new;
      if (lt_old_out) lt_old_out[j] = p.log_target_old;
      if (divergent_out) divergent_out[j] = p.divergent ? 1 : 0;
      if (w_out) w_out[j] = dump.weights[(size_t)j];
      if (idx_out) idx_out[j] = dump.indices.empty() ? -1 : dump.indices[(size_t)j];
    }
  });
}

// The parallel part of smc_step (smc.hpp:118-138) for a SUBSET of particles
// whose global slots are gj[n]: propose with fork(kProposal, k, gj) and the
// incremental weight; divergent particles keep theta and get -inf.
// thetas (n*D) updated in place; inc[n], lt_new[n] out.
int oracle_propose_particles(const int* layers, int nl, int act, const double* X, const int* y, int64_t n_data,
                             int64_t prefix_end, int64_t block_end, int64_t total_n, int mode, double beta,
                             double sigma, double step_size, int leapfrog_steps, int kernel_kind, uint64_t seed,
                             int k, const int64_t* gj, int64_t n, int threads, double* thetas, double* inc,
                             double* lt_new) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n_data, input_dim(net), classes_of(net));
    TargetContext c;
    c.data = &d;
    c.window = SubsetWindow{prefix_end, block_end, total_n};
    c.mode = (TargetMode)mode;
    c.beta = beta;
    c.prior.sigma = sigma;
    c.model = net;
    validate(c);
    const int64_t D = model_param_count(net);
    KernelConfig kc{step_size, leapfrog_steps, (KernelKind)kernel_kind};
    KernelConfig::validate(kc);
    const RngStream root(seed);
    parallel_for(n, threads, [&](int64_t i) {
      RngStream s = root.fork(tag::kProposal, (std::uint64_t)k, (std::uint64_t)gj[i]);
      const Vec th(thetas + i * D, thetas + (i + 1) * D);
      const ProposalResult p = propose(ContextTarget{&c}, th, kc, s);
      if (p.divergent) {
        inc[i] = kNegInf;
        lt_new[i] = p.log_target_new;
      } else {
        std::memcpy(thetas + i * D, p.theta_new.data(), sizeof(double) * (size_t)D);
        inc[i] = incremental_log_weight(p.log_target_new, p.log_target_old, p.p_initial, p.p_final);
        lt_new[i] = p.log_target_new;
      }
    });
  });
}

// init_ensemble (smc.hpp:73-89) on a scaled/sda context.
int oracle_init_ensemble(const int* layers, int nl, int act, const double* X, const int* y, int64_t n,
                         int64_t prefix_end, int64_t block_end, int64_t total_n, int mode, double beta,
                         double sigma, uint64_t seed, int64_t J, int threads, double* thetas, double* log_w) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n, input_dim(net), classes_of(net));
    TargetContext c;
    c.data = &d;
    c.window = SubsetWindow{prefix_end, block_end, total_n};
    c.mode = (TargetMode)mode;
    c.beta = beta;
    c.prior.sigma = sigma;
    c.model = net;
    const ParticleEnsemble e = init_ensemble(J, c, RngStream(seed), threads);
    std::memcpy(thetas, e.thetas.data(), sizeof(double) * e.thetas.size());
    std::memcpy(log_w, e.log_weights.data(), sizeof(double) * (size_t)J);
  });
}

// evaluate_predictive (runner.hpp:331-364) of the ensemble thetas[J*D], log_w[J] on a test set.
int oracle_evaluate_predictive(const int* layers, int nl, int act, const double* X, const int* y, int64_t n,
                               const double* thetas, const double* log_w, int64_t J, int threads, double* log_pred,
                               double* accuracy) {
  return guarded([&] {
    const ModelSpec net = model_of(layers, nl, act);
    const Dataset d = dataset_of(X, y, n, input_dim(net), classes_of(net));
    ParticleEnsemble e;
    e.dim = model_param_count(net);
    e.count = J;
    e.thetas.assign(thetas, thetas + e.dim * J);
    e.log_weights.assign(log_w, log_w + J);
    const auto r = evaluate_predictive(e, net, d, threads);
    *log_pred = r.first;
    *accuracy = r.second;
  });
}

// ---- resampling / weights --------------------------------------------------------
// kind 0: multinomial with J given uniforms u[J]; kind 1: systematic with u[0].
int oracle_resample_indices(const double* w, const double* u, int64_t J, int kind, int* idx) {
  return guarded([&] {
    const Vec wv(w, w + J);
    check_normalized_weights(wv);
    const Vec cdf = cdf_of(wv);
    for (int64_t j = 0; j < J; ++j)
      idx[j] = kind == 0 ? upper_bound_index(cdf, u[j]) : upper_bound_index(cdf, (u[0] + (double)j) / (double)J);
  });
}
int oracle_normalize(const double* lw, int64_t J, double* w, double* ess_out) {
  return guarded([&] {
    const Vec v = normalize(Vec(lw, lw + J));
    std::memcpy(w, v.data(), sizeof(double) * (size_t)J);
    if (ess_out) *ess_out = ess(v);
  });
}

// ---- schedules / sda ---------------------------------------------------------------
int64_t oracle_batch_size(int kind, int64_t initial, int64_t increment, int iterations, int64_t n, int period,
                          int switch_iteration, int k) {
  try {
    ScheduleConfig c{(ScheduleKind)kind, initial, increment, iterations, n, period, switch_iteration};
    return batch_size(c, k);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
double oracle_sda_beta_step(double beta, double* entropy_step, double denom) {
  return sda_beta_step(beta, *entropy_step, denom);
}
int oracle_sda_moments_from(const double* prefix_nll, const double* block_nll, const double* log_w, int64_t J,
                            double* out6) {
  return guarded([&] {
    const SdaMoments m = sda_moments_from(Vec(prefix_nll, prefix_nll + J), Vec(block_nll, block_nll + J),
                                          Vec(log_w, log_w + J));
    const double v[6] = {m.mean_block, m.mean_block_sq, m.var_block, m.mean_prefix, m.mean_prod,
                         m.cov_prefix_block};
    std::memcpy(out6, v, sizeof(v));
  });
}
// state: [beta, entropy_step, beta_reset, prefix_end, block_end, total_n, stage, terminal]
int oracle_sda_advance_with(int64_t increment, int64_t n, double* state, const double* moments6) {
  return guarded([&] {
    ScheduleConfig c{ScheduleKind::kSda, 1, increment, 1, n, 1, -1};
    SdaState s;
    s.beta = state[0];
    s.entropy_step = state[1];
    s.beta_reset = state[2];
    s.window = SubsetWindow{(int64_t)state[3], (int64_t)state[4], (int64_t)state[5]};
    s.stage = (SdaStage)(int)state[6];
    s.terminal = state[7] != 0.0;
    SdaMoments m{moments6[0], moments6[1], moments6[2], moments6[3], moments6[4], moments6[5]};
    const SdaState t = s.terminal ? s : sda_advance_with(c, s, m);
    state[0] = t.beta;
    state[1] = t.entropy_step;
    state[2] = t.beta_reset;
    state[3] = (double)t.window.prefix_end;
    state[4] = (double)t.window.block_end;
    state[5] = (double)t.window.total_n;
    state[6] = (double)(int)t.stage;
    state[7] = t.terminal ? 1.0 : 0.0;
  });
}

// ---- whole-run loop (runner.hpp:453-617, hot loop only) ----------------------------
struct oracle_run_record {
  int k;
  int64_t batch;
  double beta;
  double ess;
  int resampled;
  double mean_log_target;
  double sampler_ms;
  int n_divergent;
};

// X/y: the UNSHUFFLED training set (the loop shuffles it with fork(kPermutation)).
int oracle_run(const int* layers, int nl, int act, const double* X, const int* y, int64_t n, double sigma,
               double step_size, int leapfrog_steps, int kernel_kind, int sched_kind, int64_t initial,
               int64_t increment, int period, int switch_iteration, double beta0, double entropy_step,
               int redraw, int particles, int iterations, uint64_t seed, int threads, double fraction,
               int resample_kind, int resample_always, oracle_run_record* records, double* final_thetas,
               double* final_log_w) {
  return guarded([&] {
    RunConfig cfg;
    cfg.model = model_of(layers, nl, act);
    cfg.prior.sigma = sigma;
    cfg.kernel = KernelConfig{step_size, leapfrog_steps, (KernelKind)kernel_kind};
    KernelConfig::validate(cfg.kernel);
    cfg.schedule = ScheduleConfig{(ScheduleKind)sched_kind, initial, increment, iterations, n, period,
                                  switch_iteration};
    cfg.beta0 = beta0;
    cfg.entropy_step = entropy_step;
    cfg.redraw_constant = redraw != 0;
    cfg.particles = particles;
    cfg.iterations = iterations;
    cfg.seed = seed;
    cfg.threads = threads;
    cfg.resample_fraction = fraction;
    cfg.resample_kind = (ResampleKind)resample_kind;
    cfg.resample_always = resample_always != 0;
    const Dataset d = dataset_of(X, y, n, input_dim(cfg.model), classes_of(cfg.model));
    const RunResult r = run_loop(cfg, d);
    for (size_t i = 0; i < r.records.size(); ++i) {
      const IterRecord& a = r.records[i];
      records[i] = oracle_run_record{a.k, a.batch, a.beta, a.ess, a.resampled ? 1 : 0, a.mean_log_target,
                                     a.sampler_ms, a.n_divergent};
    }
    if (final_thetas) std::memcpy(final_thetas, r.ensemble.thetas.data(), sizeof(double) * r.ensemble.thetas.size());
    if (final_log_w)
      std::memcpy(final_log_w, r.ensemble.log_weights.data(), sizeof(double) * r.ensemble.log_weights.size());
  });
}

}  // extern "C"
