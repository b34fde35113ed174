/*
 * dasmc_gpu.h -- C-ABI drop-in boundary of the B200-native SMC hot path.
 *
 * The reference (arxiv/paper_2601_21983, /root/reference/proj) is a header-only
 * C++ library whose hot-path seam is a template parameter: smc_step<Target>()
 * calls Target::value_and_grad(theta) once per particle per leapfrog
 * evaluation (kernels.hpp:17-20, 75-99; smc.hpp:109-158).  A per-particle call
 * cannot feed a GPU, so the seam moves to ENSEMBLE granularity: one call
 * evaluates / moves / reweights / resamples all J particles.  Every entry point
 * below names the reference interface it replaces.
 *
 * Conventions:
 *  - plain C types only; host pointers are borrowed for the duration of the
 *    call; device buffers are owned by the context;
 *  - int status: 0 ok, -1 invalid argument, -2 all particles dead
 *    (= SamplerError, smc.hpp:21-24), -3 CUDA error; the message of the last
 *    failure on the calling thread is returned by dasmc_last_error();
 *  - per-particle divergence is an OUTPUT FLAG, not an error
 *    (kernels.hpp:138-145);
 *  - theta crosses the boundary in the reference layout: particle j occupies
 *    theta[j*D, (j+1)*D), per layer W (out x in) column-major then bias
 *    (network.hpp:55-62).  D = param_count (network.hpp:36-42);
 *  - one host thread per context (not re-entrant), like ParticleEnsemble's
 *    single owner between barriers (SPEC.md "Concurrency Model").
 */
#ifndef DASMC_GPU_H
#define DASMC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DASMC_OK 0
#define DASMC_EINVAL (-1)
#define DASMC_EDEAD (-2)
#define DASMC_ECUDA (-3)

/* Activation (network.hpp:19). */
#define DASMC_RELU 0
#define DASMC_TANH 1
/* TargetMode (target.hpp:91). */
#define DASMC_SCALED 0
#define DASMC_SDA 1
/* KernelKind (kernels.hpp:22). */
#define DASMC_HMC 0
#define DASMC_LANGEVIN 1
/* Resampling scheme: multinomial = smc.hpp:93-103 (parity mode);
 * systematic = [EXT] north-star default. */
#define DASMC_MULTINOMIAL 0
#define DASMC_SYSTEMATIC 1
/* Arithmetic of the dense contractions. */
#define DASMC_PREC_FP32 0   /* fp32 CUDA-core path: the 1e-4 parity path */
#define DASMC_PREC_TF32 1   /* tcgen05 kind::tf32 tensor-core path (tolerance stated in DESIGN.md) */
#define DASMC_PREC_3XTF32 2 /* tcgen05 split-tf32 (3 MMAs) tensor-core path, fp32-level accuracy */
#define DASMC_PREC_F16 3    /* tcgen05 kind::f16 with fp16 operands (the same 10-bit mantissa as tf32, fp32
                               accumulation, half the operand bytes); one-hidden-layer MLPs */
#define DASMC_PREC_TF32H 4  /* tf32 forward (kind::tf32 on tf32-rounded X, [W1, b1]); the weight-gradient
                               GEMM operands (X^T, a1^T, delta1^T, delta2^T: bounded-range activations and
                               deltas) stored as fp16, which carries the same 11-bit significand as tf32,
                               and contracted with kind::f16 (fp32 accumulation).  Deep MLPs run as TF32 */
#define DASMC_PREC_F16X2 5  /* kind::f16 throughout; forward = X (fp16: the same 11-bit significand as tf32)
                               times [W1, b1] split into fp16 hi + lo (two MMAs, ~22 significand bits);
                               weight-gradient operands fp16 as in TF32H.  At least tf32 accuracy, fp16
                               exponent range (|theta| >= 65504 overflows -> the particle diverges);
                               one-hidden-layer MLPs */
/* ScheduleKind (annealing.hpp:18). */
#define DASMC_SCHED_CONSTANT 0
#define DASMC_SCHED_FULL_BATCH 1
#define DASMC_SCHED_CTR 2
#define DASMC_SCHED_LINEAR 3
#define DASMC_SCHED_AUTOMATED 4
#define DASMC_SCHED_SDA 5

typedef struct dasmc_ctx dasmc_ctx;

/* NetSpec (network.hpp:24-27).
 * [EXT] conv != NULL describes a CNN front (BASELINE.json configs[2..3]; the
 * reference is MLP-only): {in_c, in_h, in_w, nconv, (k, cout, pool) x nconv}.
 * Each stage is a valid stride-1 convolution (theta block W[cout][cin][k][k]
 * row-major, then b[cout]), the activation, and an optional 2x2/2 max-pool.
 * The last stage output is flattened in (c, y, x) order into the MLP given by
 * layer_sizes, whose layer_sizes[0] must be the flatten size.  theta = conv
 * blocks in order, then the MLP in the reference layout.  X rows are images
 * [c][h][w]. */
typedef struct {
  int num_layers;         /* entries in layer_sizes, >= 2 */
  const int* layer_sizes; /* {input, hidden..., classes} */
  int activation;         /* DASMC_RELU | DASMC_TANH */
  const int* conv;        /* NULL for an MLP */
} dasmc_net_desc;

/* KernelConfig (kernels.hpp:26-49). */
typedef struct {
  double step_size;
  int leapfrog_steps;
  int kind;
} dasmc_kernel_cfg;

/* IterRecord (smc.hpp:38-49) + divergence count. */
typedef struct {
  int k;
  int64_t batch;
  double beta;
  double ess; /* pre-resample */
  int resampled;
  double mean_log_target;
  double sampler_ms;
  int n_divergent;
} dasmc_iter_record;

/* ScheduleConfig (annealing.hpp:23-30) + [EXT] period / switch_iteration
 * (period = 1 and switch_iteration = -1 are the
 * reference semantics). */
typedef struct {
  int kind;
  int64_t initial_batch;
  int64_t increment;
  int iterations;
  int64_t dataset_size;
  int period;
  int switch_iteration;
} dasmc_schedule;

/* SdaState (annealing.hpp:89-96). */
typedef struct {
  double beta;
  double entropy_step;
  double beta_reset;
  int64_t prefix_end, block_end, total_n;
  int stage; /* 0 initial, 1 annealed */
  int terminal;
} dasmc_sda_state;

/* The whole-run configuration read by run_experiment's hot loop
 * (runner.hpp:57-70, 453-617). */
typedef struct {
  dasmc_kernel_cfg kernel;
  dasmc_schedule schedule; /* iterations / dataset_size are resolved from the run */
  double sigma;            /* PriorSpec (network.hpp:45-47) */
  double beta0, entropy_step;
  int particles;
  int iterations;
  uint64_t seed;
  double resample_fraction;
  int resample_kind;
  int resample_always; /* [EXT] Appendix A.7 */
  int redraw_constant; /* ScheduleConfig::redraw_constant: a fresh batch of initial_batch rows per
                          iteration (runner.hpp:531-556) */
} dasmc_run_cfg;

/* Last error message of the calling thread. */
const char* dasmc_last_error(void);

/* ---- context ------------------------------------------------------------------
 * Replaces: Dataset + TargetContext ownership (dataset.hpp:46-56,
 * target.hpp:95-102).  X is n x input row-major fp32 in the run's fixed
 * (already shuffled) order, y the int32 labels.  The data is copied once to
 * HBM and stays resident.  max_particles bounds J for buffer sizing (2 .. 65535 per context; larger
 * ensembles shard over dasmc_gpu_create_multi). */
int dasmc_gpu_create(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n,
                     int max_particles, int device, int precision, dasmc_ctx** out);
int dasmc_gpu_destroy(dasmc_ctx* ctx);
int dasmc_gpu_param_count(const dasmc_ctx* ctx); /* param_count (network.hpp:36-42) */

/* TargetContext fields (target.hpp:95-113): window {prefix_end, block_end,
 * total_n}, mode, beta (SDA), prior sigma.  Validated exactly as validate(ctx). */
int dasmc_gpu_set_target(dasmc_ctx* ctx, int64_t prefix_end, int64_t block_end, int64_t total_n, int mode,
                         double beta, double sigma);

/* ---- parity entry points (host buffers) -------------------------------------------
 * log_target_with_grad (target.hpp:147-173) for J particles: values[J] (fp64),
 * grads[J*D] in the reference layout (may be NULL). */
int dasmc_gpu_value_and_grad(dasmc_ctx* ctx, const double* theta, int64_t J, double* values, double* grads);
/* unscaled_loglik_parts (target.hpp:121-129) under the current window. */
int dasmc_gpu_loglik_parts(dasmc_ctx* ctx, const double* theta, int64_t J, double* prefix, double* block);
/* Momentum draws p0 of propose() (kernels.hpp:131) for iteration k, particles
 * [0, J): stream root.fork(kProposal, k, j) (smc.hpp:119-120), fp64 out. */
int dasmc_gpu_momentum(dasmc_ctx* ctx, uint64_t seed, int k, int64_t J, double* p0);
/* Resampling uniforms of iteration k as the step draws them on the device: `count` draws of
 * root.fork(kResample, k) (smc.hpp:152; numeric.hpp:95-99), chunked with the F2 jump-ahead
 * (parity hook for rng.hpp:60-64 uniform()). */
int dasmc_gpu_uniforms(dasmc_ctx* ctx, uint64_t seed, int k, int64_t count, double* u);
/* Bit-exact resampling hook: indices given normalised weights w[J] and
 * uniforms u (J of them for multinomial, u[0] for systematic)
 * (numeric.hpp:81-101 sample_categorical's CDF + upper_bound). */
int dasmc_gpu_resample_indices(dasmc_ctx* ctx, const double* w, const double* u, int64_t J, int kind,
                               int32_t* idx);

/* ---- ensemble (ParticleEnsemble, smc.hpp:28-35) ------------------------------------ */
/* init_ensemble (smc.hpp:73-89) under the current target; stream root = seed. */
int dasmc_gpu_init_ensemble(dasmc_ctx* ctx, int64_t J, uint64_t seed);
int dasmc_gpu_set_ensemble(dasmc_ctx* ctx, const double* theta, const double* log_weights, int64_t J,
                           int iteration);
int dasmc_gpu_get_ensemble(dasmc_ctx* ctx, double* theta, double* log_weights, int* iteration);
/* Same with fp32 theta (the device precision) -- halves the boundary bytes. */
int dasmc_gpu_set_ensemble_f32(dasmc_ctx* ctx, const float* theta, const double* log_weights, int64_t J,
                               int iteration);
int dasmc_gpu_get_ensemble_f32(dasmc_ctx* ctx, float* theta, double* log_weights, int* iteration);

/* ---- the hot path -------------------------------------------------------------------
 * smc_step (smc.hpp:109-158): fresh momenta, S-step leapfrog under the current
 * target (S+1 gradient evaluations, kernels.hpp:75-99), incremental weights
 * (kernels.hpp:153-163), normalise / ESS / mean_log_target, resampling iff
 * resample_always or ESS < fraction*J.  Stream root = RngStream(seed); the
 * iteration index is the ensemble's.  `record` may be NULL: then the call
 * returns without synchronising the device (records are fetched with
 * dasmc_gpu_sync_records). */
int dasmc_gpu_smc_step(dasmc_ctx* ctx, const dasmc_kernel_cfg* cfg, uint64_t seed, int resample_kind,
                       double fraction, int resample_always, dasmc_iter_record* record);
/* Blocks until queued steps finished; copies the last `count` queued records. */
int dasmc_gpu_sync_records(dasmc_ctx* ctx, dasmc_iter_record* records, int count);
/* Per-particle proposal outputs of the last smc_step (parity dumps, host fp64,
 * reference layout); any pointer may be NULL. */
int dasmc_gpu_last_proposals(dasmc_ctx* ctx, double* p_final, double* log_target_new, double* log_target_old,
                             int32_t* divergent, double* norm_weights, int32_t* indices);

/* sda_moments (annealing.hpp:153-174) of the current ensemble under window
 * {prefix_end, block_end}: out6 = {mean_block, mean_block_sq, var_block,
 * mean_prefix, mean_prod, cov_prefix_block}. */
int dasmc_gpu_sda_moments(dasmc_ctx* ctx, int64_t prefix_end, int64_t block_end, double* out6);

/* ---- host-side schedule / controller (annealing.hpp), exact ------------------------ */
int64_t dasmc_batch_size(const dasmc_schedule* cfg, int k);                 /* annealing.hpp:52-82 */
int dasmc_sda_init(const dasmc_schedule* cfg, double beta0, double entropy_step, dasmc_sda_state* out);
double dasmc_sda_beta_step(double beta, double* entropy_step, double denom); /* annealing.hpp:114-122 */
int dasmc_sda_advance_with(const dasmc_schedule* cfg, dasmc_sda_state* state, const double* moments6);
int dasmc_sda_moments_from(const double* prefix_nll, const double* block_nll, const double* log_weights,
                           int64_t J, double* out6);

/* ---- IDX data files (dataset.hpp:84-196) -----------------------------------------------
 * parse_idx / load_idx: an IDX image (magic 0x803) + label (0x801) pair -> n rows of
 * rows*cols pixels / 255 (fp32) and labels; gzip files are decompressed transparently.
 * Malformed input returns DASMC_EINVAL with the reference's FormatError message.  Call with
 * X == NULL / y == NULL to query n, d and num_classes first. */
int dasmc_parse_idx(const uint8_t* image_bytes, int64_t image_len, const uint8_t* label_bytes, int64_t label_len,
                    int64_t* n, int64_t* d, int* num_classes, float* X, int32_t* y);
int dasmc_load_idx(const char* image_path, const char* label_path, int64_t* n, int64_t* d, int* num_classes, float* X,
                   int32_t* y);

/* ---- constant-redraw batches (runner.hpp:531-556) ---------------------------------------
 * rows = draw_batch_rows(k): the first `count` entries of a partial Fisher-Yates shuffle of
 * 0..n-1 with root.fork(kRedraw, k) (bit-exact); dasmc_gpu_set_rows makes the target read
 * train[rows[0..count)] (gathered on the device; rows == NULL restores the resident set).
 * The window is then {0, count, N} as in context_for. */
int dasmc_redraw_rows(uint64_t seed, int k, int64_t n, int64_t count, int64_t* rows);
/* make_synthetic (dataset.hpp:208-267) for the runner's classification datasets: kind 0 =
 * gaussian_blobs (3 classes), 1 = two_moons (2 classes); X n x 2 (fp32), y int32. */
int dasmc_make_synthetic(int kind, int64_t n, double noise, uint64_t seed, float* X, int32_t* y);
int dasmc_gpu_set_rows(dasmc_ctx* ctx, const int64_t* rows, int64_t count);

/* ---- start-gradient cache ---------------------------------
 * Opt-in.  When the target is unchanged since the previous smc_step (same mode, window,
 * beta, sigma, data rows and J) and that step had no divergent particle, the step's first
 * leapfrog evaluation is replaced by the previous step's final log targets and gradients,
 * gathered through its resampling: the same values (deterministic kernels), S instead of
 * S+1 evaluations.  Needs the record of each step (sync).  The reference recomputes
 * (kernels.hpp:85); off by default, and bench.py leaves it off. */
int dasmc_gpu_set_cache_start(dasmc_ctx* ctx, int enable);
int dasmc_gpu_last_step_cached(dasmc_ctx* ctx); /* 1 if the last smc_step used the cache */

/* ---- evaluate_predictive (runner.hpp:331-364) ------------------------------------------
 * Ensemble-averaged predictive of the context's current ensemble on a labelled test set
 * (host buffers: n_test rows in the model's input layout, int32 labels): mean log predictive
 * probability of the true label (floor 1e-300) and argmax accuracy in percent.  Weights are
 * normalised from the context's log-weights; particles with w = 0 contribute nothing. */
int dasmc_gpu_evaluate_predictive(dasmc_ctx* ctx, const float* X_test, const int32_t* y_test, int64_t n_test,
                                  double* log_pred, double* accuracy);
/* Sharded form: pred[n_test x classes] += sum over this context's J
 * particles of w[j] * softmax_j, in ascending j (w: the globally normalised weights of the
 * local slots; y_test needed for CNN contexts only).  Ranks all-reduce pred, then call
 * dasmc_predictive_metrics. */
int dasmc_gpu_predictive_mix(dasmc_ctx* ctx, const float* X_test, const int32_t* y_test, int64_t n_test,
                             const double* w, int64_t J, double* pred);
int dasmc_predictive_metrics(const double* pred, const int32_t* y, int64_t n, int classes, double* log_pred,
                             double* accuracy);

/* ---- data (dataset.hpp) -------------------------------------------------------------- */
/* [EXT] teacher-labelled synthetic data: features of kind 0
 * (U[0,1)) or 1 (k/255), labels = argmax of a N(0,1) teacher of shape `net`. */
int dasmc_make_teacher_data(const dasmc_net_desc* net, int64_t n, int feature_kind, uint64_t seed,
                            uint64_t cfg_id, int threads, float* X, int32_t* y);
/* Permutation of shuffled(data, root.fork(kPermutation)) (runner.hpp:486-489;
 * dataset.hpp:294-316): row i of the shuffled set is source row perm[i]. */
int dasmc_shuffle_permutation(uint64_t seed, int64_t n, int64_t* perm);

/* Pre-size the window-dependent activation buffers for windows up to M rows
 * (otherwise they grow on first use, which synchronises the stream). */
int dasmc_gpu_reserve_rows(dasmc_ctx* ctx, int64_t M);

/* ---- particle sharding across GPUs -------------------------------------
 * Rank r of G owns global particle slots [lo, hi) = [r*J/G, (r+1)*J/G)
 * (parallel.hpp:30-31's static partition).  Every RNG stream is keyed by the
 * GLOBAL slot, so results do not depend on G.  One iteration:
 *   1. dasmc_gpu_shard_propose   -- local move + incremental weights of own slots
 *   2. all-gather of the local (log_w, log_target_new) vectors  (torch.distributed / NCCL)
 *   3. dasmc_gpu_shard_resample  -- normalise / ESS / decision / indices on the FULL
 *      vectors, computed redundantly (identically) on every rank
 *   4. dasmc_shard_plan + pack / point-to-point exchange / unpack of theta rows. */
void dasmc_shard_range(int64_t J, int world, int rank, int64_t* lo, int64_t* hi);
/* init_ensemble of the shard holding global slots [j_offset, j_offset + J)
 * (streams fork(kInit, j_offset + j), smc.hpp:82). */
int dasmc_gpu_init_ensemble_at(dasmc_ctx* ctx, int64_t J, uint64_t seed, int64_t j_offset);
/* Migration plan for `rank` given the global indices idx[J] (out[j] = in[idx[j]]):
 *   recv_src[Jr]   owner rank of each local destination slot (local slot order)
 *   recv_row[Jr]   the source's LOCAL row
 *   send_cnt[G]    rows this rank sends to each rank (self included)
 *   send_rows[..]  this rank's local rows, grouped by destination rank, each group
 *                  in the destination's slot order (size = sum send_cnt <= J). */
int dasmc_shard_plan(const int32_t* idx, int64_t J, int world, int rank, int32_t* recv_src, int32_t* recv_row,
                     int64_t* send_cnt, int32_t* send_rows);
/* Propose + reweight the context's J_local particles, which are global slots
 * [j_offset, j_offset + J_local).  Writes the new (unnormalised) log-weights and
 * log_target_new of the local slots into caller DEVICE buffers (synchronous). */
int dasmc_gpu_shard_propose(dasmc_ctx* ctx, const dasmc_kernel_cfg* cfg, uint64_t seed, int64_t j_offset,
                            double* log_w_dev, double* log_target_new_dev);
/* Normalise / ESS / mean_log_target / resample decision and indices over the
 * gathered FULL vectors (device pointers, J_total entries, reference order);
 * writes idx_dev[J_total] (identity if not resampled), updates the local
 * log-weight slice, returns the record.  Positions are finalised locally
 * (divergent particles keep theta, smc.hpp:129-131). */
int dasmc_gpu_shard_resample(dasmc_ctx* ctx, const double* log_w_full_dev, const double* log_target_new_full_dev,
                             int64_t J_total, int64_t j_offset, uint64_t seed, int resample_kind, double fraction,
                             int resample_always, int32_t* idx_dev, dasmc_iter_record* record);
/* theta rows (internal device layout, row stride dasmc_gpu_row_floats floats):
 * pack local rows[n] into dst_dev; unpack src_dev into local slots[n] of the next ensemble. */
int64_t dasmc_gpu_row_floats(const dasmc_ctx* ctx);
int dasmc_gpu_pack_rows(dasmc_ctx* ctx, const int32_t* rows, int64_t n, float* dst_dev);
int dasmc_gpu_unpack_rows(dasmc_ctx* ctx, const float* src_dev, const int32_t* slots, int64_t n);

/* ---- single-process multi-GPU group --------------------------------------
 * One ensemble of up to max_particles particles sharded over ndev shard contexts, shard r on
 * devices[r] owning global slots [r*J/G, (r+1)*J/G) (parallel.hpp:30-31).  The returned
 * handle is used with the SAME hot-path entry points as a single context: set_target,
 * init_ensemble, set/get_ensemble(_f32), smc_step, sync_records, sda_moments, reserve_rows,
 * stream / timing (lead shard), destroy.  smc_step runs every shard's propose + reweight,
 * all-gathers the log-weights and log targets into every shard (peer copies over NVLink),
 * computes the same normalise / ESS / resampling indices redundantly on every shard, and
 * migrates resampled rows with a gather kernel that reads the owners' memory directly (P2P
 * loads, no host plan).  RNG streams are keyed by the GLOBAL slot, so results are identical
 * to one context for any G.  Devices may repeat (shards sharing a GPU: the in-process
 * emulation used by the single-GPU tests).  Other entry points return DASMC_EINVAL. */
int dasmc_gpu_create_multi(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n,
                           int max_particles, const int* devices, int ndev, int precision, dasmc_ctx** out);
int dasmc_gpu_multi_shards(const dasmc_ctx* ctx); /* G (1 for a single context) */

/* CUDA-graph replay of smc_step (single contexts; SURVEY.md §7 hard part 7: small configs are
 * launch-bound).  The step's kernels read the iteration / record slot / resampling key from
 * device memory, so one instantiated graph per step signature (buffer rotation, target,
 * kernel configuration, resampling options, allocations) replays every iteration with only
 * its first node's argument updated.  Results are bit-identical to eager launches.  Off by
 * default; ignored while the start-gradient cache is on. */
int dasmc_gpu_set_graphs(dasmc_ctx* ctx, int enable);

/* ---- instrumentation (bench.py) ------------------------------------------------------ */
/* The context's CUDA stream (cudaStream_t) -- every kernel of the context runs on it. */
void* dasmc_gpu_stream(dasmc_ctx* ctx);
/* Total kernel launches issued by this library in this process. */
int64_t dasmc_launch_count(void);
/* Enable CUDA-event timing of kernel ranges (0: layer-1 forward GEMM,
 * 1: layer-1 weight-gradient GEMM with the fused leapfrog, 2: whole gradient
 * evaluation); dasmc_gpu_kernel_times synchronises, returns the accumulated
 * milliseconds and range counts since the last reset, then resets. */
int dasmc_gpu_set_timing(dasmc_ctx* ctx, int enable);
int dasmc_gpu_kernel_times(dasmc_ctx* ctx, double* ms3, int64_t* count3);
/* Isolated timing of the step's memory-bound kernels on the context's buffers
 * (bench / profiling only; tools/membench.py): reps launches each of
 * 0: resample gather theta_new[j] = theta[idx[j]] (smc.hpp:97-99),
 * 1: sum of squares of J momentum rows (the kinetic term, kernels.hpp:89-95),
 * 2: momentum generation p ~ N(0, I) (smc.hpp:118-123, rng.hpp:76-81),
 * 3: weights / normalise / ESS / CDF / systematic search (smc.hpp:28-99).
 * idx (host, J entries in [0, J)) drives kernel 0.  ms4 = mean ms per launch,
 * bytes4 = algorithmic HBM bytes per launch. */
int dasmc_gpu_bench_memory(dasmc_ctx* ctx, int64_t J, const int32_t* idx, int reps, double* ms4, double* bytes4);

/* xoshiro256++ draws [skip, skip+count) of stream `key`, reached with the
 * F2-linear jump-ahead the device generator uses (host check of rng.hpp:48-58). */
int dasmc_rng_skip(uint64_t key, uint64_t skip, int64_t count, uint64_t* out);

/* ---- whole run (runner.hpp:453-617 hot loop) ---------------------------------------------
 * X/y UNshuffled; shuffles with fork(kPermutation), resolves the schedule,
 * init_ensemble, then per iteration: context_for -> smc_step -> sda_advance.
 * records[iterations]; sda_trace[iterations] may be NULL. */
int dasmc_gpu_run(const dasmc_net_desc* net, const float* X, const int32_t* y, int64_t n,
                  const dasmc_run_cfg* cfg, int device, int precision, dasmc_iter_record* records,
                  dasmc_sda_state* sda_trace, double* final_theta, double* final_log_weights);

#ifdef __cplusplus
}
#endif

#endif /* DASMC_GPU_H */
