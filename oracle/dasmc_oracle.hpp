// dasmc CPU ORACLE -- test infrastructure only, never shipped or measured as the product.
//
// A plain-C++20 (no Eigen) fp64 restatement of the reference hot path of
// arxiv/paper_2601_21983 (/root/reference/proj/include/dasmc/*.hpp).  Every
// function cites the reference file:line it follows.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it.
//
// Parity status: the reference cannot be compiled here (Eigen3, Catch2, CLI11
// absent), so this restatement is pinned against every inline
// known answer of the reference's own Catch2 tests (ported in
// oracle/oracle_tests.cpp) and the worked examples of SPEC.md.  RNG bit
// streams, smc_step, resampling, schedules and SDA have no reference golden
// vectors ("parity unpinned by reference tests" for those);
// they are pinned by SPEC.md worked examples and by this restatement's
// line-by-line reading of the reference algorithm.
//
// Extensions marked [EXT] are not in the reference: they resolve
// BASELINE.json-vs-reference mismatches and are the
// definition the GPU path must match.
#ifndef DASMC_ORACLE_HPP
#define DASMC_ORACLE_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <variant>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;
inline constexpr double kNegInf = -std::numeric_limits<double>::infinity();
inline constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

// ---------------------------------------------------------------- dense GEMM
// Row-major C[MxN] = alpha * op(A) * op(B) + beta * C.  An optional BLAS hook
// (set by the C-ABI from numpy's OpenBLAS, single-threaded per call) stands
// in for Eigen's dgemm; the fallback is a plain blocked loop.
using DgemmFn = void (*)(bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
                         int lda, const double* B, int ldb, double beta, double* C, int ldc);
inline DgemmFn& dgemm_hook() {
  static DgemmFn fn = nullptr;
  return fn;
}

inline void gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                 const double* B, int ldb, double beta, double* C, int ldc) {
  if (M <= 0 || N <= 0) return;
  if (dgemm_hook() && K > 0) {
    dgemm_hook()(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    return;
  }
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) C[(size_t)i * ldc + j] = beta == 0.0 ? 0.0 : beta * C[(size_t)i * ldc + j];
  // i-k-j loop order keeps the innermost loop contiguous in B and C.
  std::vector<double> arow((size_t)K);
  std::vector<double> brow((size_t)N);
  for (int i = 0; i < M; ++i) {
    for (int k = 0; k < K; ++k) arow[(size_t)k] = ta ? A[(size_t)k * lda + i] : A[(size_t)i * lda + k];
    double* c = C + (size_t)i * ldc;
    for (int k = 0; k < K; ++k) {
      const double a = alpha * arow[(size_t)k];
      if (a == 0.0) continue;
      if (!tb) {
        const double* b = B + (size_t)k * ldb;
        for (int j = 0; j < N; ++j) c[j] += a * b[j];
      } else {
        for (int j = 0; j < N; ++j) c[j] += a * B[(size_t)j * ldb + k];
      }
    }
  }
}

// ---------------------------------------------------------------- rng.hpp:14-113
inline std::uint64_t splitmix64(std::uint64_t x) {  // rng.hpp:14-19
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline std::uint64_t rotl64(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

class RngStream {  // rng.hpp:34-102
 public:
  explicit RngStream(std::uint64_t seed) : key_(seed) { reset(); }
  std::uint64_t key() const { return key_; }
  RngStream fork(std::uint64_t a, std::uint64_t b = 0, std::uint64_t c = 0) const {  // rng.hpp:40-46
    std::uint64_t k = splitmix64(key_ ^ 0x8e2f0c5a61d3b947ULL);
    k = splitmix64(k ^ a);
    k = splitmix64(k ^ b);
    k = splitmix64(k ^ c);
    return RngStream(k);
  }
  std::uint64_t next_u64() {  // rng.hpp:48-58 (xoshiro256++)
    const std::uint64_t out = rotl64(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl64(s_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }  // rng.hpp:61-63
  std::uint64_t uniform_below(std::uint64_t n) {                                 // rng.hpp:66-73
    if (n == 0) throw std::invalid_argument("uniform_below: n must be positive");
    const std::uint64_t limit = ~std::uint64_t{0} - (~std::uint64_t{0} % n);
    std::uint64_t x = next_u64();
    while (x >= limit) x = next_u64();
    return x % n;
  }
  double normal() {  // rng.hpp:76-81: Box-Muller, cos branch, 2 draws per normal
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  Vec normal_vector(std::int64_t dim) {  // rng.hpp:83-88
    if (dim < 1) throw std::invalid_argument("normal_vector: dim must be >= 1");
    Vec out((size_t)dim);
    for (auto& v : out) v = normal();
    return out;
  }
  const std::uint64_t* state() const { return s_; }

 private:
  void reset() {  // rng.hpp:91-98
    std::uint64_t s = key_;
    for (auto& w : s_) {
      s = splitmix64(s);
      w = s;
    }
    if ((s_[0] | s_[1] | s_[2] | s_[3]) == 0) s_[0] = 1;
  }
  std::uint64_t key_;
  std::uint64_t s_[4];
};

namespace tag {  // rng.hpp:106-113
inline constexpr std::uint64_t kInit = 1, kProposal = 2, kResample = 3, kPermutation = 4,
                               kSynthetic = 5, kRedraw = 6;
}

// ---------------------------------------------------------------- parallel.hpp:16-44
template <typename Fn>
void parallel_for(std::int64_t n, int threads, Fn&& fn) {
  if (n <= 0) return;
  if (threads <= 1 || n == 1) {
    for (std::int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  const std::int64_t workers = std::min<std::int64_t>(threads, n);
  std::vector<std::thread> pool;
  std::exception_ptr first;
  std::mutex mu;
  for (std::int64_t t = 0; t < workers; ++t) {
    const std::int64_t lo = n * t / workers, hi = n * (t + 1) / workers;
    pool.emplace_back([lo, hi, &fn, &first, &mu] {
      try {
        for (std::int64_t i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  if (first) std::rethrow_exception(first);
}

// ---------------------------------------------------------------- numeric.hpp
inline double logsumexp(const Vec& v) {  // numeric.hpp:19-30
  if (v.empty()) throw std::invalid_argument("logsumexp: empty input");
  double m = v[0];
  for (double x : v) m = std::max(m, x);
  if (m == kNegInf) throw std::invalid_argument("logsumexp: all entries are -inf");
  double s = 0.0;
  for (double x : v) s += std::exp(x - m);
  return m + std::log(s);
}

inline void check_normalized_weights(const Vec& w) {  // numeric.hpp:38-47
  if (w.empty()) throw std::invalid_argument("weights: empty");
  double s = 0.0;
  for (double x : w) {
    if (!(x >= 0.0)) throw std::invalid_argument("weights: entries must be >= 0");
    s += x;
  }
  if (std::abs(s - 1.0) > 1e-9) throw std::invalid_argument("weights: must sum to 1");
}

inline double dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

inline double weighted_mean(const Vec& values, const Vec& w) {  // numeric.hpp:49-54
  if (values.size() != w.size()) throw std::invalid_argument("weighted_mean: length mismatch");
  check_normalized_weights(w);
  return dot(w, values);
}

inline double weighted_var(const Vec& values, const Vec& w) {  // numeric.hpp:58-65
  if (values.size() != w.size()) throw std::invalid_argument("weighted_var: length mismatch");
  check_normalized_weights(w);
  const double mean = dot(w, values);
  double msq = 0.0;
  for (size_t i = 0; i < w.size(); ++i) msq += w[i] * (values[i] * values[i]);
  return std::max(0.0, msq - mean * mean);
}

inline double weighted_cov(const Vec& x, const Vec& y, const Vec& w) {  // numeric.hpp:68-78
  if (x.size() != y.size() || x.size() != w.size())
    throw std::invalid_argument("weighted_cov: length mismatch");
  check_normalized_weights(w);
  const double mx = dot(w, x), my = dot(w, y);
  double mxy = 0.0;
  for (size_t i = 0; i < w.size(); ++i) mxy += w[i] * (x[i] * y[i]);
  return mxy - mx * my;
}

// Sequential fp64 CDF with cdf.back() = 1.0 (numeric.hpp:87-94).
inline Vec cdf_of(const Vec& w) {
  Vec cdf(w.size());
  double acc = 0.0;
  for (size_t i = 0; i < w.size(); ++i) {
    acc += w[i];
    cdf[i] = acc;
  }
  cdf.back() = 1.0;
  return cdf;
}

// First index with cdf[idx] > u (std::upper_bound, numeric.hpp:97-98).
inline int upper_bound_index(const Vec& cdf, double u) {
  return static_cast<int>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
}

inline std::vector<int> sample_categorical(RngStream& rng, const Vec& w, int count) {  // numeric.hpp:81-101
  check_normalized_weights(w);
  if (count < 1) throw std::invalid_argument("sample_categorical: count must be >= 1");
  const Vec cdf = cdf_of(w);
  std::vector<int> out((size_t)count);
  for (auto& idx : out) idx = upper_bound_index(cdf, rng.uniform());
  return out;
}

// ---------------------------------------------------------------- network.hpp
enum class Activation { kRelu = 0, kTanh = 1 };

struct NetSpec {  // network.hpp:24-27
  std::vector<int> layer_sizes;
  Activation activation = Activation::kRelu;
};

inline void validate(const NetSpec& s) {  // network.hpp:29-34
  if (s.layer_sizes.size() < 2) throw std::invalid_argument("NetSpec: need at least input and output layers");
  for (int v : s.layer_sizes)
    if (v < 1) throw std::invalid_argument("NetSpec: layer sizes must be >= 1");
}

inline int param_count(const NetSpec& s) {  // network.hpp:36-42
  validate(s);
  int total = 0;
  for (size_t l = 1; l < s.layer_sizes.size(); ++l)
    total += s.layer_sizes[l - 1] * s.layer_sizes[l] + s.layer_sizes[l];
  return total;
}

struct PriorSpec {  // network.hpp:45-51
  double sigma = 1.0;
};
inline void validate(const PriorSpec& p) {
  if (!(p.sigma > 0.0)) throw std::invalid_argument("PriorSpec: sigma must be > 0");
}

// theta layout per layer l (network.hpp:55-62): W (out x in) column-major, i.e.
// W(r, c) at off + r + c*out, equivalently a row-major [in][out] matrix W^T;
// then the bias b[out].
inline void check_theta(const NetSpec& s, const Vec& theta) {
  if ((int64_t)theta.size() != param_count(s))
    throw std::invalid_argument("parameter vector length does not match NetSpec");
}

inline void apply_activation(double* z, size_t n, Activation a) {  // network.hpp:69-74
  if (a == Activation::kRelu)
    for (size_t i = 0; i < n; ++i) z[i] = std::max(z[i], 0.0);
  else
    for (size_t i = 0; i < n; ++i) z[i] = std::tanh(z[i]);
}

// forward_batch (network.hpp:79-99): logits, row-major [m x classes].
inline Vec forward_batch(const NetSpec& s, const double* theta, const double* X, int64_t m) {
  const size_t L = s.layer_sizes.size();
  Vec a, z;
  int off = 0;
  const double* below = X;
  for (size_t l = 1; l < L; ++l) {
    const int in = s.layer_sizes[l - 1], out = s.layer_sizes[l];
    z.assign((size_t)m * out, 0.0);
    // Z = A * W^T; W^T is the row-major [in][out] view of the column-major W.
    gemm(false, false, (int)m, out, in, 1.0, below, in, theta + off, out, 0.0, z.data(), out);
    off += in * out;
    for (int64_t i = 0; i < m; ++i)
      for (int r = 0; r < out; ++r) z[(size_t)i * out + r] += theta[off + r];
    off += out;
    if (l + 1 < L) apply_activation(z.data(), z.size(), s.activation);
    a.swap(z);
    below = a.data();
  }
  return a;
}

inline Vec forward_batch(const NetSpec& s, const Vec& theta, const double* X, int64_t m) {
  check_theta(s, theta);
  return forward_batch(s, theta.data(), X, m);
}

inline double log_softmax_at(const double* logits, int C, int label) {  // network.hpp:108-114
  if (label < 0 || label >= C) throw std::invalid_argument("label out of range");
  double mx = logits[0];
  for (int c = 1; c < C; ++c) mx = std::max(mx, logits[c]);
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += std::exp(logits[c] - mx);
  return logits[label] - (mx + std::log(s));
}

inline double loglik_batch(const NetSpec& s, const double* theta, const double* X, const int* y,
                           int64_t m) {  // network.hpp:124-141
  if (m < 1) throw std::invalid_argument("loglik_batch: empty batch");
  const Vec logits = forward_batch(s, theta, X, m);
  const int C = s.layer_sizes.back();
  double total = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    if (y[i] < 0 || y[i] >= C) throw std::invalid_argument("loglik_batch: label out of range");
    total += log_softmax_at(logits.data() + (size_t)i * C, C, y[i]);
  }
  return total;
}

// loglik_and_grad_batch (network.hpp:145-219).  grad has param_count entries
// in the reference theta layout; returns the summed log-likelihood.
// [EXT] dX (optional, [m x n0]): the gradient with respect to the inputs,
// delta_1 W_1 (no activation derivative), used by the CNN head.
inline double loglik_and_grad_batch(const NetSpec& s, const double* theta, const double* X,
                                    const int* y, int64_t m, double* grad, double* dX = nullptr) {
  if (m < 1) throw std::invalid_argument("loglik_and_grad_batch: empty batch");
  const size_t L = s.layer_sizes.size();
  const int C = s.layer_sizes.back();
  std::vector<Vec> acts(L - 1);
  std::vector<int> offs(L, 0);
  int off = 0;
  const double* below = X;
  for (size_t l = 1; l < L; ++l) {  // forward keeping post-activations (159-178)
    const int in = s.layer_sizes[l - 1], out = s.layer_sizes[l];
    offs[l] = off;
    Vec z((size_t)m * out, 0.0);
    gemm(false, false, (int)m, out, in, 1.0, below, in, theta + off, out, 0.0, z.data(), out);
    off += in * out;
    for (int64_t i = 0; i < m; ++i)
      for (int r = 0; r < out; ++r) z[(size_t)i * out + r] += theta[off + r];
    off += out;
    if (l + 1 < L) apply_activation(z.data(), z.size(), s.activation);
    acts[l - 1] = std::move(z);
    below = acts[l - 1].data();
  }
  // log-likelihood and residual onehot - softmax (180-193)
  Vec& logits = acts.back();
  double total = 0.0;
  std::vector<double> e((size_t)C);
  for (int64_t i = 0; i < m; ++i) {
    const int yi = y[i];
    if (yi < 0 || yi >= C) throw std::invalid_argument("loglik_and_grad_batch: label out of range");
    double* row = logits.data() + (size_t)i * C;
    double mx = row[0];
    for (int c = 1; c < C; ++c) mx = std::max(mx, row[c]);
    double denom = 0.0;
    for (int c = 0; c < C; ++c) {
      e[(size_t)c] = std::exp(row[c] - mx);
      denom += e[(size_t)c];
    }
    total += row[yi] - (mx + std::log(denom));
    for (int c = 0; c < C; ++c) row[c] = -(e[(size_t)c] / denom);
    row[yi] += 1.0;
  }
  // backward (195-217)
  Vec delta = std::move(logits);
  for (int l = (int)L - 1; l >= 1; --l) {
    const int in = s.layer_sizes[(size_t)l - 1], out = s.layer_sizes[(size_t)l];
    const double* A = l == 1 ? X : acts[(size_t)l - 2].data();
    // dW^T [in][out] = A^T (in x m) * delta (m x out)
    gemm(true, false, in, out, (int)m, 1.0, A, in, delta.data(), out, 0.0, grad + offs[(size_t)l], out);
    double* db = grad + offs[(size_t)l] + in * out;
    for (int r = 0; r < out; ++r) db[r] = 0.0;
    for (int64_t i = 0; i < m; ++i)
      for (int r = 0; r < out; ++r) db[r] += delta[(size_t)i * out + r];
    if (l > 1) {
      Vec next((size_t)m * in, 0.0);
      // next = delta (m x out) * W (out x in) = delta * (W^T)^T
      gemm(false, true, (int)m, in, out, 1.0, delta.data(), out, theta + offs[(size_t)l], out, 0.0,
           next.data(), in);
      const Vec& a = acts[(size_t)l - 2];
      if (s.activation == Activation::kRelu) {
        for (size_t i = 0; i < next.size(); ++i) next[i] *= (a[i] > 0.0 ? 1.0 : 0.0);
      } else {
        for (size_t i = 0; i < next.size(); ++i) next[i] *= (1.0 - a[i] * a[i]);
      }
      delta = std::move(next);
    } else if (dX != nullptr) {
      gemm(false, true, (int)m, in, out, 1.0, delta.data(), out, theta + offs[(size_t)l], out, 0.0, dX, in);
    }
  }
  return total;
}

inline double sqnorm(const double* v, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i] * v[i];
  return s;
}

inline double prior_logpdf(const PriorSpec& p, const double* theta, size_t d) {  // network.hpp:221-227
  validate(p);
  constexpr double kLogTwoPi = 1.8378770664093455;
  const double var = p.sigma * p.sigma;
  return -0.5 * (double)d * (kLogTwoPi + std::log(var)) - sqnorm(theta, d) / (2.0 * var);
}

inline Vec sample_gaussian_prior(const PriorSpec& p, int64_t dim, RngStream& rng) {  // network.hpp:235-239
  validate(p);
  Vec v = rng.normal_vector(dim);
  for (auto& x : v) x *= p.sigma;
  return v;
}

// ---------------------------------------------------------------- dataset.hpp
struct SubsetWindow {  // dataset.hpp:32-41
  int64_t prefix_end = 0, block_end = 0, total_n = 0;
};
inline void validate(const SubsetWindow& w) {
  if (w.prefix_end < 0 || w.prefix_end > w.block_end || w.block_end > w.total_n)
    throw std::invalid_argument("SubsetWindow: need 0 <= prefix_end <= block_end <= total_n");
}

struct Dataset {  // dataset.hpp:46-56 (row-major fp64 features)
  int64_t n = 0;
  int d = 0;
  Vec features;
  std::vector<int> labels;
  Vec targets;
  int num_classes = 0;
  std::vector<int64_t> perm;
  const double* row(int64_t i) const { return features.data() + (size_t)i * d; }
};

inline Dataset shuffled(const Dataset& src, RngStream& rng) {  // dataset.hpp:294-316
  const int64_t n = src.n;
  std::vector<int64_t> order((size_t)n);
  for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
  for (int64_t i = n - 1; i > 0; --i) {
    const auto j = (int64_t)rng.uniform_below((std::uint64_t)(i + 1));
    std::swap(order[(size_t)i], order[(size_t)j]);
  }
  Dataset out;
  out.n = n;
  out.d = src.d;
  out.num_classes = src.num_classes;
  out.features.resize((size_t)n * src.d);
  if (!src.labels.empty()) out.labels.resize((size_t)n);
  if (!src.targets.empty()) out.targets.resize((size_t)n);
  out.perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t s = order[(size_t)i];
    std::memcpy(out.features.data() + (size_t)i * src.d, src.row(s), sizeof(double) * src.d);
    if (!src.labels.empty()) out.labels[(size_t)i] = src.labels[(size_t)s];
    if (!src.targets.empty()) out.targets[(size_t)i] = src.targets[(size_t)s];
    out.perm[(size_t)i] = src.perm.empty() ? s : src.perm[(size_t)s];
  }
  return out;
}

inline Dataset gather(const Dataset& src, const std::vector<int64_t>& rows) {  // dataset.hpp:334-351
  Dataset out;
  out.n = (int64_t)rows.size();
  out.d = src.d;
  out.num_classes = src.num_classes;
  out.features.resize(rows.size() * (size_t)src.d);
  if (!src.labels.empty()) out.labels.resize(rows.size());
  if (!src.targets.empty()) out.targets.resize(rows.size());
  out.perm.resize(rows.size());
  for (size_t i = 0; i < rows.size(); ++i) {
    const int64_t s = rows[i];
    if (s < 0 || s >= src.n) throw std::invalid_argument("gather: row index out of range");
    std::memcpy(out.features.data() + i * src.d, src.row(s), sizeof(double) * src.d);
    if (!src.labels.empty()) out.labels[i] = src.labels[(size_t)s];
    if (!src.targets.empty()) out.targets[i] = src.targets[(size_t)s];
    out.perm[i] = src.perm.empty() ? s : src.perm[(size_t)s];
  }
  return out;
}

enum class SyntheticKind { kGaussianBlobs, kTwoMoons, kLinearGaussian };

struct SyntheticData {
  Dataset data;
  Vec true_theta;
  double noise_std = 0.0;
};

inline SyntheticData make_synthetic(SyntheticKind kind, int64_t n, double noise, std::uint64_t seed,
                                    int dim = 2) {  // dataset.hpp:208-267
  if (n < 2) throw std::invalid_argument("make_synthetic: n must be >= 2");
  RngStream rng = RngStream(seed).fork(tag::kSynthetic);
  SyntheticData out;
  Dataset& d = out.data;
  d.n = n;
  constexpr double kPi = 3.141592653589793;
  switch (kind) {
    case SyntheticKind::kGaussianBlobs: {
      d.d = 2;
      d.features.resize((size_t)n * 2);
      d.labels.resize((size_t)n);
      for (int64_t i = 0; i < n; ++i) {
        const int c = (int)(i % 3);
        const double angle = 2.0 * kPi * c / 3;
        d.features[(size_t)i * 2] = 3.0 * std::cos(angle) + noise * rng.normal();
        d.features[(size_t)i * 2 + 1] = 3.0 * std::sin(angle) + noise * rng.normal();
        d.labels[(size_t)i] = c;
      }
      d.num_classes = 3;
      break;
    }
    case SyntheticKind::kTwoMoons: {
      d.d = 2;
      d.features.resize((size_t)n * 2);
      d.labels.resize((size_t)n);
      for (int64_t i = 0; i < n; ++i) {
        const int c = (int)(i % 2);
        const double t = kPi * rng.uniform();
        double x, y;
        if (c == 0) {
          x = std::cos(t);
          y = std::sin(t);
        } else {
          x = 1.0 - std::cos(t);
          y = 0.5 - std::sin(t);
        }
        d.features[(size_t)i * 2] = x + noise * rng.normal();
        d.features[(size_t)i * 2 + 1] = y + noise * rng.normal();
        d.labels[(size_t)i] = c;
      }
      d.num_classes = 2;
      break;
    }
    case SyntheticKind::kLinearGaussian: {
      d.d = dim;
      d.features.resize((size_t)n * dim);
      d.targets.resize((size_t)n);
      out.true_theta = rng.normal_vector(dim);
      out.noise_std = noise;
      for (int64_t i = 0; i < n; ++i) {
        for (int j = 0; j < dim; ++j) d.features[(size_t)i * dim + j] = rng.normal();
        double acc = 0.0;  // row . true_theta (Eigen dot; order may differ in the last ulp)
        for (int j = 0; j < dim; ++j) acc += d.features[(size_t)i * dim + j] * out.true_theta[(size_t)j];
        d.targets[(size_t)i] = acc + noise * rng.normal();
      }
      d.num_classes = 0;
      break;
    }
  }
  d.perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) d.perm[(size_t)i] = i;
  return out;
}

// [EXT] teacher-labelled synthetic data for BASELINE.json configs (SURVEY.md
// §8d, Appendix A.5).  Features from RngStream(seed).fork(kSynthetic, cfg_id, 1)
// in row-major order: kind 0 -> uniform() in [0,1); kind 1 -> k/255 with
// k = uniform_below(256).  Teacher theta ~ N(0, I) from fork(kSynthetic,
// cfg_id, 2) in the reference layout.  label = argmax of the teacher logits,
// evaluated with plain ascending-index fp64 loops (first max wins).
inline Vec teacher_logits_row(const NetSpec& s, const double* theta, const double* x) {
  Vec cur(x, x + s.layer_sizes[0]), nxt;
  int off = 0;
  for (size_t l = 1; l < s.layer_sizes.size(); ++l) {
    const int in = s.layer_sizes[l - 1], out = s.layer_sizes[l];
    nxt.assign((size_t)out, 0.0);
    for (int r = 0; r < out; ++r) {
      double acc = 0.0;
      for (int c = 0; c < in; ++c) acc += theta[off + c * out + r] * cur[(size_t)c];
      acc += theta[off + in * out + r];
      if (l + 1 < s.layer_sizes.size())
        acc = s.activation == Activation::kRelu ? (acc > 0.0 ? acc : 0.0) : std::tanh(acc);
      nxt[(size_t)r] = acc;
    }
    off += in * out + out;
    cur.swap(nxt);
  }
  return cur;
}

inline Dataset make_teacher_dataset(const NetSpec& teacher, int64_t n, int feature_kind,
                                    std::uint64_t seed, std::uint64_t cfg_id, int threads = 1) {
  validate(teacher);
  Dataset d;
  d.n = n;
  d.d = teacher.layer_sizes.front();
  d.num_classes = teacher.layer_sizes.back();
  d.features.resize((size_t)n * d.d);
  d.labels.resize((size_t)n);
  RngStream fx = RngStream(seed).fork(tag::kSynthetic, cfg_id, 1);
  for (auto& v : d.features) v = feature_kind == 0 ? fx.uniform() : (double)fx.uniform_below(256) / 255.0;
  RngStream ft = RngStream(seed).fork(tag::kSynthetic, cfg_id, 2);
  const Vec th = ft.normal_vector(param_count(teacher));
  parallel_for(n, threads, [&](int64_t i) {
    const Vec z = teacher_logits_row(teacher, th.data(), d.row(i));
    int best = 0;
    for (int c = 1; c < (int)z.size(); ++c)
      if (z[(size_t)c] > z[(size_t)best]) best = c;
    d.labels[(size_t)i] = best;
  });
  d.perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) d.perm[(size_t)i] = i;
  return d;
}

// ---------------------------------------------------------------- [EXT] CNN models
// BASELINE.json configs[2..3].  The reference is MLP-only
// (network.hpp:21-27), so these layers are new and parity here is pinned by
// finite differences / naive loops / torch fp64 autograd (tests/), not by the
// reference.  Semantics (stated in DESIGN.md):
//   * a conv stage is a valid 2-D convolution, stride 1, W[cout][cin][k][k]
//     row-major then b[cout]; the network activation follows every convolution;
//     an optional 2x2 / stride-2 max-pool follows (floor for odd sizes) whose
//     backward routes to the FIRST maximum of the window in (dy, dx) order;
//   * images are [c][h][w] (w fastest); the last stage output is flattened in
//     that order and fed to a reference MLP (`head`, network.hpp) whose input
//     size is the flatten size;
//   * theta = the conv stages in order, then the head in the reference layout.
struct ConvSpec {
  int k = 3, cout = 1;
  bool pool = false;
};
struct CnnSpec {
  int in_c = 1, in_h = 1, in_w = 1;
  std::vector<ConvSpec> convs;
  NetSpec head;
};
struct ConvDims {
  int cin, hin, win, k, cout, ho, wo, sh, sw;  // sh x sw = stage output (after the pool)
  bool pool;
  int64_t woff, boff;  // offsets in theta
};

inline std::vector<ConvDims> conv_dims(const CnnSpec& s) {
  std::vector<ConvDims> out;
  int c = s.in_c, h = s.in_h, w = s.in_w;
  int64_t off = 0;
  for (const ConvSpec& cs : s.convs) {
    ConvDims d;
    d.cin = c;
    d.hin = h;
    d.win = w;
    d.k = cs.k;
    d.cout = cs.cout;
    d.ho = h - cs.k + 1;
    d.wo = w - cs.k + 1;
    d.pool = cs.pool;
    d.sh = cs.pool ? d.ho / 2 : d.ho;
    d.sw = cs.pool ? d.wo / 2 : d.wo;
    if (cs.k < 1 || cs.cout < 1 || d.ho < 1 || d.wo < 1 || d.sh < 1 || d.sw < 1)
      throw std::invalid_argument("CnnSpec: convolution does not fit its input");
    d.woff = off;
    off += (int64_t)cs.cout * c * cs.k * cs.k;
    d.boff = off;
    off += cs.cout;
    out.push_back(d);
    c = cs.cout;
    h = d.sh;
    w = d.sw;
  }
  return out;
}
inline int64_t cnn_conv_params(const CnnSpec& s) {
  const auto d = conv_dims(s);
  return d.back().boff + d.back().cout;
}
inline int64_t flatten_size(const CnnSpec& s) {
  const auto d = conv_dims(s);
  return (int64_t)d.back().cout * d.back().sh * d.back().sw;
}
inline void validate(const CnnSpec& s) {
  if (s.in_c < 1 || s.in_h < 1 || s.in_w < 1) throw std::invalid_argument("CnnSpec: bad input shape");
  if (s.convs.empty()) throw std::invalid_argument("CnnSpec: need at least one convolution");
  validate(s.head);
  if (s.head.layer_sizes[0] != flatten_size(s))
    throw std::invalid_argument("CnnSpec: head input size must equal the flatten size");
}
inline int cnn_param_count(const CnnSpec& s) {
  validate(s);
  return (int)(cnn_conv_params(s) + param_count(s.head));
}

inline double act_of(double z, Activation a) { return a == Activation::kRelu ? (z > 0.0 ? z : 0.0) : std::tanh(z); }
inline double act_grad_from_post(double a, Activation act) {  // network.hpp:211-214 convention
  return act == Activation::kRelu ? (a > 0.0 ? 1.0 : 0.0) : 1.0 - a * a;
}

// Conv stages of one image; acts[i] = post-activation (pre-pool) [cout][ho][wo],
// outs[i] = stage output [cout][sh][sw] (== acts[i] without a pool).
inline void cnn_stages(const CnnSpec& s, const std::vector<ConvDims>& dims, const double* theta, const double* x,
                       std::vector<Vec>& acts, std::vector<Vec>& outs) {
  acts.resize(dims.size());
  outs.resize(dims.size());
  const double* in = x;
  for (size_t i = 0; i < dims.size(); ++i) {
    const ConvDims& d = dims[i];
    Vec& A = acts[i];
    A.assign((size_t)d.cout * d.ho * d.wo, 0.0);
    for (int co = 0; co < d.cout; ++co)
      for (int y = 0; y < d.ho; ++y)
        for (int xx = 0; xx < d.wo; ++xx) {
          double acc = 0.0;
          for (int ci = 0; ci < d.cin; ++ci)
            for (int ky = 0; ky < d.k; ++ky)
              for (int kx = 0; kx < d.k; ++kx)
                acc += theta[d.woff + (((int64_t)co * d.cin + ci) * d.k + ky) * d.k + kx] *
                       in[((size_t)ci * d.hin + y + ky) * d.win + xx + kx];
          acc += theta[d.boff + co];
          A[((size_t)co * d.ho + y) * d.wo + xx] = act_of(acc, s.head.activation);
        }
    if (d.pool) {
      Vec& P = outs[i];
      P.assign((size_t)d.cout * d.sh * d.sw, 0.0);
      for (int co = 0; co < d.cout; ++co)
        for (int y = 0; y < d.sh; ++y)
          for (int xx = 0; xx < d.sw; ++xx) {
            double mx = A[((size_t)co * d.ho + 2 * y) * d.wo + 2 * xx];
            for (int dy = 0; dy < 2; ++dy)
              for (int dx = 0; dx < 2; ++dx) mx = std::max(mx, A[((size_t)co * d.ho + 2 * y + dy) * d.wo + 2 * xx + dx]);
            P[((size_t)co * d.sh + y) * d.sw + xx] = mx;
          }
    } else {
      outs[i] = A;
    }
    in = outs[i].data();
  }
}

// Backward through the conv stages of one image given dflat = d ll / d(flatten);
// accumulates into grad (conv block of theta).
inline void cnn_stages_backward(const CnnSpec& s, const std::vector<ConvDims>& dims, const double* theta,
                                const double* x, const std::vector<Vec>& acts, const std::vector<Vec>& outs,
                                const double* dflat, double* grad) {
  Vec dout(dflat, dflat + outs.back().size());
  for (int i = (int)dims.size() - 1; i >= 0; --i) {
    const ConvDims& d = dims[(size_t)i];
    const Vec& A = acts[(size_t)i];
    Vec dz(A.size(), 0.0);
    if (d.pool) {
      for (int co = 0; co < d.cout; ++co)
        for (int y = 0; y < d.sh; ++y)
          for (int xx = 0; xx < d.sw; ++xx) {
            int by = 0, bx = 0;
            double mx = A[((size_t)co * d.ho + 2 * y) * d.wo + 2 * xx];
            for (int dy = 0; dy < 2; ++dy)
              for (int dx = 0; dx < 2; ++dx) {
                const double v = A[((size_t)co * d.ho + 2 * y + dy) * d.wo + 2 * xx + dx];
                if (v > mx) {
                  mx = v;
                  by = dy;
                  bx = dx;
                }
              }
            dz[((size_t)co * d.ho + 2 * y + by) * d.wo + 2 * xx + bx] = dout[((size_t)co * d.sh + y) * d.sw + xx];
          }
    } else {
      dz = dout;
    }
    for (size_t t = 0; t < dz.size(); ++t) dz[t] *= act_grad_from_post(A[t], s.head.activation);
    const double* in = i == 0 ? x : outs[(size_t)i - 1].data();
    for (int co = 0; co < d.cout; ++co) {
      double gb = 0.0;
      for (int y = 0; y < d.ho; ++y)
        for (int xx = 0; xx < d.wo; ++xx) gb += dz[((size_t)co * d.ho + y) * d.wo + xx];
      grad[d.boff + co] += gb;
      for (int ci = 0; ci < d.cin; ++ci)
        for (int ky = 0; ky < d.k; ++ky)
          for (int kx = 0; kx < d.k; ++kx) {
            double g = 0.0;
            for (int y = 0; y < d.ho; ++y)
              for (int xx = 0; xx < d.wo; ++xx)
                g += dz[((size_t)co * d.ho + y) * d.wo + xx] * in[((size_t)ci * d.hin + y + ky) * d.win + xx + kx];
            grad[d.woff + (((int64_t)co * d.cin + ci) * d.k + ky) * d.k + kx] += g;
          }
    }
    if (i > 0) {
      Vec din((size_t)d.cin * d.hin * d.win, 0.0);
      for (int ci = 0; ci < d.cin; ++ci)
        for (int y = 0; y < d.hin; ++y)
          for (int xx = 0; xx < d.win; ++xx) {
            double acc = 0.0;
            for (int co = 0; co < d.cout; ++co)
              for (int ky = 0; ky < d.k; ++ky)
                for (int kx = 0; kx < d.k; ++kx) {
                  const int oy = y - ky, ox = xx - kx;
                  if (oy < 0 || ox < 0 || oy >= d.ho || ox >= d.wo) continue;
                  acc += dz[((size_t)co * d.ho + oy) * d.wo + ox] *
                         theta[d.woff + (((int64_t)co * d.cin + ci) * d.k + ky) * d.k + kx];
                }
            din[((size_t)ci * d.hin + y) * d.win + xx] = acc;
          }
      dout.swap(din);
    }
  }
}

inline Vec cnn_flatten_batch(const CnnSpec& s, const double* theta, const double* X, int64_t m) {
  const auto dims = conv_dims(s);
  const int64_t in_sz = (int64_t)s.in_c * s.in_h * s.in_w, F = flatten_size(s);
  Vec flat((size_t)(m * F));
  std::vector<Vec> acts, outs;
  for (int64_t i = 0; i < m; ++i) {
    cnn_stages(s, dims, theta, X + i * in_sz, acts, outs);
    std::copy(outs.back().begin(), outs.back().end(), flat.begin() + i * F);
  }
  return flat;
}

inline double cnn_loglik_batch(const CnnSpec& s, const double* theta, const double* X, const int* y, int64_t m) {
  const Vec flat = cnn_flatten_batch(s, theta, X, m);
  return loglik_batch(s.head, theta + cnn_conv_params(s), flat.data(), y, m);
}

inline double cnn_loglik_and_grad_batch(const CnnSpec& s, const double* theta, const double* X, const int* y,
                                        int64_t m, double* grad) {
  if (m < 1) throw std::invalid_argument("cnn_loglik_and_grad_batch: empty batch");
  const auto dims = conv_dims(s);
  const int64_t in_sz = (int64_t)s.in_c * s.in_h * s.in_w, F = flatten_size(s), Pc = cnn_conv_params(s);
  const Vec flat = cnn_flatten_batch(s, theta, X, m);
  Vec dflat((size_t)(m * F));
  const double ll = loglik_and_grad_batch(s.head, theta + Pc, flat.data(), y, m, grad + Pc, dflat.data());
  for (int64_t t = 0; t < Pc; ++t) grad[t] = 0.0;
  std::vector<Vec> acts, outs;
  for (int64_t i = 0; i < m; ++i) {
    cnn_stages(s, dims, theta, X + i * in_sz, acts, outs);
    cnn_stages_backward(s, dims, theta, X + i * in_sz, acts, outs, dflat.data() + i * F, grad);
  }
  return ll;
}

inline Dataset make_teacher_dataset(const CnnSpec& teacher, int64_t n, int feature_kind, std::uint64_t seed,
                                    std::uint64_t cfg_id, int threads = 1) {
  validate(teacher);
  Dataset d;
  d.n = n;
  d.d = teacher.in_c * teacher.in_h * teacher.in_w;
  d.num_classes = teacher.head.layer_sizes.back();
  d.features.resize((size_t)n * d.d);
  d.labels.resize((size_t)n);
  RngStream fx = RngStream(seed).fork(tag::kSynthetic, cfg_id, 1);
  for (auto& v : d.features) v = feature_kind == 0 ? fx.uniform() : (double)fx.uniform_below(256) / 255.0;
  RngStream ft = RngStream(seed).fork(tag::kSynthetic, cfg_id, 2);
  const Vec th = ft.normal_vector(cnn_param_count(teacher));
  const auto dims = conv_dims(teacher);
  const int64_t Pc = cnn_conv_params(teacher);
  parallel_for(n, threads, [&](int64_t i) {
    std::vector<Vec> acts, outs;
    cnn_stages(teacher, dims, th.data(), d.row(i), acts, outs);
    const Vec z = teacher_logits_row(teacher.head, th.data() + Pc, outs.back().data());
    int best = 0;
    for (int c = 1; c < (int)z.size(); ++c)
      if (z[(size_t)c] > z[(size_t)best]) best = c;
    d.labels[(size_t)i] = best;
  });
  d.perm.resize((size_t)n);
  for (int64_t i = 0; i < n; ++i) d.perm[(size_t)i] = i;
  return d;
}

// ---------------------------------------------------------------- target.hpp
struct LinearGaussianSpec {  // target.hpp:19-22
  int dim = 1;
  double noise_std = 1.0;
};
using ModelSpec = std::variant<NetSpec, LinearGaussianSpec, CnnSpec>;  // CnnSpec: [EXT]

inline int model_param_count(const ModelSpec& m) {  // target.hpp:26-29
  if (const auto* net = std::get_if<NetSpec>(&m)) return param_count(*net);
  if (const auto* cnn = std::get_if<CnnSpec>(&m)) return cnn_param_count(*cnn);
  return std::get<LinearGaussianSpec>(m).dim;
}

struct ValueGrad {  // target.hpp:31-34
  double value = 0.0;
  Vec grad;
};

inline double lingauss_loglik(const LinearGaussianSpec& m, const Dataset& d, int64_t lo, int64_t hi,
                              const double* theta, double* grad) {  // target.hpp:38-58
  constexpr double kLogTwoPi = 1.8378770664093455;
  const double var = m.noise_std * m.noise_std;
  double ss = 0.0;
  if (grad)
    for (int j = 0; j < m.dim; ++j) grad[j] = 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    double pred = 0.0;
    for (int j = 0; j < m.dim; ++j) pred += d.row(i)[j] * theta[j];
    const double r = d.targets[(size_t)i] - pred;
    ss += r * r;
    if (grad)
      for (int j = 0; j < m.dim; ++j) grad[j] += d.row(i)[j] * r;
  }
  if (grad)
    for (int j = 0; j < m.dim; ++j) grad[j] /= var;
  return -0.5 * (double)(hi - lo) * (kLogTwoPi + std::log(var)) - ss / (2.0 * var);
}

// segment_loglik / segment_loglik_grad over rows [lo, hi) (target.hpp:63-89).
inline double segment_loglik(const ModelSpec& model, const Dataset& d, int64_t lo, int64_t hi,
                             const double* theta) {
  if (hi <= lo) return 0.0;
  if (const auto* net = std::get_if<NetSpec>(&model))
    return loglik_batch(*net, theta, d.row(lo), d.labels.data() + lo, hi - lo);
  if (const auto* cnn = std::get_if<CnnSpec>(&model))
    return cnn_loglik_batch(*cnn, theta, d.row(lo), d.labels.data() + lo, hi - lo);
  return lingauss_loglik(std::get<LinearGaussianSpec>(model), d, lo, hi, theta, nullptr);
}

inline double segment_loglik_grad(const ModelSpec& model, const Dataset& d, int64_t lo, int64_t hi,
                                  const double* theta, double* grad) {
  const int D = model_param_count(model);
  if (hi <= lo) {
    for (int i = 0; i < D; ++i) grad[i] = 0.0;
    return 0.0;
  }
  if (const auto* net = std::get_if<NetSpec>(&model))
    return loglik_and_grad_batch(*net, theta, d.row(lo), d.labels.data() + lo, hi - lo, grad);
  if (const auto* cnn = std::get_if<CnnSpec>(&model))
    return cnn_loglik_and_grad_batch(*cnn, theta, d.row(lo), d.labels.data() + lo, hi - lo, grad);
  return lingauss_loglik(std::get<LinearGaussianSpec>(model), d, lo, hi, theta, grad);
}

enum class TargetMode { kScaled = 0, kSda = 1 };

struct TargetContext {  // target.hpp:95-102
  const Dataset* data = nullptr;
  SubsetWindow window;
  TargetMode mode = TargetMode::kScaled;
  double beta = 1.0;
  PriorSpec prior;
  ModelSpec model;
};

inline void validate(const TargetContext& c) {  // target.hpp:104-113
  validate(c.prior);
  if (c.data == nullptr) return;
  validate(c.window);
  if (c.window.block_end < 1) throw std::invalid_argument("TargetContext: empty subset");
  if (c.window.block_end > c.data->n) throw std::invalid_argument("TargetContext: window exceeds dataset");
  if (c.mode == TargetMode::kSda && !(c.beta > 0.0 && c.beta <= 1.0))
    throw std::invalid_argument("TargetContext: sda mode needs beta in (0, 1]");
}

struct LoglikParts {
  double prefix = 0.0, block = 0.0;
};

inline LoglikParts unscaled_loglik_parts(const Dataset& d, const SubsetWindow& w,
                                         const ModelSpec& model, const double* theta) {  // target.hpp:121-129
  validate(w);
  if (w.block_end > d.n) throw std::invalid_argument("unscaled_loglik_parts: window exceeds dataset");
  return {segment_loglik(model, d, 0, w.prefix_end, theta),
          segment_loglik(model, d, w.prefix_end, w.block_end, theta)};
}

inline double log_target(const TargetContext& c, const double* theta) {  // target.hpp:131-145
  validate(c);
  const int D = model_param_count(c.model);
  double v = prior_logpdf(c.prior, theta, (size_t)D);
  if (c.data == nullptr) return v;
  if (c.mode == TargetMode::kScaled) {
    const double scale = (double)c.window.total_n / (double)c.window.block_end;
    v += scale * segment_loglik(c.model, *c.data, 0, c.window.block_end, theta);
  } else {
    v += segment_loglik(c.model, *c.data, 0, c.window.prefix_end, theta);
    v += c.beta * segment_loglik(c.model, *c.data, c.window.prefix_end, c.window.block_end, theta);
  }
  return v;
}

inline ValueGrad log_target_with_grad(const TargetContext& c, const double* theta) {  // target.hpp:147-173
  validate(c);
  const int D = model_param_count(c.model);
  ValueGrad vg;
  vg.value = prior_logpdf(c.prior, theta, (size_t)D);
  vg.grad.resize((size_t)D);
  const double inv_var = 1.0 / (c.prior.sigma * c.prior.sigma);
  for (int i = 0; i < D; ++i) vg.grad[(size_t)i] = -theta[i] * inv_var;  // network.hpp:232 (-theta/sigma^2)
  if (c.data == nullptr) return vg;
  Vec g((size_t)D);
  if (c.mode == TargetMode::kScaled) {
    const double scale = (double)c.window.total_n / (double)c.window.block_end;
    const double ll = segment_loglik_grad(c.model, *c.data, 0, c.window.block_end, theta, g.data());
    vg.value += scale * ll;
    for (int i = 0; i < D; ++i) vg.grad[(size_t)i] += scale * g[(size_t)i];
  } else {
    if (c.window.prefix_end > 0) {
      const double ll = segment_loglik_grad(c.model, *c.data, 0, c.window.prefix_end, theta, g.data());
      vg.value += ll;
      for (int i = 0; i < D; ++i) vg.grad[(size_t)i] += g[(size_t)i];
    }
    if (c.window.block_end > c.window.prefix_end) {
      const double ll =
          segment_loglik_grad(c.model, *c.data, c.window.prefix_end, c.window.block_end, theta, g.data());
      vg.value += c.beta * ll;
      for (int i = 0; i < D; ++i) vg.grad[(size_t)i] += c.beta * g[(size_t)i];
    }
  }
  return vg;
}

// ContextTarget adapter (target.hpp:180-190) generalised to any callable.
struct ContextTarget {
  const TargetContext* ctx;
  int dim() const { return model_param_count(ctx->model); }
  ValueGrad value_and_grad(const Vec& theta) const { return log_target_with_grad(*ctx, theta.data()); }
};

using TargetFn = std::function<ValueGrad(const Vec&)>;

// ---------------------------------------------------------------- kernels.hpp
enum class KernelKind { kHmc = 0, kLangevin = 1 };

struct KernelConfig {  // kernels.hpp:26-49
  double step_size = 0.0;
  int leapfrog_steps = 1;
  KernelKind kind = KernelKind::kHmc;
  static void validate(const KernelConfig& c) {
    if (!(c.step_size > 0.0)) throw std::invalid_argument("KernelConfig: step_size must be > 0");
    if (c.leapfrog_steps < 1) throw std::invalid_argument("KernelConfig: leapfrog_steps must be >= 1");
    if (c.kind == KernelKind::kLangevin && c.leapfrog_steps != 1)
      throw std::invalid_argument("KernelConfig: langevin requires leapfrog_steps == 1");
  }
  static KernelConfig hmc(double h, int s) {
    KernelConfig c{h, s, KernelKind::kHmc};
    validate(c);
    return c;
  }
  static KernelConfig langevin(double h) {
    KernelConfig c{h, 1, KernelKind::kLangevin};
    validate(c);
    return c;
  }
};

struct DivergenceError : std::runtime_error {  // kernels.hpp:53-61
  explicit DivergenceError(int s) : std::runtime_error("leapfrog diverged at step " + std::to_string(s)), step(s) {}
  int step;
};

inline bool all_finite(const Vec& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

struct Trajectory {
  Vec theta, momentum;
  double value_start = 0.0, value_end = 0.0;
};

// detail::integrate (kernels.hpp:75-99): S+1 value_and_grad evaluations.
template <typename Target>
Trajectory integrate(const Target& target, const Vec& theta0, const Vec& p0, const KernelConfig& cfg) {
  KernelConfig::validate(cfg);
  if (theta0.size() != p0.size()) throw std::invalid_argument("leapfrog: position/momentum dimension mismatch");
  const double h = cfg.step_size;
  Trajectory t{theta0, p0, 0.0, 0.0};
  ValueGrad vg = target.value_and_grad(t.theta);
  t.value_start = vg.value;
  if (!std::isfinite(vg.value) || !all_finite(vg.grad)) throw DivergenceError(0);
  const size_t D = theta0.size();
  for (int s = 0; s < cfg.leapfrog_steps; ++s) {
    for (size_t i = 0; i < D; ++i) t.momentum[i] += 0.5 * h * vg.grad[i];
    for (size_t i = 0; i < D; ++i) t.theta[i] += h * t.momentum[i];
    if (!all_finite(t.theta)) throw DivergenceError(s);
    vg = target.value_and_grad(t.theta);
    if (!std::isfinite(vg.value) || !all_finite(vg.grad)) throw DivergenceError(s);
    for (size_t i = 0; i < D; ++i) t.momentum[i] += 0.5 * h * vg.grad[i];
    if (!all_finite(t.momentum)) throw DivergenceError(s);
  }
  t.value_end = vg.value;
  return t;
}

template <typename Target>
std::pair<Vec, Vec> leapfrog(const Target& target, const Vec& theta, const Vec& p0,
                             const KernelConfig& cfg) {  // kernels.hpp:105-112
  Trajectory t = integrate(target, theta, p0, cfg);
  return {std::move(t.theta), std::move(t.momentum)};
}

struct ProposalResult {  // kernels.hpp:117-125
  Vec theta_new, p_initial, p_final;
  double log_target_new = 0.0, log_target_old = 0.0;
  bool divergent = false;
  int divergence_step = -1;
};

template <typename Target>
ProposalResult propose(const Target& target, const Vec& theta, const KernelConfig& cfg,
                       RngStream& rng) {  // kernels.hpp:127-147
  ProposalResult r;
  r.p_initial = rng.normal_vector((int64_t)theta.size());
  try {
    Trajectory t = integrate(target, theta, r.p_initial, cfg);
    r.theta_new = std::move(t.theta);
    r.p_final = std::move(t.momentum);
    r.log_target_new = t.value_end;
    r.log_target_old = t.value_start;
  } catch (const DivergenceError& e) {
    r.theta_new = theta;
    r.p_final = r.p_initial;
    r.log_target_new = kNaN;
    r.log_target_old = kNaN;
    r.divergent = true;
    r.divergence_step = e.step;
  }
  return r;
}

inline double incremental_log_weight(double lt_new, double lt_old, const Vec& p0,
                                     const Vec& ps) {  // kernels.hpp:153-163
  if (p0.size() != ps.size()) throw std::invalid_argument("incremental_log_weight: momentum dimension mismatch");
  if (!std::isfinite(lt_new) || !std::isfinite(lt_old) || !all_finite(p0) || !all_finite(ps)) return kNegInf;
  return (lt_new - lt_old) + 0.5 * (sqnorm(p0.data(), p0.size()) - sqnorm(ps.data(), ps.size()));
}

// ---------------------------------------------------------------- smc.hpp
struct SamplerError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ParticleEnsemble (smc.hpp:28-35): thetas is D x J column-major, i.e.
// particle j occupies thetas[j*D, (j+1)*D).
struct ParticleEnsemble {
  int64_t dim = 0, count = 0;
  Vec thetas;
  Vec log_weights;
  int iteration = 0;
  double* col(int64_t j) { return thetas.data() + (size_t)j * dim; }
  const double* col(int64_t j) const { return thetas.data() + (size_t)j * dim; }
};

struct IterRecord {  // smc.hpp:38-49
  int k = 0;
  int64_t batch = 0;
  double beta = 1.0;
  double ess = 0.0;
  bool resampled = false;
  double mean_log_target = 0.0;
  double sampler_ms = 0.0;
  double test_log_pred = kNaN, test_accuracy = kNaN;
  bool evaluated = false;
  int n_divergent = 0;
};

enum class ResampleKind { kMultinomial = 0, kSystematic = 1 };

struct SmcOptions {  // smc.hpp:51-54 (+ [EXT] scheme / always)
  int num_threads = 1;
  double resample_fraction = 0.5;
  ResampleKind kind = ResampleKind::kMultinomial;
  bool resample_always = false;  // [EXT] SURVEY Appendix A.7 ("resample every iteration")
};

inline Vec normalize(const Vec& lw) {  // smc.hpp:57-64
  if (lw.empty()) throw std::invalid_argument("normalize: empty weights");
  double m = lw[0];
  for (double x : lw) m = std::max(m, x);
  if (m == kNegInf) throw SamplerError("normalize: all particles dead (every log-weight is -inf)");
  Vec w(lw.size());
  double s = 0.0;
  for (size_t i = 0; i < lw.size(); ++i) {
    w[i] = std::exp(lw[i] - m);
    s += w[i];
  }
  for (auto& x : w) x /= s;
  return w;
}

inline double ess(const Vec& w) { return 1.0 / dot(w, w); }  // smc.hpp:67-69

inline ParticleEnsemble init_ensemble(int64_t count, const TargetContext& ctx0, const RngStream& rng,
                                      int threads = 1) {  // smc.hpp:73-89
  if (count < 2) throw std::invalid_argument("init_ensemble: need at least 2 particles");
  validate(ctx0);
  const int64_t D = model_param_count(ctx0.model);
  ParticleEnsemble e;
  e.dim = D;
  e.count = count;
  e.thetas.resize((size_t)(D * count));
  e.log_weights.resize((size_t)count);
  parallel_for(count, threads, [&](int64_t j) {
    RngStream s = rng.fork(tag::kInit, (std::uint64_t)j);
    const Vec th = sample_gaussian_prior(ctx0.prior, D, s);
    std::copy(th.begin(), th.end(), e.col(j));
    e.log_weights[(size_t)j] = log_target(ctx0, th.data()) - prior_logpdf(ctx0.prior, th.data(), (size_t)D);
  });
  e.iteration = 0;
  return e;
}

// [EXT] systematic scheme: one uniform u from the same stream, positions
// (u + j) / J, the same sequential CDF and upper_bound as sample_categorical.
inline std::vector<int> systematic_indices(RngStream& rng, const Vec& w) {
  check_normalized_weights(w);
  const Vec cdf = cdf_of(w);
  const double u = rng.uniform();
  const int J = (int)w.size();
  std::vector<int> idx((size_t)J);
  for (int j = 0; j < J; ++j) idx[(size_t)j] = upper_bound_index(cdf, (u + (double)j) / (double)J);
  return idx;
}

inline ParticleEnsemble resample(const ParticleEnsemble& e, RngStream& rng, ResampleKind kind,
                                 std::vector<int>* idx_out = nullptr) {  // smc.hpp:93-103
  const Vec w = normalize(e.log_weights);
  const std::vector<int> idx = kind == ResampleKind::kMultinomial
                                   ? sample_categorical(rng, w, (int)e.count)
                                   : systematic_indices(rng, w);
  ParticleEnsemble out;
  out.dim = e.dim;
  out.count = e.count;
  out.thetas.resize(e.thetas.size());
  for (int64_t j = 0; j < e.count; ++j) std::copy(e.col(idx[(size_t)j]), e.col(idx[(size_t)j]) + e.dim, out.col(j));
  out.log_weights.assign((size_t)e.count, -std::log((double)e.count));
  out.iteration = e.iteration;
  if (idx_out) *idx_out = idx;
  return out;
}

struct StepDump {  // optional per-particle proposal outputs for golden vectors
  std::vector<ProposalResult> proposals;
  Vec weights;
  std::vector<int> indices;
};

template <typename Target>
std::pair<ParticleEnsemble, IterRecord> smc_step(const ParticleEnsemble& e, const Target& target,
                                                 const KernelConfig& cfg, const RngStream& rng,
                                                 const SmcOptions& opts = {},
                                                 StepDump* dump = nullptr) {  // smc.hpp:109-158
  KernelConfig::validate(cfg);
  const int64_t J = e.count;
  const int k = e.iteration;
  std::vector<ProposalResult> props((size_t)J);
  parallel_for(J, opts.num_threads, [&](int64_t j) {
    RngStream s = rng.fork(tag::kProposal, (std::uint64_t)k, (std::uint64_t)j);
    Vec th(e.col(j), e.col(j) + e.dim);
    props[(size_t)j] = propose(target, th, cfg, s);
  });
  ParticleEnsemble next;
  next.dim = e.dim;
  next.count = J;
  next.thetas.resize(e.thetas.size());
  next.log_weights.resize((size_t)J);
  IterRecord rec;
  for (int64_t j = 0; j < J; ++j) {
    const ProposalResult& p = props[(size_t)j];
    if (p.divergent) {
      std::copy(e.col(j), e.col(j) + e.dim, next.col(j));
      next.log_weights[(size_t)j] = kNegInf;
      ++rec.n_divergent;
    } else {
      std::copy(p.theta_new.begin(), p.theta_new.end(), next.col(j));
      next.log_weights[(size_t)j] =
          e.log_weights[(size_t)j] + incremental_log_weight(p.log_target_new, p.log_target_old, p.p_initial, p.p_final);
    }
  }
  rec.k = k;
  const Vec w = normalize(next.log_weights);
  rec.ess = ess(w);
  double mlt = 0.0;
  for (int64_t j = 0; j < J; ++j)
    if (w[(size_t)j] > 0.0) mlt += w[(size_t)j] * props[(size_t)j].log_target_new;
  rec.mean_log_target = mlt;
  next.iteration = k + 1;
  std::vector<int> idx;
  if (opts.resample_always || rec.ess < opts.resample_fraction * (double)J) {
    RngStream s = rng.fork(tag::kResample, (std::uint64_t)k);
    next = resample(next, s, opts.kind, &idx);
    next.iteration = k + 1;
    rec.resampled = true;
  }
  if (dump) {
    dump->proposals = std::move(props);
    dump->weights = w;
    dump->indices = idx;
  }
  return {std::move(next), rec};
}

// ---------------------------------------------------------------- annealing.hpp
enum class ScheduleKind { kConstant = 0, kFullBatch = 1, kCtr = 2, kLinear = 3, kAutomated = 4, kSda = 5 };

struct ScheduleConfig {  // annealing.hpp:23-37 (+ [EXT] period / switch_iteration)
  ScheduleKind kind = ScheduleKind::kFullBatch;
  int64_t initial_batch = 1, increment = 1;
  int iterations = 1;
  int64_t dataset_size = 1;
  int period = 1;             // [EXT] linear adds `increment` every `period` iterations (App. A.3)
  int switch_iteration = -1;  // [EXT] <0: reference 0.9*K double compare; else k < switch_iteration (App. A.2)
};

inline void validate(const ScheduleConfig& c) {
  if (c.initial_batch < 1 || c.initial_batch > c.dataset_size)
    throw std::invalid_argument("ScheduleConfig: need 1 <= initial_batch <= dataset_size");
  if (c.increment < 1 || c.increment > c.dataset_size)
    throw std::invalid_argument("ScheduleConfig: need 1 <= increment <= dataset_size");
  if (c.iterations < 1) throw std::invalid_argument("ScheduleConfig: iterations must be >= 1");
  if (c.period < 1) throw std::invalid_argument("ScheduleConfig: period must be >= 1");
}

inline int64_t round_to_multiple_half_up(double v, int64_t mult) {  // annealing.hpp:41-44
  return (int64_t)std::floor(v / (double)mult + 0.5) * mult;
}

inline int64_t batch_size(const ScheduleConfig& c, int k) {  // annealing.hpp:52-82
  validate(c);
  if (k < 0 || k >= c.iterations) throw std::invalid_argument("batch_size: k out of range");
  if (c.kind == ScheduleKind::kSda) throw std::invalid_argument("batch_size: the sda schedule is state-driven");
  const double switch_point = 0.9 * (double)c.iterations;
  const bool early = c.switch_iteration < 0 ? (double)k < switch_point : k < c.switch_iteration;
  switch (c.kind) {
    case ScheduleKind::kConstant: return c.initial_batch;
    case ScheduleKind::kFullBatch: return c.dataset_size;
    case ScheduleKind::kCtr: return early ? c.initial_batch : c.dataset_size;
    case ScheduleKind::kLinear:
      return early ? std::min(c.increment * (int64_t)(k / c.period) + c.initial_batch, c.dataset_size)
                   : c.dataset_size;
    case ScheduleKind::kAutomated: {
      if (!early) return c.dataset_size;
      const auto slope = (int64_t)std::floor((double)(c.dataset_size - c.initial_batch) / switch_point);
      const int64_t raw = c.initial_batch + slope * k;
      const int64_t rounded = round_to_multiple_half_up((double)raw, c.increment);
      return std::clamp(rounded, c.initial_batch, c.dataset_size);
    }
    case ScheduleKind::kSda: break;
  }
  throw std::logic_error("batch_size: unreachable");
}

enum class SdaStage { kInitial = 0, kAnnealed = 1 };

struct SdaState {  // annealing.hpp:89-96
  double beta = 0.1, entropy_step = 1.0, beta_reset = 0.1;
  SubsetWindow window;
  SdaStage stage = SdaStage::kInitial;
  bool terminal = false;
};

inline SdaState sda_init(const ScheduleConfig& c, double beta0 = 0.1, double entropy_step = 1.0) {  // 98-110
  validate(c);
  if (!(beta0 > 0.0 && beta0 <= 1.0)) throw std::invalid_argument("sda_init: beta0 must be in (0, 1]");
  SdaState s;
  s.beta = beta0;
  s.beta_reset = beta0;
  s.entropy_step = entropy_step;
  s.window = SubsetWindow{0, c.initial_batch, c.dataset_size};
  s.stage = SdaStage::kInitial;
  return s;
}

inline double sda_beta_step(double beta, double& entropy_step, double denom) {  // annealing.hpp:114-122
  if (denom == 0.0) return 1.0;
  double cand = beta - entropy_step / denom;
  if (cand <= beta) {
    entropy_step = -entropy_step;
    cand = beta - entropy_step / denom;
  }
  return std::min(cand, 1.0);
}

inline double sda_beta_update_initial(double beta, double step, double var_block) {  // 128-134
  if (var_block < 0.0) throw std::invalid_argument("sda_beta_update_initial: variance must be >= 0");
  return sda_beta_step(beta, step, var_block);
}

inline double sda_beta_update_annealed(double beta, double step, double var_block, double cov) {  // 137-140
  return sda_beta_step(beta, step, var_block + cov);
}

struct SdaMoments {  // annealing.hpp:144-151
  double mean_block = 0, mean_block_sq = 0, var_block = 0, mean_prefix = 0, mean_prod = 0,
         cov_prefix_block = 0;
};

// Moments from per-particle unscaled NLLs and the ensemble's log-weights
// (annealing.hpp:166-173).
inline SdaMoments sda_moments_from(const Vec& prefix_nll, const Vec& block_nll, const Vec& log_weights) {
  const Vec w = normalize(log_weights);
  SdaMoments m;
  Vec bsq(block_nll.size()), prod(block_nll.size());
  for (size_t i = 0; i < bsq.size(); ++i) {
    bsq[i] = block_nll[i] * block_nll[i];
    prod[i] = prefix_nll[i] * block_nll[i];
  }
  m.mean_block = weighted_mean(block_nll, w);
  m.mean_block_sq = weighted_mean(bsq, w);
  m.var_block = weighted_var(block_nll, w);
  m.mean_prefix = weighted_mean(prefix_nll, w);
  m.mean_prod = weighted_mean(prod, w);
  m.cov_prefix_block = weighted_cov(prefix_nll, block_nll, w);
  return m;
}

inline SdaMoments sda_moments(const ParticleEnsemble& e, const Dataset& d, const ModelSpec& model,
                              const SubsetWindow& w, int threads = 1, Vec* pre_out = nullptr,
                              Vec* blk_out = nullptr) {  // annealing.hpp:153-174
  validate(w);
  if (w.block_end <= w.prefix_end) throw std::invalid_argument("sda_moments: window has no new block");
  Vec pre((size_t)e.count), blk((size_t)e.count);
  parallel_for(e.count, threads, [&](int64_t j) {
    const LoglikParts p = unscaled_loglik_parts(d, w, model, e.col(j));
    pre[(size_t)j] = -p.prefix;
    blk[(size_t)j] = -p.block;
  });
  if (pre_out) *pre_out = pre;
  if (blk_out) *blk_out = blk;
  return sda_moments_from(pre, blk, e.log_weights);
}

// State transition given the moments (annealing.hpp:186-207).
inline SdaState sda_advance_with(const ScheduleConfig& c, const SdaState& s, const SdaMoments& m) {
  SdaState next = s;
  const double denom = s.stage == SdaStage::kInitial ? m.var_block : m.var_block + m.cov_prefix_block;
  const double bnew = sda_beta_step(s.beta, next.entropy_step, denom);
  if (bnew >= 1.0) {
    const int64_t absorbed = s.window.block_end;
    if (absorbed >= c.dataset_size) {
      next.beta = 1.0;
      next.window = SubsetWindow{c.dataset_size, c.dataset_size, c.dataset_size};
      next.stage = SdaStage::kAnnealed;
      next.terminal = true;
    } else {
      next.beta = s.beta_reset;
      next.window = SubsetWindow{absorbed, std::min(absorbed + c.increment, c.dataset_size), c.dataset_size};
      next.stage = SdaStage::kAnnealed;
    }
  } else {
    next.beta = bnew;
  }
  return next;
}

inline SdaState sda_advance(const ScheduleConfig& c, const SdaState& s, const ParticleEnsemble& e,
                            const Dataset& d, const ModelSpec& model, int threads = 1) {  // 181-208
  validate(c);
  if (s.terminal) return s;
  return sda_advance_with(c, s, sda_moments(e, d, model, s.window, threads));
}

// ---------------------------------------------------------------- runner.hpp (loop only)
// evaluate_predictive (runner.hpp:331-364): ensemble-averaged predictive over a labelled
// test set.  Weights normalised from the log-weights; dead particles (w = 0) skipped;
// predictive[i][c] = sum_j w_j softmax_j[i][c] in ascending j; returns (mean log
// predictive probability of the true label with a 1e-300 floor, argmax accuracy in %;
// argmax = first maximum).  The logits come from the model's forward pass.
inline std::pair<double, double> evaluate_predictive(const ParticleEnsemble& e, const ModelSpec& model,
                                                     const Dataset& test, int threads = 1) {
  if (test.n < 1 || test.labels.empty()) throw std::invalid_argument("evaluate_predictive: empty or unlabelled test set");
  const Vec w = normalize(e.log_weights);
  const int C = std::holds_alternative<CnnSpec>(model) ? std::get<CnnSpec>(model).head.layer_sizes.back()
                                                     : std::get<NetSpec>(model).layer_sizes.back();
  std::vector<Vec> probs((size_t)e.count);
  parallel_for(e.count, threads, [&](int64_t j) {
    if (w[(size_t)j] <= 0.0) return;
    Vec logits;
    if (const auto* cnn = std::get_if<CnnSpec>(&model)) {
      const Vec flat = cnn_flatten_batch(*cnn, e.col(j), test.row(0), test.n);
      logits = forward_batch(cnn->head, e.col(j) + cnn_conv_params(*cnn), flat.data(), test.n);
    } else {
      logits = forward_batch(std::get<NetSpec>(model), e.col(j), test.row(0), test.n);
    }
    for (int64_t i = 0; i < test.n; ++i) {
      double* row = logits.data() + (size_t)i * C;
      double m = row[0];
      for (int c = 1; c < C; ++c) m = std::max(m, row[c]);
      double s = 0.0;
      for (int c = 0; c < C; ++c) {
        row[c] = std::exp(row[c] - m);
        s += row[c];
      }
      for (int c = 0; c < C; ++c) row[c] /= s;
    }
    probs[(size_t)j] = std::move(logits);
  });
  Vec pred((size_t)test.n * C, 0.0);
  for (int64_t j = 0; j < e.count; ++j)
    if (w[(size_t)j] > 0.0)
      for (size_t t = 0; t < pred.size(); ++t) pred[t] += w[(size_t)j] * probs[(size_t)j][t];
  double log_pred = 0.0;
  int64_t correct = 0;
  for (int64_t i = 0; i < test.n; ++i) {
    const int y = test.labels[(size_t)i];
    const double* row = pred.data() + (size_t)i * C;
    log_pred += std::log(std::max(row[y], 1e-300));
    int am = 0;
    for (int c = 1; c < C; ++c)
      if (row[c] > row[am]) am = c;
    if (am == y) ++correct;
  }
  return {log_pred / (double)test.n, 100.0 * (double)correct / (double)test.n};
}

struct RunConfig {  // the in-memory subset of runner.hpp:57-70 the hot loop reads
  ModelSpec model;
  PriorSpec prior;
  KernelConfig kernel;
  ScheduleConfig schedule;  // iterations / dataset_size resolved by the caller
  double beta0 = 0.1, entropy_step = 1.0;
  bool redraw_constant = false;
  int particles = 128;
  int iterations = 1;
  std::uint64_t seed = 0;
  int threads = 1;
  double resample_fraction = 0.5;
  ResampleKind resample_kind = ResampleKind::kMultinomial;
  bool resample_always = false;
};

struct RunResult {
  std::vector<IterRecord> records;
  ParticleEnsemble ensemble;
  std::vector<SdaState> sda_trace;
};

// run_experiment loop (runner.hpp:486-489 shuffle, 531-564 context_for,
// 581-604 loop).  `train` is the unshuffled training set; predictive
// evaluation is out of the hot path and not run here.
inline RunResult run_loop(const RunConfig& cfg, const Dataset& train_in,
                          const std::function<void(int, double)>& on_iter = nullptr) {
  RngStream root(cfg.seed);
  Dataset train;
  {
    RngStream ps = root.fork(tag::kPermutation);
    train = shuffled(train_in, ps);
  }
  ScheduleConfig sched = cfg.schedule;
  sched.iterations = cfg.iterations;
  sched.dataset_size = train.n;
  validate(sched);
  const bool is_sda = sched.kind == ScheduleKind::kSda;
  SdaState sda;
  if (is_sda) sda = sda_init(sched, cfg.beta0, cfg.entropy_step);
  SmcOptions opts{cfg.threads, cfg.resample_fraction, cfg.resample_kind, cfg.resample_always};
  Dataset redraw;
  auto draw_rows = [&](int k) {  // runner.hpp:531-542
    std::vector<int64_t> order((size_t)train.n);
    for (int64_t i = 0; i < train.n; ++i) order[(size_t)i] = i;
    RngStream s = root.fork(tag::kRedraw, (std::uint64_t)k);
    for (int64_t i = 0; i < sched.initial_batch; ++i) {
      const int64_t j = i + (int64_t)s.uniform_below((std::uint64_t)(train.n - i));
      std::swap(order[(size_t)i], order[(size_t)j]);
    }
    order.resize((size_t)sched.initial_batch);
    return order;
  };
  auto context_for = [&](int k) {  // runner.hpp:544-564
    TargetContext ctx;
    ctx.prior = cfg.prior;
    ctx.model = cfg.model;
    if (is_sda) {
      ctx.data = &train;
      ctx.window = sda.window;
      ctx.mode = TargetMode::kSda;
      ctx.beta = sda.beta;
    } else if (cfg.redraw_constant) {
      redraw = gather(train, draw_rows(k));
      ctx.data = &redraw;
      ctx.window = SubsetWindow{0, sched.initial_batch, train.n};
      ctx.mode = TargetMode::kScaled;
    } else {
      ctx.data = &train;
      ctx.window = SubsetWindow{0, batch_size(sched, k), train.n};
      ctx.mode = TargetMode::kScaled;
    }
    return ctx;
  };
  RunResult res;
  const TargetContext ctx0 = context_for(0);
  res.ensemble = init_ensemble(cfg.particles, ctx0, root, cfg.threads);
  for (int k = 0; k < cfg.iterations; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    const TargetContext ctx = context_for(k);
    auto [next, rec] = smc_step(res.ensemble, ContextTarget{&ctx}, cfg.kernel, root, opts);
    res.ensemble = std::move(next);
    rec.batch = ctx.window.block_end;
    rec.beta = is_sda ? ctx.beta : 1.0;
    if (is_sda) {
      sda = sda_advance(sched, sda, res.ensemble, train, cfg.model, cfg.threads);
      res.sda_trace.push_back(sda);
    }
    rec.sampler_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (on_iter) on_iter(k, rec.sampler_ms);
    res.records.push_back(rec);
  }
  return res;
}

}  // namespace oracle

#endif  // DASMC_ORACLE_HPP
