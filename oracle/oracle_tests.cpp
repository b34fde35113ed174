// Pins the CPU oracle against every known answer of the reference's own test
// suite (proj/tests/test_*.cpp) plus SPEC.md worked examples for the modules
// whose reference tests are stubs (smc, annealing).  TEST INFRASTRUCTURE ONLY.
// Each CHECK cites the reference test (file:line) or SPEC example it restates.
#include <cstdio>
#include <set>

#include "dasmc_oracle.hpp"

using namespace oracle;

static int g_fail = 0, g_pass = 0;
static const char* g_case = "";
#define CASE(name) g_case = name;
#define CHECK(cond)                                                                 \
  do {                                                                              \
    if (cond) {                                                                     \
      ++g_pass;                                                                     \
    } else {                                                                        \
      ++g_fail;                                                                     \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);      \
    }                                                                               \
  } while (0)
#define CHECK_THROWS(expr)                 \
  do {                                     \
    bool thrown = false;                   \
    try {                                  \
      (void)(expr);                        \
    } catch (const std::exception&) {      \
      thrown = true;                       \
    }                                      \
    CHECK(thrown);                         \
  } while (0)

// Catch::Approx semantics: |a-b| <= margin or <= eps*(scale + max(|a|,|b|)).
static bool approx(double a, double b, double eps = 1.1920929e-05 * 100 / 100, double margin = 0.0) {
  if (std::abs(a - b) <= margin) return true;
  return std::abs(a - b) <= eps * (std::max(std::abs(a), std::abs(b)));
}

static double max_rel_error(const Vec& a, const Vec& b, double floor = 1e-3) {  // test_util.hpp:37-45
  double worst = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = std::max({std::abs(a[i]), std::abs(b[i]), floor});
    worst = std::max(worst, std::abs(a[i] - b[i]) / d);
  }
  return worst;
}

static Vec central_diff(const std::function<double(const Vec&)>& f, const Vec& th, double eps = 1e-5) {
  Vec g(th.size()), p = th;  // test_util.hpp:19-33
  for (size_t i = 0; i < th.size(); ++i) {
    p[i] = th[i] + eps;
    const double hi = f(p);
    p[i] = th[i] - eps;
    const double lo = f(p);
    p[i] = th[i];
    g[i] = (hi - lo) / (2.0 * eps);
  }
  return g;
}

static NetSpec random_net_spec(RngStream& rng) {  // test_util.hpp:47-59
  NetSpec s;
  s.layer_sizes.push_back(2 + (int)rng.uniform_below(5));
  const int classes = 2 + (int)rng.uniform_below(4);
  const int hidden = (int)rng.uniform_below(3);
  for (int l = 0; l < hidden; ++l) s.layer_sizes.push_back(2 + (int)rng.uniform_below(7));
  s.layer_sizes.push_back(classes);
  s.activation = rng.uniform() < 0.5 ? Activation::kRelu : Activation::kTanh;
  return s;
}

struct Batch {
  Vec X;
  std::vector<int> y;
  int64_t m;
};
static Batch random_batch(RngStream& rng, const NetSpec& s, int64_t m) {  // test_util.hpp:66-77
  Batch b{Vec((size_t)m * s.layer_sizes[0]), std::vector<int>((size_t)m), m};
  for (int64_t i = 0; i < m; ++i) {
    for (int j = 0; j < s.layer_sizes[0]; ++j) b.X[(size_t)i * s.layer_sizes[0] + j] = rng.normal();
    b.y[(size_t)i] = (int)rng.uniform_below((std::uint64_t)s.layer_sizes.back());
  }
  return b;
}

static Vec naive_forward(const NetSpec& s, const Vec& th, const Vec& x) {  // test_network.cpp:21-41
  return teacher_logits_row(s, th.data(), x.data());
}

struct Flat {
  size_t n;
  ValueGrad value_and_grad(const Vec&) const { return {0.0, Vec(n, 0.0)}; }
};
struct Quad {
  ValueGrad value_and_grad(const Vec& x) const {
    Vec g(x.size());
    for (size_t i = 0; i < x.size(); ++i) g[i] = -x[i];
    return {-0.5 * sqnorm(x.data(), x.size()), g};
  }
};
struct NanGrad {
  ValueGrad value_and_grad(const Vec& x) const { return {0.0, Vec(x.size(), kNaN)}; }
};

static void test_rng() {
  CASE("rng determinism");  // test_rng.cpp:10-15
  {
    RngStream a(42), b(42);
    bool same = true;
    for (int i = 0; i < 1000; ++i) same &= a.next_u64() == b.next_u64();
    CHECK(same);
  }
  CASE("rng distinct seeds");  // test_rng.cpp:17-23
  {
    RngStream a(1), b(2);
    int eq = 0;
    for (int i = 0; i < 64; ++i) eq += a.next_u64() == b.next_u64();
    CHECK(eq == 0);
  }
  CASE("fork independent of position and order");  // test_rng.cpp:25-39
  {
    RngStream parent(7);
    RngStream before = parent.fork(3, 11);
    for (int i = 0; i < 50; ++i) parent.next_u64();
    RngStream after = parent.fork(3, 11);
    bool same = true;
    for (int i = 0; i < 100; ++i) same &= before.next_u64() == after.next_u64();
    CHECK(same);
    RngStream p2(7);
    RngStream first = p2.fork(3, 12), second = p2.fork(3, 11);
    CHECK(second.next_u64() == RngStream(7).fork(3, 11).next_u64());
    CHECK(first.next_u64() != second.next_u64());
  }
  CASE("fork collisions");  // test_rng.cpp:41-51
  {
    std::set<std::uint64_t> firsts;
    for (std::uint64_t a = 0; a < 8; ++a)
      for (std::uint64_t b = 0; b < 8; ++b) firsts.insert(RngStream(123).fork(a, b).next_u64());
    CHECK(firsts.size() == 64);
  }
  CASE("uniform range");  // test_rng.cpp:53-65
  {
    RngStream r(5);
    double lo = 1, hi = 0;
    bool ok = true;
    for (int i = 0; i < 100000; ++i) {
      const double u = r.uniform();
      ok &= u >= 0.0 && u < 1.0;
      lo = std::min(lo, u);
      hi = std::max(hi, u);
    }
    CHECK(ok);
    CHECK(lo < 1e-3);
    CHECK(hi > 1.0 - 1e-3);
  }
  CASE("uniform_below");  // test_rng.cpp:67-71
  {
    RngStream r(5);
    CHECK_THROWS(r.uniform_below(0));
    bool ok = true;
    for (int i = 0; i < 10000; ++i) ok &= r.uniform_below(7) < 7;
    CHECK(ok);
  }
  CASE("xoshiro256++ reference vector");  // published xoshiro256++ algorithm, state {1,2,3,4}
  {
    // With state words s = {1, 2, 3, 4}: first output rotl(1+4, 23) + 1.
    CHECK(rotl64(5, 23) + 1 == 41943041ULL);
    CHECK(splitmix64(0) == 0xe220a8397b1dcdafULL);  // splitmix64 known first output from 0
  }
}

static void test_numeric() {
  CASE("logsumexp basics");  // test_numeric.cpp:23-31
  CHECK(approx(logsumexp({0.0, 0.0}), std::log(2.0), 1e-12));
  CHECK(approx(logsumexp({-1000.0, -1000.0}), -1000.0 + std::log(2.0), 1e-12));
  CHECK(approx(logsumexp({3.7}), 3.7));
  CHECK(std::isfinite(logsumexp({700.0, 699.0})));
  CHECK(approx(logsumexp({0.0, kNegInf}), 0.0, 1e-12, 1e-15));
  CASE("logsumexp domain");  // test_numeric.cpp:34-37
  CHECK_THROWS(logsumexp(Vec{}));
  CHECK_THROWS(logsumexp({kNegInf, kNegInf}));
  CASE("logsumexp shift invariance");  // test_numeric.cpp:39-48
  {
    RngStream r(11);
    for (double shift : {500.0, -500.0}) {
      Vec v(20), s(20);
      for (int i = 0; i < 20; ++i) {
        v[(size_t)i] = 10.0 * r.normal();
        s[(size_t)i] = v[(size_t)i] + shift;
      }
      CHECK(approx(logsumexp(s), logsumexp(v) + shift, 1e-12));
    }
  }
  CASE("weighted_mean");  // test_numeric.cpp:50-56
  CHECK(approx(weighted_mean({1, 2, 3, 4}, {0.25, 0.25, 0.25, 0.25}), 2.5));
  CHECK(approx(weighted_mean({5, 7, 9}, {1, 0, 0}), 5.0));
  CHECK(approx(weighted_mean({2, 4}, {0.25, 0.75}), 3.5));
  CHECK_THROWS(weighted_mean({1, 2}, {1.0}));
  CASE("weighted_var");  // test_numeric.cpp:58-64
  CHECK(approx(weighted_var({3, 3, 3}, {0.2, 0.3, 0.5}), 0.0, 1e-5, 1e-15));
  CHECK(approx(weighted_var({0, 2}, {0.5, 0.5}), 1.0));
  CHECK(approx(weighted_var({1, 2, 3}, {0.2, 0.5, 0.3}), 0.49));
  CHECK(weighted_var({1e8, 1e8}, {0.5, 0.5}) >= 0.0);
  CASE("weighted_cov");  // test_numeric.cpp:66-76
  CHECK(approx(weighted_cov({1, 2, 4}, {1, 2, 4}, {0.3, 0.45, 0.25}), weighted_var({1, 2, 4}, {0.3, 0.45, 0.25}),
               1e-5, 1e-12));
  CHECK(approx(weighted_cov({1, 2, 4}, {7, 7, 7}, {0.3, 0.45, 0.25}), 0.0, 1e-5, 1e-12));
  CHECK(approx(weighted_cov({1, 2}, {2, 1}, {0.5, 0.5}), -0.25));
  CHECK_THROWS(weighted_cov({1, 2}, {1, 2, 3}, {0.5, 0.5}));
  CASE("weighted_var random nonneg");  // test_numeric.cpp:78-91
  {
    RngStream r(3);
    bool ok = true;
    for (int rep = 0; rep < 200; ++rep) {
      Vec v(10), raw(10);
      double s = 0;
      for (int i = 0; i < 10; ++i) {
        v[(size_t)i] = 100.0 * r.normal();
        raw[(size_t)i] = r.uniform() + 1e-3;
        s += raw[(size_t)i];
      }
      for (auto& x : raw) x /= s;
      const double var = weighted_var(v, raw);
      ok &= var >= 0.0 && approx(weighted_cov(v, v, raw), var, 1e-5, 1e-12);
    }
    CHECK(ok);
  }
  CASE("sample_categorical degenerate");  // test_numeric.cpp:93-99
  {
    RngStream r(17);
    bool ok = true;
    for (int i : sample_categorical(r, {1, 0, 0}, 5)) ok &= i == 0;
    for (int i : sample_categorical(r, {0, 1}, 3)) ok &= i == 1;
    CHECK(ok);
    CHECK_THROWS(sample_categorical(r, {0.5, 0.2}, 3));
    CHECK_THROWS(sample_categorical(r, {1.5, -0.5}, 3));
  }
  CASE("sample_categorical chi2");  // test_numeric.cpp:101-113
  {
    RngStream r(2024);
    std::vector<int> cnt(4, 0);
    for (int i : sample_categorical(r, {0.25, 0.25, 0.25, 0.25}, 100000)) cnt[(size_t)i]++;
    double chi2 = 0;
    for (int c : cnt) chi2 += (c - 25000.0) * (c - 25000.0) / 25000.0;
    CHECK(chi2 < 16.266);
  }
  CASE("normal statistics");  // test_numeric.cpp:115-129
  {
    RngStream a(9), b(9);
    CHECK(a.normal_vector(16) == b.normal_vector(16));
    RngStream r(1234);
    const Vec z = r.normal_vector(1000000);
    double m = 0;
    for (double x : z) m += x;
    m /= (double)z.size();
    double v = 0;
    for (double x : z) v += (x - m) * (x - m);
    v /= (double)(z.size() - 1);
    CHECK(std::abs(m) < 0.01);
    CHECK(std::abs(v - 1.0) < 0.01);
    RngStream c(9);
    CHECK_THROWS(c.normal_vector(0));
  }
}

static void test_network() {
  CASE("param_count");  // test_network.cpp:45-51
  CHECK(param_count({{2, 3, 2}}) == 17);
  CHECK(param_count({{784, 32, 10}}) == 25450);
  CHECK(param_count({{1, 1}}) == 2);
  CHECK_THROWS(param_count({{4}}));
  CHECK_THROWS(param_count({{4, 0, 2}}));
  CASE("forward fixed nets");  // test_network.cpp:53-69
  {
    const Vec th{2.0, 1.0}, x{3.0};
    CHECK(approx(forward_batch({{1, 1}}, th, x.data(), 1)[0], 7.0));
    const NetSpec s{{3, 4, 2}};
    const Vec z((size_t)param_count(s), 0.0), in{0.5, -1.0, 2.0};
    const Vec out = forward_batch(s, z, in.data(), 1);
    CHECK(out[0] == 0.0 && out[1] == 0.0);
    CHECK_THROWS(forward_batch(s, Vec(2), in.data(), 1));
  }
  CASE("forward vs naive per-unit");  // test_network.cpp:71-81
  {
    RngStream r(101);
    bool ok = true;
    for (int rep = 0; rep < 20; ++rep) {
      const NetSpec s = random_net_spec(r);
      const Vec th = r.normal_vector(param_count(s));
      const Vec x = r.normal_vector(s.layer_sizes[0]);
      const Vec got = forward_batch(s, th, x.data(), 1), exp = naive_forward(s, th, x);
      for (size_t i = 0; i < got.size(); ++i) ok &= std::abs(got[i] - exp[i]) < 1e-12;
    }
    CHECK(ok);
  }
  CASE("output permutation equivariance");  // test_network.cpp:83-100
  {
    RngStream r(55);
    const NetSpec s{{4, 6, 3}};
    Vec th = r.normal_vector(param_count(s));
    const Vec x = r.normal_vector(4);
    const Vec base = forward_batch(s, th, x.data(), 1);
    const int off = 4 * 6 + 6;
    for (int c = 0; c < 6; ++c) std::swap(th[(size_t)(off + c * 3)], th[(size_t)(off + c * 3 + 2)]);
    std::swap(th[(size_t)(off + 18)], th[(size_t)(off + 20)]);
    const Vec sw = forward_batch(s, th, x.data(), 1);
    CHECK(approx(sw[0], base[2]) && approx(sw[2], base[0]) && approx(sw[1], base[1]));
  }
  CASE("loglik_point");  // test_network.cpp:102-117
  {
    const NetSpec s{{2, 10}};
    const Vec z((size_t)param_count(s), 0.0), x{0.3, -0.2};
    const Vec lg = forward_batch(s, z, x.data(), 1);
    CHECK(approx(log_softmax_at(lg.data(), 10, 4), -std::log(10.0)));
    CHECK_THROWS(log_softmax_at(lg.data(), 10, 10));
    CHECK_THROWS(log_softmax_at(lg.data(), 10, -1));
    const double big[2] = {1000.0, -1000.0};
    CHECK(approx(log_softmax_at(big, 2, 0), 0.0, 1e-5, 1e-12));
    CHECK(std::isfinite(log_softmax_at(big, 2, 1)));
  }
  CASE("naive softmax");  // test_network.cpp:119-130
  {
    RngStream r(77);
    bool ok = true;
    for (int rep = 0; rep < 10; ++rep) {
      const NetSpec s = random_net_spec(r);
      Vec th = r.normal_vector(param_count(s));
      for (auto& v : th) v *= 0.5;
      const Vec x = r.normal_vector(s.layer_sizes[0]);
      const Vec lg = forward_batch(s, th, x.data(), 1);
      const int label = (int)r.uniform_below(lg.size());
      double den = 0;
      for (double v : lg) den += std::exp(v);
      ok &= approx(log_softmax_at(lg.data(), (int)lg.size(), label), std::log(std::exp(lg[(size_t)label]) / den), 1e-10);
    }
    CHECK(ok);
  }
  CASE("likelihoods normalise");  // test_network.cpp:132-143
  {
    RngStream r(31);
    bool ok = true;
    for (int rep = 0; rep < 10; ++rep) {
      const NetSpec s = random_net_spec(r);
      const Vec th = r.normal_vector(param_count(s));
      const Vec x = r.normal_vector(s.layer_sizes[0]);
      const Vec lg = forward_batch(s, th, x.data(), 1);
      double t = 0;
      for (int c = 0; c < s.layer_sizes.back(); ++c) t += std::exp(log_softmax_at(lg.data(), (int)lg.size(), c));
      ok &= std::abs(t - 1.0) <= 1e-12;
    }
    CHECK(ok);
  }
  CASE("gradient vs central FD");  // test_network.cpp:145-160
  {
    RngStream r(2025);
    bool ok = true;
    for (int rep = 0; rep < 20; ++rep) {
      const NetSpec s = random_net_spec(r);
      const Vec th = r.normal_vector(param_count(s));
      const Batch b = random_batch(r, s, 1 + (int64_t)r.uniform_below(6));
      Vec g(th.size());
      const double v = loglik_and_grad_batch(s, th.data(), b.X.data(), b.y.data(), b.m, g.data());
      const Vec fd = central_diff([&](const Vec& t) { return loglik_batch(s, t.data(), b.X.data(), b.y.data(), b.m); }, th);
      ok &= max_rel_error(g, fd) < 1e-4;
      ok &= approx(v, loglik_batch(s, th.data(), b.X.data(), b.y.data(), b.m));
    }
    CHECK(ok);
  }
  CASE("duplicated datapoint doubles exactly");  // test_network.cpp:162-176
  {
    RngStream r(7);
    const NetSpec s{{3, 5, 2}, Activation::kTanh};
    const Vec th = r.normal_vector(param_count(s));
    const Batch one = random_batch(r, s, 1);
    Vec X2(one.X);
    X2.insert(X2.end(), one.X.begin(), one.X.end());
    const std::vector<int> y2{one.y[0], one.y[0]};
    Vec g1(th.size()), g2(th.size());
    const double v1 = loglik_and_grad_batch(s, th.data(), one.X.data(), one.y.data(), 1, g1.data());
    const double v2 = loglik_and_grad_batch(s, th.data(), X2.data(), y2.data(), 2, g2.data());
    CHECK(v2 == 2.0 * v1);
    double worst = 0;
    for (size_t i = 0; i < g1.size(); ++i) worst = std::max(worst, std::abs(g2[i] - 2.0 * g1[i]));
    CHECK(worst == 0.0);
  }
  CASE("closed-form output bias gradient");  // test_network.cpp:178-199
  {
    const NetSpec s{{2, 3, 3}};
    const Vec z((size_t)param_count(s), 0.0);
    RngStream r(13);
    Vec X(6);
    for (auto& v : X) v = r.normal();
    const std::vector<int> bal{0, 1, 2}, unb{1, 1, 2};
    Vec g(z.size());
    const double vb = loglik_and_grad_batch(s, z.data(), X.data(), bal.data(), 3, g.data());
    CHECK(approx(vb, 3.0 * -std::log(3.0)));
    double mx = 0;
    for (double v : g) mx = std::max(mx, std::abs(v));
    CHECK(mx <= 1e-15);
    loglik_and_grad_batch(s, z.data(), X.data(), unb.data(), 3, g.data());
    const int bo = 2 * 3 + 3 + 3 * 3;
    CHECK(approx(g[(size_t)bo], -1.0, 1e-5, 1e-12));
    CHECK(approx(g[(size_t)bo + 1], 1.0, 1e-5, 1e-12));
    CHECK(approx(g[(size_t)bo + 2], 0.0, 1e-5, 1e-12));
  }
  CASE("empty batch rejected");  // test_network.cpp:201-206
  {
    const NetSpec s{{2, 2}};
    Vec th((size_t)param_count(s), 0.0), g(th.size());
    CHECK_THROWS(loglik_and_grad_batch(s, th.data(), nullptr, nullptr, 0, g.data()));
  }
  CASE("prior KATs");  // test_network.cpp:208-230
  {
    constexpr double kLogTwoPi = 1.8378770664093455;
    const Vec o{0.0, 0.0};
    CHECK(approx(prior_logpdf({1.0}, o.data(), 2), -kLogTwoPi));
    const double sg = 0.7;
    const Vec at{sg};
    CHECK(approx(prior_logpdf({sg}, at.data(), 1), -0.5 * std::log(2.0 * M_PI * sg * sg) - 0.5));
    RngStream r(19);
    const Vec th = r.normal_vector(6);
    const Vec fd = central_diff([&](const Vec& t) { return prior_logpdf({sg}, t.data(), t.size()); }, th, 1e-6);
    Vec ex(6);
    for (int i = 0; i < 6; ++i) ex[(size_t)i] = -th[(size_t)i] / (sg * sg);
    CHECK(max_rel_error(ex, fd, 1e-6) < 1e-8);
  }
  CASE("prior sampling");  // test_network.cpp:232-254
  {
    RngStream bad(1);
    CHECK_THROWS(sample_gaussian_prior({0.0}, 3, bad));
    RngStream a(5), b(5);
    CHECK(sample_gaussian_prior({1.0}, 2, a) == sample_gaussian_prior({1.0}, 2, b));
    RngStream r(99);
    double s = 0, ss = 0;
    for (int i = 0; i < 100000; ++i) {
      const double v = sample_gaussian_prior({2.5}, 1, r)[0];
      s += v;
      ss += v * v;
    }
    const double m = s / 100000, sd = std::sqrt(ss / 100000 - m * m);
    CHECK(std::abs(sd - 2.5) / 2.5 < 0.01);
  }
}

struct Problem {
  Dataset d;
  NetSpec net;
  Vec th;
};
static Problem problem(std::uint64_t seed, int64_t n = 24) {  // test_target.cpp:22-41
  Problem p;
  p.d = make_synthetic(SyntheticKind::kTwoMoons, n, 0.1, seed).data;
  p.net = NetSpec{{2, 5, 2}};
  RngStream r(seed + 1);
  p.th = r.normal_vector(param_count(p.net));
  return p;
}
static TargetContext scaled_ctx(const Problem& p, int64_t m, int64_t total) {
  TargetContext c;
  c.data = &p.d;
  c.window = SubsetWindow{0, m, total};
  c.model = p.net;
  return c;
}

static void test_target() {
  CASE("scaled full = plain posterior");  // test_target.cpp:49-55
  {
    const Problem p = problem(21);
    const auto c = scaled_ctx(p, p.d.n, p.d.n);
    const double direct = loglik_batch(p.net, p.th.data(), p.d.row(0), p.d.labels.data(), p.d.n) +
                          prior_logpdf(c.prior, p.th.data(), p.th.size());
    CHECK(approx(log_target(c, p.th.data()), direct, 1e-13));
  }
  CASE("scaled N/M factor");  // test_target.cpp:57-64
  {
    const Problem p = problem(22);
    const auto c = scaled_ctx(p, 6, p.d.n);
    const double e = ((double)p.d.n / 6.0) * segment_loglik(p.net, p.d, 0, 6, p.th.data()) +
                     prior_logpdf(c.prior, p.th.data(), p.th.size());
    CHECK(approx(log_target(c, p.th.data()), e, 1e-13));
  }
  CASE("sda beta=1");  // test_target.cpp:66-75
  {
    const Problem p = problem(23);
    auto c = scaled_ctx(p, 10, p.d.n);
    c.mode = TargetMode::kSda;
    c.window = SubsetWindow{4, 10, p.d.n};
    c.beta = 1.0;
    const double e = segment_loglik(p.net, p.d, 0, 10, p.th.data()) + prior_logpdf(c.prior, p.th.data(), p.th.size());
    CHECK(approx(log_target(c, p.th.data()), e, 1e-13));
  }
  CASE("sda closed prefix = scaled");  // test_target.cpp:77-87
  {
    const Problem p = problem(24);
    auto s = scaled_ctx(p, 8, p.d.n);
    s.mode = TargetMode::kSda;
    s.window = SubsetWindow{8, 8, p.d.n};
    const auto plain = scaled_ctx(p, 8, 8);
    CHECK(approx(log_target(s, p.th.data()), log_target(plain, p.th.data()), 1e-12));
  }
  CASE("target FD both modes");  // test_target.cpp:89-106
  {
    const Problem p = problem(25, 12);
    auto c = scaled_ctx(p, 7, p.d.n);
    const auto f = [&](const TargetContext& cc) {
      const Vec g = log_target_with_grad(cc, p.th.data()).grad;
      const Vec fd = central_diff([&](const Vec& t) { return log_target(cc, t.data()); }, p.th);
      return max_rel_error(g, fd);
    };
    CHECK(f(c) < 1e-4);
    c.mode = TargetMode::kSda;
    c.window = SubsetWindow{4, 9, p.d.n};
    c.beta = 0.37;
    CHECK(f(c) < 1e-4);
  }
  CASE("brute-force full batch");  // test_target.cpp:108-115
  {
    const Problem p = problem(26, 16);
    const auto c = scaled_ctx(p, p.d.n, p.d.n);
    Vec g(p.th.size());
    loglik_and_grad_batch(p.net, p.th.data(), p.d.row(0), p.d.labels.data(), p.d.n, g.data());
    const Vec t = log_target_with_grad(c, p.th.data()).grad;
    double w = 0;
    for (size_t i = 0; i < g.size(); ++i) w = std::max(w, std::abs(t[i] - (g[i] - p.th[i])));
    CHECK(w < 1e-12);
  }
  CASE("sda linear in beta");  // test_target.cpp:117-131
  {
    const Problem p = problem(27, 10);
    auto c = scaled_ctx(p, 6, p.d.n);
    c.mode = TargetMode::kSda;
    c.window = SubsetWindow{5, 6, p.d.n};
    c.beta = 0.5;
    Vec gb(p.th.size()), gp(p.th.size());
    segment_loglik_grad(p.net, p.d, 5, 6, p.th.data(), gb.data());
    segment_loglik_grad(p.net, p.d, 0, 5, p.th.data(), gp.data());
    const Vec t = log_target_with_grad(c, p.th.data()).grad;
    double w = 0;
    for (size_t i = 0; i < t.size(); ++i) w = std::max(w, std::abs(t[i] - (gp[i] + 0.5 * gb[i] - p.th[i])));
    CHECK(w < 1e-14);
  }
  CASE("prior linearity");  // test_target.cpp:133-143
  {
    const Problem p = problem(28, 10);
    const auto c = scaled_ctx(p, 10, p.d.n);
    const ValueGrad j = log_target_with_grad(c, p.th.data());
    Vec g(p.th.size());
    const double ll = segment_loglik_grad(p.net, p.d, 0, 10, p.th.data(), g.data());
    const double sc = (double)p.d.n / 10.0;
    CHECK(approx(j.value, sc * ll + prior_logpdf(c.prior, p.th.data(), p.th.size()), 1e-12));
    double w = 0;
    for (size_t i = 0; i < g.size(); ++i) w = std::max(w, std::abs(j.grad[i] - (sc * g[i] - p.th[i])));
    CHECK(w < 1e-12);
  }
  CASE("target determinism");  // test_target.cpp:145-150
  {
    const Problem p = problem(29);
    const auto c = scaled_ctx(p, 9, p.d.n);
    CHECK(log_target(c, p.th.data()) == log_target(c, p.th.data()));
    CHECK(log_target_with_grad(c, p.th.data()).grad == log_target_with_grad(c, p.th.data()).grad);
  }
  CASE("empty subset rejected");  // test_target.cpp:152-159
  {
    const Problem p = problem(30);
    auto c = scaled_ctx(p, 5, p.d.n);
    c.window = SubsetWindow{0, 0, p.d.n};
    CHECK_THROWS(log_target(c, p.th.data()));
    c.window = SubsetWindow{0, p.d.n + 1, p.d.n + 1};
    CHECK_THROWS(log_target(c, p.th.data()));
  }
  CASE("prior-only target");  // test_target.cpp:161-170
  {
    TargetContext c;
    c.prior = PriorSpec{1.3};
    c.model = NetSpec{{2, 2}};
    RngStream r(31);
    const Vec th = r.normal_vector(6);
    CHECK(approx(log_target(c, th.data()), prior_logpdf(c.prior, th.data(), 6)));
    const Vec g = log_target_with_grad(c, th.data()).grad;
    double w = 0;
    for (int i = 0; i < 6; ++i) w = std::max(w, std::abs(g[(size_t)i] + th[(size_t)i] / (1.3 * 1.3)));
    CHECK(w < 1e-14);
  }
  CASE("linear-gaussian FD");  // test_target.cpp:172-185
  {
    const auto s = make_synthetic(SyntheticKind::kLinearGaussian, 30, 0.5, 8, 4);
    TargetContext c;
    c.data = &s.data;
    c.window = SubsetWindow{0, 30, 30};
    c.model = LinearGaussianSpec{4, 0.5};
    RngStream r(9);
    const Vec th = r.normal_vector(4);
    const Vec g = log_target_with_grad(c, th.data()).grad;
    const Vec fd = central_diff([&](const Vec& t) { return log_target(c, t.data()); }, th, 1e-6);
    CHECK(max_rel_error(g, fd, 1e-6) < 1e-7);
  }
  CASE("scaled estimate convergence");  // test_target.cpp:187-212
  {
    const int64_t n = 400;
    const NetSpec net{{2, 4, 2}};
    RngStream tr(500);
    const Vec th = tr.normal_vector(param_count(net));
    int good = 0;
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
      const auto s = make_synthetic(SyntheticKind::kTwoMoons, n, 0.15, 1000 + seed);
      RngStream r(seed);
      const Dataset d = shuffled(s.data, r);
      const double full = segment_loglik(net, d, 0, n, th.data());
      double prev = std::numeric_limits<double>::infinity();
      bool mono = true;
      for (int64_t m : {n / 4, n / 2, n}) {
        const double err = std::abs((double)n / (double)m * segment_loglik(net, d, 0, m, th.data()) - full);
        if (err > prev + 1e-12) mono = false;
        prev = err;
      }
      good += mono;
    }
    CHECK(good >= 8);
  }
}

static Vec scalar(double v) { return Vec{v}; }

static void test_kernels() {
  CASE("kernel config");  // test_kernels.cpp:47-55
  CHECK(KernelConfig::langevin(0.1).leapfrog_steps == 1);
  CHECK_THROWS(KernelConfig::hmc(0.0, 5));
  CHECK_THROWS(KernelConfig::hmc(0.1, 0));
  CHECK_THROWS(KernelConfig::validate(KernelConfig{0.1, 3, KernelKind::kLangevin}));
  CASE("free particle");  // test_kernels.cpp:57-65
  {
    RngStream r(3);
    const Vec th = r.normal_vector(4), p0 = r.normal_vector(4);
    const auto [ts, ps] = leapfrog(Flat{4}, th, p0, KernelConfig::hmc(0.25, 7));
    double w = 0;
    for (int i = 0; i < 4; ++i) w = std::max(w, std::abs(ts[(size_t)i] - (th[(size_t)i] + 7 * 0.25 * p0[(size_t)i])));
    CHECK(w < 1e-12);
    CHECK(ps == p0);
  }
  CASE("1-D leapfrog KAT");  // test_kernels.cpp:67-74
  {
    const auto [ts, ps] = leapfrog(Quad{}, scalar(1.0), scalar(0.0), KernelConfig::hmc(0.1, 1));
    CHECK(approx(ts[0], 0.995, 1e-12));
    CHECK(approx(ps[0], -0.099750, 1e-9));
  }
  CASE("reversibility on random NN targets");  // test_kernels.cpp:76-107
  {
    RngStream r(71);
    bool ok = true;
    for (int rep = 0; rep < 5; ++rep) {
      const NetSpec net = random_net_spec(r);
      Dataset d = make_synthetic(SyntheticKind::kTwoMoons, 12, 0.1, 100 + (std::uint64_t)rep).data;
      if (net.layer_sizes[0] != 2) {
        Vec wide((size_t)12 * net.layer_sizes[0]);
        for (int i = 0; i < 12; ++i)
          for (int j = 0; j < net.layer_sizes[0]; ++j) wide[(size_t)(i * net.layer_sizes[0] + j)] = d.features[(size_t)(i * 2 + j % 2)];
        d.features = wide;
        d.d = net.layer_sizes[0];
      }
      for (auto& l : d.labels) l %= net.layer_sizes.back();
      TargetContext c;
      c.data = &d;
      c.window = SubsetWindow{0, 12, 12};
      c.model = net;
      Vec th = r.normal_vector(param_count(net));
      for (auto& v : th) v *= 0.5;
      const Vec p0 = r.normal_vector((int64_t)th.size());
      const auto cfg = KernelConfig::hmc(0.05, 8);
      const auto [ts, ps] = leapfrog(ContextTarget{&c}, th, p0, cfg);
      Vec mp(ps);
      for (auto& v : mp) v = -v;
      const auto [tb, pb] = leapfrog(ContextTarget{&c}, ts, mp, cfg);
      for (size_t i = 0; i < th.size(); ++i) ok &= std::abs(tb[i] - th[i]) < 1e-9 && std::abs(pb[i] + p0[i]) < 1e-9;
    }
    CHECK(ok);
  }
  CASE("hamiltonian drift");  // test_kernels.cpp:109-121
  {
    RngStream r(5);
    const Vec th = r.normal_vector(10);
    RngStream s(17);
    const auto res = propose(Quad{}, th, KernelConfig::hmc(0.01, 20), s);
    CHECK(!res.divergent);
    const double h0 = -Quad{}.value_and_grad(th).value + 0.5 * sqnorm(res.p_initial.data(), 10);
    const double h1 = -res.log_target_new + 0.5 * sqnorm(res.p_final.data(), 10);
    CHECK(std::abs(h1 - h0) < 1e-3);
  }
  CASE("LD == HMC(S=1) bitwise");  // test_kernels.cpp:123-134
  {
    RngStream r(13);
    const Vec th = r.normal_vector(6);
    RngStream a(99), b(99);
    const auto h = propose(Quad{}, th, KernelConfig::hmc(0.07, 1), a);
    const auto l = propose(Quad{}, th, KernelConfig::langevin(0.07), b);
    CHECK(h.theta_new == l.theta_new && h.p_initial == l.p_initial && h.p_final == l.p_final &&
          h.log_target_new == l.log_target_new);
  }
  CASE("propose reproducible");  // test_kernels.cpp:136-145
  {
    RngStream r(1);
    const Vec th = r.normal_vector(3);
    RngStream a(55), b(55);
    const auto x = propose(Quad{}, th, KernelConfig::hmc(0.1, 4), a);
    const auto y = propose(Quad{}, th, KernelConfig::hmc(0.1, 4), b);
    CHECK(x.theta_new == y.theta_new && x.log_target_new == y.log_target_new);
  }
  CASE("divergence flagged");  // test_kernels.cpp:147-157
  {
    RngStream s(2);
    const auto res = propose(NanGrad{}, scalar(0.5), KernelConfig::hmc(0.1, 3), s);
    CHECK(res.divergent && res.divergence_step == 0 && res.theta_new == scalar(0.5));
    CHECK_THROWS(leapfrog(NanGrad{}, scalar(0.5), scalar(0.1), KernelConfig::hmc(0.1, 3)));
  }
  CASE("incremental weight KATs");  // test_kernels.cpp:159-168
  CHECK(incremental_log_weight(-3.0, -3.0, scalar(0.7), scalar(0.7)) == 0.0);
  CHECK(approx(incremental_log_weight(-1.0, -1.0, scalar(1.0), scalar(0.0)), 0.5));
  CHECK(approx(incremental_log_weight(-1.3, -1.0, scalar(0.0), scalar(0.0)), -0.3));
  CHECK(incremental_log_weight(kNaN, -1.0, scalar(0.0), scalar(0.0)) == kNegInf);
  CHECK_THROWS(incremental_log_weight(0.0, 0.0, scalar(0.0), Vec(2)));
  CASE("incremental weight antisymmetry");  // test_kernels.cpp:170-181
  {
    RngStream r(41);
    bool ok = true;
    for (int rep = 0; rep < 20; ++rep) {
      const double nv = r.normal(), ov = r.normal();
      const Vec p0 = r.normal_vector(5), ps = r.normal_vector(5);
      ok &= std::abs(incremental_log_weight(nv, ov, p0, ps) + incremental_log_weight(ov, nv, ps, p0)) <= 1e-12;
    }
    CHECK(ok);
  }
  CASE("jacobian cancellation");  // test_kernels.cpp:183-204
  {
    const auto cfg = KernelConfig::hmc(0.1, 3);
    const Vec th0 = scalar(0.8);
    const double p0 = -0.4, eps = 1e-5;
    const auto flow = [&](const Vec& st, double p) { return leapfrog(Quad{}, st, scalar(p), cfg).first[0]; };
    const double fj = (flow(th0, p0 + eps) - flow(th0, p0 - eps)) / (2 * eps);
    const auto [ts, ps] = leapfrog(Quad{}, th0, scalar(p0), cfg);
    const double pr = -ps[0];
    const double rj = (flow(ts, pr + eps) - flow(ts, pr - eps)) / (2 * eps);
    CHECK(std::abs(std::abs(fj) - std::abs(rj)) / std::abs(fj) < 1e-6);
  }
}

static void test_dataset() {
  CASE("two_moons geometry");  // test_dataset.cpp:133-151
  {
    const Dataset d = make_synthetic(SyntheticKind::kTwoMoons, 201, 0.0, 4).data;
    int c0 = 0;
    bool ok = true;
    for (int64_t i = 0; i < d.n; ++i) {
      const double x = d.row(i)[0], y = d.row(i)[1];
      if (d.labels[(size_t)i] == 0) {
        ++c0;
        ok &= std::abs(std::sqrt(x * x + y * y) - 1.0) <= 1e-9 && y >= -1e-12;
      } else {
        ok &= std::abs(std::sqrt((x - 1) * (x - 1) + (y - 0.5) * (y - 0.5)) - 1.0) <= 1e-9 && y <= 0.5 + 1e-12;
      }
    }
    CHECK(ok);
    CHECK(std::abs(c0 - (201 - c0)) <= 1);
  }
  CASE("synthetic reproducible");  // test_dataset.cpp:153-160
  {
    const auto a = make_synthetic(SyntheticKind::kGaussianBlobs, 50, 0.3, 12);
    const auto b = make_synthetic(SyntheticKind::kGaussianBlobs, 50, 0.3, 12);
    const auto c = make_synthetic(SyntheticKind::kGaussianBlobs, 50, 0.3, 13);
    CHECK(a.data.features == b.data.features && a.data.labels == b.data.labels);
    CHECK(a.data.features != c.data.features);
  }
  CASE("shuffle bijection");  // test_dataset.cpp:178-194
  {
    const Dataset src = make_synthetic(SyntheticKind::kGaussianBlobs, 30, 0.2, 5).data;
    RngStream r(77);
    const Dataset s = shuffled(src, r);
    std::set<int64_t> seen(s.perm.begin(), s.perm.end());
    CHECK(seen.size() == 30 && *seen.begin() == 0 && *seen.rbegin() == 29);
    bool ok = true;
    for (int64_t i = 0; i < 30; ++i) {
      const int64_t p = s.perm[(size_t)i];
      ok &= s.row(i)[0] == src.row(p)[0] && s.row(i)[1] == src.row(p)[1] && s.labels[(size_t)i] == src.labels[(size_t)p];
    }
    CHECK(ok);
  }
  CASE("window validation");  // test_dataset.cpp:196-213
  {
    CHECK_THROWS(validate(SubsetWindow{10, 5, 20}));
    CHECK_THROWS(validate(SubsetWindow{0, 25, 20}));
  }
  CASE("gather");  // test_dataset.cpp:225-237
  {
    const Dataset src = make_synthetic(SyntheticKind::kGaussianBlobs, 10, 0.2, 2).data;
    const Dataset g = gather(src, {9, 0, 4});
    CHECK(g.n == 3 && g.row(0)[0] == src.row(9)[0] && g.labels[1] == src.labels[0]);
    CHECK_THROWS(gather(src, {11}));
  }
}

static void test_smc_spec() {
  CASE("normalize KATs");  // SPEC.md smc normalize examples
  {
    const Vec w = normalize({0, 0, 0, 0});
    CHECK(w[0] == 0.25 && w[3] == 0.25);
    const Vec d = normalize({0, kNegInf});
    CHECK(d[0] == 1.0 && d[1] == 0.0);
    const Vec a = normalize({0.3, -1.2, 2.0}), b = normalize({1234.8, 1233.3, 1236.5});
    bool ok = true;
    for (int i = 0; i < 3; ++i) ok &= std::abs(a[(size_t)i] - b[(size_t)i]) < 1e-12;
    CHECK(ok);
    bool threw = false;
    try {
      normalize({kNegInf, kNegInf});
    } catch (const SamplerError&) {
      threw = true;
    }
    CHECK(threw);
  }
  CASE("ess KATs");  // SPEC.md ess examples
  CHECK(approx(ess(Vec(8, 0.125)), 8.0, 1e-12));
  CHECK(ess({1.0, 0.0, 0.0}) == 1.0);
  CHECK(approx(ess({0.5, 0.5, 0, 0}), 2.0, 1e-12));
  CASE("resample KATs");  // SPEC.md resample_multinomial examples
  {
    ParticleEnsemble e;
    e.dim = 1;
    e.count = 3;
    e.thetas = {10, 20, 30};
    e.log_weights = {0, kNegInf, kNegInf};
    RngStream r(4);
    const auto out = resample(e, r, ResampleKind::kMultinomial);
    CHECK(out.thetas == Vec({10, 10, 10}));
    CHECK(approx(out.log_weights[0], -std::log(3.0), 1e-15));
    CHECK(approx(ess(normalize(out.log_weights)), 3.0, 1e-12));
    RngStream r2(4);
    const auto sys = resample(e, r2, ResampleKind::kSystematic);
    CHECK(sys.thetas == Vec({10, 10, 10}));
  }
  CASE("systematic indices sorted and proportional");  // [EXT] definition
  {
    RngStream r(8);
    Vec w(100);
    double s = 0;
    for (auto& v : w) {
      v = r.uniform();
      s += v;
    }
    for (auto& v : w) v /= s;
    RngStream r2(9);
    const auto idx = systematic_indices(r2, w);
    bool sorted = std::is_sorted(idx.begin(), idx.end());
    CHECK(sorted);
    std::vector<int> cnt(100, 0);
    for (int i : idx) cnt[(size_t)i]++;
    bool prop = true;
    for (int j = 0; j < 100; ++j) prop &= std::abs(cnt[(size_t)j] - 100 * w[(size_t)j]) < 1.0 + 1e-9;
    CHECK(prop);
  }
  CASE("smc_step null dynamics");  // SPEC.md smc_step example 1 (prior-only, h -> 0)
  {
    TargetContext c;
    c.model = NetSpec{{2, 2}};
    const RngStream root(11);
    ParticleEnsemble e = init_ensemble(16, c, root);
    bool eq = true;
    for (double v : e.log_weights) eq &= v == 0.0;
    CHECK(eq);  // SPEC init_ensemble example 1: prior-only -> equal log-weights
    const auto [n, rec] = smc_step(e, ContextTarget{&c}, KernelConfig::hmc(1e-9, 1), root);
    CHECK(approx(rec.ess, 16.0, 1e-9));
    CHECK(!rec.resampled && n.iteration == 1);
  }
  CASE("smc_step determinism");  // SPEC.md smc_step example 2
  {
    const Problem p = problem(3, 40);
    const auto c = scaled_ctx(p, 20, 40);
    const RngStream root(5);
    const ParticleEnsemble e = init_ensemble(8, c, root);
    const auto [a, ra] = smc_step(e, ContextTarget{&c}, KernelConfig::hmc(0.05, 3), root);
    const auto [b, rb] = smc_step(e, ContextTarget{&c}, KernelConfig::hmc(0.05, 3), root);
    CHECK(a.thetas == b.thetas && a.log_weights == b.log_weights && ra.ess == rb.ess);
    SmcOptions four;
    four.num_threads = 4;
    const auto [t4, r4] = smc_step(e, ContextTarget{&c}, KernelConfig::hmc(0.05, 3), root, four);
    CHECK(t4.thetas == a.thetas && t4.log_weights == a.log_weights);  // thread-count invariance
  }
  CASE("smc conjugate 1-D posterior");  // SPEC.md smc_step example 3
  {
    const auto s = make_synthetic(SyntheticKind::kLinearGaussian, 20, 0.5, 42, 1);
    TargetContext c;
    c.data = &s.data;
    c.window = SubsetWindow{0, 20, 20};
    c.model = LinearGaussianSpec{1, 0.5};
    // analytic posterior (dataset.hpp:276-290 restated for D = 1)
    double xx = 0, xy = 0;
    for (int i = 0; i < 20; ++i) {
      xx += s.data.features[(size_t)i] * s.data.features[(size_t)i];
      xy += s.data.features[(size_t)i] * s.data.targets[(size_t)i];
    }
    const double prec = xx / 0.25 + 1.0, mean = (xy / 0.25) / prec, sd = std::sqrt(1.0 / prec);
    const RngStream root(77);
    ParticleEnsemble e = init_ensemble(512, c, root);
    double last_ess = 512;
    for (int k = 0; k < 50; ++k) {
      auto [n, rec] = smc_step(e, ContextTarget{&c}, KernelConfig::hmc(0.05, 5), root);
      e = std::move(n);
      last_ess = rec.ess;
    }
    const Vec w = normalize(e.log_weights);
    double est = 0;
    for (int64_t j = 0; j < 512; ++j) est += w[(size_t)j] * e.thetas[(size_t)j];
    CHECK(std::abs(est - mean) < 3.0 * sd / std::sqrt(std::max(1.0, ess(w))) + 3.0 * sd / std::sqrt(512.0));
    CHECK(last_ess >= 1.0);
  }
}

static void test_annealing_spec() {
  CASE("batch_size KATs");  // SPEC.md annealing batch_size examples + acceptance 4
  {
    const ScheduleConfig cst{ScheduleKind::kConstant, 500, 500, 200, 60000};
    CHECK(batch_size(cst, 0) == 500 && batch_size(cst, 199) == 500);
    const ScheduleConfig ctr{ScheduleKind::kCtr, 500, 500, 200, 60000};
    CHECK(batch_size(ctr, 180) == 60000 && batch_size(ctr, 179) == 500);
    const ScheduleConfig aut{ScheduleKind::kAutomated, 500, 500, 200, 60000};
    CHECK(batch_size(aut, 1) == 1000);
    CHECK(batch_size(aut, 0) == 500 && batch_size(aut, 180) == 60000);
    const ScheduleConfig lin{ScheduleKind::kLinear, 500, 500, 200, 60000};
    CHECK(batch_size(lin, 3) == 2000 && batch_size(lin, 179) == 60000 && batch_size(lin, 150) == 60000);
    const ScheduleConfig fb{ScheduleKind::kFullBatch, 500, 500, 200, 60000};
    CHECK(batch_size(fb, 7) == 60000);
    CHECK_THROWS(batch_size(cst, 200));
    CHECK_THROWS(batch_size(ScheduleConfig{ScheduleKind::kSda, 500, 500, 200, 60000}, 0));
    bool mono = true;
    for (int k = 1; k < 200; ++k) mono &= batch_size(aut, k) >= batch_size(aut, k - 1);
    CHECK(mono);
  }
  CASE("batch_size [EXT] period/switch");  // BASELINE C1 / C2 semantics (Appendix A.2-A.3)
  {
    const ScheduleConfig c1{ScheduleKind::kCtr, 200, 100, 50, 2000, 1, 40};
    CHECK(batch_size(c1, 39) == 200 && batch_size(c1, 40) == 2000);
    const ScheduleConfig c2{ScheduleKind::kLinear, 1000, 1000, 300, 60000, 5, 300};
    CHECK(batch_size(c2, 0) == 1000 && batch_size(c2, 4) == 1000 && batch_size(c2, 5) == 2000 &&
          batch_size(c2, 299) == 60000 && batch_size(c2, 149) == 30000);
  }
  CASE("sda beta KATs");  // SPEC.md sda_beta_update_initial / annealed examples
  CHECK(approx(sda_beta_update_initial(0.1, 1.0, 10.0), 0.2, 1e-12));
  CHECK(sda_beta_update_initial(0.9, -1.0, 5.0) == 1.0);
  CHECK(approx(sda_beta_update_initial(0.5, -1.0, 4.0), 0.75, 1e-12));
  CHECK(approx(sda_beta_update_annealed(0.9, -1.0, 5.0, 5.0), 1.0, 1e-12));
  CHECK(sda_beta_update_annealed(0.5, 1.0, 3.0, -3.0) == 1.0);
  CHECK(approx(sda_beta_update_annealed(0.2, 1.0, 2.0, 2.0), 0.45, 1e-12));
  CASE("sda flip persists");  // annealing.hpp:190 (the flip is stored in next.entropy_step)
  {
    double step = 1.0;
    sda_beta_step(0.1, step, 10.0);
    CHECK(step == -1.0);
  }
  CASE("sda_advance absorption");  // SPEC.md sda_advance example 1
  {
    const ScheduleConfig c{ScheduleKind::kSda, 500, 500, 200, 60000};
    SdaState s = sda_init(c);
    s.window = SubsetWindow{500, 1000, 60000};
    s.stage = SdaStage::kAnnealed;
    s.beta = 0.9;
    s.entropy_step = -1.0;
    SdaMoments m;
    m.var_block = 5.0;
    m.cov_prefix_block = 5.0;  // -> beta 1.0
    const SdaState t = sda_advance_with(c, s, m);
    CHECK(t.window.prefix_end == 1000 && t.window.block_end == 1500 && t.beta == 0.1);
    SdaState term = s;
    term.window = SubsetWindow{59500, 60000, 60000};
    const SdaState u = sda_advance_with(c, term, m);
    CHECK(u.terminal && u.beta == 1.0 && u.window.prefix_end == 60000);
  }
  CASE("sda moments KATs");  // SPEC.md sda_moments examples
  {
    const SdaMoments m = sda_moments_from({1, 1, 1}, {2, 2, 2}, {0, 0, 0});
    CHECK(approx(m.var_block, 0.0, 1e-5, 1e-12) && approx(m.cov_prefix_block, 0.0, 1e-5, 1e-12));
    const SdaMoments h = sda_moments_from({1, 2, 4}, {3, 1, 2}, {std::log(0.2), std::log(0.5), std::log(0.3)});
    // hand evaluation: E[B]=0.6+0.5+0.6=1.7; E[B^2]=1.8+0.5+1.2=3.5; Var=0.61
    CHECK(approx(h.mean_block, 1.7, 1e-12) && approx(h.mean_block_sq, 3.5, 1e-12) && approx(h.var_block, 0.61, 1e-10));
    // E[P]=0.2+1+1.2=2.4; E[PB]=0.6+1+2.4=4.0; Cov=4.0-2.4*1.7=-0.08
    CHECK(approx(h.mean_prefix, 2.4, 1e-12) && approx(h.mean_prod, 4.0, 1e-12) && approx(h.cov_prefix_block, -0.08, 1e-9));
  }
}

int main() {
  test_rng();
  test_numeric();
  test_network();
  test_target();
  test_kernels();
  test_dataset();
  test_smc_spec();
  test_annealing_spec();
  std::printf("oracle_tests: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
