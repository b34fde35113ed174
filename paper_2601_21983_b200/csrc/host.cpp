// Host-side pieces of the B200 driver (see host.h).
#include "host.h"

#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <thread>

namespace dasmc_b200 {

uint64_t HostRng::uniform_below(uint64_t n) {  // rng.hpp:66-73
  if (n == 0) throw std::invalid_argument("uniform_below: n must be positive");
  const uint64_t limit = ~uint64_t{0} - (~uint64_t{0} % n);
  uint64_t v = next_u64();
  while (v >= limit) v = next_u64();
  return v % n;
}

double HostRng::normal() {  // rng.hpp:76-81
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

// ---- GF(2)[x] arithmetic for the jump-ahead ----------------------------------------------
namespace {

using Poly = std::array<uint64_t, 9>;  // up to 576 bits

int poly_deg(const Poly& p) {
  for (int w = 8; w >= 0; --w)
    if (p[(size_t)w]) return w * 64 + 63 - __builtin_clzll(p[(size_t)w]);
  return -1;
}
bool poly_bit(const Poly& p, int i) { return (p[(size_t)(i >> 6)] >> (i & 63)) & 1ULL; }
void poly_flip(Poly& p, int i) { p[(size_t)(i >> 6)] ^= 1ULL << (i & 63); }

Poly poly_mulmod(const Poly& a, const Poly& b, const Poly& m, int dm) {
  Poly r{};
  const int da = poly_deg(a);
  for (int i = 0; i <= da; ++i) {
    if (!poly_bit(a, i)) continue;
    // r ^= b << i
    const int ws = i >> 6, bs = i & 63;
    for (int w = 8; w >= 0; --w) {
      if (w - ws < 0) break;
      uint64_t v = b[(size_t)(w - ws)] << bs;
      if (bs && w - ws - 1 >= 0) v |= b[(size_t)(w - ws - 1)] >> (64 - bs);
      r[(size_t)w] ^= v;
    }
  }
  for (int d = poly_deg(r); d >= dm; d = poly_deg(r)) {
    const int sh = d - dm;
    const int ws = sh >> 6, bs = sh & 63;
    for (int w = 8; w >= 0; --w) {
      if (w - ws < 0) break;
      uint64_t v = m[(size_t)(w - ws)] << bs;
      if (bs && w - ws - 1 >= 0) v |= m[(size_t)(w - ws - 1)] >> (64 - bs);
      r[(size_t)w] ^= v;
    }
  }
  return r;
}

struct CharPoly {
  Poly p{};
  int deg = 0;
};

// Berlekamp-Massey on bit 0 of state word 0 gives the minimal polynomial of
// the F2-linear state transition (degree 256: xoshiro256 has full period).
const CharPoly& char_poly() {
  static const CharPoly cp = [] {
    Xoshiro x;
    x.seed(0x1234567ULL);
    const int N = 1024;
    std::vector<int> s((size_t)N);
    for (int t = 0; t < N; ++t) {
      s[(size_t)t] = (int)(x.s[0] & 1ULL);
      x.step();
    }
    std::vector<int> C((size_t)N + 1, 0), B((size_t)N + 1, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < N; ++n) {
      int d = s[(size_t)n];
      for (int i = 1; i <= L; ++i) d ^= C[(size_t)i] & s[(size_t)(n - i)];
      if (d == 0) {
        ++m;
      } else if (2 * L <= n) {
        T = C;
        for (int i = 0; i + m <= N; ++i) C[(size_t)(i + m)] ^= B[(size_t)i];
        L = n + 1 - L;
        B = T;
        m = 1;
      } else {
        for (int i = 0; i + m <= N; ++i) C[(size_t)(i + m)] ^= B[(size_t)i];
        ++m;
      }
    }
    if (L != 256) throw std::runtime_error("xoshiro char poly: unexpected degree");
    CharPoly out;
    out.deg = L;
    // P(x) = x^L C(1/x): coefficient of x^(L-i) is C[i].
    for (int i = 0; i <= L; ++i)
      if (C[(size_t)i]) poly_flip(out.p, L - i);
    return out;
  }();
  return cp;
}

std::array<uint64_t, 4> to4(const Poly& p) { return {p[0], p[1], p[2], p[3]}; }

Poly x_pow_mod(uint64_t n) {  // x^n mod P by square-and-multiply
  const CharPoly& cp = char_poly();
  Poly result{};
  result[0] = 1;
  Poly base{};
  base[0] = 2;  // x
  while (n) {
    if (n & 1ULL) result = poly_mulmod(result, base, cp.p, cp.deg);
    base = poly_mulmod(base, base, cp.p, cp.deg);
    n >>= 1;
  }
  return result;
}

}  // namespace

const std::array<uint64_t, 4>& jump_poly_unit() {
  static const std::array<uint64_t, 4> u = to4(x_pow_mod(1));
  return u;
}

std::vector<std::array<uint64_t, 4>> jump_table(uint64_t chunk_steps, int64_t nchunks) {
  const CharPoly& cp = char_poly();
  std::vector<std::array<uint64_t, 4>> out((size_t)nchunks);
  const Poly step = x_pow_mod(chunk_steps);
  Poly cur{};
  cur[0] = 1;
  for (int64_t c = 0; c < nchunks; ++c) {
    out[(size_t)c] = to4(cur);
    cur = poly_mulmod(cur, step, cp.p, cp.deg);
  }
  return out;
}

// ---- schedules (annealing.hpp:23-82) ------------------------------------------------------
void validate_schedule(const dasmc_schedule& c) {
  if (c.initial_batch < 1 || c.initial_batch > c.dataset_size)
    throw std::invalid_argument("ScheduleConfig: need 1 <= initial_batch <= dataset_size");
  if (c.increment < 1 || c.increment > c.dataset_size)
    throw std::invalid_argument("ScheduleConfig: need 1 <= increment <= dataset_size");
  if (c.iterations < 1) throw std::invalid_argument("ScheduleConfig: iterations must be >= 1");
  if (c.period < 1) throw std::invalid_argument("ScheduleConfig: period must be >= 1");
}

int64_t batch_size(const dasmc_schedule& c, int k) {
  validate_schedule(c);
  if (k < 0 || k >= c.iterations) throw std::invalid_argument("batch_size: k out of range");
  if (c.kind == DASMC_SCHED_SDA) throw std::invalid_argument("batch_size: the sda schedule is state-driven");
  const double switch_point = 0.9 * (double)c.iterations;
  const bool early = c.switch_iteration < 0 ? (double)k < switch_point : k < c.switch_iteration;
  switch (c.kind) {
    case DASMC_SCHED_CONSTANT: return c.initial_batch;
    case DASMC_SCHED_FULL_BATCH: return c.dataset_size;
    case DASMC_SCHED_CTR: return early ? c.initial_batch : c.dataset_size;
    case DASMC_SCHED_LINEAR:
      return early ? std::min(c.increment * (int64_t)(k / c.period) + c.initial_batch, c.dataset_size)
                   : c.dataset_size;
    case DASMC_SCHED_AUTOMATED: {
      if (!early) return c.dataset_size;
      const auto slope = (int64_t)std::floor((double)(c.dataset_size - c.initial_batch) / switch_point);
      const int64_t raw = c.initial_batch + slope * k;
      const int64_t rounded = (int64_t)std::floor((double)raw / (double)c.increment + 0.5) * c.increment;
      return std::clamp(rounded, c.initial_batch, c.dataset_size);
    }
    default: break;
  }
  throw std::invalid_argument("batch_size: unknown schedule kind");
}

double sda_beta_step(double beta, double& step, double denom) {  // annealing.hpp:114-122
  if (denom == 0.0) return 1.0;
  double cand = beta - step / denom;
  if (cand <= beta) {
    step = -step;
    cand = beta - step / denom;
  }
  return std::min(cand, 1.0);
}

std::vector<double> normalize(const double* lw, int64_t J) {  // smc.hpp:57-64
  if (J < 1) throw std::invalid_argument("normalize: empty weights");
  double m = lw[0];
  for (int64_t j = 0; j < J; ++j) m = std::max(m, lw[j]);
  if (m == -INFINITY) throw std::runtime_error("normalize: all particles dead (every log-weight is -inf)");
  std::vector<double> w((size_t)J);
  double s = 0.0;
  for (int64_t j = 0; j < J; ++j) {
    w[(size_t)j] = std::exp(lw[j] - m);
    s += w[(size_t)j];
  }
  for (auto& v : w) v /= s;
  return w;
}

// sda_moments's six estimators (annealing.hpp:166-173; numeric.hpp:49-78).
void sda_moments_from(const double* pre, const double* blk, const double* lw, int64_t J, double* out6) {
  const std::vector<double> w = normalize(lw, J);
  double sum = 0.0;
  for (double v : w) sum += v;
  if (std::abs(sum - 1.0) > 1e-9) throw std::invalid_argument("weights: must sum to 1");
  double mb = 0, mbsq = 0, mp = 0, mprod = 0;
  for (int64_t j = 0; j < J; ++j) mb += w[(size_t)j] * blk[j];
  for (int64_t j = 0; j < J; ++j) mbsq += w[(size_t)j] * (blk[j] * blk[j]);
  const double var = std::max(0.0, mbsq - mb * mb);
  for (int64_t j = 0; j < J; ++j) mp += w[(size_t)j] * pre[j];
  for (int64_t j = 0; j < J; ++j) mprod += w[(size_t)j] * (pre[j] * blk[j]);
  out6[0] = mb;
  out6[1] = mbsq;
  out6[2] = var;
  out6[3] = mp;
  out6[4] = mprod;
  out6[5] = mprod - mp * mb;
}

dasmc_sda_state sda_init(const dasmc_schedule& c, double beta0, double entropy_step) {  // annealing.hpp:98-110
  validate_schedule(c);
  if (!(beta0 > 0.0 && beta0 <= 1.0)) throw std::invalid_argument("sda_init: beta0 must be in (0, 1]");
  dasmc_sda_state s{};
  s.beta = beta0;
  s.beta_reset = beta0;
  s.entropy_step = entropy_step;
  s.prefix_end = 0;
  s.block_end = c.initial_batch;
  s.total_n = c.dataset_size;
  s.stage = 0;
  s.terminal = 0;
  return s;
}

dasmc_sda_state sda_advance_with(const dasmc_schedule& c, const dasmc_sda_state& s, const double* m) {
  if (s.terminal) return s;  // annealing.hpp:185
  dasmc_sda_state n = s;
  const double denom = s.stage == 0 ? m[2] : m[2] + m[5];
  const double bnew = sda_beta_step(s.beta, n.entropy_step, denom);
  if (bnew >= 1.0) {
    const int64_t absorbed = s.block_end;
    if (absorbed >= c.dataset_size) {
      n.beta = 1.0;
      n.prefix_end = n.block_end = n.total_n = c.dataset_size;
      n.stage = 1;
      n.terminal = 1;
    } else {
      n.beta = s.beta_reset;
      n.prefix_end = absorbed;
      n.block_end = std::min(absorbed + c.increment, c.dataset_size);
      n.total_n = c.dataset_size;
      n.stage = 1;
    }
  } else {
    n.beta = bnew;
  }
  return n;
}

// ---- data ----------------------------------------------------------------------------------
std::vector<int64_t> shuffle_permutation(uint64_t seed, int64_t n) {  // dataset.hpp:294-301
  std::vector<int64_t> order((size_t)n);
  for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
  HostRng r(fork_key(seed, tag::kPermutation, 0, 0));
  for (int64_t i = n - 1; i > 0; --i) {
    const auto j = (int64_t)r.uniform_below((uint64_t)(i + 1));
    std::swap(order[(size_t)i], order[(size_t)j]);
  }
  return order;
}

// ---- IDX data files (dataset.hpp:84-196) -------------------------------------------------
namespace {
uint32_t read_be32(const std::vector<unsigned char>& b, size_t off, const char* field) {
  if (off + 4 > b.size())
    throw FormatError(std::string("IDX: truncated while reading ") + field + " at offset " + std::to_string(off));
  return (uint32_t(b[off]) << 24) | (uint32_t(b[off + 1]) << 16) | (uint32_t(b[off + 2]) << 8) | uint32_t(b[off + 3]);
}

std::vector<unsigned char> gunzip(const std::vector<unsigned char>& in) {
  z_stream zs{};
  if (inflateInit2(&zs, 15 + 16) != Z_OK) throw FormatError("gzip: inflateInit failed");
  std::vector<unsigned char> out;
  out.reserve(in.size() * 4);
  std::vector<unsigned char> buf(1 << 16);
  zs.next_in = const_cast<unsigned char*>(in.data());
  zs.avail_in = (uInt)in.size();
  int rc = Z_OK;
  do {
    zs.next_out = buf.data();
    zs.avail_out = (uInt)buf.size();
    rc = inflate(&zs, Z_NO_FLUSH);
    if (rc != Z_OK && rc != Z_STREAM_END) {
      inflateEnd(&zs);
      throw FormatError("gzip: corrupt stream (zlib rc " + std::to_string(rc) + ")");
    }
    out.insert(out.end(), buf.data(), buf.data() + (buf.size() - zs.avail_out));
    if (rc != Z_STREAM_END && zs.avail_in == 0 && zs.avail_out != 0) {
      inflateEnd(&zs);
      throw FormatError("gzip: truncated stream");
    }
  } while (rc != Z_STREAM_END);
  inflateEnd(&zs);
  return out;
}
}  // namespace

IdxData parse_idx(const std::vector<unsigned char>& img, const std::vector<unsigned char>& lab) {
  constexpr uint32_t kImageMagic = 0x00000803, kLabelMagic = 0x00000801;
  const uint32_t im = read_be32(img, 0, "image magic");
  if (im != kImageMagic) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), "IDX image magic: expected 0x%08x, got 0x%08x at offset 0", kImageMagic, im);
    throw FormatError(buf);
  }
  const uint32_t n = read_be32(img, 4, "image count");
  const uint32_t rows = read_be32(img, 8, "image rows");
  const uint32_t cols = read_be32(img, 12, "image cols");
  const size_t pixels = size_t(n) * rows * cols;
  if (img.size() != 16 + pixels)
    throw FormatError("IDX image payload: expected " + std::to_string(16 + pixels) + " bytes, got " +
                      std::to_string(img.size()));
  const uint32_t lm = read_be32(lab, 0, "label magic");
  if (lm != kLabelMagic) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), "IDX label magic: expected 0x%08x, got 0x%08x at offset 0", kLabelMagic, lm);
    throw FormatError(buf);
  }
  const uint32_t nl = read_be32(lab, 4, "label count");
  if (lab.size() != 8 + size_t(nl))
    throw FormatError("IDX label payload: expected " + std::to_string(8 + size_t(nl)) + " bytes, got " +
                      std::to_string(lab.size()));
  if (nl != n)
    throw FormatError("IDX count mismatch: " + std::to_string(n) + " images vs " + std::to_string(nl) + " labels");
  IdxData d;
  d.n = n;
  d.d = (int64_t)rows * cols;
  d.X.resize(pixels);
  d.y.resize(n);
  int max_label = 0;
  for (size_t p = 0; p < pixels; ++p) d.X[p] = (float)((double)img[16 + p] / 255.0);
  for (uint32_t i = 0; i < n; ++i) {
    d.y[i] = lab[8 + i];
    max_label = std::max(max_label, (int)d.y[i]);
  }
  d.num_classes = max_label + 1;
  return d;
}

std::vector<unsigned char> read_file_bytes(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw FormatError("cannot open file: " + path);
  std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (bytes.size() >= 2 && bytes[0] == 0x1f && bytes[1] == 0x8b) return gunzip(bytes);
  return bytes;
}

// make_synthetic (dataset.hpp:208-267), the classification kinds the runner feeds to an MLP:
// kind 0 = gaussian_blobs (3 classes), 1 = two_moons (2 classes); 2-D features, stream
// RngStream(seed).fork(kSynthetic).
void make_synthetic(int kind, int64_t n, double noise, uint64_t seed, float* X, int32_t* y) {
  if (n < 2) throw std::invalid_argument("make_synthetic: n must be >= 2");
  if (kind != 0 && kind != 1) throw std::invalid_argument("make_synthetic: classification kinds only (blobs, moons)");
  HostRng r(fork_key(seed, tag::kSynthetic, 0, 0));
  constexpr double kPi = 3.141592653589793;
  for (int64_t i = 0; i < n; ++i) {
    double x0, x1;
    if (kind == 0) {
      const int c = (int)(i % 3);
      const double angle = 2.0 * kPi * c / 3;
      x0 = 3.0 * std::cos(angle) + noise * r.normal();
      x1 = 3.0 * std::sin(angle) + noise * r.normal();
      y[i] = c;
    } else {
      const int c = (int)(i % 2);
      const double t = kPi * r.uniform();
      double a, b;
      if (c == 0) {
        a = std::cos(t);
        b = std::sin(t);
      } else {
        a = 1.0 - std::cos(t);
        b = 0.5 - std::sin(t);
      }
      x0 = a + noise * r.normal();
      x1 = b + noise * r.normal();
      y[i] = c;
    }
    X[2 * i] = (float)x0;
    X[2 * i + 1] = (float)x1;
  }
}

// draw_batch_rows (runner.hpp:531-542): partial Fisher-Yates over 0..n-1 with the
// stream root.fork(kRedraw, k), i = 0..count-1, j = i + uniform_below(n - i).
std::vector<int64_t> redraw_rows(uint64_t seed, int k, int64_t n, int64_t count) {
  std::vector<int64_t> order((size_t)n);
  for (int64_t i = 0; i < n; ++i) order[(size_t)i] = i;
  HostRng r(fork_key(seed, tag::kRedraw, (uint64_t)k, 0));
  for (int64_t i = 0; i < count; ++i) {
    const auto j = i + (int64_t)r.uniform_below((uint64_t)(n - i));
    std::swap(order[(size_t)i], order[(size_t)j]);
  }
  order.resize((size_t)count);
  return order;
}

void make_teacher_data(const std::vector<int>& layers, int act, int64_t n, int feature_kind, uint64_t seed,
                       uint64_t cfg_id, int threads, float* X, int32_t* y, const int* conv) {
  // [EXT] conv != nullptr: a CNN teacher (dasmc_gpu.h), same loops as the oracle's cnn_stages
  struct Stage {
    int cin, hin, win, k, cout, ho, wo, sh, sw, pool;
    int64_t woff, boff;
  };
  std::vector<Stage> st;
  int64_t D = 0;
  int d = layers.front();
  if (conv != nullptr) {
    int ch = conv[0], h = conv[1], w = conv[2];
    d = ch * h * w;
    for (int i = 0; i < conv[3]; ++i) {
      Stage s{ch, h, w, conv[4 + 3 * i], conv[5 + 3 * i], 0, 0, 0, 0, conv[6 + 3 * i] != 0 ? 1 : 0, 0, 0};
      s.ho = h - s.k + 1;
      s.wo = w - s.k + 1;
      s.sh = s.pool ? s.ho / 2 : s.ho;
      s.sw = s.pool ? s.wo / 2 : s.wo;
      s.woff = D;
      D += (int64_t)s.cout * s.cin * s.k * s.k;
      s.boff = D;
      D += s.cout;
      st.push_back(s);
      ch = s.cout;
      h = s.sh;
      w = s.sw;
    }
  }
  const int64_t Dconv = D;
  std::vector<double> F((size_t)n * d);
  HostRng fx(fork_key(seed, tag::kSynthetic, cfg_id, 1));
  for (auto& v : F) v = feature_kind == 0 ? fx.uniform() : (double)fx.uniform_below(256) / 255.0;
  for (size_t l = 1; l < layers.size(); ++l) D += (int64_t)layers[l - 1] * layers[l] + layers[l];
  HostRng ft(fork_key(seed, tag::kSynthetic, cfg_id, 2));
  std::vector<double> th((size_t)D);
  for (auto& v : th) v = ft.normal();
  auto actf = [&](double z) { return act == DASMC_RELU ? (z > 0.0 ? z : 0.0) : std::tanh(z); };
  auto label_rows = [&](int64_t lo, int64_t hi) {
    std::vector<double> cur, nxt, A;
    for (int64_t i = lo; i < hi; ++i) {
      cur.assign(F.begin() + i * d, F.begin() + (i + 1) * d);
      for (const Stage& s : st) {
        A.assign((size_t)s.cout * s.ho * s.wo, 0.0);
        for (int co = 0; co < s.cout; ++co)
          for (int yy = 0; yy < s.ho; ++yy)
            for (int xx = 0; xx < s.wo; ++xx) {
              double acc = 0.0;
              for (int ci = 0; ci < s.cin; ++ci)
                for (int ky = 0; ky < s.k; ++ky)
                  for (int kx = 0; kx < s.k; ++kx)
                    acc += th[(size_t)(s.woff + (((int64_t)co * s.cin + ci) * s.k + ky) * s.k + kx)] *
                           cur[((size_t)ci * s.hin + yy + ky) * s.win + xx + kx];
              acc += th[(size_t)(s.boff + co)];
              A[((size_t)co * s.ho + yy) * s.wo + xx] = actf(acc);
            }
        if (s.pool) {
          nxt.assign((size_t)s.cout * s.sh * s.sw, 0.0);
          for (int co = 0; co < s.cout; ++co)
            for (int yy = 0; yy < s.sh; ++yy)
              for (int xx = 0; xx < s.sw; ++xx) {
                double mx = A[((size_t)co * s.ho + 2 * yy) * s.wo + 2 * xx];
                for (int dy = 0; dy < 2; ++dy)
                  for (int dx = 0; dx < 2; ++dx)
                    mx = std::max(mx, A[((size_t)co * s.ho + 2 * yy + dy) * s.wo + 2 * xx + dx]);
                nxt[((size_t)co * s.sh + yy) * s.sw + xx] = mx;
              }
          cur.swap(nxt);
        } else {
          cur.swap(A);
        }
      }
      int64_t off = Dconv;
      for (size_t l = 1; l < layers.size(); ++l) {
        const int in = layers[l - 1], out = layers[l];
        nxt.assign((size_t)out, 0.0);
        for (int r = 0; r < out; ++r) {
          double acc = 0.0;
          for (int c = 0; c < in; ++c) acc += th[(size_t)(off + (int64_t)c * out + r)] * cur[(size_t)c];
          acc += th[(size_t)(off + (int64_t)in * out + r)];
          if (l + 1 < layers.size()) acc = actf(acc);
          nxt[(size_t)r] = acc;
        }
        off += (int64_t)in * out + out;
        cur.swap(nxt);
      }
      int best = 0;
      for (int c = 1; c < (int)cur.size(); ++c)
        if (cur[(size_t)c] > cur[(size_t)best]) best = c;
      y[i] = best;
    }
  };
  const int T = std::max(1, std::min<int>(threads, (int)std::max<int64_t>(1, n / 64)));
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) pool.emplace_back(label_rows, n * t / T, n * (t + 1) / T);
  for (auto& p : pool) p.join();
  for (size_t i = 0; i < F.size(); ++i) X[i] = (float)F[i];
}

}  // namespace dasmc_b200
