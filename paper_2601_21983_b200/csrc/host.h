// Host-side (CPU) pieces of the B200 driver: the splittable RNG
// (rng.hpp:14-113), xoshiro256++ jump-ahead polynomials used to parallelise a
// stream on the device, the annealing schedules and SDA controller
// (annealing.hpp), the data permutation and the teacher-labelled synthetic
// data generator.  This is product code (not the oracle); it is kept in plain
// C++ compiled with -ffp-contract=off so its double arithmetic matches the
// reference's IEEE semantics bit for bit.
#pragma once

#include <array>
#include <stdexcept>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dasmc_gpu.h"

namespace dasmc_b200 {

// ---- RngStream (rng.hpp:14-113) ---------------------------------------------------
#if defined(__CUDACC__)
#define DASMC_HD __host__ __device__ __forceinline__
#else
#define DASMC_HD inline
#endif

DASMC_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
DASMC_HD uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// Child key of fork(a, b, c) (rng.hpp:40-46).
DASMC_HD uint64_t fork_key(uint64_t key, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t k = splitmix64(key ^ 0x8e2f0c5a61d3b947ULL);
  k = splitmix64(k ^ a);
  k = splitmix64(k ^ b);
  return splitmix64(k ^ c);
}

struct Xoshiro {  // rng.hpp:48-58, 91-98
  uint64_t s[4];
  DASMC_HD void seed(uint64_t key) {
    uint64_t x = key;
    for (int i = 0; i < 4; ++i) {
      x = splitmix64(x);
      s[i] = x;
    }
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
  }
  DASMC_HD void step() {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
  }
  DASMC_HD uint64_t next() {
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    step();
    return out;
  }
  DASMC_HD double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  // Jump by n steps given r(x) = x^n mod P(x) (256 coefficient bits, LSB first).
  DASMC_HD void jump(const uint64_t* r) {
    uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    for (int w = 0; w < 4; ++w) {
      uint64_t bits = r[w];
      for (int b = 0; b < 64; ++b) {
        if (bits & 1ULL) {
          t0 ^= s[0];
          t1 ^= s[1];
          t2 ^= s[2];
          t3 ^= s[3];
        }
        bits >>= 1;
        step();
      }
    }
    s[0] = t0;
    s[1] = t1;
    s[2] = t2;
    s[3] = t3;
  }
};

namespace tag {  // rng.hpp:106-113
constexpr uint64_t kInit = 1, kProposal = 2, kResample = 3, kPermutation = 4, kSynthetic = 5, kRedraw = 6;
}

struct HostRng {
  Xoshiro x;
  explicit HostRng(uint64_t key) { x.seed(key); }
  uint64_t next_u64() { return x.next(); }
  double uniform() { return x.uniform(); }
  uint64_t uniform_below(uint64_t n);  // rng.hpp:66-73
  double normal();                     // rng.hpp:76-81
};

// Jump polynomials r_c(x) = x^(c*L) mod P(x), P = characteristic polynomial
// of the xoshiro256 state transition (found by Berlekamp-Massey).
const std::array<uint64_t, 4>& jump_poly_unit();  // x^1 mod P (sanity)
std::vector<std::array<uint64_t, 4>> jump_table(uint64_t chunk_steps, int64_t nchunks);

// ---- schedules / SDA (annealing.hpp) -------------------------------------------------
void validate_schedule(const dasmc_schedule& c);
int64_t batch_size(const dasmc_schedule& c, int k);
double sda_beta_step(double beta, double& entropy_step, double denom);
void sda_moments_from(const double* pre_nll, const double* blk_nll, const double* log_w, int64_t J,
                      double* out6);
dasmc_sda_state sda_init(const dasmc_schedule& c, double beta0, double entropy_step);
dasmc_sda_state sda_advance_with(const dasmc_schedule& c, const dasmc_sda_state& s, const double* m6);

// normalize (smc.hpp:57-64); throws on all -inf.
std::vector<double> normalize(const double* lw, int64_t J);

// ---- data -------------------------------------------------------------------------------
std::vector<int64_t> shuffle_permutation(uint64_t seed, int64_t n);
std::vector<int64_t> redraw_rows(uint64_t seed, int k, int64_t n, int64_t count);  // runner.hpp:531-542
void make_synthetic(int kind, int64_t n, double noise, uint64_t seed, float* X, int32_t* y);  // dataset.hpp:208-267

// IDX image/label files (dataset.hpp:84-196): FormatError texts as the reference.
struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IdxData {
  int64_t n = 0, d = 0;
  int num_classes = 0;
  std::vector<float> X;   // pixels / 255
  std::vector<int32_t> y;
};
IdxData parse_idx(const std::vector<unsigned char>& image_bytes, const std::vector<unsigned char>& label_bytes);
std::vector<unsigned char> read_file_bytes(const std::string& path);  // gzip decompressed transparently
void make_teacher_data(const std::vector<int>& layers, int act, int64_t n, int feature_kind, uint64_t seed,
                       uint64_t cfg_id, int threads, float* X, int32_t* y, const int* conv = nullptr);

// ---- errors ------------------------------------------------------------------------------
struct Error {
  int code;
  std::string msg;
};
void set_last_error(const std::string& m);

}  // namespace dasmc_b200
