// The reference generator (random.hpp:21-38, random.cpp:11-56), bit for bit:
// std::mt19937_64 + cache-free Box-Muller (two engine words per normal, sine
// partner discarded), column-major block fills. Host-side by design: it
// supplies the Ω blocks / right-hand sides / power vectors the GPU consumes.
// Bulk fills draw the engine words sequentially (the stream is inherently
// serial) and run the Box-Muller transform on all host cores — same bits,
// same stream position as the reference's scalar loop.
#pragma once

#include <cstdint>
#include <random>

namespace npcg {

/// std::mt19937_64, restated with its state in the open (the GPU generator
/// continues the stream from it and hands it back). Output-for-output equal
/// to libstdc++'s engine (same seeding, twist and tempering; a URBG with the
/// same min/max, so std::uniform_int_distribution takes the same branches).
struct Mt64 {
  static constexpr int kN = 312, kM = 156;
  static constexpr std::uint64_t kA = 0xB5026F5AA96619E9ull, kUpper = ~std::uint64_t{0} << 31,
                                 kLower = (std::uint64_t{1} << 31) - 1;
  using result_type = std::uint64_t;
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~result_type{0}; }
  std::uint64_t x[kN];
  int p = kN;      // next output is temper(x[p]); kN: the block is used up
  std::uint64_t words = 0;  // outputs drawn so far (diagnostics)
  explicit Mt64(std::uint64_t seed = 5489u) {
    x[0] = seed;
    for (int i = 1; i < kN; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    p = kN;
  }
  static std::uint64_t temper(std::uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
  }
  static std::uint64_t mix(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    const std::uint64_t y = (a & kUpper) | (b & kLower);
    return c ^ (y >> 1) ^ ((y & 1) ? kA : 0);
  }
  void twist() {  // in place, as libstdc++'s _M_gen_rand
    int k = 0;
    for (; k < kN - kM; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM]);
    for (; k < kN - 1; ++k) x[k] = mix(x[k], x[k + 1], x[k + kM - kN]);
    x[kN - 1] = mix(x[kN - 1], x[0], x[kM - 1]);
    p = 0;
  }
  result_type operator()() {
    if (p >= kN) twist();
    ++words;
    return temper(x[p++]);
  }
  void discard(std::uint64_t z) {
    for (; z > 0; --z) (*this)();
  }
};

struct HostRng {
  explicit HostRng(std::uint64_t seed) : engine(seed) {}
  Mt64 engine;
  double normal();
  double uniform();
  std::uint64_t integer(std::uint64_t bound);
  /// gaussian_matrix(rows, cols) into dst (col-major, ld = rows).
  void gaussian(std::int64_t rows, std::int64_t cols, double* dst);
};

/// GPU continuation of the stream (rng_gpu.cu): `count` tempered engine words
/// into device memory, the engine advanced exactly as `count` host calls.
struct Ctx;
void device_words(Ctx& ctx, Mt64& e, std::int64_t count, unsigned long long* out);
/// gaussian_matrix(rows, cols) generated on the device (bitwise engine words,
/// CUDA log / cos); rows [r0, r0 + rcnt) of each column into dst (device, ld).
void device_gaussian(Ctx& ctx, Mt64& e, std::int64_t rows, std::int64_t cols, std::int64_t r0, std::int64_t rcnt,
                     double* dst, std::int64_t ld);

}  // namespace npcg
