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

struct HostRng {
  explicit HostRng(std::uint64_t seed) : engine(seed) {}
  std::mt19937_64 engine;
  double normal();
  double uniform();
  std::uint64_t integer(std::uint64_t bound);
  /// gaussian_matrix(rows, cols) into dst (col-major, ld = rows).
  void gaussian(std::int64_t rows, std::int64_t cols, double* dst);
};

}  // namespace npcg
