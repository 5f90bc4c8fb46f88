#include "rng.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>
#include <thread>
#include <vector>

namespace npcg {

namespace {
inline double box_muller(std::uint64_t w1, std::uint64_t w2) {
  // random.cpp:11-18
  const double u1 = (static_cast<double>(w1) + 1.0) * 0x1.0p-64;
  const double u2 = static_cast<double>(w2) * 0x1.0p-64;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}
}  // namespace

double HostRng::normal() {
  const std::uint64_t w1 = engine();
  const std::uint64_t w2 = engine();
  return box_muller(w1, w2);
}

double HostRng::uniform() { return static_cast<double>(engine()) * 0x1.0p-64; }

std::uint64_t HostRng::integer(std::uint64_t bound) {
  if (bound == 0) throw std::invalid_argument("Rng - integer: bound must be positive");
  return std::uniform_int_distribution<std::uint64_t>(0, bound - 1)(engine);
}

void HostRng::gaussian(std::int64_t rows, std::int64_t cols, double* dst) {
  const std::int64_t total = rows * cols;
  if (total <= 0) return;
  if (total < (1 << 16)) {
    for (std::int64_t k = 0; k < total; ++k) dst[k] = normal();
    return;
  }
  // Words are drawn in stream order in chunks; the transform is parallel.
  const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  constexpr std::int64_t kChunk = 1 << 20;
  std::vector<std::uint64_t> words(static_cast<size_t>(2 * std::min(total, kChunk)));
  for (std::int64_t base = 0; base < total; base += kChunk) {
    const std::int64_t cnt = std::min(kChunk, total - base);
    for (std::int64_t k = 0; k < 2 * cnt; ++k) words[static_cast<size_t>(k)] = engine();
    const std::int64_t per = (cnt + hw - 1) / hw;
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < hw; ++t) {
      const std::int64_t lo = t * per, hi = std::min(cnt, lo + per);
      if (lo >= hi) break;
      pool.emplace_back([&, lo, hi] {
        for (std::int64_t k = lo; k < hi; ++k)
          dst[base + k] = box_muller(words[static_cast<size_t>(2 * k)], words[static_cast<size_t>(2 * k + 1)]);
      });
    }
    for (auto& th : pool) th.join();
  }
}

}  // namespace npcg
