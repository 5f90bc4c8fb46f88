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
  // Words are drawn in stream order in chunks on this thread while the other
  // threads transform the previous chunk (double-buffered): the serial engine
  // and the parallel Box-Muller transform overlap.
  const unsigned hw = std::max(2u, std::min(64u, std::thread::hardware_concurrency()));
  const unsigned workers = hw - 1;
  constexpr std::int64_t kChunk = 1 << 20;
  const size_t cap = static_cast<size_t>(2 * std::min(total, kChunk));
  std::vector<std::uint64_t> buf[2] = {std::vector<std::uint64_t>(cap), std::vector<std::uint64_t>(cap)};
  auto fill = [&](std::vector<std::uint64_t>& w, std::int64_t cnt) {
    for (std::int64_t k = 0; k < 2 * cnt; ++k) w[static_cast<size_t>(k)] = engine();
  };
  std::int64_t cnt = std::min(kChunk, total);
  fill(buf[0], cnt);
  int cur = 0;
  for (std::int64_t base = 0; base < total; base += kChunk) {
    const std::vector<std::uint64_t>& words = buf[cur];
    const std::int64_t per = (cnt + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < workers; ++t) {
      const std::int64_t lo = t * per, hi = std::min(cnt, lo + per);
      if (lo >= hi) break;
      pool.emplace_back([&words, dst, base, lo, hi] {
        for (std::int64_t k = lo; k < hi; ++k)
          dst[base + k] = box_muller(words[static_cast<size_t>(2 * k)], words[static_cast<size_t>(2 * k + 1)]);
      });
    }
    const std::int64_t next = std::min(kChunk, total - base - kChunk);
    if (next > 0) fill(buf[cur ^ 1], next);  // overlaps the transform of this chunk
    for (auto& th : pool) th.join();
    cnt = next;
    cur ^= 1;
  }
}

}  // namespace npcg
