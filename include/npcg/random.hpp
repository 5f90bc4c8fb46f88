// reference: random.hpp:11-50 — the seeded mt19937_64 + Box-Muller generator,
// bit for bit (implemented host-side in libnpcg_b200, npcg_rng_*).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "types.hpp"

namespace npcg {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) { check_status(npcg_rng_create(seed, &h_)); }
  Rng(const Rng& o) { check_status(npcg_rng_clone(o.h_, &h_)); }
  Rng& operator=(const Rng& o) {
    if (this != &o) {
      npcg_rng_destroy(h_);
      check_status(npcg_rng_clone(o.h_, &h_));
    }
    return *this;
  }
  ~Rng() { npcg_rng_destroy(h_); }

  double normal() { return npcg_rng_normal(h_); }      // random.cpp:11-18
  double uniform() { return npcg_rng_uniform(h_); }    // random.cpp:20
  std::uint64_t integer(std::uint64_t bound) {         // random.cpp:22-25
    std::uint64_t out = 0;
    check_status(npcg_rng_integer(h_, bound, &out));
    return out;
  }
  npcg_rng* handle() const { return h_; }

 private:
  npcg_rng* h_ = nullptr;
};

inline Matrix gaussian_matrix(Rng& rng, Index rows, Index cols) {  // random.cpp:27-32
  Matrix g(rows, cols);
  check_status(npcg_rng_gaussian(rng.handle(), rows, cols, g.data()));
  return g;
}

inline Vector gaussian_vector(Rng& rng, Index n) {  // random.cpp:34-38
  Vector v(n);
  check_status(npcg_rng_gaussian(rng.handle(), n, 1, v.data()));
  return v;
}

inline std::vector<Index> sample_without_replacement(Rng& rng, Index n, Index k) {  // random.cpp:44-56
  std::vector<std::int64_t> tmp(static_cast<size_t>(k > 0 ? k : 0));
  check_status(npcg_rng_sample(rng.handle(), n, k, tmp.data()));
  return std::vector<Index>(tmp.begin(), tmp.end());
}

}  // namespace npcg
