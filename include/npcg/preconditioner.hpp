// reference: preconditioner.hpp:20-65 — the Nyström preconditioner, applied
// on device in O(n ell) (two skinny GEMVs + the rank-ell correction).
#pragma once

#include <memory>

#include "nystrom.hpp"

namespace npcg {

struct NystromPreconditioner {
  std::shared_ptr<npcg_pre> device;
  std::shared_ptr<npcg_nys> approx;  // keeps U, lambda alive on device
  double lambda_ell = 0.0;
  double mu = 0.0;
  Index n = 0, ell = 0;

  Index dim() const { return n; }
  Index size() const { return ell; }

  /// P^-1 r (preconditioner.cpp:27-36).
  Vector apply_inverse(const Vector& r) const {
    if (r.size() != n) throw std::invalid_argument("NystromPreconditioner - apply_inverse: length mismatch");
    Vector z(n);
    check_status(npcg_pre_apply_inverse(device.get(), 1, r.data(), std::max<Index>(n, 1), z.data(),
                                        std::max<Index>(n, 1), NPCG_HOST));
    return z;
  }
  /// P^-1 R column-wise (preconditioner.cpp:38-45).
  Matrix apply_inverse_block(const Matrix& r) const {
    if (r.rows() != n) throw std::invalid_argument("NystromPreconditioner - apply_inverse_block: row mismatch");
    Matrix z(n, r.cols());
    if (r.cols() > 0)
      check_status(npcg_pre_apply_inverse(device.get(), r.cols(), r.data(), std::max<Index>(n, 1), z.data(),
                                          std::max<Index>(n, 1), NPCG_HOST));
    return z;
  }
  /// P v (preconditioner.cpp:17-25).
  Vector apply(const Vector& v) const {
    if (v.size() != n) throw std::invalid_argument("NystromPreconditioner - apply: length mismatch");
    Vector out(n);
    check_status(npcg_pre_apply(device.get(), 1, v.data(), std::max<Index>(n, 1), out.data(),
                                std::max<Index>(n, 1), NPCG_HOST));
    return out;
  }
};

/// build_preconditioner (preconditioner.cpp:80-89); mu must be > 0.
inline NystromPreconditioner build_preconditioner(const NystromApproximation& approx, double mu) {
  npcg_pre* h = nullptr;
  check_status(npcg_pre_create(approx.device.get(), mu, &h));
  NystromPreconditioner p;
  p.device = std::shared_ptr<npcg_pre>(h, [](npcg_pre* q) { npcg_pre_destroy(q); });
  p.approx = approx.device;
  p.lambda_ell = approx.lambda_min();
  p.mu = mu;
  p.n = approx.dim();
  p.ell = approx.size();
  return p;
}

/// woodbury_inverse_apply(u, lambda, mu, b) (preconditioner.cpp:104-114) on the
/// approximation's device factors: (U diag(lambda) U^T + mu I)^-1 b.
inline Vector woodbury_inverse_apply(const NystromApproximation& approx, double mu, const Vector& b) {
  if (b.size() != approx.dim()) throw std::invalid_argument("woodbury_inverse_apply: shape mismatch");
  Vector x(b.size());
  check_status(npcg_woodbury_inverse_apply(approx.device.get(), mu, 1, b.data(), std::max<Index>(b.size(), 1),
                                           x.data(), std::max<Index>(x.size(), 1), NPCG_HOST));
  return x;
}

/// sketch_and_solve(op, b, mu, ell, rng) (preconditioner.cpp:116-121).
inline Vector sketch_and_solve(const LinearOperator& op, const Vector& b, double mu, Index ell, Rng& rng) {
  if (!(mu > 0.0)) throw std::invalid_argument("sketch_and_solve: mu must be > 0");
  return woodbury_inverse_apply(randomized_nystrom(op, ell, rng), mu, b);
}

}  // namespace npcg
