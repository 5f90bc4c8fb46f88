// reference: nystrom.hpp:19-89 — randomized Nyström approximation. The sketch
// pair and the factored approximation are device-resident (npcg_nys); u and
// lambda are mirrored to the host on construction as in the reference struct.
#pragma once

#include <memory>
#include <vector>

#include "operators.hpp"

namespace npcg {

struct NystromApproximation {  // nystrom.hpp:19-33
  Matrix u;        // n-by-ell, orthonormal columns
  Vector lambda;   // nonincreasing, >= 0
  double shift_used = 0.0;
  std::shared_ptr<npcg_nys> device;  // factored approximation on the B200

  Index dim() const { return u.rows(); }
  Index size() const { return u.cols(); }
  Index rank() const {
    Index r = 0;
    for (Index i = 0; i < lambda.size(); ++i) r += lambda(i) > 0.0;
    return r;
  }
  double lambda_min() const { return lambda.size() == 0 ? 0.0 : lambda(lambda.size() - 1); }
};

/// Cached test matrix and sketch (nystrom.hpp:42-48), on device. A value:
/// extending returns a new pair that shares the device storage copy-on-append
/// (npcg_nys_clone), so the input pair never changes.
struct SketchPair {
  std::shared_ptr<npcg_nys> device;
  Index n = 0;
  Index size() const {
    std::int64_t cols = 0;
    if (device) check_status(npcg_nys_info(device.get(), nullptr, &cols, nullptr, nullptr));
    return cols;
  }
  Index dim() const { return n; }
};

namespace detail {
inline std::shared_ptr<npcg_nys> own(npcg_nys* h) {
  return std::shared_ptr<npcg_nys>(h, [](npcg_nys* p) { npcg_nys_destroy(p); });
}
inline std::shared_ptr<npcg_nys> clone(const std::shared_ptr<npcg_nys>& h, bool factors_only) {
  npcg_nys* c = nullptr;
  check_status(npcg_nys_clone(h.get(), factors_only ? 1 : 0, &c));
  return own(c);
}
inline NystromApproximation fetch(const std::shared_ptr<npcg_nys>& nys) {
  std::int64_t n = 0, size = 0, ell = 0;
  double shift = 0.0;
  check_status(npcg_nys_info(nys.get(), &n, &size, &ell, &shift));
  NystromApproximation a;
  a.u = Matrix(n, ell);
  a.lambda = Vector(ell);
  a.shift_used = shift;
  check_status(npcg_nys_get(nys.get(), a.lambda.data(), ell ? a.u.data() : nullptr, std::max<std::int64_t>(n, 1),
                            NPCG_HOST));
  a.device = clone(nys, true);  // the approximation is a value: later refactors of the pair leave it alone
  return a;
}
}  // namespace detail

/// make_empty_sketch (nystrom.cpp:28-34), bound to its operator on device.
inline SketchPair make_empty_sketch(const LinearOperator& op) {
  npcg_nys* h = nullptr;
  const OpRef ref = device_handle(op);
  check_status(npcg_nys_create(ref, &h));
  return SketchPair{detail::own(h), op.dim()};
}

/// extend_sketch (nystrom.cpp:36-58): draws the n x extra Gaussian from rng in
/// the reference's stream order; Gram-Schmidt, QR and Y = A Omega on device.
inline SketchPair extend_sketch(const SketchPair& pair, const LinearOperator& op, Index extra, Rng& rng) {
  if (pair.dim() != op.dim()) throw std::invalid_argument("extend_sketch: dimension mismatch");
  SketchPair out{detail::clone(pair.device, false), pair.n};
  const OpRef h = device_handle(op);  // the operator of this call (a user operator is bound for the call)
  check_status(npcg_nys_bind(out.device.get(), h));
  h.check(npcg_nys_extend_rng(out.device.get(), extra, rng.handle()));
  return out;
}

/// nystrom_from_sketch (nystrom.cpp:96-140).
inline NystromApproximation nystrom_from_sketch(const SketchPair& pair) {
  check_status(npcg_nys_factor(pair.device.get()));
  return detail::fetch(pair.device);
}

/// randomized_nystrom (nystrom.cpp:142-148).
inline NystromApproximation randomized_nystrom(const LinearOperator& op, Index ell, Rng& rng) {
  if (ell < 1 || ell > op.dim()) throw std::invalid_argument("randomized_nystrom: need 1 <= ell <= dim");
  return nystrom_from_sketch(extend_sketch(make_empty_sketch(op), op, ell, rng));
}

/// extend_sketch_columns (nystrom.cpp:60-94): `extra` unused columns of A
/// drawn from rng; `used` receives every index drawn so far on this sketch.
inline SketchPair extend_sketch_columns(const SketchPair& pair, const LinearOperator& op, Index extra,
                                        std::vector<Index>& used, Rng& rng) {
  if (pair.dim() != op.dim()) throw std::invalid_argument("extend_sketch_columns: dimension mismatch");
  SketchPair out{detail::clone(pair.device, false), pair.n};
  const OpRef h = device_handle(op);
  check_status(npcg_nys_bind(out.device.get(), h));
  h.check(npcg_nys_extend_columns(out.device.get(), extra, rng.handle()));
  int64_t count = 0;
  check_status(npcg_nys_used(out.device.get(), nullptr, &count));
  std::vector<int64_t> idx(static_cast<size_t>(count));
  check_status(npcg_nys_used(out.device.get(), idx.data(), &count));
  used.assign(idx.begin(), idx.end());
  return out;
}

/// column_sampling_nystrom (nystrom.cpp:150-158): ell distinct columns from rng.
inline NystromApproximation column_sampling_nystrom(const LinearOperator& op, Index ell, Rng& rng) {
  npcg_nys* h = nullptr;
  const OpRef ref = device_handle(op);
  ref.check(npcg_column_sampling_nystrom(ref, ell, nullptr, rng.handle(), &h));
  return detail::fetch(detail::own(h));
}

/// column_sampling_nystrom with caller-chosen distinct indices (nystrom.cpp:160-184).
inline NystromApproximation column_sampling_nystrom(const LinearOperator& op, const std::vector<Index>& indices) {
  std::vector<int64_t> idx(indices.begin(), indices.end());
  npcg_nys* h = nullptr;
  const OpRef ref = device_handle(op);
  ref.check(npcg_column_sampling_nystrom(ref, static_cast<int64_t>(idx.size()), idx.data(), nullptr, &h));
  return detail::fetch(detail::own(h));
}

/// An approximation given by its factors (e.g. read from disk) placed on device.
inline NystromApproximation make_approximation(const Matrix& u, const Vector& lambda, double shift_used = 0.0) {
  npcg_nys* h = nullptr;
  check_status(npcg_nys_from_factors(default_context(), u.rows(), lambda.size(), u.data(),
                                     std::max<Index>(u.rows(), 1), lambda.data(), shift_used, NPCG_HOST, &h));
  return detail::fetch(detail::own(h));
}

}  // namespace npcg
