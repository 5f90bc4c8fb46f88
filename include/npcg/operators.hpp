// reference: operators.hpp:25-168 — the LinearOperator NVI and its concrete
// operators. Concrete operators here are device-resident (the matrix / design
// / points live in B200 HBM); matvec()/apply_block() keep the reference's
// contract (dimension + finiteness checks, invalid_argument) and copy the
// host vector in and the result out. The solvers detect a DeviceOperator and
// never leave the device.
#pragma once

#include <memory>
#include <stdexcept>
#include <utility>

#include "random.hpp"
#include "types.hpp"

namespace npcg {

class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  Index dim() const { return do_dim(); }
  Vector matvec(const Vector& v) const {  // operators.cpp:25-30
    Vector out(dim());
    do_matvec(v, out);
    return out;
  }
  Matrix apply_block(const Matrix& v) const {  // operators.cpp:32-40
    Matrix out(dim(), v.cols());
    do_apply_block(v, out);
    return out;
  }
  virtual bool has_column_access() const { return false; }
  Vector column(Index j) const {  // operators.cpp:42-50
    Vector out(dim());
    do_column(j, out);
    return out;
  }

 protected:
  virtual Index do_dim() const = 0;
  virtual void do_matvec(const Vector& v, Vector& out) const = 0;
  virtual void do_apply_block(const Matrix& v, Matrix& out) const = 0;
  virtual void do_column(Index, Vector&) const {
    throw std::runtime_error("LinearOperator - column: operator has no column access");
  }
};

/// An operator whose data lives on the B200 (npcg_op handle).
class DeviceOperator : public LinearOperator {
 public:
  explicit DeviceOperator(npcg_op* h) : h_(h, [](npcg_op* p) { npcg_op_destroy(p); }) {}
  npcg_op* handle() const { return h_.get(); }
  bool has_column_access() const override { return npcg_op_has_column_access(h_.get()) != 0; }

 protected:
  Index do_dim() const override {
    std::int64_t n = 0;
    check_status(npcg_op_dim(h_.get(), &n));
    return n;
  }
  void do_matvec(const Vector& v, Vector& out) const override {
    check_status(npcg_op_apply(h_.get(), v.size(), 1, v.data(), std::max<Index>(v.size(), 1), out.data(),
                               std::max<Index>(out.size(), 1), NPCG_HOST));
  }
  void do_apply_block(const Matrix& v, Matrix& out) const override {
    if (v.cols() == 0) return;
    check_status(npcg_op_apply(h_.get(), v.rows(), v.cols(), v.data(), std::max<Index>(v.rows(), 1), out.data(),
                               std::max<Index>(out.rows(), 1), NPCG_HOST));
  }
  void do_column(Index j, Vector& out) const override {
    check_status(npcg_op_column(h_.get(), j, out.data(), NPCG_HOST));
  }

 private:
  std::shared_ptr<npcg_op> h_;
};

/// DenseOperator(Matrix a): rejects nonsquare / asymmetric input (operators.cpp:64-70).
class DenseOperator final : public DeviceOperator {
 public:
  explicit DenseOperator(const Matrix& a) : DeviceOperator(make(a)) {}
  struct FromHandle {};
  DenseOperator(FromHandle, npcg_op* h) : DeviceOperator(h) {}
  /// The stored matrix (materialised from the device).
  Matrix dense() const {
    const Index n = dim();
    return apply_block(Matrix::Identity(n, n));
  }

 private:
  static npcg_op* make(const Matrix& a) {
    npcg_op* h = nullptr;
    check_status(npcg_op_dense_create(default_context(), a.rows(), a.cols(), a.data(),
                                      std::max<Index>(a.rows(), 1), NPCG_HOST, &h));
    return h;
  }
};

/// GramRidgeOperator(Matrix design): v -> (1/n_rows) G^T (G v) (operators.cpp:105-121).
class GramRidgeOperator final : public DeviceOperator {
 public:
  explicit GramRidgeOperator(const Matrix& g) : DeviceOperator(make(g)), rows_(g.rows()) {}
  Index n_rows() const { return rows_; }

 private:
  static npcg_op* make(const Matrix& g) {
    npcg_op* h = nullptr;
    check_status(npcg_op_gram_create(default_context(), g.rows(), g.cols(), g.data(),
                                     std::max<Index>(g.rows(), 1), NPCG_HOST, &h));
    return h;
  }
  Index rows_;
};

namespace detail {
struct HostDesign {
  Matrix design;
};
}  // namespace detail

/// GramRidgeOperator that owns its design (taken by value, as the reference's
/// constructor does) and streams it to the device: the upload overlaps the
/// first product (npcg_op_gram_create_streamed). A non-finite design raises
/// std::invalid_argument from that first product instead of the constructor.
class StreamedGramRidgeOperator final : private detail::HostDesign, public DeviceOperator {
 public:
  explicit StreamedGramRidgeOperator(Matrix g) : detail::HostDesign{std::move(g)}, DeviceOperator(make(design)) {}
  Index n_rows() const { return design.rows(); }

 private:
  static npcg_op* make(const Matrix& g) {
    if (g.rows() < 1 || g.cols() < 1) throw std::invalid_argument("GramRidgeOperator: design matrix must be nonempty");
    npcg_op* h = nullptr;
    check_status(npcg_op_gram_create_streamed(default_context(), g.rows(), g.cols(), g.data(), g.rows(), &h));
    return h;
  }
};

/// KernelOperator(points, sigma, dense_cap) (operators.cpp:141-188).
class KernelOperator final : public DeviceOperator {
 public:
  static constexpr Index kDefaultDenseCap = 20000;
  KernelOperator(const Matrix& points, double sigma, Index dense_cap = kDefaultDenseCap)
      : DeviceOperator(make(points, sigma, dense_cap)), sigma_(sigma) {}
  double sigma() const { return sigma_; }
  bool is_dense() const { return npcg_op_kind(handle()) == 2; }

 private:
  static npcg_op* make(const Matrix& p, double sigma, Index cap) {
    npcg_op* h = nullptr;
    check_status(npcg_op_kernel_create(default_context(), p.rows(), p.cols(), p.data(),
                                       std::max<Index>(p.rows(), 1), sigma, cap, NPCG_HOST, &h));
    return h;
  }
  double sigma_;
};

struct SpectrumProfile {  // operators.hpp:144-150
  Vector eigenvalues;
  explicit SpectrumProfile(Vector lambdas) : eigenvalues(std::move(lambdas)) {}
  Index size() const { return eigenvalues.size(); }
};

/// synthesize_operator (operators.cpp:211-219): Q from the seeded Gaussian,
/// A = Q diag(profile) Q^T symmetrised, built on device.
inline DenseOperator synthesize_operator(const SpectrumProfile& profile, std::uint64_t seed) {
  npcg_op* h = nullptr;
  check_status(npcg_op_synthesize(default_context(), profile.size(), profile.eigenvalues.data(), seed, &h));
  return DenseOperator(DenseOperator::FromHandle{}, h);
}

inline GramRidgeOperator gram_ridge(const Matrix& design) { return GramRidgeOperator(design); }
inline KernelOperator gaussian_kernel(const Matrix& points, double sigma,
                                      Index dense_cap = KernelOperator::kDefaultDenseCap) {
  return KernelOperator(points, sigma, dense_cap);
}

/// The device handle behind an operator (solvers run only on device operators).
inline npcg_op* device_handle(const LinearOperator& op) {
  const auto* d = dynamic_cast<const DeviceOperator*>(&op);
  if (!d) throw std::runtime_error("npcg: operator is not device-resident (use DenseOperator/GramRidgeOperator/KernelOperator)");
  return d->handle();
}

}  // namespace npcg
