// reference: operators.hpp:25-168 — the LinearOperator NVI and its concrete
// operators. Concrete operators here are device-resident (the matrix / design
// / points live in B200 HBM); matvec()/apply_block() keep the reference's
// contract (dimension + finiteness checks, invalid_argument) and copy the
// host vector in and the result out. The solvers detect a DeviceOperator and
// never leave the device.
#pragma once

#include <cmath>
#include <exception>
#include <string>
#include <memory>
#include <stdexcept>
#include <utility>

#include "random.hpp"
#include "types.hpp"

namespace npcg {

/// The NVI plug-in point (operators.hpp:25-47; operators.cpp:14-63): user
/// subclasses implement do_dim / do_matvec (and optionally do_apply_block,
/// do_column + has_column_access) and are accepted by every solver entry point
/// -- the library calls back into them (OpRef below).
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  Index dim() const { return do_dim(); }
  Vector matvec(const Vector& v) const {  // operators.cpp:25-30
    if (v.size() != dim())
      throw std::invalid_argument("LinearOperator - matvec: dimension mismatch (got " + std::to_string(v.size()) +
                                  ", operator dim " + std::to_string(dim()) + ")");
    if (!all_finite(v.data(), v.size()))
      throw std::invalid_argument("LinearOperator - matvec: input has non-finite entries");
    Vector out(dim());
    do_matvec(v, out);
    return out;
  }
  Matrix apply_block(const Matrix& v) const {  // operators.cpp:32-40
    if (v.rows() != dim()) throw std::invalid_argument("LinearOperator - apply_block: dimension mismatch");
    if (!all_finite(v.data(), v.size()))
      throw std::invalid_argument("LinearOperator - apply_block: input has non-finite entries");
    Matrix out(dim(), v.cols());
    do_apply_block(v, out);
    return out;
  }
  virtual bool has_column_access() const { return false; }
  Vector column(Index j) const {  // operators.cpp:42-50
    if (!has_column_access()) throw std::runtime_error("LinearOperator - column: operator has no column access");
    if (j < 0 || j >= dim()) throw std::invalid_argument("LinearOperator - column: index out of range");
    Vector out(dim());
    do_column(j, out);
    return out;
  }

 protected:
  virtual Index do_dim() const = 0;
  virtual void do_matvec(const Vector& v, Vector& out) const = 0;
  /// Default: one do_matvec per column (operators.cpp:52-58).
  virtual void do_apply_block(const Matrix& v, Matrix& out) const {
    Vector col(v.rows()), col_out(dim());
    for (Index j = 0; j < v.cols(); ++j) {
      std::copy(v.col(j), v.col(j) + v.rows(), col.data());
      do_matvec(col, col_out);
      std::copy(col_out.data(), col_out.data() + col_out.size(), out.col(j));
    }
  }
  virtual void do_column(Index, Vector&) const {
    throw std::runtime_error("LinearOperator - column: operator has no column access");
  }

 private:
  static bool all_finite(const double* p, Index n) {
    for (Index i = 0; i < n; ++i)
      if (!std::isfinite(p[i])) return false;
    return true;
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

/// RegularizedOperator: A_mu = A + mu I, matvec(v) = base.matvec(v) + mu v
/// exactly (operators.hpp:69-94; operators.cpp:82-103). Over a device operator
/// it is a device operator too (npcg_op_regularize), so cg(regularize(op, mu),
/// b) runs the same fused B200 kernels as nystrom_pcg(op, b, mu, ...); over a
/// user operator it is evaluated on the host through the base's NVI.
class RegularizedOperator final : public LinearOperator {
 public:
  RegularizedOperator(std::shared_ptr<const LinearOperator> base, double mu) : owned_(std::move(base)), mu_(mu) {
    if (owned_ == nullptr) throw std::invalid_argument("RegularizedOperator: base operator is null");
    base_ = owned_.get();
    init();
  }
  /// Non-owning view; the base operator must outlive the result.
  RegularizedOperator(const LinearOperator& base, double mu) : base_(&base), mu_(mu) { init(); }
  double mu() const { return mu_; }
  const LinearOperator& base() const { return *base_; }
  bool has_column_access() const override { return false; }
  /// The device handle (null when the base is a host-side user operator).
  npcg_op* handle() const { return dev_.get(); }

 protected:
  Index do_dim() const override { return base_->dim(); }
  void do_matvec(const Vector& v, Vector& out) const override {
    if (dev_) {
      check_status(npcg_op_apply(dev_.get(), v.size(), 1, v.data(), std::max<Index>(v.size(), 1), out.data(),
                                 std::max<Index>(out.size(), 1), NPCG_HOST));
      return;
    }
    out = base_->matvec(v);
    for (Index i = 0; i < out.size(); ++i) out[i] += mu_ * v[i];
  }
  void do_apply_block(const Matrix& v, Matrix& out) const override {
    if (v.cols() == 0) return;
    if (dev_) {
      check_status(npcg_op_apply(dev_.get(), v.rows(), v.cols(), v.data(), std::max<Index>(v.rows(), 1), out.data(),
                                 std::max<Index>(out.rows(), 1), NPCG_HOST));
      return;
    }
    out = base_->apply_block(v);
    for (Index i = 0; i < out.size(); ++i) out.data()[i] += mu_ * v.data()[i];
  }

 private:
  void init();
  std::shared_ptr<const LinearOperator> owned_;
  const LinearOperator* base_ = nullptr;
  double mu_;
  std::shared_ptr<npcg_op> dev_;
};

/// regularize(op, mu) (operators.hpp:153; operators.cpp:201-203).
inline RegularizedOperator regularize(std::shared_ptr<const LinearOperator> op, double mu) {
  return RegularizedOperator(std::move(op), mu);
}

namespace detail {
/// A user LinearOperator bound to the C-ABI for the duration of one library
/// call (npcg_op_callback_create, host buffers): the library calls back into
/// the operator's NVI (matvec for one column, apply_block otherwise), so its
/// dimension / finiteness checks and exceptions are the user's own. An
/// exception thrown by the operator is carried across the C boundary and
/// rethrown by OpRef::rethrow().
struct UserBinding {
  const LinearOperator* op = nullptr;
  std::exception_ptr error;
  static int apply(void* u, std::int64_t n, std::int64_t k, const double* v, std::int64_t ldv, double* out,
                   std::int64_t ldo, void*) {
    auto* b = static_cast<UserBinding*>(u);
    try {
      if (k == 1) {
        Vector x(n);
        std::copy(v, v + n, x.data());
        const Vector y = b->op->matvec(x);
        std::copy(y.data(), y.data() + n, out);
      } else {
        Matrix x(n, k);
        for (std::int64_t j = 0; j < k; ++j) std::copy(v + j * ldv, v + j * ldv + n, x.col(j));
        const Matrix y = b->op->apply_block(x);
        for (std::int64_t j = 0; j < k; ++j) std::copy(y.col(j), y.col(j) + n, out + j * ldo);
      }
      return 0;
    } catch (...) {
      b->error = std::current_exception();
      return 1;
    }
  }
  static int column(void* u, std::int64_t j, double* out, void*) {
    auto* b = static_cast<UserBinding*>(u);
    try {
      const Vector c = b->op->column(j);
      std::copy(c.data(), c.data() + c.size(), out);
      return 0;
    } catch (...) {
      b->error = std::current_exception();
      return 1;
    }
  }
};
}  // namespace detail

/// The device handle an entry point runs on: the operator's own (device /
/// regularized-device operators) or, for any other LinearOperator subclass, a
/// callback operator that lives as long as this object.
class OpRef {
 public:
  explicit OpRef(const LinearOperator& op) {
    if (const auto* d = dynamic_cast<const DeviceOperator*>(&op)) {
      h_ = d->handle();
    } else if (const auto* r = dynamic_cast<const RegularizedOperator*>(&op); r && r->handle()) {
      h_ = r->handle();
    } else {
      bind_ = std::make_unique<detail::UserBinding>();
      bind_->op = &op;
      npcg_op* h = nullptr;
      check_status(npcg_op_callback_create(default_context(), op.dim(), &detail::UserBinding::apply,
                                           op.has_column_access() ? &detail::UserBinding::column : nullptr,
                                           bind_.get(), NPCG_HOST, &h));
      owned_ = std::shared_ptr<npcg_op>(h, [](npcg_op* p) { npcg_op_destroy(p); });
      h_ = h;
    }
  }
  npcg_op* get() const { return h_; }
  operator npcg_op*() const { return h_; }
  /// The user operator's own exception, if a callback threw one.
  void rethrow() const {
    if (bind_ && bind_->error) std::rethrow_exception(bind_->error);
  }
  /// check_status that prefers the user operator's exception.
  void check(int rc) const {
    if (rc != NPCG_OK) rethrow();
    check_status(rc);
  }

 private:
  npcg_op* h_ = nullptr;
  std::unique_ptr<detail::UserBinding> bind_;
  std::shared_ptr<npcg_op> owned_;
};

/// The device handle behind an operator (see OpRef).
inline OpRef device_handle(const LinearOperator& op) { return OpRef(op); }

inline void RegularizedOperator::init() {
  if (!(mu_ >= 0.0)) throw std::invalid_argument("RegularizedOperator: mu must be >= 0");
  const DeviceOperator* d = dynamic_cast<const DeviceOperator*>(base_);
  npcg_op* bh = d ? d->handle() : nullptr;
  if (!bh)
    if (const auto* r = dynamic_cast<const RegularizedOperator*>(base_)) bh = r->handle();
  if (!bh) return;  // host-side user operator: NVI evaluation
  npcg_op* h = nullptr;
  check_status(npcg_op_regularize(bh, mu_, &h));
  // the device view borrows the base handle: keep the base's handle alive with it
  std::shared_ptr<const LinearOperator> keep = owned_;
  dev_ = std::shared_ptr<npcg_op>(h, [keep](npcg_op* p) { npcg_op_destroy(p); });
}

}  // namespace npcg
