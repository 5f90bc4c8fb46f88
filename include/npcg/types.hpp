// C++ facade of the B200 Nyström-PCG library: the reference's npcg:: API
// (/root/reference/proj/core/include/npcg/*.hpp) over the C-ABI in
// include/npcg_capi.h. Eigen is not required: Matrix/Vector are minimal
// column-major containers with Eigen::MatrixXd's memory layout, so an Eigen
// user can Eigen::Map them zero-copy (types.hpp:7-9 of the reference).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <vector>

#include "../npcg_capi.h"

namespace npcg {

using Index = std::ptrdiff_t;

/// Column-major dense matrix, ld == rows (Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * r_)]; }
  double* col(Index j) { return a_.data() + j * r_; }
  const double* col(Index j) const { return a_.data() + j * r_; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};

/// Dense vector (Eigen::VectorXd layout).
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : a_(static_cast<size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> v) : a_(v) {}
  static Vector Zero(Index n) { return Vector(n); }
  Index size() const { return static_cast<Index>(a_.size()); }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(Index i) { return a_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return a_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return a_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return a_[static_cast<size_t>(i)]; }

 private:
  std::vector<double> a_;
};

/// Maps C-ABI status codes to the reference's exception types
/// (invalid_argument / runtime_error; SolveDivergenceError in solvers.hpp).
inline void check_status(int rc) {
  if (rc == NPCG_OK) return;
  const std::string msg = npcg_last_error();
  if (rc == NPCG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

/// The process-wide device context (one B200; NPCG_DEVICE env selects it).
inline npcg_ctx* default_context() {
  static npcg_ctx* ctx = [] {
    npcg_ctx* c = nullptr;
    const char* dev = std::getenv("NPCG_DEVICE");
    check_status(npcg_ctx_create(dev ? std::atoi(dev) : 0, &c));
    return c;
  }();
  return ctx;
}

}  // namespace npcg
