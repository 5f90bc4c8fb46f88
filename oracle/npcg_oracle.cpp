// TEST INFRASTRUCTURE ONLY — see npcg_oracle.hpp for scope and who may use it.
// Every function below restates the reference function named in its comment
// (paths relative to /root/reference/proj/core/src/).
#include "npcg_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <numbers>
#include <sstream>

#include "blas_lapack.h"

namespace npcg_oracle {

namespace {
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
bool all_finite(const double* p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}
double norm2(const double* p, size_t n) {  // Eigen norm(): sqrt(squaredNorm())
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += p[i] * p[i];
  return std::sqrt(s);
}
double dot(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
int I(Index v) { return static_cast<int>(v); }
// C = op(A) * op(B) (+ beta C); col-major, tight leading dimensions.
void gemm(bool ta, bool tb, Index m, Index n, Index k, double alpha, const double* a, Index lda,
          const double* b, Index ldb, double beta, double* c, Index ldc) {
  if (m == 0 || n == 0) return;
  if (k == 0) {
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) c[i + j * ldc] = beta == 0.0 ? 0.0 : beta * c[i + j * ldc];
    return;
  }
  cblas_dgemm(kCblasColMajor, ta ? kCblasTrans : kCblasNoTrans, tb ? kCblasTrans : kCblasNoTrans,
              I(m), I(n), I(k), alpha, a, I(std::max<Index>(lda, 1)), b,
              I(std::max<Index>(ldb, 1)), beta, c, I(std::max<Index>(ldc, 1)));
}
void gemv(bool t, Index m, Index n, double alpha, const double* a, Index lda, const double* x,
          double beta, double* y) {
  const Index ylen = t ? n : m;
  if (ylen == 0) return;
  if ((t ? m : n) == 0) {
    for (Index i = 0; i < ylen; ++i) y[i] = beta == 0.0 ? 0.0 : beta * y[i];
    return;
  }
  cblas_dgemv(kCblasColMajor, t ? kCblasTrans : kCblasNoTrans, I(m), I(n), alpha, a,
              I(std::max<Index>(lda, 1)), x, 1, beta, y, 1);
}
}  // namespace

// ============================ random.cpp =====================================
// random.cpp:11-18 — Box-Muller, sine partner discarded, exactly two words.
double Rng::normal() {
  const double u1 = (static_cast<double>(engine()) + 1.0) * 0x1.0p-64;
  const double u2 = static_cast<double>(engine()) * 0x1.0p-64;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}
// random.cpp:20
double Rng::uniform() { return static_cast<double>(engine()) * 0x1.0p-64; }
// random.cpp:22-25 (libstdc++ uniform_int_distribution, as the reference)
std::uint64_t Rng::integer(std::uint64_t bound) {
  if (bound == 0) throw std::invalid_argument("Rng - integer: bound must be positive");
  return std::uniform_int_distribution<std::uint64_t>(0, bound - 1)(engine);
}
// random.cpp:27-32 — column-major fill
Matrix gaussian_matrix(Rng& rng, Index rows, Index cols) {
  Matrix g(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) g(i, j) = rng.normal();
  return g;
}
// random.cpp:34-38
Vector gaussian_vector(Rng& rng, Index n) {
  Vector v(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = rng.normal();
  return v;
}
// random.cpp:40-42
Matrix random_orthogonal(Rng& rng, Index n) {
  return dense::orthonormal_columns(gaussian_matrix(rng, n, n));
}
// random.cpp:44-56
std::vector<Index> sample_without_replacement(Rng& rng, Index n, Index k) {
  if (k < 0 || k > n) throw std::invalid_argument("sample_without_replacement: need 0 <= k <= n");
  std::vector<Index> pool(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) pool[static_cast<size_t>(i)] = i;
  for (Index i = 0; i < k; ++i) {
    const Index j = i + static_cast<Index>(rng.integer(static_cast<std::uint64_t>(n - i)));
    std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
  }
  pool.resize(static_cast<size_t>(k));
  return pool;
}

// ============================ dense.cpp ======================================
namespace dense {
namespace {
void reverse_inplace(Vector& values, Matrix* vectors) {  // dense.cpp:14-20
  std::reverse(values.begin(), values.end());
  if (vectors != nullptr) {
    const Index n = vectors->cols;
    for (Index j = 0; j < n / 2; ++j)
      std::swap_ranges(vectors->col(j), vectors->col(j) + vectors->rows, vectors->col(n - 1 - j));
  }
}
}  // namespace
Eig sym_eig(const Matrix& a) {  // dense.cpp:29-41
  if (a.rows != a.cols) throw std::invalid_argument("sym_eig: matrix must be square");
  Eig out;
  out.vectors = a;
  out.values.assign(static_cast<size_t>(a.rows), 0.0);
  if (a.rows == 0) return out;
  const int info = LAPACKE_dsyevd(kLapackColMajor, 'V', 'L', I(a.rows), out.vectors.data(),
                                  I(a.rows), out.values.data());
  if (info != 0) throw std::runtime_error("sym_eig: dsyevd failed with info = " + std::to_string(info));
  reverse_inplace(out.values, &out.vectors);
  return out;
}
Vector sym_eigenvalues(const Matrix& a) {  // dense.cpp:43-55
  if (a.rows != a.cols) throw std::invalid_argument("sym_eigenvalues: matrix must be square");
  Matrix work = a;
  Vector values(static_cast<size_t>(a.rows));
  if (a.rows == 0) return values;
  const int info =
      LAPACKE_dsyevd(kLapackColMajor, 'N', 'L', I(a.rows), work.data(), I(a.rows), values.data());
  if (info != 0)
    throw std::runtime_error("sym_eigenvalues: dsyevd failed with info = " + std::to_string(info));
  reverse_inplace(values, nullptr);
  return values;
}
ThinSvd thin_svd(const Matrix& b) {  // dense.cpp:81-96
  const Index m = b.rows, n = b.cols;
  if (m < n) throw std::invalid_argument("thin_svd: expected a tall (m >= n) matrix");
  ThinSvd out;
  Matrix work = b;
  out.u = Matrix(m, n);
  out.singular.assign(static_cast<size_t>(n), 0.0);
  if (n == 0) return out;
  Matrix vt(n, n);
  const int info = LAPACKE_dgesdd(kLapackColMajor, 'S', I(m), I(n), work.data(), I(m),
                                  out.singular.data(), out.u.data(), I(m), vt.data(), I(n));
  if (info != 0) throw std::runtime_error("thin_svd: dgesdd failed with info = " + std::to_string(info));
  return out;
}
Matrix orthonormal_columns(const Matrix& g) {  // dense.cpp:98-117
  const Index m = g.rows, n = g.cols;
  if (m < n) throw std::invalid_argument("orthonormal_columns: expected a tall (m >= n) matrix");
  Matrix q = g;
  if (n == 0) return q;
  Vector tau(static_cast<size_t>(std::min(m, n)));
  int info = LAPACKE_dgeqrf(kLapackColMajor, I(m), I(n), q.data(), I(m), tau.data());
  if (info != 0)
    throw std::runtime_error("orthonormal_columns: dgeqrf failed with info = " + std::to_string(info));
  info = LAPACKE_dorgqr(kLapackColMajor, I(m), I(n), I(n), q.data(), I(m), tau.data());
  if (info != 0)
    throw std::runtime_error("orthonormal_columns: dorgqr failed with info = " + std::to_string(info));
  return q;
}
double ulp_spacing(double x) {  // dense.cpp:119-122
  const double ax = std::abs(x);
  return std::nextafter(ax, std::numeric_limits<double>::infinity()) - ax;
}
}  // namespace dense

// ============================ operators.cpp ==================================
namespace {
void check_vector(const LinearOperator& op, const Vector& v, const char* who) {  // operators.cpp:14-21
  if (static_cast<Index>(v.size()) != op.dim())
    throw std::invalid_argument(std::string(who) + ": dimension mismatch (got " +
                                std::to_string(v.size()) + ", operator dim " +
                                std::to_string(op.dim()) + ")");
  if (!all_finite(v.data(), v.size()))
    throw std::invalid_argument(std::string(who) + ": input has non-finite entries");
}
}  // namespace

Vector LinearOperator::matvec(const Vector& v) const {  // operators.cpp:25-30
  check_vector(*this, v, "LinearOperator - matvec");
  Vector out(static_cast<size_t>(dim()));
  do_matvec(v, out);
  return out;
}
Matrix LinearOperator::apply_block(const Matrix& v) const {  // operators.cpp:32-40
  if (v.rows != dim()) throw std::invalid_argument("LinearOperator - apply_block: dimension mismatch");
  if (!all_finite(v.data(), v.size()))
    throw std::invalid_argument("LinearOperator - apply_block: input has non-finite entries");
  Matrix out(dim(), v.cols);
  do_apply_block(v, out);
  return out;
}
Vector LinearOperator::column(Index j) const {  // operators.cpp:42-50
  if (!has_column_access())
    throw std::runtime_error("LinearOperator - column: operator has no column access");
  if (j < 0 || j >= dim()) throw std::invalid_argument("LinearOperator - column: index out of range");
  Vector out(static_cast<size_t>(dim()));
  do_column(j, out);
  return out;
}
void LinearOperator::do_apply_block(const Matrix& v, Matrix& out) const {  // operators.cpp:52-58
  Vector in(static_cast<size_t>(dim())), col_out(static_cast<size_t>(dim()));
  for (Index j = 0; j < v.cols; ++j) {
    std::copy(v.col(j), v.col(j) + v.rows, in.begin());
    do_matvec(in, col_out);
    std::copy(col_out.begin(), col_out.end(), out.col(j));
  }
}
void LinearOperator::do_column(Index, Vector&) const {
  throw std::runtime_error("LinearOperator - column: operator has no column access");
}

DenseOperator::DenseOperator(Matrix a) : a_(std::move(a)) {  // operators.cpp:64-70
  if (a_.rows != a_.cols) throw std::invalid_argument("DenseOperator: matrix must be square");
  double mx = 0.0;
  for (double x : a_.a) mx = std::max(mx, std::abs(x));
  const double scale = std::max(1.0, mx);
  double asym = 0.0;
  for (Index j = 0; j < a_.cols; ++j)
    for (Index i = 0; i < a_.rows; ++i) asym = std::max(asym, std::abs(a_(i, j) - a_(j, i)));
  if (asym > 1e-12 * scale) throw std::invalid_argument("DenseOperator: matrix must be symmetric");
}
void DenseOperator::do_matvec(const Vector& v, Vector& out) const {  // operators.cpp:72-74
  gemv(false, a_.rows, a_.cols, 1.0, a_.data(), a_.rows, v.data(), 0.0, out.data());
}
void DenseOperator::do_apply_block(const Matrix& v, Matrix& out) const {  // operators.cpp:76-78
  gemm(false, false, a_.rows, v.cols, a_.cols, 1.0, a_.data(), a_.rows, v.data(), v.rows, 0.0,
       out.data(), out.rows);
}
void DenseOperator::do_column(Index j, Vector& out) const {  // operators.cpp:80
  std::copy(a_.col(j), a_.col(j) + a_.rows, out.begin());
}

GramRidgeOperator::GramRidgeOperator(Matrix design) : g_(std::move(design)) {  // operators.cpp:105-110
  if (g_.rows < 1 || g_.cols < 1)
    throw std::invalid_argument("GramRidgeOperator: design matrix must be nonempty");
  if (!all_finite(g_.data(), g_.size()))
    throw std::invalid_argument("GramRidgeOperator: design matrix has non-finite entries");
}
void GramRidgeOperator::do_matvec(const Vector& v, Vector& out) const {  // operators.cpp:112-116
  Vector gv(static_cast<size_t>(g_.rows));
  gemv(false, g_.rows, g_.cols, 1.0, g_.data(), g_.rows, v.data(), 0.0, gv.data());
  gemv(true, g_.rows, g_.cols, 1.0, g_.data(), g_.rows, gv.data(), 0.0, out.data());
  const double m = static_cast<double>(g_.rows);
  for (double& o : out) o /= m;
}
void GramRidgeOperator::do_apply_block(const Matrix& v, Matrix& out) const {  // operators.cpp:118-121
  Matrix gv(g_.rows, v.cols);
  gemm(false, false, g_.rows, v.cols, g_.cols, 1.0, g_.data(), g_.rows, v.data(), v.rows, 0.0,
       gv.data(), gv.rows);
  gemm(true, false, g_.cols, v.cols, g_.rows, 1.0, g_.data(), g_.rows, gv.data(), gv.rows, 0.0,
       out.data(), out.rows);
  const double m = static_cast<double>(g_.rows);
  for (double& o : out.a) o /= m;
}

namespace {
// operators.cpp:125-137 — rows [row_begin, row_begin+rows) of the Gaussian kernel.
Matrix kernel_block(const Matrix& points, const Vector& norms, double sigma, Index row_begin,
                    Index rows) {
  const Index n = points.rows, d = points.cols;
  Matrix sq(rows, n);
  // sq = -2 * (block * points^T)
  gemm(false, true, rows, n, d, -2.0, points.data() + row_begin, n, points.data(), n, 0.0,
       sq.data(), rows);
  const double c = -1.0 / (2.0 * sigma * sigma);
  for (Index j = 0; j < n; ++j) {
    double* col = sq.col(j);
    for (Index i = 0; i < rows; ++i) {
      double s = col[i] + norms[static_cast<size_t>(row_begin + i)];  // colwise += norms_i
      s = s + norms[static_cast<size_t>(j)];                          // rowwise += norms_j
      col[i] = std::exp(std::max(s, 0.0) * c);
    }
  }
  for (Index i = 0; i < rows; ++i) sq(i, row_begin + i) = 1.0;
  return sq;
}
Vector row_sq_norms(const Matrix& p) {  // points.rowwise().squaredNorm()
  Vector out(static_cast<size_t>(p.rows), 0.0);
  for (Index i = 0; i < p.rows; ++i) {
    double s = 0.0;
    for (Index c = 0; c < p.cols; ++c) s += p(i, c) * p(i, c);
    out[static_cast<size_t>(i)] = s;
  }
  return out;
}
}  // namespace

KernelOperator::KernelOperator(Matrix points, double sigma, Index dense_cap)  // operators.cpp:141-150
    : points_(std::move(points)), sigma_(sigma) {
  if (points_.rows < 1) throw std::invalid_argument("KernelOperator: need at least one point");
  if (!(sigma_ > 0.0)) throw std::invalid_argument("KernelOperator: sigma must be > 0");
  if (!all_finite(points_.data(), points_.size()))
    throw std::invalid_argument("KernelOperator: points have non-finite entries");
  if (points_.rows <= dense_cap)
    kernel_ = kernel_block(points_, row_sq_norms(points_), sigma_, 0, points_.rows);
}
void KernelOperator::do_matvec(const Vector& v, Vector& out) const {  // operators.cpp:152-164
  if (is_dense()) {
    gemv(false, kernel_.rows, kernel_.cols, 1.0, kernel_.data(), kernel_.rows, v.data(), 0.0, out.data());
    return;
  }
  constexpr Index kBlock = 512;
  const Index n = points_.rows;
  const Vector norms = row_sq_norms(points_);
  for (Index begin = 0; begin < n; begin += kBlock) {
    const Index rows = std::min(kBlock, n - begin);
    const Matrix kb = kernel_block(points_, norms, sigma_, begin, rows);
    gemv(false, rows, n, 1.0, kb.data(), rows, v.data(), 0.0, out.data() + begin);
  }
}
void KernelOperator::do_apply_block(const Matrix& v, Matrix& out) const {  // operators.cpp:166-177
  if (is_dense()) {
    gemm(false, false, kernel_.rows, v.cols, kernel_.cols, 1.0, kernel_.data(), kernel_.rows,
         v.data(), v.rows, 0.0, out.data(), out.rows);
    return;
  }
  constexpr Index kBlock = 512;
  const Index n = points_.rows;
  const Vector norms = row_sq_norms(points_);
  for (Index begin = 0; begin < n; begin += kBlock) {
    const Index rows = std::min(kBlock, n - begin);
    const Matrix kb = kernel_block(points_, norms, sigma_, begin, rows);
    gemm(false, false, rows, v.cols, n, 1.0, kb.data(), rows, v.data(), v.rows, 0.0,
         out.data() + begin, out.rows);
  }
}
void KernelOperator::do_column(Index j, Vector& out) const {  // operators.cpp:179-188
  if (is_dense()) {
    std::copy(kernel_.col(j), kernel_.col(j) + kernel_.rows, out.begin());
    return;
  }
  const double c = -1.0 / (2.0 * sigma_ * sigma_);
  for (Index i = 0; i < points_.rows; ++i) {
    double s = 0.0;
    for (Index k = 0; k < points_.cols; ++k) {
      const double d = points_(i, k) - points_(j, k);
      s += d * d;
    }
    out[static_cast<size_t>(i)] = std::exp(s * c);
  }
  out[static_cast<size_t>(j)] = 1.0;
}

// operators.cpp:211-219
DenseOperator synthesize_operator(const Vector& lam, std::uint64_t seed) {
  const Index n = static_cast<Index>(lam.size());
  if (n < 1) throw std::invalid_argument("SpectrumProfile: need at least one eigenvalue");
  for (Index i = 0; i < n; ++i) {  // SpectrumProfile ctor, operators.cpp:190-199
    const double l = lam[static_cast<size_t>(i)];
    if (!(l >= 0.0) || !std::isfinite(l))
      throw std::invalid_argument("SpectrumProfile: eigenvalues must be finite and >= 0");
    if (i > 0 && l > lam[static_cast<size_t>(i - 1)])
      throw std::invalid_argument("SpectrumProfile: eigenvalues must be nonincreasing");
  }
  Rng rng(seed);
  const Matrix q = random_orthogonal(rng, n);
  Matrix qd = q;  // q * diag(lambda)
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) qd(i, j) *= lam[static_cast<size_t>(j)];
  Matrix a(n, n);
  gemm(false, true, n, n, n, 1.0, qd.data(), n, q.data(), n, 0.0, a.data(), n);
  Matrix s(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) s(i, j) = (a(i, j) + a(j, i)) / 2.0;
  return DenseOperator(std::move(s));
}

// ============================ nystrom.cpp ====================================
SketchPair make_empty_sketch(Index n) {  // nystrom.cpp:28-34
  if (n < 1) throw std::invalid_argument("make_empty_sketch: dimension must be positive");
  SketchPair p;
  p.omega = Matrix(n, 0);
  p.y = Matrix(n, 0);
  return p;
}

SketchPair extend_sketch_with(const SketchPair& pair, const LinearOperator& op, Matrix fresh) {
  // nystrom.cpp:36-58 after the Gaussian draw (the caller drew `fresh`).
  const Index n = op.dim();
  const Index extra = fresh.cols;
  const Index old = pair.size();
  for (int pass = 0; pass < 2 && old > 0; ++pass) {
    Matrix coef(old, extra);  // omega^T fresh
    gemm(true, false, old, extra, n, 1.0, pair.omega.data(), n, fresh.data(), n, 0.0, coef.data(), old);
    gemm(false, false, n, extra, old, -1.0, pair.omega.data(), n, coef.data(), old, 1.0,
         fresh.data(), n);
  }
  const Matrix q_new = dense::orthonormal_columns(fresh);
  SketchPair grown;
  grown.omega = Matrix(n, old + extra);
  grown.y = Matrix(n, old + extra);
  std::copy(pair.omega.a.begin(), pair.omega.a.end(), grown.omega.a.begin());
  std::copy(q_new.a.begin(), q_new.a.end(), grown.omega.a.begin() + old * n);
  std::copy(pair.y.a.begin(), pair.y.a.end(), grown.y.a.begin());
  const Matrix y_new = op.apply_block(q_new);
  std::copy(y_new.a.begin(), y_new.a.end(), grown.y.a.begin() + old * n);
  return grown;
}

SketchPair extend_sketch(const SketchPair& pair, const LinearOperator& op, Index extra, Rng& rng) {
  const Index n = op.dim();  // nystrom.cpp:36-45
  if (pair.omega.rows != n) throw std::invalid_argument("extend_sketch: dimension mismatch");
  if (extra < 1) throw std::invalid_argument("extend_sketch: extra must be >= 1");
  if (pair.size() + extra > n)
    throw std::invalid_argument("extend_sketch: sketch size would exceed dimension");
  return extend_sketch_with(pair, op, gaussian_matrix(rng, n, extra));
}

SketchPair extend_sketch_columns(const SketchPair& pair, const LinearOperator& op, Index extra,
                                 std::vector<Index>& used, Rng& rng) {  // nystrom.cpp:60-94
  const Index n = op.dim();
  if (!op.has_column_access())
    throw std::runtime_error("extend_sketch_columns: operator has no column access");
  if (extra < 1) throw std::invalid_argument("extend_sketch_columns: extra must be >= 1");
  if (static_cast<Index>(used.size()) + extra > n)
    throw std::invalid_argument("extend_sketch_columns: sketch size would exceed dimension");
  std::vector<bool> taken(static_cast<size_t>(n), false);
  for (Index j : used) taken[static_cast<size_t>(j)] = true;
  std::vector<Index> remaining;
  for (Index j = 0; j < n; ++j)
    if (!taken[static_cast<size_t>(j)]) remaining.push_back(j);
  for (Index i = 0; i < extra; ++i) {
    const Index pick =
        i + static_cast<Index>(rng.integer(static_cast<std::uint64_t>(remaining.size() - i)));
    std::swap(remaining[static_cast<size_t>(i)], remaining[static_cast<size_t>(pick)]);
  }
  const Index old = pair.size();
  SketchPair grown;
  grown.omega = Matrix(n, old + extra);
  grown.y = Matrix(n, old + extra);
  std::copy(pair.omega.a.begin(), pair.omega.a.end(), grown.omega.a.begin());
  std::copy(pair.y.a.begin(), pair.y.a.end(), grown.y.a.begin());
  for (Index i = 0; i < extra; ++i) {
    const Index j = remaining[static_cast<size_t>(i)];
    grown.omega(j, old + i) = 1.0;
    const Vector c = op.column(j);
    std::copy(c.begin(), c.end(), grown.y.col(old + i));
    used.push_back(j);
  }
  return grown;
}

NystromApproximation column_sampling_nystrom(const LinearOperator& op, const std::vector<Index>& indices) {
  // nystrom.cpp:160-184: Omega = distinct unit columns, Y = the matching columns of A
  const Index n = op.dim();
  const Index ell = static_cast<Index>(indices.size());
  if (ell < 1 || ell > n) throw std::invalid_argument("column_sampling_nystrom: need 1 <= #indices <= dim");
  if (!op.has_column_access())
    throw std::runtime_error("column_sampling_nystrom: operator has no column access");
  SketchPair pair;
  pair.omega = Matrix(n, ell);
  pair.y = Matrix(n, ell);
  std::vector<bool> seen(static_cast<size_t>(n), false);
  for (Index i = 0; i < ell; ++i) {
    const Index j = indices[static_cast<size_t>(i)];
    if (j < 0 || j >= n) throw std::invalid_argument("column_sampling_nystrom: index out of range");
    if (seen[static_cast<size_t>(j)]) throw std::invalid_argument("column_sampling_nystrom: indices must be distinct");
    seen[static_cast<size_t>(j)] = true;
    pair.omega(j, i) = 1.0;
    const Vector c = op.column(j);
    std::copy(c.begin(), c.end(), pair.y.col(i));
  }
  return nystrom_from_sketch(pair);
}

NystromApproximation column_sampling_nystrom(const LinearOperator& op, Index ell, Rng& rng) {  // nystrom.cpp:150-158
  const Index n = op.dim();
  if (ell < 1 || ell > n) throw std::invalid_argument("column_sampling_nystrom: need 1 <= ell <= dim");
  if (!op.has_column_access())
    throw std::runtime_error("column_sampling_nystrom: operator has no column access");
  return column_sampling_nystrom(op, sample_without_replacement(rng, n, ell));
}

NystromApproximation nystrom_from_sketch(const SketchPair& pair) {  // nystrom.cpp:96-140
  const Index n = pair.omega.rows;
  const Index ell = pair.size();
  NystromApproximation approx;
  if (ell == 0) {
    approx.u = Matrix(n, 0);
    return approx;
  }
  if (!all_finite(pair.y.data(), pair.y.size()))
    throw std::runtime_error("nystrom_from_sketch: sketch has non-finite entries");
  const double ynorm = norm2(pair.y.data(), pair.y.size());
  const double nu0 = dense::ulp_spacing(ynorm);
  double nu = nu0;
  Matrix b;
  bool factored = false;
  for (int attempt = 0; attempt <= 3; ++attempt, nu *= 10.0) {
    Matrix y_nu(n, ell);
    for (size_t i = 0; i < y_nu.size(); ++i) y_nu.a[i] = pair.y.a[i] + nu * pair.omega.a[i];
    Matrix core(ell, ell);
    gemm(true, false, ell, ell, n, 1.0, pair.omega.data(), n, y_nu.data(), n, 0.0, core.data(), ell);
    // Eigen::LLT<Matrix> (lower) reads only the lower triangle: dpotrf('L').
    if (LAPACKE_dpotrf(kLapackColMajor, 'L', I(ell), core.data(), I(ell)) != 0) continue;
    // llt.matrixU().solve<OnTheRight>(y_nu): X L^T = Y_nu.
    cblas_dtrsm(kCblasColMajor, kCblasRight, kCblasLower, kCblasTrans, kCblasNonUnit, I(n), I(ell),
                1.0, core.data(), I(ell), y_nu.data(), I(n));
    if (!all_finite(y_nu.data(), y_nu.size())) continue;
    b = std::move(y_nu);
    approx.shift_used = nu;
    factored = true;
    break;
  }
  if (!factored) {
    std::ostringstream msg;
    msg << "nystrom_from_sketch: Cholesky failed after 3 shift escalations"
        << " (n = " << n << ", ell = " << ell << ", initial shift = " << nu0
        << ", final shift = " << nu / 10.0 << ", ||Y||_F = " << ynorm << ")";
    throw std::runtime_error(msg.str());
  }
  dense::ThinSvd svd = dense::thin_svd(b);
  approx.u = std::move(svd.u);
  approx.lambda.resize(svd.singular.size());
  for (size_t i = 0; i < svd.singular.size(); ++i)
    approx.lambda[i] = std::max(svd.singular[i] * svd.singular[i] - approx.shift_used, 0.0);
  for (size_t i = 1; i < approx.lambda.size(); ++i)
    if (approx.lambda[i] > approx.lambda[i - 1])
      throw std::runtime_error("nystrom_from_sketch: eigenvalue estimates out of order");
  return approx;
}

NystromApproximation randomized_nystrom(const LinearOperator& op, Index ell, Rng& rng) {
  const Index n = op.dim();  // nystrom.cpp:142-148
  if (ell < 1 || ell > n) throw std::invalid_argument("randomized_nystrom: need 1 <= ell <= dim");
  return nystrom_from_sketch(extend_sketch(make_empty_sketch(n), op, ell, rng));
}

// ============================ preconditioner.cpp =============================
Vector NystromPreconditioner::apply(const Vector& v) const {  // preconditioner.cpp:17-25
  if (static_cast<Index>(v.size()) != dim())
    throw std::invalid_argument("NystromPreconditioner - apply: length mismatch");
  if (size() == 0) return v;
  Vector t(static_cast<size_t>(size()));
  gemv(true, u.rows, u.cols, 1.0, u.data(), u.rows, v.data(), 0.0, t.data());
  for (size_t j = 0; j < t.size(); ++j) t[j] *= ((lambda[j] + mu) / (lambda_ell + mu) - 1.0);
  Vector us(v.size());
  gemv(false, u.rows, u.cols, 1.0, u.data(), u.rows, t.data(), 0.0, us.data());
  Vector out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i] + us[i];
  return out;
}
// preconditioner.cpp:104-114: (U diag(lambda) U^T + mu I)^-1 b
Vector woodbury_inverse_apply(const Matrix& u, const Vector& lambda, double mu, const Vector& b) {
  if (!(mu > 0.0)) throw std::invalid_argument("woodbury_inverse_apply: mu must be > 0");
  if (u.rows != static_cast<Index>(b.size()) || u.cols != static_cast<Index>(lambda.size()))
    throw std::invalid_argument("woodbury_inverse_apply: shape mismatch");
  Vector out(b.size());
  if (u.cols == 0) {
    for (size_t i = 0; i < b.size(); ++i) out[i] = b[i] / mu;
    return out;
  }
  Vector t(static_cast<size_t>(u.cols));
  gemv(true, u.rows, u.cols, 1.0, u.data(), u.rows, b.data(), 0.0, t.data());
  Vector core(t.size());
  for (size_t j = 0; j < t.size(); ++j) core[j] = (1.0 / (lambda[j] + mu)) * t[j];
  Vector uc(b.size()), ut(b.size());
  gemv(false, u.rows, u.cols, 1.0, u.data(), u.rows, core.data(), 0.0, uc.data());
  gemv(false, u.rows, u.cols, 1.0, u.data(), u.rows, t.data(), 0.0, ut.data());
  for (size_t i = 0; i < b.size(); ++i) out[i] = uc[i] + (b[i] - ut[i]) / mu;
  return out;
}

Vector NystromPreconditioner::apply_inverse(const Vector& r) const {  // preconditioner.cpp:27-36
  if (static_cast<Index>(r.size()) != dim())
    throw std::invalid_argument("NystromPreconditioner - apply_inverse: length mismatch");
  if (size() == 0) return r;
  Vector t(static_cast<size_t>(size()));
  gemv(true, u.rows, u.cols, 1.0, u.data(), u.rows, r.data(), 0.0, t.data());
  for (size_t j = 0; j < t.size(); ++j) t[j] = ((lambda_ell + mu) / (lambda[j] + mu) - 1.0) * t[j];
  Vector us(r.size());
  gemv(false, u.rows, u.cols, 1.0, u.data(), u.rows, t.data(), 0.0, us.data());
  Vector out(r.size());
  for (size_t i = 0; i < r.size(); ++i) out[i] = r[i] + us[i];
  return out;
}
Matrix NystromPreconditioner::apply_inverse_block(const Matrix& r) const {  // preconditioner.cpp:38-45
  if (r.rows != dim())
    throw std::invalid_argument("NystromPreconditioner - apply_inverse_block: row mismatch");
  if (size() == 0) return r;
  const Index l = size(), s = r.cols, n = r.rows;
  Matrix t(l, s);
  gemm(true, false, l, s, n, 1.0, u.data(), n, r.data(), n, 0.0, t.data(), l);
  for (Index j = 0; j < s; ++j)
    for (Index i = 0; i < l; ++i)
      t(i, j) = ((lambda_ell + mu) / (lambda[static_cast<size_t>(i)] + mu) - 1.0) * t(i, j);
  Matrix us(n, s);
  gemm(false, false, n, s, l, 1.0, u.data(), n, t.data(), l, 0.0, us.data(), n);
  Matrix out(n, s);
  for (size_t i = 0; i < out.size(); ++i) out.a[i] = r.a[i] + us.a[i];
  return out;
}
NystromPreconditioner build_preconditioner(const NystromApproximation& approx, double mu) {
  if (!(mu > 0.0)) throw std::invalid_argument("build_preconditioner: mu must be > 0");  // :80-89
  NystromPreconditioner p;
  p.u = approx.u;
  p.lambda = approx.lambda;
  p.lambda_ell = approx.lambda.empty() ? 0.0 : approx.lambda.back();
  p.mu = mu;
  return p;
}

// ============================ solvers.cpp ====================================
namespace {
void check_solver_inputs(Index n, const Vector& b, const Vector& x0, const SolveOptions& opt,
                         const char* context) {  // solvers.cpp:23-32
  if (static_cast<Index>(b.size()) != n)
    throw std::invalid_argument(std::string(context) + ": right-hand side length mismatch");
  if (static_cast<Index>(x0.size()) != n)
    throw std::invalid_argument(std::string(context) + ": initial guess length mismatch");
  if (!(opt.eta > 0.0)) throw std::invalid_argument(std::string(context) + ": eta must be > 0");
  if (opt.max_iter < 0) throw std::invalid_argument(std::string(context) + ": max_iter must be >= 0");
}

// solvers.cpp:40-107 — the shared (P)CG state machine.
template <class MatvecFn, class PrecondFn>
SolveReport pcg_loop(Index n, MatvecFn&& apply_op, PrecondFn&& apply_precond, const Vector& b,
                     const Vector& x0, const SolveOptions& opt, const char* context) {
  const auto start = Clock::now();
  check_solver_inputs(n, b, x0, opt, context);
  SolveReport report;
  report.eta_used = opt.relative ? opt.eta * norm2(b.data(), b.size()) : opt.eta;
  report.x = x0;
  if (opt.record_iterates) report.iterates.push_back(report.x);
  const size_t N = static_cast<size_t>(n);
  Vector r = apply_op(x0);
  for (size_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
  report.matvec_count = 1;
  double res = norm2(r.data(), N);
  report.residual_history.push_back(res);
  if (!std::isfinite(res)) {
    report.wall_time = seconds_since(start);
    throw SolveDivergenceError(std::string(context) + ": non-finite initial residual", std::move(report));
  }
  if (res <= report.eta_used) {
    report.converged = true;
    report.wall_time = seconds_since(start);
    return report;
  }
  Vector z = apply_precond(r);
  Vector p = z;
  double rz = dot(r.data(), z.data(), N);
  for (Index t = 1; t <= opt.max_iter; ++t) {
    const Vector v = apply_op(p);
    ++report.matvec_count;
    const double pv = dot(p.data(), v.data(), N);
    report.iterations = t;
    if (!(pv > 0.0) || !std::isfinite(pv)) {
      report.wall_time = seconds_since(start);
      std::ostringstream msg;
      msg << context << ": breakdown at iteration " << t << " (p'Ap = " << pv << ")";
      throw SolveDivergenceError(msg.str(), std::move(report));
    }
    const double alpha = rz / pv;
    for (size_t i = 0; i < N; ++i) report.x[i] += alpha * p[i];
    for (size_t i = 0; i < N; ++i) r[i] -= alpha * v[i];
    res = norm2(r.data(), N);
    report.residual_history.push_back(res);
    if (opt.record_iterates) report.iterates.push_back(report.x);
    if (!std::isfinite(res)) {
      report.wall_time = seconds_since(start);
      std::ostringstream msg;
      msg << context << ": non-finite residual at iteration " << t;
      throw SolveDivergenceError(msg.str(), std::move(report));
    }
    if (res <= report.eta_used) {
      report.converged = true;
      break;
    }
    z = apply_precond(r);
    const double rz_next = dot(r.data(), z.data(), N);
    const double beta = rz_next / rz;
    for (size_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_next;
  }
  report.wall_time = seconds_since(start);
  return report;
}
}  // namespace

SolveReport cg(const LinearOperator& op_mu, const Vector& b, const Vector& x0,
               const SolveOptions& opt) {  // solvers.cpp:111-120
  return pcg_loop(
      op_mu.dim(), [&](const Vector& v) { return op_mu.matvec(v); },
      [](const Vector& r) { return r; }, b, x0, opt, "cg");
}

SolveReport nystrom_pcg(const LinearOperator& op, const Vector& b, const Vector& x0, double mu,
                        const NystromPreconditioner& precond, const SolveOptions& opt) {
  if (!(mu >= 0.0)) throw std::invalid_argument("nystrom_pcg: mu must be >= 0");  // :122-148
  if (precond.size() > 0) {
    if (precond.dim() != op.dim())
      throw std::invalid_argument("nystrom_pcg: preconditioner dimension mismatch");
    if (precond.mu != mu)
      throw std::invalid_argument("nystrom_pcg: preconditioner built with a different mu");
  }
  const auto apply_op = [&](const Vector& v) {
    Vector out = op.matvec(v);
    for (size_t i = 0; i < out.size(); ++i) out[i] += mu * v[i];
    return out;
  };
  if (precond.size() == 0)
    return pcg_loop(op.dim(), apply_op, [](const Vector& r) { return r; }, b, x0, opt, "nystrom_pcg");
  return pcg_loop(
      op.dim(), apply_op, [&](const Vector& r) { return precond.apply_inverse(r); }, b, x0, opt,
      "nystrom_pcg");
}

namespace {
// Minimum-norm solve via SVD pseudo-inverse (stands in for Eigen's
// completeOrthogonalDecomposition().pseudoInverse() in the damped fallback).
Matrix pinv_solve(const Matrix& a, const Matrix& rhs) {
  const Index k = a.rows;
  Matrix work = a, u(k, k), vt(k, k);
  Vector s(static_cast<size_t>(k));
  if (LAPACKE_dgesdd(kLapackColMajor, 'A', I(k), I(k), work.data(), I(k), s.data(), u.data(), I(k),
                     vt.data(), I(k)) != 0)
    throw std::runtime_error("block_nystrom_pcg: pseudo-inverse SVD failed");
  const double tol = std::numeric_limits<double>::epsilon() * static_cast<double>(k) * (k ? s[0] : 0.0);
  Matrix utb(k, rhs.cols);
  gemm(true, false, k, rhs.cols, k, 1.0, u.data(), k, rhs.data(), k, 0.0, utb.data(), k);
  for (Index j = 0; j < rhs.cols; ++j)
    for (Index i = 0; i < k; ++i) utb(i, j) = s[static_cast<size_t>(i)] > tol ? utb(i, j) / s[static_cast<size_t>(i)] : 0.0;
  Matrix out(k, rhs.cols);
  gemm(true, false, k, rhs.cols, k, 1.0, vt.data(), k, utb.data(), k, 0.0, out.data(), k);
  return out;
}
bool llt_solve(const Matrix& a, const Matrix& rhs, Matrix& out) {
  Matrix f = a;
  if (LAPACKE_dpotrf(kLapackColMajor, 'L', I(a.rows), f.data(), I(a.rows)) != 0) return false;
  out = rhs;
  LAPACKE_dpotrs(kLapackColMajor, 'L', I(a.rows), I(rhs.cols), f.data(), I(a.rows), out.data(), I(rhs.rows));
  return true;
}
double fro(const Matrix& m) { return norm2(m.data(), m.size()); }
}  // namespace

// solvers.cpp:150-279 — O'Leary block PCG.
BlockSolveReport block_nystrom_pcg(const LinearOperator& op, const Matrix& b, double mu,
                                   const NystromPreconditioner& precond, const SolveOptions& opt) {
  const auto start = Clock::now();
  const Index n = op.dim(), s = b.cols;
  if (b.rows != n) throw std::invalid_argument("block_nystrom_pcg: right-hand side row mismatch");
  if (s < 1) throw std::invalid_argument("block_nystrom_pcg: need at least one column");
  if (!all_finite(b.data(), b.size()))
    throw std::invalid_argument("block_nystrom_pcg: right-hand side has non-finite entries");
  if (!(opt.eta > 0.0)) throw std::invalid_argument("block_nystrom_pcg: eta must be > 0");
  if (!(mu >= 0.0)) throw std::invalid_argument("block_nystrom_pcg: mu must be >= 0");
  if (precond.size() > 0 && precond.dim() != n)
    throw std::invalid_argument("block_nystrom_pcg: preconditioner dimension mismatch");
  BlockSolveReport report;
  report.eta_used = opt.eta;
  Vector threshold(static_cast<size_t>(s));
  for (Index j = 0; j < s; ++j)
    threshold[static_cast<size_t>(j)] = opt.relative ? opt.eta * norm2(b.col(j), static_cast<size_t>(n)) : opt.eta;
  // ColPivHouseholderQR -> dgeqp3.
  Matrix qr = b;
  std::vector<int> jpvt(static_cast<size_t>(s), 0);
  Vector tau(static_cast<size_t>(std::min(n, s)));
  if (LAPACKE_dgeqp3(kLapackColMajor, I(n), I(s), qr.data(), I(n), jpvt.data(), tau.data()) != 0)
    throw std::runtime_error("block_nystrom_pcg: dgeqp3 failed");
  const Index kmin = std::min(n, s);
  Matrix r_upper(kmin, s);
  for (Index j = 0; j < s; ++j)
    for (Index i = 0; i <= std::min(j, kmin - 1); ++i) r_upper(i, j) = qr(i, j);
  const double pivot_max = std::abs(r_upper(0, 0));
  Index rank = 0;
  for (Index i = 0; i < kmin; ++i)
    if (std::abs(r_upper(i, i)) > 1e-12 * pivot_max) ++rank;
  for (Index i = rank; i < s; ++i) report.deflated.push_back(jpvt[static_cast<size_t>(i)] - 1);
  std::sort(report.deflated.begin(), report.deflated.end());
  report.residual_history.assign(static_cast<size_t>(s), {});
  report.converged.assign(static_cast<size_t>(s), false);
  if (rank == 0) {
    report.x = Matrix(n, s);
    for (Index j = 0; j < s; ++j) {
      const double res = norm2(b.col(j), static_cast<size_t>(n));
      report.residual_history[static_cast<size_t>(j)].push_back(res);
      report.converged[static_cast<size_t>(j)] = res <= threshold[static_cast<size_t>(j)];
    }
    report.wall_time = seconds_since(start);
    return report;
  }
  Matrix q_r(n, rank);
  std::copy(qr.a.begin(), qr.a.begin() + n * rank, q_r.a.begin());
  if (LAPACKE_dorgqr(kLapackColMajor, I(n), I(rank), I(rank), q_r.data(), I(n), tau.data()) != 0)
    throw std::runtime_error("block_nystrom_pcg: dorgqr failed");
  Matrix mix(rank, s);  // R[0:rank, :] * P^T
  for (Index k = 0; k < s; ++k)
    for (Index i = 0; i < rank; ++i) mix(i, jpvt[static_cast<size_t>(k)] - 1) = r_upper(i, k);
  Matrix defl_error = b;  // b - q_r * mix
  gemm(false, false, n, s, rank, -1.0, q_r.data(), n, mix.data(), rank, 1.0, defl_error.data(), n);

  const auto apply_op_block = [&](const Matrix& blk) {
    Matrix out = op.apply_block(blk);
    for (size_t i = 0; i < out.size(); ++i) out.a[i] += mu * blk.a[i];
    return out;
  };
  const auto apply_precond_block = [&](const Matrix& blk) {
    return precond.size() == 0 ? blk : precond.apply_inverse_block(blk);
  };
  Matrix x_tilde(n, rank);
  Matrix resid = q_r;
  Matrix z = apply_precond_block(resid);
  Matrix p = z;
  Matrix zr(rank, rank);
  gemm(true, false, rank, rank, n, 1.0, z.data(), n, resid.data(), n, 0.0, zr.data(), rank);
  const auto record_residuals = [&]() -> bool {
    Matrix original = defl_error;  // resid * mix + defl_error
    gemm(false, false, n, s, rank, 1.0, resid.data(), n, mix.data(), rank, 1.0, original.data(), n);
    bool all_done = true;
    for (Index j = 0; j < s; ++j) {
      const double res = norm2(original.col(j), static_cast<size_t>(n));
      if (!std::isfinite(res)) throw std::runtime_error("block_nystrom_pcg: non-finite residual");
      report.residual_history[static_cast<size_t>(j)].push_back(res);
      report.converged[static_cast<size_t>(j)] = res <= threshold[static_cast<size_t>(j)];
      all_done = all_done && report.converged[static_cast<size_t>(j)];
    }
    return all_done;
  };
  bool done = record_residuals();
  for (Index t = 1; t <= opt.max_iter && !done; ++t) {
    report.iterations = t;
    const Matrix v = apply_op_block(p);
    Matrix gram(rank, rank);
    gemm(true, false, rank, rank, n, 1.0, p.data(), n, v.data(), n, 0.0, gram.data(), rank);
    Matrix alpha;
    if (!llt_solve(gram, zr, alpha)) {
      ++report.fallback_count;
      const double damp = 10.0 * dense::ulp_spacing(fro(gram));
      Matrix damped = gram;
      for (Index i = 0; i < rank; ++i) damped(i, i) += damp;
      alpha = pinv_solve(damped, zr);
    }
    gemm(false, false, n, rank, rank, 1.0, p.data(), n, alpha.data(), rank, 1.0, x_tilde.data(), n);
    gemm(false, false, n, rank, rank, -1.0, v.data(), n, alpha.data(), rank, 1.0, resid.data(), n);
    done = record_residuals();
    if (done) break;
    z = apply_precond_block(resid);
    Matrix zr_next(rank, rank);
    gemm(true, false, rank, rank, n, 1.0, z.data(), n, resid.data(), n, 0.0, zr_next.data(), rank);
    Matrix beta;
    if (!llt_solve(zr, zr_next, beta)) {
      ++report.fallback_count;
      const double damp = 10.0 * dense::ulp_spacing(fro(zr));
      Matrix damped = zr;
      for (Index i = 0; i < rank; ++i) damped(i, i) += damp;
      beta = pinv_solve(damped, zr_next);
    }
    Matrix pn = z;  // p = z + p * beta
    gemm(false, false, n, rank, rank, 1.0, p.data(), n, beta.data(), rank, 1.0, pn.data(), n);
    p = std::move(pn);
    zr = std::move(zr_next);
  }
  report.x = Matrix(n, s);
  gemm(false, false, n, s, rank, 1.0, x_tilde.data(), n, mix.data(), rank, 0.0, report.x.data(), n);
  report.wall_time = seconds_since(start);
  return report;
}

Index iteration_bound(double kappa, double epsilon) {  // solvers.cpp:281-291
  if (!(kappa >= 1.0)) throw std::invalid_argument("iteration_bound: kappa must be >= 1");
  if (!(epsilon > 0.0 && epsilon < 1.0))
    throw std::invalid_argument("iteration_bound: epsilon must lie in (0, 1)");
  if (kappa == 1.0) return 1;
  const double root = std::sqrt(kappa);
  const double rate = std::log((root + 1.0) / (root - 1.0));
  const double t = std::ceil(std::log(2.0 / epsilon) / rate);
  return std::max<Index>(1, static_cast<Index>(t));
}

// ============================ adaptive.cpp ===================================
double AdaptiveConfig::resolved_tau() const {  // adaptive.cpp:9-15
  if (tau.has_value()) {
    if (!(*tau > 0.0)) throw std::invalid_argument("AdaptiveConfig: tau must be > 0");
    return *tau;
  }
  return tol_mode == TolMode::ratio ? 10.0 : 30.0;
}

namespace {
void validate_config(const LinearOperator& op, const AdaptiveConfig& c) {  // adaptive.cpp:19-28
  const Index n = op.dim();
  if (c.ell0 < 1 || c.ell0 > c.ell_max || c.ell_max > n)
    throw std::invalid_argument("AdaptiveConfig: need 1 <= ell0 <= ell_max <= dim");
  if (!(c.mu > 0.0)) throw std::invalid_argument("AdaptiveConfig: mu must be > 0");
  if (c.q < 1) throw std::invalid_argument("AdaptiveConfig: q must be >= 1");
  c.resolved_tau();
  if (c.sketch == SketchKind::column_sampling && !op.has_column_access())
    throw std::runtime_error("AdaptiveConfig: column sampling needs column access");
}
SketchPair grow(const SketchPair& pair, const LinearOperator& op, Index extra,
                std::vector<Index>& used, const AdaptiveConfig& c, Rng& rng) {  // :30-35
  if (c.sketch == SketchKind::column_sampling) return extend_sketch_columns(pair, op, extra, used, rng);
  return extend_sketch(pair, op, extra, rng);
}
void finalize(AdaptiveOutcome& o, double mu) {  // :37-42
  o.ell_final = o.approximation.size();
  const double err = o.error_estimate ? std::max(0.0, *o.error_estimate) : 0.0;
  o.posterior_condition_estimate = posterior_condition_estimate(o.approximation.lambda_min(), mu, err);
}
template <class StopFn>
AdaptiveOutcome doubling_loop(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng,
                              StopFn&& should_stop) {  // adaptive.cpp:50-79
  validate_config(op, c);
  AdaptiveOutcome outcome;
  std::vector<Index> used;
  SketchPair pair = grow(make_empty_sketch(op.dim()), op, c.ell0, used, c, rng);
  outcome.approximation = nystrom_from_sketch(pair);
  while (true) {
    if (should_stop(outcome)) break;
    const Index ell = pair.size();
    if (ell >= c.ell_max) {
      outcome.hit_cap = true;
      break;
    }
    const Index extra = 2 * ell <= c.ell_max ? ell : c.ell_max - ell;
    pair = grow(pair, op, extra, used, c, rng);
    ++outcome.doublings;
    outcome.approximation = nystrom_from_sketch(pair);
    if (pair.size() == c.ell_max && 2 * ell > c.ell_max) {
      outcome.hit_cap = true;
      break;
    }
  }
  finalize(outcome, c.mu);
  return outcome;
}
}  // namespace

double estimate_error_power(const LinearOperator& op, const Matrix& u, const Vector& lambda,
                            Index q, Rng& rng) {  // adaptive.cpp:83-109
  const Index n = op.dim();
  if (q < 1) throw std::invalid_argument("estimate_error_power: q must be >= 1");
  if (u.cols != static_cast<Index>(lambda.size()) || (u.cols > 0 && u.rows != n))
    throw std::invalid_argument("estimate_error_power: factor shape mismatch");
  Vector v = gaussian_vector(rng, n);
  const double v0 = norm2(v.data(), v.size());
  if (v0 == 0.0) return 0.0;
  for (double& x : v) x /= v0;
  double estimate = 0.0;
  Vector t(static_cast<size_t>(u.cols)), corr(static_cast<size_t>(n));
  for (Index i = 0; i < q; ++i) {
    Vector w = op.matvec(v);
    if (u.cols > 0) {
      gemv(true, n, u.cols, 1.0, u.data(), n, v.data(), 0.0, t.data());
      for (size_t j = 0; j < t.size(); ++j) t[j] = lambda[j] * t[j];
      gemv(false, n, u.cols, 1.0, u.data(), n, t.data(), 0.0, corr.data());
      for (size_t k = 0; k < w.size(); ++k) w[k] -= corr[k];
    }
    estimate = dot(v.data(), w.data(), v.size());
    const double nrm = norm2(w.data(), w.size());
    if (nrm == 0.0) return 0.0;
    for (size_t k = 0; k < w.size(); ++k) v[k] = w[k] / nrm;
  }
  return estimate;
}

AdaptiveOutcome adaptive_nystrom(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::error)  // adaptive.cpp:111-123
    throw std::invalid_argument("adaptive_nystrom: config.tol_mode must be error");
  const double tol = c.resolved_tau() * c.mu;
  return doubling_loop(op, c, rng, [&](AdaptiveOutcome& o) {
    const double est = estimate_error_power(op, o.approximation.u, o.approximation.lambda, c.q, rng);
    o.error_estimate = est;
    if (est > tol) return false;
    return !c.secondary_criterion || o.approximation.lambda_min() <= tol / 11.0;
  });
}
AdaptiveOutcome adaptive_nystrom_ratio(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::ratio)  // adaptive.cpp:125-133
    throw std::invalid_argument("adaptive_nystrom_ratio: config.tol_mode must be ratio");
  const double tau = c.resolved_tau();
  return doubling_loop(op, c, rng, [&](AdaptiveOutcome& o) {
    return o.approximation.lambda_min() <= tau * c.mu;
  });
}
AdaptiveOutcome fixed_rank_nystrom(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::fixed)  // adaptive.cpp:135-148
    throw std::invalid_argument("fixed_rank_nystrom: config.tol_mode must be fixed");
  validate_config(op, c);
  AdaptiveOutcome o;
  std::vector<Index> used;
  const SketchPair pair = grow(make_empty_sketch(op.dim()), op, c.ell_max, used, c, rng);
  o.approximation = nystrom_from_sketch(pair);
  o.error_estimate = estimate_error_power(op, o.approximation.u, o.approximation.lambda, c.q, rng);
  finalize(o, c.mu);
  return o;
}
double posterior_condition_estimate(double lambda_ell, double mu, double err) {  // :150-156
  if (!(mu > 0.0)) throw std::invalid_argument("posterior_condition_estimate: mu must be > 0");
  if (lambda_ell < 0.0 || err < 0.0)
    throw std::invalid_argument("posterior_condition_estimate: inputs must be >= 0");
  return (lambda_ell + mu + err) / mu;
}

std::uint64_t synthetic_operator_seed(std::uint64_t seed) {  // bench.cpp:180-185
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

}  // namespace npcg_oracle
