// =============================================================================
// npcg ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's Nyström-PCG hot path
// (/root/reference/proj/core/src/{random,dense,operators,nystrom,
//  preconditioner,solvers,adaptive,bench}.cpp), written from the reference's
// behaviour, line by line, over plain col-major storage + LAPACK/CBLAS from the
// OpenBLAS that ships in this image (the reference needs Eigen3 + LAPACKE,
// neither of which exists here, so the reference itself cannot be compiled —
// see DESIGN.md §Oracle).
//
// Who may use this: tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs — as the CHECKER or the CPU baseline,
// never as the product. The product (paper_2110_02820_b200/, libnpcg_b200.so)
// never links or loads anything under oracle/.
//
// Parity pins: the oracle is checked (tests/test_oracle_kat.py) against every
// known-answer test and property the reference's own suites hold for this path
// (SURVEY.md §8c), plus the C++-standard mt19937_64 known answer. The
// reference has no golden data files; there is no runnable reference build to
// generate more (parity pinned by KATs/properties, not by reference outputs).
// =============================================================================
#pragma once

#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace npcg_oracle {

using Index = std::int64_t;

/// Column-major dense matrix (Eigen::MatrixXd layout: ld == rows).
struct Matrix {
  Index rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return a[static_cast<size_t>(i + j * rows)]; }
  double operator()(Index i, Index j) const { return a[static_cast<size_t>(i + j * rows)]; }
  double* col(Index j) { return a.data() + j * rows; }
  const double* col(Index j) const { return a.data() + j * rows; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
  size_t size() const { return a.size(); }
};
using Vector = std::vector<double>;

// ---- random.cpp -------------------------------------------------------------
/// reference: random.hpp:21-38, random.cpp:11-25
struct Rng {
  explicit Rng(std::uint64_t seed) : engine(seed) {}
  double normal();
  double uniform();
  std::uint64_t integer(std::uint64_t bound);
  std::mt19937_64 engine;
};
Matrix gaussian_matrix(Rng& rng, Index rows, Index cols);        // random.cpp:27-32
Vector gaussian_vector(Rng& rng, Index n);                       // random.cpp:34-38
Matrix random_orthogonal(Rng& rng, Index n);                     // random.cpp:40-42
std::vector<Index> sample_without_replacement(Rng&, Index n, Index k);  // random.cpp:44-56

// ---- dense.cpp --------------------------------------------------------------
namespace dense {
struct Eig { Vector values; Matrix vectors; };
struct ThinSvd { Matrix u; Vector singular; };
Eig sym_eig(const Matrix& a);                 // dense.cpp:29-41
Vector sym_eigenvalues(const Matrix& a);      // dense.cpp:43-55
ThinSvd thin_svd(const Matrix& b);            // dense.cpp:81-96
Matrix orthonormal_columns(const Matrix& g);  // dense.cpp:98-117
double ulp_spacing(double x);                 // dense.cpp:119-122
}  // namespace dense

// ---- operators.cpp ----------------------------------------------------------
/// NVI contract of operators.hpp:25-47 / operators.cpp:14-50.
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  Index dim() const { return do_dim(); }
  Vector matvec(const Vector& v) const;
  Matrix apply_block(const Matrix& v) const;
  virtual bool has_column_access() const { return false; }
  Vector column(Index j) const;

 protected:
  virtual Index do_dim() const = 0;
  virtual void do_matvec(const Vector& v, Vector& out) const = 0;
  virtual void do_apply_block(const Matrix& v, Matrix& out) const;
  virtual void do_column(Index j, Vector& out) const;
};

class DenseOperator final : public LinearOperator {   // operators.cpp:64-80
 public:
  explicit DenseOperator(Matrix a);
  bool has_column_access() const override { return true; }
  const Matrix& dense() const { return a_; }
 protected:
  Index do_dim() const override { return a_.rows; }
  void do_matvec(const Vector& v, Vector& out) const override;
  void do_apply_block(const Matrix& v, Matrix& out) const override;
  void do_column(Index j, Vector& out) const override;
 private:
  Matrix a_;
};

class GramRidgeOperator final : public LinearOperator {  // operators.cpp:105-121
 public:
  explicit GramRidgeOperator(Matrix design);
  Index n_rows() const { return g_.rows; }
 protected:
  Index do_dim() const override { return g_.cols; }
  void do_matvec(const Vector& v, Vector& out) const override;
  void do_apply_block(const Matrix& v, Matrix& out) const override;
 private:
  Matrix g_;
};

class KernelOperator final : public LinearOperator {  // operators.cpp:125-188
 public:
  static constexpr Index kDefaultDenseCap = 20000;
  KernelOperator(Matrix points, double sigma, Index dense_cap = kDefaultDenseCap);
  bool has_column_access() const override { return true; }
  bool is_dense() const { return kernel_.size() > 0; }
  const Matrix& kernel() const { return kernel_; }
 protected:
  Index do_dim() const override { return points_.rows; }
  void do_matvec(const Vector& v, Vector& out) const override;
  void do_apply_block(const Matrix& v, Matrix& out) const override;
  void do_column(Index j, Vector& out) const override;
 private:
  Matrix points_;
  double sigma_;
  Matrix kernel_;
};

/// operators.cpp:211-219
DenseOperator synthesize_operator(const Vector& eigenvalues, std::uint64_t seed);

// ---- nystrom.cpp ------------------------------------------------------------
struct NystromApproximation {  // nystrom.hpp:19-33
  Matrix u;
  Vector lambda;
  double shift_used = 0.0;
  Index size() const { return u.cols; }
  double lambda_min() const { return lambda.empty() ? 0.0 : lambda.back(); }
};
struct SketchPair { Matrix omega, y; Index size() const { return omega.cols; } };
SketchPair make_empty_sketch(Index n);                                          // nystrom.cpp:28-34
SketchPair extend_sketch(const SketchPair&, const LinearOperator&, Index extra, Rng&);  // :36-58
/// Same as extend_sketch but with the raw Gaussian block supplied by the caller
/// (the exact matrix `gaussian_matrix(rng, n, extra)` would return).
SketchPair extend_sketch_with(const SketchPair&, const LinearOperator&, Matrix fresh);
SketchPair extend_sketch_columns(const SketchPair&, const LinearOperator&, Index extra,
                                 std::vector<Index>& used, Rng&);               // :60-94
NystromApproximation nystrom_from_sketch(const SketchPair&);                    // :96-140
NystromApproximation column_sampling_nystrom(const LinearOperator&, const std::vector<Index>&);  // :160-184
NystromApproximation column_sampling_nystrom(const LinearOperator&, Index ell, Rng&);          // :150-158
NystromApproximation randomized_nystrom(const LinearOperator&, Index ell, Rng&);  // :142-148

// ---- preconditioner.cpp -----------------------------------------------------
struct NystromPreconditioner {  // preconditioner.hpp:20-37
  Matrix u;
  Vector lambda;
  double lambda_ell = 0.0;
  double mu = 0.0;
  Index dim() const { return u.rows; }
  Index size() const { return u.cols; }
  Vector apply(const Vector& v) const;           // preconditioner.cpp:17-25
  Vector apply_inverse(const Vector& r) const;   // :27-36
  Matrix apply_inverse_block(const Matrix& r) const;  // :38-45
};
NystromPreconditioner build_preconditioner(const NystromApproximation&, double mu);  // :80-89
Vector woodbury_inverse_apply(const Matrix& u, const Vector& lambda, double mu, const Vector& b);  // :104-114

// ---- solvers.cpp ------------------------------------------------------------
struct SolveOptions { double eta = 1e-10; Index max_iter = 500; bool relative = false; bool record_iterates = false; };
struct SolveReport {
  Vector x;
  Index iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  Index matvec_count = 0;
  double wall_time = 0.0;
  double eta_used = 0.0;
  std::vector<Vector> iterates;
};
struct BlockSolveReport {
  Matrix x;
  Index iterations = 0;
  std::vector<std::vector<double>> residual_history;
  std::vector<bool> converged;
  std::vector<Index> deflated;
  Index fallback_count = 0;
  double wall_time = 0.0;
  double eta_used = 0.0;
};
class SolveDivergenceError : public std::runtime_error {
 public:
  SolveDivergenceError(const std::string& w, SolveReport r) : std::runtime_error(w), report(std::move(r)) {}
  SolveReport report;
};
SolveReport cg(const LinearOperator& op_mu, const Vector& b, const Vector& x0, const SolveOptions&);
SolveReport nystrom_pcg(const LinearOperator& op, const Vector& b, const Vector& x0, double mu,
                        const NystromPreconditioner& p, const SolveOptions& opt);
BlockSolveReport block_nystrom_pcg(const LinearOperator& op, const Matrix& b, double mu,
                                   const NystromPreconditioner& p, const SolveOptions& opt);
Index iteration_bound(double kappa, double epsilon);

// ---- adaptive.cpp -----------------------------------------------------------
enum class TolMode { error = 0, ratio = 1, fixed = 2 };
enum class SketchKind { gaussian = 0, column_sampling = 1 };
struct AdaptiveConfig {
  Index ell0 = 10, ell_max = 0;
  double mu = 0.0;
  TolMode tol_mode = TolMode::error;
  std::optional<double> tau;
  Index q = 5;
  bool secondary_criterion = true;
  SketchKind sketch = SketchKind::gaussian;
  double resolved_tau() const;
};
struct AdaptiveOutcome {
  NystromApproximation approximation;
  std::optional<double> error_estimate;
  Index doublings = 0;
  bool hit_cap = false;
  double posterior_condition_estimate = 0.0;
  Index ell_final = 0;
};
double estimate_error_power(const LinearOperator&, const Matrix& u, const Vector& lambda, Index q, Rng&);
AdaptiveOutcome adaptive_nystrom(const LinearOperator&, const AdaptiveConfig&, Rng&);
AdaptiveOutcome adaptive_nystrom_ratio(const LinearOperator&, const AdaptiveConfig&, Rng&);
AdaptiveOutcome fixed_rank_nystrom(const LinearOperator&, const AdaptiveConfig&, Rng&);
double posterior_condition_estimate(double lambda_ell, double mu, double err);

// ---- bench.cpp ---------------------------------------------------------------
std::uint64_t synthetic_operator_seed(std::uint64_t seed);  // bench.cpp:180-185

}  // namespace npcg_oracle
