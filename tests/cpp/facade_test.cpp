// Drop-in check of the C++ facade (include/npcg/*.hpp): reference-style calls
// (names, signatures, exception types of /root/reference/proj/core) running
// on the B200 through libnpcg_b200.so. Mirrors cases of the reference's
// operators/preconditioner/solvers/nystrom tests. Exit code 0 = all passed.
#include <cmath>
#include <cstdio>
#include <memory>
#include <stdexcept>

#include "npcg/npcg.hpp"

using namespace npcg;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

// A user-defined operator: the reference's plug-in point (operators.hpp:25-47).
// 1-D Laplacian-like tridiagonal SPD matrix, diag 2 + i/n, off-diagonals -1;
// only do_dim / do_matvec are implemented (do_apply_block is the NVI default).
class TridiagOperator final : public LinearOperator {
 public:
  explicit TridiagOperator(Index n) : n_(n) {}
  mutable Index calls = 0;
  static double diag(Index i, Index n) { return 2.0 + static_cast<double>(i) / static_cast<double>(n); }

 protected:
  Index do_dim() const override { return n_; }
  void do_matvec(const Vector& v, Vector& out) const override {
    ++calls;
    for (Index i = 0; i < n_; ++i) {
      double s = diag(i, n_) * v(i);
      if (i > 0) s -= v(i - 1);
      if (i + 1 < n_) s -= v(i + 1);
      out(i) = s;
    }
  }

 private:
  Index n_;
};

class ThrowingOperator final : public LinearOperator {
 protected:
  Index do_dim() const override { return 4; }
  void do_matvec(const Vector&, Vector&) const override { throw std::domain_error("user operator failed"); }
};

static void dump(FILE* f, const char* name, Index iters, const Vector& x) {
  if (!f) return;
  std::fprintf(f, "%s %td", name, iters);
  for (Index i = 0; i < x.size(); ++i) std::fprintf(f, " %.17g", x(i));
  std::fprintf(f, "\n");
}

int main(int argc, char** argv) {
  FILE* out = argc > 1 ? std::fopen(argv[1], "w") : nullptr;
  // operators_test.cpp:55-62 — dense matvec on a 2x2 example
  Matrix a(2, 2);
  a(0, 0) = 2; a(0, 1) = 1; a(1, 0) = 1; a(1, 1) = 2;
  const DenseOperator op(a);
  const Vector y = op.matvec(Vector{1.0, 0.0});
  CHECK(y(0) == 2.0 && y(1) == 1.0);
  CHECK(op.has_column_access());
  const Vector c1 = op.column(1);
  CHECK(c1(0) == 1.0 && c1(1) == 2.0);
  // operators_test.cpp:64-70 — dimension / finiteness contract
  bool threw = false;
  try { op.matvec(Vector{1.0, 2.0, 3.0}); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  // preconditioner_test.cpp:80-86 — U = [e1 e2], Lambda = (4, 2), mu = 1: (5,3,7) -> (3,3,7)
  Matrix u(3, 2);
  u(0, 0) = 1; u(1, 1) = 1;
  const NystromApproximation basis = make_approximation(u, Vector{4.0, 2.0}, 1e-16);
  const NystromPreconditioner p = build_preconditioner(basis, 1.0);
  const Vector z = p.apply_inverse(Vector{5.0, 3.0, 7.0});
  CHECK(std::abs(z(0) - 3.0) < 1e-14 && std::abs(z(1) - 3.0) < 1e-14 && std::abs(z(2) - 7.0) < 1e-14);
  threw = false;
  try { build_preconditioner(basis, 0.0); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  // nystrom_test.cpp:12-20 — zero matrix gives exactly zero eigenvalues
  {
    const DenseOperator zero(Matrix::Zero(10, 10));
    Rng rng(1);
    const NystromApproximation ap = randomized_nystrom(zero, 3, rng);
    CHECK(ap.lambda.size() == 3);
    for (Index i = 0; i < 3; ++i) CHECK(ap.lambda(i) == 0.0);
  }
  // nystrom_test.cpp:84-103 — column sampling on diag(5, 0, 0) reconstructs exactly
  {
    Matrix d = Matrix::Zero(3, 3);
    d(0, 0) = 5.0;
    const DenseOperator dop(d);
    const NystromApproximation ap = column_sampling_nystrom(dop, std::vector<Index>{0});
    CHECK(ap.lambda.size() == 1 && std::abs(ap.lambda(0) - 5.0) < 1e-12);
    threw = false;
    try { column_sampling_nystrom(dop, std::vector<Index>{1, 1}); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
  }
  // solvers_test.cpp:112-127 — known solution through Nyström PCG
  {
    const Index n = 60;
    Vector lam(n);
    for (Index j = 0; j < n; ++j) lam(j) = std::pow(j + 1.0, -2.0);
    const DenseOperator A = synthesize_operator(SpectrumProfile(lam), 5);
    Rng rng(5);
    const Vector star = gaussian_vector(rng, n);
    const double mu = 0.01;
    Vector b = A.matvec(star);
    for (Index i = 0; i < n; ++i) b(i) += mu * star(i);
    const NystromApproximation ap = randomized_nystrom(A, 10, rng);
    const NystromPreconditioner pre = build_preconditioner(ap, mu);
    SolveOptions opt;
    opt.relative = true;
    const SolveReport rep = nystrom_pcg(A, b, mu, pre, opt);
    double err = 0.0, nrm = 0.0;
    for (Index i = 0; i < n; ++i) {
      err += (rep.x(i) - star(i)) * (rep.x(i) - star(i));
      nrm += star(i) * star(i);
    }
    CHECK(rep.converged);
    CHECK(std::sqrt(err / nrm) < 1e-8);
    CHECK(rep.matvec_count == rep.iterations + 1);
    threw = false;
    try { nystrom_pcg(A, b, 0.2, pre, opt); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // adaptive_test.cpp:220-226
    CHECK(posterior_condition_estimate(1.0, 1.0, 2.0) == 4.0);
    AdaptiveConfig cfg;
    cfg.ell0 = 4;
    cfg.ell_max = 32;
    cfg.mu = mu;
    cfg.tau = 10.0;
    Rng r2(7);
    const AdaptiveOutcome out = adaptive_nystrom(A, cfg, r2);
    CHECK(out.ell_final >= 4 && out.ell_final <= 32);
    CHECK(out.error_estimate.has_value());
  }
  // regularisation path: cold starts batch the mu over each pass of A;
  // every column must reproduce its own nystrom_pcg call
  {
    const Index n = 1500;
    Vector lam(n);
    for (Index j = 0; j < n; ++j) lam(j) = std::pow(j + 1.0, -1.5);
    const DenseOperator A = synthesize_operator(SpectrumProfile(lam), 11);
    Rng rng(11);
    const Matrix B = gaussian_matrix(rng, n, 4);
    const NystromApproximation ap = randomized_nystrom(A, 40, rng);
    const std::vector<double> mus{1e-4, 1e-3, 1e-2};
    SolveOptions opt;
    opt.relative = true;
    const auto path = regularization_path(A, B, mus, ap, /*warm_start=*/false, opt);
    CHECK(path.size() == 3 && path[0].size() == 4);
    for (size_t k = 0; k < mus.size(); ++k) {
      const NystromPreconditioner pre = build_preconditioner(ap, mus[k]);
      for (Index j = 0; j < 4; ++j) {
        Vector bj(n);
        for (Index i = 0; i < n; ++i) bj(i) = B(i, j);
        const SolveReport one = nystrom_pcg(A, bj, mus[k], pre, opt);
        const SolveReport& got = path[k][static_cast<size_t>(j)];
        CHECK(got.converged && one.converged);
        CHECK(std::abs(static_cast<long>(got.iterations) - static_cast<long>(one.iterations)) <= 1);
        double err = 0.0, nrm = 0.0;
        for (Index i = 0; i < n; ++i) {
          err += (got.x(i) - one.x(i)) * (got.x(i) - one.x(i));
          nrm += one.x(i) * one.x(i);
        }
        CHECK(std::sqrt(err / nrm) < 1e-8);
      }
    }
  }
  // solvers_test.cpp:76-90 — breakdown raises SolveDivergenceError with its report
  {
    Matrix ind = Matrix::Identity(2, 2);
    ind(1, 1) = -1.0;
    const DenseOperator bad(ind);
    threw = false;
    try {
      cg(bad, 0.0, Vector{1.0, 1.0});
    } catch (const SolveDivergenceError& e) {
      threw = e.report.iterations == 1 && !e.report.converged;
    }
    CHECK(threw);
  }
  // streamed Gram upload: same products as the synchronous constructor
  {
    Matrix g(300, 20);
    for (Index j = 0; j < 20; ++j)
      for (Index i = 0; i < 300; ++i) g(i, j) = std::sin(0.37 * i + 1.3 * j) / (1.0 + j);
    const GramRidgeOperator sync(g);
    const StreamedGramRidgeOperator streamed(g);
    CHECK(streamed.n_rows() == 300 && streamed.dim() == 20);
    Vector v(20);
    for (Index j = 0; j < 20; ++j) v(j) = 1.0 / (1.0 + j);
    const Vector a = sync.matvec(v), b = streamed.matvec(v);
    double d = 0.0;
    for (Index j = 0; j < 20; ++j) d = std::max(d, std::abs(a(j) - b(j)));
    CHECK(d < 1e-14);
    Matrix bad = g;
    bad(7, 3) = std::nan("");
    threw = false;
    try {
      const StreamedGramRidgeOperator s2(bad);
      (void)s2.matvec(v);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  CHECK(iteration_bound(56.0, 1e-6) == 54);
  // The plug-in point: a user LinearOperator subclass through every solver
  // entry point, and cg(regularize(op, mu), b) -- the reference bench's call
  // (bench.cpp:218-220). The pytest side compares these against the oracle.
  {
    const Index n = 200;
    auto user = std::make_shared<TridiagOperator>(n);
    Vector b(n);
    for (Index i = 0; i < n; ++i) b(i) = std::cos(0.1 * i);
    const double mu = 0.05;
    SolveOptions opt;
    opt.relative = true;
    const RegularizedOperator reg = regularize(user, mu);
    CHECK(reg.handle() == nullptr);  // host-side user operator
    const SolveReport r1 = cg(reg, b, opt);
    CHECK(r1.converged && r1.matvec_count == r1.iterations + 1);
    CHECK(user->calls >= r1.iterations);
    dump(out, "user_cg_regularized", r1.iterations, r1.x);
    Rng rng(11);
    const NystromApproximation ap = randomized_nystrom(*user, 20, rng);
    CHECK(ap.lambda.size() == 20);
    const NystromPreconditioner pre = build_preconditioner(ap, mu);
    const SolveReport r2 = nystrom_pcg(*user, b, mu, pre, opt);
    CHECK(r2.converged);
    dump(out, "user_nystrom_pcg", r2.iterations, r2.x);
    Vector lam_dump(ap.lambda.size());
    for (Index i = 0; i < ap.lambda.size(); ++i) lam_dump(i) = ap.lambda(i);
    dump(out, "user_lambda", 0, lam_dump);
    Matrix B2(n, 3);
    for (Index j = 0; j < 3; ++j)
      for (Index i = 0; i < n; ++i) B2(i, j) = std::sin(0.05 * (i + 1) * (j + 1));
    const BlockSolveReport br = block_nystrom_pcg(*user, B2, mu, pre, opt);
    for (Index j = 0; j < 3; ++j) {
      CHECK(br.converged[static_cast<size_t>(j)]);
      CHECK(static_cast<Index>(br.residual_history[static_cast<size_t>(j)].size()) == br.iterations + 1);
    }
    Vector bx(n);
    for (Index i = 0; i < n; ++i) bx(i) = br.x(i, 1);
    dump(out, "user_block_col1", br.iterations, bx);
    // a device operator regularized on device: the same kernels as nystrom_pcg(op, b, mu, empty)
    Vector lam(n);
    for (Index j = 0; j < n; ++j) lam(j) = std::pow(j + 1.0, -2.0);
    auto A = std::make_shared<DenseOperator>(synthesize_operator(SpectrumProfile(lam), 9));
    const RegularizedOperator dreg = regularize(A, 1e-3);
    CHECK(dreg.handle() != nullptr && !dreg.has_column_access());
    const SolveReport r3 = cg(dreg, b, opt);
    const SolveReport r4 = cg(*A, 1e-3, b, opt);
    CHECK(r3.iterations == r4.iterations);
    double d = 0.0;
    for (Index i = 0; i < n; ++i) d = std::max(d, std::abs(r3.x(i) - r4.x(i)));
    CHECK(d == 0.0);
    const Vector m1 = dreg.matvec(b), m2 = A->matvec(b);
    d = 0.0;
    for (Index i = 0; i < n; ++i) d = std::max(d, std::abs(m1(i) - (m2(i) + 1e-3 * b(i))));
    CHECK(d == 0.0);
    threw = false;
    try { regularize(A, -1.0); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // a user operator's own exception crosses the library unchanged
    threw = false;
    try {
      cg(ThrowingOperator(), Vector{1.0, 2.0, 3.0, 4.0}, opt);
    } catch (const std::domain_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  if (out) std::fclose(out);
  if (failures == 0) std::printf("facade ok\n");
  return failures == 0 ? 0 : 1;
}
