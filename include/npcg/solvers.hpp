// reference: solvers.hpp:20-93 — (P)CG drivers. The loop runs on the B200
// (pcg.cu); reports and exceptions follow the reference exactly.
#pragma once

#include <chrono>
#include <cmath>
#include <vector>

#include "preconditioner.hpp"

namespace npcg {

struct SolveOptions {  // solvers.hpp:20-25
  double eta = 1e-10;
  Index max_iter = 500;
  bool relative = false;
  bool record_iterates = false;
};

struct SolveReport {  // solvers.hpp:28-37
  Vector x;
  Index iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  Index matvec_count = 0;
  double wall_time = 0.0;
  double eta_used = 0.0;
  std::vector<Vector> iterates;
};

struct BlockSolveReport {  // solvers.hpp:40-49
  Matrix x;
  Index iterations = 0;
  std::vector<std::vector<double>> residual_history;  // per column, one entry per iteration (+ the initial)
  std::vector<bool> converged;
  std::vector<Index> deflated;
  Index fallback_count = 0;
  double wall_time = 0.0;
  double eta_used = 0.0;
};

class SolveDivergenceError : public std::runtime_error {  // solvers.hpp:51-57
 public:
  SolveDivergenceError(const std::string& what, SolveReport report)
      : std::runtime_error(what), report(std::move(report)) {}
  SolveReport report;
};

namespace detail {
inline SolveReport pcg_call(const LinearOperator& op, npcg_pre* pre, double mu, const Vector& b, const Vector* x0,
                            const SolveOptions& opt) {
  const Index n = op.dim();
  if (b.size() != n) throw std::invalid_argument("nystrom_pcg: right-hand side length mismatch");
  if (x0 && x0->size() != n) throw std::invalid_argument("nystrom_pcg: initial guess length mismatch");
  npcg_solve_opts o{opt.eta, static_cast<std::int64_t>(opt.max_iter), opt.relative ? 1 : 0, opt.record_iterates ? 1 : 0};
  SolveReport rep;
  rep.x = Vector(n);
  npcg_solve_report r{};
  const Index hl = std::max<Index>(opt.max_iter, 0) + 1;
  std::vector<double> hist(static_cast<size_t>(hl));
  std::vector<double> its(opt.record_iterates ? static_cast<size_t>(hl * n) : 0);
  const OpRef ref = device_handle(op);
  const int rc = npcg_pcg(ref, pre, mu, 1, b.data(), std::max<Index>(n, 1), x0 ? x0->data() : nullptr,
                          std::max<Index>(n, 1), &o, rep.x.data(), std::max<Index>(n, 1), &r, hist.data(),
                          opt.record_iterates ? its.data() : nullptr, NPCG_HOST);
  rep.iterations = r.iterations;
  rep.matvec_count = r.matvec_count;
  rep.converged = r.converged != 0;
  rep.eta_used = r.eta_used;
  rep.wall_time = r.wall_time;
  rep.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
  for (Index t = 0; opt.record_iterates && t < r.history_len; ++t) {
    Vector xi(n);
    std::copy(its.begin() + t * n, its.begin() + (t + 1) * n, xi.data());
    rep.iterates.push_back(std::move(xi));
  }
  if (rc == NPCG_EDIVERGED) throw SolveDivergenceError(npcg_last_error(), std::move(rep));
  ref.check(rc);
  return rep;
}
}  // namespace detail

/// cg (solvers.cpp:111-120): textbook CG on an spd operator, typically
/// regularize(op, mu) (the reference's bench calls cg(RegularizedOperator(op,
/// shift), b, options), bench.cpp:218-220).
inline SolveReport cg(const LinearOperator& op_mu, const Vector& b, const SolveOptions& opt = {}) {
  return detail::pcg_call(op_mu, nullptr, 0.0, b, nullptr, opt);
}
inline SolveReport cg(const LinearOperator& op_mu, const Vector& b, const Vector& x0, const SolveOptions& opt = {}) {
  return detail::pcg_call(op_mu, nullptr, 0.0, b, &x0, opt);
}
/// Extension: cg on op + mu I without building the regularized operator.
inline SolveReport cg(const LinearOperator& op, double mu, const Vector& b, const SolveOptions& opt = {}) {
  return detail::pcg_call(op, nullptr, mu, b, nullptr, opt);
}

/// nystrom_pcg (solvers.cpp:122-148).
inline SolveReport nystrom_pcg(const LinearOperator& op, const Vector& b, double mu,
                               const NystromPreconditioner& precond, const SolveOptions& opt = {}) {
  return detail::pcg_call(op, precond.device.get(), mu, b, nullptr, opt);
}
inline SolveReport nystrom_pcg(const LinearOperator& op, const Vector& b, const Vector& x0, double mu,
                               const NystromPreconditioner& precond, const SolveOptions& opt = {}) {
  return detail::pcg_call(op, precond.device.get(), mu, b, &x0, opt);
}

/// Regularisation path (extension; the paper's protocol):
/// nystrom_pcg for every mu of `mus` on one approximation, the preconditioner
/// rebuilt per mu. warm_start starts mu_k from the solutions of mu_{k-1};
/// with cold starts consecutive mu share each pass over a stored dense A
/// (npcg_regularization_path). Returns reports[k][j] for mu k, column j of b.
inline std::vector<std::vector<SolveReport>> regularization_path(const LinearOperator& op, const Matrix& b,
                                                                 const std::vector<double>& mus,
                                                                 const NystromApproximation& approx,
                                                                 bool warm_start = true,
                                                                 const SolveOptions& opt = {}) {
  const Index n = op.dim(), s = b.cols();
  const Index nmu = static_cast<Index>(mus.size());
  if (b.rows() != n) throw std::invalid_argument("regularization_path: right-hand side row mismatch");
  if (!approx.device) throw std::runtime_error("build_preconditioner: approximation not factored");
  npcg_solve_opts o{opt.eta, static_cast<std::int64_t>(opt.max_iter), opt.relative ? 1 : 0, 0};
  std::vector<npcg_solve_report> reps(static_cast<size_t>(std::max<Index>(nmu * s, 1)));
  std::vector<double> x(static_cast<size_t>(std::max<Index>(n * s * nmu, 1)));
  const OpRef ref = device_handle(op);
  ref.check(npcg_regularization_path(ref, approx.device.get(), nmu, mus.data(), s, b.data(), std::max<Index>(n, 1), &o,
                                     warm_start ? 1 : 0, x.data(), std::max<Index>(n, 1), reps.data(), NPCG_HOST));
  std::vector<std::vector<SolveReport>> out(static_cast<size_t>(nmu));
  for (Index k = 0; k < nmu; ++k)
    for (Index j = 0; j < s; ++j) {
      const npcg_solve_report& r = reps[static_cast<size_t>(k * s + j)];
      SolveReport rep;
      rep.x = Vector(n);
      std::copy(x.begin() + (k * s + j) * n, x.begin() + (k * s + j + 1) * n, rep.x.data());
      rep.iterations = r.iterations;
      rep.matvec_count = r.matvec_count;
      rep.converged = r.converged != 0;
      rep.eta_used = r.eta_used;
      rep.wall_time = r.wall_time;
      out[static_cast<size_t>(k)].push_back(std::move(rep));
    }
  return out;
}

/// block_nystrom_pcg (solvers.cpp:150-279).
inline BlockSolveReport block_nystrom_pcg(const LinearOperator& op, const Matrix& b, double mu,
                                          const NystromPreconditioner& precond, const SolveOptions& opt = {}) {
  const Index n = op.dim(), s = b.cols();
  if (b.rows() != n) throw std::invalid_argument("block_nystrom_pcg: right-hand side row mismatch");
  npcg_solve_opts o{opt.eta, static_cast<std::int64_t>(opt.max_iter), opt.relative ? 1 : 0, 0};
  BlockSolveReport rep;
  rep.x = Matrix(n, s);
  npcg_block_report r{};
  std::vector<int> conv(static_cast<size_t>(s));
  std::vector<std::int64_t> defl(static_cast<size_t>(s));
  std::vector<double> fres(static_cast<size_t>(s));
  const Index hl = std::max<Index>(opt.max_iter, 0) + 1;
  std::vector<double> hist(static_cast<size_t>(hl * s));
  std::vector<std::int64_t> hlen(static_cast<size_t>(s));
  const OpRef ref = device_handle(op);
  ref.check(npcg_block_pcg(ref, precond.device.get(), mu, s, b.data(), std::max<Index>(n, 1), &o, rep.x.data(),
                           std::max<Index>(n, 1), &r, conv.data(), defl.data(), fres.data(), hist.data(), hlen.data(),
                           NPCG_HOST));
  rep.iterations = r.iterations;
  rep.fallback_count = r.fallback_count;
  rep.eta_used = r.eta_used;
  rep.wall_time = r.wall_time;
  for (Index j = 0; j < s; ++j) {
    rep.converged.push_back(conv[static_cast<size_t>(j)] != 0);
    rep.residual_history.emplace_back(hist.begin() + j * hl, hist.begin() + j * hl + hlen[static_cast<size_t>(j)]);
  }
  rep.deflated.assign(defl.begin(), defl.begin() + r.n_deflated);
  return rep;
}

/// iteration_bound (solvers.cpp:281-291).
inline Index iteration_bound(double kappa, double epsilon) {
  std::int64_t out = 0;
  check_status(npcg_iteration_bound(kappa, epsilon, &out));
  return out;
}

}  // namespace npcg
