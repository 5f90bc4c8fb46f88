// TEST INFRASTRUCTURE ONLY. extern "C" surface of the CPU oracle so the
// Python tests (tests/) and bench.py's CPU-baseline leg can drive it through
// ctypes. Status codes mirror the product C-ABI (include/npcg_capi.h):
// 0 ok, 1 invalid_argument, 2 runtime_error, 3 SolveDivergenceError.
#include <cstring>
#include <memory>
#include <string>

#include "blas_lapack.h"
#include "npcg_oracle.hpp"

using namespace npcg_oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const SolveDivergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
Matrix mat(Index r, Index c, const double* p) {
  Matrix m(r, c);
  if (r > 0 && c > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}
Vector vec(Index n, const double* p) { return Vector(p, p + n); }

// RegularizedOperator (operators.cpp:82-103): matvec = base.matvec(v); out += mu v.
class Regularized final : public LinearOperator {
 public:
  Regularized(const LinearOperator& b, double mu) : b_(b), mu_(mu) {
    if (!(mu_ >= 0.0)) throw std::invalid_argument("RegularizedOperator: mu must be >= 0");
  }
 protected:
  Index do_dim() const override { return b_.dim(); }
  void do_matvec(const Vector& v, Vector& out) const override {
    out = b_.matvec(v);
    for (size_t i = 0; i < out.size(); ++i) out[i] += mu_ * v[i];
  }
 private:
  const LinearOperator& b_;
  double mu_;
};

struct SolveOut {
  double* x;
  int64_t* iterations;
  int* converged;
  int64_t* matvec_count;
  double* eta_used;
  double* wall_time;
  double* history;      // capacity max_iter+1
  int64_t* history_len;
  double* iterates;     // nullable, capacity (max_iter+1)*n
};
void fill(const SolveReport& r, Index n, const SolveOut& o) {
  if (o.x) std::memcpy(o.x, r.x.data(), sizeof(double) * static_cast<size_t>(n));
  *o.iterations = r.iterations;
  *o.converged = r.converged ? 1 : 0;
  *o.matvec_count = r.matvec_count;
  *o.eta_used = r.eta_used;
  *o.wall_time = r.wall_time;
  *o.history_len = static_cast<int64_t>(r.residual_history.size());
  if (o.history)
    std::memcpy(o.history, r.residual_history.data(), sizeof(double) * r.residual_history.size());
  if (o.iterates)
    for (size_t t = 0; t < r.iterates.size(); ++t)
      std::memcpy(o.iterates + t * static_cast<size_t>(n), r.iterates[t].data(), sizeof(double) * static_cast<size_t>(n));
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int n) { openblas_set_num_threads(n); }
int orc_get_threads(void) { return openblas_get_num_threads(); }
const char* orc_corename(void) { return openblas_get_corename(); }

// ---- RNG --------------------------------------------------------------------
void* orc_rng_new(uint64_t seed) { return new Rng(seed); }
void* orc_rng_clone(void* r) { return new Rng(*static_cast<Rng*>(r)); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
double orc_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
double orc_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
uint64_t orc_rng_word(void* r) { return static_cast<Rng*>(r)->engine(); }
void orc_rng_discard(void* r, uint64_t k) { static_cast<Rng*>(r)->engine.discard(k); }
int orc_rng_integer(void* r, uint64_t bound, uint64_t* out) {
  return guard([&] { *out = static_cast<Rng*>(r)->integer(bound); });
}
void orc_gaussian_matrix(void* r, int64_t rows, int64_t cols, double* out) {
  Matrix g = gaussian_matrix(*static_cast<Rng*>(r), rows, cols);
  if (rows > 0 && cols > 0) std::memcpy(out, g.data(), sizeof(double) * g.size());
}
int orc_sample_without_replacement(void* r, int64_t n, int64_t k, int64_t* out) {
  return guard([&] {
    auto s = sample_without_replacement(*static_cast<Rng*>(r), n, k);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  });
}
uint64_t orc_splitmix64(uint64_t s) { return synthetic_operator_seed(s); }
void orc_rng_uniform_fill(void* r, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = static_cast<Rng*>(r)->uniform();
}

// ---- dense ------------------------------------------------------------------
double orc_ulp_spacing(double x) { return dense::ulp_spacing(x); }
int orc_orthonormal_columns(int64_t m, int64_t n, const double* g, double* q) {
  return guard([&] {
    Matrix out = dense::orthonormal_columns(mat(m, n, g));
    std::memcpy(q, out.data(), sizeof(double) * out.size());
  });
}
int orc_thin_svd(int64_t m, int64_t n, const double* b, double* u, double* s) {
  return guard([&] {
    auto out = dense::thin_svd(mat(m, n, b));
    std::memcpy(u, out.u.data(), sizeof(double) * out.u.size());
    std::memcpy(s, out.singular.data(), sizeof(double) * out.singular.size());
  });
}
int orc_sym_eig(int64_t n, const double* a, double* vals, double* vecs) {
  return guard([&] {
    auto e = dense::sym_eig(mat(n, n, a));
    std::memcpy(vals, e.values.data(), sizeof(double) * e.values.size());
    if (vecs) std::memcpy(vecs, e.vectors.data(), sizeof(double) * e.vectors.size());
  });
}

// ---- operators --------------------------------------------------------------
int orc_op_dense(int64_t n, int64_t ncols, const double* a, void** out) {
  return guard([&] { *out = new DenseOperator(mat(n, ncols, a)); });
}
int orc_op_gram(int64_t m, int64_t n, const double* g, void** out) {
  return guard([&] { *out = new GramRidgeOperator(mat(m, n, g)); });
}
int orc_op_kernel(int64_t n, int64_t d, const double* pts, double sigma, int64_t cap, void** out) {
  return guard([&] { *out = new KernelOperator(mat(n, d, pts), sigma, cap); });
}
int orc_op_synth(int64_t n, const double* lam, uint64_t seed, void** out) {
  return guard([&] { *out = new DenseOperator(synthesize_operator(vec(n, lam), seed)); });
}
void orc_op_free(void* op) { delete static_cast<LinearOperator*>(op); }
int64_t orc_op_dim(void* op) { return static_cast<LinearOperator*>(op)->dim(); }
int orc_op_apply(void* op, int64_t rows, int64_t k, const double* v, double* out) {
  return guard([&] {
    auto* o = static_cast<LinearOperator*>(op);
    if (k == 1 && rows == o->dim()) {  // matvec path (checks + do_matvec)
      Vector r = o->matvec(vec(rows, v));
      std::memcpy(out, r.data(), sizeof(double) * r.size());
    } else {
      Matrix r = o->apply_block(mat(rows, k, v));
      std::memcpy(out, r.data(), sizeof(double) * r.size());
    }
  });
}
int orc_op_apply_block(void* op, int64_t rows, int64_t k, const double* v, double* out) {
  return guard([&] {
    Matrix r = static_cast<LinearOperator*>(op)->apply_block(mat(rows, k, v));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}
int orc_op_column(void* op, int64_t j, double* out) {
  return guard([&] {
    Vector r = static_cast<LinearOperator*>(op)->column(j);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}
// Dense matrix behind a DenseOperator or a stored KernelOperator (n*n doubles).
int orc_op_dense_data(void* op, double* out) {
  return guard([&] {
    auto* o = static_cast<LinearOperator*>(op);
    if (auto* d = dynamic_cast<DenseOperator*>(o)) {
      std::memcpy(out, d->dense().data(), sizeof(double) * d->dense().size());
    } else if (auto* k = dynamic_cast<KernelOperator*>(o); k && k->is_dense()) {
      std::memcpy(out, k->kernel().data(), sizeof(double) * k->kernel().size());
    } else {
      throw std::runtime_error("orc_op_dense_data: operator has no stored matrix");
    }
  });
}

// ---- Nyström ----------------------------------------------------------------
int orc_sketch_empty(int64_t n, void** out) {
  return guard([&] { *out = new SketchPair(make_empty_sketch(n)); });
}
void orc_sketch_free(void* p) { delete static_cast<SketchPair*>(p); }
int64_t orc_sketch_size(void* p) { return static_cast<SketchPair*>(p)->size(); }
void orc_sketch_get(void* p, double* omega, double* y) {
  auto* s = static_cast<SketchPair*>(p);
  if (omega) std::memcpy(omega, s->omega.data(), sizeof(double) * s->omega.size());
  if (y) std::memcpy(y, s->y.data(), sizeof(double) * s->y.size());
}
int orc_sketch_extend(void* p, void* op, int64_t extra, void* rng, void** out) {
  return guard([&] {
    *out = new SketchPair(extend_sketch(*static_cast<SketchPair*>(p), *static_cast<LinearOperator*>(op),
                                        extra, *static_cast<Rng*>(rng)));
  });
}
int orc_sketch_extend_with(void* p, void* op, int64_t extra, const double* fresh, void** out) {
  return guard([&] {
    auto* o = static_cast<LinearOperator*>(op);
    *out = new SketchPair(
        extend_sketch_with(*static_cast<SketchPair*>(p), *o, mat(o->dim(), extra, fresh)));
  });
}
int orc_sketch_extend_columns(void* p, void* op, int64_t extra, const int64_t* used_in, int64_t n_used, void* rng,
                              int64_t* used_out, void** out) {
  return guard([&] {
    std::vector<Index> used(used_in, used_in + n_used);
    *out = new SketchPair(extend_sketch_columns(*static_cast<SketchPair*>(p), *static_cast<LinearOperator*>(op), extra,
                                                used, *static_cast<Rng*>(rng)));
    std::copy(used.begin(), used.end(), used_out);
  });
}
int orc_column_sampling_nystrom(void* op, int64_t k, const int64_t* indices, void** out) {
  return guard([&] {
    *out = new NystromApproximation(column_sampling_nystrom(*static_cast<LinearOperator*>(op),
                                                            std::vector<Index>(indices, indices + k)));
  });
}
int orc_column_sampling_nystrom_rng(void* op, int64_t ell, void* rng, void** out) {
  return guard([&] {
    *out = new NystromApproximation(
        column_sampling_nystrom(*static_cast<LinearOperator*>(op), ell, *static_cast<Rng*>(rng)));
  });
}
int orc_nystrom_from_sketch(void* p, void** out) {
  return guard([&] { *out = new NystromApproximation(nystrom_from_sketch(*static_cast<SketchPair*>(p))); });
}
int orc_randomized_nystrom(void* op, int64_t ell, void* rng, void** out) {
  return guard([&] {
    *out = new NystromApproximation(
        randomized_nystrom(*static_cast<LinearOperator*>(op), ell, *static_cast<Rng*>(rng)));
  });
}
int orc_approx_make(int64_t n, int64_t ell, const double* u, const double* lam, double shift, void** out) {
  return guard([&] {
    auto* a = new NystromApproximation;
    a->u = mat(n, ell, u);
    a->lambda = vec(ell, lam);
    a->shift_used = shift;
    *out = a;
  });
}
void orc_approx_info(void* a, int64_t* n, int64_t* ell, double* shift) {
  auto* x = static_cast<NystromApproximation*>(a);
  *n = x->u.rows;
  *ell = x->u.cols;
  *shift = x->shift_used;
}
void orc_approx_get(void* a, double* u, double* lam) {
  auto* x = static_cast<NystromApproximation*>(a);
  if (u) std::memcpy(u, x->u.data(), sizeof(double) * x->u.size());
  if (lam) std::memcpy(lam, x->lambda.data(), sizeof(double) * x->lambda.size());
}
void orc_approx_free(void* a) { delete static_cast<NystromApproximation*>(a); }

// ---- preconditioner ---------------------------------------------------------
int orc_pre_build(void* approx, double mu, void** out) {
  return guard([&] {
    *out = new NystromPreconditioner(build_preconditioner(*static_cast<NystromApproximation*>(approx), mu));
  });
}
void orc_pre_free(void* p) { delete static_cast<NystromPreconditioner*>(p); }
int orc_woodbury(void* approx, double mu, int64_t n, const double* b, double* x) {
  return guard([&] {
    auto* a = static_cast<NystromApproximation*>(approx);
    const Vector out = woodbury_inverse_apply(a->u, a->lambda, mu, vec(n, b));
    std::memcpy(x, out.data(), sizeof(double) * static_cast<size_t>(n));
  });
}
int orc_pre_apply_inverse(void* p, int64_t n, int64_t s, const double* r, double* z) {
  return guard([&] {
    auto* pre = static_cast<NystromPreconditioner*>(p);
    if (s == 1) {
      Vector out = pre->apply_inverse(vec(n, r));
      std::memcpy(z, out.data(), sizeof(double) * out.size());
    } else {
      Matrix out = pre->apply_inverse_block(mat(n, s, r));
      std::memcpy(z, out.data(), sizeof(double) * out.size());
    }
  });
}
int orc_pre_apply(void* p, int64_t n, const double* v, double* out) {
  return guard([&] {
    Vector o = static_cast<NystromPreconditioner*>(p)->apply(vec(n, v));
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

// ---- solvers ----------------------------------------------------------------
// pre == nullptr -> empty (identity) preconditioner built with `mu`.
int orc_pcg(void* op, const double* b, const double* x0, double mu, void* pre, double eta,
            int64_t max_iter, int relative, int record_iterates, double* x, int64_t* iterations,
            int* converged, int64_t* matvec_count, double* eta_used, double* wall_time,
            double* history, int64_t* history_len, double* iterates) {
  auto* o = static_cast<LinearOperator*>(op);
  const Index n = o->dim();
  SolveOut so{x, iterations, converged, matvec_count, eta_used, wall_time, history, history_len, iterates};
  SolveOptions opt{eta, max_iter, relative != 0, record_iterates != 0};
  *history_len = 0;
  try {
    NystromPreconditioner identity;
    identity.u = Matrix(n, 0);
    identity.mu = mu;
    const NystromPreconditioner& p = pre ? *static_cast<NystromPreconditioner*>(pre) : identity;
    const Vector x0v = x0 ? vec(n, x0) : Vector(static_cast<size_t>(n), 0.0);
    fill(nystrom_pcg(*o, vec(n, b), x0v, mu, p, opt), n, so);
    return 0;
  } catch (const SolveDivergenceError& e) {
    g_err = e.what();
    fill(e.report, n, so);
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
// cg() on A + mu I (RegularizedOperator), solvers.cpp:111-120.
int orc_cg(void* op, double mu, const double* b, const double* x0, double eta, int64_t max_iter,
           int relative, double* x, int64_t* iterations, int* converged, int64_t* matvec_count,
           double* eta_used, double* wall_time, double* history, int64_t* history_len) {
  auto* o = static_cast<LinearOperator*>(op);
  const Index n = o->dim();
  SolveOut so{x, iterations, converged, matvec_count, eta_used, wall_time, history, history_len, nullptr};
  *history_len = 0;
  try {
    Regularized reg(*o, mu);
    const Vector x0v = x0 ? vec(n, x0) : Vector(static_cast<size_t>(n), 0.0);
    fill(cg(reg, vec(n, b), x0v, SolveOptions{eta, max_iter, relative != 0, false}), n, so);
    return 0;
  } catch (const SolveDivergenceError& e) {
    g_err = e.what();
    fill(e.report, n, so);
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
int orc_block_pcg(void* op, int64_t s, const double* b, double mu, void* pre, double eta,
                  int64_t max_iter, int relative, double* x, int64_t* iterations, int* converged,
                  int64_t* deflated, int64_t* n_deflated, int64_t* fallback_count, double* final_res,
                  double* history, int64_t* history_len) {
  return guard([&] {
    auto* o = static_cast<LinearOperator*>(op);
    const Index n = o->dim();
    NystromPreconditioner identity;
    identity.u = Matrix(n, 0);
    identity.mu = mu;
    const NystromPreconditioner& p = pre ? *static_cast<NystromPreconditioner*>(pre) : identity;
    auto r = block_nystrom_pcg(*o, mat(n, s, b), mu, p, SolveOptions{eta, max_iter, relative != 0, false});
    std::memcpy(x, r.x.data(), sizeof(double) * r.x.size());
    *iterations = r.iterations;
    for (Index j = 0; j < s; ++j) {
      converged[j] = r.converged[static_cast<size_t>(j)] ? 1 : 0;
      const auto& h = r.residual_history[static_cast<size_t>(j)];
      final_res[j] = h.back();
      if (history_len) history_len[j] = static_cast<int64_t>(h.size());
      if (history) std::memcpy(history + j * (max_iter + 1), h.data(), sizeof(double) * h.size());
    }
    *n_deflated = static_cast<int64_t>(r.deflated.size());
    for (size_t i = 0; i < r.deflated.size(); ++i) deflated[i] = r.deflated[i];
    *fallback_count = r.fallback_count;
  });
}
int orc_iteration_bound(double kappa, double eps, int64_t* out) {
  return guard([&] { *out = iteration_bound(kappa, eps); });
}

// ---- adaptive ---------------------------------------------------------------
int orc_estimate_error_power(void* op, void* approx, int64_t q, void* rng, double* out) {
  return guard([&] {
    auto* a = static_cast<NystromApproximation*>(approx);
    *out = estimate_error_power(*static_cast<LinearOperator*>(op), a->u, a->lambda, q, *static_cast<Rng*>(rng));
  });
}
// mode: 0 error, 1 ratio, 2 fixed; sketch: 0 gaussian, 1 column sampling.
int orc_adaptive(void* op, int mode, int64_t ell0, int64_t ell_max, double mu, int has_tau,
                 double tau, int64_t q, int secondary, int sketch, void* rng, void** approx_out,
                 int* has_err, double* err, int64_t* doublings, int* hit_cap, double* posterior,
                 int64_t* ell_final) {
  return guard([&] {
    AdaptiveConfig c;
    c.ell0 = ell0;
    c.ell_max = ell_max;
    c.mu = mu;
    c.tol_mode = static_cast<TolMode>(mode);
    if (has_tau) c.tau = tau;
    c.q = q;
    c.secondary_criterion = secondary != 0;
    c.sketch = static_cast<SketchKind>(sketch);
    auto& o = *static_cast<LinearOperator*>(op);
    auto& r = *static_cast<Rng*>(rng);
    AdaptiveOutcome out = mode == 0 ? adaptive_nystrom(o, c, r)
                          : mode == 1 ? adaptive_nystrom_ratio(o, c, r)
                                      : fixed_rank_nystrom(o, c, r);
    *has_err = out.error_estimate.has_value() ? 1 : 0;
    *err = out.error_estimate.value_or(0.0);
    *doublings = out.doublings;
    *hit_cap = out.hit_cap ? 1 : 0;
    *posterior = out.posterior_condition_estimate;
    *ell_final = out.ell_final;
    *approx_out = new NystromApproximation(std::move(out.approximation));
  });
}
int orc_posterior(double l, double mu, double e, double* out) {
  return guard([&] { *out = posterior_condition_estimate(l, mu, e); });
}

}  // extern "C"
