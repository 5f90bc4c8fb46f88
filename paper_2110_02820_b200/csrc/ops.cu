// Operators, Nyström sketch/factorisation and the preconditioner on device.
// Reference: operators.cpp, nystrom.cpp, preconditioner.cpp (file:line per
// function below; paths relative to /root/reference/proj/core/src/).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "blas.cuh"
#include "factor.cuh"
#include "gemm.cuh"
#include "ops.cuh"
#include "ozaki.cuh"

namespace npcg {

// =============================== operators ===================================
void Op::apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate) {
  // RegularizedOperator / nystrom_pcg apply_op (operators.cpp:95-103, solvers.cpp:137-141):
  // out = A p; out += mu p.
  apply(P, ldp, S, out, ldo, gate);
  if (ldp == ldo) {
    axpby(*ctx, nloc, S, mu, P, 1.0, out, ldo);
  } else {
    for (int s = 0; s < S; ++s) axpby(*ctx, nloc, 1, mu, P + s * ldp, 1.0, out + s * ldo, ldo);
  }
}

void Op::column(i64, double*) { fail(NPCG_ERUNTIME, "LinearOperator - column: operator has no column access"); }

void Op::columns(const i64* idx, i64 k, double* out, i64 ldo) {
  for (i64 c = 0; c < k; ++c) column(idx[c], out + c * ldo);
}

namespace {
__global__ void gather_cols_kernel2(const double* __restrict__ a, i64 lda, i64 n, const i64* __restrict__ idx, i64 k,
                                    double* __restrict__ out, i64 ldo) {
  const i64 total = n * k;
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = t % n, c = t / n;
    out[i + c * ldo] = a[i + idx[c] * lda];
  }
}
// omega(:, c) = e_idx[c], restricted to this rank's rows [off, off + nloc)
__global__ void unit_cols_kernel(double* __restrict__ om, i64 ldo, const i64* __restrict__ idx, i64 k, i64 off,
                                 i64 nloc) {
  const i64 c = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < k && idx[c] >= off && idx[c] < off + nloc) om[idx[c] - off + c * ldo] = 1.0;
}
}  // namespace

void DenseOp::columns(const i64* idx, i64 k, double* out, i64 ldo) {
  DBuf<i64> d(k, ctx->stream);
  NPCG_CUDA(cudaMemcpyAsync(d.p, idx, sizeof(i64) * k, cudaMemcpyHostToDevice, ctx->stream));
  NPCG_LAUNCH(*ctx, gather_cols_kernel2, static_cast<unsigned>(std::min<i64>(cdiv(n * k, 256), 4096)), 256, 0,
              a.p(), a.ld, n, d.p, k, out, ldo);
  ctx->sync();  // the host index buffer is the caller's
}

// DenseOperator::do_matvec / do_apply_block (operators.cpp:72-78). A is
// symmetric, so A V is computed as A^T V: each output entry is a dot of a
// contiguous column with V (coldot for <= 8 columns; DMMA GEMM beyond; the
// sketch-sized blocks of a large A on the INT8 tensor cores by digit-plane
// splitting, which costs two passes over A and pays from ~130 columns on).
bool ozaki_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NPCG_OZAKI");  // diagnostics: NPCG_OZAKI=0 keeps every product on DMMA
    return e == nullptr || std::string(e) != "0";
  }();
  return on;
}
void DenseOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  if (k <= 8) {
    coldot(*ctx, a.p(), a.ld, n, n, V, ldv, static_cast<int>(k), out, ldo, 0.0, nullptr, 0, gate);
  } else if (k >= 192 && n >= 4096 && a.rows == n && a.cols == n && ozaki_enabled()) {
    gemm_ozaki(*ctx, n, k, n, a.p(), a.ld, true, V, ldv, 0.0, out, ldo);
  } else {
    gemm(*ctx, n, k, n, 1.0, Operand{a.p(), a.ld, true}, Operand{V, ldv, true}, 0.0, out, ldo);
  }
}
void DenseOp::apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate) {
  if (S <= 8) {  // fused epilogue: v_i = (A p)_i + mu p_i
    coldot(*ctx, a.p(), a.ld, n, n, P, ldp, S, out, ldo, mu, P, ldp, gate);
  } else {
    Op::apply_shift(P, ldp, S, mu, out, ldo, gate);
  }
}
void DenseOp::column(i64 j, double* out) { copy2d(*ctx, n, 1, a.col(j), a.ld, out, n); }

void KernelFreeOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  kernel_apply_free(*ctx, *this, V, ldv, k, out, ldo, gate);
}

// User operator callbacks (npcg_op_callback_create). The gate is the PCG
// loop's "any column running" flag: a product of a finished solve is skipped,
// so the user's operator sees exactly the products the reference would make.
void CallbackOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  Ctx& c = *ctx;
  if (gate) {
    int h = 1;
    NPCG_CUDA(cudaMemcpyAsync(&h, gate, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (h == 0) return;
  }
  int rc = 0;
  if (where == NPCG_DEVICE) {
    rc = fn(user, n, k, V, ldv, out, ldo, c.stream);
  } else {
    std::vector<double> hv(static_cast<size_t>(n * k)), ho(static_cast<size_t>(n * k));
    NPCG_CUDA(cudaMemcpy2DAsync(hv.data(), n * 8, V, ldv * 8, n * 8, k, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    rc = fn(user, n, k, hv.data(), n, ho.data(), n, nullptr);
    if (rc == 0) {
      NPCG_CUDA(cudaMemcpy2DAsync(out, ldo * 8, ho.data(), n * 8, n * 8, k, cudaMemcpyHostToDevice, c.stream));
      c.sync();  // ho is released on return
    }
  }
  if (rc != 0) fail(NPCG_ERUNTIME, "LinearOperator callback failed (apply returned " + std::to_string(rc) + ")");
}

void CallbackOp::column(i64 j, double* out) {
  Ctx& c = *ctx;
  if (!col) Op::column(j, out);
  int rc = 0;
  if (where == NPCG_DEVICE) {
    rc = col(user, j, out, c.stream);
  } else {
    std::vector<double> h(static_cast<size_t>(n));
    c.sync();
    rc = col(user, j, h.data(), nullptr);
    if (rc == 0) {
      NPCG_CUDA(cudaMemcpyAsync(out, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
      c.sync();
    }
  }
  if (rc != 0) fail(NPCG_ERUNTIME, "LinearOperator callback failed (column returned " + std::to_string(rc) + ")");
}

// RegularizedOperator::do_matvec / do_apply_block (operators.cpp:95-103):
// out = base V; out += mu V -- the base's fused shift epilogue has exactly
// this rounding order.
void RegOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  if (k <= 8) {
    base->apply_shift(V, ldv, static_cast<int>(k), mu, out, ldo, gate);
  } else {
    base->apply(V, ldv, k, out, ldo, gate);
    for (i64 s = 0; s < k; ++s) axpby(*ctx, nloc, 1, mu, V + s * ldv, 1.0, out + s * ldo, ldo);
  }
}
void RegOp::apply_shift(const double* P, i64 ldp, int S, double mu2, double* out, i64 ldo, const int* gate) {
  apply(P, ldp, S, out, ldo, gate);
  if (mu2 != 0.0) {  // (A_mu p) += mu2 p (nystrom_pcg on a regularized operator, solvers.cpp:137-141)
    for (int s = 0; s < S; ++s) axpby(*ctx, nloc, 1, mu2, P + s * ldp, 1.0, out + s * ldo, ldo);
  }
}

// ================================ Nyström ====================================
namespace {
/// Make columns [0, cols) of s's sketch writable by s: in place when s owns
/// the written end of its store and the capacity suffices, otherwise a fresh
/// store (doubling growth) with s's `size` columns copied over.
void ensure_capacity(Nys& s, i64 cols) {
  if (s.sk && s.sk->omega.cols >= cols && s.sk->filled == s.size) return;
  const i64 have = s.sk ? s.sk->omega.cols : 0;
  const i64 cap = std::min<i64>(s.n, std::max<i64>(cols, 2 * have));
  auto st = std::make_shared<SketchStore>();
  st->omega.alloc(s.nloc, cap, s.ctx->stream, true);
  st->y.alloc(s.nloc, cap, s.ctx->stream, true);
  if (s.size > 0) {
    copy2d(*s.ctx, s.nloc, s.size, s.sk->omega.p(), s.sk->omega.ld, st->omega.p(), st->omega.ld);
    copy2d(*s.ctx, s.nloc, s.size, s.sk->y.p(), s.sk->y.ld, st->y.p(), st->y.ld);
  }
  st->filled = s.size;
  s.sk = std::move(st);
}
}  // namespace

// extend_sketch (nystrom.cpp:36-58) after the Gaussian draw. `raw` is this
// rank's row block of the n x extra Gaussian (all of it unsharded). On a
// sharded context the Gram-Schmidt projections and the CholeskyQR Grams are
// all-reduced (l_old x extra, extra x extra) and Y_new = A Q_new all-gathers Q.
void nys_extend(Nys& s, const double* raw, i64 ld, i64 extra, int where) {
  Ctx& ctx = *s.ctx;
  if (!s.op) fail(NPCG_ERUNTIME, "extend_sketch: approximation has no operator");
  if (extra < 1) invalid("extend_sketch: extra must be >= 1");
  if (s.size + extra > s.n) invalid("extend_sketch: sketch size would exceed dimension");
  const i64 n = s.nloc, old = s.size;
  DMat fresh;
  upload(ctx, fresh, n, extra, raw, ld, where);
  ensure_capacity(s, old + extra);
  SketchStore& st = *s.sk;
  // Two passes of block Gram-Schmidt against the existing columns.
  if (old > 0) {
    DMat coef;
    coef.alloc(old, extra, ctx.stream, false);
    for (int pass = 0; pass < 2; ++pass) {
      gemm(ctx, old, extra, n, 1.0, Operand{st.omega.p(), st.omega.ld, true}, Operand{fresh.p(), fresh.ld, true}, 0.0,
           coef.p(), coef.ld);
      rows_allreduce(ctx, coef.p(), coef.ld * extra);  // Omega^T fresh over all row blocks
      gemm(ctx, n, extra, old, -1.0, Operand{st.omega.p(), st.omega.ld, false}, Operand{coef.p(), coef.ld, true}, 1.0,
           fresh.p(), fresh.ld);
    }
  }
  double* q_new = st.omega.col(old);
  orthonormalize(ctx, fresh.p(), fresh.ld, n, extra, q_new, st.omega.ld, nullptr, 0, /*dist=*/true);
  s.op->apply(q_new, st.omega.ld, extra, st.y.col(old), st.y.ld);
  s.size = st.filled = old + extra;
  s.fac.reset();  // the handle now holds an unfactored, larger sketch
}

void nys_extend_columns(Nys& s, const std::vector<i64>& idx) {
  Ctx& ctx = *s.ctx;
  const i64 old = s.size, extra = static_cast<i64>(idx.size());
  if (extra == 0) return;
  ensure_capacity(s, old + extra);
  SketchStore& st = *s.sk;
  // omega columns: e_j (fresh capacity is zero; reused capacity is cleared first)
  NPCG_CUDA(cudaMemset2DAsync(st.omega.col(old), st.omega.ld * 8, 0, s.nloc * 8, extra, ctx.stream));
  DBuf<i64> d(extra, ctx.stream);
  NPCG_CUDA(cudaMemcpyAsync(d.p, idx.data(), sizeof(i64) * extra, cudaMemcpyHostToDevice, ctx.stream));
  NPCG_LAUNCH(ctx, unit_cols_kernel, static_cast<unsigned>(cdiv(extra, 256)), 256, 0, st.omega.col(old), st.omega.ld,
              d.p, extra, s.off, s.nloc);
  s.op->columns(idx.data(), extra, st.y.col(old), st.y.ld);
  ctx.sync();
  s.size = st.filled = old + extra;
  s.fac.reset();
}

namespace {
__global__ void clamp_lambda_kernel(const double* sigma, i64 ell, double nu, double* lambda) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < ell) lambda[i] = fmax(sigma[i] * sigma[i] - nu, 0.0);
}
double ulp_spacing(double x) {
  const double ax = std::abs(x);
  return std::nextafter(ax, std::numeric_limits<double>::infinity()) - ax;
}
}  // namespace

// nystrom_from_sketch (nystrom.cpp:96-140). The result is built in a fresh
// Factors and published only after every check passed. Sharded: ||Y||_F, the
// finiteness checks and the core Omega^T Y_nu are all-reduced, so every rank
// takes the same shift / Cholesky branch on bitwise-identical l x l data;
// B = Y_nu L^-T and U keep the local rows.
void nys_factor(Nys& s) {
  Ctx& ctx = *s.ctx;
  const i64 n = s.nloc, ell = s.size;
  auto f = std::make_shared<Factors>();
  f->ell = ell;
  if (ell == 0) {
    f->u.alloc(n, 0, ctx.stream, false);
    s.fac = std::move(f);
    return;
  }
  const DMat& om = s.omega();
  const DMat& y = s.y();
  if (!all_finite_rows(ctx, y.p(), n, ell, y.ld))
    fail(NPCG_ERUNTIME, "nystrom_from_sketch: sketch has non-finite entries");
  const double ynorm = std::sqrt(sum_squares_rows(ctx, y.p(), n, ell, y.ld));
  const double nu0 = ulp_spacing(ynorm);
  double nu = nu0;
  DMat ynu, core, b;
  ynu.alloc(n, ell, ctx.stream, false);
  core.alloc(ell, ell, ctx.stream, false);
  b.alloc(n, ell, ctx.stream, false);
  bool factored = false;
  for (int attempt = 0; attempt <= 3; ++attempt, nu *= 10.0) {
    add_scaled(ctx, n, ell, y.p(), nu, om.p(), ynu.p(), ynu.ld);  // Y + nu Omega (shared ld)
    gemm(ctx, ell, ell, n, 1.0, Operand{om.p(), om.ld, true}, Operand{ynu.p(), ynu.ld, true}, 0.0,
         core.p(), core.ld);
    rows_allreduce(ctx, core.p(), core.ld * ell);  // Omega^T Y_nu over all row blocks
    CholFactor cf;
    if (!cholesky(ctx, core.p(), ell, core.ld, cf)) continue;
    trsm_right_lt(ctx, n, ell, ynu.p(), ynu.ld, core.p(), core.ld, cf, b.p(), b.ld);
    if (!all_finite_rows(ctx, b.p(), n, ell, b.ld)) continue;
    f->shift = nu;
    factored = true;
    break;
  }
  if (!factored) {
    std::ostringstream msg;
    msg << "nystrom_from_sketch: Cholesky failed after 3 shift escalations"
        << " (n = " << s.n << ", ell = " << ell << ", initial shift = " << nu0 << ", final shift = " << nu / 10.0
        << ", ||Y||_F = " << ynorm << ")";
    fail(NPCG_ERUNTIME, msg.str());
  }
  ynu.buf.release();
  core.buf.release();
  f->u.alloc(n, ell, ctx.stream, false);
  DBuf<double> sigma(ell, ctx.stream);
  thin_svd(ctx, b.p(), b.ld, n, ell, f->u.p(), f->u.ld, sigma.p, /*dist=*/true);
  f->lambda.alloc(ell, ctx.stream);
  NPCG_LAUNCH(ctx, clamp_lambda_kernel, static_cast<unsigned>(cdiv(ell, 256)), 256, 0, sigma.p, ell, f->shift,
              f->lambda.p);
  f->lambda_host.assign(static_cast<size_t>(ell), 0.0);
  NPCG_CUDA(cudaMemcpyAsync(f->lambda_host.data(), f->lambda.p, sizeof(double) * ell, cudaMemcpyDeviceToHost,
                            ctx.stream));
  ctx.sync();
  for (i64 i = 1; i < ell; ++i)
    if (f->lambda_host[i] > f->lambda_host[i - 1])
      fail(NPCG_ERUNTIME, "nystrom_from_sketch: eigenvalue estimates out of order");
  s.fac = std::move(f);
}

// ============================ preconditioner =================================
namespace {
__global__ void gains_kernel(const double* lambda, i64 ell, double lambda_ell, double mu, double* inv, double* fwd) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ell) return;
  inv[i] = (lambda_ell + mu) / (lambda[i] + mu) - 1.0;  // preconditioner.cpp:33
  fwd[i] = (lambda[i] + mu) / (lambda_ell + mu) - 1.0;  // preconditioner.cpp:22
}
__global__ void scale_rows_kernel(double* T, i64 ell, i64 S, i64 ldt, const double* g, const int* gate) {
  if (gate && *gate == 0) return;
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= ell * S) return;
  const i64 j = idx % ell, s = idx / ell;
  T[j + s * ldt] = g[j] * T[j + s * ldt];
}
}  // namespace

// build_preconditioner (preconditioner.cpp:80-89).
void pre_build(Pre& p, const Nys& s, double mu) {
  if (!(mu > 0.0)) invalid("build_preconditioner: mu must be > 0");
  if (!s.factored()) fail(NPCG_ERUNTIME, "build_preconditioner: approximation not factored");
  p.ctx = s.ctx;
  p.fac = s.fac;
  p.n = s.n;
  p.nloc = s.nloc;
  p.ell = s.fac->ell;
  p.mu = mu;
  p.lambda_ell = s.fac->lambda_min();
  if (p.ell > 0) {
    p.gain_inv.alloc(p.ell, s.ctx->stream);
    p.gain_fwd.alloc(p.ell, s.ctx->stream);
    NPCG_LAUNCH(*s.ctx, gains_kernel, static_cast<unsigned>(cdiv(p.ell, 256)), 256, 0, s.fac->lambda.p, p.ell,
                p.lambda_ell, mu, p.gain_inv.p, p.gain_fwd.p);
  }
}

namespace {
// out = V + U diag(g) U^T V   (preconditioner.cpp:17-45 shapes). Sharded: U
// and V are this rank's rows; T = U^T V is all-reduced (l x S).
void lowrank_update(Pre& p, const double* g, const double* V, i64 ldv, i64 S, double* out, i64 ldo,
                    const int* gate) {
  Ctx& ctx = *p.ctx;
  const i64 n = p.nloc;
  if (p.ell == 0) {
    copy2d(ctx, n, S, V, ldv, out, ldo);
    return;
  }
  const Factors& s = *p.fac;
  DMat T;
  T.alloc(p.ell, S, ctx.stream, false);
  if (S <= 8) {
    coldot(ctx, s.u.p(), s.u.ld, n, p.ell, V, ldv, static_cast<int>(S), T.p(), T.ld, 0.0, nullptr, 0, gate);
  } else {
    gemm(ctx, p.ell, S, n, 1.0, Operand{s.u.p(), s.u.ld, true}, Operand{V, ldv, true}, 0.0, T.p(), T.ld);
  }
  rows_allreduce(ctx, T.p(), T.ld * S);
  NPCG_LAUNCH(ctx, scale_rows_kernel, static_cast<unsigned>(cdiv(p.ell * S, 256)), 256, 0, T.p(), p.ell, S, T.ld, g,
              gate);
  if (S <= 8) {
    rowdot(ctx, s.u.p(), s.u.ld, n, p.ell, T.p(), T.ld, static_cast<int>(S), V, ldv, out, ldo, gate);
  } else {
    DMat us;
    us.alloc(n, S, ctx.stream, false);
    gemm(ctx, n, S, p.ell, 1.0, Operand{s.u.p(), s.u.ld, false}, Operand{T.p(), T.ld, true}, 0.0, us.p(), us.ld);
    add2d(ctx, n, S, V, ldv, us.p(), us.ld, out, ldo);  // r + (U scaled)
  }
}
}  // namespace

void pre_apply_inverse(Pre& p, const double* R, i64 ldr, i64 S, double* Z, i64 ldz, const int* gate) {
  lowrank_update(p, p.gain_inv.p, R, ldr, S, Z, ldz, gate);
}
void pre_apply(Pre& p, const double* V, i64 ldv, i64 S, double* out, i64 ldo) {
  lowrank_update(p, p.gain_fwd.p, V, ldv, S, out, ldo, nullptr);
}

namespace {
__global__ void inv_shift_scale_kernel(const double* __restrict__ T, i64 ell, i64 S, i64 ldt,
                                       const double* __restrict__ lambda, double mu, double* __restrict__ core) {
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= ell * S) return;
  const i64 j = idx % ell, s = idx / ell;
  core[j + s * ldt] = __dmul_rn(__ddiv_rn(1.0, __dadd_rn(lambda[j], mu)), T[j + s * ldt]);
}
// X = W1 + (B - W2) / mu   (preconditioner.cpp:113, same association)
__global__ void woodbury_combine_kernel(i64 n, i64 S, const double* __restrict__ W1, i64 ldw,
                                        const double* __restrict__ W2, const double* __restrict__ B, i64 ldb,
                                        double mu, double* __restrict__ X, i64 ldx) {
  const i64 total = n * S;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, s = idx / n;
    X[i + s * ldx] = __dadd_rn(W1[i + s * ldw], __ddiv_rn(__dsub_rn(B[i + s * ldb], W2[i + s * ldw]), mu));
  }
}
}  // namespace

void woodbury_apply(Ctx& ctx, const Factors& f, i64 n, double mu, const double* B, i64 ldb, i64 S, double* X,
                    i64 ldx) {
  if (!(mu > 0.0)) invalid("woodbury_inverse_apply: mu must be > 0");
  if (S <= 0) return;
  const i64 ell = f.ell;
  DMat W1, W2;
  W1.alloc(n, S, ctx.stream, false);
  W2.alloc(n, S, ctx.stream, false);
  if (ell == 0) {  // b / mu
    NPCG_CUDA(cudaMemset2DAsync(W1.p(), W1.ld * 8, 0, n * 8, S, ctx.stream));
    NPCG_CUDA(cudaMemset2DAsync(W2.p(), W2.ld * 8, 0, n * 8, S, ctx.stream));
  } else {
    DMat T, core;
    T.alloc(ell, S, ctx.stream, false);
    core.alloc(ell, S, ctx.stream, false);
    gemm(ctx, ell, S, n, 1.0, Operand{f.u.p(), f.u.ld, true}, Operand{B, ldb, true}, 0.0, T.p(), T.ld);  // U^T b
    rows_allreduce(ctx, T.p(), T.ld * S);
    NPCG_LAUNCH(ctx, inv_shift_scale_kernel, static_cast<unsigned>(cdiv(ell * S, 256)), 256, 0, T.p(), ell, S, T.ld,
                f.lambda.p, mu, core.p());
    gemm(ctx, n, S, ell, 1.0, Operand{f.u.p(), f.u.ld, false}, Operand{core.p(), core.ld, true}, 0.0, W1.p(), W1.ld);
    gemm(ctx, n, S, ell, 1.0, Operand{f.u.p(), f.u.ld, false}, Operand{T.p(), T.ld, true}, 0.0, W2.p(), W2.ld);
  }
  NPCG_LAUNCH(ctx, woodbury_combine_kernel, static_cast<unsigned>(std::min<i64>(cdiv(n * S, 256), 4096)), 256, 0, n,
              S, W1.p(), W1.ld, W2.p(), B, ldb, mu, X, ldx);
}

}  // namespace npcg
