// O'Leary block PCG (block_nystrom_pcg, solvers.cpp:150-279) on device.
//
//   B P = Q R     column-pivoted Householder QR of the n x s right-hand block
//                 (one CTA; s is a handful of columns), rank by |R_ii| >
//                 1e-12 |R_00|, deflated columns recorded.
//   then the block recurrence on the rank retained directions:
//     V = A_mu P, alpha = (P^T V)^-1 (Z^T R), X += P alpha, R -= V alpha,
//     Z = P^-1 R, beta = (Z^T R)_old^-1 (Z^T R)_new, P = Z + P beta,
//   with the k x k solves by Cholesky on device and the reference's damped
//   pseudo-inverse fallback (10 ulps of the Frobenius norm) when it fails.
// Every n-length product is a coldot/rowdot skinny kernel or a DMMA GEMM; the
// k x k algebra runs in single-CTA kernels; the host only reads the per-
// iteration residual norms to decide convergence, as the reference does.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <vector>

#include "blas.cuh"
#include "gemm.cuh"
#include "pcg.cuh"

namespace npcg {
namespace {

constexpr int KMAX = 32;

// Column-pivoted Householder QR in place on A (n x s, ld lda). Outputs tau,
// jpvt (original column index per position), and R stays in the upper
// triangle of A (Householder vectors below, v_0 = 1 implicit).
__global__ void __launch_bounds__(1024) colpiv_qr_kernel(double* A, i64 lda, i64 n, int s, double* tau, int* jpvt) {
  __shared__ double sh[32];
  __shared__ double norms[KMAX];
  __shared__ int perm[KMAX];
  __shared__ double s_beta, s_tau, s_scale;
  const int tid = threadIdx.x;
  if (tid < s) perm[tid] = tid;
  __syncthreads();
  const int kmin = static_cast<int>(n < s ? n : static_cast<i64>(s));
  for (int i = 0; i < kmin; ++i) {
    // remaining column norms (rows i..n-1), exact each step
    for (int j = i; j < s; ++j) {
      double acc = 0.0;
      const double* col = A + static_cast<i64>(j) * lda;
      for (i64 r = i + tid; r < n; r += blockDim.x) acc += col[r] * col[r];
      acc = block_sum(acc, sh);
      if (tid == 0) norms[j] = acc;
      __syncthreads();
    }
    if (tid == 0) {  // first maximal remaining column (Eigen maxCoeff)
      int best = i;
      for (int j = i + 1; j < s; ++j)
        if (norms[j] > norms[best]) best = j;
      if (best != i) {
        const int t = perm[i];
        perm[i] = perm[best];
        perm[best] = t;
        norms[best] = norms[i];
      }
      s_scale = static_cast<double>(best);
    }
    __syncthreads();
    const int best = static_cast<int>(s_scale);
    if (best != i) {  // swap full columns
      double* ci = A + static_cast<i64>(i) * lda;
      double* cb = A + static_cast<i64>(best) * lda;
      for (i64 r = tid; r < n; r += blockDim.x) {
        const double t = ci[r];
        ci[r] = cb[r];
        cb[r] = t;
      }
    }
    __syncthreads();
    // Householder for column i rows i..n-1
    double* ci = A + static_cast<i64>(i) * lda;
    double tail = 0.0;
    for (i64 r = i + 1 + tid; r < n; r += blockDim.x) tail += ci[r] * ci[r];
    tail = block_sum(tail, sh);
    if (tid == 0) {
      const double alpha = ci[i];
      if (tail == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scale = 0.0;
      } else {
        const double beta = -copysign(sqrt(alpha * alpha + tail), alpha);
        s_tau = (beta - alpha) / beta;
        s_beta = beta;
        s_scale = 1.0 / (alpha - beta);
      }
      tau[i] = s_tau;
    }
    __syncthreads();
    const double t = s_tau, sc = s_scale;
    for (i64 r = i + 1 + tid; r < n; r += blockDim.x) ci[r] *= sc;
    __syncthreads();
    if (tid == 0) ci[i] = s_beta;
    // apply H = I - t v v^T to columns j > i
    for (int j = i + 1; j < s && t != 0.0; ++j) {
      double* cj = A + static_cast<i64>(j) * lda;
      double w = 0.0;
      for (i64 r = i + tid; r < n; r += blockDim.x) w += (r == i ? 1.0 : ci[r]) * cj[r];
      w = block_sum(w, sh);
      for (i64 r = i + tid; r < n; r += blockDim.x) cj[r] -= t * w * (r == i ? 1.0 : ci[r]);
      __syncthreads();
    }
    __syncthreads();
  }
  if (tid < s) jpvt[tid] = perm[tid];
}

// Q(:, 0:rank) = H_0 ... H_{rank-1} [I; 0], one CTA per column.
__global__ void form_q_kernel(const double* A, i64 lda, i64 n, int rank, const double* tau, double* Q, i64 ldq) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double* q = Q + static_cast<i64>(c) * ldq;
  for (i64 r = threadIdx.x; r < n; r += blockDim.x) q[r] = r == c ? 1.0 : 0.0;
  __syncthreads();
  for (int k = rank - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t == 0.0) continue;
    const double* v = A + static_cast<i64>(k) * lda;
    double w = 0.0;
    for (i64 r = k + threadIdx.x; r < n; r += blockDim.x) w += (r == k ? 1.0 : v[r]) * q[r];
    w = block_sum(w, sh);
    for (i64 r = k + threadIdx.x; r < n; r += blockDim.x) q[r] -= t * w * (r == k ? 1.0 : v[r]);
    __syncthreads();
  }
}

// Cholesky solve of the k x k SPD system A X = B (B k x m), LLT on the lower
// triangle (Eigen::LLT); on failure the damped pseudo-inverse
// (A + 10 ulp(||A||_F) I)^+ B via a Jacobi eigendecomposition. One thread.
__global__ void small_solve_kernel(const double* A, i64 lda, int k, const double* B, i64 ldb, int m, double* X,
                                   i64 ldx, int* fallback) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double L[KMAX][KMAX];
  bool ok = true;
  for (int j = 0; j < k && ok; ++j) {
    for (int i = j; i < k; ++i) {
      double s = A[i + j * lda];
      for (int p = 0; p < j; ++p) s -= L[i][p] * L[j][p];
      if (i == j) {
        if (!(s > 0.0) || !isfinite(s)) {
          ok = false;
          break;
        }
        L[j][j] = sqrt(s);
      } else {
        L[i][j] = s / L[j][j];
      }
    }
  }
  if (ok) {
    for (int c = 0; c < m; ++c) {
      double y[KMAX];
      for (int i = 0; i < k; ++i) {
        double s = B[i + c * ldb];
        for (int p = 0; p < i; ++p) s -= L[i][p] * y[p];
        y[i] = s / L[i][i];
      }
      for (int i = k - 1; i >= 0; --i) {
        double s = y[i];
        for (int p = i + 1; p < k; ++p) s -= L[p][i] * X[p + c * ldx];
        X[i + c * ldx] = s / L[i][i];
      }
    }
    *fallback = 0;
    return;
  }
  *fallback = 1;
  double M[KMAX][KMAX], Vv[KMAX][KMAX];
  double fro = 0.0;
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) {
      const double a = 0.5 * (A[i + j * lda] + A[j + i * lda]);
      M[i][j] = a;
      fro += A[i + j * lda] * A[i + j * lda];
      Vv[i][j] = i == j ? 1.0 : 0.0;
    }
  fro = sqrt(fro);
  const double ulp = nextafter(fro, INFINITY) - fro;
  for (int i = 0; i < k; ++i) M[i][i] += 10.0 * ulp;
  for (int sweep = 0; sweep < 60; ++sweep) {  // cyclic Jacobi
    double off = 0.0;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) off += M[p][q] * M[p][q];
    if (off <= 1e-30 * fro * fro + 1e-300) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        if (M[p][q] == 0.0) continue;
        const double th = (M[q][q] - M[p][p]) / (2.0 * M[p][q]);
        const double t = copysign(1.0, th) / (fabs(th) + sqrt(1.0 + th * th));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < k; ++r) {
          const double mp = M[r][p], mq = M[r][q];
          M[r][p] = c * mp - sn * mq;
          M[r][q] = sn * mp + c * mq;
        }
        for (int r = 0; r < k; ++r) {
          const double mp = M[p][r], mq = M[q][r];
          M[p][r] = c * mp - sn * mq;
          M[q][r] = sn * mp + c * mq;
        }
        for (int r = 0; r < k; ++r) {
          const double vp = Vv[r][p], vq = Vv[r][q];
          Vv[r][p] = c * vp - sn * vq;
          Vv[r][q] = sn * vp + c * vq;
        }
      }
  }
  double emax = 0.0;
  for (int i = 0; i < k; ++i) emax = fmax(emax, fabs(M[i][i]));
  const double thr = 2.220446049250313e-16 * k * emax;
  for (int c = 0; c < m; ++c) {
    double t[KMAX];
    for (int i = 0; i < k; ++i) {
      double s = 0.0;
      for (int r = 0; r < k; ++r) s += Vv[r][i] * B[r + c * ldb];
      t[i] = fabs(M[i][i]) > thr ? s / M[i][i] : 0.0;
    }
    for (int r = 0; r < k; ++r) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += Vv[r][i] * t[i];
      X[r + c * ldx] = s;
    }
  }
}

// squared column norms (the square root is taken on the host after the
// row-sharded all-reduce; sqrt is correctly rounded on both sides)
__global__ void colnorms_kernel(const double* A, i64 lda, i64 n, int s, double* out) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (i64 r = threadIdx.x; r < n; r += blockDim.x) acc += A[r + c * lda] * A[r + c * lda];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) out[c] = acc;
}

__global__ void negate_kernel(const double* a, i64 lda, int rows, int cols, double* out, i64 ldo) {
  const int i = threadIdx.x, j = blockIdx.x;
  if (i < rows && j < cols) out[i + j * ldo] = -a[i + j * lda];
}

}  // namespace

BlockPcgResult block_pcg_solve(Ctx& ctx, Op& op, Pre* pre, double mu, i64 s, const double* B, i64 ldb,
                               const PcgOptions& opt, double* X, i64 ldx) {
  using Clock = std::chrono::steady_clock;
  const auto t0 = Clock::now();
  // Sharded: B, X and every n x k block are this rank's rows; the k x k Grams
  // and column norms are all-reduced, and the one upfront QR of B runs
  // replicated on the all-gathered B (s is a handful of columns).
  const i64 n = op.nloc, nfull = op.n;
  BlockPcgResult res;
  res.converged.assign(static_cast<size_t>(s), false);
  res.history.assign(static_cast<size_t>(s), {});
  if (s > KMAX) fail(NPCG_EINVAL, "block_nystrom_pcg: at most 32 right-hand sides per block");
  if (!all_finite_rows(ctx, B, n, s, ldb)) invalid("block_nystrom_pcg: right-hand side has non-finite entries");
  std::vector<double> thr(static_cast<size_t>(s));
  DBuf<double> nrm(s, ctx.stream);
  auto colnorms = [&](const double* A, i64 lda, std::vector<double>& outv) {
    NPCG_LAUNCH(ctx, colnorms_kernel, static_cast<unsigned>(s), 256, 0, A, lda, n, static_cast<int>(s), nrm.p);
    rows_allreduce(ctx, nrm.p, s);
    NPCG_CUDA(cudaMemcpyAsync(outv.data(), nrm.p, sizeof(double) * s, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    for (auto& v : outv) v = std::sqrt(v);
  };
  std::vector<double> bnorm(static_cast<size_t>(s));
  colnorms(B, ldb, bnorm);
  for (i64 j = 0; j < s; ++j) thr[j] = opt.relative ? opt.eta * bnorm[j] : opt.eta;
  res.eta_used = opt.eta;

  // ---- column-pivoted QR of B
  DMat Aq;
  Aq.alloc(nfull, s, ctx.stream, false);
  rows_allgather(ctx, ctx.split(nfull), B, ldb, s, Aq.p(), Aq.ld);
  DBuf<double> tau(s, ctx.stream);
  DBuf<int> jp(s, ctx.stream);
  NPCG_LAUNCH(ctx, colpiv_qr_kernel, 1, 1024, 0, Aq.p(), Aq.ld, nfull, static_cast<int>(s), tau.p, jp.p);
  std::vector<double> hq(static_cast<size_t>(s * s));
  std::vector<int> jpvt(static_cast<size_t>(s));
  download(ctx, Aq.p(), Aq.ld, std::min<i64>(nfull, s), s, hq.data(), s, NPCG_HOST);
  NPCG_CUDA(cudaMemcpy(jpvt.data(), jp.p, sizeof(int) * s, cudaMemcpyDeviceToHost));
  const i64 kmin = std::min<i64>(nfull, s);
  const double pivot_max = std::abs(hq[0]);
  i64 rank = 0;
  for (i64 i = 0; i < kmin; ++i)
    if (std::abs(hq[i + i * s]) > 1e-12 * pivot_max) ++rank;
  for (i64 i = rank; i < s; ++i) res.deflated.push_back(jpvt[i]);
  std::sort(res.deflated.begin(), res.deflated.end());
  if (rank == 0) {  // solvers.cpp:199-209
    NPCG_CUDA(cudaMemset2DAsync(X, ldx * 8, 0, n * 8, s, ctx.stream));
    for (i64 j = 0; j < s; ++j) {
      res.history[j].push_back(bnorm[j]);
      res.converged[j] = bnorm[j] <= thr[j];
    }
    ctx.sync();
    res.wall_time = std::chrono::duration<double>(Clock::now() - t0).count();
    return res;
  }
  DMat Qr, mix, negmix, defl;
  {
    DMat Qf;  // Q_r over all n rows (replicated), then this rank's rows
    Qf.alloc(nfull, rank, ctx.stream, false);
    NPCG_LAUNCH(ctx, form_q_kernel, static_cast<unsigned>(rank), 256, 0, Aq.p(), Aq.ld, nfull, static_cast<int>(rank),
                tau.p, Qf.p(), Qf.ld);
    Qr.alloc(n, rank, ctx.stream, false);
    copy2d(ctx, n, rank, Qf.p() + op.off, Qf.ld, Qr.p(), Qr.ld);
    ctx.sync();
  }
  std::vector<double> hmix(static_cast<size_t>(rank * s), 0.0);  // R[0:rank, :] P^T (solvers.cpp:203-208)
  for (i64 k = 0; k < s; ++k)
    for (i64 i = 0; i < rank && i <= k; ++i) hmix[i + jpvt[k] * rank] = hq[i + k * s];
  mix.alloc(rank, s, ctx.stream, false);
  upload(ctx, mix, rank, s, hmix.data(), rank, NPCG_HOST);
  negmix.alloc(rank, s, ctx.stream, false);
  NPCG_LAUNCH(ctx, negate_kernel, static_cast<unsigned>(s), 32, 0, mix.p(), mix.ld, static_cast<int>(rank),
              static_cast<int>(s), negmix.p(), negmix.ld);
  defl.alloc(n, s, ctx.stream, false);  // B - Q_r mix
  rowdot(ctx, Qr.p(), Qr.ld, n, rank, negmix.p(), negmix.ld, static_cast<int>(s), B, ldb, defl.p(), defl.ld);

  const int k = static_cast<int>(rank);
  DMat Xt, R, Z, P, V, ZR, ZRn, G, alpha, beta, negalpha, orig;
  Xt.alloc(n, k, ctx.stream, true);
  R.alloc(n, k, ctx.stream, false);
  copy2d(ctx, n, k, Qr.p(), Qr.ld, R.p(), R.ld);
  Z.alloc(n, k, ctx.stream, false);
  P.alloc(n, k, ctx.stream, false);
  V.alloc(n, k, ctx.stream, false);
  ZR.alloc(k, k, ctx.stream, false);
  ZRn.alloc(k, k, ctx.stream, false);
  G.alloc(k, k, ctx.stream, false);
  alpha.alloc(k, k, ctx.stream, false);
  beta.alloc(k, k, ctx.stream, false);
  negalpha.alloc(k, k, ctx.stream, false);
  orig.alloc(n, s, ctx.stream, false);
  DBuf<int> fb(1, ctx.stream);
  auto precond = [&](const double* in, i64 ldi, double* out, i64 ldo) {
    if (pre && pre->ell > 0) pre_apply_inverse(*pre, in, ldi, k, out, ldo);
    else copy2d(ctx, n, k, in, ldi, out, ldo);
  };
  auto gram = [&](const double* a, i64 lda, const double* b, i64 ldbb, double* out, i64 ldo) {  // a^T b
    gemm(ctx, k, k, n, 1.0, Operand{a, lda, true}, Operand{b, ldbb, true}, 0.0, out, ldo);
    rows_allreduce(ctx, out, ldo * k);
  };
  auto solve = [&](const DMat& A, const DMat& rhs, DMat& out) {
    NPCG_LAUNCH(ctx, small_solve_kernel, 1, 32, 0, A.p(), A.ld, k, rhs.p(), rhs.ld, k, out.p(), out.ld, fb.p);
    int h = 0;
    NPCG_CUDA(cudaMemcpyAsync(&h, fb.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    res.fallback_count += h;
  };
  std::vector<double> hres(static_cast<size_t>(s));
  auto record = [&]() -> bool {  // solvers.cpp:225-237
    rowdot(ctx, R.p(), R.ld, n, k, mix.p(), mix.ld, static_cast<int>(s), defl.p(), defl.ld, orig.p(), orig.ld);
    colnorms(orig.p(), orig.ld, hres);
    bool all = true;
    for (i64 j = 0; j < s; ++j) {
      if (!std::isfinite(hres[j])) fail(NPCG_ERUNTIME, "block_nystrom_pcg: non-finite residual");
      res.history[j].push_back(hres[j]);
      res.converged[j] = hres[j] <= thr[j];
      all = all && res.converged[j];
    }
    return all;
  };
  precond(R.p(), R.ld, Z.p(), Z.ld);
  copy2d(ctx, n, k, Z.p(), Z.ld, P.p(), P.ld);
  gram(Z.p(), Z.ld, R.p(), R.ld, ZR.p(), ZR.ld);
  bool done = record();
  for (i64 t = 1; t <= opt.max_iter && !done; ++t) {
    res.iterations = t;
    op.apply_shift(P.p(), P.ld, k, mu, V.p(), V.ld, nullptr);
    gram(P.p(), P.ld, V.p(), V.ld, G.p(), G.ld);
    solve(G, ZR, alpha);
    rowdot(ctx, P.p(), P.ld, n, k, alpha.p(), alpha.ld, k, Xt.p(), Xt.ld, Xt.p(), Xt.ld);  // X += P alpha
    NPCG_LAUNCH(ctx, negate_kernel, static_cast<unsigned>(k), 32, 0, alpha.p(), alpha.ld, k, k, negalpha.p(),
                negalpha.ld);
    rowdot(ctx, V.p(), V.ld, n, k, negalpha.p(), negalpha.ld, k, R.p(), R.ld, R.p(), R.ld);  // R -= V alpha
    done = record();
    if (done) break;
    precond(R.p(), R.ld, Z.p(), Z.ld);
    gram(Z.p(), Z.ld, R.p(), R.ld, ZRn.p(), ZRn.ld);
    solve(ZR, ZRn, beta);
    rowdot(ctx, P.p(), P.ld, n, k, beta.p(), beta.ld, k, Z.p(), Z.ld, V.p(), V.ld);  // V <- Z + P beta
    copy2d(ctx, n, k, V.p(), V.ld, P.p(), P.ld);
    copy2d(ctx, k, k, ZRn.p(), ZRn.ld, ZR.p(), ZR.ld);
  }
  rowdot(ctx, Xt.p(), Xt.ld, n, k, mix.p(), mix.ld, static_cast<int>(s), nullptr, 0, X, ldx);  // X = X~ mix
  ctx.sync();
  res.wall_time = std::chrono::duration<double>(Clock::now() - t0).count();
  return res;
}

}  // namespace npcg
