// Dense FP64 factorisations of the Nyström pipeline, on device:
// blocked Cholesky (lower, LLT semantics), blocked right triangular solve,
// CholeskyQR2 (shifted CholeskyQR3 fallback) and a one-sided Jacobi SVD.
#pragma once

#include "context.cuh"

namespace npcg {

constexpr int kCholNB = 64;

/// What cholesky() leaves besides L: the diagonal-block inverses (block b,
/// rows/cols b*nb.., stored nb x nb col-major at dinv + b*nb*nb) and, from
/// the fused path (n <= kCholFusedMax), the full inverse L^{-1} in `linv`.
struct CholFactor {
  DBuf<double> dinv;
  DMat linv;
  i64 n = 0;
  int nb = kCholNB;
};

constexpr i64 kCholFusedMax = 4096;

/// Fused single-launch Cholesky + L^{-1} (chol.cu); same contract as cholesky().
bool cholesky_fused(Ctx& ctx, double* a, i64 n, i64 lda, CholFactor& f);

/// In-place lower Cholesky of the n x n matrix at `a` (ld lda), reading only
/// the lower triangle (Eigen::LLT / dpotrf('L') semantics). On return the
/// lower triangle holds L and the strict upper triangle is zero. Returns
/// false when a pivot is <= 0 or non-finite (synchronises).
bool cholesky(Ctx& ctx, double* a, i64 n, i64 lda, CholFactor& f);

/// X (m x n) = Y * L^{-T} for the lower factor L of `f` (X L^T = Y;
/// Eigen `llt.matrixU().solve<OnTheRight>(Y)`). Y is used as workspace and
/// overwritten. X must not alias Y.
void trsm_right_lt(Ctx& ctx, i64 m, i64 n, double* Y, i64 ldy, const double* L, i64 ldl, const CholFactor& f,
                   double* X, i64 ldx);

/// Orthonormal basis Q (m x n) of range(G) (m >= n, full column rank),
/// by CholeskyQR2 with a shifted CholeskyQR3 fallback. If R != nullptr the
/// upper-triangular factor (G = Q R) is written there (n x n, ld ldr).
/// `dist`: G's rows are this rank's block of a row-sharded matrix (the Grams
/// and norms are all-reduced; R is replicated, Q keeps the local rows).
void orthonormalize(Ctx& ctx, const double* G, i64 ldg, i64 m, i64 n, double* Q, i64 ldq,
                    double* R = nullptr, i64 ldr = 0, bool dist = false);

/// max_ij |G_ij - delta_ij| of an n x n matrix (synchronises the stream).
double identity_deviation(Ctx& ctx, const double* G, i64 ldg, i64 n);

/// orthonormalize() that reports a CholeskyQR breakdown instead of throwing.
bool try_orthonormalize(Ctx& ctx, const double* G, i64 ldg, i64 m, i64 n, double* Q, i64 ldq);

/// Thin SVD of a tall matrix (dgesdd('S') equivalent up to column signs):
/// U (m x n) left singular vectors, sigma (n) descending, on device.
void thin_svd(Ctx& ctx, const double* B, i64 ldb, i64 m, i64 n, double* U, i64 ldu, double* sigma,
              bool dist = false);

/// One-sided Jacobi on the n x n matrix W (ld ldw, overwritten): finds an
/// orthogonal V with W V orthogonal columns. sigma(j) = ||(W V)(:,j)||,
/// columns of V and sigma sorted descending into Vs / sigma.
void jacobi_svd_small(Ctx& ctx, double* W, i64 ldw, i64 n, double* Vs, i64 ldv, double* sigma);

/// Same contract via the symmetric eigenvectors of W^T W (eig.cu) and
/// sigma_j = ||(W V)(:, j)||. The default path (NPCG_SVD=jacobi selects the
/// one-sided Jacobi instead).
void small_svd_eig(Ctx& ctx, double* W, i64 ldw, i64 n, double* Vs, i64 ldv, double* sigma);

}  // namespace npcg
