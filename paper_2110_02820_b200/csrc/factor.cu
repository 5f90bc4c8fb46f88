// Dense factorisations of the Nyström pipeline (see factor.cuh).
//
// Cholesky: right-looking, 64-wide blocks. The 64x64 diagonal block is
// factored and inverted by one CTA in shared memory; panel (A_ik L_kk^-T)
// and trailing update (A -= L_ik L_jk^T) are DMMA GEMMs (gemm.cu). The
// triangular solve on the right is blocked the same way, so every O(n l^2)
// flop of nystrom_from_sketch runs on the FP64 tensor pipe.
//
// SVD of the tall B: CholeskyQR2 (B = Q R, Gram matrices on DMMA, shifted
// CholeskyQR3 when the Gram Cholesky breaks down), then a one-sided Jacobi
// SVD of the l x l R^T in one cooperative kernel (round-robin pairs, one
// warp per pair, grid-wide barrier between rounds), then U = Q V on DMMA.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "blas.cuh"
#include "factor.cuh"
#include "gemm.cuh"

namespace cg = cooperative_groups;

namespace npcg {
namespace {

constexpr int NB = kCholNB;

__global__ void __launch_bounds__(256) chol_diag_kernel(double* a, i64 lda, i64 k0, int nb, double* dinv,
                                                        int* flag) {
  extern __shared__ double chol_smem[];
  double (*L)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(chol_smem);
  double (*X)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(chol_smem + NB * (NB + 1));
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    const int i = idx % NB, j = idx / NB;
    L[i][j] = (i < nb && j < nb && i >= j) ? a[(k0 + i) + (k0 + j) * lda] : 0.0;
    X[i][j] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double d = L[j][j];
      if (!(d > 0.0) || !isfinite(d)) bad = 1;
      else L[j][j] = sqrt(d);
    }
    __syncthreads();
    if (bad) break;
    const double piv = L[j][j];
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) L[i][j] /= piv;
    __syncthreads();
    const int m = nb - j - 1;
    for (int idx = tid; idx < m * m; idx += blockDim.x) {
      const int ii = idx % m, cc = idx / m;
      if (ii >= cc) L[j + 1 + ii][j + 1 + cc] -= L[j + 1 + ii][j] * L[j + 1 + cc][j];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) atomicOr(flag, 1);
    return;
  }
  // X = L^{-1} by forward substitution, one column per thread.
  if (tid < nb) {
    const int c = tid;
    X[c][c] = 1.0 / L[c][c];
    for (int i = c + 1; i < nb; ++i) {
      double s = 0.0;
      for (int k = c; k < i; ++k) s += L[i][k] * X[k][c];
      X[i][c] = -s / L[i][i];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    const int i = idx % NB, j = idx / NB;
    if (i < nb && j < nb) a[(k0 + i) + (k0 + j) * lda] = i >= j ? L[i][j] : 0.0;
    dinv[i + j * NB] = (i < nb && j < nb) ? X[i][j] : 0.0;
  }
}

__global__ void zero_upper_kernel(double* a, i64 n, i64 lda) {
  const i64 total = n * n;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    if (i < j) a[i + j * lda] = 0.0;
  }
}

__global__ void add_diag_kernel(double* a, i64 n, i64 lda, double s) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i + i * lda] += s;
}

// ---- one-sided Jacobi ----------------------------------------------------
__global__ void __launch_bounds__(256) jacobi_kernel(double* W, i64 ldw, double* V, i64 ldv, int n, double tol,
                                                     int max_sweeps, unsigned int* counters) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int N2 = n + (n & 1);
  const int half = N2 / 2;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    unsigned int* cnt = counters + (sweep & 1);
    for (int r = 0; r < N2 - 1; ++r) {
      for (int pi = gwarp; pi < half; pi += nwarps) {
        int p, q;
        if (pi == 0) {
          p = N2 - 1;
          q = r;
        } else {
          p = (r + pi) % (N2 - 1);
          q = (r - pi + N2 - 1) % (N2 - 1);
        }
        if (p >= n || q >= n) continue;
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        double* wp = W + static_cast<i64>(p) * ldw;
        double* wq = W + static_cast<i64>(q) * ldw;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double x = wp[i], y = wq[i];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al > 0.0 && be > 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < n; i += 32) {
            const double x = wp[i], y = wq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
          }
          double* vp = V + static_cast<i64>(p) * ldv;
          double* vq = V + static_cast<i64>(q) * ldv;
          for (int i = lane; i < n; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
          if (lane == 0) atomicAdd(cnt, 1u);
        }
      }
      grid.sync();
      if (r == 0 && blockIdx.x == 0 && threadIdx.x == 0) counters[(sweep + 1) & 1] = 0u;
    }
    grid.sync();
    if (*(volatile unsigned int*)cnt == 0u) break;
  }
}

__global__ void colnorm_kernel(const double* W, i64 ldw, int n, double* sigma) {
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gwarp >= n) return;
  const double* w = W + static_cast<i64>(gwarp) * ldw;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += w[i] * w[i];
  s = warp_sum(s);
  if (lane == 0) sigma[gwarp] = sqrt(s);
}

__global__ void rank_kernel(const double* sigma, int n, int* perm) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double sj = sigma[j];
  int rank = 0;
  for (int i = 0; i < n; ++i) {
    const double si = sigma[i];
    rank += (si > sj || (si == sj && i < j)) ? 1 : 0;
  }
  perm[rank] = j;
}

__global__ void gather_cols_kernel(const double* V, i64 ldv, int n, const int* perm, const double* sigma,
                                   double* Vs, i64 lds, double* sigma_s) {
  const int r = blockIdx.x;
  const int j = perm[r];
  for (int i = threadIdx.x; i < n; i += blockDim.x) Vs[i + static_cast<i64>(r) * lds] = V[i + static_cast<i64>(j) * ldv];
  if (threadIdx.x == 0) sigma_s[r] = sigma[j];
}

}  // namespace

bool cholesky(Ctx& ctx, double* a, i64 n, i64 lda, CholFactor& f) {
  f.n = n;
  if (n <= 0) return true;
  const i64 nblk = cdiv(n, NB);
  f.dinv.alloc(nblk * NB * NB, ctx.stream);
  DBuf<int> flag(1, ctx.stream);
  flag.zero();
  DMat panel;
  constexpr int kSmem = 2 * NB * (NB + 1) * 8;
  static bool attr_set = false;
  if (!attr_set) {
    NPCG_CUDA(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_set = true;
  }
  for (i64 b = 0; b < nblk; ++b) {
    const i64 k0 = b * NB, kb = std::min<i64>(NB, n - k0);
    NPCG_LAUNCH(ctx, chol_diag_kernel, 1, 256, kSmem, a, lda, k0, static_cast<int>(kb), f.dinv.p + b * NB * NB, flag.p);
    const i64 r0 = k0 + kb, m = n - r0;
    if (m <= 0) break;
    if (panel.rows != m) panel.alloc(m, NB, ctx.stream, false);
    copy2d(ctx, m, kb, a + r0 + k0 * lda, lda, panel.p(), panel.ld);
    // L_ik = A_ik * Dinv^T
    gemm(ctx, m, kb, kb, 1.0, Operand{panel.p(), panel.ld, false}, Operand{f.dinv.p + b * NB * NB, NB, false}, 0.0,
         a + r0 + k0 * lda, lda);
    // A[r0:, r0:] -= L_ik L_ik^T  (full square; only the lower part is used)
    gemm(ctx, m, m, kb, -1.0, Operand{a + r0 + k0 * lda, lda, false}, Operand{a + r0 + k0 * lda, lda, false}, 1.0,
         a + r0 + r0 * lda, lda);
  }
  NPCG_LAUNCH(ctx, zero_upper_kernel, static_cast<unsigned>(std::min<i64>(cdiv(n * n, 256), 4096)), 256, 0, a, n,
              lda);
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return h == 0;
}

void trsm_right_lt(Ctx& ctx, i64 m, i64 n, double* Y, i64 ldy, const double* L, i64 ldl, const CholFactor& f,
                   double* X, i64 ldx) {
  const i64 nblk = cdiv(n, NB);
  for (i64 b = 0; b < nblk; ++b) {
    const i64 k0 = b * NB, kb = std::min<i64>(NB, n - k0);
    gemm(ctx, m, kb, kb, 1.0, Operand{Y + k0 * ldy, ldy, false}, Operand{f.dinv.p + b * NB * NB, NB, false}, 0.0,
         X + k0 * ldx, ldx);
    const i64 r0 = k0 + kb, rem = n - r0;
    if (rem <= 0) break;
    gemm(ctx, m, rem, kb, -1.0, Operand{X + k0 * ldx, ldx, false}, Operand{L + r0 + k0 * ldl, ldl, false}, 1.0,
         Y + r0 * ldy, ldy);
  }
}

namespace {
// One CholeskyQR pass: Q = Y L^{-T} with L L^T = Y^T Y (+ shift I). `Y` is
// consumed. Returns false on Cholesky breakdown. L is left in `Lm`.
bool cholqr_pass(Ctx& ctx, double* Y, i64 ldy, i64 m, i64 n, double shift, DMat& Lm, double* Q, i64 ldq) {
  Lm.alloc(n, n, ctx.stream, false);
  gemm(ctx, n, n, m, 1.0, Operand{Y, ldy, true}, Operand{Y, ldy, true}, 0.0, Lm.p(), Lm.ld);
  if (shift > 0.0) NPCG_LAUNCH(ctx, add_diag_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, Lm.p(), n, Lm.ld, shift);
  CholFactor f;
  if (!cholesky(ctx, Lm.p(), n, Lm.ld, f)) return false;
  trsm_right_lt(ctx, m, n, Y, ldy, Lm.p(), Lm.ld, f, Q, ldq);
  return true;
}
}  // namespace

void orthonormalize(Ctx& ctx, const double* G_in, i64 ldg_in, i64 m, i64 n, double* Q, i64 ldq, double* Rt, i64 ldr) {
  if (n <= 0) return;
  // Scale by an exact power of two so max|G| ~ 1: the Gram G^T G neither
  // underflows (e.g. the nu-shifted zero matrix, whose B ~ sqrt(nu) ~ 1e-162)
  // nor overflows. Q is scale-invariant; R^T is scaled back exactly.
  const double amax = max_abs(ctx, G_in, m, n, ldg_in);
  int e2 = 0;
  if (amax > 0.0 && std::isfinite(amax)) std::frexp(amax, &e2);
  DMat scaled;
  const double* G = G_in;
  i64 ldg = ldg_in;
  if (e2 != 0) {
    scaled.alloc(m, n, ctx.stream, false);
    copy2d(ctx, m, n, G_in, ldg_in, scaled.p(), scaled.ld);
    scale_pow2(ctx, m, n, scaled.p(), scaled.ld, -e2);
    G = scaled.p();
    ldg = scaled.ld;
  }
  DMat work;
  work.alloc(m, n, ctx.stream, false);
  copy2d(ctx, m, n, G, ldg, work.p(), work.ld);
  DMat L1, L2, L3;
  int passes = 2;
  if (!cholqr_pass(ctx, work.p(), work.ld, m, n, 0.0, L1, Q, ldq)) {
    // Shifted CholeskyQR (Fukaya et al.): s = 11 (m n + n(n+1)) u ||G||_F^2.
    const double fro2 = sum_squares(ctx, G, m, n, ldg);
    const double s = 11.0 * (static_cast<double>(m) * n + static_cast<double>(n) * (n + 1)) * 2.220446049250313e-16 * fro2;
    copy2d(ctx, m, n, G, ldg, work.p(), work.ld);
    if (!cholqr_pass(ctx, work.p(), work.ld, m, n, s, L1, Q, ldq))
      fail(NPCG_ERUNTIME, "orthonormal_columns: shifted CholeskyQR broke down (rank-deficient input)");
    passes = 3;
  }
  // second (and third) pass on Q
  copy2d(ctx, m, n, Q, ldq, work.p(), work.ld);
  if (!cholqr_pass(ctx, work.p(), work.ld, m, n, 0.0, L2, Q, ldq))
    fail(NPCG_ERUNTIME, "orthonormal_columns: CholeskyQR2 second pass broke down");
  if (passes == 3) {
    copy2d(ctx, m, n, Q, ldq, work.p(), work.ld);
    if (!cholqr_pass(ctx, work.p(), work.ld, m, n, 0.0, L3, Q, ldq))
      fail(NPCG_ERUNTIME, "orthonormal_columns: CholeskyQR3 third pass broke down");
  }
  if (Rt) {  // R^T = L1 L2 (L3)
    if (passes == 2) {
      gemm(ctx, n, n, n, 1.0, Operand{L1.p(), L1.ld, false}, Operand{L2.p(), L2.ld, true}, 0.0, Rt, ldr);
    } else {
      DMat t;
      t.alloc(n, n, ctx.stream, false);
      gemm(ctx, n, n, n, 1.0, Operand{L1.p(), L1.ld, false}, Operand{L2.p(), L2.ld, true}, 0.0, t.p(), t.ld);
      gemm(ctx, n, n, n, 1.0, Operand{t.p(), t.ld, false}, Operand{L3.p(), L3.ld, true}, 0.0, Rt, ldr);
    }
    if (e2 != 0) scale_pow2(ctx, n, n, Rt, ldr, e2);
  }
}

void jacobi_svd_small(Ctx& ctx, double* W, i64 ldw, i64 n, double* Vs, i64 ldv, double* sigma) {
  if (n <= 0) return;
  DMat V;
  V.alloc(n, n, ctx.stream, false);
  set_identity(ctx, V.p(), n, n, V.ld);
  DBuf<unsigned int> counters(2, ctx.stream);
  counters.zero();
  int nn = static_cast<int>(n);
  double tol = 2.220446049250313e-16 * std::sqrt(static_cast<double>(n));
  int max_sweeps = 60;
  int per_sm = 0;
  NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, 256, 0));
  const int want = static_cast<int>(cdiv((n + 1) / 2, 8));
  const int grid = std::max(1, std::min(want, per_sm * ctx.sm_count));
  double* Wp = W;
  double* Vp = V.p();
  i64 ldvv = V.ld;
  unsigned int* cp = counters.p;
  void* args[] = {&Wp, &ldw, &Vp, &ldvv, &nn, &tol, &max_sweeps, &cp};
  ctx.prof_begin("jacobi_kernel");
  NPCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_kernel), grid, 256, args, 0, ctx.stream));
  ctx.check_launch("jacobi_kernel");
  ctx.prof_end();
  DBuf<double> sig(n, ctx.stream);
  DBuf<int> perm(n, ctx.stream);
  NPCG_LAUNCH(ctx, colnorm_kernel, static_cast<unsigned>(cdiv(n * 32, 256)), 256, 0, W, ldw, nn, sig.p);
  NPCG_LAUNCH(ctx, rank_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, sig.p, nn, perm.p);
  NPCG_LAUNCH(ctx, gather_cols_kernel, static_cast<unsigned>(n), 128, 0, V.p(), V.ld, nn, perm.p, sig.p, Vs, ldv,
              sigma);
}

void thin_svd(Ctx& ctx, const double* B, i64 ldb, i64 m, i64 n, double* U, i64 ldu, double* sigma) {
  if (m < n) invalid("thin_svd: expected a tall (m >= n) matrix");
  if (n <= 0) return;
  DMat Q, Rt, Vs;
  Q.alloc(m, n, ctx.stream, false);
  Rt.alloc(n, n, ctx.stream, false);
  Vs.alloc(n, n, ctx.stream, false);
  orthonormalize(ctx, B, ldb, m, n, Q.p(), Q.ld, Rt.p(), Rt.ld);
  jacobi_svd_small(ctx, Rt.p(), Rt.ld, n, Vs.p(), Vs.ld, sigma);
  gemm(ctx, m, n, n, 1.0, Operand{Q.p(), Q.ld, false}, Operand{Vs.p(), Vs.ld, true}, 0.0, U, ldu);
}

}  // namespace npcg
