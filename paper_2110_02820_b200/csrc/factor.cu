// Dense factorisations of the Nyström pipeline (see factor.cuh).
//
// Cholesky: right-looking, 64-wide blocks. The 64x64 diagonal block is
// factored and inverted by one CTA in shared memory; panel (A_ik L_kk^-T)
// and trailing update (A -= L_ik L_jk^T) are DMMA GEMMs (gemm.cu). The
// triangular solve on the right is blocked the same way, so every O(n l^2)
// flop of nystrom_from_sketch runs on the FP64 tensor pipe.
//
// SVD of the tall B: CholeskyQR2 (B = Q R, Gram matrices on DMMA, shifted
// CholeskyQR3 when the Gram Cholesky breaks down; a re-orthogonalisation pass
// is skipped when Q^T Q is already I to 1e-14), then the SVD of the l x l R^T
// (small_svd_eig: tridiagonal eigenvectors of R R^T + Jacobi refinement, or a
// one-CTA one-sided Jacobi for l <= 110), then U = Q V on DMMA.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <string>

#include "blas.cuh"
#include "eig.cuh"
#include "factor.cuh"
#include "gemm.cuh"
#include "ozaki.cuh"

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
  // Right-looking: every thread reads the pivot and takes its square root
  // itself (no single-thread step), scales its share of column j, then the
  // trailing lower triangle is updated. Two barriers per column. A pivot that
  // is <= 0 or not finite is seen by all threads at once (uniform exit).
  for (int j = 0; j < nb; ++j) {
    const double dj = L[j][j];
    if (!(dj > 0.0) || !isfinite(dj)) {
      if (tid == 0) bad = 1;
      break;
    }
    const double piv = sqrt(dj);
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) L[i][j] /= piv;
    __syncthreads();
    if (tid == 0) L[j][j] = piv;
    {  // trailing lower triangle, 16 x 16 thread tile (no div/mod in the loop)
      const int ty = tid >> 4, tx = tid & 15;
      for (int i = j + 1 + ty; i < nb; i += 16) {
        const double lij = L[i][j];
        for (int c = j + 1 + tx; c <= i; c += 16) L[i][c] -= lij * L[c][j];
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) atomicOr(flag, 1);
    return;
  }
  // X = L^{-1}, row by row: X[i][c] = (delta_ic - sum_{k<i} L[i][k] X[k][c]) / L[i][i],
  // four threads per column c split the k-sum (shuffle-combined).
  {
    const int c = tid >> 2, part = tid & 3;
    for (int i = 0; i < nb; ++i) {
      double s = 0.0;
      if (c < i)
        for (int k = c + part; k < i; k += 4) s += L[i][k] * X[k][c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (part == 0 && c <= i) X[i][c] = ((c == i ? 1.0 : 0.0) - s) / L[i][i];
      __syncthreads();
    }
  }
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

// C_ij = G_ij / (G_jj - G_ii) (skew), zero when the pair is too close for a
// first-order step (|G_ij| > 0.1 |G_jj - G_ii|). One warp per column j also
// predicts the column-norm error of j, sum_i min(G_ij^2/|G_jj - G_ii|, |G_ij|)
// relative to G_jj, and max-reduces it into *qual.
__global__ void refine_angles_kernel(const double* G, i64 ldg, i64 n, double* C, i64 ldc, double* qual) {
  const i64 j = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double gjj = G[j + j * ldg];
  double err = 0.0;
  for (i64 i = lane; i < n; i += 32) {
    double c = 0.0;
    if (i != j) {
      const double gij = 0.5 * (G[i + j * ldg] + G[j + i * ldg]);
      const double den = gjj - G[i + i * ldg];
      if (fabs(gij) <= 0.1 * fabs(den)) c = gij / den;
      err += fabs(den) > 0.0 ? fmin(gij * gij / fabs(den), fabs(gij)) : fabs(gij);
    }
    C[i + j * ldc] = c;
  }
  err = warp_sum(err);
  if (lane == 0) {
    const double rel = gjj > 0.0 ? err / gjj : (err > 0.0 ? 1.0 : 0.0);
    atomicMax(reinterpret_cast<unsigned long long*>(qual), static_cast<unsigned long long>(__double_as_longlong(rel)));
  }
}

__global__ void identity_dev_kernel(const double* G, i64 ldg, i64 n, double* out) {
  const i64 total = n * n;
  double m = 0.0;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    const double d = fabs(G[i + j * ldg] - (i == j ? 1.0 : 0.0));
    m = isnan(d) ? 1e308 : fmax(m, d);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out), static_cast<unsigned long long>(__double_as_longlong(m)));
}

__global__ void add_diag_kernel(double* a, i64 n, i64 lda, double s) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i + i * lda] += s;
}

// ---- block one-sided Jacobi ---------------------------------------------
// Columns are grouped in blocks of b; blocks are paired round-robin and one
// CTA owns a pair S (m = 2b columns). The CTA stages W_S (all n rows) in
// shared memory and runs one-sided Jacobi sweeps on it there (one warp per
// column pair, rotations from direct column dot products, __syncthreads
// between rounds), accumulating the rotations in an m x m J; then writes W_S
// back and applies V_S <- V_S J. A grid-wide barrier separates rounds of
// disjoint block pairs; a sweep without rotations ends the iteration. With a
// single pair (m >= n) the whole problem lives in one CTA.
__device__ __forceinline__ void rr_pair(int k, int r, int N, int& p, int& q) {
  if (k == 0) {
    p = N - 1;
    q = r;
  } else {
    p = (r + k) % (N - 1);
    q = (r - k + N - 1) % (N - 1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

constexpr int JOS_THREADS = 512;
constexpr int JOS_MAXM = 160;
constexpr double tol_conv = 1e-12;  // relative column non-orthogonality that ends the sweeps

// Jacobi rotation zeroing ga = w_p.w_q (al = |w_p|^2, be = |w_q|^2). The
// angle only has to be good, not exact: t is formed in FP32 when the inputs
// fit its range, and (c, s) are then normalised in FP64 by Newton steps on
// rsqrt, so c^2 + s^2 = 1 to FP64 rounding and the accumulated V stays
// orthogonal. This keeps the FP64 sqrt/div latency chains off the critical
// path of every round.
__device__ __forceinline__ void rotation(double al, double be, double ga, double& c, double& s) {
  const double zeta = (be - al) * 0.5;  // zeta * ga
  double t;
  const double az = fabs(zeta), ag = fabs(ga);
  if (az < 1e30 && ag < 1e30 && ag > 1e-30 && az > 1e-30) {
    const float zf = static_cast<float>(zeta) / static_cast<float>(ga);
    const float tf = copysignf(1.0f, zf) / (fabsf(zf) + sqrtf(1.0f + zf * zf));
    t = static_cast<double>(tf);
  } else {
    const double z = zeta / ga;
    t = copysign(1.0, z) / (fabs(z) + sqrt(1.0 + z * z));
  }
  const double u = 1.0 + t * t;
  double r = static_cast<double>(rsqrtf(static_cast<float>(u)));
  r = r * (1.5 - 0.5 * u * r * r);
  r = r * (1.5 - 0.5 * u * r * r);
  r = r * (1.5 - 0.5 * u * r * r);
  c = r;
  s = r * t;
}

__global__ void __launch_bounds__(JOS_THREADS) jacobi_os_kernel(double* W, i64 ldw, double* V, i64 ldv, int n, int b,
                                                                int nbp, double tol, int max_sweeps, int inner_sweeps,
                                                                unsigned int* counters) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double jos_smem[];
  __shared__ int cols[JOS_MAXM];
  __shared__ int s_m, s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int nld = n + (n & 1);  // smem column stride
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    unsigned int* cnt = counters + (sweep & 1);
    for (int r = 0; r < nbp - 1; ++r) {
      for (int pi = blockIdx.x; pi < nbp / 2; pi += gridDim.x) {
        int P, Q;
        rr_pair(pi, r, nbp, P, Q);
        __syncthreads();
        if (tid == 0) {
          int m = 0;
          for (int k = 0; k < b; ++k)
            if (P * b + k < n) cols[m++] = P * b + k;
          for (int k = 0; k < b; ++k)
            if (Q * b + k < n) cols[m++] = Q * b + k;
          s_m = m;
        }
        __syncthreads();
        const int m = s_m;
        if (m < 2) continue;
        double* Ws = jos_smem;                    // m columns x nld
        double* Js = jos_smem + m * nld;          // m x m, column-major
        for (int idx = tid; idx < m * n; idx += blockDim.x) {
          const int k = idx / n, i = idx % n;
          Ws[k * nld + i] = W[i + static_cast<i64>(cols[k]) * ldw];
        }
        for (int idx = tid; idx < m * m; idx += blockDim.x) Js[idx] = (idx % m == idx / m) ? 1.0 : 0.0;
        const int m2 = m + (m & 1);
        int any = 0;
        for (int isw = 0; isw < inner_sweeps; ++isw) {
          if (tid == 0) s_rot = 0;
          __syncthreads();
          for (int ir = 0; ir < m2 - 1; ++ir) {
            for (int k = warp; k < m2 / 2; k += nwarp) {
              int p, q;
              rr_pair(k, ir, m2, p, q);
              if (q >= m) continue;
              double* wp = Ws + p * nld;
              double* wq = Ws + q * nld;
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
              // rotate when |ga| > tol sqrt(al be) (squared; al, be >= 0)
              if (al > 0.0 && be > 0.0 && ga * ga > tol * tol * al * be) {
                double c, s;
                rotation(al, be, ga, c, s);
                for (int i = lane; i < n; i += 32) {
                  const double x = wp[i], y = wq[i];
                  wp[i] = c * x - s * y;
                  wq[i] = s * x + c * y;
                }
                double* jp = Js + p * m;
                double* jq = Js + q * m;
                for (int i = lane; i < m; i += 32) {
                  const double x = jp[i], y = jq[i];
                  jp[i] = c * x - s * y;
                  jq[i] = s * x + c * y;
                }
                // convergence counts only rotations above the (looser) sweep
                // tolerance; rounding-level rotations are applied but do not
                // keep the iteration alive.
                if (lane == 0 && ga * ga > tol_conv * tol_conv * al * be) s_rot = 1;
              }
            }
            __syncthreads();
          }
          if (!s_rot) break;
          any = 1;
        }
        if (!any) continue;
        if (tid == 0) atomicAdd(cnt, 1u);
        for (int idx = tid; idx < m * n; idx += blockDim.x) {
          const int k = idx / n, i = idx % n;
          W[i + static_cast<i64>(cols[k]) * ldw] = Ws[k * nld + i];
        }
        __syncthreads();
        for (int idx = tid; idx < m * n; idx += blockDim.x) {  // stage V_S (reusing the W_S space)
          const int k = idx / n, i = idx % n;
          Ws[k * nld + i] = V[i + static_cast<i64>(cols[k]) * ldv];
        }
        __syncthreads();
        for (int idx = tid; idx < m * n; idx += blockDim.x) {  // V_S <- V_S J
          const int k = idx / n, i = idx % n;
          const double* jk = Js + k * m;
          double acc = 0.0;
          for (int j = 0; j < m; ++j) acc += Ws[j * nld + i] * jk[j];
          V[i + static_cast<i64>(cols[k]) * ldv] = acc;
        }
      }
      grid.sync();
      if (r == 0 && blockIdx.x == 0 && threadIdx.x == 0) counters[(sweep + 1) & 1] = 0u;
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[2] = sweep + 1;
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
  static const bool blocked_only = std::getenv("NPCG_CHOL") && std::string(std::getenv("NPCG_CHOL")) == "blocked";
  if (n <= kCholFusedMax && !blocked_only) return cholesky_fused(ctx, a, n, lda, f);
  f.nb = NB;
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
  if (f.linv.p()) {  // X = Y L^{-T}: one DMMA GEMM with the explicit inverse
    GemmEpi tri;
    tri.tri = true;  // L^{-T} is upper triangular: an n-tile's K loop stops at its last column
    gemm(ctx, m, n, n, 1.0, Operand{Y, ldy, false}, Operand{f.linv.p(), f.linv.ld, false}, 0.0, X, ldx, tri);
    return;
  }
  const i64 nb = f.nb;
  const i64 nblk = cdiv(n, nb);
  for (i64 b = 0; b < nblk; ++b) {
    const i64 k0 = b * nb, kb = std::min<i64>(nb, n - k0);
    gemm(ctx, m, kb, kb, 1.0, Operand{Y + k0 * ldy, ldy, false}, Operand{f.dinv.p + b * nb * nb, nb, false}, 0.0,
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
bool cholqr_pass(Ctx& ctx, double* Y, i64 ldy, i64 m, i64 n, double shift, DMat& Lm, double* Q, i64 ldq, bool dist) {
  Lm.alloc(n, n, ctx.stream, false);
  GemmEpi gram;
  gram.sym = true;  // Y^T Y: upper tiles + mirror
  gemm(ctx, n, n, m, 1.0, Operand{Y, ldy, true}, Operand{Y, ldy, true}, 0.0, Lm.p(), Lm.ld, gram);
  if (dist) rows_allreduce(ctx, Lm.p(), Lm.ld * n);  // Y^T Y over all row blocks
  if (shift > 0.0) NPCG_LAUNCH(ctx, add_diag_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, Lm.p(), n, Lm.ld, shift);
  CholFactor f;
  if (!cholesky(ctx, Lm.p(), n, Lm.ld, f)) return false;
  trsm_right_lt(ctx, m, n, Y, ldy, Lm.p(), Lm.ld, f, Q, ldq);
  return true;
}
}  // namespace

void orthonormalize(Ctx& ctx, const double* G_in, i64 ldg_in, i64 m, i64 n, double* Q, i64 ldq, double* Rt, i64 ldr,
                    bool dist) {
  if (n <= 0) return;
  dist = dist && ctx.sharded();
  // Scale by an exact power of two so max|G| ~ 1: the Gram G^T G neither
  // underflows (e.g. the nu-shifted zero matrix, whose B ~ sqrt(nu) ~ 1e-162)
  // nor overflows. Q is scale-invariant; R^T is scaled back exactly.
  const double amax = dist ? max_abs_rows(ctx, G_in, m, n, ldg_in) : max_abs(ctx, G_in, m, n, ldg_in);
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
  std::vector<DMat> Ls(1);
  bool shifted = false;
  if (!cholqr_pass(ctx, work.p(), work.ld, m, n, 0.0, Ls[0], Q, ldq, dist)) {
    // Shifted CholeskyQR (Fukaya et al.): s = 11 (m n + n(n+1)) u ||G||_F^2.
    const double fro2 = dist ? sum_squares_rows(ctx, G, m, n, ldg) : sum_squares(ctx, G, m, n, ldg);
    const double mt = dist ? rows_allreduce_host(ctx, static_cast<double>(m), false) : static_cast<double>(m);
    const double s = 11.0 * (mt * n + static_cast<double>(n) * (n + 1)) * 2.220446049250313e-16 * fro2;
    copy2d(ctx, m, n, G, ldg, work.p(), work.ld);
    if (!cholqr_pass(ctx, work.p(), work.ld, m, n, s, Ls[0], Q, ldq, dist))
      fail(NPCG_ERUNTIME, "orthonormal_columns: shifted CholeskyQR broke down (rank-deficient input)");
    shifted = true;
  }
  // Further passes on Q (CholeskyQR2 / shifted CholeskyQR3). The Gram Q^T Q of
  // the next pass is formed first; when Q is already orthonormal to working
  // accuracy (well-conditioned input, e.g. a Gaussian Omega) the pass is skipped.
  for (int more = 0; more < (shifted ? 2 : 1); ++more) {
    DMat L;
    L.alloc(n, n, ctx.stream, false);
    GemmEpi gram;
    gram.sym = true;
    gemm(ctx, n, n, m, 1.0, Operand{Q, ldq, true}, Operand{Q, ldq, true}, 0.0, L.p(), L.ld, gram);
    if (dist) rows_allreduce(ctx, L.p(), L.ld * n);
    if (!shifted || more > 0) {
      // (sharded: m is the local row count; ~world x m rows in all)
      const double tol = std::max(1e-14, 4.0 * std::sqrt(static_cast<double>(m) * (dist ? ctx.world() : 1)) *
                                             2.220446049250313e-16);
      if (identity_deviation(ctx, L.p(), L.ld, n) <= tol) break;
    }
    CholFactor f;
    if (!cholesky(ctx, L.p(), n, L.ld, f))
      fail(NPCG_ERUNTIME, "orthonormal_columns: CholeskyQR re-orthogonalisation pass broke down");
    copy2d(ctx, m, n, Q, ldq, work.p(), work.ld);
    trsm_right_lt(ctx, m, n, work.p(), work.ld, L.p(), L.ld, f, Q, ldq);
    Ls.push_back(std::move(L));
  }
  if (Rt) {  // R^T = L1 L2 (L3)
    if (Ls.size() == 1) {
      copy2d(ctx, n, n, Ls[0].p(), Ls[0].ld, Rt, ldr);
    } else {
      DMat acc, t;
      acc.alloc(n, n, ctx.stream, false);
      copy2d(ctx, n, n, Ls[0].p(), Ls[0].ld, acc.p(), acc.ld);
      for (size_t k = 1; k < Ls.size(); ++k) {
        double* dst = k + 1 == Ls.size() ? Rt : nullptr;
        if (!dst) t.alloc(n, n, ctx.stream, false);
        gemm(ctx, n, n, n, 1.0, Operand{acc.p(), acc.ld, false}, Operand{Ls[k].p(), Ls[k].ld, true}, 0.0,
             dst ? dst : t.p(), dst ? ldr : t.ld);
        if (!dst) std::swap(acc, t);
      }
    }
    if (e2 != 0) scale_pow2(ctx, n, n, Rt, ldr, e2);
  }
}

// max |G_ij - delta_ij| (synchronises).
double identity_deviation(Ctx& ctx, const double* G, i64 ldg, i64 n) {
  DBuf<double> out(1, ctx.stream);
  out.zero();
  NPCG_LAUNCH(ctx, identity_dev_kernel, static_cast<unsigned>(std::min<i64>(cdiv(n * n, 256), 1024)), 256, 0, G, ldg,
              n, out.p);
  double h = 0.0;
  NPCG_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return h;
}

void jacobi_svd_small(Ctx& ctx, double* W, i64 ldw, i64 n, double* Vs, i64 ldv, double* sigma) {
  if (n <= 0) return;
  DMat V;
  V.alloc(n, n, ctx.stream, false);
  set_identity(ctx, V.p(), n, n, V.ld);
  DBuf<unsigned int> counters(3, ctx.stream);
  counters.zero();
  int nn = static_cast<int>(n);
  double tol = 2.220446049250313e-16 * std::sqrt(static_cast<double>(n));
  int max_sweeps = 60;
  // Shared memory holds the pair's m columns (n rows each) plus J (m x m).
  constexpr i64 kSmemBudget = 200 * 1024;
  const i64 nld = n + (n & 1);
  int bsz, nbp, inner;
  if ((nld * n + n * n) * 8 <= kSmemBudget && n <= JOS_MAXM) {  // whole problem in one CTA
    bsz = static_cast<int>((n + 1) / 2);
    nbp = 2;
    inner = max_sweeps;
  } else {
    i64 m = 2;
    while (m * 2 <= JOS_MAXM && (2 * m * nld + 4 * m * m) * 8 <= kSmemBudget && m < 32) m *= 2;
    bsz = static_cast<int>(m / 2);
    if (const char* e = std::getenv("NPCG_JACOBI_B")) bsz = std::max(1, std::min(bsz, std::atoi(e)));
    const int nblk = static_cast<int>(cdiv(n, bsz));
    nbp = nblk + (nblk & 1);
    inner = 1;
    if (const char* e = std::getenv("NPCG_JACOBI_INNER")) inner = std::max(1, std::atoi(e));
  }
  const i64 mcols = 2 * static_cast<i64>(bsz);
  const int smem = static_cast<int>((mcols * nld + mcols * mcols) * 8);
  NPCG_CUDA(cudaFuncSetAttribute(jacobi_os_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_os_kernel, JOS_THREADS, smem));
  const int grid = std::max(1, std::min(nbp / 2, std::max(per_sm, 1) * ctx.sm_count));
  double* Wp = W;
  double* Vp = V.p();
  i64 ldvv = V.ld;
  unsigned int* cp = counters.p;
  void* args[] = {&Wp, &ldw, &Vp, &ldvv, &nn, &bsz, &nbp, &tol, &max_sweeps, &inner, &cp};
  ctx.prof_begin("jacobi_os_kernel");
  NPCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_os_kernel), grid, JOS_THREADS, args, smem,
                                        ctx.stream));
  ctx.check_launch("jacobi_os_kernel");
  ctx.prof_end();
  if (std::getenv("NPCG_DEBUG")) {
    unsigned int h[3];
    NPCG_CUDA(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    std::fprintf(stderr, "[npcg] jacobi n=%lld b=%d pairs/round=%d grid=%d sweeps=%u\n", static_cast<long long>(n), bsz,
                 nbp / 2, grid, h[2]);
  }
  DBuf<double> sig(n, ctx.stream);
  DBuf<int> perm(n, ctx.stream);
  NPCG_LAUNCH(ctx, colnorm_kernel, static_cast<unsigned>(cdiv(n * 32, 256)), 256, 0, W, ldw, nn, sig.p);
  NPCG_LAUNCH(ctx, rank_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, sig.p, nn, perm.p);
  NPCG_LAUNCH(ctx, gather_cols_kernel, static_cast<unsigned>(n), 128, 0, V.p(), V.ld, nn, perm.p, sig.p, Vs, ldv,
              sigma);
}

void thin_svd(Ctx& ctx, const double* B, i64 ldb, i64 m, i64 n, double* U, i64 ldu, double* sigma, bool dist) {
  dist = dist && ctx.sharded();
  if (!dist && m < n) invalid("thin_svd: expected a tall (m >= n) matrix");
  if (n <= 0) return;
  DMat Q, Rt, Vs;
  Q.alloc(m, n, ctx.stream, false);
  Rt.alloc(n, n, ctx.stream, false);
  Vs.alloc(n, n, ctx.stream, false);
  orthonormalize(ctx, B, ldb, m, n, Q.p(), Q.ld, Rt.p(), Rt.ld, dist);
  const char* mode = std::getenv("NPCG_SVD");
  if (mode && std::string(mode) == "jacobi") {
    jacobi_svd_small(ctx, Rt.p(), Rt.ld, n, Vs.p(), Vs.ld, sigma);
  } else {
    small_svd_eig(ctx, Rt.p(), Rt.ld, n, Vs.p(), Vs.ld, sigma);
  }
  gemm(ctx, m, n, n, 1.0, Operand{Q.p(), Q.ld, false}, Operand{Vs.p(), Vs.ld, true}, 0.0, U, ldu);
}

// Orthonormalise a square, nearly orthogonal Z by Newton-Schulz iteration
// towards its polar factor, V <- 1.5 V - 0.5 V (V^T V): two DMMA GEMMs per
// step, quadratic convergence, no factorisation. Returns false when Z is too
// far from orthogonal for the iteration (max |Z^T Z - I| > 0.5).
bool polar_orthonormalize(Ctx& ctx, const double* Z, i64 ldz, i64 n, double* V, i64 ldv) {
  DMat G, Y;
  G.alloc(n, n, ctx.stream, false);
  Y.alloc(n, n, ctx.stream, false);
  copy2d(ctx, n, n, Z, ldz, V, ldv);
  const double tol = std::max(1e-14, 4.0 * std::sqrt(static_cast<double>(n)) * 2.220446049250313e-16);
  double prev = 1e300;
  for (int it = 0; it < 8; ++it) {
    gemm(ctx, n, n, n, 1.0, Operand{V, ldv, true}, Operand{V, ldv, true}, 0.0, G.p(), G.ld);
    const double dev = identity_deviation(ctx, G.p(), G.ld, n);
    if (dev <= tol || (dev <= 1e-12 && dev > 0.25 * prev)) return true;  // converged / at the rounding floor
    if (!(dev <= 0.5)) return false;
    prev = dev;
    copy2d(ctx, n, n, V, ldv, Y.p(), Y.ld);
    gemm(ctx, n, n, n, -0.5, Operand{Y.p(), Y.ld, false}, Operand{G.p(), G.ld, true}, 1.5, V, ldv);
  }
  return false;
}

// SVD of R via the eigenvectors of R R^T = W^T W (W = R^T): the eigensolver
// only has to deliver an orthogonal V that diagonalises W^T W to working
// accuracy; the singular values are then the column norms of W V, which are
// accurate relative to each sigma_j (an O(eps sigma_1^2) perturbation of the
// Gram moves them only at second order), not just relative to sigma_1.
void small_svd_eig(Ctx& ctx, double* W, i64 ldw, i64 n, double* Vs, i64 ldv, double* sigma) {
  if (n <= 0) return;
  // Tiny R: one-CTA one-sided Jacobi (its sweeps cost O(n^3) per CTA, so beyond
  // a few dozen columns the eigenvector path is faster; Jacobi stays the fallback).
  static const int jacobi_max = std::getenv("NPCG_JACOBI_MAX") ? std::atoi(std::getenv("NPCG_JACOBI_MAX")) : 24;
  if (n <= jacobi_max) {
    jacobi_svd_small(ctx, W, ldw, n, Vs, ldv, sigma);
    return;
  }
  const int nn = static_cast<int>(n);
  // W scaled by an exact power of two (singular vectors are scale-invariant;
  // keeps W^T W clear of underflow/overflow); sigma is scaled back at the end.
  const double amax = max_abs(ctx, W, n, n, ldw);
  int e2 = 0;
  if (amax > 0.0 && std::isfinite(amax)) std::frexp(amax, &e2);
  DMat Ws, M, Z, V, W1, G, Cm, T;
  Ws.alloc(n, n, ctx.stream, false);
  M.alloc(n, n, ctx.stream, false);
  Z.alloc(n, n, ctx.stream, true);
  V.alloc(n, n, ctx.stream, false);
  W1.alloc(n, n, ctx.stream, false);
  G.alloc(n, n, ctx.stream, false);
  Cm.alloc(n, n, ctx.stream, false);
  T.alloc(n, n, ctx.stream, false);
  copy2d(ctx, n, n, W, ldw, Ws.p(), Ws.ld);
  scale_pow2(ctx, n, n, Ws.p(), Ws.ld, -e2);
  gemm(ctx, n, n, n, 1.0, Operand{Ws.p(), Ws.ld, true}, Operand{Ws.p(), Ws.ld, true}, 0.0, M.p(), M.ld);  // W^T W
  sym_eigvecs(ctx, M.p(), M.ld, n, Z.p(), Z.ld);
  bool ok = polar_orthonormalize(ctx, Z.p(), Z.ld, n, V.p(), V.ld) || try_orthonormalize(ctx, Z.p(), Z.ld, n, n, V.p(), V.ld);
  // Simultaneous-Jacobi refinement: G = (W V)^T (W V) has entries accurate
  // relative to the column norms; the first-order angles C_ij = G_ij/(G_jj -
  // G_ii) rotate V towards the singular vectors of the small sigma too (the
  // error squares each pass), then V is re-orthonormalised. The pass repeats
  // until the predicted column-norm error is below 1e-13 relative; if inverse
  // iteration mis-resolved a cluster, the robust one-sided Jacobi takes over.
  DBuf<double> qual(1, ctx.stream);
  for (int pass = 0; ok && pass < 4; ++pass) {
    gemm(ctx, n, n, n, 1.0, Operand{Ws.p(), Ws.ld, false}, Operand{V.p(), V.ld, true}, 0.0, W1.p(), W1.ld);
    gemm(ctx, n, n, n, 1.0, Operand{W1.p(), W1.ld, true}, Operand{W1.p(), W1.ld, true}, 0.0, G.p(), G.ld);
    NPCG_CUDA(cudaMemsetAsync(qual.p, 0, sizeof(double), ctx.stream));
    NPCG_LAUNCH(ctx, refine_angles_kernel, static_cast<unsigned>(cdiv(n, 8)), 256, 0, G.p(), G.ld, n, Cm.p(), Cm.ld,
                qual.p);
    double q = 0.0;
    NPCG_CUDA(cudaMemcpyAsync(&q, qual.p, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    if (std::getenv("NPCG_DEBUG")) std::fprintf(stderr, "[npcg] svd refine pass %d predicted rel err %.3e\n", pass, q);
    if (q <= 1e-13) break;
    if (pass == 3) {
      ok = false;
      break;
    }
    copy2d(ctx, n, n, V.p(), V.ld, T.p(), T.ld);
    gemm(ctx, n, n, n, 1.0, Operand{V.p(), V.ld, false}, Operand{Cm.p(), Cm.ld, true}, 1.0, T.p(), T.ld);
    ok = polar_orthonormalize(ctx, T.p(), T.ld, n, V.p(), V.ld) || try_orthonormalize(ctx, T.p(), T.ld, n, n, V.p(), V.ld);
  }
  if (!ok) {
    if (std::getenv("NPCG_DEBUG")) std::fprintf(stderr, "[npcg] svd: eigenvector path fell back to Jacobi\n");
    jacobi_svd_small(ctx, W, ldw, n, Vs, ldv, sigma);
    return;
  }
  DBuf<double> sig(n, ctx.stream);
  DBuf<int> perm(n, ctx.stream);
  NPCG_LAUNCH(ctx, colnorm_kernel, static_cast<unsigned>(cdiv(n * 32, 256)), 256, 0, W1.p(), W1.ld, nn, sig.p);
  NPCG_LAUNCH(ctx, rank_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, sig.p, nn, perm.p);
  NPCG_LAUNCH(ctx, gather_cols_kernel, static_cast<unsigned>(n), 128, 0, V.p(), V.ld, nn, perm.p, sig.p, Vs, ldv,
              sigma);
  scale_pow2(ctx, n, 1, sigma, n, e2);
}

}  // namespace npcg

namespace npcg {
bool try_orthonormalize(Ctx& ctx, const double* G, i64 ldg, i64 m, i64 n, double* Q, i64 ldq) {
  try {
    orthonormalize(ctx, G, ldg, m, n, Q, ldq);
    return true;
  } catch (const Error& e) {
    if (e.code == NPCG_ERUNTIME) return false;
    throw;
  }
}
}  // namespace npcg
