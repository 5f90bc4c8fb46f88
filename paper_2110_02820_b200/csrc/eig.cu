// Symmetric eigenvectors of a small dense l x l matrix on device, for the
// thin SVD of the Nyström pipeline (factor.cu).
//
//   1. Householder tridiagonalisation: per column, every CTA forms the
//      reflector redundantly; the previous step's rank-2 update and this
//      step's trailing symmetric matvec are fused in one pass split over CTAs
//      by column. n <= 512: one thread-block cluster with the matrix in
//      registers (one cluster barrier per column); larger n: one cooperative
//      kernel (one grid-wide barrier per column).
//   2. Bisection with Sturm counts, one eigenvalue per thread.
//   3. Inverse iteration on the tridiagonal (partial-pivoting LU), one
//      eigenvector per thread, deterministic pseudo-random starts; exact
//      repeats are split by a tiny shift.
//   4. Back-transformation by the stored reflectors, one warp per column.
// The caller re-orthonormalises the vectors (CholeskyQR2) and takes the
// singular values as column norms of W V, so their relative accuracy does not
// depend on this solver's eigenvalue accuracy (see factor.cu).
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <string>

#include "eig.cuh"
#include "gemm.cuh"

namespace cg = cooperative_groups;

namespace npcg {
namespace {

constexpr int TRI_THREADS = 256;

// Fast reciprocal (MUFU seed + Newton steps in the FP64 pipe, about 1 ulp): the
// Sturm counts and inverse iteration only need it to a few ulps, and an IEEE
// division on their sequential recurrences costs several times more.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);  // one more Newton step: the approximation alone is not full precision
  return fma(r, e, r);
}


// One grid-wide barrier per column: the rank-2 update of step k-1 is kept
// pending (vp, wp) and applied on the fly -- redundantly by every CTA to
// column k (which yields the reflector of step k), and by the column owners
// in the same pass that forms p = tau A22 v for step k (each trailing column
// is read and written once per step). p is double-buffered across steps.
__global__ void __launch_bounds__(TRI_THREADS) tridiag_kernel(double* M, i64 ld, int n, double* d, double* e,
                                                               double* tau, double* H, i64 ldh, double* p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double tsm[];  // v (n), vp (n), wp (n)
  __shared__ double red[32];
  double* v = tsm;           // step k reflector: v[i] <-> row k+1+i
  double* vp = tsm + n;      // pending update of step k-1: index i <-> row k+i
  double* wp = tsm + 2 * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int G = gridDim.x, bid = blockIdx.x;
  bool pend = false;
  for (int k = 0; k < n - 2; ++k) {
    const int L = n - k - 1;
    const double* colk = M + k + static_cast<i64>(k) * ld;  // column k, rows k..n-1
    // ---- column k with the pending update applied; reflector (redundant in every CTA)
    double s = 0.0;
    for (int j = tid; j < L; j += blockDim.x) {
      double x = colk[j + 1];
      if (pend) x -= vp[j + 1] * wp[0] + wp[j + 1] * vp[0];
      v[j] = x;
      if (j > 0) s += x * x;
    }
    s = block_sum(s, red);  // (barrier: v complete)
    const double alpha = v[0];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (s > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + s), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    for (int j = tid; j < L; j += blockDim.x) v[j] = j == 0 ? 1.0 : v[j] * scal;
    if (bid == 0 && tid == 0) {
      d[k] = pend ? colk[0] - (vp[0] * wp[0] + wp[0] * vp[0]) : colk[0];
      e[k] = beta;
      tau[k] = t;
    }
    __syncthreads();
    if (bid == 0)
      for (int i = tid; i < L; i += blockDim.x) H[(k + 1 + i) + static_cast<i64>(k) * ldh] = v[i];
    // ---- owners: A22 -= pending (written back), p = tau A22 v
    double* pk = p + (k & 1) * n;
    for (int c = bid * nw + warp; c < L; c += G * nw) {
      double* col = M + (k + 1) + static_cast<i64>(k + 1 + c) * ld;
      const double vc = pend ? vp[c + 1] : 0.0, wc = pend ? wp[c + 1] : 0.0;
      double acc = 0.0;
      if (pend) {
        for (int i = lane; i < L; i += 32) {
          const double a = col[i] - (vp[i + 1] * wc + wp[i + 1] * vc);
          col[i] = a;
          acc += a * v[i];
        }
      } else {
        for (int i = lane; i < L; i += 32) acc += col[i] * v[i];
      }
      acc = warp_sum(acc);
      if (lane == 0) pk[c] = t * acc;
    }
    grid.sync();
    // ---- w = p - (tau/2)(p.v) v (redundant per CTA) becomes the pending update
    double pv = 0.0;
    for (int i = tid; i < L; i += blockDim.x) pv += pk[i] * v[i];
    pv = block_sum(pv, red);
    const double K = 0.5 * t * pv;
    for (int i = tid; i < L; i += blockDim.x) {
      double w = pk[i];
      w -= K * v[i];
      wp[i] = w;
      vp[i] = v[i];
    }
    pend = true;
    __syncthreads();
  }
  if (bid == 0 && tid == 0) {
    if (n >= 3) {  // last 2 x 2 block with the pending update of step n-3
      const double* m2 = M + (n - 2) + static_cast<i64>(n - 2) * ld;
      d[n - 2] = m2[0] - (vp[0] * wp[0] + wp[0] * vp[0]);
      e[n - 2] = m2[1] - (vp[1] * wp[0] + wp[1] * vp[0]);
      d[n - 1] = m2[1 + ld] - (vp[1] * wp[1] + wp[1] * vp[1]);
      tau[n - 2] = 0.0;
    } else if (n == 2) {
      d[0] = M[0];
      d[1] = M[1 + ld];
      e[0] = M[1];
      tau[0] = 0.0;
    } else {
      d[0] = M[0];
    }
    if (n >= 1) {
      e[n - 1] = 0.0;
      tau[n - 1] = 0.0;
    }
  }
}

// The same algorithm inside one thread-block cluster (n <= 512, no global
// memory traffic but the outputs). Warp w of CTA r keeps
// its owned columns c = (w + 8q) C + r (q < 4) in registers, lane l holding
// rows l + 32 m (m < MR), so the fused pass (pending rank-2 update + the
// column's dot with v) touches shared memory only for the vectors. The next
// step's column k+1 is taken as row k+1 (A is symmetric): every CTA publishes
// the row's entries of its own columns next to their p values, and one
// gather per step (half-warp h reads CTA h's 32 (p, row) pairs, contiguous)
// moves both -- no CTA serves a whole column to the cluster (DSMEM bandwidth
// per SM is ~21 B/clk; a 3.2 KB column to 15 peers costs ~1 us).
template <int MR>
__global__ void __launch_bounds__(TRI_THREADS, 1) tridiag_reg_kernel(const double* M, i64 ld, int n, double* d,
                                                                      double* e, double* tau, double* H, i64 ldh,
                                                                      unsigned long long* trace) {
  constexpr int QMAX = 4, NW = TRI_THREADS / 32;
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
  extern __shared__ double trs[];
  double* v = trs;               // [n] reflector of the step (v[j] <-> row k+1+j)
  double* vp = v + n;            // [n] previous step's v, w (vp[i] <-> row k+i)
  double* wp = vp + n;
  double* pt = wp + n;           // [n] gathered p (pt[i] <-> column k+1+i)
  double* xcol = pt + n;         // [n] row k of the updated matrix (xcol[i] <-> column k+i)
  __shared__ double2 pr[2][32];  // (p, row k+1 entry) of this CTA's owned columns
  __shared__ double redA[NW], redB[NW];
  __shared__ double alpha_sh, lastd;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncl = (n + C - 1) / C;
  auto bsum1 = [&](double x, double* buf) {
    x = warp_sum(x);
    if (lane == 0) buf[warp] = x;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += buf[w];
    return t;
  };
  double a[QMAX][MR];
  int cq[QMAX];
#pragma unroll
  for (int q = 0; q < QMAX; ++q) {
    const int lc = warp + NW * q;
    cq[q] = lc < ncl ? lc * C + rank : n;  // n = no column
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int r = lane + 32 * m;
      a[q][m] = (cq[q] < n && r < n) ? M[r + static_cast<i64>(cq[q]) * ld] : 0.0;
    }
    if (lane == 0 && cq[q] < n) pr[1][lc].y = a[q][0];  // row 0 for the first step
  }
  if (trace && tid == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    trace[64 * 6 + rank] = sm;
  }
  // gather (p, row k+1) of step k-1 from every CTA: half-warp h <- CTA h
  auto gather = [&](int k, int buf) {
    const int src = tid >> 4, l0 = tid & 15;
    if (src < C) {
      const double2* rp = cl.map_shared_rank(&pr[buf][0], src);
      const int c0 = l0 * C + src, c1 = (l0 + 16) * C + src;
      const bool ok0 = l0 < ncl && c0 > k && c0 < n, ok1 = l0 + 16 < ncl && c1 > k && c1 < n;
      const double2 g0 = ok0 ? rp[l0] : make_double2(0.0, 0.0), g1 = ok1 ? rp[l0 + 16] : make_double2(0.0, 0.0);
      if (ok0) {
        pt[c0 - k - 1] = g0.x;
        xcol[c0 - k - 1] = g0.y;
      }
      if (ok1) {
        pt[c1 - k - 1] = g1.x;
        xcol[c1 - k - 1] = g1.y;
      }
    }
  };
  cl.sync();
  gather(-1, 1);  // row 0 (its p entries are unused)
  __syncthreads();
  bool pend = false;
  auto tick = [&](int k, int ph) {
    if (trace && rank == 0 && tid == 0 && k < 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      trace[k * 6 + ph] = t;
    }
  };
  for (int k = 0; k < n - 2; ++k) {
    tick(k, 0);
    const int L = n - k - 1;  // <= 511: rows k+1+tid and k+1+tid+256
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = tid + u * TRI_THREADS;
      if (j < L) {
        double x = xcol[j + 1];
        if (pend) x -= vp[j + 1] * wp[0] + wp[j + 1] * vp[0];
        v[j] = x;
        if (j > 0) s += x * x;
        else alpha_sh = x;
      }
    }
    s = bsum1(s, redA);  // (its barrier also publishes v and alpha)
    tick(k, 1);
    const double alpha = alpha_sh;
    double t = 0.0, beta = alpha, scal = 0.0;
    if (s > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + s), alpha);
      t = (beta - alpha) * fast_rcp(beta);
      scal = fast_rcp(alpha - beta);
    }
    for (int j = tid; j < L; j += TRI_THREADS) v[j] = j == 0 ? 1.0 : v[j] * scal;  // this thread's own entries
    if (rank == 0 && tid == 0) {
      d[k] = pend ? xcol[0] - (vp[0] * wp[0] + wp[0] * vp[0]) : xcol[0];
      e[k] = beta;
      tau[k] = t;
    }
    __syncthreads();
    if (rank == 0)
      for (int i = tid; i < L; i += TRI_THREADS) H[(k + 1 + i) + static_cast<i64>(k) * ldh] = v[i];
    tick(k, 2);
    const int buf = k & 1;
    {
      double vcq[QMAX], wcq[QMAX], accq[QMAX], rowq[QMAX];
      bool lq[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        lq[q] = cq[q] > k && cq[q] < n;
        vcq[q] = lq[q] && pend ? vp[cq[q] - k] : 0.0;
        wcq[q] = lq[q] && pend ? wp[cq[q] - k] : 0.0;
        accq[q] = 0.0;
        rowq[q] = 0.0;
      }
      // Branch-free inside a group of 4 warp-rows (loads hoisted, 4 x QMAX
      // independent chains): rows outside the trailing block and dead columns
      // get zero coefficients, which leaves a unchanged and adds +0 to acc.
#pragma unroll
      for (int g = 0; g < MR / 4; ++g) {
        if (32 * (4 * g + 3) + 31 <= k || 128 * g >= n) continue;  // whole group outside (uniform)
        double vpi[4], wpi[4], vi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = lane + 32 * (4 * g + u);
          const bool rl = r > k && r < n;
          const int ix = rl ? r - k : 1;
          const double x0 = vp[ix], x1 = wp[ix], x2 = v[ix - 1];
          vpi[u] = rl && pend ? x0 : 0.0;
          wpi[u] = rl && pend ? x1 : 0.0;
          vi[u] = rl ? x2 : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < QMAX; ++q) {
            const double x = fma(-vpi[u], wcq[q], fma(-wpi[u], vcq[q], a[q][4 * g + u]));  // two FMAs
            a[q][4 * g + u] = x;
            accq[q] = fma(x, vi[u], accq[q]);
          }
      }
      const int m1 = (k + 1) >> 5;  // warp-row holding row k+1 (uniform branch per m)
#pragma unroll
      for (int m = 0; m < MR; ++m)
        if (m == m1)
#pragma unroll
          for (int q = 0; q < QMAX; ++q) rowq[q] = a[q][m];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        if (lq[q] && lane == ((k + 1) & 31)) pr[buf][warp + NW * q].y = rowq[q];  // row k+1 of column cq
        if (k == n - 3 && cq[q] == n - 1)  // a(n-1, n-1) after the last update, for the final 2 x 2 block
#pragma unroll
          for (int m = 0; m < MR; ++m)
            if (lane + 32 * m == n - 1) lastd = a[q][m];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < QMAX; ++q) accq[q] += __shfl_xor_sync(0xffffffffu, accq[q], o);
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < QMAX; ++q)
          if (lq[q]) pr[buf][warp + NW * q].x = t * accq[q];
    }
    tick(k, 3);
    cl.sync();
    tick(k, 4);
    gather(k, buf);
    __syncthreads();
    double pv = 0.0;
    for (int i = tid; i < L; i += TRI_THREADS) pv += pt[i] * v[i];
    pv = bsum1(pv, redB);
    tick(k, 5);
    const double K = 0.5 * t * pv;
    for (int i = tid; i < L; i += TRI_THREADS) {
      double w = pt[i];
      w -= K * v[i];
      wp[i] = w;
      vp[i] = v[i];
    }
    pend = true;
    __syncthreads();
  }
  if (rank == 0 && tid == 0) {
    const double* ld1 = cl.map_shared_rank(&lastd, (n - 1) % C);
    d[n - 2] = xcol[0] - (vp[0] * wp[0] + wp[0] * vp[0]);
    e[n - 2] = xcol[1] - (vp[1] * wp[0] + wp[1] * vp[0]);
    d[n - 1] = *ld1 - (vp[1] * wp[1] + wp[1] * vp[1]);
    tau[n - 2] = 0.0;
    e[n - 1] = 0.0;
    tau[n - 1] = 0.0;
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

// number of eigenvalues of T strictly below x (Sturm sequence of LDL^T)
__device__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n, double x,
                           double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
#pragma unroll 8
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e2[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// Gershgorin interval, ||T|| bound, pivmin and e_i^2 (one CTA).
__global__ void tri_bounds_kernel(const double* d, const double* e, int n, double* e2, double* info) {
  __shared__ double sh[32];
  double lo = 1e308, hi = -1e308, emax = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i < n - 1) {
      emax = fmax(emax, fabs(e[i]));
      e2[i] = e[i] * e[i];
    }
  }
  lo = -block_max(-lo, sh);
  hi = block_max(hi, sh);
  emax = block_max(emax, sh);
  if (threadIdx.x == 0) {
    const double tnorm = fmax(fmax(fabs(lo), fabs(hi)), 1e-300);
    const double eps = 2.220446049250313e-16;
    info[0] = lo - 4.0 * eps * tnorm - 1e-300;
    info[1] = hi + 4.0 * eps * tnorm + 1e-300;
    info[2] = fmax(1e-300, 4.0 * 2.2250738585072014e-308 * fmax(1.0, emax * emax));
    info[3] = tnorm;
  }
}

// Multisection: one warp per eigenvalue, 32 Sturm counts per step shrink the
// bracket 33x (about 9 steps to 1e-13 ||T||). Eigenvalue j is the (j+1)-th
// smallest. Only inverse-iteration shifts are needed from here.
__global__ void bisect_kernel(const double* d, const double* e2, int n, const double* info, double* lam) {
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (j >= n) return;
  double lo = info[0], hi = info[1];
  const double pivmin = info[2], tnorm = info[3];
  const double eps = 2.220446049250313e-16;
  for (int it = 0; it < 40; ++it) {
    const double tol = fmax(2.0 * eps * fmax(fabs(lo), fabs(hi)), 1e-13 * tnorm);
    if (hi - lo <= tol) break;
    const double x = lo + (hi - lo) * static_cast<double>(lane + 1) / 33.0;
    const int c = sturm_count(d, e2, n, x, pivmin);
    const unsigned ball = __ballot_sync(0xffffffffu, c > j);
    const int k = ball ? __ffs(ball) - 1 : 32;
    const double xk = __shfl_sync(0xffffffffu, x, k < 32 ? k : 31);
    const double xk1 = __shfl_sync(0xffffffffu, x, k > 0 ? k - 1 : 0);
    const double nlo = k == 0 ? lo : xk1;
    const double nhi = k == 32 ? hi : xk;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) lam[j] = 0.5 * (lo + hi);
}

__device__ __forceinline__ double hash_unit(unsigned long long a) {
  a ^= a >> 33;
  a *= 0xff51afd7ed558ccdULL;
  a ^= a >> 33;
  a *= 0xc4ceb9fe1a85ec53ULL;
  a ^= a >> 33;
  return static_cast<double>(a >> 11) * 0x1.0p-53 - 0.5;
}

// Inverse iteration on T for eigenvalue lam[j] (three solves), one thread per
// eigenvector. Work arrays are interleaved [i][j] so a warp's threads touch
// consecutive addresses at every step; the vector lands in Zr[i][j]
// (row-major n x n, i.e. Z^T column-major).
__global__ void invit_kernel(const double* d, const double* e, const double* lam, int n, const double* info,
                             double* Zr, double* wk, unsigned char* pvk) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double eps = 2.220446049250313e-16;
  const double tnorm = info[3];
  const i64 N = n;
  int rep = 0;  // exact repeats get distinct shifts so the solves differ
  while (j - rep - 1 >= 0 && lam[j] - lam[j - rep - 1] <= 4.0 * eps * tnorm) ++rep;
  const double shift = lam[j] + rep * 8.0 * eps * tnorm;
  const double tiny = fmax(eps * tnorm, 1e-300);
  double* u0 = wk;
  double* u1 = wk + N * N;
  double* u2 = wk + 2 * N * N;
  double* lm = wk + 3 * N * N;
#define IX(i) (static_cast<i64>(i) * N + j)
  for (int i = 0; i < n; ++i) {
    u0[IX(i)] = d[i] - shift;
    u1[IX(i)] = i < n - 1 ? e[i] : 0.0;
    u2[IX(i)] = 0.0;
  }
  for (int i = 0; i < n - 1; ++i) {  // dgttrf on T - shift I
    const double sub = e[i];
    const double a = u0[IX(i)];
    if (fabs(a) >= fabs(sub)) {
      pvk[IX(i)] = 0;
      const double piv = a == 0.0 ? tiny : a;
      u0[IX(i)] = piv;
      const double f = sub / piv;
      lm[IX(i)] = f;
      u0[IX(i + 1)] -= f * u1[IX(i)];
    } else {
      pvk[IX(i)] = 1;
      const double f = a / sub;
      lm[IX(i)] = f;
      u0[IX(i)] = sub;
      const double old_u1 = u1[IX(i)];
      const double old_d1 = u0[IX(i + 1)];
      u1[IX(i)] = old_d1;
      u0[IX(i + 1)] = old_u1 - f * old_d1;
      if (i < n - 2) {
        const double old_u1n = u1[IX(i + 1)];
        u2[IX(i)] = old_u1n;
        u1[IX(i + 1)] = -f * old_u1n;
      }
    }
  }
  if (u0[IX(n - 1)] == 0.0) u0[IX(n - 1)] = tiny;
  double* z = Zr;
  for (int i = 0; i < n; ++i) z[IX(i)] = hash_unit((static_cast<unsigned long long>(j) << 32) ^ static_cast<unsigned>(i));
  for (int it = 0; it < 3; ++it) {
    for (int i = 0; i < n - 1; ++i) {
      const double zi = z[IX(i)], zi1 = z[IX(i + 1)], f = lm[IX(i)];
      if (pvk[IX(i)]) {
        z[IX(i)] = zi1;
        z[IX(i + 1)] = zi - f * zi1;
      } else {
        z[IX(i + 1)] = zi1 - f * zi;
      }
    }
    z[IX(n - 1)] /= u0[IX(n - 1)];
    if (n >= 2) z[IX(n - 2)] = (z[IX(n - 2)] - u1[IX(n - 2)] * z[IX(n - 1)]) / u0[IX(n - 2)];
    for (int i = n - 3; i >= 0; --i)
      z[IX(i)] = (z[IX(i)] - u1[IX(i)] * z[IX(i + 1)] - u2[IX(i)] * z[IX(i + 2)]) / u0[IX(i)];
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) nrm += z[IX(i)] * z[IX(i)];
    const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
    for (int i = 0; i < n; ++i) z[IX(i)] *= inv;
  }
#undef IX
}

// Inverse iteration with the working set in shared memory: V eigenvectors per
// CTA, one per thread, layout [i][v]. The LU of T - shift I (partial
// pivoting, dgttrf) is recomputed in each of the three iterations and applied
// to z on the fly, so only U (three diagonals) and z are stored. Writes
// Zr[i][j] like invit_kernel.
__global__ void invit_smem_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                  const double* __restrict__ lam, int n, const double* __restrict__ info,
                                  double* __restrict__ Zr) {
  extern __shared__ double ism[];
  const int V = blockDim.x, v = threadIdx.x;
  const int j = blockIdx.x * V + v;
  double* u0 = ism;
  double* u1 = ism + static_cast<i64>(n) * V;
  double* u2 = ism + 2 * static_cast<i64>(n) * V;
  double* z = ism + 3 * static_cast<i64>(n) * V;
#define SX(i) (static_cast<i64>(i) * V + v)
  if (j >= n) return;
  const double eps = 2.220446049250313e-16;
  const double tnorm = info[3];
  int rep = 0;
  while (j - rep - 1 >= 0 && lam[j] - lam[j - rep - 1] <= 4.0 * eps * tnorm) ++rep;
  const double shift = lam[j] + rep * 8.0 * eps * tnorm;
  const double tiny = fmax(eps * tnorm, 1e-300);
  for (int i = 0; i < n; ++i) z[SX(i)] = hash_unit((static_cast<unsigned long long>(j) << 32) ^ static_cast<unsigned>(i));
  double scale = 1.0;
  for (int it = 0; it < 3; ++it) {
    // factor + forward elimination; a/b: diagonal/superdiagonal of row i, nd/nb: of row i+1
    double a = d[0] - shift, b = n > 1 ? e[0] : 0.0;
    double zi = z[SX(0)] * scale;
    for (int i = 0; i < n - 1; ++i) {
      const double sub = e[i];
      double nd = d[i + 1] - shift, nb = i + 1 < n - 1 ? e[i + 1] : 0.0;
      const double zi1 = z[SX(i + 1)] * scale;
      double nz;
      if (fabs(a) >= fabs(sub)) {
        const double piv = a == 0.0 ? tiny : a;
        const double pinv = fast_rcp(piv);
        const double f = sub * pinv;
        u0[SX(i)] = pinv;  // U's diagonal is kept as its reciprocal (back substitution multiplies)
        u1[SX(i)] = b;
        u2[SX(i)] = 0.0;
        nd -= f * b;
        z[SX(i)] = zi;
        nz = zi1 - f * zi;
      } else {
        const double f = a * fast_rcp(sub);
        u0[SX(i)] = fast_rcp(sub);
        u1[SX(i)] = nd;
        u2[SX(i)] = nb;
        const double nd2 = b - f * nd;
        nb = -f * nb;
        nd = nd2;
        z[SX(i)] = zi1;
        nz = zi - f * zi1;
      }
      a = nd;
      b = nb;
      zi = nz;
    }
    u0[SX(n - 1)] = fast_rcp(a == 0.0 ? tiny : a);
    z[SX(n - 1)] = zi;
    // back substitution (u0 holds reciprocals)
    double x2 = 0.0, x1 = z[SX(n - 1)] * u0[SX(n - 1)];
    z[SX(n - 1)] = x1;
    double nrm = x1 * x1;
    for (int i = n - 2; i >= 0; --i) {
      const double x = (z[SX(i)] - u1[SX(i)] * x1 - u2[SX(i)] * x2) * u0[SX(i)];
      z[SX(i)] = x;
      nrm += x * x;
      x2 = x1;
      x1 = x;
    }
    scale = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
  }
  for (int i = 0; i < n; ++i) Zr[static_cast<i64>(i) * n + j] = z[SX(i)] * scale;
#undef SX
}

__global__ void transpose_sq_kernel(const double* __restrict__ src, int n, double* __restrict__ dst, i64 ldd) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = by + k, c = bx + threadIdx.x;
    tile[k][threadIdx.x] = (r < n && c < n) ? src[static_cast<i64>(r) * n + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = bx + k, c = by + threadIdx.x;  // dst(c, r) = src(r', c')
    if (r < n && c < n) dst[c + static_cast<i64>(r) * ldd] = tile[threadIdx.x][k];
  }
}
// Z <- H_0 H_1 ... H_{n-3} Z, one warp per column of Z.
__global__ void backtransform_kernel(const double* H, i64 ldh, const double* tau, int n, double* Z, i64 ldz) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= n) return;
  double* z = Z + static_cast<i64>(col) * ldz;
  for (int k = n - 3; k >= 0; --k) {
    const double t = tau[k];
    if (t == 0.0) continue;
    const double* v = H + static_cast<i64>(k) * ldh;  // v_0 = 1 at row k+1
    double s = 0.0;
    for (int i = k + 1 + lane; i < n; i += 32) s += v[i] * z[i];
    s = warp_sum(s);
    const double ts = t * s;
    for (int i = k + 1 + lane; i < n; i += 32) z[i] -= ts * v[i];
  }
}

// Blocked: reflectors are staged 32 at a time in shared memory (one
// coalesced load per block, shared by the CTA's 8 columns), each warp applies
// them to its column of Z, also held in shared memory.
constexpr int BT_KB = 32;
__global__ void __launch_bounds__(256) backtransform_smem_kernel(const double* __restrict__ H, i64 ldh,
                                                                 const double* __restrict__ tau, int n, double* Z,
                                                                 i64 ldz) {
  extern __shared__ double bsm[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * nw + warp;
  double* vb = bsm;                                   // [BT_KB][n]: reflector k1 - kk at vb + kk*n
  double* z = bsm + static_cast<i64>(BT_KB) * n + static_cast<i64>(warp) * n;
  __shared__ double tb[BT_KB];
  if (col < n)
    for (int i = lane; i < n; i += 32) z[i] = Z[i + static_cast<i64>(col) * ldz];
  for (int k1 = n - 3; k1 >= 0; k1 -= BT_KB) {
    const int kb = min(BT_KB, k1 + 1);
    __syncthreads();
    for (int kk = warp; kk < kb; kk += nw) {
      const int k = k1 - kk;
      const double* v = H + static_cast<i64>(k) * ldh;
      for (int i = lane; i < n; i += 32) vb[static_cast<i64>(kk) * n + i] = i > k ? v[i] : 0.0;
      if (lane == 0) tb[kk] = tau[k];
    }
    __syncthreads();
    if (col < n) {
      for (int kk = 0; kk < kb; ++kk) {
        const double t = tb[kk];
        if (t == 0.0) continue;
        const int k = k1 - kk;
        const double* v = vb + static_cast<i64>(kk) * n;
        const int i0 = ((k + 1) & ~31) + lane;
        double s = 0.0;
        for (int i = i0; i < n; i += 32) s += v[i] * z[i];
        s = warp_sum(s);
        const double ts = t * s;
        for (int i = i0; i < n; i += 32) z[i] -= ts * v[i];
      }
    }
  }
  if (col < n)
    for (int i = lane; i < n; i += 32) Z[i + static_cast<i64>(col) * ldz] = z[i];
}

// Compact-WY back-transformation: the reflectors k in block b = [32b, 32b+31]
// multiply to P_b = H_{32b} ... H_{32b+31} = I - V_b T_b V_b^T (T_b upper
// triangular, dlarft 'F','C'), and Z <- P_0 P_1 ... Z is applied block by block
// (last block first) as Z -= V_b (T_b (V_b^T Z)): 32 independent dots per
// column instead of 32 dependent reflector applications.
constexpr int WY = 32;

// T_b from the Gram S = H^T H (its 32x32 diagonal blocks) and tau; one warp per block.
__global__ void wy_t_kernel(const double* __restrict__ S, i64 lds, const double* __restrict__ tau, int nref,
                            double* __restrict__ T) {
  __shared__ double Ts[WY][WY + 1];
  const int b = blockIdx.x, lane = threadIdx.x;
  const int k0 = b * WY, kb = min(WY, nref - k0);
  for (int idx = lane; idx < WY * (WY + 1); idx += 32) (&Ts[0][0])[idx] = 0.0;
  __syncwarp();
  for (int j = 0; j < kb; ++j) {
    const double tj = tau[k0 + j];
    // T[0:j, j] = -tau_j T[0:j, 0:j] (V^T v_j)[0:j]
    double acc = 0.0;
    if (lane < j)
      for (int c = lane; c < j; ++c) acc += Ts[lane][c] * S[(k0 + c) + static_cast<i64>(k0 + j) * lds];
    __syncwarp();
    if (lane < j) Ts[lane][j] = -tj * acc;
    if (lane == j) Ts[j][j] = tj;
    __syncwarp();
  }
  for (int idx = lane; idx < WY * WY; idx += 32) {
    const int r = idx % WY, c = idx / WY;
    T[static_cast<i64>(b) * WY * WY + r + c * WY] = Ts[r][c];
  }
}

// Z <- P_0 ... P_{nb-1} Z; CTA = 8 columns of Z (one warp each) kept in shared memory.
__global__ void __launch_bounds__(256) wy_apply_kernel(const double* __restrict__ H, i64 ldh,
                                                       const double* __restrict__ T, int nref, int n, double* Z,
                                                       i64 ldz) {
  extern __shared__ double wsm[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * nw + warp;
  double* vb = wsm;                                    // [WY][n]
  double* tb = vb + static_cast<i64>(WY) * n;          // [WY][WY] col-major
  double* z = tb + WY * WY + static_cast<i64>(warp) * n;
  if (col < n)
    for (int i = lane; i < n; i += 32) z[i] = Z[i + static_cast<i64>(col) * ldz];
  const int nblk = (nref + WY - 1) / WY;
  for (int b = nblk - 1; b >= 0; --b) {
    const int k0 = b * WY, kb = min(WY, nref - k0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < WY * n; idx += blockDim.x) {
      const int c = idx / n, i = idx % n;
      vb[idx] = c < kb ? H[i + static_cast<i64>(k0 + c) * ldh] : 0.0;
    }
    for (int idx = threadIdx.x; idx < WY * WY; idx += blockDim.x) tb[idx] = T[static_cast<i64>(b) * WY * WY + idx];
    __syncthreads();
    if (col >= n) continue;
    // w = V^T z: per-lane partials of all 32 dots, then a reduce-scatter (lane j ends with w_j)
    double acc[WY];
#pragma unroll
    for (int c = 0; c < WY; ++c) acc[c] = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double zi = z[i];
#pragma unroll
      for (int c = 0; c < WY; ++c) acc[c] += vb[c * n + i] * zi;
    }
#pragma unroll
    for (int sft = 16; sft >= 1; sft >>= 1) {
      const bool up = lane & sft;
#pragma unroll
      for (int c = 0; c < sft; ++c) {
        const double send = up ? acc[c] : acc[sft + c];
        const double keep = up ? acc[sft + c] : acc[c];
        acc[c] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
    const double w = acc[0];
    // u = T w (T upper triangular): lane j sums T[j][k] w_k, k >= j
    double u = 0.0;
#pragma unroll
    for (int k = 0; k < WY; ++k) {
      const double wk = __shfl_sync(0xffffffffu, w, k);
      if (k >= lane) u += tb[lane + k * WY] * wk;
    }
    double ua[WY];
#pragma unroll
    for (int c = 0; c < WY; ++c) ua[c] = __shfl_sync(0xffffffffu, u, c);
    // z -= V u
    for (int i = lane; i < n; i += 32) {
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < WY; ++c) sum += vb[c * n + i] * ua[c];
      z[i] -= sum;
    }
  }
  if (col < n)
    for (int i = lane; i < n; i += 32) Z[i + static_cast<i64>(col) * ldz] = z[i];
}

// The same back-transformation on the FP64 tensor pipe: CTA = 8 columns of Z
// in shared memory; per block, W = V_b^T Z_t (k split over the 8 warps,
// partials summed in fixed order), W' = T_b W, Z_t -= V_b W' (m-tiles over
// the warps), all products mma.sync.m8n8k4.f64. V_b is read from L2 once per
// CTA and block; shared rows padded to 33 doubles (conflict-free fragments).
constexpr int WYC = 8;
constexpr int VS = WY + 1;
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256) wy_apply_dmma_kernel(const double* __restrict__ H, i64 ldh,
                                                            const double* __restrict__ T, int nref, int n, double* Z,
                                                            i64 ldz) {
  extern __shared__ double wsm2[];
  const int np = (n + 7) & ~7;
  double* zt = wsm2;                             // [np][WYC]
  double* vb = zt + static_cast<i64>(np) * WYC;  // [np][VS]
  double* tb = vb + static_cast<i64>(np) * VS;   // [WY][WY] col-major
  double* wpart = tb + WY * WY;                  // [8][WY][WYC]
  double* wsh = wpart + 8 * WY * WYC;            // [WY][WYC]
  double* wq = wsh + WY * WYC;                   // [WY][WYC]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int col0 = blockIdx.x * WYC;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row / k index
  for (int idx = tid; idx < np * WYC; idx += 256) {
    const int i = idx / WYC, j = idx % WYC;
    zt[idx] = (i < n && col0 + j < n) ? Z[i + static_cast<i64>(col0 + j) * ldz] : 0.0;
  }
  const int nblk = (nref + WY - 1) / WY;
  const int ksteps = np / 4;
  const int kw0 = warp * ksteps / 8, kw1 = (warp + 1) * ksteps / 8;
  // V_b is prefetched into registers (thread: reflector tid / 8, rows tid % 8 + 8u)
  // while the previous block computes
  constexpr int NPRE = 64;  // np <= 512
  double pre[NPRE], tpre[WY * WY / 256];
  const int pc = tid >> 3, pr0 = tid & 7;
  auto issue = [&](int b) {
    const int k0 = b * WY, kb = min(WY, nref - k0);
#pragma unroll
    for (int u = 0; u < NPRE; ++u) {
      const int i = pr0 + 8 * u;
      pre[u] = (i < n && pc < kb) ? H[i + static_cast<i64>(k0 + pc) * ldh] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < WY * WY / 256; ++u) tpre[u] = T[static_cast<i64>(b) * WY * WY + tid + 256 * u];
  };
  issue(nblk - 1);
  for (int b = nblk - 1; b >= 0; --b) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NPRE; ++u)
      if (pr0 + 8 * u < np) vb[(pr0 + 8 * u) * VS + pc] = pre[u];
#pragma unroll
    for (int u = 0; u < WY * WY / 256; ++u) tb[tid + 256 * u] = tpre[u];
    __syncthreads();
    if (b > 0) issue(b - 1);
    // W = V_b^T Z_t: 4 m-tiles (reflectors) x 1 n-tile (columns), this warp's k-range
    double c[4][2] = {};
    for (int ks = kw0; ks < kw1; ++ks) {
      const int kr = ks * 4 + fk;
      const double bf = zt[kr * WYC + fr];
#pragma unroll
      for (int m = 0; m < 4; ++m) dmma884(c[m][0], c[m][1], vb[kr * VS + m * 8 + fr], bf);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int e = 0; e < 2; ++e) wpart[(warp * WY + m * 8 + fr) * WYC + 2 * fk + e] = c[m][e];
    __syncthreads();
    {
      const int r = tid / WYC, j = tid % WYC;
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += wpart[(w * WY + r) * WYC + j];  // fixed order
      wsh[r * WYC + j] = sacc;
    }
    __syncthreads();
    {
      const int r = tid / WYC, j = tid % WYC;  // W' = T W, T upper triangular
      double sacc = 0.0;
#pragma unroll
      for (int k = 0; k < WY; ++k) sacc += k >= r ? tb[r + k * WY] * wsh[k * WYC + j] : 0.0;
      wq[r * WYC + j] = sacc;
    }
    __syncthreads();
    // Z_t -= V_b W': m-tiles of 8 rows over the warps, K = 32 (8 k-steps)
    double bq[WY / 4];  // W' fragments, shared by every m-tile of the warp
#pragma unroll
    for (int ks = 0; ks < WY / 4; ++ks) bq[ks] = wq[(ks * 4 + fk) * WYC + fr];
    for (int mt = warp; mt < np / 8; mt += 16) {  // two m-tiles per pass: independent chains
      const int mt2 = mt + 8;
      const bool two = mt2 < np / 8;
      const int row = mt * 8 + fr, row2 = mt2 * 8 + fr;
      double c0 = zt[row * WYC + 2 * fk], c1 = zt[row * WYC + 2 * fk + 1];
      double d0 = two ? zt[row2 * WYC + 2 * fk] : 0.0, d1 = two ? zt[row2 * WYC + 2 * fk + 1] : 0.0;
#pragma unroll
      for (int ks = 0; ks < WY / 4; ++ks) {
        dmma884(c0, c1, -vb[row * VS + ks * 4 + fk], bq[ks]);
        if (two) dmma884(d0, d1, -vb[row2 * VS + ks * 4 + fk], bq[ks]);
      }
      zt[row * WYC + 2 * fk] = c0;
      zt[row * WYC + 2 * fk + 1] = c1;
      if (two) {
        zt[row2 * WYC + 2 * fk] = d0;
        zt[row2 * WYC + 2 * fk + 1] = d1;
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < n * WYC; idx += 256) {
    const int j = idx / n, i = idx % n;
    if (col0 + j < n) Z[i + static_cast<i64>(col0 + j) * ldz] = zt[i * WYC + j];
  }
}

}  // namespace

void sym_eigvecs(Ctx& ctx, double* M, i64 ldm, i64 n, double* Z, i64 ldz) {
  if (n <= 0) return;
  int nn = static_cast<int>(n);
  DBuf<double> d(n, ctx.stream), e(n, ctx.stream), tau(n, ctx.stream), p(2 * n, ctx.stream), lam(n, ctx.stream);
  DMat H;
  H.alloc(n, n, ctx.stream, true);
  bool done_tri = false;
  const char* tri_env = std::getenv("NPCG_TRIDIAG");  // diagnostics: "global"
  const std::string tri_mode = tri_env ? tri_env : "";
  if (n >= 3 && n <= 512 && tri_mode.empty()) {
    // register-resident cluster kernel: 8 CTAs up to n = 256, 16 up to 512
    const int C = n <= 256 ? 8 : 16;
    const size_t smem = static_cast<size_t>(5 * n * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(TRI_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = n <= 128 ? tridiag_reg_kernel<4> : n <= 256 ? tridiag_reg_kernel<8> : tridiag_reg_kernel<16>;
    NPCG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters >= 1) {
      static const bool tracing = std::getenv("NPCG_TRI_TRACE") != nullptr;  // diagnostics
      DBuf<unsigned long long> tr;
      if (tracing) {
        tr.alloc(64 * 6 + 16, ctx.stream);
        tr.zero();
      }
      ctx.prof_begin("tridiag_reg_kernel");
      NPCG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<const double*>(M), ldm, nn, d.p, e.p, tau.p, H.p(), H.ld,
                                   tracing ? tr.p : static_cast<unsigned long long*>(nullptr)));
      ctx.check_launch("tridiag_reg_kernel");
      ctx.prof_end();
      if (tracing) {
        ctx.sync();
        std::vector<unsigned long long> h(64 * 6 + 16);
        NPCG_CUDA(cudaMemcpy(h.data(), tr.p, 8 * h.size(), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[tri smid]");
        for (int r = 0; r < 16; ++r) std::fprintf(stderr, " %llu", h[64 * 6 + r]);
        std::fprintf(stderr, "\n");
        for (int k = 1; k < 40 && k + 1 < n - 2; k += 8)
          std::fprintf(stderr, "[tri-reg n=%d] k=%d colred %.2f scal %.2f fused %.2f csync %.2f gather %.2f tail %.2f us\n",
                       nn, k, (h[k * 6 + 1] - h[k * 6]) * 1e-3, (h[k * 6 + 2] - h[k * 6 + 1]) * 1e-3,
                       (h[k * 6 + 3] - h[k * 6 + 2]) * 1e-3, (h[k * 6 + 4] - h[k * 6 + 3]) * 1e-3,
                       (h[k * 6 + 5] - h[k * 6 + 4]) * 1e-3, (h[(k + 1) * 6] - h[k * 6 + 5]) * 1e-3);
      }
      done_tri = true;
    } else {
      (void)cudaGetLastError();
    }
  }
  if (n >= 3 && !done_tri) {
    const int smem = static_cast<int>(3 * n * 8);
    NPCG_CUDA(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   std::max(smem, 48 * 1024)));
    int per_sm = 0;
    NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_kernel, TRI_THREADS, smem));
    // enough CTAs to stream the trailing matrix, few enough for cheap barriers
    const int want = static_cast<int>(std::max<i64>(1, std::min<i64>(cdiv(n, 8), ctx.sm_count)));
    int grid = std::max(1, std::min(want, std::max(per_sm, 1) * ctx.sm_count));
    double* Mp = M;
    double* dp = d.p;
    double* ep = e.p;
    double* tp = tau.p;
    double* Hp = H.p();
    i64 ldh = H.ld;
    double* pp = p.p;
    void* args[] = {&Mp, &ldm, &nn, &dp, &ep, &tp, &Hp, &ldh, &pp};
    ctx.prof_begin("tridiag_kernel");
    NPCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tridiag_kernel), grid, TRI_THREADS, args, smem,
                                          ctx.stream));
    ctx.check_launch("tridiag_kernel");
    ctx.prof_end();
  } else if (n < 3) {
    // n <= 2: already tridiagonal
    std::vector<double> h(static_cast<size_t>(n * n));
    download(ctx, M, ldm, n, n, h.data(), n, NPCG_HOST);
    double hd[2] = {h[0], n == 2 ? h[3] : 0.0}, he[2] = {n == 2 ? h[1] : 0.0, 0.0}, ht[2] = {0.0, 0.0};
    NPCG_CUDA(cudaMemcpyAsync(d.p, hd, 8 * n, cudaMemcpyHostToDevice, ctx.stream));
    NPCG_CUDA(cudaMemcpyAsync(e.p, he, 8 * n, cudaMemcpyHostToDevice, ctx.stream));
    NPCG_CUDA(cudaMemcpyAsync(tau.p, ht, 8 * n, cudaMemcpyHostToDevice, ctx.stream));
    ctx.sync();
  }
  DBuf<double> e2(n, ctx.stream), info(4, ctx.stream);
  NPCG_LAUNCH(ctx, tri_bounds_kernel, 1, 256, 0, d.p, e.p, nn, e2.p, info.p);
  NPCG_LAUNCH(ctx, bisect_kernel, static_cast<unsigned>(cdiv(n * 32, 256)), 256, 0, d.p, e2.p, nn, info.p, lam.p);
  DBuf<double> zr(n * n, ctx.stream);
  const i64 per_vec = 4 * n * 8;
  const int V = static_cast<int>(std::min<i64>(8, (200 * 1024) / per_vec));
  if (V >= 1) {
    const int smem = static_cast<int>(V * per_vec);
    NPCG_CUDA(cudaFuncSetAttribute(invit_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    NPCG_LAUNCH(ctx, invit_smem_kernel, static_cast<unsigned>(cdiv(n, V)), V, smem, d.p, e.p, lam.p, nn, info.p,
                zr.p);
  } else {
    DBuf<double> iw(4 * n * n, ctx.stream);
    DBuf<unsigned char> ipv(n * n, ctx.stream);
    NPCG_LAUNCH(ctx, invit_kernel, static_cast<unsigned>(cdiv(n, 64)), 64, 0, d.p, e.p, lam.p, nn, info.p, zr.p,
                iw.p, ipv.p);
  }
  NPCG_LAUNCH(ctx, transpose_sq_kernel, dim3(static_cast<unsigned>(cdiv(n, 32)), static_cast<unsigned>(cdiv(n, 32))),
              dim3(32, 8), 0, zr.p, nn, Z, ldz);
  const int nref = nn - 2;  // reflectors k = 0 .. n-3
  if (nref >= 1 && (static_cast<i64>(WY + 8) * n + WY * WY) * 8 <= 200 * 1024) {
    // compact WY: T blocks from the diagonal blocks of H^T H (one DMMA GEMM)
    const int nblk = (nref + WY - 1) / WY;
    DMat S;
    S.alloc(n, n, ctx.stream, false);
    gemm(ctx, n, n, n, 1.0, Operand{H.p(), H.ld, true}, Operand{H.p(), H.ld, true}, 0.0, S.p(), S.ld);
    DBuf<double> Tw(static_cast<i64>(nblk) * WY * WY, ctx.stream);
    NPCG_LAUNCH(ctx, wy_t_kernel, static_cast<unsigned>(nblk), 32, 0, S.p(), S.ld, tau.p, nref, Tw.p);
    const i64 np = round_up(n, 8);
    const i64 smem2 = (np * (WYC + VS) + WY * WY + 10 * WY * WYC) * 8;  // (np <= 512: the register prefetch)
    static const bool no_dmma = std::getenv("NPCG_WY") && std::string(std::getenv("NPCG_WY")) == "fma";  // diagnostics
    if (np <= 512 && smem2 <= 220 * 1024 && !no_dmma) {
      NPCG_CUDA(cudaFuncSetAttribute(wy_apply_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem2)));
      NPCG_LAUNCH(ctx, wy_apply_dmma_kernel, static_cast<unsigned>(cdiv(n, WYC)), 256, static_cast<int>(smem2), H.p(),
                  H.ld, Tw.p, nref, nn, Z, ldz);
    } else {
      const int smem = static_cast<int>((static_cast<i64>(WY + 8) * n + WY * WY) * 8);
      NPCG_CUDA(cudaFuncSetAttribute(wy_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      NPCG_LAUNCH(ctx, wy_apply_kernel, static_cast<unsigned>(cdiv(n, 8)), 256, smem, H.p(), H.ld, Tw.p, nref, nn,
                  Z, ldz);
    }
  } else {
    NPCG_LAUNCH(ctx, backtransform_kernel, static_cast<unsigned>(cdiv(n * 32, 256)), 256, 0, H.p(), H.ld, tau.p, nn,
                Z, ldz);
  }
}

}  // namespace npcg
