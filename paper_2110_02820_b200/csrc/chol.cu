// Fused Cholesky + explicit inverse of the lower factor, one cooperative
// launch (see factor.cuh: cholesky()).
//
// Right-looking, 32 x 32 tiles, one grid-wide barrier per block column b:
//   D(b)  one warp factors the diagonal tile (lane = row; pivots broadcast by
//         shuffle, l = a * rsqrt(d) -- no division on the serial chain) and
//         inverts it (lane = column of the inverse).
//   U(b)  every CTA takes tiles of the remaining work, all independent:
//           trailing  A_ij -= L_ib L_jb^T              b < j <= i
//           inverse   W_ij -= L_ib X_bj                b < i, j <= b
//         where L_ib = A_ib Dinv_b^T and X_bj = Dinv_b W_bj are recomputed
//         per tile from tiles nobody writes during U(b) (the factor goes to a
//         separate buffer), so U(b) needs no internal barrier. W starts as I:
//         solving L X = I rides along with the factorisation (X = L^{-1}).
//         CTA 0 owns tile (b+1, b+1) and factors D(b+1) right after its update.
// The inverse turns every triangular solve of the pipeline (Y L^{-T}) into
// one DMMA GEMM. Tiles are FP64 CUDA-core products staged in shared memory
// (32^3 per tile; the whole factorisation is latency-, not flop-bound).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "factor.cuh"

namespace npcg {
namespace {

namespace cg = cooperative_groups;

constexpr int CB = 32;           // tile size
constexpr int CT = 256;          // threads per CTA
constexpr int TS = CB + 1;       // smem row stride (conflict-free column reads)
constexpr int NTILE = 6;         // smem tiles per CTA

struct CholArgs {
  double* a;     // working matrix (lower part read, trailing part updated in place)
  i64 lda;
  int n, nb;
  double* L;     // factor (n x n, ld ldw)
  double* W;     // inverse workspace, starts as I (n x n)
  double* X;     // L^{-1} (n x n)
  i64 ldw;
  double* dinv;  // nb tiles CB x CB col-major
  int* flag;
  unsigned long long* trace;  // diagnostics (NPCG_CHOL_TRACE): CTA 0 phase timestamps, nullable
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

using Tile = double[CB][TS];

// rows/cols of tile index t (clipped to n)
__device__ __forceinline__ int tile_rows(int t, int n) { return min(CB, n - t * CB); }

// smem T[r][k] = M(r0 + r, c0 + k) (zero outside rows < nr, cols < nc)
__device__ __forceinline__ void load_tile(Tile& T, const double* M, i64 ld, i64 r0, i64 c0, int nr, int nc) {
  for (int idx = threadIdx.x; idx < CB * CB; idx += CT) {
    const int r = idx & 31, k = idx >> 5;
    T[r][k] = (r < nr && k < nc) ? M[(r0 + r) + (c0 + k) * ld] : 0.0;
  }
}
// smem T[c][k] = M(r0 + k, c0 + c)  (transposed load)
__device__ __forceinline__ void load_tile_t(Tile& T, const double* M, i64 ld, i64 r0, i64 c0, int nr, int nc) {
  for (int idx = threadIdx.x; idx < CB * CB; idx += CT) {
    const int k = idx & 31, c = idx >> 5;
    T[c][k] = (k < nr && c < nc) ? M[(r0 + k) + (c0 + c) * ld] : 0.0;
  }
}
// dinv tile b (col-major CB x CB) -> smem D[r][k]
__device__ __forceinline__ void load_dinv(Tile& D, const double* dinv) {
  for (int idx = threadIdx.x; idx < CB * CB; idx += CT) {
    const int r = idx & 31, k = idx >> 5;
    D[r][k] = dinv[r + k * CB];
  }
}

// acc[q] = sum_k A[r][k] B[c0+q][k]  with r = tid & 31, c0 = 4 (tid >> 5)
__device__ __forceinline__ void mul_abt(const Tile& A, const Tile& B, double acc[4]) {
  const int r = threadIdx.x & 31, c0 = (threadIdx.x >> 5) * 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = 0.0;
#pragma unroll 8
  for (int k = 0; k < CB; ++k) {
    const double av = A[r][k];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += av * B[c0 + q][k];
  }
}
__device__ __forceinline__ void store_acc(Tile& C, const double acc[4]) {
  const int r = threadIdx.x & 31, c0 = (threadIdx.x >> 5) * 4;
#pragma unroll
  for (int q = 0; q < 4; ++q) C[r][c0 + q] = acc[q];
}
// Factor + invert the diagonal tile held in smem T (lower part; rows >= nr
// padded with the identity). Warp 0 only: L goes back to T, L^{-1} to Xs
// (both [row][col]); the caller publishes them with the whole CTA. Returns
// false (uniform in the warp) on a non-positive pivot.
__device__ __noinline__ bool diag_factor(Tile& T, Tile& Xs, int nr) {
  const int lane = threadIdx.x & 31;
  double row[CB];
#pragma unroll
  for (int k = 0; k < CB; ++k) row[k] = lane < nr ? (k < nr ? T[lane][k] : 0.0) : (k == lane ? 1.0 : 0.0);
  __shared__ double rs[CB];      // 1 / L_jj (identical in every lane)
  __shared__ double lv[2][CB];   // column j of L, broadcast through shared memory
  bool ok = true;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    double d = __shfl_sync(0xffffffffu, row[j], j);
    if (!(d > 0.0) || !isfinite(d)) {  // uniform: d is the broadcast pivot
      ok = false;
      d = 1.0;
    }
    const double r = rsqrt(d);
    if (lane == 0) rs[j] = r;
    const double l = lane == j ? d * r : row[j] * r;
    if (lane >= j) row[j] = l;
    // the next pivot's column first: its multiplier comes by one shuffle, so
    // the chain to the next step is shfl -> rsqrt -> mul -> shfl -> fma
    if (j + 1 < CB) {
      const double ln = __shfl_sync(0xffffffffu, l, j + 1);
      if (lane >= j + 1) row[j + 1] -= l * ln;
    }
    lv[j & 1][lane] = l;
    __syncwarp();
#pragma unroll
    for (int c = j + 2; c < CB; ++c) {  // off the critical path
      const double lc = lv[j & 1][c];
      if (lane >= c) row[c] -= l * lc;
    }
  }
  if (!ok) return false;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < CB; ++k) T[lane][k] = k <= lane ? row[k] : 0.0;
  __syncwarp();
  // X = L^{-1}, lane c computes column c, right-looking: once x_k is final,
  // every later row takes its contribution at once (short dependency chain).
  double x[CB];
#pragma unroll
  for (int i = 0; i < CB; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < CB; ++k) {
    x[k] *= rs[k];  // rows < lane stay exactly 0
#pragma unroll
    for (int i = k + 1; i < CB; ++i) x[i] -= T[i][k] * x[k];
  }
#pragma unroll
  for (int i = 0; i < CB; ++i) Xs[i][lane] = x[i];
  return true;
}

// Publish the factored diagonal tile b (T = L_bb, Xs = L_bb^{-1}) with the whole CTA.
__device__ __forceinline__ void publish_diag(const Tile& T, const Tile& Xs, int b, int nr, const CholArgs& a) {
  const i64 o = static_cast<i64>(b) * CB;
  double* dv = a.dinv + static_cast<i64>(b) * CB * CB;
  for (int idx = threadIdx.x; idx < CB * CB; idx += CT) {
    const int i = idx & 31, k = idx >> 5;
    dv[i + k * CB] = Xs[i][k];
    if (i < nr && k < nr) a.L[(o + i) + (o + k) * a.ldw] = k <= i ? T[i][k] : 0.0;
  }
}

__global__ void __launch_bounds__(CT) chol_fused_kernel(const CholArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double csm[];
  Tile* tl = reinterpret_cast<Tile*>(csm);
  Tile &Dn = tl[0], &Ai = tl[1], &Aj = tl[2], &Li = tl[3], &Lj = tl[4], &Ct = tl[5];
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, nb = a.nb;
  const int r = tid & 31, c0 = (tid >> 5) * 4;
  volatile int* flag = a.flag;

  // W = I (lower tiles only are ever read)
  for (i64 idx = static_cast<i64>(bid) * CT + tid; idx < static_cast<i64>(n) * n; idx += static_cast<i64>(G) * CT) {
    const i64 i = idx % n, j = idx / n;
    a.W[i + j * a.ldw] = i == j ? 1.0 : 0.0;
  }
  if (bid == 0) {
    load_tile(Ct, a.a, a.lda, 0, 0, tile_rows(0, n), tile_rows(0, n));
    __syncthreads();
    if (tid < 32 && !diag_factor(Ct, Lj, tile_rows(0, n)) && tid == 0) *flag = 1;
    __syncthreads();
    if (!*flag) publish_diag(Ct, Lj, 0, tile_rows(0, n), a);
  }
  grid.sync();
  if (*flag) return;

  for (int b = 0; b < nb - 1; ++b) {
    const int T = nb - 1 - b;
    const int ntrail = T * (T + 1) / 2, ninv = T * (b + 1);
    const i64 ob = static_cast<i64>(b) * CB;
    const int nrb = tile_rows(b, n);
    bool have_dinv = false;
    if (a.trace && bid == 0 && tid == 0) a.trace[4 * b] = gtimer();
    for (int q = bid; q < ntrail + ninv; q += G) {
      if (!have_dinv) {
        load_dinv(Dn, a.dinv + static_cast<i64>(b) * CB * CB);
        have_dinv = true;
      }
      double acc[4];
      if (q < ntrail) {  // ---- trailing tile (i, j), b < j <= i
        int ii = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
        while (ii * (ii + 1) / 2 > q) --ii;
        while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
        const int jj = q - ii * (ii + 1) / 2;
        const int ti = b + 1 + ii, tj = b + 1 + jj;
        const int nri = tile_rows(ti, n), nrj = tile_rows(tj, n);
        const i64 oi = static_cast<i64>(ti) * CB, oj = static_cast<i64>(tj) * CB;
        load_tile(Ai, a.a, a.lda, oi, ob, nri, nrb);
        if (tj != ti) load_tile(Aj, a.a, a.lda, oj, ob, nrj, nrb);
        double old[4];  // destination values, fetched early (off the dependency chain)
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int c = c0 + qq;
          old[qq] = (r < nri && c < nrj && (ti != tj || c <= r)) ? a.a[(oi + r) + (oj + c) * a.lda] : 0.0;
        }
        __syncthreads();
        mul_abt(Ai, Dn, acc);  // L_ib = A_ib Dinv_b^T
        store_acc(Li, acc);
        if (tj != ti) {
          mul_abt(Aj, Dn, acc);
          store_acc(Lj, acc);
        }
        __syncthreads();
        if (ti == tj) {  // the diagonal-tile owner publishes L_ib
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            if (r < nri && c0 + qq < nrb) a.L[(oi + r) + (ob + c0 + qq) * a.ldw] = Li[r][c0 + qq];
        }
        mul_abt(Li, ti == tj ? Li : Lj, acc);  // A_ij -= L_ib L_jb^T
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int c = c0 + qq;
          if (r < nri && c < nrj && (ti != tj || c <= r)) {
            const double v = old[qq] - acc[qq];
            a.a[(oi + r) + (oj + c) * a.lda] = v;
            if (ti == b + 1 && tj == b + 1) Ct[r][c] = v;
          }
        }
        if (ti == b + 1 && tj == b + 1) {  // D(b+1) right away (CTA 0, q == 0)
          __syncthreads();
          if (a.trace && tid == 0) a.trace[4 * b + 1] = gtimer();
          if (tid < 32 && !diag_factor(Ct, Lj, nri) && tid == 0) *flag = 1;
          __syncthreads();
          if (!*flag) publish_diag(Ct, Lj, b + 1, nri, a);
          if (a.trace && tid == 0) a.trace[4 * b + 2] = gtimer();
        }
        __syncthreads();
      } else {  // ---- inverse tile: W_ij -= L_ib X_bj,  b < i, j <= b
        const int qi = q - ntrail;
        const int ti = b + 1 + qi / (b + 1), tj = qi % (b + 1);
        const int nri = tile_rows(ti, n), nrj = tile_rows(tj, n);
        const i64 oi = static_cast<i64>(ti) * CB, oj = static_cast<i64>(tj) * CB;
        load_tile(Ai, a.a, a.lda, oi, ob, nri, nrb);       // A_ib
        load_tile_t(Aj, a.W, a.ldw, ob, oj, nrb, nrj);     // W_bj^T
        double old[4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int c = c0 + qq;
          old[qq] = (r < nri && c < nrj) ? a.W[(oi + r) + (oj + c) * a.ldw] : 0.0;
        }
        __syncthreads();
        mul_abt(Ai, Dn, acc);                              // L_ib
        store_acc(Li, acc);
        mul_abt(Aj, Dn, acc);                              // (Dinv_b W_bj)^T = X_bj^T
        store_acc(Lj, acc);
        __syncthreads();
        if (ti == b + 1) {  // one owner per j publishes X_bj
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int c = c0 + qq;  // X_bj[c][r] = Lj[r][c]... (Lj holds X_bj^T: Lj[col][row])
            if (c < nrb && r < nrj) a.X[(ob + c) + (oj + r) * a.ldw] = Lj[r][c];
          }
        }
        mul_abt(Li, Lj, acc);  // (L_ib X_bj)[r][c] = sum_k L_ib[r][k] X_bj^T[c][k]
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int c = c0 + qq;
          if (r < nri && c < nrj) a.W[(oi + r) + (oj + c) * a.ldw] = old[qq] - acc[qq];
        }
        __syncthreads();
      }
    }
    if (a.trace && bid == 0 && tid == 0) a.trace[4 * b + 3] = gtimer();
    grid.sync();
    if (*flag) return;
  }
  // last block row of X: X_{nb-1, j} = Dinv W_{nb-1, j}; zero the upper triangle of X
  {
    const int b = nb - 1;
    const i64 ob = static_cast<i64>(b) * CB;
    const int nrb = tile_rows(b, n);
    for (int tj = bid; tj < nb; tj += G) {
      const int nrj = tile_rows(tj, n);
      const i64 oj = static_cast<i64>(tj) * CB;
      load_dinv(Dn, a.dinv + static_cast<i64>(b) * CB * CB);
      load_tile_t(Aj, a.W, a.ldw, ob, oj, nrb, nrj);
      __syncthreads();
      double acc[4];
      mul_abt(Aj, Dn, acc);  // X_bj^T[r = col j][c = row b]
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int c = c0 + qq;
        if (c < nrb && r < nrj) a.X[(ob + c) + (oj + r) * a.ldw] = acc[qq];
      }
      __syncthreads();
    }
  }
  for (i64 idx = static_cast<i64>(bid) * CT + tid; idx < static_cast<i64>(n) * n; idx += static_cast<i64>(G) * CT) {
    const i64 i = idx % n, j = idx / n;
    if (i < j) {
      a.X[i + j * a.ldw] = 0.0;
      a.a[i + j * a.lda] = 0.0;
    } else {
      a.a[i + j * a.lda] = a.L[i + j * a.ldw];
    }
  }
}

}  // namespace

bool cholesky_fused(Ctx& ctx, double* A, i64 n, i64 lda, CholFactor& f) {
  const int nb = static_cast<int>(cdiv(n, CB));
  DMat Lw, Ww;
  Lw.alloc(n, n, ctx.stream, false);
  Ww.alloc(n, n, ctx.stream, false);
  f.linv.alloc(n, n, ctx.stream, false);
  f.dinv.alloc(static_cast<i64>(nb) * CB * CB, ctx.stream);
  f.n = n;
  f.nb = CB;
  DBuf<int> flag(1, ctx.stream);
  flag.zero();
  if (Lw.ld != f.linv.ld || Ww.ld != f.linv.ld) fail(NPCG_ERUNTIME, "cholesky_fused: layout");
  DBuf<unsigned long long> trace;
  static const bool tracing = std::getenv("NPCG_CHOL_TRACE") != nullptr;
  if (tracing) {
    trace.alloc(4 * nb, ctx.stream);
    trace.zero();
  }
  CholArgs args{A, lda, static_cast<int>(n), nb, Lw.p(), Ww.p(), f.linv.p(), f.linv.ld, f.dinv.p, flag.p,
                tracing ? trace.p : nullptr};
  constexpr int smem = NTILE * CB * TS * 8;
  static bool attr = false;
  if (!attr) {
    NPCG_CUDA(cudaFuncSetAttribute(chol_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  int per_sm = 0;
  NPCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_fused_kernel, CT, smem));
  const i64 t1 = static_cast<i64>(nb - 1) * nb / 2 + (nb - 1);  // widest U phase (b = 0)
  const int G = static_cast<int>(std::max<i64>(1, std::min<i64>(t1, static_cast<i64>(std::max(per_sm, 1)) * ctx.sm_count)));
  int G2 = G;
  if (const char* g = std::getenv("NPCG_CHOL_GRID")) G2 = std::max(1, std::min(G, std::atoi(g)));  // diagnostics
  void* kargs[] = {&args};
  ctx.prof_begin("chol_fused_kernel");
  NPCG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(chol_fused_kernel), G2, CT, kargs, smem, ctx.stream));
  ctx.check_launch("chol_fused_kernel");
  ctx.prof_end();
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (tracing) {
    std::vector<unsigned long long> tr(4 * nb);
    NPCG_CUDA(cudaMemcpy(tr.data(), trace.p, 8 * tr.size(), cudaMemcpyDeviceToHost));
    for (int b = 0; b + 1 < nb; ++b)
      std::fprintf(stderr, "[chol n=%lld] b=%d tile->D %.2f us  D %.2f us  D->end %.2f us  end->next %.2f us\n",
                   static_cast<long long>(n), b, (tr[4 * b + 1] - tr[4 * b]) * 1e-3,
                   (tr[4 * b + 2] - tr[4 * b + 1]) * 1e-3, (tr[4 * b + 3] - tr[4 * b + 2]) * 1e-3,
                   b + 2 < nb ? (tr[4 * b + 4] - tr[4 * b + 3]) * 1e-3 : 0.0);
  }
  return h == 0;
}

}  // namespace npcg
