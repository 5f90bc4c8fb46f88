// Level-1/2 kernels. The two skinny GEMV shapes of the hot path:
//
//  coldot  out(j,s) = M(:,j) . X(:,s)   — each output is a dot of one
//          contiguous column with X. Serves A·p for symmetric stored A
//          (column i of A == row i) and U^T r of the preconditioner.
//          A warp streams 4 columns at once with 16-byte loads (4 x 16 B per
//          lane per step, unrolled x4 -> 256 B in flight per lane), X is read
//          through L1 and reused across the 4 columns. Short/wide problems
//          split the rows across CTAs; partials are summed in fixed order.
//  rowdot  out(i,s) = base(i,s) + M(i,:) . c(:,s) — a thread owns a row pair
//          (16-byte loads, coalesced across the warp), c is broadcast from
//          L1. Serves U (g ⊙ t) of the preconditioner and X v of the Gram op.
//
// Both are HBM-bound: algorithmic bytes = 8 * nrows * ncols per call.
#include <math_constants.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "blas.cuh"

namespace npcg {
namespace {

constexpr int CPW = 4;            // columns per warp (coldot)
constexpr int CD_WARPS = 8;       // warps per CTA (coldot)
constexpr int CD_COLS = CPW * CD_WARPS;
constexpr int RD_THREADS = 256;   // rowdot: 2 rows per thread, c staged in shared memory
constexpr int RD_SMEM_MAX = 48 * 1024;

template <int S>
__global__ void __launch_bounds__(256) coldot_kernel(const double* __restrict__ M, i64 ldm, i64 nrows, i64 ncols,
                                                     const double* __restrict__ X, i64 ldx, i64 rows_per_split,
                                                     double* __restrict__ out, i64 ldo, double mu,
                                                     const double* __restrict__ shift, i64 ldsh,
                                                     double* __restrict__ partial, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 j0 = static_cast<i64>(blockIdx.x) * CD_COLS + warp * CPW;
  if (j0 >= ncols) return;
  const i64 r0 = static_cast<i64>(blockIdx.y) * rows_per_split;
  const i64 r1 = min(nrows, r0 + rows_per_split);
  double acc[CPW][S];
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int s = 0; s < S; ++s) acc[c][s] = 0.0;
  const double* col[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) col[c] = M + min(j0 + c, ncols - 1) * ldm;

  i64 i = r0 + 2 * lane;
  // main loop: UN row-pairs per lane per trip (fewer for many right-hand
  // sides: the x registers would cap occupancy)
  constexpr int UN = S <= 2 ? 4 : 2;
  for (; i + (UN - 1) * 64 + 1 < r1; i += UN * 64) {
    double2 a[UN][CPW], x[UN][S];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
#pragma unroll
      for (int c = 0; c < CPW; ++c) a[u][c] = __ldg(reinterpret_cast<const double2*>(col[c] + i + u * 64));
#pragma unroll
      for (int s = 0; s < S; ++s) x[u][s] = __ldg(reinterpret_cast<const double2*>(X + s * ldx + i + u * 64));
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
#pragma unroll
      for (int c = 0; c < CPW; ++c)
#pragma unroll
        for (int s = 0; s < S; ++s) acc[c][s] += a[u][c].x * x[u][s].x + a[u][c].y * x[u][s].y;
  }
  for (; i < r1; i += 64) {
    const bool two = i + 1 < r1;
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const double a0 = col[c][i], a1 = two ? col[c][i + 1] : 0.0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double x0 = X[s * ldx + i], x1 = two ? X[s * ldx + i + 1] : 0.0;
        acc[c][s] += a0 * x0 + a1 * x1;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c)
#pragma unroll
    for (int s = 0; s < S; ++s) acc[c][s] = warp_sum(acc[c][s]);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const i64 j = j0 + c;
      if (j >= ncols) break;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (partial) {
          partial[(static_cast<i64>(blockIdx.y) * S + s) * ncols + j] = acc[c][s];
        } else {
          double v = acc[c][s];
          if (shift) v = __dadd_rn(v, __dmul_rn(mu, shift[j + s * ldsh]));  // out += mu v, unfused (operators.cpp:97)
          out[j + s * ldo] = v;
        }
      }
    }
  }
}

__global__ void coldot_reduce_kernel(const double* __restrict__ partial, int splits, i64 ncols, int S,
                                     double* __restrict__ out, i64 ldo, double mu,
                                     const double* __restrict__ shift, i64 ldsh, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= ncols * S) return;
  const i64 j = idx % ncols, s = idx / ncols;
  double v = 0.0;
  for (int k = 0; k < splits; ++k) v += partial[(static_cast<i64>(k) * S + s) * ncols + j];
  if (shift) v = __dadd_rn(v, __dmul_rn(mu, shift[j + s * ldsh]));  // out += mu v, unfused (operators.cpp:97)
  out[j + s * ldo] = v;
}

template <int S>
__global__ void __launch_bounds__(RD_THREADS) rowdot_kernel(const double* __restrict__ M, i64 ldm, i64 nrows,
                                                            i64 ncols, const double* __restrict__ c, i64 ldc,
                                                            i64 cols_per_split, const double* __restrict__ base,
                                                            i64 ldb, double* __restrict__ out, i64 ldo,
                                                            double* __restrict__ partial,
                                                            const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  extern __shared__ double cs[];  // c[k0:k1, :] as [k][S]
  const i64 k0 = static_cast<i64>(blockIdx.y) * cols_per_split;
  const i64 k1 = min(ncols, k0 + cols_per_split);
  const int kc = static_cast<int>(k1 - k0);
  for (int idx = threadIdx.x; idx < kc * S; idx += RD_THREADS) {
    const int kk = idx / S, s = idx % S;
    cs[idx] = c[s * ldc + k0 + kk];
  }
  __syncthreads();
  const i64 i = (static_cast<i64>(blockIdx.x) * RD_THREADS + threadIdx.x) * 2;
  if (i >= nrows) return;
  const bool two = i + 1 < nrows;
  double acc0[S], acc1[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc0[s] = acc1[s] = 0.0;
  const double* mp = M + k0 * ldm + i;
  int k = 0;
  constexpr int U = 8;  // 8 x 16 B loads in flight per thread
  for (; k + U - 1 < kc; k += U) {
    double2 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldg(reinterpret_cast<const double2*>(mp + (k + u) * ldm));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const double cv = cs[(k + u) * S + s];
        acc0[s] += a[u].x * cv;
        acc1[s] += a[u].y * cv;
      }
  }
  for (; k < kc; ++k) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(mp + k * ldm));
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double cv = cs[k * S + s];
      acc0[s] += a.x * cv;
      acc1[s] += a.y * cv;
    }
  }
  if (partial) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double* pp = partial + (static_cast<i64>(blockIdx.y) * S + s) * nrows;
      pp[i] = acc0[s];
      if (two) pp[i + 1] = acc1[s];
    }
  } else {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double b0 = base ? base[s * ldb + i] : 0.0;
      out[s * ldo + i] = b0 + acc0[s];
      if (two) out[s * ldo + i + 1] = (base ? base[s * ldb + i + 1] : 0.0) + acc1[s];
    }
  }
}

__global__ void rowdot_reduce_kernel(const double* __restrict__ partial, int splits, i64 nrows, int S,
                                     const double* __restrict__ base, i64 ldb, double* __restrict__ out,
                                     i64 ldo, const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  const i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= nrows * S) return;
  const i64 i = idx % nrows, s = idx / nrows;
  double v = 0.0;
  for (int k = 0; k < splits; ++k) v += partial[(static_cast<i64>(k) * S + s) * nrows + i];
  out[s * ldo + i] = (base ? base[s * ldb + i] : 0.0) + v;
}

__global__ void copy2d_kernel(i64 rows, i64 cols, const double* __restrict__ src, i64 lds, double* __restrict__ dst,
                              i64 ldd) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

__global__ void nonfinite_kernel(const double* __restrict__ p, i64 rows, i64 cols, i64 ld, int* flag) {
  const i64 total = rows * cols;
  int bad = 0;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    if (!isfinite(p[i + j * ld])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void sumsq_partial_kernel(const double* __restrict__ p, i64 rows, i64 cols, i64 ld, double* partial) {
  __shared__ double sh[32];
  const i64 total = rows * cols;
  double s = 0.0;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    const double v = p[i + j * ld];
    s += v * v;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int n, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += partial[k];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__device__ __forceinline__ unsigned long long dbits(double v) { return static_cast<unsigned long long>(__double_as_longlong(v)); }

__global__ void symstats_kernel(const double* __restrict__ a, i64 n, i64 ld, unsigned long long* out) {
  const i64 total = n * n;
  double asym = 0.0, amax = 0.0;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    const double v = a[i + j * ld];
    amax = fmax(amax, fabs(v));
    asym = fmax(asym, fabs(v - a[j + i * ld]));
    if (isnan(v)) amax = CUDART_INF;  // NaN never passes max-based checks
  }
  asym = warp_max(asym);
  amax = warp_max(amax);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out + 0, dbits(asym));
    atomicMax(out + 1, dbits(amax));
  }
}

__global__ void axpby_kernel(i64 rows, i64 cols, double a, const double* __restrict__ x, double b, double* y, i64 ld) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 o = idx % rows + idx / rows * ld;
    y[o] = __dadd_rn(__dmul_rn(a, x[o]), __dmul_rn(b, y[o]));  // unfused, as Eigen evaluates it
  }
}

__global__ void add_scaled_kernel(i64 rows, i64 cols, const double* __restrict__ a, double nu,
                                  const double* __restrict__ b, double* __restrict__ out, i64 ld) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 o = idx % rows + idx / rows * ld;
    out[o] = __dadd_rn(a[o], __dmul_rn(nu, b[o]));  // Y + nu Omega unfused (nystrom.cpp:113)
  }
}

__global__ void add2d_kernel(i64 rows, i64 cols, const double* __restrict__ a, i64 lda,
                             const double* __restrict__ b, i64 ldb, double* __restrict__ out, i64 ldo) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    out[i + j * ldo] = a[i + j * lda] + b[i + j * ldb];
  }
}

__global__ void symmetrize_kernel(const double* __restrict__ a, i64 n, i64 lda, double* __restrict__ out, i64 ldo) {
  const i64 total = n * n;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    out[i + j * ldo] = (a[i + j * lda] + a[j + i * lda]) / 2.0;
  }
}

// in place: each lower/upper pair is averaged by one thread (diagonal unchanged)
__global__ void symmetrize_inplace_kernel(double* __restrict__ a, i64 n, i64 lda) {
  const i64 total = n * n;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    if (i > j) {
      const double v = (a[i + j * lda] + a[j + i * lda]) / 2.0;
      a[i + j * lda] = v;
      a[j + i * lda] = v;
    }
  }
}

__global__ void scale_cols_kernel(double* a, i64 rows, i64 cols, i64 lda, const double* __restrict__ d) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    a[i + j * lda] *= d[j];
  }
}

__global__ void divide_kernel(i64 rows, i64 cols, double* y, i64 ld, double d) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 o = idx % rows + idx / rows * ld;
    y[o] = y[o] / d;
  }
}

__global__ void identity_kernel(double* a, i64 rows, i64 cols, i64 ld) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    a[i + j * ld] = i == j ? 1.0 : 0.0;
  }
}

unsigned grid_for(Ctx& ctx, i64 total) {
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cdiv(total, 256), ctx.sm_count * 8)));
}

}  // namespace

void copy2d(Ctx& ctx, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd) {
  if (rows <= 0 || cols <= 0) return;
  if (lds == ldd && lds == rows) {
    NPCG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  NPCG_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, rows * 8, cols, cudaMemcpyDeviceToDevice, ctx.stream));
}

namespace {
// Host (pageable) -> device copy of a rows x cols column-major block through the
// context's pinned ring: chunks of whole columns (or row pieces of one column)
// are packed into a 32 MB pinned slot by several host threads, then copied
// asynchronously on the context stream; the next chunk is packed while the
// previous one crosses PCIe. (A plain cudaMemcpy from pageable memory runs at
// ~12 GB/s here; the PCIe 5 x16 link carries ~54 GB/s.)
void h2d_pinned(Ctx& ctx, double* dst, i64 ldd, const double* src, i64 lds, i64 rows, i64 cols) {
  constexpr int NS = Ctx::kPinSlots;
  const i64 slot_doubles = Ctx::kPinSlotBytes / 8;
  if (!ctx.pin) {
    NPCG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx.pin), Ctx::kPinSlotBytes * NS, cudaHostAllocDefault));
    for (auto& ev : ctx.pin_free) NPCG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : ctx.pin_free) NPCG_CUDA(cudaEventRecord(ev, ctx.stream));
  }
  const i64 rpc = std::min(rows, slot_doubles);                       // rows per piece
  const i64 cpc = rpc == rows ? std::max<i64>(1, slot_doubles / rows) : 1;  // columns per chunk
  const int nthr = static_cast<int>(std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2)));
  int q = 0;
  for (i64 c0 = 0; c0 < cols; c0 += cpc) {
    const i64 nc = std::min(cpc, cols - c0);
    for (i64 r0 = 0; r0 < rows; r0 += rpc, q = (q + 1) % NS) {
      const i64 nr = std::min(rpc, rows - r0);
      double* slot = reinterpret_cast<double*>(ctx.pin + q * Ctx::kPinSlotBytes);
      NPCG_CUDA(cudaEventSynchronize(ctx.pin_free[q]));  // the slot's previous copy has landed
      auto pack = [&](int t) {  // thread t: an equal share of the chunk's bytes
        const i64 total = nr * nc, a = total * t / nthr, b = total * (t + 1) / nthr;
        for (i64 e = a; e < b;) {
          const i64 c = e / nr, r = e % nr, len = std::min(nr - r, b - e);
          std::memcpy(slot + c * nr + r, src + (c0 + c) * lds + r0 + r, len * 8);
          e += len;
        }
      };
      if (nr * nc * 8 < (i64{4} << 20) || nthr == 1) {
        for (int t = 0; t < nthr; ++t) pack(t);
      } else {
        std::vector<std::thread> th;
        for (int t = 1; t < nthr; ++t) th.emplace_back(pack, t);
        pack(0);
        for (auto& x : th) x.join();
      }
      NPCG_CUDA(cudaMemcpy2DAsync(dst + r0 + c0 * ldd, ldd * 8, slot, nr * 8, nr * 8, nc, cudaMemcpyHostToDevice,
                                  ctx.stream));
      NPCG_CUDA(cudaEventRecord(ctx.pin_free[q], ctx.stream));
    }
  }
}
}  // namespace

void upload(Ctx& ctx, DMat& dst, i64 rows, i64 cols, const double* src, i64 lds, int where) {
  if (rows <= 0 || cols <= 0) {
    dst.alloc(rows, cols, ctx.stream, true);
    return;
  }
  if (lds < rows) invalid("leading dimension smaller than the row count");
  dst.alloc(rows, cols, ctx.stream, false);
  if (dst.ld > rows)  // only the column pads need zeroing; the copy fills the rest
    NPCG_CUDA(cudaMemset2DAsync(dst.p() + rows, dst.ld * 8, 0, (dst.ld - rows) * 8, cols, ctx.stream));
  if (where == NPCG_HOST && rows * cols * 8 >= (i64{16} << 20)) {
    h2d_pinned(ctx, dst.p(), dst.ld, src, lds, rows, cols);
    return;
  }
  NPCG_CUDA(cudaMemcpy2DAsync(dst.p(), dst.ld * 8, src, lds * 8, rows * 8, cols,
                              where == NPCG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx.stream));
}

void download(Ctx& ctx, const double* src, i64 lds, i64 rows, i64 cols, double* dst, i64 ldd, int where) {
  if (rows <= 0 || cols <= 0) return;
  if (ldd < rows) invalid("leading dimension smaller than the row count");
  NPCG_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, rows * 8, cols,
                              where == NPCG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx.stream));
  if (where == NPCG_HOST) ctx.sync();
}

bool all_finite(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld) {
  if (rows <= 0 || cols <= 0) return true;
  DBuf<int> flag(1, ctx.stream);
  flag.zero();
  NPCG_LAUNCH(ctx, nonfinite_kernel, grid_for(ctx, rows * cols), 256, 0, p, rows, cols, ld, flag.p);
  int h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return h == 0;
}

double sum_squares(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld) {
  if (rows <= 0 || cols <= 0) return 0.0;
  const int nb = static_cast<int>(std::min<i64>(cdiv(rows * cols, 256), ctx.sm_count * 4));
  DBuf<double> part(nb + 1, ctx.stream);
  NPCG_LAUNCH(ctx, sumsq_partial_kernel, nb, 256, 0, p, rows, cols, ld, part.p);
  NPCG_LAUNCH(ctx, sum_partials_kernel, 1, 1024, 0, part.p, nb, part.p + nb);
  double h = 0.0;
  NPCG_CUDA(cudaMemcpyAsync(&h, part.p + nb, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return h;
}

bool all_finite_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld) {
  const bool ok = all_finite(ctx, p, rows, cols, ld);
  return rows_allreduce_host(ctx, ok ? 0.0 : 1.0, true) == 0.0;
}
double sum_squares_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld) {
  return rows_allreduce_host(ctx, sum_squares(ctx, p, rows, cols, ld), false);
}
double max_abs_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld) {
  return rows_allreduce_host(ctx, max_abs(ctx, p, rows, cols, ld), true);
}

void symmetry_stats(Ctx& ctx, const double* a, i64 n, i64 ld, double* asym, double* amax) {
  DBuf<unsigned long long> out(2, ctx.stream);
  out.zero();
  NPCG_LAUNCH(ctx, symstats_kernel, grid_for(ctx, n * n), 256, 0, a, n, ld, out.p);
  unsigned long long h[2];
  NPCG_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  std::memcpy(asym, &h[0], 8);
  std::memcpy(amax, &h[1], 8);
}

void axpby(Ctx& ctx, i64 rows, i64 cols, double a, const double* x, double b, double* y, i64 ld) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, axpby_kernel, grid_for(ctx, rows * cols), 256, 0, rows, cols, a, x, b, y, ld);
}
void add_scaled(Ctx& ctx, i64 rows, i64 cols, const double* a, double nu, const double* b, double* out, i64 ld) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, add_scaled_kernel, grid_for(ctx, rows * cols), 256, 0, rows, cols, a, nu, b, out, ld);
}
void add2d(Ctx& ctx, i64 rows, i64 cols, const double* a, i64 lda, const double* b, i64 ldb, double* out, i64 ldo) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, add2d_kernel, grid_for(ctx, rows * cols), 256, 0, rows, cols, a, lda, b, ldb, out, ldo);
}
void symmetrize(Ctx& ctx, const double* a, i64 n, i64 lda, double* out, i64 ldo) {
  if (n <= 0) return;
  if (a == out && lda == ldo) {
    NPCG_LAUNCH(ctx, symmetrize_inplace_kernel, grid_for(ctx, n * n), 256, 0, out, n, ldo);
    return;
  }
  NPCG_LAUNCH(ctx, symmetrize_kernel, grid_for(ctx, n * n), 256, 0, a, n, lda, out, ldo);
}
void scale_cols(Ctx& ctx, double* a, i64 rows, i64 cols, i64 lda, const double* d) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, scale_cols_kernel, grid_for(ctx, rows * cols), 256, 0, a, rows, cols, lda, d);
}
void divide(Ctx& ctx, i64 rows, i64 cols, double* y, i64 ld, double d) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, divide_kernel, grid_for(ctx, rows * cols), 256, 0, rows, cols, y, ld, d);
}
namespace {
__global__ void maxabs_kernel(const double* __restrict__ a, i64 rows, i64 cols, i64 ld, unsigned long long* out) {
  const i64 total = rows * cols;
  double m = 0.0;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double v = fabs(a[idx % rows + idx / rows * ld]);
    m = isnan(v) ? CUDART_INF : fmax(m, v);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, dbits(m));
}
__global__ void scale_pow2_kernel(i64 rows, i64 cols, double* a, i64 ld, int e) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    double* p = a + idx % rows + idx / rows * ld;
    *p = ldexp(*p, e);
  }
}
}  // namespace

namespace {
__global__ void transpose_tile_kernel(const double* __restrict__ src, i64 lds, i64 rows, i64 cols,
                                      double* __restrict__ dst, i64 ldd, int* bad) {
  __shared__ double tile[32][33];
  const i64 r0 = static_cast<i64>(blockIdx.x) * 32, c0 = static_cast<i64>(blockIdx.y) * 32;
  int nonfinite = 0;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const i64 r = r0 + threadIdx.x, c = c0 + k;
    const double x = (r < rows && c < cols) ? src[r + c * lds] : 0.0;
    nonfinite |= !isfinite(x);
    tile[k][threadIdx.x] = x;
  }
  if (__syncthreads_or(nonfinite) && bad && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(bad, 1);
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const i64 c = c0 + threadIdx.x, r = r0 + k;  // dst(c, r) = src(r, c)
    if (r < rows && c < cols) dst[c + r * ldd] = tile[threadIdx.x][k];
  }
}
}  // namespace

void transpose(Ctx& ctx, const double* src, i64 lds, i64 rows, i64 cols, double* dst, i64 ldd) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, transpose_tile_kernel, dim3(static_cast<unsigned>(cdiv(rows, 32)), static_cast<unsigned>(cdiv(cols, 32))),
              dim3(32, 8), 0, src, lds, rows, cols, dst, ldd, static_cast<int*>(nullptr));
}

void transpose_checked(Ctx& ctx, cudaStream_t s, const double* src, i64 lds, i64 rows, i64 cols, double* dst,
                       i64 ldd, int* bad) {
  if (rows <= 0 || cols <= 0) return;
  transpose_tile_kernel<<<dim3(static_cast<unsigned>(cdiv(rows, 32)), static_cast<unsigned>(cdiv(cols, 32))),
                          dim3(32, 8), 0, s>>>(src, lds, rows, cols, dst, ldd, bad);
  ctx.check_launch("transpose_tile_kernel");
}

double max_abs(Ctx& ctx, const double* a, i64 rows, i64 cols, i64 ld) {
  if (rows <= 0 || cols <= 0) return 0.0;
  DBuf<unsigned long long> out(1, ctx.stream);
  out.zero();
  NPCG_LAUNCH(ctx, maxabs_kernel, grid_for(ctx, rows * cols), 256, 0, a, rows, cols, ld, out.p);
  unsigned long long h = 0;
  NPCG_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  double r;
  std::memcpy(&r, &h, 8);
  return r;
}

void scale_pow2(Ctx& ctx, i64 rows, i64 cols, double* a, i64 ld, int e) {
  if (rows <= 0 || cols <= 0 || e == 0) return;
  NPCG_LAUNCH(ctx, scale_pow2_kernel, grid_for(ctx, rows * cols), 256, 0, rows, cols, a, ld, e);
}

void set_identity(Ctx& ctx, double* a, i64 rows, i64 cols, i64 ld) {
  if (rows <= 0 || cols <= 0) return;
  NPCG_LAUNCH(ctx, identity_kernel, grid_for(ctx, rows * cols), 256, 0, a, rows, cols, ld);
}

namespace {
template <int S>
void coldot_s(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* X, i64 ldx, double* out,
              i64 ldo, double mu, const double* shift, i64 ldsh, const int* gate) {
  const i64 cblocks = cdiv(ncols, CD_COLS);
  i64 splits = 1;
  const i64 target = 2 * ctx.sm_count;
  if (cblocks < target) splits = std::max<i64>(1, std::min<i64>(cdiv(target, cblocks), nrows / 256));
  i64 rps = round_up(cdiv(nrows, splits), 64);
  splits = cdiv(nrows, rps);
  if (splits <= 1) {
    NPCG_LAUNCH(ctx, coldot_kernel<S>, dim3(static_cast<unsigned>(cblocks), 1), 256, 0, M, ldm, nrows, ncols, X,
                ldx, std::max<i64>(nrows, 1), out, ldo, mu, shift, ldsh, static_cast<double*>(nullptr), gate);
    ctx.prof_work(2.0 * nrows * ncols * S, 8.0 * (nrows * ncols + S * (nrows + ncols)));
    return;
  }
  DBuf<double> part(splits * S * ncols, ctx.stream);
  NPCG_LAUNCH(ctx, coldot_kernel<S>, dim3(static_cast<unsigned>(cblocks), static_cast<unsigned>(splits)), 256, 0, M,
              ldm, nrows, ncols, X, ldx, rps, out, ldo, mu, shift, ldsh, part.p, gate);
  ctx.prof_work(2.0 * nrows * ncols * S, 8.0 * (nrows * ncols + S * (nrows + ncols)));
  NPCG_LAUNCH(ctx, coldot_reduce_kernel, static_cast<unsigned>(cdiv(ncols * S, 256)), 256, 0, part.p,
              static_cast<int>(splits), ncols, S, out, ldo, mu, shift, ldsh, gate);
}

template <int S>
void rowdot_s(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* c, i64 ldc,
              const double* base, i64 ldb, double* out, i64 ldo, const int* gate) {
  const i64 rblocks = cdiv(nrows, 2 * RD_THREADS);
  // enough CTAs for the bytes in flight (~8 per SM), at least 16 columns each,
  // and the CTA's slice of c in 48 KB of shared memory
  i64 splits = 1;
  const i64 target = 8 * ctx.sm_count;
  if (rblocks < target) splits = std::max<i64>(1, std::min<i64>(cdiv(target, rblocks), ncols / 16));
  splits = std::max<i64>(splits, cdiv(ncols * S * 8, RD_SMEM_MAX));
  i64 cps = cdiv(ncols, splits);
  splits = cdiv(ncols, std::max<i64>(cps, 1));
  const int smem = static_cast<int>(std::max<i64>(cps, 1) * S * 8);
  if (splits <= 1) {
    NPCG_LAUNCH(ctx, rowdot_kernel<S>, dim3(static_cast<unsigned>(rblocks), 1), RD_THREADS, smem, M, ldm, nrows,
                ncols, c, ldc, std::max<i64>(ncols, 1), base, ldb, out, ldo, static_cast<double*>(nullptr), gate);
    ctx.prof_work(2.0 * nrows * ncols * S, 8.0 * (nrows * ncols + S * (2 * nrows + ncols)));
    return;
  }
  DBuf<double> part(splits * S * nrows, ctx.stream);
  NPCG_LAUNCH(ctx, rowdot_kernel<S>, dim3(static_cast<unsigned>(rblocks), static_cast<unsigned>(splits)), RD_THREADS,
              smem, M, ldm, nrows, ncols, c, ldc, cps, base, ldb, out, ldo, part.p, gate);
  ctx.prof_work(2.0 * nrows * ncols * S, 8.0 * (nrows * ncols + S * (2 * nrows + ncols)));
  NPCG_LAUNCH(ctx, rowdot_reduce_kernel, static_cast<unsigned>(cdiv(nrows * S, 256)), 256, 0, part.p,
              static_cast<int>(splits), nrows, S, base, ldb, out, ldo, gate);
}
}  // namespace

#define NPCG_DISPATCH_S(S, FN, ...)                                            \
  switch (S) {                                                                 \
    case 1: FN<1>(__VA_ARGS__); break;                                         \
    case 2: FN<2>(__VA_ARGS__); break;                                         \
    case 3: FN<3>(__VA_ARGS__); break;                                         \
    case 4: FN<4>(__VA_ARGS__); break;                                         \
    case 5: FN<5>(__VA_ARGS__); break;                                         \
    case 6: FN<6>(__VA_ARGS__); break;                                         \
    case 7: FN<7>(__VA_ARGS__); break;                                         \
    case 8: FN<8>(__VA_ARGS__); break;                                         \
    default: fail(NPCG_EINVAL, "skinny kernels support 1..8 right-hand sides"); \
  }

void coldot(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* X, i64 ldx, int S, double* out,
            i64 ldo, double mu, const double* shift, i64 ldsh, const int* gate) {
  if (ncols <= 0 || S <= 0) return;
  NPCG_DISPATCH_S(S, coldot_s, ctx, M, ldm, nrows, ncols, X, ldx, out, ldo, mu, shift, ldsh, gate);
}

void rowdot(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* c, i64 ldc, int S,
            const double* base, i64 ldb, double* out, i64 ldo, const int* gate) {
  if (nrows <= 0 || S <= 0) return;
  if (ncols <= 0) {
    if (base) {
      copy2d(ctx, nrows, S, base, ldb, out, ldo);
    } else {
      NPCG_CUDA(cudaMemset2DAsync(out, ldo * 8, 0, nrows * 8, S, ctx.stream));
    }
    return;
  }
  NPCG_DISPATCH_S(S, rowdot_s, ctx, M, ldm, nrows, ncols, c, ldc, base, ldb, out, ldo, gate);
}

}  // namespace npcg
