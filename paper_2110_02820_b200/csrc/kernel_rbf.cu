// Gaussian (RBF) kernel operator on device (operators.cpp:125-188).
//
// Entry formula (kernel_block, operators.cpp:125-137):
//   K_ij = exp( max(0, (-2 x_i.x_j + ||x_i||^2) + ||x_j||^2) * (-1/(2 sigma^2)) ),  K_ii = 1.
// Stored path: the -2 X X^T product runs on the DMMA GEMM, then one pass adds
// the norms, clamps, exponentiates and pins the diagonal.
// Matrix-free path: tiles of points are staged in shared memory and K tiles are
// recomputed on the fly; column access uses the difference formula
// (operators.cpp:184-187).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "blas.cuh"
#include "gemm.cuh"
#include "ops.cuh"

namespace npcg {
namespace {

__global__ void row_norms_kernel(const double* __restrict__ pts, i64 ld, i64 n, i64 d, double* __restrict__ norms) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (i64 c = 0; c < d; ++c) {
    const double x = pts[i + c * ld];
    s += x * x;
  }
  norms[i] = s;
}

__global__ void kernel_epilogue_kernel(double* __restrict__ K, i64 ldk, i64 n, const double* __restrict__ norms,
                                       double c) {
  const i64 total = n * n;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % n, j = idx / n;
    double* p = K + i + j * ldk;
    double s = *p + norms[i];
    s = s + norms[j];
    *p = i == j ? 1.0 : exp(fmax(s, 0.0) * c);
  }
}

// Column block [r0, r0+cols) of K (= row block, K symmetric) from the DMMA
// product -2 X X_R^T (n x cols, in place): entry (j, i) is K(r0+i, j) with the
// reference rounding order (-2 x.x + ||x_{r0+i}||^2) + ||x_j||^2.
__global__ void kernel_colblock_epilogue_kernel(double* __restrict__ K, i64 ldk, i64 n, i64 cols, i64 r0,
                                                const double* __restrict__ norms, double c) {
  const i64 total = n * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 j = idx % n, i = idx / n;
    double* p = K + j + i * ldk;
    double s = *p + norms[r0 + i];
    s = s + norms[j];
    *p = r0 + i == j ? 1.0 : exp(fmax(s, 0.0) * c);
  }
}

__global__ void transpose_kernel(const double* __restrict__ src, i64 lds, i64 rows, i64 cols, double* __restrict__ dst,
                                 i64 ldd) {
  const i64 total = rows * cols;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % rows, j = idx / rows;
    dst[j + i * ldd] = src[i + j * lds];
  }
}

// Matrix-free K V: one thread per output row, tiles of 32 points in smem.
constexpr int FT = 32;
constexpr int FDMAX = 64;
template <int S>
__global__ void __launch_bounds__(128) kernel_free_apply_kernel(const double* __restrict__ prm, i64 ldp, i64 n, int d,
                                                                const double* __restrict__ norms, double c,
                                                                const double* __restrict__ V, i64 ldv,
                                                                double* __restrict__ out, i64 ldo,
                                                                const int* __restrict__ gate) {
  if (gate && *gate == 0) return;
  __shared__ double xs[FT][FDMAX + 1];
  __shared__ double ns[FT];
  __shared__ double vs[S][FT];
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double xi[FDMAX];
  double ni = 0.0;
  if (i < n) {
    for (int k = 0; k < d; ++k) xi[k] = prm[k + i * ldp];
    ni = norms[i];
  }
  double acc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = 0.0;
  for (i64 j0 = 0; j0 < n; j0 += FT) {
    const int cnt = static_cast<int>(n - j0 < FT ? n - j0 : FT);
    __syncthreads();
    for (int idx = threadIdx.x; idx < FT * d; idx += blockDim.x) {
      const int jj = idx / d, k = idx % d;
      xs[jj][k] = jj < cnt ? prm[k + (j0 + jj) * ldp] : 0.0;
    }
    for (int jj = threadIdx.x; jj < FT; jj += blockDim.x) {
      ns[jj] = jj < cnt ? norms[j0 + jj] : 0.0;
#pragma unroll
      for (int s = 0; s < S; ++s) vs[s][jj] = jj < cnt ? V[(j0 + jj) + s * ldv] : 0.0;
    }
    __syncthreads();
    if (i < n) {
      for (int jj = 0; jj < cnt; ++jj) {
        double dot = 0.0;
        for (int k = 0; k < d; ++k) dot += xi[k] * xs[jj][k];
        double sq = -2.0 * dot + ni;
        sq = sq + ns[jj];
        const double kij = (j0 + jj == i) ? 1.0 : exp(fmax(sq, 0.0) * c);
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] += kij * vs[s][jj];
      }
    }
  }
  if (i < n) {
#pragma unroll
    for (int s = 0; s < S; ++s) out[i + s * ldo] = acc[s];
  }
}

__global__ void kernel_column_kernel(const double* __restrict__ pts, i64 ld, i64 n, i64 d, i64 j, double c,
                                     double* __restrict__ out) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (i64 k = 0; k < d; ++k) {
    const double diff = pts[i + k * ld] - pts[j + k * ld];
    s += diff * diff;
  }
  out[i] = i == j ? 1.0 : exp(s * c);
}

template <int S>
void free_apply_s(Ctx& ctx, const KernelFreeOp& op, const double* V, i64 ldv, double* out, i64 ldo, const int* gate) {
  const double c = -1.0 / (2.0 * op.sigma * op.sigma);
  NPCG_LAUNCH(ctx, kernel_free_apply_kernel<S>, static_cast<unsigned>(cdiv(op.n, 128)), 128, 0, op.pts_rm.p(),
              op.pts_rm.ld, op.n, static_cast<int>(op.d), op.norms.p, c, V, ldv, out, ldo, gate);
}

}  // namespace

void build_kernel_matrix(Ctx& ctx, const DMat& pts, i64 n, i64 d, double sigma, DMat& K) {
  DBuf<double> norms(n, ctx.stream);
  NPCG_LAUNCH(ctx, row_norms_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, pts.p(), pts.ld, n, d, norms.p);
  K.alloc(n, n, ctx.stream, false);
  // K = -2 X X^T  (A = X M-major, B = X^T N-major)
  gemm(ctx, n, n, d, -2.0, Operand{pts.p(), pts.ld, false}, Operand{pts.p(), pts.ld, false}, 0.0, K.p(), K.ld);
  const double c = -1.0 / (2.0 * sigma * sigma);
  NPCG_LAUNCH(ctx, kernel_epilogue_kernel, static_cast<unsigned>(std::min<i64>(cdiv(n * n, 256), ctx.sm_count * 16)),
              256, 0, K.p(), K.ld, n, norms.p, c);
}

void prepare_kernel_free(Ctx& ctx, KernelFreeOp& op) {
  op.norms.alloc(op.n, ctx.stream);
  NPCG_LAUNCH(ctx, row_norms_kernel, static_cast<unsigned>(cdiv(op.n, 256)), 256, 0, op.pts.p(), op.pts.ld, op.n,
              op.d, op.norms.p);
  op.pts_rm.alloc(op.d, op.n, ctx.stream, true);
  NPCG_LAUNCH(ctx, transpose_kernel, static_cast<unsigned>(std::min<i64>(cdiv(op.n * op.d, 256), 4096)), 256, 0,
              op.pts.p(), op.pts.ld, op.n, op.d, op.pts_rm.p(), op.pts_rm.ld);
}

void kernel_apply_free(Ctx& ctx, const KernelFreeOp& op, const double* V, i64 ldv, i64 k, double* out, i64 ldo,
                       const int* gate) {
  if (k > 0 && !(std::getenv("NPCG_KFREE") && std::string(std::getenv("NPCG_KFREE")) == "fused")) {
    // Recompute K by row blocks like do_apply_block (operators.cpp:166-177):
    // K_R = kernel(-2 X_R X^T on DMMA + norms, clamp, exp), then out_R = K_R V
    // on DMMA (k > 8) or the coldot GEMV; the exps are paid once per block,
    // not once per column chunk. (Measured at n = 50 000: 2.7x faster than the
    // one-thread-per-row kernel below even for a single vector.)
    const i64 n = op.n;
    const double c = -1.0 / (2.0 * op.sigma * op.sigma);
    const i64 budget = i64{4} << 30;  // bytes of one K row block
    const i64 R = std::min<i64>(n, std::max<i64>(128, budget / (8 * std::max<i64>(n, 1)) / 128 * 128));
    DMat Kt;  // K[:, r0 : r0+R] = (K_R)^T, n x R: its columns are contiguous
    Kt.alloc(n, R, ctx.stream, false);
    for (i64 r0 = 0; r0 < n; r0 += R) {
      const i64 rb = std::min(R, n - r0);
      gemm(ctx, n, rb, op.d, -2.0, Operand{op.pts.p(), op.pts.ld, false}, Operand{op.pts.p() + r0, op.pts.ld, false},
           0.0, Kt.p(), Kt.ld);
      NPCG_LAUNCH(ctx, kernel_colblock_epilogue_kernel,
                  static_cast<unsigned>(std::min<i64>(cdiv(rb * n, 256), ctx.sm_count * 16)), 256, 0, Kt.p(), Kt.ld, n,
                  rb, r0, op.norms.p, c);
      if (k <= 8) {  // few vectors: out_R = (K_R^T)^T V as column dots (HBM-bound on the block)
        coldot(ctx, Kt.p(), Kt.ld, n, rb, V, ldv, static_cast<int>(k), out + r0, ldo, 0.0, nullptr, 0, gate);
      } else {
        gemm(ctx, rb, k, n, 1.0, Operand{Kt.p(), Kt.ld, true}, Operand{V, ldv, true}, 0.0, out + r0, ldo);
      }
    }
    return;
  }
  if (op.d > FDMAX) fail(NPCG_ERUNTIME, "KernelOperator: matrix-free path supports d <= 64");
  for (i64 s0 = 0; s0 < k; s0 += 4) {
    const int S = static_cast<int>(std::min<i64>(4, k - s0));
    const double* v = V + s0 * ldv;
    double* o = out + s0 * ldo;
    switch (S) {
      case 1: free_apply_s<1>(ctx, op, v, ldv, o, ldo, gate); break;
      case 2: free_apply_s<2>(ctx, op, v, ldv, o, ldo, gate); break;
      case 3: free_apply_s<3>(ctx, op, v, ldv, o, ldo, gate); break;
      default: free_apply_s<4>(ctx, op, v, ldv, o, ldo, gate); break;
    }
  }
}

void KernelFreeOp::column(i64 j, double* out) {
  const double c = -1.0 / (2.0 * sigma * sigma);
  NPCG_LAUNCH(*ctx, kernel_column_kernel, static_cast<unsigned>(cdiv(n, 256)), 256, 0, pts.p(), pts.ld, n, d, j, c,
              out);
}

}  // namespace npcg
