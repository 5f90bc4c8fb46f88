// Row-sharded operators for one-process-per-GPU runs.
//
// Every n-vector is split into balanced contiguous row blocks R_g (comm.cuh).
// A product V -> A V on a sharded context:
//   1. all-gather V's row blocks into the full n x k block (NCCL all-gather;
//      the PCG's search direction p, a sketch block Q);
//   2. the local operator on the full block:
//        stored A (dense, stored kernel, low-rank; cfgs 1, 3, 5): rank g holds
//          the column block A[:, R_g] = rows R_g (A symmetric) and produces its
//          rows of A V directly;
//        Gram ridge (cfg 2): rank g holds the row block X_g of the design and
//          produces the full-length partial X_g^T (X_g V) / m;
//        matrix-free kernel (cfg 4): rank g evaluates its share of the
//          symmetric 128 x 128 block pairs (or of the sketch's column blocks)
//          and produces a full-length partial;
//   3. partial outputs are reduce-scattered (NCCL) into the row blocks.
// Everything downstream (factorisation, preconditioner, PCG vector updates)
// works on the local row blocks with all-reduced row reductions.
#include "blas.cuh"
#include "gemm.cuh"
#include "ops.cuh"

namespace npcg {
namespace {
// out (cols) <- row j of the n x cols block (ld)
__global__ void block_row_kernel(const double* __restrict__ a, i64 lda, i64 j, i64 cols, double* __restrict__ out) {
  for (i64 c = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; c < cols;
       c += static_cast<i64>(gridDim.x) * blockDim.x)
    out[c] = a[j + c * lda];
}
}  // namespace

void DenseColBlockOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  if (k <= 8) {
    coldot(*ctx, a.p(), a.ld, n, nloc, V, ldv, static_cast<int>(k), out, ldo, 0.0, nullptr, 0, gate);
  } else {
    gemm(*ctx, nloc, k, n, 1.0, Operand{a.p(), a.ld, true}, Operand{V, ldv, true}, 0.0, out, ldo);
  }
}

void DenseColBlockOp::column(i64 j, double* out) {
  NPCG_LAUNCH(*ctx, block_row_kernel, static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cdiv(nloc, 256), 1024))),
              256, 0, a.p(), a.ld, j, nloc, out);
}

void ShardOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  Ctx& c = *ctx;
  const RowSplit sp = c.split(n);
  DMat full;
  full.alloc(n, k, c.stream, false);
  rows_allgather(c, sp, V, ldv, k, full.p(), full.ld);
  if (local->partial_output(k)) {
    DMat part;
    part.alloc(n, k, c.stream, false);
    local->apply(full.p(), full.ld, k, part.p(), part.ld, gate);
    rows_reduce_scatter(c, sp, part.p(), part.ld, k, out, ldo);
  } else {
    local->apply(full.p(), full.ld, k, out, ldo, gate);
  }
}

void ShardOp::column(i64 j, double* out) {
  if (auto* blk = dynamic_cast<DenseColBlockOp*>(local.get())) {
    blk->column(j, out);
    return;
  }
  // full column on every rank, keep the local rows
  DBuf<double> full(n, ctx->stream);
  local->column(j, full.p);
  NPCG_CUDA(cudaMemcpyAsync(out, full.p + off, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->sync();
}

}  // namespace npcg
