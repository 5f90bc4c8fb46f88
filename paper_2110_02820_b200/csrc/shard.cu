// Row-sharded operators for multi-GPU runs: one process per GPU,
// vectors replicated, the operator split by rows.
//
//   Gram (ridge, cfg 2): rank g holds the row block X_g of the design; its
//     local product X_g^T (X_g v) / m is a partial n-vector and one in-place
//     all-reduce (n doubles per RHS) completes A v.
//   Dense / stored kernel (cfgs 1, 3, 5): rank g holds the column block
//     A[:, R_g] (= rows R_g, A symmetric); its local product is rows R_g of
//     A v and one all-gather (ceil(n/G) doubles per rank per RHS) completes it.
//
// The exchange is a callback enqueued on the library stream (the host binds
// it to NCCL through torch.distributed), so the PCG loop, the sketch and the
// power iterations run unchanged on a ShardOp: everything downstream of the
// operator (factorisation, preconditioner, vector updates) is replicated and
// deterministic, hence identical on every rank.
#include "blas.cuh"
#include "gemm.cuh"
#include "ops.cuh"

namespace npcg {
namespace {

// send (nmax x k, contiguous) <- local block (nloc x k, ld)
__global__ void pack_block_kernel(const double* __restrict__ src, i64 lds, i64 nloc, i64 nmax, i64 k,
                                  double* __restrict__ dst) {
  const i64 total = nmax * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = idx % nmax, s = idx / nmax;
    dst[idx] = i < nloc ? src[i + s * lds] : 0.0;
  }
}

// out (n x k, ldo) <- gathered blocks recv[r][s][i] (rank-major, nmax x k each)
__global__ void unpack_gather_kernel(const double* __restrict__ recv, i64 nranks, i64 nmax, i64 k, i64 n,
                                     double* __restrict__ out, i64 ldo) {
  const i64 total = n * k;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 row = idx % n, s = idx / n;
    const i64 r = row / nmax, i = row % nmax;
    out[row + s * ldo] = recv[(r * k + s) * nmax + i];
  }
}

}  // namespace

void DenseColBlockOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  if (k <= 8) {
    coldot(*ctx, a.p(), a.ld, n, nloc, V, ldv, static_cast<int>(k), out, ldo, 0.0, nullptr, 0, gate);
  } else {
    gemm(*ctx, nloc, k, n, 1.0, Operand{a.p(), a.ld, true}, Operand{V, ldv, true}, 0.0, out, ldo);
  }
}

void ShardOp::apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) {
  Ctx& c = *ctx;
  if (mode == 0) {
    local->apply(V, ldv, k, out, ldo, gate);
    const i64 count = ldo * (k - 1) + n;  // one contiguous span (column pads ride along)
    if (fn(user, 0, out, out, count, c.stream) != 0) fail(NPCG_ECUDA, "sharded operator: all-reduce failed");
    return;
  }
  // mode 1: local rows -> padded send block -> all-gather -> scatter into out
  DMat loc;
  loc.alloc(nmax, k, c.stream, false);
  local->apply(V, ldv, k, loc.p(), loc.ld, gate);
  DBuf<double> send(nmax * k, c.stream), recv(nranks * nmax * k, c.stream);
  const i64 nloc = static_cast<DenseColBlockOp*>(local.get())->nloc;
  NPCG_LAUNCH(c, pack_block_kernel, static_cast<unsigned>(std::min<i64>(cdiv(nmax * k, 256), 4096)), 256, 0,
              loc.p(), loc.ld, nloc, nmax, k, send.p);
  if (fn(user, 1, send.p, recv.p, nmax * k, c.stream) != 0) fail(NPCG_ECUDA, "sharded operator: all-gather failed");
  NPCG_LAUNCH(c, unpack_gather_kernel, static_cast<unsigned>(std::min<i64>(cdiv(n * k, 256), 4096)), 256, 0,
              recv.p, nranks, nmax, k, n, out, ldo);
}

}  // namespace npcg
