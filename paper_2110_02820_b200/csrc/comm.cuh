// Row-sharded data plane for one process per GPU.
//
// A sharded context splits every operator dimension n into G contiguous,
// balanced row blocks R_g (floor(n/G) or floor(n/G)+1 rows; RowSplit). Every
// n-length object of the path -- Omega, Y, U, x, r, z, p, the right-hand
// sides -- lives on its owner as the local row block; the only exchanges are
//   * all-gather of a row-sharded block (the search direction p before A p,
//     an Omega block before Y = A Omega),
//   * sum all-reduce of row reductions (the l x l Grams Omega^T Y_nu and the
//     CholeskyQR Grams, ||Y||_F, U^T r, the PCG dots), and
//   * reduce-scatter of full-length partial products (Gram ridge operator,
//     the symmetric matrix-free kernel product),
// enqueued on the library stream. NcclComm drives NCCL from C++ (NVLink /
// NVSwitch on a B200 node; libnccl is loaded at run time, so unsharded use
// needs no NCCL); CallbackComm forwards to a host-supplied npcg_exchange_fn.
#pragma once

#include <memory>
#include <string>

#include "common.cuh"

namespace npcg {

struct Ctx;

/// Balanced contiguous row blocks of n rows over `world` ranks.
struct RowSplit {
  i64 n = 0;
  int world = 1;
  i64 q = 0, r = 0;  // n = q * world + r: ranks < r own q + 1 rows
  RowSplit() = default;
  RowSplit(i64 n_, int world_) : n(n_), world(world_), q(n_ / world_), r(n_ % world_) {}
  i64 count(int g) const { return q + (g < r ? 1 : 0); }
  i64 offset(int g) const { return g * q + (g < r ? g : r); }
  i64 nmax() const { return q + (r > 0 ? 1 : 0); }
};

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  virtual const char* name() const = 0;
  /// In-place sum over ranks of `count` doubles; every rank receives the same bits.
  virtual void allreduce_sum(double* buf, i64 count, cudaStream_t s) = 0;
  /// recv (world * count, rank-major) <- every rank's `count` doubles.
  virtual void allgather(const double* send, double* recv, i64 count, cudaStream_t s) = 0;
  /// recv (count) <- sum over ranks of send[rank * count .. (rank+1) * count).
  virtual void reduce_scatter_sum(const double* send, double* recv, i64 count, cudaStream_t s) = 0;
};

/// NCCL communicator created inside the library (ncclCommInitRank).
std::shared_ptr<Comm> make_nccl_comm(int device, int rank, int world, const void* unique_id128);
/// 128-byte ncclUniqueId for rank 0 to distribute.
void nccl_unique_id(void* out128);
/// Host-callback transport (npcg_exchange_fn kinds 0 all-reduce, 1 all-gather, 2 reduce-scatter).
std::shared_ptr<Comm> make_callback_comm(int rank, int world, npcg_exchange_fn fn, void* user);

// ---- row-sharded helpers (no-ops on an unsharded context) -----------------
/// Sum over ranks of a device buffer, in place (enqueued on ctx.stream).
void rows_allreduce(Ctx& ctx, double* buf, i64 count);
/// Host scalar combined over ranks (sum or max), synchronising.
double rows_allreduce_host(Ctx& ctx, double v, bool max);
/// full (n x k, ldf) <- all ranks' local row blocks (split.count(rank) x k, ldl).
void rows_allgather(Ctx& ctx, const RowSplit& split, const double* local, i64 ldl, i64 k, double* full, i64 ldf);
/// local (count(rank) x k, ldl) <- sum over ranks of each rank's full-length partial (n x k, ldp).
void rows_reduce_scatter(Ctx& ctx, const RowSplit& split, const double* partial, i64 ldp, i64 k, double* local,
                         i64 ldl);

}  // namespace npcg
