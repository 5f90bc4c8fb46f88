// Device-resident operators, Nyström state and preconditioner behind the
// C-ABI handles (npcg_op / npcg_nys / npcg_pre).
#pragma once

#include <memory>
#include <vector>

#include "context.cuh"

namespace npcg {

enum OpKind { kDense = 0, kGram = 1, kKernelStored = 2, kKernelFree = 3, kCallback = 4, kRegularized = 5 };

/// LinearOperator (operators.hpp:25-47) on device. apply() is the unchecked
/// do_apply_block(); the C-ABI layer does the reference's dim/finite checks.
struct Op {
  Ctx* ctx = nullptr;
  i64 n = 0;              // operator dimension
  i64 nloc = 0, off = 0;  // this rank's row block of every n-vector (nloc = n, off = 0 unsharded)
  int kind = kDense;
  /// Set n and the local row block from the context's layout.
  void set_dim(Ctx& c, i64 n_) {
    ctx = &c;
    n = n_;
    nloc = c.local_rows(n_);
    off = c.row_offset(n_);
  }
  virtual ~Op() = default;
  /// out (n x k) = A V  (device pointers; on a sharded context V and out are
  /// this rank's row blocks, nloc x k).
  virtual void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate = nullptr) = 0;
  /// out = A P + mu P with the reference's rounding order (out = A p; out += mu p).
  virtual void apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate);
  virtual bool has_column() const { return false; }
  virtual void column(i64 j, double* out);
  /// A product costs far more than a host round trip (matrix-free kernel):
  /// the PCG driver then keeps one iteration in flight instead of several.
  virtual bool costly() const { return false; }
  /// For the local operator of a ShardOp: apply() on a full-length input
  /// yields a full-length partial (reduce-scattered by the ShardOp) rather
  /// than this rank's rows.
  virtual bool partial_output(i64 /*k*/) const { return false; }
  /// out(:, c) = A(:, idx[c]) for c < k (host indices; ld ldo). Default: column() per index.
  virtual void columns(const i64* idx, i64 k, double* out, i64 ldo);
};

struct DenseOp : Op {  // DenseOperator (operators.cpp:64-80); also the stored kernel
  DMat a;
  void columns(const i64* idx, i64 k, double* out, i64 ldo) override;
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  void apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate) override;
  bool has_column() const override { return true; }
  void column(i64 j, double* out) override;
};

struct GramOp : Op {  // GramRidgeOperator (operators.cpp:105-121): (1/m) G^T (G v)
  DMat xr;            // design stored row-major: n x m col-major, data row a contiguous
  i64 m = 0;
  double div = 0.0;   // out /= div (operators.cpp:115); the global row count when X is a row shard
  // Streamed construction (npcg_op_gram_create_streamed): row blocks of X
  // landing in `stage` (caller layout) on the copy stream (`copied` fires),
  // then transposed into xr and checked for non-finite entries on the
  // transpose stream (`ready` fires).
  struct Chunk {
    i64 r0, r1;
    cudaEvent_t copied, ready;
  };
  std::vector<Chunk> pending;
  DMat stage;  // m x n column-major copy of X while the streamed upload is pending
  DBuf<int> bad;  // non-finite flag of the streamed upload
  int nonfinite = 0;  // latched: every later use raises the constructor's error
  /// Order the context stream after every pending block, wait for the upload
  /// (the caller's host buffer is free afterwards) and raise the constructor's
  /// non-finite error (operators.cpp:108-109) if the flag is set.
  void settle();
  bool shard_partial = false;  // local operator of a ShardOp over a row block of X: full-length partial output
  bool partial_output(i64) const override { return shard_partial; }
  ~GramOp() override;
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  void apply_shift(const double* P, i64 ldp, int S, double mu, double* out, i64 ldo, const int* gate) override;
};
/// Upload the design `g` (m x n, ld ldg; host or device) into op.xr, checking
/// for non-finite entries in the same pass (synchronous, raises the
/// constructor's error).
void gram_upload(Ctx& c, GramOp& op, const double* g, i64 ldg, int where);
/// Enqueue the upload of the host design `g` (m x n, ld ldg) into op.xr in
/// row blocks on the context's side stream; returns without waiting.
void gram_upload_streamed(Ctx& c, GramOp& op, const double* g, i64 ldg);

struct KernelFreeOp : Op {  // KernelOperator beyond dense_cap (operators.cpp:152-188)
  DMat pts;                 // n x d col-major (reference layout)
  DMat pts_rm;              // d x n col-major == points row-major (point-contiguous)
  DBuf<double> norms;       // ||x_i||^2
  double max_norm = INFINITY;  // max_i ||x_i||^2 (bounds the kernel exponent)
  DMat pts_s;               // points * sqrt(1/sigma^2) (symmetric fused kernel)
  DBuf<double> norms_s;     // -||x_i||^2 / (2 sigma^2)
  i64 d = 0;
  double sigma = 1.0;
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  bool has_column() const override { return true; }
  void column(i64 j, double* out) override;
  void columns(const i64* idx, i64 k, double* out, i64 ldo) override;
  bool costly() const override { return true; }
  bool partial_output(i64 k) const override;
  // Row-sharded use (the local operator of a ShardOp): this rank's share of
  // the work -- a range of the symmetric block pairs (k <= 2), of the column
  // blocks (k > 8), or its own row block (3..8 vectors).
  int shard_rank = 0, shard_world = 1;
  i64 shard_off = 0, shard_rows = 0;
};

/// A user operator behind C callbacks (npcg_op_callback_create): the
/// reference's LinearOperator plug-in point (operators.hpp:25-47).
struct CallbackOp : Op {
  npcg_apply_fn fn = nullptr;
  npcg_column_fn col = nullptr;
  void* user = nullptr;
  int where = NPCG_HOST;
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  bool has_column() const override { return col != nullptr; }
  void column(i64 j, double* out) override;
  bool costly() const override { return true; }  // unknown cost: keep one PCG iteration in flight
};

/// RegularizedOperator (operators.cpp:82-103): out = base V; out += mu V.
struct RegOp : Op {
  Op* base = nullptr;  // not owned (the reference's non-owning view)
  double mu = 0.0;
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  void apply_shift(const double* P, i64 ldp, int S, double mu2, double* out, i64 ldo, const int* gate) override;
  bool costly() const override { return base->costly(); }
};

/// Column block A[:, off : off+nloc] of a symmetric A held by one rank; on a
/// full-length input V its apply gives rows off.. of A V (A^T V restricted to
/// the block).
struct DenseColBlockOp : Op {
  DMat a;  // n x nloc
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  bool has_column() const override { return true; }
  /// Local rows of A(:, j) = row j of the block (A symmetric).
  void column(i64 j, double* out) override;
};

/// Row-sharded operator (sharded context, one process per GPU): apply()
/// takes and returns this rank's row blocks. It all-gathers the input over
/// the ranks (NCCL), runs `local` on the full-length block and keeps the local
/// rows `local` produced (column block A[:, R_g]: the stored dense / kernel /
/// low-rank operators) or reduce-scatters the full-length partial it produced
/// (Gram ridge over a row block of X, the symmetric matrix-free kernel).
struct ShardOp : Op {
  std::unique_ptr<Op> local;  // works on full-length inputs
  void apply(const double* V, i64 ldv, i64 k, double* out, i64 ldo, const int* gate) override;
  bool has_column() const override { return local->has_column(); }
  void column(i64 j, double* out) override;
  bool costly() const override { return local->costly(); }
};

/// Build the stored Gaussian kernel matrix (operators.cpp:125-150) on device.
void build_kernel_matrix(Ctx& ctx, const DMat& pts, i64 n, i64 d, double sigma, DMat& K);
void prepare_kernel_free(Ctx& ctx, KernelFreeOp& op);
/// Column block K[:, r0 : r0+cols] (n x cols) of the stored Gaussian kernel.
void build_kernel_colblock(Ctx& ctx, const DMat& pts, i64 n, i64 d, double sigma, i64 r0, i64 cols, DMat& K);
void kernel_apply_free(Ctx& ctx, const KernelFreeOp& op, const double* V, i64 ldv, i64 k, double* out, i64 ldo,
                       const int* gate);

/// Device storage of a sketch pair (Omega, Y), capacity-managed. Several
/// Nys handles may share one store (npcg_nys_clone, the facade's value-
/// semantics extend_sketch): a handle of size s views the first s columns,
/// and appending writes only columns >= s, so the store records how many
/// columns have been written; a handle extending behind that mark (a branch)
/// or past the capacity copies its own columns to a fresh store first.
struct SketchStore {
  DMat omega, y;
  i64 filled = 0;
};

/// The factored approximation (nystrom.hpp:19-33): U, lambda, shift. It is
/// immutable once published -- a Nys handle and every preconditioner built
/// from it share it, so extending or refactoring the handle later never
/// changes an existing preconditioner (the reference's value semantics).
struct Factors {
  DMat u;                         // n x ell (this rank's rows on a sharded context)
  DBuf<double> lambda;            // ell, nonincreasing
  std::vector<double> lambda_host;
  i64 ell = 0;
  double shift = 0.0;
  double lambda_min() const { return ell == 0 ? 0.0 : lambda_host.back(); }
};

/// Cached sketch + factored approximation (nystrom.hpp:19-48).
struct Nys {
  Ctx* ctx = nullptr;
  Op* op = nullptr;  // not owned; nullptr for from_factors
  i64 n = 0;              // dimension
  i64 nloc = 0, off = 0;  // this rank's rows of Omega, Y, U (nloc = n unsharded)
  std::shared_ptr<SketchStore> sk;  // first `size` columns are this handle's pair
  i64 size = 0;
  std::shared_ptr<const Factors> fac;  // null until factored; replaced only by a successful nys_factor
  std::vector<i64> used;  // column-sampling sketches: indices drawn so far (extend_sketch_columns)
  bool factored() const { return static_cast<bool>(fac); }
  const DMat& omega() const { return sk->omega; }
  const DMat& y() const { return sk->y; }
};
void nys_extend(Nys& s, const double* raw, i64 ld, i64 extra, int where);
/// Append unit columns e_j and A(:, j) for the given distinct indices
/// (extend_sketch_columns / column_sampling_nystrom, nystrom.cpp:60-94,160-184).
void nys_extend_columns(Nys& s, const std::vector<i64>& idx);
/// nystrom_from_sketch: publishes a new Factors on success; on failure the
/// handle keeps what it had (nothing is half-updated).
void nys_factor(Nys& s);

/// NystromPreconditioner (preconditioner.hpp:20-37). Holds its own reference
/// to the factors it was built from.
struct Pre {
  Ctx* ctx = nullptr;
  std::shared_ptr<const Factors> fac;  // U, lambda (device)
  i64 n = 0, ell = 0;
  i64 nloc = 0;  // local rows of U and of the vectors it is applied to
  double mu = 0.0, lambda_ell = 0.0;
  DBuf<double> gain_inv;  // (lambda_ell + mu)/(lambda + mu) - 1
  DBuf<double> gain_fwd;  // (lambda + mu)/(lambda_ell + mu) - 1
};
void pre_build(Pre& p, const Nys& s, double mu);
/// Z = P^{-1} R (n x S). Z may alias nothing of R.
void pre_apply_inverse(Pre& p, const double* R, i64 ldr, i64 S, double* Z, i64 ldz, const int* gate = nullptr);
void pre_apply(Pre& p, const double* V, i64 ldv, i64 S, double* out, i64 ldo);
/// woodbury_inverse_apply (preconditioner.cpp:104-114): X = (U diag(lambda) U^T + mu I)^-1 B
/// = U ((lambda + mu)^-1 .* (U^T B)) + (B - U U^T B) / mu, on the factored approximation f.
void woodbury_apply(Ctx& ctx, const Factors& f, i64 nloc, double mu, const double* B, i64 ldb, i64 S, double* X,
                    i64 ldx);

}  // namespace npcg
