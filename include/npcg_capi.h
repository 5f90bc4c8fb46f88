/*
 * npcg_capi.h — drop-in C-ABI of the B200-native Nyström-PCG hot path.
 *
 * The reference (/root/reference/proj/core) exposes only a C++ API
 * (the npcg headers, Eigen types) and no FFI. This header is the boundary a
 * maintainer binds instead: plain pointers + sizes, column-major FP64
 * (Eigen::MatrixXd layout, ld >= rows), 64-bit indices, status codes.
 * Each entry point names the reference interface it replaces (file:line,
 * paths relative to /root/reference/proj/core/). The C++ façade in
 * include/npcg/ maps these back onto the reference's class/func names and
 * exception types; INTEGRATION.md shows the bindings.
 *
 * Everything computes on one B200 (sm_100a) through hand-written CUDA kernels
 * in libnpcg_b200.so. There is no CPU fallback: without a usable device every
 * compute entry point returns NPCG_ECUDA.
 *
 * Pointers tagged `where` are host memory (NPCG_HOST) or device memory of the
 * context's GPU (NPCG_DEVICE). Host buffers are copied in/out inside the call.
 */
#ifndef NPCG_CAPI_H
#define NPCG_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference's exception types) -------------- */
enum {
  NPCG_OK = 0,
  NPCG_EINVAL = 1,    /* std::invalid_argument  (operators.cpp:14-21, nystrom.cpp:144-145, ...) */
  NPCG_ERUNTIME = 2,  /* std::runtime_error     (nystrom.cpp:124-130, operators.cpp:42-50)        */
  NPCG_EDIVERGED = 3, /* npcg::SolveDivergenceError (solvers.hpp:51-57); report is filled        */
  NPCG_ECUDA = 4,     /* CUDA failure / no device                                                 */
  NPCG_ENCCL = 5      /* collective failure (multi-GPU builds)                                    */
};
enum { NPCG_HOST = 0, NPCG_DEVICE = 1 };

typedef struct npcg_ctx npcg_ctx;
typedef struct npcg_rng npcg_rng;
typedef struct npcg_op npcg_op;
typedef struct npcg_nys npcg_nys;
typedef struct npcg_pre npcg_pre;

/* Thread-local message of the last failing call, formatted like the
 * reference's what() strings. */
const char* npcg_last_error(void);
const char* npcg_version(void);

/* ---- context ------------------------------------------------------------ */
int npcg_ctx_create(int device, npcg_ctx** out);
int npcg_ctx_destroy(npcg_ctx* ctx);
int npcg_ctx_sync(npcg_ctx* ctx);
/* ---- row-sharded contexts: one process per GPU --------------
 * No reference counterpart (the reference is single-process). On a sharded
 * context every dimension n of an operator is split into balanced contiguous
 * row blocks R_g (npcg_ctx_layout) and every n-length argument of every entry
 * point -- right-hand sides, solutions, raw Omega blocks, U, power vectors,
 * columns -- is this rank's row block (count rows, ld >= count). Rng-drawn
 * blocks are drawn whole on every rank (the reference's stream) and each rank
 * keeps its rows. The exchanges -- all-gather of p / sketch blocks, sum
 * all-reduce of the row reductions (Omega^T Y, Grams, dots, U^T r),
 * reduce-scatter of partial products -- are issued by the library from C++
 * on its stream: NCCL (npcg_ctx_create_sharded), or a host callback
 * (npcg_ctx_create_exchange; kind 0 in-place sum all-reduce of `count`
 * doubles, 1 all-gather of `count` doubles per rank into recv rank-major,
 * 2 reduce-scatter: recv (count) = sum over ranks of send[rank*count ..]). */
typedef int (*npcg_exchange_fn)(void* user, int kind, double* send, double* recv, int64_t count, void* stream);
/* 128-byte ncclUniqueId (rank 0 creates it, the host distributes it). */
int npcg_nccl_unique_id(void* out128);
int npcg_ctx_create_sharded(int device, int rank, int world, const void* nccl_id128, npcg_ctx** out);
int npcg_ctx_create_exchange(int device, int rank, int world, npcg_exchange_fn fn, void* user, npcg_ctx** out);
/* rank, world and this rank's row block [offset, offset + count) of dimension n. */
int npcg_ctx_layout(const npcg_ctx* ctx, int64_t n, int* rank, int* world, int64_t* offset, int64_t* count);

/* The CUDA stream all of this context's work is ordered on (cudaStream_t). */
void* npcg_ctx_stream(npcg_ctx* ctx);
/* Device memory owned by the context's allocator (for NPCG_DEVICE inputs). */
int npcg_dev_alloc(npcg_ctx* ctx, int64_t bytes, void** out);
int npcg_dev_free(npcg_ctx* ctx, void* p);
int npcg_memcpy(npcg_ctx* ctx, void* dst, int dst_where, const void* src, int src_where, int64_t bytes);
/* Number of this library's kernel launches issued on ctx so far. */
int64_t npcg_ctx_launches(npcg_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (on != 0 clears and
 * starts recording). Report: one "name\tlaunches\ttotal_ms\n" line per kernel. */
int npcg_prof_enable(npcg_ctx* ctx, int on);
int npcg_prof_report(npcg_ctx* ctx, char* buf, int64_t cap);

/* ---- random (random.hpp:21-50, random.cpp:11-56) -------------------------
 * The reference generator, bit for bit: std::mt19937_64 + cache-free
 * Box-Muller, two engine words per normal, column-major fills. Host-side:
 * it produces the Ω blocks, right-hand sides and power-method start vectors
 * the GPU path consumes. */
int npcg_rng_create(uint64_t seed, npcg_rng** out);
int npcg_rng_clone(const npcg_rng* rng, npcg_rng** out);
int npcg_rng_destroy(npcg_rng* rng);
double npcg_rng_normal(npcg_rng* rng);                         /* random.cpp:11-18 */
double npcg_rng_uniform(npcg_rng* rng);                        /* random.cpp:20    */
uint64_t npcg_rng_word(npcg_rng* rng);                         /* engine()         */
void npcg_rng_discard(npcg_rng* rng, uint64_t words);
int npcg_rng_integer(npcg_rng* rng, uint64_t bound, uint64_t* out);   /* random.cpp:22-25 */
/* gaussian_matrix (random.cpp:27-32) into dst (col-major, ld = rows). */
int npcg_rng_gaussian(npcg_rng* rng, int64_t rows, int64_t cols, double* dst);
int npcg_rng_sample(npcg_rng* rng, int64_t n, int64_t k, int64_t* out); /* random.cpp:44-56 */
/* count successive Rng::uniform() draws (random.cpp:20) into dst. */
int npcg_rng_uniform_fill(npcg_rng* rng, int64_t count, double* dst);
uint64_t npcg_splitmix64(uint64_t seed);                       /* bench.cpp:180-185 */
/* The reference generator continued on the GPU: the same
 * mt19937_64 word stream as the host calls above (bitwise), produced by a
 * device kernel from the engine's state; the Rng advances exactly as the host
 * draw would. npcg_rng_gaussian_device fills dst (device, col-major rows x
 * cols, ld) like npcg_rng_gaussian, with the Box-Muller transform on the GPU
 * (CUDA log/cos: deviates within a few ulp of libm's). On a row-sharded ctx
 * only this rank's rows land in dst (ld >= its row count). */
int npcg_rng_words_device(npcg_ctx* ctx, npcg_rng* rng, int64_t count, uint64_t* dst);
int npcg_rng_gaussian_device(npcg_ctx* ctx, npcg_rng* rng, int64_t rows, int64_t cols, double* dst, int64_t ld);

/* ---- operators (operators.hpp:25-168) ----------------------------------- */
/* DenseOperator(Matrix a), operators.cpp:64-70 (square + symmetry check). */
int npcg_op_dense_create(npcg_ctx* ctx, int64_t rows, int64_t cols, const double* a, int64_t lda,
                         int where, npcg_op** out);
/* GramRidgeOperator(Matrix design) = (1/m) G^T G, operators.cpp:105-121. */
int npcg_op_gram_create(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, int64_t ldg,
                        int where, npcg_op** out);
/* GramRidgeOperator(Matrix design) with a streamed upload (host buffer only).
 * Replaces the same constructor (operators.cpp:105-110) for large designs:
 * returns once the copy is enqueued, in ~80 MB row blocks on a side stream,
 * and the first product (the sketch) starts on each block as it lands.
 * Contract: `g` must stay valid and unchanged until the first call that
 * applies the operator returns (or npcg_op_destroy); that call raises the
 * constructor's non-finite error (NPCG_EINVAL, same message) in its place.
 * Device memory: two copies of X until then (the synchronous constructor
 * streams host designs through a 4 x ~80 MB staging ring instead). */
int npcg_op_gram_create_streamed(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, int64_t ldg,
                                 npcg_op** out);
/* KernelOperator(points n x d, sigma, dense_cap), operators.cpp:141-150:
 * stored (built on device) when n <= dense_cap, otherwise matrix-free. */
int npcg_op_kernel_create(npcg_ctx* ctx, int64_t n, int64_t d, const double* pts, int64_t ldp,
                          double sigma, int64_t dense_cap, int where, npcg_op** out);
/* synthesize_operator(profile, seed), operators.cpp:211-219: Q from a seeded
 * Gaussian, A = Q diag(lambda) Q^T symmetrised — on the device. */
int npcg_op_synthesize(npcg_ctx* ctx, int64_t n, const double* lambda, uint64_t seed,
                       npcg_op** out);
/* A = G diag(lambda) G^T / r (low-rank synthetic psd; BASELINE config 5). */
int npcg_op_lowrank_create(npcg_ctx* ctx, int64_t n, int64_t r, const double* g, int64_t ldg,
                           const double* lambda, int where, npcg_op** out);
/* Row-sharded operators for an explicit local block (sharded contexts, see
 * npcg_ctx_create_sharded): the column block A[:, R_g] (n x count(rank)) of a
 * symmetric A, and the row block X_g (m_local x n) of a ridge design with
 * m_total rows. The regular constructors above take the full data on a
 * sharded context and keep this rank's share themselves (dense: A[:, R_g];
 * Gram: the rows of X; kernel: K[:, R_g] built from all points, or a share
 * of the matrix-free work; low-rank: G diag(lambda) G[R_g]^T / r). */
int npcg_op_dense_shard_create(npcg_ctx* ctx, int64_t n, const double* a_block, int64_t lda, int where,
                               npcg_op** out);
int npcg_op_gram_shard_create(npcg_ctx* ctx, int64_t m_local, int64_t n, const double* g, int64_t ldg,
                              int where, int64_t m_total, npcg_op** out);
/* The reference's plug-in point: a user subclass of LinearOperator
 * (operators.hpp:25-47, NVI do_matvec / do_apply_block / do_column) as a
 * device operator every entry point accepts (sketch, power method, PCG,
 * block PCG). `apply` computes out = A V for k columns (n x k, col-major):
 *   where = NPCG_HOST:   host buffers; the library synchronises its stream,
 *                        copies V out, calls `apply`, copies out back in;
 *   where = NPCG_DEVICE: device pointers of the context's GPU; `stream` is the
 *                        library's cudaStream_t and the callback must order
 *                        its work on it (no host synchronisation needed).
 * `column` (nullable: no column access, operators.cpp:42-50) writes A(:, j).
 * A non-zero return from a callback fails the calling entry point with
 * NPCG_ERUNTIME ("LinearOperator callback failed ..."). `user` is borrowed
 * and must outlive the operator. */
typedef int (*npcg_apply_fn)(void* user, int64_t n, int64_t k, const double* v, int64_t ldv, double* out,
                             int64_t ldo, void* stream);
typedef int (*npcg_column_fn)(void* user, int64_t j, double* out, void* stream);
int npcg_op_callback_create(npcg_ctx* ctx, int64_t n, npcg_apply_fn apply, npcg_column_fn column, void* user,
                            int where, npcg_op** out);
/* RegularizedOperator(base, mu) / regularize (operators.hpp:69-94,153;
 * operators.cpp:82-103,201-203): A_mu v = base v; += mu v (the reference's
 * rounding order). mu >= 0 (invalid_argument otherwise). Non-owning view of
 * `base`, which must outlive the result (the reference's reference
 * constructor; the C++ facade holds a shared_ptr for the owning one). No
 * column access, as in the reference. cg on it (npcg_pcg with pre = NULL,
 * mu = 0) runs the same fused kernels as nystrom_pcg on base with mu. */
int npcg_op_regularize(npcg_op* base, double mu, npcg_op** out);
int npcg_op_destroy(npcg_op* op);
int npcg_op_dim(const npcg_op* op, int64_t* n);
/* This rank's row block [offset, offset + count) of the operator's vectors
 * (offset 0, count n on an unsharded context). */
int npcg_op_rows(const npcg_op* op, int64_t* offset, int64_t* count);
int npcg_op_kind(const npcg_op* op); /* 0 dense, 1 gram, 2 kernel stored, 3 kernel matrix-free, 4 user callback,
                                        5 regularized */
int npcg_op_has_column_access(const npcg_op* op);
/* LinearOperator::matvec / apply_block (operators.cpp:25-40): dim + finiteness
 * checks, then A V. V and out are rows x k col-major. */
int npcg_op_apply(npcg_op* op, int64_t rows, int64_t k, const double* v, int64_t ldv, double* out,
                  int64_t ldo, int where);
/* LinearOperator::column (operators.cpp:42-50). */
int npcg_op_column(npcg_op* op, int64_t j, double* out, int where);

/* ---- Nyström (nystrom.hpp:19-89) ---------------------------------------- */
/* make_empty_sketch(n) bound to op (nystrom.cpp:28-34). */
int npcg_nys_create(npcg_op* op, npcg_nys** out);
/* Rebind the sketch pair to `op` (same dimension) for the next extend: the
 * reference passes the operator to every extend_sketch call
 * (nystrom.cpp:36-58) rather than storing it in the SketchPair. */
int npcg_nys_bind(npcg_nys* nys, npcg_op* op);
/* extend_sketch (nystrom.cpp:36-58) with the raw n x extra Gaussian block the
 * reference Rng would draw (gaussian_matrix); block Gram-Schmidt x2 against
 * the existing columns, orthonormalisation and Y_new = A Q_new on device. */
int npcg_nys_extend(npcg_nys* nys, int64_t extra, const double* omega_raw, int64_t ld, int where);
/* Same, drawing the block from `rng` (exact reference stream order). */
int npcg_nys_extend_rng(npcg_nys* nys, int64_t extra, npcg_rng* rng);
/* extend_sketch_columns (nystrom.cpp:60-94): `extra` distinct unused columns
 * drawn from `rng` (Fisher-Yates over the unused indices); Omega gets unit
 * columns, Y the columns of A. The drawn indices accumulate in the handle. */
int npcg_nys_extend_columns(npcg_nys* nys, int64_t extra, npcg_rng* rng);
/* Indices drawn so far by column-sampling sketches (out nullable: count only). */
int npcg_nys_used(const npcg_nys* nys, int64_t* out, int64_t* count);
/* column_sampling_nystrom (nystrom.cpp:150-184): `ell` indices drawn from rng
 * (indices == NULL), or the caller's distinct indices; returns the factored handle. */
int npcg_column_sampling_nystrom(npcg_op* op, int64_t ell, const int64_t* indices, npcg_rng* rng, npcg_nys** out);
/* nystrom_from_sketch (nystrom.cpp:96-140): shift, Cholesky (x10 escalation,
 * <= 3 retries), triangular solve, thin SVD, clamp. */
int npcg_nys_factor(npcg_nys* nys);
/* A factored approximation given directly (U n x ell, lambda ell). */
int npcg_nys_from_factors(npcg_ctx* ctx, int64_t n, int64_t ell, const double* u, int64_t ldu,
                          const double* lambda, double shift_used, int where, npcg_nys** out);
int npcg_nys_info(const npcg_nys* nys, int64_t* n, int64_t* sketch_cols, int64_t* ell_factored,
                  double* shift_used);
/* This rank's rows [offset, offset + count) of Omega, Y and U. */
int npcg_nys_rows(const npcg_nys* nys, int64_t* offset, int64_t* count);
/* lambda (ell), U (n x ell, nullable) of the factored approximation. */
int npcg_nys_get(npcg_nys* nys, double* lambda, double* u, int64_t ldu, int where);
/* The cached sketch pair (omega, y: n x size), nullable outputs. */
int npcg_nys_get_sketch(npcg_nys* nys, double* omega, double* y, int64_t ld, int where);
/* A second handle on the same sketch pair and factored approximation, O(1):
 * the sketch storage is shared copy-on-append (appending through one handle
 * never changes what the other sees), the factors are immutable and shared.
 * This gives the reference's value semantics -- extend_sketch returns a new
 * SketchPair and leaves its input unchanged (nystrom.cpp:36-58), and a
 * NystromApproximation / preconditioner is unaffected by later extends or
 * refactors of the pair it came from. factors_only != 0: the clone holds only
 * the approximation (no sketch, no operator). */
int npcg_nys_clone(const npcg_nys* nys, int factors_only, npcg_nys** out);
int npcg_nys_destroy(npcg_nys* nys);

/* ---- preconditioner (preconditioner.hpp:20-65) --------------------------- */
/* build_preconditioner(approx, mu), preconditioner.cpp:80-89 (mu > 0). The
 * preconditioner keeps its own reference to the factors: later extends /
 * refactors of `nys` (or destroying it) do not affect it. */
int npcg_pre_create(npcg_nys* nys, double mu, npcg_pre** out);
/* apply_inverse / apply_inverse_block (preconditioner.cpp:27-45), R n x s. */
int npcg_pre_apply_inverse(npcg_pre* pre, int64_t s, const double* r, int64_t ldr, double* z,
                           int64_t ldz, int where);
/* apply (preconditioner.cpp:17-25). */
int npcg_pre_apply(npcg_pre* pre, int64_t s, const double* v, int64_t ldv, double* out,
                   int64_t ldo, int where);
int npcg_pre_destroy(npcg_pre* pre);
/* woodbury_inverse_apply(approx.u, approx.lambda, mu, B) (preconditioner.cpp:104-114):
 * X = (U diag(lambda) U^T + mu I)^-1 B for B n x s, mu > 0. sketch_and_solve
 * (:116-121) = randomized_nystrom + this (C++/Python facades). */
int npcg_woodbury_inverse_apply(npcg_nys* nys, double mu, int64_t s, const double* b, int64_t ldb, double* x,
                                int64_t ldx, int where);

/* ---- solvers (solvers.hpp:20-93) ----------------------------------------- */
typedef struct {
  double eta;        /* SolveOptions::eta      (default 1e-10) */
  int64_t max_iter;  /* SolveOptions::max_iter (default 500)   */
  int relative;      /* SolveOptions::relative                 */
  int record_iterates;
} npcg_solve_opts;

typedef struct {
  int64_t iterations;
  int64_t matvec_count;
  int converged;
  int status;        /* 0 ok/max_iter, 1 breakdown (p'Ap <= 0), 2 non-finite residual, 3 non-finite initial */
  double eta_used;
  double wall_time;
  int64_t history_len;
} npcg_solve_report;

/* nystrom_pcg (solvers.cpp:122-148) on s independent right-hand sides that
 * share one pass over A per iteration (column j == nystrom_pcg on column j).
 * pre == NULL -> identity (cg on A + mu I, solvers.cpp:111-120).
 * history: s x (max_iter+1) col-major residual norms (nullable).
 * iterates: (max_iter+1) x n x s (nullable; needs record_iterates); only the
 * rows t < max history_len are written (device memory grows with the loop).
 * Returns NPCG_EDIVERGED if any column diverged (its report says which). */
int npcg_pcg(npcg_op* op, npcg_pre* pre, double mu, int64_t s, const double* b, int64_t ldb,
             const double* x0, int64_t ldx0, const npcg_solve_opts* opts, double* x, int64_t ldx,
             npcg_solve_report* reports, double* history, double* iterates, int where);

/* Regularisation path (the paper's protocol):
 * one Nystrom approximation `nys` reused for every mu; for k = 0..nmu-1 the
 * preconditioner is rebuilt for mus[k] (only its l gains change) and the s
 * right-hand sides are solved together (npcg_pcg). warm_start != 0 starts mu_k
 * from the solutions of mu_{k-1} (the paper goes from the largest mu down),
 * otherwise from 0. With cold starts the systems of different mu are
 * independent: on a stored dense operator 8 / s consecutive mu (s = 1, 2, 4)
 * run as one 8-column solve, every column with its own shift and gains, so a
 * pass over A serves all of them; each column reports what its own solve
 * would. x: n x s per mu, mu-major (x + k * s * ldx), nullable;
 * reports: nmu x s, mu-major. A diverged column is reported (status), not
 * fatal: the path goes on. */
int npcg_regularization_path(npcg_op* op, npcg_nys* nys, int64_t nmu, const double* mus, int64_t s,
                             const double* b, int64_t ldb, const npcg_solve_opts* opts, int warm_start,
                             double* x, int64_t ldx, npcg_solve_report* reports, int where);

/* block_nystrom_pcg (solvers.cpp:150-279), O'Leary block PCG, 1 <= s <= 32
 * (one joint Krylov space; not separable into batches).
 * history: s x (max_iter+1) col-major per-column residual norms of every
 * iteration (BlockSolveReport::residual_history, solvers.hpp:40-49), with
 * history_len[j] entries valid (both nullable). */
typedef struct {
  int64_t iterations;
  int64_t fallback_count;
  int64_t n_deflated;
  double eta_used;
  double wall_time;
} npcg_block_report;
int npcg_block_pcg(npcg_op* op, npcg_pre* pre, double mu, int64_t s, const double* b, int64_t ldb,
                   const npcg_solve_opts* opts, double* x, int64_t ldx, npcg_block_report* rep,
                   int* converged, int64_t* deflated, double* final_residual, double* history,
                   int64_t* history_len, int where);

/* iteration_bound (solvers.cpp:281-291). */
int npcg_iteration_bound(double kappa, double epsilon, int64_t* out);

/* ---- adaptive (adaptive.hpp:26-85) -------------------------------------- */
/* estimate_error_power (adaptive.cpp:83-109) from a caller-drawn raw start
 * vector g (n; the Rng's gaussian_vector). */
int npcg_power_estimate(npcg_op* op, npcg_nys* nys, int64_t q, const double* g_raw, int where,
                        double* estimate);
int npcg_power_estimate_rng(npcg_op* op, npcg_nys* nys, int64_t q, npcg_rng* rng, double* estimate);

typedef struct {
  int64_t ell0, ell_max;
  double mu;
  int tol_mode;       /* 0 error (strategy 1), 1 ratio (strategy 2), 2 fixed (strategy 3) */
  int has_tau;
  double tau;         /* default 30 (error) / 10 (ratio) */
  int64_t q;          /* power iterations, default 5 */
  int secondary_criterion;
  int sketch;         /* 0 gaussian, 1 column sampling (needs column access) */
} npcg_adaptive_cfg;

typedef struct {
  int64_t ell_final, doublings;
  int hit_cap;
  int has_error_estimate;
  double error_estimate;
  double posterior_condition;
} npcg_adaptive_outcome;

/* adaptive_nystrom / adaptive_nystrom_ratio / fixed_rank_nystrom
 * (adaptive.cpp:50-148). Ω blocks and power-method start vectors are drawn
 * from `rng` in the reference's exact stream order. */
int npcg_adaptive(npcg_op* op, const npcg_adaptive_cfg* cfg, npcg_rng* rng, npcg_nys** out,
                  npcg_adaptive_outcome* outcome);
/* posterior_condition_estimate (adaptive.cpp:150-156). */
int npcg_posterior_condition(double lambda_ell, double mu, double err, double* out);

/* ---- dense helpers (dense.hpp:26-50), on device ------------------------- */
int npcg_orthonormal_columns(npcg_ctx* ctx, int64_t m, int64_t n, const double* g, double* q,
                             int where);                                    /* dense.cpp:98-117 */
int npcg_thin_svd(npcg_ctx* ctx, int64_t m, int64_t n, const double* b, double* u, double* s,
                  int where);                                               /* dense.cpp:81-96  */
double npcg_ulp_spacing(double x);                                          /* dense.cpp:119-122 */
/* The FP64 DMMA GEMM every O(n l^2) / O(n^2 l) step runs on:
 * C = alpha op(A) op(B) + beta C. a_kmajor: A stored K x M (A^T), else M x K;
 * b_kmajor: B stored K x N, else N x K (B^T). (Eigen GEMM call sites:
 * operators.cpp:76-78,118-121; nystrom.cpp:48-49,116; dense.cpp:98-117.) */
int npcg_gemm(npcg_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha, const double* a, int64_t lda,
              int a_kmajor, const double* b, int64_t ldb, int b_kmajor, double beta, double* c, int64_t ldc,
              int where);

/* C = A B run on the INT8 tensor cores by digit-plane splitting (ozaki.cuh):
 * the sketch products Y = A Omega of stored and matrix-free kernel operators
 * (nystrom.cpp:56 through operators.cpp:76-78) and the factorisation's
 * Grams / triangular solve / U = Q V (nystrom.cpp:115-122, dense.cpp:81-117).
 * A stored K x M (a_kmajor) or M x K; B stored K x N (b_kmajor) or N x K. */
int npcg_gemm_ozaki(npcg_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int a_kmajor,
                    const double* b, int64_t ldb, int b_kmajor, double* c, int64_t ldc, int where);
/* Diagnostics: C32 (m x n col-major int32) = A8 B8^T, A8 m x kp and B8 n x kp
 * row-major int8 host arrays (kp % 128 == 0), on the tcgen05 INT8 GEMM. */
int npcg_gemm_i8(npcg_ctx* ctx, int64_t m, int64_t n, int64_t kp, const int8_t* a8, const int8_t* b8,
                 int32_t* c32);

#ifdef __cplusplus
}
#endif
#endif /* NPCG_CAPI_H */
