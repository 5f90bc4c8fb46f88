// Level-1/2 building blocks on device (all FP64, column-major, deterministic
// reductions). These are the HBM-streaming kernels of the PCG loop and the
// Nyström pipeline; see blas.cu for the layouts and roofline notes.
#pragma once

#include "context.cuh"

namespace npcg {

/// dst(rows x cols, ldd) = src(rows x cols, lds), device to device.
void copy2d(Ctx& ctx, i64 rows, i64 cols, const double* src, i64 lds, double* dst, i64 ldd);
/// Host/device -> device matrix with ld conversion (pads stay zero).
void upload(Ctx& ctx, DMat& dst, i64 rows, i64 cols, const double* src, i64 lds, int where);
/// Device matrix -> host/device buffer with leading dimension ldd.
void download(Ctx& ctx, const double* src, i64 lds, i64 rows, i64 cols, double* dst, i64 ldd, int where);
/// true iff every entry of the rows x cols block is finite (synchronises).
bool all_finite(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld);
/// sum of squares of a rows x cols block, deterministic (synchronises).
double sum_squares(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld);
/// Row-sharded reductions: the same over this rank's row block, combined over
/// every rank of a sharded context (collective: every rank must call, also
/// with zero local rows). Identical to the plain ones unsharded.
bool all_finite_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld);
double sum_squares_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld);
double max_abs_rows(Ctx& ctx, const double* p, i64 rows, i64 cols, i64 ld);
/// max |a_ij - a_ji| and max |a_ij| of a square matrix (synchronises).
void symmetry_stats(Ctx& ctx, const double* a, i64 n, i64 ld, double* asym, double* amax);
/// Y = X + a * Y  elementwise on rows x cols (ld shared).
void axpby(Ctx& ctx, i64 rows, i64 cols, double a, const double* x, double b, double* y, i64 ld);
/// out = a + nu * b (rows x cols, shared ld).
void add_scaled(Ctx& ctx, i64 rows, i64 cols, const double* a, double nu, const double* b, double* out, i64 ld);
/// out = a + b (each with its own leading dimension).
void add2d(Ctx& ctx, i64 rows, i64 cols, const double* a, i64 lda, const double* b, i64 ldb, double* out, i64 ldo);
/// y /= d elementwise (division, as the reference's `out /= n_rows`).
void divide(Ctx& ctx, i64 rows, i64 cols, double* y, i64 ld, double d);
/// out = (a + a^T) / 2 for a square n x n matrix (out must not alias a).
void symmetrize(Ctx& ctx, const double* a, i64 n, i64 lda, double* out, i64 ldo);
/// a(:, j) *= d(j)  (d on device).
void scale_cols(Ctx& ctx, double* a, i64 rows, i64 cols, i64 lda, const double* d);
/// dst (cols x rows) = src^T (src rows x cols).
void transpose(Ctx& ctx, const double* src, i64 lds, i64 rows, i64 cols, double* dst, i64 ldd);
/// transpose() on stream `s`, OR-ing 1 into *bad (device) when src holds a non-finite entry.
void transpose_checked(Ctx& ctx, cudaStream_t s, const double* src, i64 lds, i64 rows, i64 cols, double* dst,
                       i64 ldd, int* bad);
/// max |a_ij| of a block (synchronises).
double max_abs(Ctx& ctx, const double* a, i64 rows, i64 cols, i64 ld);
/// a *= 2^e exactly (ldexp).
void scale_pow2(Ctx& ctx, i64 rows, i64 cols, double* a, i64 ld, int e);
/// Set to the identity (rows x cols).
void set_identity(Ctx& ctx, double* a, i64 rows, i64 cols, i64 ld);

/// out(j, s) = sum_i M(i, j) * X(i, s) for j < ncols, s < S (partial over row
/// splits summed in fixed order). M is nrows x ncols col-major. When
/// `shift_src` != nullptr: out(j, s) += mu * shift_src(j, s) (symmetric A_mu p).
void coldot(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* X, i64 ldx, int S,
            double* out, i64 ldo, double mu = 0.0, const double* shift_src = nullptr, i64 ldsh = 0,
            const int* gate = nullptr);
/// out(i, s) = base(i, s) + sum_j M(i, j) * c(j, s)   (M nrows x ncols, c ncols x S).
/// base may be nullptr (treated as 0). `gate` (device int, nullable): when it
/// reads 0 every CTA exits at once (lets a converged PCG loop run dry cheaply).
void rowdot(Ctx& ctx, const double* M, i64 ldm, i64 nrows, i64 ncols, const double* c, i64 ldc, int S,
            const double* base, i64 ldb, double* out, i64 ldo, const int* gate = nullptr);

}  // namespace npcg
