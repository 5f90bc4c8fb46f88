// FP64 GEMM emulated on the INT8 tensor cores (tcgen05.mma kind::i8, TMEM
// accumulators, TMA-fed) by operand splitting (the Ozaki scheme).
//
// Every row r of the K-major operands A (M x K) and B^T (N x K) is scaled by
// 2^-E_r (E_r the exponent of the row's largest |entry|) and cut into NS
// signed 7-bit digit planes by round-to-nearest:
//     a = 2^E * sum_t d_t 2^(-6-7(t-1)),  |d_t| <= 64,  residual < 2^(E-7NS+1)
// (NS = 8: 55 bits below the row maximum, finer than an FP64 ulp of it). The
// digit products are exact integers, so
//     (AB)_ij = 2^(E_i+F_j) sum_g 2^(-12-7(g-2)) P_g,  P_g = sum_{t+u=g} (D_t D'_u)_ij
// and P_g (g = 2 .. NS+1) is one int8 GEMM over the concatenated K of its g-1
// plane pairs, accumulated exactly in int32 (|P_g| < 2^31 for K <= 65408;
// longer K is chunked). The planes g > NS+1 are below the truncation error and
// are not formed. The FP64 result is assembled in fixed order (deterministic).
#pragma once

#include "context.cuh"
#include "gemm.cuh"

namespace npcg {

/// C (M x N, col-major, ldc) = A B + beta C (beta 0 or 1). A K-major (entry
/// (m,k) at A[k + m*lda]) or M-major (at A[m + k*lda]); B K-major (entry (k,n)
/// at B[k + n*ldb]). FP64 in and out; the products run on the INT8 tensor pipe.
void gemm_ozaki(Ctx& ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, bool a_kmajor, const double* B, i64 ldb,
                double beta, double* C, i64 ldc, bool b_kmajor = true);


/// Digit planes of one operand: `rows` rows of K entries (planes [NS][rows][Kp]
/// int8, K contiguous, zero-padded to Kp), one exponent per row.
struct OzakiPlanes {
  DBuf<int8_t> d;
  DBuf<int> e;     // row exponents (entries < 2^e)
  DBuf<double> s;  // 2^e
  i64 rows = 0, K = 0, Kp = 0;
};
/// Split rows x K operand P (kmajor: row r at P + r*ld, contiguous; else entry
/// (r, k) at P[r + k*ld]) into planes.
void ozaki_split(Ctx& ctx, const double* P, i64 ld, bool kmajor, i64 rows, i64 K, OzakiPlanes& out);
/// Whether ozaki_split can read P (K-major rows must be 16-byte aligned pairs).
bool ozaki_splittable(const double* P, i64 ld, bool kmajor);
/// C (A.rows x B.rows) = A B^T over A's K entries + beta C, B's planes taken from
/// K offset k_off_b (a multiple of 128): one split of a long operand serves
/// products over any 128-aligned range of it.
void gemm_ozaki_planes(Ctx& ctx, const OzakiPlanes& A, const OzakiPlanes& B, i64 k_off_b, double beta, double* C,
                       i64 ldc);

/// False when NPCG_OZAKI=0 (diagnostics: every product stays on the FP64 DMMA GEMM).
bool ozaki_enabled();

/// Raw INT8 GEMM (diagnostics / tests): C32 (M x N col-major int32) = A8 B8^T,
/// A8 M x Kp and B8 N x Kp row-major int8 (K contiguous, Kp % 128 == 0).
void gemm_i8_raw(Ctx& ctx, int M, int N, i64 Kp, const int8_t* A8, const int8_t* B8, int32_t* C32);

}  // namespace npcg
