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

namespace npcg {

/// C (M x N, col-major, ldc) = A B, A K-major (entry (m,k) at A[k + m*lda]),
/// B K-major (entry (k,n) at B[k + n*ldb]). FP64 in and out; the products run
/// on the INT8 tensor pipe.
void gemm_ozaki(Ctx& ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* B, i64 ldb, double* C,
                i64 ldc);

/// False when NPCG_OZAKI=0 (diagnostics: every product stays on the FP64 DMMA GEMM).
bool ozaki_enabled();

/// Raw INT8 GEMM (diagnostics / tests): C32 (M x N col-major int32) = A8 B8^T,
/// A8 M x Kp and B8 N x Kp row-major int8 (K contiguous, Kp % 128 == 0).
void gemm_i8_raw(Ctx& ctx, int M, int N, i64 Kp, const int8_t* A8, const int8_t* B8, int32_t* C32);

}  // namespace npcg
