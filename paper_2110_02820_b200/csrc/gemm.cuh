// FP64 tensor-core GEMM for sm_100a: TMA (cp.async.bulk.tensor, 128B swizzle)
// feeds a multi-stage mbarrier pipeline; 8 consumer warps run DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; tcgen05 has no f64 kind).
#pragma once

#include "context.cuh"

namespace npcg {

/// One GEMM operand in column-major device memory.
///  A (logical M x K): kmajor -> stored K x M (elem (m,k) at k + m*ld), i.e. A^T;
///                     else   -> stored M x K (elem (m,k) at m + k*ld).
///  B (logical K x N): kmajor -> stored K x N (elem (k,n) at k + n*ld);
///                     else   -> stored N x K (elem (k,n) at n + k*ld), i.e. B^T.
struct Operand {
  const double* p;
  i64 ld;
  bool kmajor;
};

/// Optional epilogue: the Gaussian kernel entry K_ij = exp(max(0, (alpha AB_ij
/// + norms_i) + norms_j) * c), K_ii = 1 (operators.cpp:125-137), applied to the
/// tile in registers instead of a second pass over C (beta must be 0).
struct GemmEpi {
  const double* norms = nullptr;
  double c = 0.0;
  /// Gram product (B = A^T, M = N, beta = 0): C is symmetric, so only the tiles
  /// that reach the diagonal or lie above it are computed (36 of 64 at n =
  /// 1000) and the strict lower triangle is mirrored from the upper one.
  bool sym = false;
  /// Triangular B (logical K x N with B[k, n] = 0 for k > n, e.g. L^{-T}):
  /// the K loop of an n-tile stops at the tile's last column.
  bool tri = false;
};

/// C (M x N, col-major, ldc) = alpha * A B + beta * C. Deterministic (split-K
/// partials are reduced in fixed order). All leading dimensions must be
/// multiples of 2 and pointers 16-byte aligned (dev_ld() matrices are).
void gemm(Ctx& ctx, i64 M, i64 N, i64 K, double alpha, Operand A, Operand B, double beta,
          double* C, i64 ldc, GemmEpi epi = GemmEpi{});

}  // namespace npcg
