// Symmetric eigenvectors of a small dense matrix on device (see eig.cu).
#pragma once

#include <vector>

#include "blas.cuh"
#include "context.cuh"

namespace npcg {

/// Z (n x n, ld ldz) <- eigenvectors of the symmetric n x n matrix M
/// (overwritten), in increasing eigenvalue order. Backward-stable
/// (Householder tridiagonalisation + bisection + inverse iteration); the
/// columns are orthonormal to the working accuracy of inverse iteration and
/// should be re-orthonormalised by the caller.
void sym_eigvecs(Ctx& ctx, double* M, i64 ldm, i64 n, double* Z, i64 ldz);

}  // namespace npcg
