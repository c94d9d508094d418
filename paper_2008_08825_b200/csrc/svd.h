// svd.h — bidiagonalisation and its back-transformations (the zgesvd replacement).
#pragma once

#include "common.cuh"

namespace bseg {

constexpr int kGebrdNB = 32;

// A (n x n) = Q B P^H, B upper bidiagonal (d: n, e: n-1, real). Reflectors: column j of A
// below the diagonal holds v_j (unit at j); row j right of the superdiagonal holds u_j
// (unit at j+1, stored unconjugated). tauq: n, taup: n-1.
size_t gebrd_workspace_bytes(int64_t n);
void zgebrd_upper(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tauq, z_t* taup, void* ws);

// Z <- Q Z and Z <- P Z (n x ncols).
size_t unmbr_workspace_bytes(int64_t n, int64_t ncols);
void zunmbr_q(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tauq, z_t* Z,
              int64_t ldz, int64_t ncols, void* ws);
void zunmbr_p(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* taup, z_t* Z,
              int64_t ldz, int64_t ncols, void* ws);

}  // namespace bseg
