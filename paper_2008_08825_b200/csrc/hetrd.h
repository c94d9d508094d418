// hetrd.h — tridiagonalisation / back-transformation and tridiagonal divide & conquer.
#pragma once

#include "common.cuh"

namespace bseg {

constexpr int kHetrdNB = 32;

// A (lower) := reflectors; d (n), e (n-1) real tridiagonal; tau (n-1).
size_t hetrd_workspace_bytes(int64_t n);
void zhetrd_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tau, void* ws);

// Z (n x ncols) <- Q Z with Q from zhetrd_lower's reflectors.
size_t unmtr_workspace_bytes(int64_t n, int64_t ncols);
void zunmtr_lower(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau, z_t* Z,
                  int64_t ldz, int64_t ncols, void* ws);

// Z <- H(0)..H(nref-1) Z ; mode 0: zhetrd 'L' reflectors, 1: zgebrd Q (columns),
// 2: zgebrd P (rows). Workspace: unmtr_workspace_bytes(n, ncols).
void apply_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                      int64_t lda, const z_t* tau, z_t* Z, int64_t ldz, int64_t ncols, void* ws);

// Symmetric tridiagonal eigensolver (Cuppen divide & conquer with Gu-Eisenstat vectors).
// d (n) diagonal, e (n-1) off-diagonal (device). On exit d holds eigenvalues ascending and
// Q (n x n, ld n, real) the orthonormal eigenvectors. Returns nonzero on failure.
size_t stedc_workspace_bytes(int64_t n);
void dstedc(cudaStream_t s, int64_t n, double* d, const double* e, double* Q, void* ws,
            int* d_info,
            int64_t keep_from = 0);

}  // namespace bseg
