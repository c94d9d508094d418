// blas.h — host-side declarations of the library's BLAS-like device operations.
#pragma once

#include "common.cuh"

namespace bseg {

enum OpShape : int;

// C = alpha * op(A) * op(B) + beta * C   (complex128, DMMA). opa/opb: 0 = N, 1 = adjoint.
// a_shape/b_shape: 0 general, 1 lower, 2 upper — the shape of op(X); entries outside it are
// treated as zero (TRMM semantics). c_lower: write only the lower triangle of C.
// splitk_ws: optional scratch enabling a deterministic K-split on under-filled grids.
void zgemm(cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, z_t alpha,
           const z_t* A, int64_t lda, const z_t* B, int64_t ldb, z_t beta, z_t* C, int64_t ldc,
           int a_shape, int b_shape, int c_lower, z_t* splitk_ws, int64_t splitk_ws_elems);
void zgemm_batched(cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, z_t alpha,
                   const z_t* A, int64_t lda, int64_t sA, const z_t* B, int64_t ldb, int64_t sB,
                   z_t beta, z_t* C, int64_t ldc, int64_t sC, int batch);
void dgemm_nn(cudaStream_t s, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
              int batch, int64_t sA, int64_t sB, int64_t sC);

void zcopy2d(cudaStream_t s, int64_t rows, int64_t cols, const z_t* src, int64_t lds, z_t* dst,
             int64_t ldd);
// Device -> page-locked host copy by SM loads that leave the block out of L2 (evict-first) and
// streaming stores over PCIe. A copy-engine D2H of a large block streams it through L2 and
// evicts the working sets of the kernels running beside it (the batch lanes' panels and
// GEMMs: measured 5 % slower under a concurrent 512 MB D2H at 12 GB/s, 0.5 % when the source
// stays in L2). Returns false (nothing launched) when dst is not device-accessible pinned
// memory; the caller then uses cudaMemcpy2DAsync.
bool zcopy2d_to_host_streaming(cudaStream_t s, int64_t rows, int64_t cols, const z_t* src,
                               int64_t lds, z_t* dst_host, int64_t ldd);
void ztrtri_diag_blocks(cudaStream_t s, int64_t n, const z_t* L, int64_t ldl, int nb, z_t* inv);

// In-place triangular solve with lower L: side 0 = left, 1 = right; op 0 = N, 1 = adjoint.
// `other` is the extent of X along the non-solved dimension.
size_t trsm_workspace_elems(int64_t n, int64_t other, int nb);
void ztrsm_lower(cudaStream_t s, int side, int op, int64_t n, int64_t other, const z_t* L,
                 int64_t ldl, z_t* X, int64_t ldx, z_t* ws, int nb);

// Blocked Cholesky (lower) in place; *d_info receives LAPACK's info (0 ok, j+1 = first
// failing pivot). Workspace: nb*nb complex. Strict upper left untouched unless zero_upper.
// With s2 and ev[2]: look-ahead, the trailing update beyond the next block column runs on s2
// (the factor is complete when s reaches the end of the enqueued work).
void zpotrf_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, int* d_info, z_t* ws,
                  bool zero_upper, cudaStream_t s2 = nullptr, cudaEvent_t* ev = nullptr);

}  // namespace bseg
