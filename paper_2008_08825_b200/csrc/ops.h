// ops.h — O(n^2) glue kernels of the hot path (see ops.cu).
#pragma once

#include <algorithm>

#include "common.cuh"

namespace bseg {

void zaddsub(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
             z_t* M1, z_t* M2, int64_t ldm);
void real_to_complex(cudaStream_t s, int64_t rows, int64_t cols, const double* Z, int64_t ldz,
                     z_t* out, int64_t ldo);
// counts[0] = #flagged, counts[1] = #nonpositive, counts[2] = status (1: no positive entry)
void clamp_spectrum(cudaStream_t s, int64_t n, const double* d, int mode, double* lambda,
                    int64_t* flagged, int64_t* nonpos, int64_t* counts, double* floor_out);
void assemble(cudaStream_t s, int64_t n, int64_t k, const z_t* V1, int64_t ld1, const z_t* V2,
              int64_t ld2, const double* l1, const double* l2, int l2_is_one, const double* dsq,
              const double* floor_p, z_t* V, int64_t ldv);
void check_scales(cudaStream_t s, int64_t k, const double* l1, const double* l2, int* bad);
void tgk_build(cudaStream_t s, int64_t n, const double* d, const double* e, double* td,
               double* te);
void tgk_extract(cudaStream_t s, int64_t n, const double* X, z_t* Ub, int64_t ldu, z_t* Vb,
                 int64_t ldv);
// Re-orthonormalises the extracted bidiagonal singular vectors Ub, Vb (n x n, columns in
// ascending-sigma order sasc) whose sigma is below 1e-3 sigma_max, from the largest of them
// down, each against every column with a larger sigma (block CGS2 + in-block MGS; a column
// that collapses onto later ones -- numerically zero sigma, where the TGK eigenvectors of +s
// and -s mix -- is replaced by a pseudo-random direction and orthonormalised again). The
// change of such a column is of the size of its error, so sigma_j |du_j| stays at the
// eps ||B|| level (backward stable). ws: n * 32 complex; kcount: one device int. Syncs the
// stream once (to size the work); no further work when no sigma is that small.
void tgk_reorthogonalize(cudaStream_t s, int64_t n, const double* sasc, z_t* Ub, z_t* Vb,
                         int64_t ld, z_t* ws, int* kcount);
// Relative-accuracy bisection refinement of ascending bidiagonal singular values (in place).
// scratch: 2n + 2 doubles.
void tgk_refine(cudaStream_t s, int64_t n, const double* d, const double* e, double* sig,
                double* scratch);
void scale_cols_rsqrt(cudaStream_t s, int64_t rows, int64_t cols, z_t* X, int64_t ldx,
                      const double* lam);
void square_vec(cudaStream_t s, int64_t n, const double* a, double* b);
// A(i,i) *= f
void scale_diag(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double f);
// M(i,j) = X(i,j) + conj(X(j,i)) for i >= j (lower triangle of X + X^H)
void herm_lower_sum(cudaStream_t s, int64_t n, const z_t* X, int64_t ldx, z_t* M, int64_t ldm);
void reverse_real(cudaStream_t s, int64_t n, const double* a, double* b);
void reverse_cols(cudaStream_t s, int64_t rows, int64_t cols, const z_t* a, int64_t lda, z_t* b,
                  int64_t ldb);
void herm_dev_partials(cudaStream_t s, int64_t n, const z_t* M, int64_t ld, double* part,
                       int nblocks);

}  // namespace bseg
