// potrf.cu — blocked right-looking Cholesky, lower (replaces LAPACKE_zpotrf 'L' at
// proj/src/backend.cpp:51 and its NotPositiveDefinite pivot report, backend.cpp:52-56).
//
// Per nb = 64 block column j:
//   1. one CTA factors the nb x nb diagonal block in shared memory (unblocked, right-looking),
//      reports the first non-positive / NaN pivot (LAPACK info = j+1), and inverts L_jj;
//   2. panel TRSM  A21 <- A21 * L_jj^{-H}            (DMMA GEMM, in place, one CTA per row block)
//   3. HERK update A22 <- A22 - A21 * A21^H (lower)  (DMMA GEMM, lower tiles only)
#include "blas.h"
#include "gemm.cuh"

namespace bseg {

namespace {
constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
}

__global__ void __launch_bounds__(256) zpotrf_diag_kernel(z_t* A, int64_t lda, int jb,
                                                          int64_t j0, int* info, z_t* inv) {
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* Ls = reinterpret_cast<z_t*>(sm);   // column-major, ld kLD
  z_t* Xs = Ls + kNB * kLD;              // Xs[i*kLD + j] = inv(i, j)
  __shared__ int failed;
  const int tid = threadIdx.x;
  if (tid == 0) failed = (*info != 0) ? 1 : 0;  // an earlier block already failed
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e % kNB, j = e / kNB;
    z_t v = make_double2(0.0, 0.0);
    if (i < jb && j < jb && i >= j) v = A[i + int64_t(j) * lda];
    Ls[i + j * kLD] = v;
    Xs[i * kLD + j] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (failed) return;
  for (int c = 0; c < jb; ++c) {
    const double d = Ls[c + c * kLD].x;  // zpotf2 uses the real part of the diagonal
    if (!(d > 0.0)) {                    // also catches NaN (LAPACK: AJJ <= 0 or DISNAN)
      if (tid == 0) {
        if (atomicCAS(info, 0, int(j0 + c + 1)) == 0) {}
        failed = 1;
      }
      __syncthreads();
      return;
    }
    const double l = sqrt(d);
    const double rl = 1.0 / l;
    __syncthreads();
    for (int r = c + 1 + tid; r < jb; r += blockDim.x) Ls[r + c * kLD] = zscale(Ls[r + c * kLD], rl);
    if (tid == 0) Ls[c + c * kLD] = make_double2(l, 0.0);
    __syncthreads();
    // trailing rank-1 update of the lower part: a(r,k) -= l(r,c) * conj(l(k,c)), r >= k > c
    const int rem = jb - c - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int r = c + 1 + e % rem, k = c + 1 + e / rem;
      if (r >= k) {
        z_t v = Ls[r + k * kLD];
        const z_t x = Ls[r + c * kLD], y = Ls[k + c * kLD];
        // v -= x * conj(y)
        v.x -= x.x * y.x + x.y * y.y;
        v.y -= x.y * y.x - x.x * y.y;
        Ls[r + k * kLD] = v;
      }
    }
  }
  __syncthreads();
  // write the factor back (strict upper of the diagonal block zeroed)
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    A[i + int64_t(j) * lda] = (i >= j) ? Ls[i + j * kLD] : make_double2(0.0, 0.0);
  }
  // inverse by forward substitution, 4 lanes per column
  const int col = tid >> 2, q = tid & 3;
  for (int i = 0; i < jb; ++i) {
    z_t part = make_double2(0.0, 0.0);
    if (col < jb && i > col)
      for (int k = col + q; k < i; k += 4) zfma(part, Ls[i + k * kLD], Xs[k * kLD + col]);
    part.x += __shfl_xor_sync(0xffffffffu, part.x, 1);
    part.y += __shfl_xor_sync(0xffffffffu, part.y, 1);
    part.x += __shfl_xor_sync(0xffffffffu, part.x, 2);
    part.y += __shfl_xor_sync(0xffffffffu, part.y, 2);
    if (col < jb && q == 0 && i >= col) {
      const double rl = 1.0 / Ls[i + i * kLD].x;  // diagonal is real positive
      Xs[i * kLD + col] = (i == col) ? make_double2(rl, 0.0) : make_double2(-part.x * rl, -part.y * rl);
    }
    __syncthreads();
  }
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e % kNB, j = e / kNB;
    inv[i + j * kNB] = Xs[i * kLD + j];
  }
}

__global__ void zero_strict_upper_kernel(int64_t n, z_t* A, int64_t lda) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    if (i < j) A[i + j * lda] = make_double2(0.0, 0.0);
  }
}

void zpotrf_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, int* d_info, z_t* ws,
                  bool zero_upper) {
  const size_t smem = size_t(2) * kNB * kLD * sizeof(z_t);
  static bool configured = false;
  if (!configured) {
    BSE_CUDA(cudaFuncSetAttribute(zpotrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    configured = true;
  }
  BSE_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), s));
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0}, mone = {-1.0, 0.0};
  for (int64_t j = 0; j < n; j += kNB) {
    const int jb = int(min64(kNB, n - j));
    z_t* Ajj = A + j + j * lda;
    zpotrf_diag_kernel<<<1, 256, smem, s>>>(Ajj, lda, jb, j, d_info, ws);
    BSE_LAUNCH_CHECK();
    const int64_t rest = n - j - jb;
    if (rest <= 0) break;
    z_t* A21 = A + (j + jb) + j * lda;
    // A21 <- A21 * inv(L_jj)^H : in place is safe because one CTA owns a full row block
    // (jb <= BN) and reads all of it before its epilogue writes.
    zgemm(s, 0, 1, rest, jb, jb, one, A21, lda, ws, kNB, zero, A21, lda, kGeneral, kUpperOp, 0,
          nullptr, 0);
    z_t* A22 = A + (j + jb) + (j + jb) * lda;
    zgemm(s, 0, 1, rest, rest, jb, mone, A21, lda, A21, lda, one, A22, lda, kGeneral, kGeneral, 1,
          nullptr, 0);
  }
  if (zero_upper && n > 1) {
    const int blocks = int(min64(ceil_div(n * n, 256), 148 * 32));
    zero_strict_upper_kernel<<<blocks, 256, 0, s>>>(n, A, lda);
    BSE_LAUNCH_CHECK();
  }
}

}  // namespace bseg
