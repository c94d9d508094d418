// potrf.cu — blocked right-looking Cholesky, lower (replaces LAPACKE_zpotrf 'L' at
// proj/src/backend.cpp:51 and its NotPositiveDefinite pivot report, backend.cpp:52-56).
//
// Per nb = 64 block column j:
//   1. one CTA factors the nb x nb diagonal block in shared memory (8-column warp panels +
//      rank-8 updates), reports the first non-positive / NaN pivot (LAPACK info = j+1), and
//      inverts L_jj (8x8 block inverses + block-wavefront products);
//   2. panel TRSM  A21 <- A21 * L_jj^{-H}            (DMMA GEMM, in place, one CTA per row block)
//   3. HERK update A22 <- A22 - A21 * A21^H (lower)  (DMMA GEMM, lower tiles only)
#include "blas.h"
#include "gemm.cuh"

namespace bseg {

namespace {
constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
}

// Factor + invert one jb x jb (jb <= 64) diagonal block in shared memory.
//  factorisation: 8 panels of 8 columns; warp 0 factors a panel (lanes own rows, no block
//    barrier), then all 256 threads apply the rank-8 update to the trailing lower block;
//  inverse: 8x8 diagonal-block inverses (8 warps in parallel), then the block
//    sub-diagonals X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ one wavefront at a time.
// Reports the first non-positive / NaN pivot as LAPACK's info (j0 + c + 1).
__global__ void __launch_bounds__(256) zpotrf_diag_kernel(z_t* A, int64_t lda, int jb,
                                                          int64_t j0, int* info, z_t* inv) {
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* Ls = reinterpret_cast<z_t*>(sm);  // column-major, ld kLD
  z_t* Xs = Ls + kNB * kLD;             // column-major, ld kLD: inverse
  z_t* Ss = Xs + kNB * kLD;             // column-major, ld kLD: wavefront scratch
  __shared__ int failed;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) failed = (*info != 0) ? 1 : 0;  // an earlier block already failed
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e % kNB, j = e / kNB;
    z_t v = make_double2(0.0, 0.0);
    if (i < jb && j < jb && i >= j) v = A[i + int64_t(j) * lda];
    if (i >= jb && i == j) v = make_double2(1.0, 0.0);  // identity padding beyond jb
    Ls[i + j * kLD] = v;
    Xs[i + j * kLD] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (failed) return;
  for (int p0 = 0; p0 < kNB; p0 += 8) {
    if (warp == 0) {
      // panel columns p0..p0+7, rows p0..63 (lanes own rows lane and lane+32)
      for (int c = p0; c < p0 + 8; ++c) {
        const double d = Ls[c + c * kLD].x;  // zpotf2 uses the real part of the diagonal
        const bool bad = !(d > 0.0) && c < jb;  // also catches NaN
        if (bad) {
          if (lane == 0) {
            atomicCAS(info, 0, int(j0 + c + 1));
            failed = 1;
          }
          break;
        }
        const double l = c < jb ? sqrt(d) : 1.0;
        const double rl = 1.0 / l;
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
          if (r > c) Ls[r + c * kLD] = zscale(Ls[r + c * kLD], rl);
        }
        if (lane == 0) Ls[c + c * kLD] = make_double2(l, 0.0);
        __syncwarp();
        // rank-1 update of the remaining panel columns k in (c, p0+8), rows r >= k
        for (int k = c + 1; k < p0 + 8; ++k) {
          const z_t y = Ls[k + c * kLD];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            if (r >= k) {
              const z_t x = Ls[r + c * kLD];
              z_t v = Ls[r + k * kLD];
              v.x -= x.x * y.x + x.y * y.y;  // v -= x conj(y)
              v.y -= x.y * y.x - x.x * y.y;
              Ls[r + k * kLD] = v;
            }
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (failed) return;
    // rank-8 update of the trailing lower block: A(r,k) -= sum_c L(r,c) conj(L(k,c))
    const int t0 = p0 + 8, rem = kNB - t0;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int r = t0 + e % rem, k = t0 + e / rem;
      if (r >= k) {
        z_t v = Ls[r + k * kLD];
#pragma unroll
        for (int c = p0; c < p0 + 8; ++c) {
          const z_t x = Ls[r + c * kLD], y = Ls[k + c * kLD];
          v.x -= x.x * y.x + x.y * y.y;
          v.y -= x.y * y.x - x.x * y.y;
        }
        Ls[r + k * kLD] = v;
      }
    }
    __syncthreads();
  }
  // write the factor back (strict upper of the diagonal block zeroed)
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    A[i + int64_t(j) * lda] = (i >= j) ? Ls[i + j * kLD] : make_double2(0.0, 0.0);
  }
  // 8x8 diagonal-block inverses: warp w inverts block w, lane j < 8 owns column j
  if (lane < 8) {
    const int b0 = warp * 8, j = b0 + lane;
    for (int i = b0; i < b0 + 8; ++i) {
      if (i < j) continue;
      z_t s = (i == j) ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0);
      for (int k = j; k < i; ++k) {
        const z_t lk = Ls[i + k * kLD], xk = Xs[k + j * kLD];
        s.x -= lk.x * xk.x - lk.y * xk.y;
        s.y -= lk.x * xk.y + lk.y * xk.x;
      }
      const double rd = 1.0 / Ls[i + i * kLD].x;  // diagonal is real positive
      Xs[i + j * kLD] = zscale(s, rd);
    }
  }
  __syncthreads();
  // block sub-diagonal wavefronts d = 1..7: X_{J+d,J} = -X_II (sum_{K=J}^{I-1} L_IK X_KJ)
  for (int d = 1; d < 8; ++d) {
    const int nblk = 8 - d;
    for (int e = tid; e < nblk * 64; e += blockDim.x) {
      const int J = e / 64, ij = e % 64, ii = ij % 8, jj = ij / 8;
      const int I = J + d;
      const int row = I * 8 + ii, col = J * 8 + jj;
      z_t s = make_double2(0.0, 0.0);
      for (int k = J * 8; k < I * 8; ++k) zfma(s, Ls[row + k * kLD], Xs[k + col * kLD]);
      Ss[row + col * kLD] = s;
    }
    __syncthreads();
    for (int e = tid; e < nblk * 64; e += blockDim.x) {
      const int J = e / 64, ij = e % 64, ii = ij % 8, jj = ij / 8;
      const int I = J + d;
      const int row = I * 8 + ii, col = J * 8 + jj;
      z_t s = make_double2(0.0, 0.0);
      for (int k = I * 8; k <= row; ++k) zfma(s, Xs[row + k * kLD], Ss[k + col * kLD]);
      Xs[row + col * kLD] = make_double2(-s.x, -s.y);
    }
    __syncthreads();
  }
  for (int e = tid; e < kNB * kNB; e += blockDim.x) {
    const int i = e % kNB, j = e / kNB;
    inv[i + j * kNB] = (i < jb && j < jb) ? Xs[i + j * kLD] : make_double2(0.0, 0.0);
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
  const size_t smem = size_t(3) * kNB * kLD * sizeof(z_t);
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
