// potrf.cu — blocked right-looking Cholesky, lower (replaces LAPACKE_zpotrf 'L' at
// proj/src/backend.cpp:51 and its NotPositiveDefinite pivot report, backend.cpp:52-56).
//
// Per nb = 64 block column j (panels grouped three at a time, see zpotrf_lower):
//   1. zpotrf_panel_kernel: every CTA factors the nb x nb diagonal block in shared memory,
//      CTA 0 writes it back and reports the first non-positive / NaN pivot (LAPACK info),
//      and each CTA solves its 32-row blocks of the panel A21 <- A21 L_jj^{-H} in place;
//   2. HERK update A22 <- A22 - A21 * A21^H (lower)  (DMMA GEMM, lower tiles only)
#include <cstdlib>

#include "blas.h"
#include "gemm.cuh"

namespace bseg {

namespace {
constexpr int kNB = 64;
constexpr int kLD = kNB + 1;
constexpr int kPR = 32;  // panel rows per solve block
}

__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, 256;" ::"r"(id) : "memory");
}

// One block column of the right-looking Cholesky in a single launch: every CTA factors the
// jb x jb diagonal block redundantly in shared memory (identical arithmetic, so identical
// factors), CTA 0 writes L_jj back and reports the first non-positive / NaN pivot as LAPACK's
// info (j0 + c + 1), and each CTA then solves its kPR-row blocks of the panel below,
// A21 <- A21 L_jj^{-H}, by forward substitution in registers. No inverse, no second launch.
//
//  factorisation: warp w owns columns w, w+8, ... (register slots, rotated every 8 steps so
//    the active column is always slot 0), lanes own rows lane and lane+32. Column c is
//    published through a triple-buffered shared column; its producer signals named barrier
//    1 + (c & 1) with bar.arrive and the other warps bar.sync on it. Look-ahead: the owner
//    of column c+1 first applies column c to that one column, pivots and publishes it, and
//    only then updates the rest of its columns, so the pivot chain (shuffle, rsqrt, scale)
//    overlaps the other warps' rank-1 updates.
//  panel solve: 8 threads per row (thread q owns columns q, q+8, ...), the owner of column c
//    finishes X(r,c) and shuffles it to the 7 others, which update their columns k > c. The
//    CTA's first row block is fetched before the factorisation starts.
__global__ void __launch_bounds__(256, 1)
    zpotrf_panel_kernel(z_t* A, int64_t lda, int jb, int64_t j0, int64_t rest, int* info,
                        unsigned* loaded) {
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* Ls = reinterpret_cast<z_t*>(sm);  // factor, column-major, ld kLD
  z_t* col = Ls + kNB * kLD;             // 3 x 64 published columns
  z_t* Bs = col + 3 * kNB;               // kPR x 64 panel rows, ld kPR + 1
  double* rd = reinterpret_cast<double*>(Bs + kNB * (kPR + 1));  // 1 / L(c,c)
  __shared__ int failed;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) failed = (*info != 0) ? 1 : 0;  // an earlier block column already failed
  auto load_rows = [&](int64_t rb) {
    const z_t* B = A + jb + rb * kPR;
    const int rows = int(min64(kPR, rest - rb * kPR));
    for (int e = tid; e < kPR * kNB; e += blockDim.x) {
      const int i = e % kPR, k = e / kPR;
      Bs[i + k * (kPR + 1)] =
          (i < rows && k < jb) ? B[i + int64_t(k) * lda] : make_double2(0.0, 0.0);
    }
  };
  if (int64_t(blockIdx.x) * kPR < rest) load_rows(blockIdx.x);
  // registers: slot j = column warp + 8 j, rows lane (h = 0) and lane + 32 (h = 1)
  z_t reg[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h, k = warp + 8 * j;
      z_t v = make_double2(0.0, 0.0);
      if (r < jb && k < jb && r >= k) v = A[r + int64_t(k) * lda];
      if (r >= jb && r == k) v = make_double2(1.0, 0.0);  // identity padding beyond jb
      reg[j][h] = v;
    }
  __syncthreads();
  if (failed) return;
  // The factor is written back over the diagonal block the CTAs read: only the CTA that
  // loads last (acq_rel count of loaded CTAs; CTAs of one launch need not be co-resident,
  // e.g. behind a concurrent factorisation on another stream) may write it.
  __shared__ int writer;
  if (tid == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(loaded) : "memory");
    writer = (old == gridDim.x - 1) ? 1 : 0;
  }
  // pivot + scale + publish of column c held in register slot `sl` of the owner warp
  auto pivot = [&](int c, z_t (&v)[2]) {
    warp_converge();
    const double d = __shfl_sync(0xffffffffu, c < 32 ? v[0].x : v[1].x, c & 31);
    // zpotf2 uses the real part of the diagonal; !(d > 0) also catches NaN (padding: d = 1)
    if (!(d > 0.0) && lane == 0) {
      if (blockIdx.x == 0) atomicCAS(info, 0, int(j0 + c + 1));
      failed = 1;
    }
    const double rl = rsqrt(d), l = d * rl;
    z_t* cb = col + (c % 3) * kNB;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r > c) v[h] = zscale(v[h], rl);
      if (r == c) v[h] = make_double2(l, 0.0);
      cb[r] = v[h];
    }
    if (lane == 0) rd[c] = rl;
    named_arrive(1 + (c & 1));
  };
  if (warp == 0) pivot(0, reg[0]);
  // fully unrolled: the slot masks (j < 8 - cc) become compile-time, so a step issues only
  // the rank-1 updates of live slots (half the FP64 instructions of the masked loop)
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int c = 8 * cc + s;
      const z_t* cb = col + (c % 3) * kNB;
      if (warp != s) named_sync(1 + (c & 1));
      else __syncwarp();
      // column c at this lane's rows, read once (the look-ahead pivot below writes another
      // buffer, but the compiler cannot prove it and would reload per slot)
      const z_t xc[2] = {cb[lane], cb[lane + 32]};
      // look-ahead: the owner of column c+1 (warp (s+1)&7, slot ps) updates and pivots it
      const int ps = (s == 7) ? 1 : 0;
      const bool ahead = (warp == ((s + 1) & 7)) && (c + 1 < kNB);
      if (ahead) {
        const int k = c + 1;
        const z_t y = cb[k];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = lane + 32 * h;
          if ((h == 1 || k < 32) && r >= k) {
            const z_t x = xc[h];
            z_t& v = reg[ps][h];
            v.x -= x.x * y.x + x.y * y.y;  // v -= x conj(y)
            v.y -= x.y * y.x - x.x * y.y;
          }
        }
        pivot(k, reg[ps]);
      }
      // rank-1 update of the other trailing columns k > c owned by this warp
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = warp + 8 * (cc + j);
        if (j < 8 - cc && k > c && !(ahead && j == ps)) {
          const z_t y = cb[k];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            if ((h == 1 || k < 32) && r >= k) {
              const z_t x = xc[h];
              z_t& v = reg[j][h];
              v.x -= x.x * y.x + x.y * y.y;
              v.y -= x.y * y.x - x.x * y.y;
            }
          }
        }
      }
    }
    // slot 0 (column warp + 8 cc) is final: store it (zeros above the diagonal), rotate
    {
      const int k = warp + 8 * cc;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = lane + 32 * h;
        Ls[r + k * kLD] = (r >= k) ? reg[0][h] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        reg[j][0] = reg[j + 1][0];
        reg[j][1] = reg[j + 1][1];
      }
    }
  }
  __syncthreads();
  if (failed) return;
  if (writer) {
    for (int e = tid; e < jb * jb; e += blockDim.x) {
      const int i = e % jb, j = e / jb;
      A[i + int64_t(j) * lda] = Ls[i + j * kLD];
    }
    if (tid == 0) *loaded = 0u;  // every CTA of this launch has counted; ready for the next
  }
  // panel solve X L^H = B on kPR-row blocks of A21 = A + jb
  const int pr = tid >> 3, q = tid & 7;
  for (int64_t rb = blockIdx.x; rb * kPR < rest; rb += gridDim.x) {
    z_t* B = A + jb + rb * kPR;
    const int rows = int(min64(kPR, rest - rb * kPR));
    if (rb != blockIdx.x) {
      __syncthreads();  // Bs reuse
      load_rows(rb);
      __syncthreads();
    }
    z_t b[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) b[m] = Bs[pr + (q + 8 * m) * (kPR + 1)];
    for (int cc = 0; cc < 8; ++cc) {  // (unrolling this one costs registers: 255, slower)
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int c = 8 * cc + s;
        z_t x = zscale(b[0], rd[c]);
        if (q == s) b[0] = x;
        warp_converge();
        x.x = __shfl_sync(0xffffffffu, x.x, (lane & 24) | s);
        x.y = __shfl_sync(0xffffffffu, x.y, (lane & 24) | s);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int k = q + 8 * (cc + m);
          if (m < 8 - cc && k > c) {
            const z_t y = Ls[k + c * kLD];
            b[m].x -= x.x * y.x + x.y * y.y;  // b -= x conj(L(k,c))
            b[m].y -= x.y * y.x - x.x * y.y;
          }
        }
      }
      Bs[pr + (q + 8 * cc) * (kPR + 1)] = b[0];
#pragma unroll
      for (int m = 0; m < 7; ++m) b[m] = b[m + 1];
    }
    __syncthreads();
    for (int e = tid; e < kPR * jb; e += blockDim.x) {
      const int i = e % kPR, k = e / kPR;
      if (i < rows) B[i + int64_t(k) * lda] = Bs[i + k * (kPR + 1)];
    }
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
                  bool zero_upper, cudaStream_t s2, cudaEvent_t* ev) {
  // ws (>= 64 bytes, distinct per concurrent call) holds the panel kernel's loaded-CTA count
  unsigned* loaded = reinterpret_cast<unsigned*>(ws);
  const size_t smem = size_t(kNB * kLD + 3 * kNB + kNB * (kPR + 1)) * sizeof(z_t) +
                      kNB * sizeof(double);
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(zpotrf_panel_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    return true;
  });
  (void)configured;
  BSE_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), s));
  BSE_CUDA(cudaMemsetAsync(loaded, 0, sizeof(unsigned), s));
  const z_t mone = {-1.0, 0.0}, one = {1.0, 0.0};
  // Look-ahead (with a second stream): the rank-jb update is split into the next block
  // column (on s, so the next panel can start) and the rest of the trailing matrix (on s2,
  // overlapping that panel). ev[0]: panel j done; ev[1]: the s2 update of step j-1 done.
  static const bool no_la = getenv("BSE_POTRF_NO_LA") != nullptr;  // A/B switch
  const bool la = s2 != nullptr && ev != nullptr && !no_la;
  // panels per group (A/B switch BSE_POTRF_GROUP; 1 = the one-panel look-ahead below). n = 4096
  // CHOL zpotrf: 5.48 ms with 1, 5.26 with 2, 5.25 with 3, 5.29 with 4, 5.70 with 6; the two
  // concurrent factorisations of CHOL+SVD: 8.66, 8.18, 7.96, 8.04, 8.21 ms.
  static const int group_env = getenv("BSE_POTRF_GROUP") ? atoi(getenv("BSE_POTRF_GROUP")) : 3;
  const int G = std::max(1, std::min(group_env, 8));
  if (la && G > 1) {
    // Panels in groups of G (left-looking inside the group, right-looking across groups):
    // block column a+q of the group first takes the group's panels a..a+q-1 in ONE rank-64q
    // update, then is factored; after the group the trailing matrix takes ONE rank-64G
    // update (k = 64G instead of G rank-64 updates: fewer C round trips per flop), split
    // into the next group's first block column (s: the critical chain), its other G-1 block
    // columns (s2 first, ev[1]) and the rest (s2, ev[2]). ev[0]: the group's panels done.
    bool pend = false;
    for (int64_t a0 = 0; a0 < n; a0 += int64_t(G) * kNB) {
      bool done = false;
      for (int q = 0; q < G && !done; ++q) {
        const int64_t c = a0 + int64_t(q) * kNB;
        if (c >= n) {
          done = true;
          break;
        }
        const int jbq = int(min64(kNB, n - c));
        const int64_t restq = n - c - jbq;
        if (q > 0) {  // the group's previous panels -> block column c (rows >= c)
          if (q == 1 && pend) BSE_CUDA(cudaStreamWaitEvent(s, ev[1], 0));
          const z_t* P = A + c + a0 * lda;
          zgemm(s, 0, 1, n - c, jbq, int(c - a0), mone, P, lda, P, lda, one, A + c + c * lda,
                lda, kGeneral, kGeneral, 1, nullptr, 0);
        }
        const int grid = int(std::max<int64_t>(1, std::min<int64_t>(148, ceil_div(restq, kPR))));
        zpotrf_panel_kernel<<<grid, 256, smem, s>>>(A + c + c * lda, lda, jbq, c, restq, d_info,
                                                    loaded);
        BSE_LAUNCH_CHECK();
        if (restq <= 0) done = true;
      }
      const int64_t r0 = a0 + int64_t(G) * kNB;  // first row / column after the group
      if (done || r0 >= n) break;
      BSE_CUDA(cudaEventRecord(ev[0], s));
      const int kk = G * kNB;
      const z_t* P = A + r0 + a0 * lda;  // rows >= r0 of the group's block columns
      const int64_t rest = n - r0;
      const int64_t w1 = min64(kNB, rest), w2 = min64(int64_t(G - 1) * kNB, rest - w1);
      const int64_t n3 = rest - w1 - w2;
      if (pend) BSE_CUDA(cudaStreamWaitEvent(s, ev[2], 0));
      zgemm(s, 0, 1, rest, w1, kk, mone, P, lda, P, lda, one, A + r0 + r0 * lda, lda, kGeneral,
            kGeneral, 1, nullptr, 0);
      pend = false;
      if (w2 > 0) {
        BSE_CUDA(cudaStreamWaitEvent(s2, ev[0], 0));
        const int64_t c2 = r0 + w1;
        zgemm(s2, 0, 1, rest - w1, w2, kk, mone, P + w1, lda, P + w1, lda, one,
              A + c2 + c2 * lda, lda, kGeneral, kGeneral, 1, nullptr, 0);
        BSE_CUDA(cudaEventRecord(ev[1], s2));
        if (n3 > 0) {
          const int64_t c3 = c2 + w2;
          zgemm(s2, 0, 1, n3, n3, kk, mone, P + w1 + w2, lda, P + w1 + w2, lda, one,
                A + c3 + c3 * lda, lda, kGeneral, kGeneral, 1, nullptr, 0);
        }
        BSE_CUDA(cudaEventRecord(ev[2], s2));
        pend = true;
      }
    }
    if (pend) BSE_CUDA(cudaStreamWaitEvent(s, ev[2], 0));
    if (zero_upper && n > 1) {
      const int blocks = int(min64(ceil_div(n * n, 256), 148 * 32));
      zero_strict_upper_kernel<<<blocks, 256, 0, s>>>(n, A, lda);
      BSE_LAUNCH_CHECK();
    }
    return;
  }
  bool big_pending = false;
  for (int64_t j = 0; j < n; j += kNB) {
    const int jb = int(min64(kNB, n - j));
    z_t* Ajj = A + j + j * lda;
    const int64_t rest = n - j - jb;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(148, ceil_div(rest, kPR))));
    zpotrf_panel_kernel<<<grid, 256, smem, s>>>(Ajj, lda, jb, j, rest, d_info, loaded);
    BSE_LAUNCH_CHECK();
    if (rest <= 0) break;
    z_t* A21 = A + (j + jb) + j * lda;
    z_t* A22 = A + (j + jb) + (j + jb) * lda;
    if (!la) {
      // HERK update A22 <- A22 - A21 A21^H (lower tiles only)
      zgemm(s, 0, 1, rest, rest, jb, mone, A21, lda, A21, lda, one, A22, lda, kGeneral, kGeneral,
            1, nullptr, 0);
      continue;
    }
    const int64_t jb2 = min64(kNB, rest), n2 = rest - jb2;
    BSE_CUDA(cudaEventRecord(ev[0], s));
    // next block column (rows >= j+jb): ordered after the s2 update of step j-1, which
    // wrote the same columns
    if (big_pending) BSE_CUDA(cudaStreamWaitEvent(s, ev[1], 0));
    zgemm(s, 0, 1, rest, jb2, jb, mone, A21, lda, A21, lda, one, A22, lda, kGeneral, kGeneral, 1,
          nullptr, 0);
    if (n2 > 0) {
      BSE_CUDA(cudaStreamWaitEvent(s2, ev[0], 0));
      zgemm(s2, 0, 1, n2, n2, jb, mone, A21 + jb2, lda, A21 + jb2, lda, one,
            A22 + jb2 + jb2 * lda, lda, kGeneral, kGeneral, 1, nullptr, 0);
      BSE_CUDA(cudaEventRecord(ev[1], s2));
      big_pending = true;
    }
  }
  if (la && big_pending) BSE_CUDA(cudaStreamWaitEvent(s, ev[1], 0));
  if (zero_upper && n > 1) {
    const int blocks = int(min64(ceil_div(n * n, 256), 148 * 32));
    zero_strict_upper_kernel<<<blocks, 256, 0, s>>>(n, A, lda);
    BSE_LAUNCH_CHECK();
  }
}

}  // namespace bseg
