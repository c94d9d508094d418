// blas.cu — launchers for the DMMA GEMM engine plus the GEMM-based triangular kernels
// (TRSM by recursive splitting over inverted nb x nb diagonal blocks).
//
// Replaces cblas_ztrsm (backend.cpp:124-127), cblas_ztrmm (backend.cpp:151-155, 161-165)
// and cblas_zgemm (backend.cpp:170-173).
#include "blas.h"

#include <cstdio>
#include <cstdlib>

#include <cudaTypedefs.h>

#include "tile_ring.cuh"
#include "gemm.cuh"

namespace bseg {

thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelTimer* g_timer = nullptr;
thread_local int g_panel_ctas = 0;
int panel_cta_cap() {
  static const int solo = getenv("BSE_SOLO_PANEL_CTAS") ? atoi(getenv("BSE_SOLO_PANEL_CTAS")) : 0;
  return g_panel_ctas > 0 ? g_panel_ctas : solo;
}

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 8, kWM = 32, kWN = 32, kST = 4;

template <bool CA, bool CB>
void launch_z(cudaStream_t s, const ZGemmParams& p, dim3 grid) {
  using T = ZGemmTile<kBM, kBN, kBK, kWM, kWN, kST, CA, CB>;
  auto kern = zgemm_dmma_kernel<kBM, kBN, kBK, kWM, kWN, kST, CA, CB>;
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(T::SMEM)));
    return true;
  });
  (void)configured;
  kern<<<grid, T::NTHREADS, T::SMEM, s>>>(p);
  BSE_LAUNCH_CHECK();
}

// Short-K variant (k <= 128: the panel trailing updates, HERK steps, back-transform
// applications): 8 warps of 32x16 per 64x64 tile (half the accumulators per thread), so
// twice the warps per SM hide each tile's prologue and C round trips.
constexpr int kSTs = 4, kMinBs = 2, kWNs = 16;  // 8 warps of 32x16 per 64x64 tile

template <bool CA, bool CB>
void launch_z_short(cudaStream_t s, const ZGemmParams& p, dim3 grid) {
  using T = ZGemmTile<kBM, kBN, kBK, kWM, kWNs, kSTs, CA, CB>;
  auto kern = zgemm_dmma_kernel<kBM, kBN, kBK, kWM, kWNs, kSTs, CA, CB, kMinBs>;
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(T::SMEM)));
    return true;
  });
  (void)configured;
  kern<<<grid, T::NTHREADS, T::SMEM, s>>>(p);
  BSE_LAUNCH_CHECK();
}

// Three-multiplication variant (gemm.cuh M3): the third accumulator set costs registers, so
// the tile shrinks to 64x32 with 4 warps of 32x16 and 3 CTAs per SM.
template <int BN, int BK, int ST, int MINB, bool CA, bool CB>
void launch_z_3m_cfg(cudaStream_t s, const ZGemmParams& p, dim3 grid) {
  using T = ZGemmTile<kBM, BN, BK, kWM, kWNs, ST, CA, CB>;
  auto kern = zgemm_dmma_kernel<kBM, BN, BK, kWM, kWNs, ST, CA, CB, MINB, true>;
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(T::SMEM)));
    return true;
  });
  (void)configured;
  kern<<<grid, T::NTHREADS, T::SMEM, s>>>(p);
  BSE_LAUNCH_CHECK();
}

// 0: four-multiplication kernels only; 3 (default): the 3M 64x32 kernel for every complex
// product; 5: 3M only for k > 128 (A/B switch BSE_GEMM_3M)
int g3m_mode() {
  static const int m = getenv("BSE_GEMM_3M") ? atoi(getenv("BSE_GEMM_3M")) : 3;
  return m;
}

template <bool CA, bool CB>
void launch_z_3m(cudaStream_t s, const ZGemmParams& p, dim3 grid) {
  // 64x32 tiles, 4 warps of 32x16, 3 CTAs per SM (measured 40-41 TFLOP/s complex-equivalent
  // on 4096^3 against 33-35 for the four-multiplication 64x64 kernel)
  const dim3 g2(grid.x, unsigned(ceil_div(p.n, 32)), grid.z);
  launch_z_3m_cfg<32, 8, 4, 3, CA, CB>(s, p, g2);  // 3 or 4 stages measure alike; 6+ lose
}

void launch_z_any(cudaStream_t s, int opa, int opb, const ZGemmParams& p, dim3 grid) {
  static const bool no_short = getenv("BSE_GEMM_NO_SHORT") != nullptr;  // A/B switch
  if (g3m_mode() == 3 || (g3m_mode() && p.k > 128)) {
    if (!opa && !opb) launch_z_3m<false, false>(s, p, grid);
    else if (!opa && opb) launch_z_3m<false, true>(s, p, grid);
    else if (opa && !opb) launch_z_3m<true, false>(s, p, grid);
    else launch_z_3m<true, true>(s, p, grid);
    return;
  }
  if (p.k <= 128 && p.ksplit == 1 && !no_short) {
    if (!opa && !opb) launch_z_short<false, false>(s, p, grid);
    else if (!opa && opb) launch_z_short<false, true>(s, p, grid);
    else if (opa && !opb) launch_z_short<true, false>(s, p, grid);
    else launch_z_short<true, true>(s, p, grid);
    return;
  }
  if (!opa && !opb) launch_z<false, false>(s, p, grid);
  else if (!opa && opb) launch_z<false, true>(s, p, grid);
  else if (opa && !opb) launch_z<true, false>(s, p, grid);
  else launch_z<true, true>(s, p, grid);
}

}  // namespace

__global__ void zgemm_splitk_reduce(int64_t m, int64_t n, int ksplit, const z_t* __restrict__ P,
                                    z_t* C, int64_t ldc, z_t alpha, z_t beta, int c_lower) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    if (c_lower && i < j) continue;
    z_t acc = P[e];
    for (int sidx = 1; sidx < ksplit; ++sidx) acc = zadd(acc, P[int64_t(sidx) * total + e]);
    z_t out = zmul(alpha, acc);
    if (beta.x != 0.0 || beta.y != 0.0) out = zadd(out, zmul(beta, C[i + j * ldc]));
    C[i + j * ldc] = out;
  }
}

namespace {
// Executed real flops of one zgemm call (8 per complex MAC) with triangular K skipping and
// skipped upper tiles, counted per 64x64 tile exactly as the kernel bounds its K loop.
double zgemm_exec_flops(int64_t m, int64_t n, int64_t k, int a_shape, int b_shape, int c_lower) {
  double f = 0.0;
  for (int64_t m0 = 0; m0 < m; m0 += kBM)
    for (int64_t n0 = 0; n0 < n; n0 += kBN) {
      if (c_lower && m0 + kBM <= n0) continue;
      int64_t lo = 0, hi = k;
      if (a_shape == kLowerOp) hi = min64(hi, m0 + kBM);
      if (a_shape == kUpperOp) lo = max64(lo, m0);
      if (b_shape == kLowerOp) lo = max64(lo, n0);
      if (b_shape == kUpperOp) hi = min64(hi, n0 + kBN);
      if (hi > lo) f += 8.0 * double(min64(kBM, m - m0)) * double(min64(kBN, n - n0)) * double(hi - lo);
    }
  return f;
}
}  // namespace

void zgemm(cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, z_t alpha,
           const z_t* A, int64_t lda, const z_t* B, int64_t ldb, z_t beta, z_t* C, int64_t ldc,
           int a_shape, int b_shape, int c_lower, z_t* ws, int64_t ws_elems) {
  if (m <= 0 || n <= 0) return;
  // the 3M kernel runs 64x32 tiles, 3 resident CTAs per SM; the 4M kernels 64x64, 2 per SM
  const bool m3 = g3m_mode() == 3 || (g3m_mode() && k > 128);
  int slot = -1;
  if (g_timer) {  // complex-equivalent flops, and the DMMA flops: 3 real MACs per complex MAC in 3M
    const double f = zgemm_exec_flops(m, n, k, a_shape, b_shape, c_lower);
    slot = timer_begin(s, 0, f, m3 ? 0.75 * f : f);
  }
  struct End {
    cudaStream_t s;
    int slot;
    ~End() { timer_end(s, slot); }
  } end_guard{s, slot};
  ZGemmParams p{};
  p.m = m; p.n = n; p.k = k;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  p.a_shape = a_shape; p.b_shape = b_shape; p.c_lower = c_lower;
  p.ksplit = 1;
  const int64_t tiles_m = ceil_div(m, kBM), tiles_n = ceil_div(n, m3 ? 32 : kBN);
  int ksplit = 1;
  // Under-filled grid with a long K: split K across CTAs (deterministic two-pass reduce).
  // The split maximises the occupancy of the last wave, with a 1% per-slice penalty for the
  // extra reduction traffic, and keeps >= 16 k-tiles per slice.
  const int64_t tiles = tiles_m * tiles_n, slots = (m3 ? 3 : 2) * 148;
  if (ws && tiles < slots && k >= 8 * kBK * 4) {
    double best = double(tiles) / double(slots);
    for (int ks = 2; ks <= 32 && int64_t(ks) * kBK * 16 <= k; ++ks) {
      if (int64_t(ks) * m * n > ws_elems) break;
      const int64_t ctas = tiles * ks;
      const double eff = double(ctas) / double(ceil_div(ctas, slots) * slots) * (1.0 - 0.01 * ks);
      if (eff > best + 1e-9) {
        best = eff;
        ksplit = ks;
      }
    }
  }
  static const bool log = getenv("BSE_GEMM_LOG") != nullptr;  // developer shape log
  if (log)
    fprintf(stderr, "zgemm %lld %lld %lld op%d%d sh%d%d cl%d ks%d gflop %.3f\n", (long long)m,
            (long long)n, (long long)k, opa, opb, a_shape, b_shape, c_lower, ksplit,
            1e-9 * zgemm_exec_flops(m, n, k, a_shape, b_shape, c_lower));
  if (ksplit > 1) {
    p.ksplit = ksplit;
    p.P = ws;
    launch_z_any(s, opa, opb, p, dim3(unsigned(tiles_m), unsigned(tiles_n), unsigned(ksplit)));
    const int64_t total = m * n;
    const int threads = 256;
    const int blocks = int(min64(ceil_div(total, threads), 148 * 16));
    zgemm_splitk_reduce<<<blocks, threads, 0, s>>>(m, n, ksplit, ws, C, ldc, alpha, beta,
                                                   c_lower);
    BSE_LAUNCH_CHECK();
    return;
  }
  launch_z_any(s, opa, opb, p, dim3(unsigned(tiles_m), unsigned(tiles_n), 1));
}

void zgemm_batched(cudaStream_t s, int opa, int opb, int64_t m, int64_t n, int64_t k, z_t alpha,
                   const z_t* A, int64_t lda, int64_t sA, const z_t* B, int64_t ldb, int64_t sB,
                   z_t beta, z_t* C, int64_t ldc, int64_t sC, int batch) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  ZGemmParams p{};
  p.m = m; p.n = n; p.k = k;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  p.sA = sA; p.sB = sB; p.sC = sC;
  p.ksplit = 1;
  if (getenv("BSE_GEMM_LOG"))
    fprintf(stderr, "zgemm %lld %lld %lld op%d%d batch%d gflop %.3f\n", (long long)m, (long long)n,
            (long long)k, opa, opb, batch, 8e-9 * double(m) * double(n) * double(k) * batch);
  launch_z_any(s, opa, opb, p,
               dim3(unsigned(ceil_div(m, kBM)), unsigned(ceil_div(n, kBN)), unsigned(batch)));
}

void dgemm_nn(cudaStream_t s, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
              int batch, int64_t sA, int64_t sB, int64_t sC) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  constexpr int BM = 64, BN = 64, BK = 16, WM = 32, WN = 32, ST = 3;
  using T = DGemmTile<BM, BN, BK, WM, WN, ST>;
  auto kern = dgemm_dmma_kernel<BM, BN, BK, WM, WN, ST>;
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(T::SMEM)));
    return true;
  });
  (void)configured;
  DGemmParams p{};
  p.m = m; p.n = n; p.k = k;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  p.sA = sA; p.sB = sB; p.sC = sC;
  kern<<<dim3(unsigned(ceil_div(m, BM)), unsigned(ceil_div(n, BN)), unsigned(batch)),
         T::NTHREADS, T::SMEM, s>>>(p);
  BSE_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------------
// Inverse of each nb x nb diagonal block of a lower-triangular L (one CTA per block,
// 4 threads per column doing strided partial dot products). Out: blocks stored
// consecutively, each nb x nb (ld nb), strict upper zeroed.
__global__ void __launch_bounds__(256) ztrtri_diag_kernel(int64_t n, const z_t* __restrict__ L,
                                                          int64_t ldl, int nb, z_t* inv) {
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* Ls = reinterpret_cast<z_t*>(sm);      // nb x (nb+1), column-major
  z_t* Xs = Ls + nb * (nb + 1);             // nb x (nb+1): Xs[i*(nb+1)+j] = X(i,j)
  const int64_t b0 = int64_t(blockIdx.x) * nb;
  const int jb = int(min64(nb, n - b0));
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    z_t v = make_double2(0.0, 0.0);
    if (i < jb && j < jb && i >= j) v = L[(b0 + i) + (b0 + j) * ldl];
    Ls[i + j * (nb + 1)] = v;
    Xs[i * (nb + 1) + j] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int col = threadIdx.x >> 2, q = threadIdx.x & 3;
  // Solve L x = e_col by forward substitution; 4 lanes share each column.
  for (int i = 0; i < jb; ++i) {
    z_t part = make_double2(0.0, 0.0);
    if (col < jb && i > col) {
      for (int kk = col + q; kk < i; kk += 4) zfma(part, Ls[i + kk * (nb + 1)], Xs[kk * (nb + 1) + col]);
    }
    warp_converge();
    part.x += __shfl_xor_sync(0xffffffffu, part.x, 1);
    part.y += __shfl_xor_sync(0xffffffffu, part.y, 1);
    part.x += __shfl_xor_sync(0xffffffffu, part.x, 2);
    part.y += __shfl_xor_sync(0xffffffffu, part.y, 2);
    if (col < jb && q == 0 && i >= col) {
      const z_t lii = Ls[i + i * (nb + 1)];
      const z_t rhs = (i == col) ? make_double2(1.0, 0.0) : make_double2(-part.x, -part.y);
      // x_i = rhs / l_ii  (complex division; l_ii is real-positive for Cholesky factors)
      const double den = lii.x * lii.x + lii.y * lii.y;
      Xs[i * (nb + 1) + col] =
          make_double2((rhs.x * lii.x + rhs.y * lii.y) / den, (rhs.y * lii.x - rhs.x * lii.y) / den);
    }
    __syncthreads();
  }
  z_t* out = inv + int64_t(blockIdx.x) * nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    out[i + int64_t(j) * nb] = Xs[i * (nb + 1) + j];
  }
}

void ztrtri_diag_blocks(cudaStream_t s, int64_t n, const z_t* L, int64_t ldl, int nb, z_t* inv) {
  const int64_t nblk = ceil_div(n, nb);
  const size_t smem = size_t(2) * nb * (nb + 1) * sizeof(z_t);
  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(ztrtri_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    return true;
  });
  (void)configured;
  ztrtri_diag_kernel<<<unsigned(nblk), 256, smem, s>>>(n, L, ldl, nb, inv);
  BSE_LAUNCH_CHECK();
}

__global__ void zcopy2d_kernel(int64_t rows, int64_t cols, const z_t* __restrict__ src,
                               int64_t lds, z_t* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

__global__ void __launch_bounds__(256) zcopy_d2h_stream_kernel(int64_t rows, int64_t cols,
                                                                const z_t* __restrict__ src,
                                                                int64_t lds, z_t* dst,
                                                                int64_t ldd) {
  constexpr int U = 4;  // loads in flight per thread
  const int64_t total = rows * cols;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e0 < total; e0 += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < total) {
        const double2* p = src + (e % rows) + (e / rows) * lds;
        asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];"  // streaming: evict-first in L2
                     : "=d"(v[u].x), "=d"(v[u].y)
                     : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < total) {
        double2* q = dst + (e % rows) + (e / rows) * ldd;
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(q), "d"(v[u].x), "d"(v[u].y)
                     : "memory");
      }
    }
  }
}

bool zcopy2d_to_host_streaming(cudaStream_t s, int64_t rows, int64_t cols, const z_t* src,
                               int64_t lds, z_t* dst_host, int64_t ldd) {
  // 8 CTAs keep the lanes' downloads ahead of the next item (measured e2e 42.1-42.5 TFLOP/s
  // with 8 or 16 CTAs against 39.5-40.8 through the copy engine); BSE_D2H_CTAS=0: copy engine
  static const int ctas = getenv("BSE_D2H_CTAS") ? atoi(getenv("BSE_D2H_CTAS")) : 8;
  if (ctas <= 0 || rows <= 0 || cols <= 0) return false;
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, dst_host, 0) != cudaSuccess || !dptr) {
    (void)cudaGetLastError();
    return false;
  }
  // 16-byte vector accesses: an 8-byte-aligned complex buffer goes to the copy engine
  if ((reinterpret_cast<uintptr_t>(dptr) | reinterpret_cast<uintptr_t>(src)) & 15u) return false;
  zcopy_d2h_stream_kernel<<<ctas, 256, 0, s>>>(rows, cols, src, lds, static_cast<z_t*>(dptr), ldd);
  BSE_LAUNCH_CHECK();
  return true;
}

void zcopy2d(cudaStream_t s, int64_t rows, int64_t cols, const z_t* src, int64_t lds, z_t* dst,
             int64_t ldd) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t total = rows * cols;
  const int blocks = int(min64(ceil_div(total, 256), 148 * 32));
  zcopy2d_kernel<<<blocks, 256, 0, s>>>(rows, cols, src, lds, dst, ldd);
  BSE_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------------
// Recursive TRSM on a lower-triangular L (n x n), in place on X:
//   side L, op N : L   X = B        side L, op C : L^H X = B
//   side R, op N : X L   = B        side R, op C : X L^H = B
// Leaves are nb-blocks solved as out-of-place products with the inverted diagonal block;
// all off-diagonal work is DMMA GEMM on the largest possible panels.
namespace {

struct TrsmCtx {
  cudaStream_t s;
  const z_t* L;
  int64_t ldl;
  const z_t* inv;  // inverted diagonal blocks
  int nb;
  int side, op;
  z_t* tmp;  // leaf scratch: nb x rhs_extent
  z_t* ws;
  int64_t ws_elems;
};

const z_t kOne = {1.0, 0.0}, kZero = {0.0, 0.0}, kMinusOne = {-1.0, 0.0};

// Solve on the diagonal range [r0, r0+len) of L; X points at the full right-hand side.
void trsm_rec(const TrsmCtx& c, int64_t r0, int64_t len, z_t* X, int64_t ldx, int64_t other) {
  if (len <= c.nb) {
    const z_t* Li = c.inv + (r0 / c.nb) * int64_t(c.nb) * c.nb;
    if (c.side == 0) {
      // X[r0:r0+len, :] = op(Linv) * X[r0:r0+len, :]
      zgemm(c.s, c.op, 0, len, other, len, kOne, Li, c.nb, X + r0, ldx, kZero, c.tmp, len,
            c.op ? kUpperOp : kLowerOp, kGeneral, 0, nullptr, 0);
      zcopy2d(c.s, len, other, c.tmp, len, X + r0, ldx);
    } else {
      // X[:, r0:r0+len] = X[:, r0:r0+len] * op(Linv)
      zgemm(c.s, 0, c.op, other, len, len, kOne, X + r0 * ldx, ldx, Li, c.nb, kZero, c.tmp,
            other, kGeneral, c.op ? kUpperOp : kLowerOp, 0, nullptr, 0);
      zcopy2d(c.s, other, len, c.tmp, other, X + r0 * ldx, ldx);
    }
    return;
  }
  const int64_t nblk = ceil_div(len, c.nb);
  const int64_t n1 = ((nblk + 1) / 2) * c.nb;
  const int64_t n2 = len - n1;
  const z_t* L21 = c.L + (r0 + n1) + r0 * c.ldl;  // n2 x n1 block below the first half
  if (c.side == 0 && c.op == 0) {
    trsm_rec(c, r0, n1, X, ldx, other);
    zgemm(c.s, 0, 0, n2, other, n1, kMinusOne, L21, c.ldl, X + r0, ldx, kOne, X + r0 + n1, ldx,
          kGeneral, kGeneral, 0, c.ws, c.ws_elems);
    trsm_rec(c, r0 + n1, n2, X, ldx, other);
  } else if (c.side == 0 && c.op == 1) {
    trsm_rec(c, r0 + n1, n2, X, ldx, other);
    zgemm(c.s, 1, 0, n1, other, n2, kMinusOne, L21, c.ldl, X + r0 + n1, ldx, kOne, X + r0, ldx,
          kGeneral, kGeneral, 0, c.ws, c.ws_elems);
    trsm_rec(c, r0, n1, X, ldx, other);
  } else if (c.side == 1 && c.op == 0) {
    trsm_rec(c, r0 + n1, n2, X, ldx, other);
    zgemm(c.s, 0, 0, other, n1, n2, kMinusOne, X + (r0 + n1) * ldx, ldx, L21, c.ldl, kOne,
          X + r0 * ldx, ldx, kGeneral, kGeneral, 0, c.ws, c.ws_elems);
    trsm_rec(c, r0, n1, X, ldx, other);
  } else {
    trsm_rec(c, r0, n1, X, ldx, other);
    zgemm(c.s, 0, 1, other, n2, n1, kMinusOne, X + r0 * ldx, ldx, L21, c.ldl, kOne,
          X + (r0 + n1) * ldx, ldx, kGeneral, kGeneral, 0, c.ws, c.ws_elems);
    trsm_rec(c, r0 + n1, n2, X, ldx, other);
  }
}

}  // namespace

size_t trsm_workspace_elems(int64_t n, int64_t other, int nb) {
  // inverted blocks + leaf scratch + split-K partials
  return size_t(ceil_div(n, nb)) * nb * nb + size_t(nb) * size_t(other) +
         size_t(8) * size_t(n) * size_t(nb);
}

void ztrsm_lower(cudaStream_t s, int side, int op, int64_t n, int64_t other, const z_t* L,
                 int64_t ldl, z_t* X, int64_t ldx, z_t* ws, int nb) {
  if (n <= 0 || other <= 0) return;
  z_t* inv = ws;
  z_t* tmp = inv + ceil_div(n, nb) * int64_t(nb) * nb;
  z_t* part = tmp + int64_t(nb) * other;
  ztrtri_diag_blocks(s, n, L, ldl, nb, inv);
  TrsmCtx c{s, L, ldl, inv, nb, side, op, tmp, part, 8 * n * int64_t(nb)};
  trsm_rec(c, 0, n, X, ldx, other);
}

CUtensorMap make_tile_map(const z_t* A, int64_t lda, int64_t n) {
  return make_tile_map_box(A, lda, n, kRingT, kRingT);
}

CUtensorMap make_tile_map_box(const z_t* A, int64_t lda, int64_t n, int box_rows, int box_cols) {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    BSE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&f),
                                     cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return f;
  }();
  CUtensorMap map;
  const cuuint64_t dims[2] = {cuuint64_t(2 * n), cuuint64_t(n)};
  const cuuint64_t strides[1] = {cuuint64_t(lda) * sizeof(z_t)};
  const cuuint32_t box[2] = {cuuint32_t(2 * box_rows), cuuint32_t(box_cols)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<z_t*>(A), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
  return map;
}

}  // namespace bseg
