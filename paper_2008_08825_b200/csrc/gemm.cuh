// gemm.cuh — FP64 tensor-core (DMMA.8x8x4) GEMM engine for complex128 and float64.
//
// Every O(n^3) stage of the hot path (Cholesky HERK/TRSM updates, the L^H M1 L and L1^H L2
// triangular products, the her2k trailing updates of the tridiagonal/bidiagonal
// reductions, the Householder back-transforms, the divide-and-conquer merges and the
// eigenvector recovery) funnels into the two kernels below. They replace the reference's
// cblas_ztrmm / cblas_zgemm / cblas_ztrsm call sites (proj/src/backend.cpp:124-173) and the
// BLAS-3 inside LAPACK's zpotrf/zheevd/zgesvd (backend.cpp:34,51,74).
//
// B200 has no FP64 tcgen05 kind (tcgen05.mma kinds are f16/tf32/f8f6f4/i8/mx*), so FP64
// tensor work is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4, measured 37 TFLOP/s peak on
// this pool). Operands are staged global->shared with a multi-stage cp.async ring and read
// into fragments with bank-conflict-free padded layouts (see the stride notes below).
//
// Complex product: 4 real DMMAs per 8x8x4 complex sub-tile on interleaved (re,im) smem
// tiles — one 16-byte LDS per lane yields both parts of a fragment element.
#pragma once

#include "common.cuh"

namespace bseg {

// Shape of op(X) as seen by the product (after the adjoint, if any).
enum OpShape : int { kGeneral = 0, kLowerOp = 1, kUpperOp = 2 };

struct ZGemmParams {
  int64_t m, n, k;
  const z_t* A;
  int64_t lda;
  const z_t* B;
  int64_t ldb;
  z_t* C;
  int64_t ldc;
  z_t alpha, beta;
  int a_shape;  // OpShape of op(A): lower => entries with k > i are zero; upper => k < i zero
  int b_shape;  // OpShape of op(B): lower => entries with k < j zero; upper => k > j zero
  int c_lower;  // write only C(i,j) with i >= j (HERK / HER2K); fully-upper tiles skipped
  int64_t sA, sB, sC;  // batch strides (blockIdx.z) when ksplit == 1
  int ksplit;          // > 1: blockIdx.z is the K-split; partial sums go to P
  z_t* P;              // ksplit slices of m x n (ld = m), raw sums (no alpha/beta)
};

struct DGemmParams {
  int64_t m, n, k;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int64_t sA, sB, sC;
};

// ----------------------------------------------------------------------------------------
// Complex kernel. CONJ_A: op(A) = A^H (A stored k x m); CONJ_B: op(B) = B^H (B stored n x k).
// Shared layouts (complex units), chosen so the 8 lanes of each 16-byte LDS phase hit 8
// distinct 4-bank groups:
//   op(A)=A   : As[kk][i], row stride BM+2   (group = 2kk + i mod 8)
//   op(A)=A^H : As[i][kk], row stride BK+4   (group = 4i + kk mod 8)
//   op(B)=B   : Bs[j][kk], row stride BK+4
//   op(B)=B^H : Bs[kk][j], row stride BN+2
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool CONJ_A, bool CONJ_B>
struct ZGemmTile {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NTHREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int A_LD = CONJ_A ? (BK + 4) : (BM + 2);
  static constexpr int A_ELEMS = CONJ_A ? BM * (BK + 4) : BK * (BM + 2);
  static constexpr int B_LD = CONJ_B ? (BN + 2) : (BK + 4);
  static constexpr int B_ELEMS = CONJ_B ? BK * (BN + 2) : BN * (BK + 4);
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(z_t);
  static_assert(BM % 8 == 0 && BN % 8 == 0 && BK % 4 == 0, "tile");
  static_assert((BM * BK) % NTHREADS == 0 && (BN * BK) % NTHREADS == 0, "loader");
};

// M3: Gauss's three-multiplication form, P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi),
// Re = P1 - P2, Im = P3 - P1 - P2: 3 DMMAs per complex 8x8x4 instead of 4 (normwise error
// bound of the same order, Higham ASNA 23.2.4), at 1.5x the accumulator registers.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool CONJ_A, bool CONJ_B,
          int MINB = 1, bool M3 = false>
__global__ void __launch_bounds__(ZGemmTile<BM, BN, BK, WM, WN, STAGES, CONJ_A, CONJ_B>::NTHREADS,
                                  MINB)
    zgemm_dmma_kernel(ZGemmParams p) {
  using T = ZGemmTile<BM, BN, BK, WM, WN, STAGES, CONJ_A, CONJ_B>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  z_t* smem = reinterpret_cast<z_t*>(smem_raw);

  // Grouped rasterisation: the hardware dispatches CTAs x-fastest, so consecutive CTAs walk
  // down a group of kGroupM tile rows before moving to the next tile column. The CTAs in
  // flight then share A row panels and B column panels in L2 (instead of every resident
  // tile column re-streaming all of A from HBM).
  constexpr int kGroupM = 16;
  int bm = blockIdx.x, bn = blockIdx.y;
  {
    const int tm = gridDim.x, tn = gridDim.y;
    const int lin = blockIdx.y * tm + blockIdx.x;
    const int per_group = kGroupM * tn;
    const int first = (lin / per_group) * kGroupM;
    const int gsz = min(tm - first, kGroupM);
    const int r = lin % per_group;
    bm = first + r % gsz;
    bn = r / gsz;
  }
  const int64_t m0 = int64_t(bm) * BM;
  const int64_t n0 = int64_t(bn) * BN;
  if (p.c_lower && m0 + BM <= n0) return;  // tile strictly above the diagonal

  const z_t* A = p.A;
  const z_t* B = p.B;
  z_t* C = p.C;
  int split = 0;
  if (p.ksplit > 1) {
    split = blockIdx.z;
  } else {
    A += int64_t(blockIdx.z) * p.sA;
    B += int64_t(blockIdx.z) * p.sB;
    C += int64_t(blockIdx.z) * p.sC;
  }

  // K range with triangular skipping.
  int64_t k_lo = 0, k_hi = p.k;
  if (p.a_shape == kLowerOp) k_hi = min(k_hi, m0 + BM);
  if (p.a_shape == kUpperOp) k_lo = max(k_lo, m0);
  if (p.b_shape == kLowerOp) k_lo = max(k_lo, n0);
  if (p.b_shape == kUpperOp) k_hi = min(k_hi, n0 + BN);
  k_lo = (k_lo / BK) * BK;
  if (p.ksplit > 1) {
    const int64_t nkt = ceil_div(max64(k_hi - k_lo, 0), BK);
    const int64_t per = ceil_div(nkt, p.ksplit);
    const int64_t a = k_lo + int64_t(split) * per * BK;
    const int64_t b = min(k_hi, a + per * BK);
    k_lo = a;
    k_hi = b;
  }
  const int64_t ktiles = k_hi > k_lo ? ceil_div(k_hi - k_lo, BK) : 0;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / T::WARPS_N) * WM;
  const int wn0 = (warp % T::WARPS_N) * WN;

  auto load_stage = [&](int stage, int64_t kt) {
    z_t* As = smem + stage * T::STAGE_ELEMS;
    z_t* Bs = As + T::A_ELEMS;
    const int64_t k0 = k_lo + kt * BK;
#pragma unroll
    for (int r = 0; r < (BM * BK) / T::NTHREADS; ++r) {
      const int e = tid + r * T::NTHREADS;
      int i, kk;
      if (!CONJ_A) { i = e % BM; kk = e / BM; } else { kk = e % BK; i = e / BK; }
      const int64_t gi = m0 + i, gk = k0 + kk;
      bool ok = gi < p.m && gk < k_hi;
      if (p.a_shape == kLowerOp) ok = ok && gk <= gi;
      if (p.a_shape == kUpperOp) ok = ok && gk >= gi;
      const z_t* src = CONJ_A ? (A + gk + gi * p.lda) : (A + gi + gk * p.lda);
      z_t* dst = CONJ_A ? (As + i * T::A_LD + kk) : (As + kk * T::A_LD + i);
      cp_async16(dst, ok ? src : A, ok);
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / T::NTHREADS; ++r) {
      const int e = tid + r * T::NTHREADS;
      int j, kk;
      if (!CONJ_B) { kk = e % BK; j = e / BK; } else { j = e % BN; kk = e / BN; }
      const int64_t gj = n0 + j, gk = k0 + kk;
      bool ok = gj < p.n && gk < k_hi;
      if (p.b_shape == kLowerOp) ok = ok && gk >= gj;
      if (p.b_shape == kUpperOp) ok = ok && gk <= gj;
      const z_t* src = CONJ_B ? (B + gj + gk * p.ldb) : (B + gk + gj * p.ldb);
      z_t* dst = CONJ_B ? (Bs + kk * T::B_LD + j) : (Bs + j * T::B_LD + kk);
      cp_async16(dst, ok ? src : B, ok);
    }
  };

  // 4M: acc_re / acc_im. M3: acc_re = P1, acc_im = P3, acc_p2 = P2.
  double acc_re[T::MT][T::NT][2], acc_im[T::MT][T::NT][2];
  double acc_p2[M3 ? T::MT : 1][M3 ? T::NT : 1][2];
#pragma unroll
  for (int a = 0; a < T::MT; ++a)
#pragma unroll
    for (int b = 0; b < T::NT; ++b) {
      acc_re[a][b][0] = acc_re[a][b][1] = 0.0;
      acc_im[a][b][0] = acc_im[a][b][1] = 0.0;
      if constexpr (M3) acc_p2[a][b][0] = acc_p2[a][b][1] = 0.0;
    }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(int(nk % STAGES), nk);
      cp_async_commit();
    }
    const z_t* As = smem + int(kt % STAGES) * T::STAGE_ELEMS;
    const z_t* Bs = As + T::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double ar[T::MT], ai[T::MT], nai[T::MT], br[T::NT], bi[T::NT];
#pragma unroll
      for (int a = 0; a < T::MT; ++a) {
        const int i = wm0 + a * 8 + fr, kk = ks + fk;
        const z_t v = CONJ_A ? As[i * T::A_LD + kk] : As[kk * T::A_LD + i];
        ar[a] = v.x;
        ai[a] = CONJ_A ? -v.y : v.y;
        nai[a] = -ai[a];
      }
#pragma unroll
      for (int b = 0; b < T::NT; ++b) {
        const int j = wn0 + b * 8 + fr, kk = ks + fk;
        const z_t v = CONJ_B ? Bs[kk * T::B_LD + j] : Bs[j * T::B_LD + kk];
        br[b] = v.x;
        bi[b] = CONJ_B ? -v.y : v.y;
      }
      if constexpr (M3) {
        double sa[T::MT], sb[T::NT];
#pragma unroll
        for (int a = 0; a < T::MT; ++a) sa[a] = ar[a] + ai[a];
#pragma unroll
        for (int b = 0; b < T::NT; ++b) sb[b] = br[b] + bi[b];
#pragma unroll
        for (int a = 0; a < T::MT; ++a)
#pragma unroll
          for (int b = 0; b < T::NT; ++b) {
            dmma884(acc_re[a][b][0], acc_re[a][b][1], ar[a], br[b]);
            dmma884(acc_p2[a][b][0], acc_p2[a][b][1], ai[a], bi[b]);
            dmma884(acc_im[a][b][0], acc_im[a][b][1], sa[a], sb[b]);
          }
      } else {
#pragma unroll
        for (int a = 0; a < T::MT; ++a)
#pragma unroll
          for (int b = 0; b < T::NT; ++b) {
            dmma884(acc_re[a][b][0], acc_re[a][b][1], ar[a], br[b]);
            dmma884(acc_re[a][b][0], acc_re[a][b][1], nai[a], bi[b]);
            dmma884(acc_im[a][b][0], acc_im[a][b][1], ar[a], bi[b]);
            dmma884(acc_im[a][b][0], acc_im[a][b][1], ai[a], br[b]);
          }
      }
    }
  }
  cp_async_wait<0>();
  if constexpr (M3) {
#pragma unroll
    for (int a = 0; a < T::MT; ++a)
#pragma unroll
      for (int b = 0; b < T::NT; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double p1 = acc_re[a][b][h], p2 = acc_p2[a][b][h];
          acc_re[a][b][h] = p1 - p2;
          acc_im[a][b][h] = acc_im[a][b][h] - p1 - p2;
        }
  }

  // Epilogue. The C reads of a row pair are issued before any store (stores to C could alias
  // later reads, so the compiler cannot hoist loads over them): 2 memory round trips per tile
  // instead of one per element, which dominates short-K products (k = 64 trailing updates).
  const bool use_beta = p.ksplit == 1 && (p.beta.x != 0.0 || p.beta.y != 0.0);
  constexpr int ER = 2;  // fragment rows per C read round
#pragma unroll
  for (int a0 = 0; a0 < T::MT; a0 += ER) {
    z_t cv[ER][T::NT][2];
#pragma unroll
    for (int da = 0; da < ER; ++da)
#pragma unroll
      for (int b = 0; b < T::NT; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t gi = m0 + wm0 + (a0 + da) * 8 + fr;
          const int64_t gj = n0 + wn0 + b * 8 + 2 * fk + h;
          const bool live = use_beta && gi < p.m && gj < p.n && !(p.c_lower && gi < gj);
          cv[da][b][h] = live ? C[gi + gj * p.ldc] : make_double2(0.0, 0.0);
        }
#pragma unroll
    for (int da = 0; da < ER; ++da)
#pragma unroll
      for (int b = 0; b < T::NT; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = a0 + da;
          const int64_t gi = m0 + wm0 + a * 8 + fr;
          const int64_t gj = n0 + wn0 + b * 8 + 2 * fk + h;
          if (gi >= p.m || gj >= p.n) continue;
          const z_t acc = make_double2(acc_re[a][b][h], acc_im[a][b][h]);
          if (p.ksplit > 1) {
            p.P[int64_t(split) * p.m * p.n + gi + gj * p.m] = acc;
            continue;
          }
          if (p.c_lower && gi < gj) continue;
          z_t out = zmul(p.alpha, acc);
          if (use_beta) out = zadd(out, zmul(p.beta, cv[da][b][h]));
          C[gi + gj * p.ldc] = out;
        }
  }
}

// Reduces K-split partials: C = alpha * sum_s P_s + beta * C.
__global__ void zgemm_splitk_reduce(int64_t m, int64_t n, int ksplit, const z_t* __restrict__ P,
                                    z_t* C, int64_t ldc, z_t alpha, z_t beta, int c_lower);

// ----------------------------------------------------------------------------------------
// Real kernel (op N, N): the divide-and-conquer eigenvector merges Q_new = Q * U.
//   As[kk][i] row stride BM+4 ; Bs[j][kk] row stride BK+4 (8-byte LDS phases of 16 lanes).
template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct DGemmTile {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int NTHREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int A_LD = BM + 4, B_LD = BK + 4;
  static constexpr int A_ELEMS = BK * A_LD, B_ELEMS = BN * B_LD;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(DGemmTile<BM, BN, BK, WM, WN, STAGES>::NTHREADS)
    dgemm_dmma_kernel(DGemmParams p) {
  using T = DGemmTile<BM, BN, BK, WM, WN, STAGES>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int64_t n0 = int64_t(blockIdx.y) * BN;
  const double* A = p.A + int64_t(blockIdx.z) * p.sA;
  const double* B = p.B + int64_t(blockIdx.z) * p.sB;
  double* C = p.C + int64_t(blockIdx.z) * p.sC;
  const int64_t ktiles = ceil_div(p.k, BK);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / T::WARPS_N) * WM;
  const int wn0 = (warp % T::WARPS_N) * WN;

  auto load_stage = [&](int stage, int64_t kt) {
    double* As = smem + stage * T::STAGE_ELEMS;
    double* Bs = As + T::A_ELEMS;
    const int64_t k0 = kt * BK;
#pragma unroll
    for (int r = 0; r < (BM * BK) / T::NTHREADS; ++r) {
      const int e = tid + r * T::NTHREADS;
      const int i = e % BM, kk = e / BM;
      const int64_t gi = m0 + i, gk = k0 + kk;
      const bool ok = gi < p.m && gk < p.k;
      cp_async8(As + kk * T::A_LD + i, ok ? A + gi + gk * p.lda : A, ok);
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / T::NTHREADS; ++r) {
      const int e = tid + r * T::NTHREADS;
      const int kk = e % BK, j = e / BK;
      const int64_t gj = n0 + j, gk = k0 + kk;
      const bool ok = gj < p.n && gk < p.k;
      cp_async8(Bs + j * T::B_LD + kk, ok ? B + gk + gj * p.ldb : B, ok);
    }
  };

  double acc[T::MT][T::NT][2];
#pragma unroll
  for (int a = 0; a < T::MT; ++a)
#pragma unroll
    for (int b = 0; b < T::NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(int(nk % STAGES), nk);
      cp_async_commit();
    }
    const double* As = smem + int(kt % STAGES) * T::STAGE_ELEMS;
    const double* Bs = As + T::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double av[T::MT], bv[T::NT];
#pragma unroll
      for (int a = 0; a < T::MT; ++a) av[a] = As[(ks + fk) * T::A_LD + wm0 + a * 8 + fr];
#pragma unroll
      for (int b = 0; b < T::NT; ++b) bv[b] = Bs[(wn0 + b * 8 + fr) * T::B_LD + ks + fk];
#pragma unroll
      for (int a = 0; a < T::MT; ++a)
#pragma unroll
        for (int b = 0; b < T::NT; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < T::MT; ++a)
#pragma unroll
    for (int b = 0; b < T::NT; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = m0 + wm0 + a * 8 + fr;
        const int64_t gj = n0 + wn0 + b * 8 + 2 * fk + h;
        if (gi >= p.m || gj >= p.n) continue;
        double out = p.alpha * acc[a][b][h];
        if (p.beta != 0.0) out += p.beta * C[gi + gj * p.ldc];
        C[gi + gj * p.ldc] = out;
      }
}

// Host launchers: see blas.h.

}  // namespace bseg
