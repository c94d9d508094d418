// hetrd2.cu — two-stage Householder tridiagonalisation of a Hermitian matrix (lower storage)
// and its back-transformation, an alternative to hetrd.cu's one-stage reduction for the
// zheevd('V','L') replacement (proj/src/backend.cpp:34).
//
// The one-stage panels are latency-bound (two grid barriers per column). The two-stage form
// moves the O(n^3) work to DMMA GEMMs and leaves an O(n^2 b) bulge chase:
//
//  stage 1  he2hb  (LAPACK zhetrd_he2hb structure): per panel of b = kBand2 columns, the
//           panel below the band is QR-factored by one cooperative kernel (rows in registers,
//           two grid barriers per column over <= n/256 CTAs) that also forms T and V T; then
//           X = A22 (V T) as two triangular DMMA GEMMs over the lower triangle,
//           W = X - 1/2 V (T^H V^H X), and the her2k A22 -= V W^H + W V^H (lower tiles only).
//  stage 2  hb2st  bulge chasing on a packed band (2b rows per column, L2-resident). Task
//           (s, j) of sweep s: right-apply the previous reflector to the bulge block Bk_j,
//           annihilate its first column, left-apply to the rest of Bk_j, two-sided update of
//           the diagonal block D_j. One warp per sweep, smem-staged 32x32 blocks; sweep s runs
//           task j once sweep s-1 has finished task j+1 (progress counters, acquire/release).
//  back     Z <- Q1 Q2 Z. Q2: the chase reflectors in groups of 32 sweeps x one task index,
//           groups ordered (sweep block descending, task ascending), each thread keeping a
//           64-row window of one column in registers and streaming down the column; Q1: the
//           stage-1 reflectors through apply_reflectors (mode 3, compact WY on DMMA).
//
// The bookkeeping (task extents, schedule rule, group order) is modelled in numpy by
// tools/two_stage_model.py. Every sum has a fixed order: results are bit-deterministic.
#include <cooperative_groups.h>

#include <atomic>
#include <cstdlib>
#include <cstring>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "ops.h"

namespace bseg {

namespace {
constexpr int kB = kBand2;       // band width
constexpr int kQrT = 256;        // panel rows per QR CTA (one row per thread)
constexpr int kLdab = 2 * kB;    // packed band: offsets 0 .. 2b-1 below the diagonal
constexpr int kChW = 4;          // chase warps per CTA
constexpr int kBp = kB + 1;      // padded smem block stride
constexpr int kQ2Rows = 64;      // back-transform window rows (b + 32 - 1, padded)
constexpr int kQ2Res = 8;        // row residues per column (lanes per column)
constexpr int kQ2Reg = kQ2Rows / kQ2Res;  // window rows per thread
constexpr int kQ2Warps = 4;      // warps per back-transform CTA (4 columns each)

__device__ __forceinline__ z_t zdiv1(z_t a) {
  const double den = a.x * a.x + a.y * a.y;
  return make_double2(a.x / den, -a.y / den);
}

// zlarfg on (alpha, ||x||^2): beta (real), tau, scale = 1 / (alpha - beta) (1 if tau == 0).
__device__ __forceinline__ void larfg2(z_t alpha, double xnorm2, double& beta, z_t& tau,
                                       z_t& scale) {
  if (xnorm2 == 0.0 && alpha.y == 0.0) {
    beta = alpha.x;
    tau = make_double2(0.0, 0.0);
    scale = make_double2(1.0, 0.0);
    return;
  }
  const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2);
  beta = alpha.x >= 0.0 ? -nrm : nrm;
  tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
  scale = zdiv1(make_double2(alpha.x - beta, alpha.y));
}

__device__ __forceinline__ z_t shfl_z(z_t v, int o) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, o);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, o);
  return v;
}
}  // namespace

// ------------------------------------------------------------------------ stage 1: he2hb
struct QrArgs {
  z_t* P;          // panel (m x kB) inside A
  int64_t ldp, m;
  int k;           // reflectors: min(m, kB)
  z_t* VW;         // V -> VW[:, 0:kB]
  z_t* WV;         //   and WV[:, kB:2kB]
  z_t* VT;         // V T (m x kB)
  int64_t ldw;
  z_t* T;          // kB x kB upper (ld kB)
  z_t* tau;        // kB
  double* normp;   // gridDim.x partial norms
  z_t* alphab;     // alpha of the current column
  z_t* part;       // gridDim.x x kB partial sums
  unsigned* bar;   // grid barrier counter (zeroed)
};

// Householder QR of the m x kB panel (zgeqr2 column order, zlarfg reflectors), V and T
// (zlarft forward/columnwise) and V T. Thread = panel row; the CTA's 256 x kB rows live in
// shared memory (element (r, c) at c * kQrLd + r: a thread walks its row conflict-free).
// Per column: (1) partial norms + alpha -> grid barrier -> (2) reflector (redundantly per
// CTA), v, partial w = v^H P(:, c>j) and g = V(:, i<j)^H v in one kB-slot vector ->
// grid barrier -> (3) totals (fixed order), rank-1 update, T column.
namespace {
constexpr int kQrLd = kQrT + 1;
constexpr size_t kQrSmem = size_t(kB) * kQrLd * sizeof(z_t);
}  // namespace
__global__ void __launch_bounds__(kQrT, 1) he2hb_qr_kernel(const __grid_constant__ QrArgs a) {
  GridBarrier grid(a.bar);
  extern __shared__ __align__(16) unsigned char qsm[];
  z_t* sP = reinterpret_cast<z_t*>(qsm);
  __shared__ z_t Ts[kB * kB];
  __shared__ z_t wred[kQrT / 32][kB];
  __shared__ z_t wsum[kB];
  __shared__ z_t taus[kB];
  __shared__ double dred[kQrT / 32 + 2];
  __shared__ z_t alpha_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int64_t r = int64_t(blockIdx.x) * kQrT + tid;
  const bool valid = r < a.m;
  const z_t zero = make_double2(0.0, 0.0), one = make_double2(1.0, 0.0);
  z_t* pr = sP + tid;  // this thread's row: pr[c * kQrLd]
#pragma unroll 8
  for (int c = 0; c < kB; ++c) pr[c * kQrLd] = valid ? a.P[r + c * a.ldp] : zero;
  for (int e = tid; e < kB * kB; e += kQrT) Ts[e] = zero;
  if (tid < kB) taus[tid] = zero;

  for (int j = 0; j < a.k; ++j) {
    // (1) partial ||P(j+1:, j)||^2 and alpha = P(j, j)
    const z_t pj = pr[j * kQrLd];
    const double bs = block_sum((valid && r > j) ? zabs2(pj) : 0.0, dred);
    if (tid == 0) a.normp[blockIdx.x] = bs;
    if (r == j) *a.alphab = pj;
    grid.sync();
    // (2) reflector
    if (warp == 0) {
      double x = 0.0;
      for (int g = lane; g < G; g += 32) x += a.normp[g];
      x = warp_sum(x);
      if (lane == 0) {
        dred[kQrT / 32] = x;
        alpha_s = *a.alphab;
      }
    }
    __syncthreads();
    double beta;
    z_t tau, scale;
    larfg2(alpha_s, dred[kQrT / 32], beta, tau, scale);
    z_t v = zero;
    if (valid) v = (r == j) ? one : (r > j ? zmul(scale, pj) : zero);
    if (valid && r > j) pr[j * kQrLd] = v;
    if (r == j) pr[j * kQrLd] = make_double2(beta, 0.0);
    // slot c > j: conj(v) P(r, c); slot i < j: conj(V(r, i)) v ; slot j: 0
    z_t sl[16], sh[16];
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      const z_t pc = pr[c * kQrLd];
      const z_t vi = r > c ? pc : (r == c ? one : zero);
      const z_t t = c > j ? zcmul(v, pc) : (c < j ? zcmul(vi, v) : zero);
      if (c < 16) sl[c] = t; else sh[c - 16] = t;
    }
    __syncthreads();  // re-converge before the butterflies
    const z_t tl = warp_transpose_zsum16(sl);  // lane l: slot l >> 1
    const z_t th = warp_transpose_zsum16(sh);  // lane l: slot 16 + (l >> 1)
    if ((lane & 1) == 0) {
      wred[warp][lane >> 1] = tl;
      wred[warp][16 + (lane >> 1)] = th;
    }
    __syncthreads();
    if (tid < kB) {
      z_t t = wred[0][tid];
#pragma unroll
      for (int w = 1; w < kQrT / 32; ++w) t = zadd(t, wred[w][tid]);
      a.part[int64_t(blockIdx.x) * kB + tid] = t;
    }
    grid.sync();
    // (3) totals (warp w sums CTAs w, w+8, ...; then a fixed-order sum over the warps), update,
    // T(:, j)
    {
      z_t t = zero;
      for (int g = warp; g < G; g += kQrT / 32) t = zadd(t, a.part[int64_t(g) * kB + lane]);
      wred[warp][lane] = t;
    }
    __syncthreads();
    if (tid < kB) {
      z_t t = wred[0][tid];
#pragma unroll
      for (int w = 1; w < kQrT / 32; ++w) t = zadd(t, wred[w][tid]);
      wsum[tid] = t;
    }
    __syncthreads();
    const z_t cv = zmul(zconj(tau), v);
    for (int c = j + 1; c < kB; ++c) pr[c * kQrLd] = zsub(pr[c * kQrLd], zmul(cv, wsum[c]));
    if (tid < kB) {
      z_t t = zero;
      if (tid < j) {  // T(i, j) = -tau sum_{i' = i}^{j-1} T(i, i') g(i')
        for (int i2 = tid; i2 < j; ++i2) zfma(t, Ts[tid + i2 * kB], wsum[i2]);
        t = zscale(zmul(tau, t), -1.0);
      } else if (tid == j) {
        t = tau;
        taus[j] = tau;
      }
      if (tid <= j) Ts[tid + j * kB] = t;
    }
  }
  __syncthreads();
  if (valid) {
    z_t vx[kB];
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      const z_t pc = pr[c * kQrLd];
      a.P[r + c * a.ldp] = pc;
      vx[c] = c < a.k ? (r > c ? pc : (r == c ? one : zero)) : zero;
      a.VW[r + c * a.ldw] = vx[c];
      a.WV[r + (kB + c) * a.ldw] = vx[c];
    }
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      z_t t = zero;
#pragma unroll
      for (int i = 0; i <= c; ++i) zfma(t, vx[i], Ts[i + c * kB]);
      a.VT[r + c * a.ldw] = t;
    }
  }
  if (blockIdx.x == 0) {
    for (int e = tid; e < kB * kB; e += kQrT) a.T[e] = Ts[e];
    if (tid < kB) a.tau[tid] = taus[tid];
  }
}

// W = X - 1/2 V (T^H Y), Y = V^H X (kB x kB). Writes W to VW[:, kB:2kB] and WV[:, 0:kB].
// Thread = (row, column); every CTA forms M = T^H Y in shared memory.
__global__ void __launch_bounds__(256) he2hb_w_kernel(int64_t m, const z_t* __restrict__ X,
                                                      const z_t* __restrict__ Y,
                                                      const z_t* __restrict__ T, z_t* VW,
                                                      z_t* WV, int64_t ldw) {
  __shared__ z_t Ms[kB * kBp];
  for (int e = threadIdx.x; e < kB * kB; e += blockDim.x) {
    const int i = e % kB, c = e / kB;
    z_t t = make_double2(0.0, 0.0);
    for (int q = 0; q <= i; ++q) zcfma(t, T[q + i * kB], Y[q + c * kB]);  // T upper
    Ms[i + c * kBp] = t;
  }
  __syncthreads();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * kB) return;
  const int64_t r = e % m;
  const int c = int(e / m);
  z_t acc = make_double2(0.0, 0.0);
#pragma unroll 8
  for (int i = 0; i < kB; ++i) zfma(acc, VW[r + i * ldw], Ms[i + c * kBp]);
  const z_t x = X[r + c * ldw];
  const z_t w = make_double2(x.x - 0.5 * acc.x, x.y - 0.5 * acc.y);
  VW[r + (kB + c) * ldw] = w;
  WV[r + c * ldw] = w;
}

// Packs the lower band (offsets 0..kB) of A into AB (kLdab per column; offsets > kB zero),
// diagonal real.
__global__ void band_pack_kernel(int64_t n, const z_t* __restrict__ A, int64_t lda,
                                 z_t* __restrict__ AB) {
  const int64_t total = n * kLdab;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int o = int(e % kLdab);
    const int64_t c = e / kLdab;
    z_t v = make_double2(0.0, 0.0);
    if (o <= kB && c + o < n) {
      v = A[(c + o) + c * lda];
      if (o == 0) v.y = 0.0;
    }
    AB[e] = v;
  }
}

// ------------------------------------------------------------------------ stage 2: hb2st
struct ChaseArgs {
  z_t* AB;        // packed band, kLdab per column
  int64_t n;
  double* e;      // e[s] = beta of task (s, 0)
  z_t* V2;        // [j][s][kB] reflectors (v[0] = 1), zero padded
  z_t* tau2;      // [j][s]
  int* prog;      // tasks finished per sweep (zeroed; published for each group's last sweep)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Bulge chasing. A CTA takes groups of kChW consecutive sweeps (groups dealt round-robin over
// a cooperative grid) and runs each group as a wavefront: at step t warp w does task
// j = t - 2w of sweep sb + w, and one CTA barrier per step orders the warps (task j of sweep s
// needs task j+1 of sweep s-1, done by warp w-1 a step earlier; the two tasks running side by
// side touch disjoint entries). The group's first sweep waits on the previous group's last
// sweep through its progress counter (acquire/release). Per task the 32x32 blocks are staged
// with cp.async (one round trip), lane r owning row r for row-wise products and column r for
// column-wise ones; sB / sD hold the bulge block Bk_j and the Hermitian-expanded D_j.
__global__ void __launch_bounds__(32 * kChW, 1) hb2st_kernel(const __grid_constant__ ChaseArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  z_t* sB = reinterpret_cast<z_t*>(smraw) + warp * (2 * kB * kBp + 3 * kB);
  z_t* sD = sB + kB * kBp;
  z_t* sv = sD + kB * kBp;  // current reflector
  z_t* sw = sv + kB;        // two-sided w
  z_t* svp = sw + kB;       // previous reflector of the sweep
  const int64_t n = a.n, nsw = n - 1;
  const z_t zero = make_double2(0.0, 0.0), one = make_double2(1.0, 0.0);
  const int r = lane;
  for (int64_t g = blockIdx.x; g * kChW < nsw; g += gridDim.x) {
    const int64_t sb = g * kChW, s = sb + warp;
    const int nt = s < nsw ? int(ceil_div(nsw - s, kB)) : 0;
    const int nt0 = int(ceil_div(nsw - sb, kB));
    const int ntp = sb > 0 ? int(ceil_div(nsw - sb + 1, kB)) : 0;  // tasks of sweep sb - 1
    const int steps = nt0 + 2 * (kChW - 1);
    z_t taup = zero;
    for (int t = 0; t < steps; ++t) {
      if (warp == 0 && sb > 0 && t < nt0) {
        const int need = min(t + 2, ntp);
        while (ld_acquire(a.prog + sb - 1) < need) {
        }
      }
      __syncthreads();
      const int j = t - 2 * warp;
      if (j < 0 || j >= nt) continue;
      const int64_t lo = s + 1 + int64_t(j) * kB;
      const int L = int(min64(kB, n - lo));
      const int64_t plo = lo - kB;
      // ---- stage D_j (lower, zero outside L x L) and Bk_j in one round trip
#pragma unroll 8
      for (int c = 0; c < kB; ++c) {
        const bool okd = c < L && r >= c && r < L;
        if (r >= c) cp_async16(sD + c * kBp + r, okd ? a.AB + (r - c) + (lo + c) * kLdab : a.AB, okd);
      }
      if (j > 0) {
#pragma unroll 8
        for (int c = 0; c < kB; ++c) {
          const bool okb = r < L;
          cp_async16(sB + c * kBp + r, okb ? a.AB + (kB + r - c) + (plo + c) * kLdab : a.AB, okb);
        }
      }
      z_t xr = zero;
      if (j == 0 && r < L) xr = a.AB[(1 + r) + s * kLdab];
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      {  // mirror of D (row r's lane writes the upper entries of column r), real diagonal
        sD[r * kBp + r].y = 0.0;
        for (int c = 0; c < r; ++c) sD[r * kBp + c] = zconj(sD[c * kBp + r]);
      }
      if (j > 0) {
        // right-apply the previous reflector: Bk -= taup (Bk vp) vp^H (lane = row)
        z_t u = zero;
#pragma unroll 8
        for (int c = 0; c < kB; ++c) zfma(u, sB[c * kBp + r], svp[c]);
        const z_t tu = zmul(taup, u);
#pragma unroll 8
        for (int c = 0; c < kB; ++c) {
          const z_t vc = svp[c];
          z_t b = sB[c * kBp + r];
          b.x -= tu.x * vc.x + tu.y * vc.y;  // b -= tu conj(vc)
          b.y -= tu.y * vc.x - tu.x * vc.y;
          sB[c * kBp + r] = b;
        }
        xr = sB[r];
      }
      // ---- reflector of the column (rows lo .. lo+L-1)
      const double xn2 = warp_sum((r >= 1 && r < L) ? zabs2(xr) : 0.0);
      z_t alpha;
      alpha.x = __shfl_sync(0xffffffffu, xr.x, 0);
      alpha.y = __shfl_sync(0xffffffffu, xr.y, 0);
      double beta;
      z_t tau, scale;
      larfg2(alpha, xn2, beta, tau, scale);
      const z_t v = r == 0 ? one : (r < L ? zmul(scale, xr) : zero);
      sv[r] = v;
      a.V2[(int64_t(j) * n + s) * kB + r] = v;
      if (r == 0) a.tau2[int64_t(j) * n + s] = tau;
      __syncwarp();
      if (j == 0) {
        if (r < L) a.AB[(1 + r) + s * kLdab] = r == 0 ? make_double2(beta, 0.0) : zero;
        if (r == 0) a.e[s] = beta;
      } else {
        // left-apply H^H to Bk columns 1.. (lane = column); column 0 becomes (beta, 0, ...)
        const int c = r;
        if (c >= 1) {
          z_t w = zero;
          for (int q = 0; q < L; ++q) zcfma(w, sv[q], sB[c * kBp + q]);
          const z_t tw = zmul(zconj(tau), w);
          for (int q = 0; q < L; ++q) {
            z_t b = sB[c * kBp + q];
            const z_t vq = sv[q];
            b.x -= vq.x * tw.x - vq.y * tw.y;
            b.y -= vq.x * tw.y + vq.y * tw.x;
            sB[c * kBp + q] = b;
          }
        } else {
          sB[0] = make_double2(beta, 0.0);
          for (int q = 1; q < L; ++q) sB[q] = zero;
        }
        __syncwarp();
        if (r < L) {
#pragma unroll 8
          for (int cc = 0; cc < kB; ++cc)
            a.AB[(kB + r - cc) + (plo + cc) * kLdab] = sB[cc * kBp + r];
        }
      }
      // ---- two-sided on D_j: x = tau D v, alpha2 = -1/2 tau x^H v, w = x + alpha2 v
      z_t xv = zero;
#pragma unroll 8
      for (int c = 0; c < kB; ++c) zfma(xv, sD[c * kBp + r], sv[c]);
      xv = zmul(tau, xv);
      const z_t dot = warp_zsum(zcmul(xv, v));
      const z_t al = zscale(zmul(tau, dot), -0.5);
      const z_t w = zadd(xv, zmul(al, v));
      sw[r] = w;
      __syncwarp();
      if (r < L) {
        for (int c = 0; c <= r; ++c) {
          const z_t vc = sv[c], wc = sw[c];
          z_t d = sD[c * kBp + r];
          // d -= v_r conj(w_c) + w_r conj(v_c)
          d.x -= (v.x * wc.x + v.y * wc.y) + (w.x * vc.x + w.y * vc.y);
          d.y -= (v.y * wc.x - v.x * wc.y) + (w.y * vc.x - w.x * vc.y);
          if (c == r) d.y = 0.0;
          a.AB[(r - c) + (lo + c) * kLdab] = d;
        }
      }
      svp[r] = v;
      taup = tau;
      if (warp == kChW - 1) {  // the next group's first sweep waits on this one
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.prog + s, j + 1);
      }
    }
    __syncthreads();
  }
}

__global__ void band_diag_kernel(int64_t n, const z_t* __restrict__ AB, double* d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = AB[i * kLdab].x;
}

// ------------------------------------------------------------------------ back-transform Q2
struct Q2Args {
  z_t* Z;
  int64_t ldz, n, ncols;
  const z_t* V2;    // [j][s][kB]
  const z_t* tau2;  // [j][s]
};

// Z <- Q2 Z. Group (S, j) = reflectors of sweeps s0..s0+31 (s0 = 32 S) at task j, acting on
// window rows [s0+1+j kB, s0+j kB+64); groups run S descending, j ascending, s descending
// inside a group (tools/two_stage_model.py). Warp = 4 columns x 8 row residues: lane
// (rho, col) keeps window rows rho + 8k (k < 8) of its column in registers; reflector i
// (rows [i, i+31]) is a dot over the lane's rows in range (the others meet the zero padding
// of vs), a 3-step butterfly over rho and an axpy. The next group's reflectors stream into
// the other shared buffer (cp.async) while a group computes. Between groups of a pass the
// window moves 32 rows down: rows k < 4 are stored, k >= 4 move to k - 4, new rows load.
namespace {
constexpr int kVsW = 46;  // padded reflector row: v(t) at [7 + t], zeros at [0, 7) and [39, 46)
__device__ __forceinline__ bool q2_valid(int64_t s, int j, int64_t n) {
  return s < n - 1 && j < ceil_div(n - 1 - s, kB);
}
}  // namespace

__global__ void __launch_bounds__(32 * kQ2Warps) hb2st_q2_kernel(const __grid_constant__ Q2Args a) {
  __shared__ __align__(16) z_t vs[2][32][kVsW];
  __shared__ __align__(16) z_t ts[2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rho = lane >> 2, cl = lane & 3;
  const int64_t col = (int64_t(blockIdx.x) * kQ2Warps + warp) * 4 + cl;
  const bool cvalid = col < a.ncols;
  z_t* Zc = a.Z + (cvalid ? col : 0) * a.ldz;
  const int64_t n = a.n;
  const z_t zero = make_double2(0.0, 0.0);
  for (int e = threadIdx.x; e < 2 * 32 * kVsW; e += blockDim.x) (&vs[0][0][0])[e] = zero;
  __syncthreads();
  auto prefetch = [&](int buf, int S, int j) {
    const int64_t s0 = int64_t(S) * 32;
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
      const int i = e >> 5, t = e & 31;
      const bool ok = q2_valid(s0 + i, j, n);
      cp_async16(&vs[buf][i][7 + t], ok ? a.V2 + (int64_t(j) * n + s0 + i) * kB + t : a.V2, ok);
    }
    if (threadIdx.x < 32) {
      const bool ok = q2_valid(s0 + threadIdx.x, j, n);
      cp_async16(&ts[buf][threadIdx.x], ok ? a.tau2 + int64_t(j) * n + s0 + threadIdx.x : a.tau2,
                 ok);
    }
  };
  auto tasks = [&](int S) { return int(ceil_div(n - 1 - int64_t(S) * 32, kB)); };
  const int nS = int(ceil_div(n - 1, 32));
  int S = nS - 1, j = 0, buf = 0;
  int64_t wb = int64_t(S) * 32 + 1;
  z_t z[kQ2Reg];
#pragma unroll
  for (int k = 0; k < kQ2Reg; ++k) {
    const int64_t row = wb + rho + 8 * k;
    z[k] = (cvalid && row < n) ? Zc[row] : zero;
  }
  prefetch(0, S, 0);
  cp_async_commit();
  while (S >= 0) {
    const bool same = j + 1 < tasks(S);
    const int S2 = same ? S : S - 1, j2 = same ? j + 1 : 0;
    if (S2 >= 0) prefetch(buf ^ 1, S2, j2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
#pragma unroll
    for (int i = 31; i >= 0; --i) {
      const int klo = i / 8, khi = min((i + 31) / 8, kQ2Reg - 1);
      z_t w0 = zero, w1 = zero;
#pragma unroll
      for (int k = 0; k < kQ2Reg; ++k)
        if (k >= klo && k <= khi) {
          if (k & 1)
            zcfma(w1, vs[buf][i][7 + rho + 8 * k - i], z[k]);
          else
            zcfma(w0, vs[buf][i][7 + rho + 8 * k - i], z[k]);
        }
      z_t w = zadd(w0, w1);
      w = zadd(w, shfl_z(w, 4));
      w = zadd(w, shfl_z(w, 8));
      w = zadd(w, shfl_z(w, 16));
      const z_t tw = zmul(ts[buf][i], w);
#pragma unroll
      for (int k = 0; k < kQ2Reg; ++k)
        if (k >= klo && k <= khi) {
          const z_t vk = vs[buf][i][7 + rho + 8 * k - i];
          z[k].x -= vk.x * tw.x - vk.y * tw.y;
          z[k].y -= vk.x * tw.y + vk.y * tw.x;
        }
    }
    __syncthreads();  // vs[buf] is refilled by the next iteration's prefetch
    if (same) {  // window 32 rows down
#pragma unroll
      for (int k = 0; k < kQ2Reg / 2; ++k) {
        const int64_t row = wb + rho + 8 * k;
        if (cvalid && row < n) Zc[row] = z[k];
        z[k] = z[k + kQ2Reg / 2];
        const int64_t nrow = wb + 64 + rho + 8 * k;
        z[k + kQ2Reg / 2] = (cvalid && nrow < n) ? Zc[nrow] : zero;
      }
      wb += 32;
    } else {  // pass done: store the window, load the next pass's first window
#pragma unroll
      for (int k = 0; k < kQ2Reg; ++k) {
        const int64_t row = wb + rho + 8 * k;
        if (cvalid && row < n) Zc[row] = z[k];
      }
      if (S2 >= 0) {
        wb = int64_t(S2) * 32 + 1;
#pragma unroll
        for (int k = 0; k < kQ2Reg; ++k) {
          const int64_t row = wb + rho + 8 * k;
          z[k] = (cvalid && row < n) ? Zc[row] : zero;
        }
      }
    }
    S = S2;
    j = j2;
    buf ^= 1;
  }
}

// ------------------------------------------------------------------------ host side
namespace {
struct Ws2 {
  unsigned* bar;
  z_t *VW, *WV, *VT, *X, *Y, *T, *alphab, *part, *splitk, *hsplit, *AB, *V2, *tau2;
  double* normp;
  int* prog;
  int64_t nt, splitk_elems, hsplit_elems;
};

Ws2 carve(void* ws, int64_t n) {
  Ws2 w{};
  char* p = reinterpret_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) & ~size_t(255);
    return q;
  };
  const int64_t G = ceil_div(n, kQrT);
  w.nt = ceil_div(max64(n - 1, 1), kB);
  w.splitk_elems = int64_t(16) * kB * kB;
  w.bar = reinterpret_cast<unsigned*>(take(256));
  w.VW = reinterpret_cast<z_t*>(take(size_t(n) * 2 * kB * sizeof(z_t)));
  w.WV = reinterpret_cast<z_t*>(take(size_t(n) * 2 * kB * sizeof(z_t)));
  w.VT = reinterpret_cast<z_t*>(take(size_t(n) * kB * sizeof(z_t)));
  w.X = reinterpret_cast<z_t*>(take(size_t(n) * kB * sizeof(z_t)));
  w.Y = reinterpret_cast<z_t*>(take(size_t(kB) * kB * sizeof(z_t)));
  w.T = reinterpret_cast<z_t*>(take(size_t(kB) * kB * sizeof(z_t)));
  w.alphab = reinterpret_cast<z_t*>(take(sizeof(z_t)));
  w.part = reinterpret_cast<z_t*>(take(size_t(G) * kB * sizeof(z_t)));
  w.normp = reinterpret_cast<double*>(take(size_t(G) * sizeof(double)));
  w.splitk = reinterpret_cast<z_t*>(take(size_t(w.splitk_elems) * sizeof(z_t)));
  w.hsplit_elems = int64_t(16) * n * kB;
  w.hsplit = reinterpret_cast<z_t*>(take(size_t(w.hsplit_elems) * sizeof(z_t)));
  w.AB = reinterpret_cast<z_t*>(take(size_t(n) * kLdab * sizeof(z_t)));
  w.V2 = reinterpret_cast<z_t*>(take(size_t(w.nt) * n * kB * sizeof(z_t)));
  w.tau2 = reinterpret_cast<z_t*>(take(size_t(w.nt) * n * sizeof(z_t)));
  w.prog = reinterpret_cast<int*>(take(size_t(n) * sizeof(int)));
  return w;
}

size_t chase_smem() { return size_t(kChW) * (2 * kB * kBp + 3 * kB) * sizeof(z_t); }
}  // namespace

size_t hetrd2_workspace_bytes(int64_t n) {
  const int64_t G = ceil_div(n, kQrT);
  const int64_t nt = ceil_div(max64(n - 1, 1), kB);
  size_t b = 256;
  b += size_t(n) * kB * 6 * sizeof(z_t);
  b += size_t(kB) * kB * 2 * sizeof(z_t) + sizeof(z_t);
  b += size_t(G) * (kB * sizeof(z_t) + sizeof(double));
  b += size_t(16) * kB * kB * sizeof(z_t);
  b += size_t(16) * n * kB * sizeof(z_t);
  b += size_t(n) * kLdab * sizeof(z_t);
  b += size_t(nt) * n * (kB + 1) * sizeof(z_t);
  b += size_t(n) * sizeof(int);
  return b + 20 * 256;
}

namespace {
// 0 = one-stage (default: measured faster on B200), 1 = two-stage
std::atomic<int> g_tridiag_mode{[] {
  const char* e = getenv("BSE_TWO_STAGE");
  return e && atoi(e) != 0 ? 1 : 0;
}()};
}  // namespace

// Per-call snapshot: a solve decides workspace size, reduction and back-transform from one
// reading, so a concurrent bse_set_tridiagonal_reduction cannot split a solve's choices.
thread_local int g_tridiag_snap = -1;

int set_tridiag_mode(int mode) { return g_tridiag_mode.exchange(mode != 0 ? 1 : 0); }

int current_tridiag_mode() { return g_tridiag_snap >= 0 ? g_tridiag_snap : g_tridiag_mode.load(); }

TridiagModeScope::TridiagModeScope(int mode) : owner(g_tridiag_snap < 0) {
  if (owner) g_tridiag_snap = mode >= 0 ? mode : g_tridiag_mode.load();
}
TridiagModeScope::~TridiagModeScope() {
  if (owner) g_tridiag_snap = -1;
}

bool use_two_stage(int64_t n) { return n >= 4 * kB && current_tridiag_mode() != 0; }

void zhetrd_2stage(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                   z_t* tau1, void* ws) {
  if (n <= 0) return;
  Ws2 w = carve(ws, n);
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0}, mone = {-1.0, 0.0};
  BSE_CUDA(cudaMemsetAsync(tau1, 0, sizeof(z_t) * size_t(n), s));
  const bool& attr = per_device([] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(hb2st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(chase_smem())));
    BSE_CUDA(cudaFuncSetAttribute(he2hb_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kQrSmem)));
    return true;
  });
  (void)attr;
  // ---- stage 1: panels c0 = 0, kB, ... while the panel has >= 2 rows below the band
  for (int64_t c0 = 0; c0 + kB <= n - 2; c0 += kB) {
    const int64_t r0 = c0 + kB, m = n - r0;
    QrArgs q{};
    q.P = A + r0 + c0 * lda;
    q.ldp = lda;
    q.m = m;
    q.k = int(min64(m, kB));
    q.VW = w.VW;
    q.WV = w.WV;
    q.VT = w.VT;
    q.ldw = n;
    q.T = w.T;
    q.tau = tau1 + c0;
    q.normp = w.normp;
    q.alphab = w.alphab;
    q.part = w.part;
    q.bar = w.bar;
    BSE_CUDA(cudaMemsetAsync(w.bar, 0, 256, s));
    const int G = int(ceil_div(m, kQrT));
    void* args[] = {&q};
    BSE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(he2hb_qr_kernel), dim3(G),
                                         dim3(kQrT), args, kQrSmem, s));
    count_launch();
    z_t* A22 = A + r0 + r0 * lda;
    // X = A22 (V T) over the lower triangle: E (V T) + E^H (V T), E = lower(A22), diagonal
    // halved (exact power-of-two scaling, restored below)
    scale_diag(s, m, A22, lda, 0.5);
    zgemm(s, 0, 0, m, kB, m, one, A22, lda, w.VT, n, zero, w.X, n, kLowerOp, kGeneral, 0,
          w.hsplit, w.hsplit_elems);
    zgemm(s, 1, 0, m, kB, m, one, A22, lda, w.VT, n, one, w.X, n, kUpperOp, kGeneral, 0,
          w.hsplit, w.hsplit_elems);
    scale_diag(s, m, A22, lda, 2.0);
    // Y = V^H X ; W = X - 1/2 V T^H Y
    zgemm(s, 1, 0, kB, kB, m, one, w.VW, n, w.X, n, zero, w.Y, kB, kGeneral, kGeneral, 0,
          w.splitk, w.splitk_elems);
    {
      const int64_t tot = m * kB;
      he2hb_w_kernel<<<unsigned(ceil_div(tot, 256)), 256, 0, s>>>(m, w.X, w.Y, w.T, w.VW, w.WV,
                                                                   n);
      BSE_LAUNCH_CHECK();
    }
    // A22 -= V W^H + W V^H (lower tiles)
    zgemm(s, 0, 1, m, m, 2 * kB, mone, w.VW, n, w.WV, n, one, A22, lda, kGeneral, kGeneral, 1,
          nullptr, 0);
  }
  // ---- stage 2
  band_pack_kernel<<<unsigned(min64(ceil_div(n * kLdab, 256), 148 * 8)), 256, 0, s>>>(n, A, lda,
                                                                                     w.AB);
  BSE_LAUNCH_CHECK();
  BSE_CUDA(cudaMemsetAsync(w.prog, 0, sizeof(int) * size_t(n), s));
  {
    const int64_t nt0 = ceil_div(n - 1, kB);
    int G = int(min64(ceil_div(nt0, 2 * kChW) + 2, 148));
    if (g_panel_ctas > 0) G = int(min64(G, max64(g_panel_ctas / 2, 1)));
    ChaseArgs c{};
    c.AB = w.AB;
    c.n = n;
    c.e = e;
    c.V2 = w.V2;
    c.tau2 = w.tau2;
    c.prog = w.prog;
    void* args[] = {&c};
    BSE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(hb2st_kernel), dim3(G),
                                         dim3(32 * kChW), args, chase_smem(), s));
    count_launch();
  }
  band_diag_kernel<<<unsigned(min64(ceil_div(n, 256), 148)), 256, 0, s>>>(n, w.AB, d);
  BSE_LAUNCH_CHECK();
}

void zunmtr_2stage(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau1,
                   void* ws2, z_t* Z, int64_t ldz, int64_t ncols, void* ws) {
  if (n <= 1 || ncols <= 0) return;
  Ws2 w = carve(ws2, n);
  Q2Args q{};
  q.Z = Z;
  q.ldz = ldz;
  q.n = n;
  q.ncols = ncols;
  q.V2 = w.V2;
  q.tau2 = w.tau2;
  const int64_t blocks = ceil_div(ncols, 4 * kQ2Warps);
  hb2st_q2_kernel<<<unsigned(blocks), 32 * kQ2Warps, 0, s>>>(q);
  BSE_LAUNCH_CHECK();
  if (n > kB + 1) apply_prepared_reflectors(s, 3, n, n - kB, Z, ldz, ncols, ws);  // Q1
}

size_t tridiag_workspace_bytes(int64_t n) {
  return use_two_stage(n) ? hetrd2_workspace_bytes(n) : hetrd_workspace_bytes(n);
}

void tridiag_reduce(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                    z_t* tau, void* ws) {
  if (use_two_stage(n))
    zhetrd_2stage(s, n, A, lda, d, e, tau, ws);
  else
    zhetrd_lower(s, n, A, lda, d, e, tau, ws);
}

void tridiag_back_prepare(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau,
                          void* ws_unmtr) {
  if (use_two_stage(n)) {
    if (n > kB + 1) prepare_reflectors(s, 3, n, n - kB, A, lda, tau, ws_unmtr);
  } else {
    prepare_reflectors(s, 0, n, n - 1, A, lda, tau, ws_unmtr);
  }
}

void tridiag_back(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau,
                  void* ws, z_t* Z, int64_t ldz, int64_t ncols, void* ws_unmtr, bool prepared) {
  if (!prepared) tridiag_back_prepare(s, n, A, lda, tau, ws_unmtr);
  if (use_two_stage(n)) {
    zunmtr_2stage(s, n, A, lda, tau, ws, Z, ldz, ncols, ws_unmtr);
  } else {
    apply_prepared_reflectors(s, 0, n, n - 1, Z, ldz, ncols, ws_unmtr);
  }
}

}  // namespace bseg
