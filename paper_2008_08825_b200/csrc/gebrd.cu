// gebrd.cu — Householder bidiagonalisation C = Q B P^H (B upper bidiagonal) and the
// back-transformations U = Q U_B, V = P V_B.
//
// Replaces zgebrd + zungbr inside LAPACKE_zgesvd('A','A') at proj/src/backend.cpp:74
// (SURVEY §8a rows a9.1, a9.2). The singular values/vectors of B come from the
// Golub–Kahan tridiagonal through the GPU divide & conquer (stedc.cu) instead of zbdsqr.
//
// Same algorithm as LAPACK's zlabrd panel + two trailing GEMMs, restructured for B200 as
// one persistent cooperative kernel per nb-column panel with four grid-wide phases per
// column g (fixed-order partial sums => deterministic):
//   P1 rows : finalise X(:,g-1); column update a(:,g) -= V Y(g,:)^H + X U(g,:)^H; partials
//   P2      : column reflector (zlarfg, redundant per CTA); y' = A(g:,g+1:)^H v (64x64 tiles)
//   P3 cols : Y(:,g) = tauq (y' - Y t1 - U t2); row update w = conj(a(g,:)) - ...; partials
//   P4      : row reflector; x' = A(g+1:,g+1:) u (64x64 tiles)
// The two matrix-vector products stream the whole trailing matrix (10.7 n^3 bytes over the
// reduction — the HBM-bound half of zgebrd); the trailing update
// A -= [V X][Y U]^H is a single DMMA GEMM with k = 2 nb.
#include <cooperative_groups.h>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "svd.h"

namespace cg = cooperative_groups;

namespace bseg {

namespace {
constexpr int kT = 64;
constexpr int kRB = 256;
constexpr int kThreads = 256;
constexpr int kNB = kGebrdNB;
}  // namespace

struct GebrdArgs {
  z_t* A;
  int64_t lda, n;
  double* d;
  double* e;
  z_t* tauq;
  z_t* taup;
  z_t* VX;  // n x 2NB: [V | X]
  z_t* YU;  // n x 2NB: [Y | U]
  z_t* wrow;     // n
  z_t* P;        // nch * nch * kT tile partials
  double* normp; // nrb
  z_t* s12;      // nrb x 2NB
  z_t* s34;      // nrb x 2(NB+1)
  z_t* t;        // 4 (NB+1): t1 | t2 | t3 | t4
  int64_t p0;
  int nbp, nch, nrb;
};

__device__ __forceinline__ void larfg_params2(z_t alpha, double xnorm2, double& beta, z_t& tau,
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
  const z_t am = make_double2(alpha.x - beta, alpha.y);
  const double den = am.x * am.x + am.y * am.y;
  scale = make_double2(am.x / den, -am.y / den);
}

__global__ void __launch_bounds__(kThreads) gebrd_panel_kernel(GebrdArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* tile = reinterpret_cast<z_t*>(sm);  // kT x (kT+1)
  z_t* vt = tile + kT * (kT + 1);          // kT vector over the reduced dimension
  z_t* red = vt + kT;                      // 4 x kT
  z_t* sa = red + 4 * kT;                  // NB+1
  z_t* sb = sa + 64;                       // NB+1
  z_t* xs = sb + 64;                       // kRB
  z_t* xc = xs + kRB;                      // kRB : X(r, i-1) of this block
  double* dred = reinterpret_cast<double*>(xc + kRB);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t n = a.n, lda = a.lda, ldp = n;
  z_t* V = a.VX;
  z_t* X = a.VX + int64_t(kNB) * ldp;
  z_t* Y = a.YU;
  z_t* U = a.YU + int64_t(kNB) * ldp;
  z_t* t1 = a.t;
  z_t* t2 = a.t + (kNB + 1);
  z_t* t3 = a.t + 2 * (kNB + 1);
  z_t* t4 = a.t + 3 * (kNB + 1);
  const z_t zero = make_double2(0.0, 0.0);

  for (int i = 0; i <= a.nbp; ++i) {
    const int64_t g = a.p0 + i;
    const bool last = (i == a.nbp);
    // ---------------------------------------------------------------- P1 (rows)
    const bool have_prev_row = (i > 0) && (g - 1 + 1 < n);  // previous column had a row reflector
    z_t taup_prev = zero;
    if (have_prev_row) taup_prev = a.taup[g - 1];
    if (!last) {
      for (int p = tid; p < i; p += blockDim.x) {
        sa[p] = Y[g + int64_t(p) * ldp];
        sb[p] = U[g + int64_t(p) * ldp];
      }
    }
    __syncthreads();
    for (int rb = cta; rb < a.nrb; rb += G) {
      const int64_t r = int64_t(rb) * kRB + tid;
      const bool valid = r < n && r >= g;
      z_t xprev = zero;
      if (have_prev_row && valid) {
        // X(r, i-1) = taup (x' - V(r, 0:i) t3 - X(r, 0:i-1) t4), x' from the tile partials
        const int ch = int(r / kT), off = int(r % kT);
        z_t xp = zero;
        for (int cc = int(g / kT); cc < a.nch; ++cc) xp = zadd(xp, a.P[(int64_t(ch) * a.nch + cc) * kT + off]);
        for (int p = 0; p < i; ++p) xp = zsub(xp, zmul(V[r + int64_t(p) * ldp], t3[p]));
        for (int p = 0; p < i - 1; ++p) xp = zsub(xp, zmul(X[r + int64_t(p) * ldp], t4[p]));
        xprev = zmul(taup_prev, xp);
        X[r + int64_t(i - 1) * ldp] = xprev;
      }
      xc[tid] = xprev;
      if (last) continue;
      z_t x = zero;
      if (valid) {
        x = a.A[r + g * lda];
        for (int p = 0; p < i; ++p) {
          const z_t xrp = (p == i - 1) ? xprev : X[r + int64_t(p) * ldp];
          x = zsub(x, zmul(V[r + int64_t(p) * ldp], zconj(sa[p])));
          x = zsub(x, zmul(xrp, zconj(sb[p])));
        }
        a.A[r + g * lda] = x;
      }
      const bool inx = valid && r > g;
      xs[tid] = inx ? x : zero;
      const double nrm = block_sum(inx ? zabs2(x) : 0.0, dred);  // contains __syncthreads
      if (tid == 0) a.normp[rb] = nrm;
      for (int p = warp; p < i; p += kThreads / 32) {
        z_t s1 = zero, s2 = zero;
        for (int j = lane; j < kRB; j += 32) {
          const int64_t rr = int64_t(rb) * kRB + j;
          if (rr > g && rr < n) {
            const z_t xv = xs[j];
            zcfma(s1, V[rr + int64_t(p) * ldp], xv);
            const z_t xx = (p == i - 1) ? xc[j] : X[rr + int64_t(p) * ldp];
            zcfma(s2, xx, xv);
          }
        }
        s1 = warp_zsum(s1);
        s2 = warp_zsum(s2);
        if (lane == 0) {
          a.s12[int64_t(rb) * 2 * kNB + p] = s1;
          a.s12[int64_t(rb) * 2 * kNB + kNB + p] = s2;
        }
      }
      __syncthreads();
    }
    if (last) break;
    grid.sync();
    // ---------------------------------------------------------------- P2: column reflector + y'
    double xn2 = 0.0;
    for (int rb = int(g / kRB); rb < a.nrb; ++rb) xn2 += a.normp[rb];
    const z_t alpha = a.A[g + g * lda];
    double beta;
    z_t tq, scale;
    larfg_params2(alpha, xn2, beta, tq, scale);
    if (cta == 0) {
      if (tid == 0) {
        a.d[g] = beta;
        a.tauq[g] = tq;
      }
      for (int p = tid; p < i; p += blockDim.x) {
        z_t s1 = zero, s2 = zero;
        for (int rb = int(g / kRB); rb < a.nrb; ++rb) {
          s1 = zadd(s1, a.s12[int64_t(rb) * 2 * kNB + p]);
          s2 = zadd(s2, a.s12[int64_t(rb) * 2 * kNB + kNB + p]);
        }
        t1[p] = zadd(zconj(V[g + int64_t(p) * ldp]), zmul(scale, s1));
        t2[p] = zadd(zconj(X[g + int64_t(p) * ldp]), zmul(scale, s2));
      }
    }
    for (int rb = cta; rb < a.nrb; rb += G) {
      const int64_t r = int64_t(rb) * kRB + tid;
      if (r < n) {
        z_t v = zero;
        if (r == g) v = make_double2(1.0, 0.0);
        else if (r > g) v = zmul(scale, a.A[r + g * lda]);
        V[r + int64_t(i) * ldp] = v;
      }
    }
    const bool has_cols = (g + 1 < n);
    if (has_cols) {
      const int r0c = int(g / kT), c0c = int((g + 1) / kT);
      const int Kr = a.nch - r0c, Kc = a.nch - c0c;
      const int64_t ntiles = int64_t(Kr) * Kc;
      for (int64_t t = cta; t < ntiles; t += G) {
        const int rc = r0c + int(t % Kr), cc = c0c + int(t / Kr);
        const int64_t R0 = int64_t(rc) * kT, C0 = int64_t(cc) * kT;
        __syncthreads();
        if (tid < kT) {
          const int64_t r = R0 + tid;
          z_t v = zero;
          if (r == g) v = make_double2(1.0, 0.0);
          else if (r > g && r < n) v = zmul(scale, a.A[r + g * lda]);
          vt[tid] = v;
        }
        for (int e = tid; e < kT * kT; e += kThreads) {
          const int rr = e % kT, cl = e / kT;
          const int64_t r = R0 + rr, c = C0 + cl;
          z_t val = zero;
          if (r < n && c < n && r >= g && c > g) val = a.A[r + c * lda];
          tile[rr + cl * (kT + 1)] = val;
        }
        __syncthreads();
        const int q = tid >> 6, x = tid & 63;
        z_t yc = zero;
        for (int k = q * 16; k < q * 16 + 16; ++k) zcfma(yc, tile[k + x * (kT + 1)], vt[k]);
        red[q * kT + x] = yc;
        __syncthreads();
        if (q == 0) {
          z_t s = zadd(zadd(red[x], red[kT + x]), zadd(red[2 * kT + x], red[3 * kT + x]));
          a.P[(int64_t(cc) * a.nch + rc) * kT + x] = s;
        }
      }
    }
    grid.sync();
    // ---------------------------------------------------------------- P3 (columns): Y(:,i), row update
    for (int p = tid; p <= i; p += blockDim.x) {
      sa[p] = (p == i) ? make_double2(1.0, 0.0) : V[g + int64_t(p) * ldp];  // V(g, p)
      sb[p] = (p == i) ? zero : X[g + int64_t(p) * ldp];                    // X(g, p)
    }
    __syncthreads();
    // reflector storage of column g (own row blocks; P2 readers are done)
    for (int rb = cta; rb < a.nrb; rb += G) {
      const int64_t r = int64_t(rb) * kRB + tid;
      if (r < n && r > g) a.A[r + g * lda] = V[r + int64_t(i) * ldp];
    }
    if (has_cols) {
      for (int cb = cta; cb < a.nrb; cb += G) {
        const int64_t c = int64_t(cb) * kRB + tid;
        const bool valid = c < n && c > g;
        z_t w = zero, ycur = zero;
        if (valid) {
          const int ch = int(c / kT), off = int(c % kT);
          z_t y = zero;
          for (int rc = int(g / kT); rc < a.nch; ++rc) y = zadd(y, a.P[(int64_t(ch) * a.nch + rc) * kT + off]);
          for (int p = 0; p < i; ++p) {
            y = zsub(y, zmul(Y[c + int64_t(p) * ldp], t1[p]));
            y = zsub(y, zmul(U[c + int64_t(p) * ldp], t2[p]));
          }
          ycur = zmul(tq, y);
          Y[c + int64_t(i) * ldp] = ycur;
          w = zconj(a.A[g + c * lda]);
          for (int p = 0; p < i; ++p) {
            w = zsub(w, zmul(Y[c + int64_t(p) * ldp], zconj(sa[p])));
            w = zsub(w, zmul(U[c + int64_t(p) * ldp], zconj(sb[p])));
          }
          w = zsub(w, ycur);  // p = i: Y(c,i) * conj(V(g,i)) with V(g,i) = 1
          a.wrow[c] = w;
        }
        const bool inx = valid && c >= g + 2;
        xs[tid] = inx ? w : zero;
        xc[tid] = valid ? ycur : zero;
        const double nrm = block_sum(inx ? zabs2(w) : 0.0, dred);
        if (tid == 0) a.normp[cb] = nrm;
        for (int p = warp; p <= i; p += kThreads / 32) {
          z_t s3 = zero, s4 = zero;
          for (int j = lane; j < kRB; j += 32) {
            const int64_t cc2 = int64_t(cb) * kRB + j;
            if (cc2 >= g + 2 && cc2 < n) {
              const z_t wv = xs[j];
              const z_t yy = (p == i) ? xc[j] : Y[cc2 + int64_t(p) * ldp];
              zcfma(s3, yy, wv);
              if (p < i) zcfma(s4, U[cc2 + int64_t(p) * ldp], wv);
            }
          }
          s3 = warp_zsum(s3);
          s4 = warp_zsum(s4);
          if (lane == 0) {
            a.s34[int64_t(cb) * 2 * (kNB + 1) + p] = s3;
            a.s34[int64_t(cb) * 2 * (kNB + 1) + (kNB + 1) + p] = s4;
          }
        }
        __syncthreads();
      }
    }
    grid.sync();
    // ---------------------------------------------------------------- P4: row reflector + x'
    if (has_cols) {
      double xr2 = 0.0;
      for (int cb = int((g + 1) / kRB); cb < a.nrb; ++cb) xr2 += a.normp[cb];
      const z_t alpha2 = a.wrow[g + 1];
      double beta2;
      z_t tp, scale2;
      larfg_params2(alpha2, xr2, beta2, tp, scale2);
      if (cta == 0) {
        if (tid == 0) {
          a.e[g] = beta2;
          a.taup[g] = tp;
        }
        for (int p = tid; p <= i; p += blockDim.x) {
          z_t s3 = zero, s4 = zero;
          for (int cb = int((g + 1) / kRB); cb < a.nrb; ++cb) {
            s3 = zadd(s3, a.s34[int64_t(cb) * 2 * (kNB + 1) + p]);
            s4 = zadd(s4, a.s34[int64_t(cb) * 2 * (kNB + 1) + (kNB + 1) + p]);
          }
          t3[p] = zadd(zconj(Y[(g + 1) + int64_t(p) * ldp]), zmul(scale2, s3));
          if (p < i) t4[p] = zadd(zconj(U[(g + 1) + int64_t(p) * ldp]), zmul(scale2, s4));
        }
      }
      for (int cb = cta; cb < a.nrb; cb += G) {
        const int64_t c = int64_t(cb) * kRB + tid;
        if (c < n) {
          z_t u = zero;
          if (c == g + 1) u = make_double2(1.0, 0.0);
          else if (c >= g + 2) {
            u = zmul(scale2, a.wrow[c]);
            a.A[g + c * lda] = u;  // row reflector storage (unconjugated)
          }
          U[c + int64_t(i) * ldp] = u;
        }
      }
      const int r0c = int((g + 1) / kT), c0c = int((g + 1) / kT);
      const int Kr = a.nch - r0c, Kc = a.nch - c0c;
      const int64_t ntiles = int64_t(Kr) * Kc;
      for (int64_t t = cta; t < ntiles; t += G) {
        const int rc = r0c + int(t % Kr), cc = c0c + int(t / Kr);
        const int64_t R0 = int64_t(rc) * kT, C0 = int64_t(cc) * kT;
        __syncthreads();
        if (tid < kT) {
          const int64_t c = C0 + tid;
          z_t u = zero;
          if (c == g + 1) u = make_double2(1.0, 0.0);
          else if (c >= g + 2 && c < n) u = zmul(scale2, a.wrow[c]);
          vt[tid] = u;
        }
        for (int e = tid; e < kT * kT; e += kThreads) {
          const int rr = e % kT, cl = e / kT;
          const int64_t r = R0 + rr, c = C0 + cl;
          z_t val = zero;
          if (r < n && c < n && r > g && c > g) val = a.A[r + c * lda];
          tile[rr + cl * (kT + 1)] = val;
        }
        __syncthreads();
        const int q = tid >> 6, x = tid & 63;
        z_t xr = zero;
        for (int k = q * 16; k < q * 16 + 16; ++k) zfma(xr, tile[x + k * (kT + 1)], vt[k]);
        red[q * kT + x] = xr;
        __syncthreads();
        if (q == 0) {
          z_t s = zadd(zadd(red[x], red[kT + x]), zadd(red[2 * kT + x], red[3 * kT + x]));
          a.P[(int64_t(rc) * a.nch + cc) * kT + x] = s;
        }
      }
    }
    grid.sync();
  }
}

size_t gebrd_workspace_bytes(int64_t n) {
  const int64_t nch = ceil_div(n, kT), nrb = ceil_div(n, kRB);
  size_t z = 0;
  z += size_t(n) * 2 * kNB * 2;  // VX, YU
  z += size_t(n);                // wrow
  z += size_t(nch) * nch * kT;   // P
  z += size_t(nrb) * 2 * kNB;    // s12
  z += size_t(nrb) * 2 * (kNB + 1);
  z += size_t(4) * (kNB + 1);
  return z * sizeof(z_t) + size_t(nrb) * sizeof(double) + 1024;
}

void zgebrd_upper(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tauq, z_t* taup, void* ws) {
  if (n <= 0) return;
  const int nch = int(ceil_div(n, kT)), nrb = int(ceil_div(n, kRB));
  z_t* base = reinterpret_cast<z_t*>(ws);
  GebrdArgs a{};
  a.A = A; a.lda = lda; a.n = n; a.d = d; a.e = e; a.tauq = tauq; a.taup = taup;
  a.VX = base; base += n * 2 * kNB;
  a.YU = base; base += n * 2 * kNB;
  a.wrow = base; base += n;
  a.P = base; base += int64_t(nch) * nch * kT;
  a.s12 = base; base += int64_t(nrb) * 2 * kNB;
  a.s34 = base; base += int64_t(nrb) * 2 * (kNB + 1);
  a.t = base; base += 4 * (kNB + 1);
  a.normp = reinterpret_cast<double*>(base);
  a.nch = nch; a.nrb = nrb;
  const size_t smem = (size_t(kT) * (kT + 1) + kT + 4 * kT + 128 + 2 * kRB) * sizeof(z_t) +
                      32 * sizeof(double);
  static int blocks_per_sm = -1, num_sms = 0;
  if (blocks_per_sm < 0) {
    BSE_CUDA(cudaFuncSetAttribute(gebrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    int dev;
    BSE_CUDA(cudaGetDevice(&dev));
    BSE_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    BSE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, gebrd_panel_kernel,
                                                           kThreads, smem));
    if (blocks_per_sm < 1) throw std::runtime_error("gebrd: kernel cannot be resident");
  }
  const z_t mone = {-1.0, 0.0}, one = {1.0, 0.0};
  for (int64_t p0 = 0; p0 < n; p0 += kNB) {
    const int nbp = int(min64(kNB, n - p0));
    BSE_CUDA(cudaMemsetAsync(a.VX, 0, sizeof(z_t) * size_t(n) * 2 * kNB * 2, s));
    a.p0 = p0;
    a.nbp = nbp;
    const int64_t m = n - p0;
    const int64_t tiles = ceil_div(m, kT) * ceil_div(m, kT);
    int G = int(min64(int64_t(blocks_per_sm) * num_sms, max64(tiles, ceil_div(m, kRB))));
    G = max(G, 1);
    void* args[] = {&a};
    double bytes = 0.0;  // algorithmic: A^H v over (n-g) x (n-g-1) and A u over (n-g-1)^2
    for (int i = 0; i < nbp; ++i) {
      const double r = double(n - (p0 + i));
      bytes += (r * (r - 1.0) + (r - 1.0) * (r - 1.0)) * sizeof(z_t);
    }
    const int slot = g_timer ? timer_begin(s, 1, bytes) : -1;
    BSE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(gebrd_panel_kernel), dim3(G),
                                         dim3(kThreads), args, smem, s));
    timer_end(s, slot);
    count_launch();
    const int64_t q = p0 + nbp;
    if (q < n) {
      // A(q:, q:) -= [V X](q:, :) [Y U](q:, :)^H
      zgemm(s, 0, 1, n - q, n - q, 2 * kNB, mone, a.VX + q, n, a.YU + q, n, one, A + q + q * lda,
            lda, kGeneral, kGeneral, 0, nullptr, 0);
    }
  }
}

size_t unmbr_workspace_bytes(int64_t n, int64_t ncols) { return unmtr_workspace_bytes(n, ncols); }

void zunmbr_q(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tauq, z_t* Z,
              int64_t ldz, int64_t ncols, void* ws) {
  apply_reflectors(s, 1, n, n, A, lda, tauq, Z, ldz, ncols, ws);
}

void zunmbr_p(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* taup, z_t* Z,
              int64_t ldz, int64_t ncols, void* ws) {
  apply_reflectors(s, 2, n, n - 1, A, lda, taup, Z, ldz, ncols, ws);
}

}  // namespace bseg
