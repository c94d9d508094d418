// hetrd.cu — Householder tridiagonalisation of a Hermitian matrix (lower storage) and the
// blocked back-transformation V = Q Z.
//
// Replaces the zhetrd + zunmtr halves of LAPACKE_zheevd('V','L') called at
// proj/src/backend.cpp:34. Same algorithm as LAPACK's zlatrd
// ('L') panel + zher2k trailing update, re-laid-out for B200:
//
//  * One persistent cooperative kernel per nb-column panel. Per column g three grid-wide
//    phases (separated by grid barriers) replace LAPACK's ~8 BLAS-2 calls:
//      P1  finalize W(:,g-1); column update a(:,g) -= V W(g,:)^H + W V(g,:)^H; partial
//          norms and partial V^H x / W^H x products per 256-row block (fixed-order partials,
//          deterministic);
//      P2  reflector (zlarfg, recomputed redundantly by every CTA from the partials) and the
//          Hermitian matrix-vector product y = A22 v over the LOWER triangle only: 64x64
//          tiles staged in shared memory, each tile contributes A_t v to its row chunk and
//          A_t^H v to its column chunk (2.67 n^3 bytes total, the HBM-bound half of zhetrd);
//      P3  reduce the tile partials, w = tau (y - V t1 - W t2), partial dot w^H v.
//  * The trailing update A22 -= V W^H + W V^H is one DMMA GEMM with k = 2 nb writing only
//    lower tiles.
#include <cooperative_groups.h>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"

namespace cg = cooperative_groups;

namespace bseg {

namespace {
constexpr int kT = 64;     // hemv tile
constexpr int kRB = 256;   // row block of phases 1/3 (= threads per CTA)
constexpr int kThreads = 256;
}  // namespace

struct HetrdArgs {
  z_t* A;
  int64_t lda, n;
  double* d;
  double* e;
  z_t* tau;
  z_t* VW;  // n x 2NB: [V | W]
  z_t* WV;  // n x 2NB: [W | V]
  int64_t ldp;
  z_t* wtmp;      // n   : unscaled-then-tau'd w before the alpha correction
  z_t* Y;         // nch * nch * kT
  double* normp;  // nrb
  z_t* s1p;       // nrb x NB
  z_t* s2p;       // nrb x NB
  z_t* t12;       // 2 NB
  z_t* dotp;      // nrb
  int64_t p0;
  int nbp, nb, nch, nrb;
};

__device__ __forceinline__ z_t zdiv1(z_t a) {  // 1 / a
  const double den = a.x * a.x + a.y * a.y;
  return make_double2(a.x / den, -a.y / den);
}

// zlarfg on (alpha, ||x||): returns beta (real), tau, scale = 1/(alpha-beta) (1 if tau == 0).
__device__ __forceinline__ void larfg_params(z_t alpha, double xnorm2, double& beta, z_t& tau,
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

__global__ void __launch_bounds__(kThreads) hetrd_panel_kernel(HetrdArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char sm[];
  z_t* tile = reinterpret_cast<z_t*>(sm);  // kT x (kT+1) column-major
  z_t* vr = tile + kT * (kT + 1);          // kT : v over tile rows
  z_t* vc = vr + kT;                       // kT : v over tile cols
  z_t* red = vc + kT;                      // 4 x kT reduction scratch
  z_t* wg = red + 4 * kT;                  // NB : W(g, p)
  z_t* vg = wg + 64;                       // NB : V(g, p)
  z_t* xs = vg + 64;                       // kRB : updated column values
  double* dred = reinterpret_cast<double*>(xs + kRB);  // 32 doubles
  z_t* zred = reinterpret_cast<z_t*>(dred + 32);        // 8 x 64 complex

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t n = a.n, lda = a.lda, ldp = a.ldp;
  const int NB = a.nb;
  z_t* V = a.VW;
  z_t* W = a.VW + int64_t(NB) * ldp;

  for (int i = 0; i <= a.nbp; ++i) {
    const int64_t g = a.p0 + i;
    const bool last = (i == a.nbp);  // finalisation-only step
    // ------------------------------------------------------------------ phase 1
    z_t alpha_prev = make_double2(0.0, 0.0);
    if (i > 0) {
      z_t dot = make_double2(0.0, 0.0);
      for (int rb = int(g / kRB); rb < a.nrb; ++rb) dot = zadd(dot, a.dotp[rb]);
      const z_t tp = a.tau[g - 1];
      alpha_prev = zscale(zmul(tp, dot), -0.5);
    }
    // row g of V and W (W(g, i-1) finalised here redundantly)
    if (!last) {
      for (int p = tid; p < i; p += blockDim.x) {
        z_t vgp = V[g + int64_t(p) * ldp];
        z_t wgp;
        if (p == i - 1) wgp = zadd(a.wtmp[g], zmul(alpha_prev, vgp));
        else wgp = W[g + int64_t(p) * ldp];
        wg[p] = wgp;
        vg[p] = vgp;
      }
    }
    __syncthreads();
    for (int rb = cta; rb < a.nrb; rb += G) {
      const int64_t r = int64_t(rb) * kRB + tid;
      const int64_t rlo = last ? g : g;  // rows >= g
      const bool valid = r < n && r >= rlo;
      z_t wprev = make_double2(0.0, 0.0);
      if (i > 0 && valid) {
        wprev = zadd(a.wtmp[r], zmul(alpha_prev, V[r + int64_t(i - 1) * ldp]));
        W[r + int64_t(i - 1) * ldp] = wprev;
        a.WV[r + int64_t(i - 1) * ldp] = wprev;
      }
      if (last) continue;
      z_t x = make_double2(0.0, 0.0);
      if (valid) {
        x = a.A[r + g * lda];
        for (int p = 0; p < i; ++p) {
          const z_t vrp = V[r + int64_t(p) * ldp];
          const z_t wrp = (p == i - 1) ? wprev : W[r + int64_t(p) * ldp];
          // x -= V(r,p) conj(W(g,p)) + W(r,p) conj(V(g,p))
          const z_t t1 = zmul(vrp, zconj(wg[p]));
          const z_t t2 = zmul(wrp, zconj(vg[p]));
          x = zsub(x, zadd(t1, t2));
        }
        if (r == g) {
          x.y = 0.0;
          a.d[g] = x.x;
        }
        a.A[r + g * lda] = x;
      }
      const bool inx = valid && r >= g + 2;
      xs[tid] = inx ? x : make_double2(0.0, 0.0);
      const double nrm = block_sum(inx ? zabs2(x) : 0.0, dred);
      if (tid == 0) a.normp[rb] = nrm;
      // s1[p] = sum conj(W(r,p)) x(r), s2[p] = sum conj(V(r,p)) x(r), r in this block
      for (int p = warp; p < i; p += kThreads / 32) {
        z_t s1 = make_double2(0.0, 0.0), s2 = make_double2(0.0, 0.0);
        for (int j = lane; j < kRB; j += 32) {
          const int64_t rr = int64_t(rb) * kRB + j;
          if (rr >= g + 2 && rr < n) {
            const z_t xv = xs[j];
            const z_t wv = (p == i - 1) ? zadd(a.wtmp[rr], zmul(alpha_prev, V[rr + int64_t(p) * ldp]))
                                        : W[rr + int64_t(p) * ldp];
            zcfma(s1, wv, xv);
            zcfma(s2, V[rr + int64_t(p) * ldp], xv);
          }
        }
        s1 = warp_zsum(s1);
        s2 = warp_zsum(s2);
        if (lane == 0) {
          a.s1p[int64_t(rb) * NB + p] = s1;
          a.s2p[int64_t(rb) * NB + p] = s2;
        }
      }
      __syncthreads();
    }
    if (last) break;
    grid.sync();
    // ------------------------------------------------------------------ phase 2
    if (g + 1 >= n) {
      // last column: no reflector; e/tau undefined
      grid.sync();
      grid.sync();
      continue;
    }
    double xn2 = 0.0;
    for (int rb = int(g / kRB); rb < a.nrb; ++rb) xn2 += a.normp[rb];
    const z_t alpha = a.A[(g + 1) + g * lda];
    double beta;
    z_t tau, scale;
    larfg_params(alpha, xn2, beta, tau, scale);
    if (cta == 0) {
      if (tid == 0) {
        a.e[g] = beta;
        a.tau[g] = tau;
      }
      // t1 = W^H v, t2 = V^H v over rows >= g+1 (v(g+1) = 1, v(r) = scale x(r))
      for (int p = tid; p < i; p += blockDim.x) {
        z_t s1 = make_double2(0.0, 0.0), s2 = make_double2(0.0, 0.0);
        for (int rb = int(g / kRB); rb < a.nrb; ++rb) {
          s1 = zadd(s1, a.s1p[int64_t(rb) * NB + p]);
          s2 = zadd(s2, a.s2p[int64_t(rb) * NB + p]);
        }
        const z_t w1 = W[(g + 1) + int64_t(p) * ldp];
        const z_t v1 = V[(g + 1) + int64_t(p) * ldp];
        a.t12[p] = zadd(zconj(w1), zmul(scale, s1));
        a.t12[NB + p] = zadd(zconj(v1), zmul(scale, s2));
      }
    }
    // reflector vector into the panels (own row blocks)
    for (int rb = cta; rb < a.nrb; rb += G) {
      const int64_t r = int64_t(rb) * kRB + tid;
      if (r < n) {
        z_t v = make_double2(0.0, 0.0);
        if (r == g + 1) v = make_double2(1.0, 0.0);
        else if (r >= g + 2) v = zmul(scale, a.A[r + g * lda]);
        V[r + int64_t(i) * ldp] = v;
        a.WV[r + int64_t(NB + i) * ldp] = v;
      }
    }
    // hemv over lower tiles of the trailing matrix rows/cols [g+1, n)
    {
      const int c0 = int((g + 1) / kT);
      const int K = a.nch - c0;
      const int64_t ntiles = int64_t(K) * (K + 1) / 2;
      for (int64_t t = cta; t < ntiles; t += G) {
        int bi = int((sqrt(8.0 * double(t) + 1.0) - 1.0) * 0.5);
        while (int64_t(bi + 1) * (bi + 2) / 2 <= t) ++bi;
        while (int64_t(bi) * (bi + 1) / 2 > t) --bi;
        const int bj = int(t - int64_t(bi) * (bi + 1) / 2);
        const int64_t R0 = int64_t(c0 + bi) * kT, C0 = int64_t(c0 + bj) * kT;
        const bool diag = (bi == bj);
        __syncthreads();
        // v over rows and cols of the tile
        if (tid < kT) {
          const int64_t r = R0 + tid;
          z_t v = make_double2(0.0, 0.0);
          if (r == g + 1) v = make_double2(1.0, 0.0);
          else if (r >= g + 2 && r < n) v = zmul(scale, a.A[r + g * lda]);
          vr[tid] = v;
        } else if (tid < 2 * kT) {
          const int64_t c = C0 + (tid - kT);
          z_t v = make_double2(0.0, 0.0);
          if (c == g + 1) v = make_double2(1.0, 0.0);
          else if (c >= g + 2 && c < n) v = zmul(scale, a.A[c + g * lda]);
          vc[tid - kT] = v;
        }
        // tile load (masked: rows/cols >= g+1, < n, lower incl. diagonal)
        for (int e = tid; e < kT * kT; e += kThreads) {
          const int rr = e % kT, cc = e / kT;
          const int64_t r = R0 + rr, c = C0 + cc;
          z_t val = make_double2(0.0, 0.0);
          if (r < n && c < n && c >= g + 1 && r >= g + 1 && r >= c) {
            val = a.A[r + c * lda];
            if (r == c) val.y = 0.0;
          }
          tile[rr + cc * (kT + 1)] = val;
        }
        __syncthreads();
        // y_R(r) = sum_c A(r,c) v(c) ; y_C(c) = sum_{r} conj(A(r,c)) v(r) (strictly lower if diag)
        const int q = tid >> 6, x = tid & 63;
        z_t yr = make_double2(0.0, 0.0), yc = make_double2(0.0, 0.0);
        for (int k = q * 16; k < q * 16 + 16; ++k) {
          zfma(yr, tile[x + k * (kT + 1)], vc[k]);
          if (!diag || k > x) zcfma(yc, tile[k + x * (kT + 1)], vr[k]);
        }
        red[q * kT + x] = yr;
        __syncthreads();
        if (q == 0) {
          z_t s = red[x];
          s = zadd(s, red[kT + x]);
          s = zadd(s, red[2 * kT + x]);
          s = zadd(s, red[3 * kT + x]);
          yr = s;
        }
        __syncthreads();
        red[q * kT + x] = yc;
        __syncthreads();
        if (q == 0) {
          z_t s = red[x];
          s = zadd(s, red[kT + x]);
          s = zadd(s, red[2 * kT + x]);
          s = zadd(s, red[3 * kT + x]);
          yc = s;
          const int gi = c0 + bi, gj = c0 + bj;
          if (diag) {
            a.Y[(int64_t(gi) * a.nch + gi) * kT + x] = zadd(yr, yc);
          } else {
            a.Y[(int64_t(gi) * a.nch + gj) * kT + x] = yr;
            a.Y[(int64_t(gj) * a.nch + gi) * kT + x] = yc;
          }
        }
      }
    }
    grid.sync();
    // ------------------------------------------------------------------ phase 3
    {
      const int c0 = int((g + 1) / kT);
      for (int rb = cta; rb < a.nrb; rb += G) {
        const int64_t r = int64_t(rb) * kRB + tid;
        const bool valid = r < n && r >= g + 1;
        z_t w = make_double2(0.0, 0.0), v = make_double2(0.0, 0.0);
        if (valid) {
          const int ch = int(r / kT), off = int(r % kT);
          z_t y = make_double2(0.0, 0.0);
          for (int b = c0; b < a.nch; ++b) y = zadd(y, a.Y[(int64_t(ch) * a.nch + b) * kT + off]);
          for (int p = 0; p < i; ++p) {
            y = zsub(y, zmul(V[r + int64_t(p) * ldp], a.t12[p]));
            y = zsub(y, zmul(W[r + int64_t(p) * ldp], a.t12[NB + p]));
          }
          w = zmul(tau, y);
          a.wtmp[r] = w;
          v = V[r + int64_t(i) * ldp];
          if (r >= g + 2) a.A[r + g * lda] = v;  // reflector storage below the subdiagonal
        }
        // dot partial: conj(w) v
        z_t pd = make_double2(0.0, 0.0);
        if (valid) zcfma(pd, w, v);
        pd = warp_zsum(pd);
        __syncthreads();
        if (lane == 0) zred[warp] = pd;
        __syncthreads();
        if (tid == 0) {
          z_t s = make_double2(0.0, 0.0);
          for (int ww = 0; ww < kThreads / 32; ++ww) s = zadd(s, zred[ww]);
          a.dotp[rb] = s;
        }
      }
    }
    grid.sync();
  }
}

__global__ void set_last_diag_kernel(const z_t* A, int64_t lda, int64_t n, double* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d[n - 1] = A[(n - 1) + (n - 1) * lda].x;
}

size_t hetrd_workspace_bytes(int64_t n) {
  const int64_t nb = kHetrdNB;
  const int64_t nch = ceil_div(n, kT), nrb = ceil_div(n, kRB);
  size_t z = 0;
  z += size_t(n) * 2 * nb * 2;           // VW, WV
  z += size_t(n);                        // wtmp
  z += size_t(nch) * nch * kT;           // Y
  z += size_t(nrb) * nb * 2;             // s1p, s2p
  z += size_t(2 * nb);                   // t12
  z += size_t(nrb);                      // dotp
  return z * sizeof(z_t) + size_t(nrb) * sizeof(double) + 256;
}

void zhetrd_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tau, void* ws) {
  if (n <= 0) return;
  const int nb = kHetrdNB;
  const int nch = int(ceil_div(n, kT)), nrb = int(ceil_div(n, kRB));
  z_t* base = reinterpret_cast<z_t*>(ws);
  HetrdArgs a{};
  a.A = A; a.lda = lda; a.n = n; a.d = d; a.e = e; a.tau = tau;
  a.ldp = n;
  a.VW = base; base += n * 2 * nb;
  a.WV = base; base += n * 2 * nb;
  a.wtmp = base; base += n;
  a.Y = base; base += int64_t(nch) * nch * kT;
  a.s1p = base; base += int64_t(nrb) * nb;
  a.s2p = base; base += int64_t(nrb) * nb;
  a.t12 = base; base += 2 * nb;
  a.dotp = base; base += nrb;
  a.normp = reinterpret_cast<double*>(base);
  a.nb = nb; a.nch = nch; a.nrb = nrb;

  const size_t smem = (size_t(kT) * (kT + 1) + 2 * kT + 4 * kT + 128 + kRB) * sizeof(z_t) +
                      32 * sizeof(double) + 8 * 64 * sizeof(z_t);
  static int blocks_per_sm = -1;
  static int num_sms = 0;
  if (blocks_per_sm < 0) {
    BSE_CUDA(cudaFuncSetAttribute(hetrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    int dev;
    BSE_CUDA(cudaGetDevice(&dev));
    BSE_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    BSE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, hetrd_panel_kernel,
                                                           kThreads, smem));
    if (blocks_per_sm < 1) throw std::runtime_error("hetrd: kernel cannot be resident");
  }
  const z_t mone = {-1.0, 0.0}, one = {1.0, 0.0};
  for (int64_t p0 = 0; p0 < n - 1; p0 += nb) {
    const int nbp = int(min64(nb, n - 1 - p0));
    BSE_CUDA(cudaMemsetAsync(a.VW, 0, sizeof(z_t) * size_t(n) * 2 * nb * 2, s));
    a.p0 = p0;
    a.nbp = nbp;
    // shrink the grid with the trailing size (fewer CTAs => cheaper grid barriers)
    const int64_t m = n - p0;
    const int64_t tiles = ceil_div(m, kT) * (ceil_div(m, kT) + 1) / 2;
    int G = int(min64(int64_t(blocks_per_sm) * num_sms, max64(tiles, ceil_div(m, kRB))));
    G = max(G, 1);
    void* args[] = {&a};
    double bytes = 0.0;  // algorithmic: lower triangle of each column's trailing matrix
    for (int i = 0; i < nbp; ++i) {
      const double mt = double(n - (p0 + i) - 1);
      bytes += 0.5 * mt * (mt + 1.0) * sizeof(z_t);
    }
    const int slot = g_timer ? timer_begin(s, 1, bytes) : -1;
    BSE_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(hetrd_panel_kernel), dim3(G),
                                         dim3(kThreads), args, smem, s));
    timer_end(s, slot);
    count_launch();
    const int64_t q = p0 + nbp;
    if (q < n) {
      zgemm(s, 0, 1, n - q, n - q, 2 * nb, mone, a.VW + q, n, a.WV + q, n, one, A + q + q * lda,
            lda, kGeneral, kGeneral, 1, nullptr, 0);
    }
  }
  set_last_diag_kernel<<<1, 32, 0, s>>>(A, lda, n, d);
  BSE_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------------
// Back-transformation  Z <- Q Z,  Q = H(0) H(1) ... H(n-2),  H(j) = I - tau_j v_j v_j^H with
// v_j(j+1) = 1 and v_j(j+2:n) stored in A(j+2:n, j)  (zunmtr 'L','L','N').
// Blocks of kBT reflectors, last block first:  Z <- (I - V T V^H) Z  with T from zlarft
// (forward, columnwise): three DMMA GEMMs + one small triangular kernel per block.
namespace {
constexpr int kBT = 64;
}

// Build the reflector block Vb (m x kb, explicit unit and zeros) for reflectors j0..j0+kb-1,
// covering rows off+j0 .. n-1 (row offset r = row - (j0+off)):
//   mode 0 (zhetrd 'L', off 1): v_j(j+1) = 1, v_j(r) = A(r, j)  for r > j+1
//   mode 1 (zgebrd Q,   off 0): v_j(j)   = 1, v_j(r) = A(r, j)  for r > j
//   mode 2 (zgebrd P,   off 1): u_j(j+1) = 1, u_j(c) = A(j, c)  for c > j+1 (row storage)
__global__ void build_v_kernel(const z_t* __restrict__ A, int64_t lda, int64_t n, int64_t j0,
                               int kb, int mode, z_t* __restrict__ Vb, int64_t ldv) {
  const int off = mode == 1 ? 0 : 1;
  const int64_t m = n - j0 - off;
  const int64_t total = m * kb;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e % m;
    const int c = int(e / m);
    const int64_t row = j0 + off + r;  // global row of the reflector vector
    const int64_t jc = j0 + c;         // reflector index
    const int64_t unit = jc + off;
    z_t v = make_double2(0.0, 0.0);
    if (row == unit) v = make_double2(1.0, 0.0);
    else if (row > unit) v = (mode == 2) ? A[jc + row * lda] : A[row + jc * lda];
    Vb[r + int64_t(c) * ldv] = v;
  }
}

// T (kb x kb upper) from the Gram matrix G = V^H V (kb x kb) and tau:
// T(i,i) = tau_i ; T(0:i,i) = -tau_i T(0:i,0:i) G(0:i,i).
__global__ void larft_kernel(const z_t* __restrict__ Gm, int kb, const z_t* __restrict__ tau,
                             z_t* __restrict__ T) {
  extern __shared__ __align__(16) unsigned char smraw[];
  z_t (*Ts)[kBT + 1] = reinterpret_cast<z_t (*)[kBT + 1]>(smraw);
  z_t* col = reinterpret_cast<z_t*>(smraw) + kBT * (kBT + 1);
  const int tid = threadIdx.x;
  for (int e = tid; e < kBT * kBT; e += blockDim.x) Ts[e % kBT][e / kBT] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = 0; i < kb; ++i) {
    const z_t ti = tau[i];
    if (tid < i) col[tid] = Gm[tid + int64_t(i) * kb];
    __syncthreads();
    if (tid < i) {
      z_t s = make_double2(0.0, 0.0);
      for (int k = tid; k < i; ++k) zfma(s, Ts[tid][k], col[k]);
      Ts[tid][i] = zscale(zmul(ti, s), -1.0);
    }
    if (tid == 0) Ts[i][i] = ti;
    __syncthreads();
  }
  for (int e = tid; e < kb * kb; e += blockDim.x) T[(e % kb) + int64_t(e / kb) * kb] = Ts[e % kb][e / kb];
}

size_t unmtr_workspace_bytes(int64_t n, int64_t ncols) {
  size_t z = size_t(n) * kBT            // Vb
             + size_t(kBT) * kBT * 2    // G, T
             + size_t(kBT) * ncols * 2  // W1, W2
             + size_t(32) * kBT * ncols;  // split-K partials
  return z * sizeof(z_t);
}

// Z <- H(0) H(1) ... H(nref-1) Z for the reflector family `mode` (see build_v_kernel).
void apply_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                      int64_t lda, const z_t* tau, z_t* Z, int64_t ldz, int64_t ncols, void* ws) {
  if (nref <= 0 || ncols <= 0) return;
  const int off = mode == 1 ? 0 : 1;
  z_t* Vb = reinterpret_cast<z_t*>(ws);
  z_t* Gm = Vb + n * kBT;
  z_t* T = Gm + kBT * kBT;
  z_t* W1 = T + kBT * kBT;
  z_t* W2 = W1 + int64_t(kBT) * ncols;
  z_t* part = W2 + int64_t(kBT) * ncols;
  const int64_t part_elems = int64_t(32) * kBT * ncols;
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0}, mone = {-1.0, 0.0};
  const int64_t nblk = ceil_div(nref, kBT);
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t j0 = b * kBT;
    const int kb = int(min64(kBT, nref - j0));
    const int64_t m = n - j0 - off;
    if (m <= 0) continue;
    {
      const int blocks = int(min64(ceil_div(m * kb, 256), 148 * 8));
      build_v_kernel<<<blocks, 256, 0, s>>>(A, lda, n, j0, kb, mode, Vb, m);
      BSE_LAUNCH_CHECK();
    }
    // G = V^H V
    zgemm(s, 1, 0, kb, kb, m, one, Vb, m, Vb, m, zero, Gm, kb, kGeneral, kGeneral, 0, part,
          part_elems);
    {
      const size_t sm = sizeof(z_t) * (kBT * (kBT + 1) + kBT);
      static bool configured = false;
      if (!configured) {
        BSE_CUDA(cudaFuncSetAttribute(larft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sm)));
        configured = true;
      }
      larft_kernel<<<1, 64, sm, s>>>(Gm, kb, tau + j0, T);
    }
    BSE_LAUNCH_CHECK();
    z_t* Zb = Z + (j0 + off);
    // W1 = V^H Z  (kb x ncols)
    zgemm(s, 1, 0, kb, ncols, m, one, Vb, m, Zb, ldz, zero, W1, kb, kGeneral, kGeneral, 0, part,
          part_elems);
    // W2 = T W1
    zgemm(s, 0, 0, kb, ncols, kb, one, T, kb, W1, kb, zero, W2, kb, kUpperOp, kGeneral, 0,
          nullptr, 0);
    // Z -= V W2
    zgemm(s, 0, 0, m, ncols, kb, mone, Vb, m, W2, kb, one, Zb, ldz, kGeneral, kGeneral, 0,
          nullptr, 0);
  }
}

void zunmtr_lower(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau, z_t* Z,
                  int64_t ldz, int64_t ncols, void* ws) {
  apply_reflectors(s, 0, n, n - 1, A, lda, tau, Z, ldz, ncols, ws);
}

}  // namespace bseg
