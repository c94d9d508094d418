// stedc.cu — symmetric tridiagonal eigensolver: Cuppen divide & conquer with
// Gu–Eisenstat eigenvectors, entirely on the GPU.
//
// Replaces the zstedc stage inside LAPACKE_zheevd (proj/src/backend.cpp:34; SURVEY §8a
// row a8.2) and, through the Golub–Kahan (TGK) embedding, the bidiagonal SVD inside
// zgesvd (row a9.3) — the reference's single-threaded zbdsqr rotation accumulation is the
// CPU hot spot the GPU design must not copy.
//
// Structure (all levels batched, no host synchronisation):
//   tear     : d[s-1], d[s] -= |e[s-1]| at every split point of a complete binary tree
//              whose 2^L leaves have <= 32 rows;
//   leaves   : one warp per leaf, implicit QL (tql2) computed redundantly by all lanes,
//              each lane owning one row of the leaf eigenvector block (no barriers);
//   merges   : per tree level, one batched launch per stage:
//              K1 prepare  : z from the boundary rows, merge of the two sorted halves,
//                            LAPACK dlaed2-style deflation (small z / close-pair Givens),
//                            column types (top-only / mixed / bottom-only);
//              K2 secular  : one warp per root, safeguarded "middle way" rational iteration
//                            (dlaed4 model) stored as (origin pole, offset) for accuracy;
//              K3 vectors  : Gu–Eisenstat z-hat (Löwner products), merged output order;
//              K4 U        : normalised secular eigenvectors, split by column type;
//              K5 GEMM     : grouped DMMA GEMM  Q_new = Q_old(:, type-ordered) * U
//                            (top and bottom halves separately — block structure halves
//                            the flops), epilogue scatters to the merged order;
//              K6 finish   : deflated columns + merged eigenvalues.
#include <algorithm>
#include <cfloat>
#include <vector>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"

namespace bseg {

namespace {
constexpr int kLeaf = 32;
constexpr double kEps = DBL_EPSILON * 0.5;  // LAPACK dlamch('Epsilon')
}  // namespace

struct MergeDesc {
  int s, n1, n2;
};

// Per-merge device state (indexed by merge id within a level).
struct MergeState {
  int K, k1, k2, k3, ndef;
  double rho;
};

struct StedcLevel {
  const MergeDesc* md;
  MergeState* ms;
  int nmerge;
  int64_t n;
  double* D;        // n: eigenvalues of the children (sorted per child) -> merged
  const double* E;  // n-1 original off-diagonal (scaled)
  double* Qold;     // n x n
  double* Qnew;     // n x n
  // scratch, indexed by absolute position s + local
  double* dl;       // dlamda (non-deflated poles, ascending)
  double* w;        // z components of the non-deflated
  int* ndcol;       // local column of each non-deflated entry
  int* ndtype;      // column type 1/2/3
  double* defval;   // deflated eigenvalues (ascending)
  int* defcol;      // their local columns
  int* orig;        // root origin (index into dl)
  double* tau;      // root offset from dl[orig]
  double* what;     // Gu–Eisenstat z-hat
  int* pos;         // merged output position of root j
  int* defpos;      // merged output position of deflated t
  int* rowT;        // type-ordered row of non-deflated i in the top GEMM (or -1)
  int* rowB;        // ... bottom GEMM
  int* acolT;       // absolute Q column for top-GEMM k index
  int* acolB;
  int* ccol;        // absolute output column for root j
  double* UT;       // (k1+k2) x K, ld n, column block at s
  double* UB;       // (k2+k3) x K
  int* info;
  int64_t keep_from;  // > 0 on the last level: output columns below it are not needed
};

// ----------------------------------------------------------------------------- setup
__global__ void stedc_scale_kernel(int64_t n, const double* d, const double* e, double* D,
                                   double* E, double* scale_out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(d[i]));
  for (int64_t i = threadIdx.x; i < n - 1; i += blockDim.x) m = fmax(m, fabs(e[i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  double mm = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) mm = fmax(mm, red[i]);
  const double sc = mm > 0.0 ? mm : 1.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) D[i] = d[i] / sc;
  for (int64_t i = threadIdx.x; i < n - 1; i += blockDim.x) E[i] = e[i] / sc;
  if (threadIdx.x == 0) *scale_out = sc;
}

// split points: s = start of every right child in the complete tree of depth L
__global__ void stedc_tear_kernel(int64_t n, int L, double* D, const double* E) {
  const int64_t nleaf = int64_t(1) << L;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nleaf;
       t += int64_t(gridDim.x) * blockDim.x) {
    if (t == 0) continue;
    const int64_t s = (t * n) >> L;  // leaf start = split point (every leaf start but 0)
    if (s <= 0 || s >= n) continue;
    const double b = fabs(E[s - 1]);
    D[s - 1] -= b;
    D[s] -= b;
  }
}

// One warp per leaf; tql2 with lanes = rows of the leaf eigenvector block.
__global__ void __launch_bounds__(128) stedc_leaf_kernel(int64_t n, int L, double* D,
                                                         const double* E, double* Q,
                                                         int* info) {
  __shared__ double zs[4][kLeaf][kLeaf + 1];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t leaf = int64_t(blockIdx.x) * 4 + wib;
  const int64_t nleaf = int64_t(1) << L;
  if (leaf >= nleaf) return;
  const int64_t s = (leaf * n) >> L, t = ((leaf + 1) * n) >> L;
  const int m = int(t - s);
  double d[kLeaf], e[kLeaf];
  for (int i = 0; i < kLeaf; ++i) {
    d[i] = i < m ? D[s + i] : 0.0;
    e[i] = (i < m - 1) ? E[s + i] : 0.0;
  }
  double (*z)[kLeaf + 1] = zs[wib];
  for (int j = 0; j < kLeaf; ++j) z[lane][j] = (lane == j) ? 1.0 : 0.0;
  __syncwarp();
  // implicit QL (EISPACK tql2 / Numerical Recipes tqli), e[i] couples i and i+1
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= DBL_EPSILON * dd) break;
      }
      if (mm != l) {
        if (iter++ == 90) {
          if (lane == 0) atomicCAS(info, 0, int(s + l + 1));
          break;
        }
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
        double sn = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          const double f = sn * e[i], b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          sn = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * sn + 2.0 * c * b;
          p = sn * r;
          d[i + 1] = g + p;
          g = c * r - b;
          // rotate columns i, i+1 of the eigenvector block (lane = row)
          const double zf = z[lane][i + 1];
          z[lane][i + 1] = sn * z[lane][i] + c * zf;
          z[lane][i] = c * z[lane][i] - sn * zf;
        }
        if (early) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  // selection sort ascending with column swaps
  for (int i = 0; i < m - 1; ++i) {
    int k = i;
    double p = d[i];
    for (int j = i + 1; j < m; ++j)
      if (d[j] < p) { k = j; p = d[j]; }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      const double tz = z[lane][i];
      z[lane][i] = z[lane][k];
      z[lane][k] = tz;
    }
  }
  __syncwarp();
  if (lane < m) {
    D[s + lane] = d[lane];
    for (int j = 0; j < m; ++j) Q[(s + lane) + (s + j) * n] = z[lane][j];
  }
}

// ----------------------------------------------------------------------------- K0 zero
// The previous level wrote only the diagonal blocks [s, s+n1)^2 and [s+n1, s+N)^2 of each
// merge; the off-diagonal blocks hold stale data of older levels (the two Q buffers
// alternate). Rotations (K1) and deflated-column copies (K6) read whole columns, so the
// off-diagonal blocks must be zero. grid = (chunks, merges).
__global__ void stedc_zero_offdiag_kernel(StedcLevel lv) {
  const MergeDesc md = lv.md[blockIdx.y];
  const int s = md.s, n1 = md.n1, n2 = md.n2;
  const int64_t n = lv.n;
  const int64_t blk = int64_t(n1) * n2;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < 2 * blk;
       e += int64_t(gridDim.x) * blockDim.x) {
    if (e < blk) {  // rows of the right child in columns of the left child
      const int64_t i = e % n2, j = e / n2;
      lv.Qold[(s + n1 + i) + (s + j) * n] = 0.0;
    } else {        // rows of the left child in columns of the right child
      const int64_t f = e - blk;
      const int64_t i = f % n1, j = f / n1;
      lv.Qold[(s + i) + (s + n1 + j) * n] = 0.0;
    }
  }
}

// ----------------------------------------------------------------------------- K1 prepare
// One CTA per merge. Parallel: z from the boundary rows, merge ranks of the two sorted
// halves, gathers into sorted order. Sequential (thread 0, contiguous L1-friendly reads):
// the dlaed2 deflation scan. Parallel again: Givens rotations of Q columns (in order) and
// the type-ordered row maps of the two half GEMMs (block prefix sums).
__global__ void __launch_bounds__(256) stedc_prepare_kernel(StedcLevel lv) {
  const int mid = blockIdx.x;
  const MergeDesc md = lv.md[mid];
  const int s = md.s, n1 = md.n1, n2 = md.n2, N = n1 + n2;
  const int64_t n = lv.n;
  const double* D = lv.D + s;
  double* Q = lv.Qold;
  // scratch (absolute offset s), all overwritten by later stages of the same level:
  double* zs = lv.what + s;     // z in sorted order
  double* ds = lv.tau + s;      // D in sorted order
  int* perm = lv.pos + s;       // sorted index -> local column
  int* rot_a = lv.defpos + s;   // rotation pairs (local columns)
  int* rot_b = lv.orig + s;
  double* rot_c = lv.UT + int64_t(s) * n;  // UT/UB column s: rewritten by K4
  double* rot_s = lv.UB + int64_t(s) * n;
  const double beta = lv.E[s + n1 - 1];
  const double sigma = beta >= 0.0 ? 1.0 : -1.0;
  const double rinv2 = 0.70710678118654752440;
  // merge ranks (stable: ties -> left half first), then gather D and z in sorted order
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    const double x = D[c];
    int rank;
    if (c < n1) {
      int lo = 0, hi = n2;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (D[n1 + m] < x) lo = m + 1; else hi = m; }
      rank = c + lo;
    } else {
      int lo = 0, hi = n1;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (D[m] <= x) lo = m + 1; else hi = m; }
      rank = (c - n1) + lo;
    }
    const double zv = (c < n1) ? Q[(s + n1 - 1) + int64_t(s + c) * n]
                               : sigma * Q[(s + n1) + int64_t(s + c) * n];
    perm[rank] = c;
    ds[rank] = x;
    zs[rank] = zv * rinv2;
  }
  __shared__ int sh_npairs, sh_K, sh_ndef;
  __shared__ double sh_rho, sh_max[32];
  __syncthreads();
  {  // max(|D|, |z|) over the merge: block-parallel (max is order independent)
    double mx = 0.0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) mx = fmax(mx, fmax(fabs(ds[j]), fabs(zs[j])));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) sh_max[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double rho = 2.0 * fabs(beta);
    double dzmax = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) dzmax = fmax(dzmax, sh_max[w]);
    const double tol = 8.0 * kEps * dzmax;
    int K = 0, ndef = 0, npairs = 0;
    double* dl = lv.dl + s;
    double* w = lv.w + s;
    int* ndcol = lv.ndcol + s;
    int* ndtype = lv.ndtype + s;
    double* defval = lv.defval + s;
    int* defcol = lv.defcol + s;
    double lastdef = -DBL_MAX;
    auto push_def = [&](double val, int col) {
      if (val >= lastdef) {
        defval[ndef] = val;
        defcol[ndef] = col;
        ++ndef;
        lastdef = val;
        return;
      }
      int t = ndef++;
      while (t > 0 && defval[t - 1] > val) {
        defval[t] = defval[t - 1];
        defcol[t] = defcol[t - 1];
        --t;
      }
      defval[t] = val;
      defcol[t] = col;
    };
    int pj = -1, tpj = 0;
    double dpj = 0.0, zpj = 0.0;
    // The scan is inherently sequential; its inputs are streamed through registers in
    // chunks of kCh (fully unrolled, so no local memory), the next chunk's loads issued before
    // the current chunk is processed.
    constexpr int kCh = 8;
    auto step = [&](int nj, double dnj, double znj) {
      const int tnj = nj < n1 ? 1 : 3;
      if (rho * fabs(znj) <= tol) {
        push_def(dnj, nj);
        return;
      }
      if (pj < 0) {
        pj = nj; dpj = dnj; zpj = znj; tpj = tnj;
        return;
      }
      const double t = dnj - dpj;
      // dlaed2's close-pair test |t c s| <= tol with c = z_j / tau, s = -z_p / tau equals
      // |t z_j z_p| <= tol (z_j^2 + z_p^2); that cheap form (no hypot / divisions on the
      // sequential path) screens out the pairs that are clearly not deflated, the exact
      // LAPACK arithmetic decides the rest.
      const double zz = znj * znj + zpj * zpj;
      if (fabs(t * znj * zpj) > 2.0 * tol * zz) {
        dl[K] = dpj; w[K] = zpj; ndcol[K] = pj; ndtype[K] = tpj;
        ++K;
        pj = nj; dpj = dnj; zpj = znj; tpj = tnj;
        return;
      }
      const double tau = hypot(znj, zpj);
      const double cv = znj / tau, sv = -zpj / tau;
      if (fabs(t * cv * sv) <= tol) {
        rot_a[npairs] = pj;
        rot_b[npairs] = nj;
        rot_c[npairs] = cv;
        rot_s[npairs] = sv;
        ++npairs;
        const double tnew = dpj * cv * cv + dnj * sv * sv;
        const double dsurv = dpj * sv * sv + dnj * cv * cv;
        push_def(tnew, pj);
        tpj = (tnj != tpj) ? 2 : tnj;
        pj = nj; dpj = dsurv; zpj = tau;
      } else {
        dl[K] = dpj; w[K] = zpj; ndcol[K] = pj; ndtype[K] = tpj;
        ++K;
        pj = nj; dpj = dnj; zpj = znj; tpj = tnj;
      }
    };
    int cn[kCh], xn[kCh];
    double cd[kCh], cz[kCh], xd[kCh], xz[kCh];
#pragma unroll
    for (int u = 0; u < kCh; ++u) {
      cn[u] = u < N ? perm[u] : 0;
      cd[u] = u < N ? ds[u] : 0.0;
      cz[u] = u < N ? zs[u] : 0.0;
    }
    for (int j0 = 0; j0 < N; j0 += kCh) {
#pragma unroll
      for (int u = 0; u < kCh; ++u) {  // next chunk in flight
        const int jj = j0 + kCh + u;
        xn[u] = jj < N ? perm[jj] : 0;
        xd[u] = jj < N ? ds[jj] : 0.0;
        xz[u] = jj < N ? zs[jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kCh; ++u)
        if (j0 + u < N) step(cn[u], cd[u], cz[u]);
#pragma unroll
      for (int u = 0; u < kCh; ++u) {
        cn[u] = xn[u];
        cd[u] = xd[u];
        cz[u] = xz[u];
      }
    }
    if (pj >= 0) {
      dl[K] = dpj; w[K] = zpj; ndcol[K] = pj; ndtype[K] = tpj;
      ++K;
    }
    sh_npairs = npairs;
    sh_K = K;
    sh_ndef = ndef;
    sh_rho = rho;
  }
  __syncthreads();
  // rotations of Q columns (rows s .. s+N), in discovery order
  const int npairs = sh_npairs;
  for (int r = 0; r < npairs; ++r) {
    const int64_t ca = s + rot_a[r], cb = s + rot_b[r];
    const double c = rot_c[r], sn = rot_s[r];
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double x = Q[(s + i) + ca * n], y = Q[(s + i) + cb * n];
      Q[(s + i) + ca * n] = c * x + sn * y;
      Q[(s + i) + cb * n] = c * y - sn * x;
    }
    __syncthreads();
  }
  // type-ordered row maps via a block prefix count: top = [type1 | type2], bottom = [type2 | type3]
  const int K = sh_K;
  __shared__ int cnt[3][257];
  const int T = blockDim.x;
  const int seg = (K + T - 1) / T;
  const int b0 = min(K, int(threadIdx.x) * seg), b1 = min(K, b0 + seg);
  int c1 = 0, c2 = 0, c3 = 0;
  for (int i = b0; i < b1; ++i) {
    const int ty = lv.ndtype[s + i];
    c1 += ty == 1; c2 += ty == 2; c3 += ty == 3;
  }
  cnt[0][threadIdx.x + 1] = c1;
  cnt[1][threadIdx.x + 1] = c2;
  cnt[2][threadIdx.x + 1] = c3;
  if (threadIdx.x == 0) { cnt[0][0] = cnt[1][0] = cnt[2][0] = 0; }
  __syncthreads();
  if (threadIdx.x < 3) {
    int acc = 0;
    for (int t = 0; t <= T; ++t) { acc += cnt[threadIdx.x][t]; cnt[threadIdx.x][t] = acc; }
  }
  __syncthreads();
  const int k1 = cnt[0][T], k2 = cnt[1][T], k3 = cnt[2][T];
  int o1 = cnt[0][threadIdx.x], o2 = cnt[1][threadIdx.x], o3 = cnt[2][threadIdx.x];
  for (int i = b0; i < b1; ++i) {
    const int ty = lv.ndtype[s + i];
    const int col = s + lv.ndcol[s + i];
    int rt = -1, rb = -1;
    if (ty == 1) { rt = o1++; }
    else if (ty == 2) { rt = k1 + o2; rb = o2; ++o2; }
    else { rb = k2 + o3++; }
    lv.rowT[s + i] = rt;
    lv.rowB[s + i] = rb;
    if (rt >= 0) lv.acolT[s + rt] = col;
    if (rb >= 0) lv.acolB[s + rb] = col;
  }
  if (threadIdx.x == 0) {
    MergeState st;
    st.K = K; st.k1 = k1; st.k2 = k2; st.k3 = k3; st.ndef = sh_ndef; st.rho = sh_rho;
    lv.ms[mid] = st;
  }
}

// ----------------------------------------------------------------------------- K2 secular
// f(tau) = 1/rho + sum_i w_i^2 / (Delta_i - tau),  Delta_i = dl_i - dl_origin.
__device__ __forceinline__ void secular_sums(const double* dl, const double* w, int K, int o,
                                             double tau, int split, double& psi, double& dpsi,
                                             double& phi, double& dphi, double& aerr) {
  // split: terms i <= split go to psi, i > split to phi. Warp-parallel.
  const int lane = threadIdx.x & 31;
  double p = 0.0, dp = 0.0, f = 0.0, df = 0.0, er = 0.0;
  const double dlo = dl[o];
  for (int i = lane; i < K; i += 32) {
    const double del = (dl[i] - dlo) - tau;
    const double t = w[i] / del;
    const double term = w[i] * t;
    if (i <= split) {
      p += term;
      dp += t * t;
    } else {
      f += term;
      df += t * t;
    }
    er += fabs(term);
  }
  psi = warp_sum(p);
  dpsi = warp_sum(dp);
  phi = warp_sum(f);
  dphi = warp_sum(df);
  aerr = warp_sum(er);
}

__global__ void __launch_bounds__(256) stedc_secular_kernel(StedcLevel lv) {
  const int mid = blockIdx.y;
  const MergeDesc md = lv.md[mid];
  const MergeState st = lv.ms[mid];
  const int K = st.K;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= K) return;
  const int s = md.s;
  const double* dl = lv.dl + s;
  const double* w = lv.w + s;
  const double rho = st.rho, rhoinv = 1.0 / rho;
  int o;
  double tau, lo, hi;
  if (K == 1) {
    if (lane == 0) {
      lv.orig[s] = 0;
      lv.tau[s] = rho * w[0] * w[0];
    }
    return;
  }
  if (j < K - 1) {
    const double del = dl[j + 1] - dl[j];
    const double midpt = 0.5 * del;
    // f at the midpoint (origin j), split so the two nearest poles are separated
    double psi, dpsi, phi, dphi, aerr;
    secular_sums(dl, w, K, j, midpt, j, psi, dpsi, phi, dphi, aerr);
    const double fmid = rhoinv + psi + phi;
    // two-pole initial guess (dlaed4): C = rest of f at midpt
    const double wj2 = w[j] * w[j], wj12 = w[j + 1] * w[j + 1];
    const double C = fmid - wj2 / (-midpt) - wj12 / (del - midpt);
    if (fmid >= 0.0) {
      o = j;
      lo = 0.0;
      hi = midpt;
      const double A = C * del + wj2 + wj12, B = wj2 * del;
      const double disc = sqrt(fabs(A * A - 4.0 * B * C));
      tau = A > 0.0 ? 2.0 * B / (A + disc) : (A - disc) / (2.0 * C);
    } else {
      o = j + 1;
      lo = -midpt;
      hi = 0.0;
      const double A = -C * del + wj2 + wj12, B = wj12 * del;
      const double disc = sqrt(fabs(A * A + 4.0 * B * C));
      tau = A > 0.0 ? -2.0 * B / (A + disc) : -(A + disc) / (2.0 * C);
    }
    if (!(tau > lo && tau < hi)) tau = 0.5 * (lo + hi);
    // iterate: psi = terms i <= j, phi = terms i > j
    for (int it = 0; it < 200; ++it) {
      secular_sums(dl, w, K, o, tau, j, psi, dpsi, phi, dphi, aerr);
      const double f = rhoinv + psi + phi;
      const double dw = dpsi + dphi;
      const double erretm = 8.0 * aerr + 2.0 * rhoinv + 3.0 * fabs(tau) * dw;
      if (fabs(f) <= kEps * erretm) break;
      if (f < 0.0) lo = fmax(lo, tau); else hi = fmin(hi, tau);
      if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) && it > 0) break;
      const double dj = (dl[j] - dl[o]) - tau;      // delta(i)   < 0
      const double dj1 = (dl[j + 1] - dl[o]) - tau; // delta(i+1) > 0
      double Cc;
      if (o == j) Cc = f - dj1 * dw - (dj - dj1) * (w[j] / dj) * (w[j] / dj);
      else Cc = f - dj * dw - (dj1 - dj) * (w[j + 1] / dj1) * (w[j + 1] / dj1);
      double A = (dj + dj1) * f - dj * dj1 * dw;
      const double B = dj * dj1 * f;
      double eta;
      if (Cc == 0.0) {
        if (A == 0.0) {
          A = (o == j) ? w[j] * w[j] + dj1 * dj1 * dw : w[j + 1] * w[j + 1] + dj * dj * dw;
        }
        eta = B / A;
      } else if (A <= 0.0) {
        eta = (A - sqrt(fabs(A * A - 4.0 * B * Cc))) / (2.0 * Cc);
      } else {
        eta = 2.0 * B / (A + sqrt(fabs(A * A - 4.0 * B * Cc)));
      }
      if (f * eta >= 0.0) eta = -f / dw;
      double tn = tau + eta;
      if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
      if (tn == tau) break;
      tau = tn;
    }
  } else {
    // last root: (dl[K-1], dl[K-1] + rho*|w|^2]
    o = K - 1;
    double wn2 = 0.0;
    for (int i = lane; i < K; i += 32) wn2 += w[i] * w[i];
    wn2 = warp_sum(wn2);
    lo = 0.0;
    hi = rho * wn2;
    tau = 0.5 * hi;
    double psi, dpsi, phi, dphi, aerr;
    for (int it = 0; it < 200; ++it) {
      secular_sums(dl, w, K, o, tau, K - 2, psi, dpsi, phi, dphi, aerr);
      // psi: terms i < K-1 ; phi: the pole term i = K-1
      const double f = rhoinv + psi + phi;
      const double dw = dpsi + dphi;
      const double erretm = 8.0 * aerr + 2.0 * rhoinv + 3.0 * fabs(tau) * dw;
      if (fabs(f) <= kEps * erretm) break;
      if (f < 0.0) lo = fmax(lo, tau); else hi = fmin(hi, tau);
      if (hi - lo <= 2.0 * DBL_EPSILON * fabs(hi) && it > 0) break;
      // model: c + S/(a - x) - wl^2/x, a = Delta_{K-2} - ... (in tau coordinates)
      const double a = (dl[K - 2] - dl[o]) - tau;  // < 0
      const double wl2 = w[K - 1] * w[K - 1];
      const double S = a * a * dpsi;
      const double c = rhoinv + psi - S / a;
      // solve c + S/(a - x) - wl2/(-tau - x)... in eta: pole term wl2/(-(tau+eta))
      // equation in eta: c + S/(a - eta) + wl2/(-tau - eta) = 0
      const double b0 = -tau;  // pole distance for the last term (delta_{K-1} = -tau)
      // c (a-eta)(b0-eta) + S (b0-eta) + wl2 (a-eta) = 0
      // c eta^2 - (c(a+b0) + S + wl2) eta + (c a b0 + S b0 + wl2 a) = 0
      const double qa = c, qb = -(c * (a + b0) + S + wl2), qc = c * a * b0 + S * b0 + wl2 * a;
      double eta;
      if (qa == 0.0) {
        eta = -qc / qb;
      } else {
        const double disc = sqrt(fabs(qb * qb - 4.0 * qa * qc));
        // numerically stable roots; take the one closest to zero (a correction)
        const double q = -0.5 * (qb + copysign(disc, qb));
        const double e1 = q / qa, e2 = (q != 0.0) ? qc / q : e1;
        eta = fabs(e1) < fabs(e2) ? e1 : e2;
      }
      if (f * eta >= 0.0 || !isfinite(eta)) eta = -f / dw;
      double tn = tau + eta;
      if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
      if (tn == tau) break;
      tau = tn;
    }
  }
  if (lane == 0) {
    lv.orig[s + j] = o;
    lv.tau[s + j] = tau;
  }
}

// ----------------------------------------------------------------------------- K3 z-hat
__global__ void __launch_bounds__(256) stedc_zhat_kernel(StedcLevel lv) {
  const int mid = blockIdx.y;
  const MergeDesc md = lv.md[mid];
  const MergeState st = lv.ms[mid];
  const int K = st.K, s = md.s, N = md.n1 + md.n2;
  const int warps = blockDim.x >> 5;
  const int i = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const double* dl = lv.dl + s;
  const int* orig = lv.orig + s;
  const double* tau = lv.tau + s;
  if (i < K) {
    // W(i) = Delta_ii * prod_{j != i} Delta_ij / (dl_i - dl_j);  zhat = sign(w_i) sqrt(-W)
    double prod = 1.0;
    for (int j = lane; j < K; j += 32) {
      const double dij = (dl[i] - dl[orig[j]]) - tau[j];
      prod *= (j == i) ? dij : dij / (dl[i] - dl[j]);
    }
    warp_converge();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, o);
    if (lane == 0) {
      const double v = sqrt(fabs(prod));
      lv.what[s + i] = copysign(v, lv.w[s + i]);
      // merged position of root i: i + #(deflated < lambda_i)
      const double lam = dl[orig[i]] + tau[i];
      const double* dv = lv.defval + s;
      int lo = 0, hi = st.ndef;
      while (lo < hi) { const int m = (lo + hi) >> 1; if (dv[m] < lam) lo = m + 1; else hi = m; }
      lv.pos[s + i] = i + lo;
      lv.ccol[s + i] = s + i + lo;
    }
  }
  // deflated positions: t + #(lambda <= def_t)
  const int tt = blockIdx.x * blockDim.x + threadIdx.x;
  if (tt < st.ndef && tt < N) {
    const double v = lv.defval[s + tt];
    int lo = 0, hi = K;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      const double lam = dl[orig[m]] + tau[m];
      if (lam <= v) lo = m + 1; else hi = m;
    }
    lv.defpos[s + tt] = tt + lo;
  }
}

// ----------------------------------------------------------------------------- K4 U
// Column j of the secular eigenvector matrix: u_ij = zhat_i / Delta_ij, normalised.
__global__ void __launch_bounds__(256) stedc_u_kernel(StedcLevel lv) {
  const int mid = blockIdx.y;
  const MergeDesc md = lv.md[mid];
  const MergeState st = lv.ms[mid];
  const int K = st.K, s = md.s;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= K) return;
  const double* dl = lv.dl + s;
  const double dlo = dl[lv.orig[s + j]];
  const double tj = lv.tau[s + j];
  double nrm = 0.0;
  for (int i = lane; i < K; i += 32) {
    const double u = lv.what[s + i] / ((dl[i] - dlo) - tj);
    nrm += u * u;
  }
  nrm = warp_sum(nrm);
  const double rn = 1.0 / sqrt(nrm);
  const int64_t n = lv.n;
  for (int i = lane; i < K; i += 32) {
    const double u = lv.what[s + i] / ((dl[i] - dlo) - tj) * rn;
    const int rt = lv.rowT[s + i], rb = lv.rowB[s + i];
    if (rt >= 0) lv.UT[rt + int64_t(s + j) * n] = u;
    if (rb >= 0) lv.UB[rb + int64_t(s + j) * n] = u;
  }
}

// ----------------------------------------------------------------------------- K5 GEMM
// Grouped real DMMA GEMM over all merges of a level: problem 2*mid (top rows) and
// 2*mid+1 (bottom rows). A columns gathered through acol, C columns scattered via ccol.
namespace {
constexpr int gBM = 64, gBN = 64, gBK = 16, gWM = 32, gWN = 32, gST = 3;
using GT = DGemmTile<gBM, gBN, gBK, gWM, gWN, gST>;
}

__global__ void __launch_bounds__(GT::NTHREADS) stedc_gemm_kernel(StedcLevel lv,
                                                                  const int* __restrict__ tile_off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  // locate problem: tile_off has nmerge*2+1 prefix entries
  const int nprob = lv.nmerge * 2;
  int lo = 0, hi = nprob;
  const int bid = blockIdx.x;
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (tile_off[m] <= bid) lo = m; else hi = m;
  }
  const int prob = lo, mid = prob >> 1, half = prob & 1;
  const MergeDesc md = lv.md[mid];
  const MergeState st = lv.ms[mid];
  const int s = md.s;
  const int64_t n = lv.n;
  const int rows = half ? md.n2 : md.n1;
  const int ncols = st.K;
  const int kdim = half ? (st.k2 + st.k3) : (st.k1 + st.k2);
  const int local = bid - tile_off[prob];
  const int tiles_m = (rows + gBM - 1) / gBM;
  const int tm = local % tiles_m, tn = local / tiles_m;
  const int64_t m0 = int64_t(tm) * gBM, n0 = int64_t(tn) * gBN;
  if (n0 >= ncols) return;
  // Wanted columns only (e.g. the positive half of the TGK spectrum): roots are ascending and
  // their merged positions monotone, so the unwanted roots are a prefix j < jlo.
  int jlo = 0;
  if (lv.keep_from > s) {
    int lo2 = 0, hi2 = ncols;  // first j with s + pos[s + j] >= keep_from
    while (lo2 < hi2) {
      const int m = (lo2 + hi2) >> 1;
      if (s + lv.pos[s + m] >= lv.keep_from) hi2 = m; else lo2 = m + 1;
    }
    jlo = lo2;
    if (n0 + gBN <= jlo) return;
  }
  const double* A = lv.Qold + (s + (half ? md.n1 : 0));
  const int* acol = half ? (lv.acolB + s) : (lv.acolT + s);
  const double* B = (half ? lv.UB : lv.UT) + int64_t(s) * n;  // ld n
  double* C = lv.Qnew + (s + (half ? md.n1 : 0));
  const int* ccol = lv.ccol + s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / GT::WARPS_N) * gWM, wn0 = (warp % GT::WARPS_N) * gWN;
  const int64_t ktiles = (kdim + gBK - 1) / gBK;
  auto load_stage = [&](int stage, int64_t kt) {
    double* As = smem + stage * GT::STAGE_ELEMS;
    double* Bs = As + GT::A_ELEMS;
    const int64_t k0 = kt * gBK;
#pragma unroll
    for (int r = 0; r < (gBM * gBK) / GT::NTHREADS; ++r) {
      const int e = tid + r * GT::NTHREADS;
      const int i = e % gBM, kk = e / gBM;
      const int64_t gi = m0 + i, gk = k0 + kk;
      const bool ok = gi < rows && gk < kdim;
      const double* src = ok ? A + gi + int64_t(acol[gk]) * n : A;
      cp_async8(As + kk * GT::A_LD + i, src, ok);
    }
#pragma unroll
    for (int r = 0; r < (gBN * gBK) / GT::NTHREADS; ++r) {
      const int e = tid + r * GT::NTHREADS;
      const int kk = e % gBK, j = e / gBK;
      const int64_t gj = n0 + j, gk = k0 + kk;
      const bool ok = gj < ncols && gk < kdim;
      cp_async8(Bs + j * GT::B_LD + kk, ok ? B + gk + gj * n : B, ok);
    }
  };
  double acc[GT::MT][GT::NT][2];
#pragma unroll
  for (int a = 0; a < GT::MT; ++a)
#pragma unroll
    for (int b = 0; b < GT::NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int st2 = 0; st2 < gST - 1; ++st2) {
    if (st2 < ktiles) load_stage(st2, st2);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<gST - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + gST - 1;
      if (nk < ktiles) load_stage(int(nk % gST), nk);
      cp_async_commit();
    }
    const double* As = smem + int(kt % gST) * GT::STAGE_ELEMS;
    const double* Bs = As + GT::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < gBK; ks += 4) {
      double av[GT::MT], bv[GT::NT];
#pragma unroll
      for (int a = 0; a < GT::MT; ++a) av[a] = As[(ks + fk) * GT::A_LD + wm0 + a * 8 + fr];
#pragma unroll
      for (int b = 0; b < GT::NT; ++b) bv[b] = Bs[(wn0 + b * 8 + fr) * GT::B_LD + ks + fk];
#pragma unroll
      for (int a = 0; a < GT::MT; ++a)
#pragma unroll
        for (int b = 0; b < GT::NT; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < GT::MT; ++a)
#pragma unroll
    for (int b = 0; b < GT::NT; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = m0 + wm0 + a * 8 + fr;
        const int64_t gj = n0 + wn0 + b * 8 + 2 * fk + h;
        if (gi >= rows || gj >= ncols || gj < jlo) continue;
        C[gi + int64_t(ccol[gj]) * n] = acc[a][b][h];
      }
}

// ----------------------------------------------------------------------------- K6 finish
__global__ void stedc_finish_kernel(StedcLevel lv) {
  const int mid = blockIdx.y;
  const MergeDesc md = lv.md[mid];
  const MergeState st = lv.ms[mid];
  const int s = md.s, N = md.n1 + md.n2;
  const int64_t n = lv.n;
  // deflated columns: copy Q_old column (already rotated) into merged position
  for (int t = blockIdx.x; t < st.ndef; t += gridDim.x) {
    const int src = s + lv.defcol[s + t];
    const int dst = s + lv.defpos[s + t];
    for (int i = threadIdx.x; i < N; i += blockDim.x)
      lv.Qnew[(s + i) + int64_t(dst) * n] = lv.Qold[(s + i) + int64_t(src) * n];
  }
  if (blockIdx.x == 0) {
    __syncthreads();
    // eigenvalues (D read in K1 only; safe to overwrite now)
    for (int j = threadIdx.x; j < st.K; j += blockDim.x)
      lv.D[s + lv.pos[s + j]] = lv.dl[s + lv.orig[s + j]] + lv.tau[s + j];
    for (int t = threadIdx.x; t < st.ndef; t += blockDim.x) lv.D[s + lv.defpos[s + t]] = lv.defval[s + t];
  }
}

__global__ void stedc_unscale_kernel(int64_t n, const double* D, const double* scale, double* d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = D[i] * (*scale);
}

// ----------------------------------------------------------------------------- driver
size_t stedc_workspace_bytes(int64_t n) {
  const size_t nn = size_t(n) * size_t(n);
  size_t b = 0;
  b += nn * sizeof(double) * 3;          // Qalt, UT, UB
  b += size_t(n) * sizeof(double) * 8;   // D, E, dl, w, defval, tau, what, scale
  b += size_t(n) * sizeof(int) * 13;     // index arrays
  b += size_t(2 * n + 2) * sizeof(MergeDesc) + size_t(n) * sizeof(MergeState) + 4096;
  b += size_t(4 * n + 130) * sizeof(int);  // tile offsets of every level
  return b + 64 * 16;
}

namespace {
template <typename T>
T* carve(char*& p, size_t count) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15);
  T* r = reinterpret_cast<T*>(a);
  p = reinterpret_cast<char*>(a + count * sizeof(T));
  return r;
}
}  // namespace

void dstedc(cudaStream_t s, int64_t n, double* d, const double* e, double* Q, void* ws,
            int* d_info, int64_t keep_from) {
  BSE_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int), s));
  if (n <= 0) return;
  char* p = reinterpret_cast<char*>(ws);
  const size_t nn = size_t(n) * size_t(n);
  double* Qalt = carve<double>(p, nn);
  double* UT = carve<double>(p, nn);
  double* UB = carve<double>(p, nn);
  double* D = carve<double>(p, n);
  double* E = carve<double>(p, n);
  double* dl = carve<double>(p, n);
  double* w = carve<double>(p, n);
  double* defval = carve<double>(p, n);
  double* tau = carve<double>(p, n);
  double* what = carve<double>(p, n);
  double* scale = carve<double>(p, 2);
  int* ndcol = carve<int>(p, n);
  int* ndtype = carve<int>(p, n);
  int* defcol = carve<int>(p, n);
  int* orig = carve<int>(p, n);
  int* pos = carve<int>(p, n);
  int* defpos = carve<int>(p, n);
  int* rowT = carve<int>(p, n);
  int* rowB = carve<int>(p, n);
  int* acolT = carve<int>(p, 2 * n);
  int* acolB = carve<int>(p, n);
  int* ccol = carve<int>(p, n);
  MergeDesc* mdesc_all = carve<MergeDesc>(p, 2 * n + 2);  // every level's merges
  MergeState* mstate = carve<MergeState>(p, n);
  int* tile_off_all = carve<int>(p, 4 * n + 130);

  stedc_scale_kernel<<<1, 1024, 0, s>>>(n, d, e, D, E, scale);
  BSE_LAUNCH_CHECK();
  int L = 0;
  while ((n >> L) > kLeaf || ((n + (int64_t(1) << L) - 1) >> L) > kLeaf) ++L;
  const int64_t nleaf = int64_t(1) << L;
  // Q buffers: level parity decides which buffer the leaves write so the final level lands
  // in Q (the caller's output).
  double* bufs[2] = {Q, Qalt};
  int cur = (L % 2 == 0) ? 0 : 1;
  BSE_CUDA(cudaMemsetAsync(bufs[cur], 0, nn * sizeof(double), s));
  if (L > 0) {
    stedc_tear_kernel<<<unsigned(ceil_div(nleaf, 256)), 256, 0, s>>>(n, L, D, E);
    BSE_LAUNCH_CHECK();
  }
  stedc_leaf_kernel<<<unsigned(ceil_div(nleaf, 4)), 128, 0, s>>>(n, L, D, E, bufs[cur], d_info);
  BSE_LAUNCH_CHECK();

  const bool& configured = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    BSE_CUDA(cudaFuncSetAttribute(stedc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(GT::SMEM)));
    return true;
  });
  (void)configured;
  // Every level's merge descriptors and GEMM tile offsets are built up front and go to the
  // device in one copy each (no host synchronisation inside the tree).
  std::vector<MergeDesc> hmd;
  std::vector<int> htile;
  std::vector<int> lvl_md(size_t(std::max(L, 1))), lvl_tile(size_t(std::max(L, 1))),
      lvl_maxn(size_t(std::max(L, 1)));
  for (int lvl = L - 1; lvl >= 0; --lvl) {
    const int nm = 1 << lvl;
    const int md0 = int(hmd.size()), t0 = int(htile.size());
    lvl_md[size_t(lvl)] = md0;
    lvl_tile[size_t(lvl)] = t0;
    htile.resize(size_t(t0 + 2 * nm + 1), 0);
    int maxN = 0;
    for (int m = 0; m < nm; ++m) {
      const int64_t a = (int64_t(m) * n) >> lvl;
      const int64_t mid = (int64_t(2 * m + 1) * n) >> (lvl + 1);
      const int64_t b = (int64_t(m + 1) * n) >> lvl;
      hmd.push_back(MergeDesc{int(a), int(mid - a), int(b - mid)});
      maxN = std::max<int>(maxN, int(b - a));
    }
    lvl_maxn[size_t(lvl)] = maxN;
    for (int m = 0; m < nm; ++m) {
      const MergeDesc& q = hmd[size_t(md0 + m)];
      const int N = q.n1 + q.n2;
      const int tn = (N + gBN - 1) / gBN;
      htile[size_t(t0 + 2 * m + 1)] = htile[size_t(t0 + 2 * m)] + ((q.n1 + gBM - 1) / gBM) * tn;
      htile[size_t(t0 + 2 * m + 2)] = htile[size_t(t0 + 2 * m + 1)] + ((q.n2 + gBM - 1) / gBM) * tn;
    }
  }
  if (L > 0) {
    if (hmd.size() > size_t(2 * n + 2) || htile.size() > size_t(4 * n + 130))
      throw std::runtime_error("stedc: level descriptors exceed the workspace");
    // pageable sources: the copies are staged before cudaMemcpyAsync returns
    BSE_CUDA(cudaMemcpyAsync(mdesc_all, hmd.data(), sizeof(MergeDesc) * hmd.size(),
                             cudaMemcpyHostToDevice, s));
    BSE_CUDA(cudaMemcpyAsync(tile_off_all, htile.data(), sizeof(int) * htile.size(),
                             cudaMemcpyHostToDevice, s));
  }
  for (int lvl = L - 1; lvl >= 0; --lvl) {
    const int nm = 1 << lvl;
    const int maxN = lvl_maxn[size_t(lvl)];
    MergeDesc* mdesc = mdesc_all + lvl_md[size_t(lvl)];
    const int* tile_off = tile_off_all + lvl_tile[size_t(lvl)];
    StedcLevel lv{};
    lv.md = mdesc; lv.ms = mstate; lv.nmerge = nm; lv.n = n;
    lv.D = D; lv.E = E; lv.Qold = bufs[cur]; lv.Qnew = bufs[cur ^ 1];
    lv.dl = dl; lv.w = w; lv.ndcol = ndcol; lv.ndtype = ndtype; lv.defval = defval;
    lv.defcol = defcol; lv.orig = orig; lv.tau = tau; lv.what = what; lv.pos = pos;
    lv.defpos = defpos; lv.rowT = rowT; lv.rowB = rowB; lv.acolT = acolT; lv.acolB = acolB;
    lv.ccol = ccol; lv.UT = UT; lv.UB = UB; lv.info = d_info;
    lv.keep_from = (lvl == 0) ? keep_from : 0;
    {
      const int64_t half = int64_t(maxN / 2 + 1) * (maxN / 2 + 1) * 2;
      const unsigned gx = unsigned(std::min<int64_t>(ceil_div(half, 256), 4096 / std::max(1, nm) + 1));
      stedc_zero_offdiag_kernel<<<dim3(gx, unsigned(nm)), 256, 0, s>>>(lv);
      BSE_LAUNCH_CHECK();
    }
    stedc_prepare_kernel<<<nm, 256, 0, s>>>(lv);
    BSE_LAUNCH_CHECK();
    const int wpb = 8;
    const dim3 gw(unsigned(ceil_div(maxN, wpb)), unsigned(nm));
    stedc_secular_kernel<<<gw, 32 * wpb, 0, s>>>(lv);
    BSE_LAUNCH_CHECK();
    const dim3 gz(unsigned(max64(ceil_div(maxN, wpb), ceil_div(maxN, 256))), unsigned(nm));
    stedc_zhat_kernel<<<gz, 256, 0, s>>>(lv);
    BSE_LAUNCH_CHECK();
    stedc_u_kernel<<<gw, 32 * wpb, 0, s>>>(lv);
    BSE_LAUNCH_CHECK();
    const int tiles = htile[size_t(lvl_tile[size_t(lvl)] + 2 * nm)];
    stedc_gemm_kernel<<<unsigned(tiles), GT::NTHREADS, GT::SMEM, s>>>(lv, tile_off);
    BSE_LAUNCH_CHECK();
    stedc_finish_kernel<<<dim3(unsigned(std::min(maxN, 1024)), unsigned(nm)), 128, 0, s>>>(lv);
    BSE_LAUNCH_CHECK();
    cur ^= 1;
  }
  stedc_unscale_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(n, D, scale, d);
  BSE_LAUNCH_CHECK();
}

}  // namespace bseg
