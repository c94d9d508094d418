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

#include <cstdlib>
#include <vector>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "svd.h"
#include "tile_ring.cuh"

namespace cg = cooperative_groups;

namespace bseg {

namespace {
constexpr int kT = 64;         // tile edge = slab of the vector phases
constexpr int kThreads = 256;  // 4 threads per slab row/column
constexpr int kQ = kThreads / kT;
constexpr int kNB = kGebrdNB;
static_assert(kNB % kQ == 0 && kNB <= 32, "panel width");
// Tile ring: every CTA keeps its last kRing trailing-matrix tiles in shared memory. Within a
// panel the trailing block A(p0:, p0:) is only read (zlabrd keeps the update in V,X,Y,U), so a
// tile loaded once stays valid for all kNB columns; the two mat-vec sweeps per column run in
// opposite directions (serpentine), each starting on the kRing tiles the previous sweep ended
// on, and the refills stream kRing tiles ahead of the consumer.
constexpr int kRing = 3;
constexpr int kTabMax = 1792;  // per-CTA tile list capacity (n <= ~32k; checked on the host)
constexpr int kTile = kT * kT;  // z_t per slot (tile_ring.cuh layout)
}  // namespace

struct alignas(64) GebrdArgs {
  z_t* A;
  int64_t lda, n;
  double* d;
  double* e;
  z_t* tauq;
  z_t* taup;
  z_t* VX;  // n x 2NB: [V | X]
  z_t* YU;  // n x 2NB: [Y | U]
  z_t* wrow;      // n : row update w = conj(a(g,:)) - ...
  z_t* P;         // nch * nch * kT tile partials
  double* normp;  // nch
  z_t* s12;       // nch x 2NB : V^H x | X^H x
  z_t* s34;       // nch x 2(NB+1) : Y^H w | U^H w
  z_t* t;         // 4 (NB+1): t1 | t2 | t3 | t4
  int64_t p0;
  int nbp, nch;
  unsigned long long* trace;  // optional per-phase timestamps (BSE_GEBRD_TRACE)
  unsigned* bar;              // grid barrier counter, zeroed before every launch
  CUtensorMap tmap;           // TMA view of A (tile_ring.cuh)
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

__device__ __forceinline__ double gb_warp_sum_range(const double* p, int lo, int hi) {
  double s[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) s[u] = 0.0;
  for (int k0 = lo + (threadIdx.x & 31); k0 < hi; k0 += 256) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + 32 * u < hi) s[u] += p[k0 + 32 * u];
  }
  return warp_sum(((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7])));
}

__device__ __forceinline__ int gb_first_owned(int lo, int cta, int G) {
  int c = cta;
  while (c < lo) c += G;
  return c;
}

// CTA 0: t_out[p] = conj(head[p]) + scale * sum_c partial[c * stride + off + p], p < pmax
// (64 sums x 4 partial lanes; entries p >= pmax are zeroed).
__device__ __forceinline__ void gb_tsum(const z_t* partial, int stride, int off, int c_lo,
                                        int c_hi, const z_t* head, int64_t head_stride, int pmax,
                                        z_t scale, z_t* t_out, int nsum) {
  const int kk = threadIdx.x >> 2, part = threadIdx.x & 3;
  z_t s = make_double2(0.0, 0.0);
  if (kk < nsum && kk < pmax) s = zsum_strided16(partial + off + kk, stride, c_lo + part, c_hi, 4);
  warp_converge();
  s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
  s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
  s.x += __shfl_xor_sync(0xffffffffu, s.x, 2);
  s.y += __shfl_xor_sync(0xffffffffu, s.y, 2);
  if (part == 0 && kk < nsum)
    t_out[kk] = kk < pmax ? zadd(zconj(head[int64_t(kk) * head_stride]), zmul(scale, s))
                          : make_double2(0.0, 0.0);
}

// Tile t of the panel's K x K tile grid starting at slab sp, column-major: each CTA owns a
// contiguous run (so consecutive tiles of a run mostly share their tile column).
__device__ __forceinline__ void gb_tile_coords(int t, int K, int sp, int& rc, int& cc) {
  rc = sp + t % K;
  cc = sp + t / K;
}

using Ring = TileRing<kRing>;

// One mat-vec sweep over this CTA's T tiles, writing one 64-vector partial per tile to P.
//  kCols (P2): y(c) = sum_r conj(A(r,c)) v(r), v = [1; scale * A(g+1:, g)] on rows >= g
//  !kCols (P4): x(r) = sum_c A(r,c) u(c),      u = [1; scale * w(g+2:)] on cols >= g+1
// Masked rows/columns of the cached tiles hold finite panel-start data that either meets a
// zero vector entry or produces a partial nobody reads (see the phase comments). Forward
// sweeps end with tiles T-kRing..T-1 resident, backward sweeps with 0..kRing-1: each sweep
// starts on the tiles the previous one ended on, and refills run kRing-1 tiles ahead.
// Mapping: warp w owns tile columns 8w..8w+7, lane l rows l and l+32; row sums reduce across
// warps through rowred (double buffered, summed by warps 0-1 after the per-tile barrier), one
// CTA barrier per tile. Column sums (P2, a forward sweep) stay in per-lane registers over a
// segment -- consecutive tiles of one tile column -- and are reduced inside the warp
// (transpose reduction) at the segment's last tile, which has its largest tile row: that
// slot of P gets the segment's sum, the segment's other slots zeros (P3 sums the slots from
// the current row slab on, and only rows >= g carry nonzero vector entries).
template <bool kCols>
__device__ __forceinline__ void gb_sweep(const GebrdArgs& a, Ring& ring, const int* ttab,
                                         z_t* vbuf, z_t* swp, int T, bool forward, int64_t g,
                                         z_t scale) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const z_t zero = make_double2(0.0, 0.0), one = make_double2(1.0, 0.0);
  // warps 6-7 stage the vectors (warps 0-1 finish P4's row sums after each tile)
  const int vtid = tid - (kThreads - kT);
  const bool vthr = vtid >= 0;
  auto vidx = [&](int k) -> int64_t {
    const int t = ttab[k];
    return int64_t(kCols ? (t & 0xffff) : (t >> 16)) * kT + vtid;
  };
  auto fetch = [&](int k) -> z_t {
    const int64_t e = vidx(k);
    if (kCols) return (e > g && e < n) ? a.A[e + g * a.lda] : zero;
    return (e >= g + 2 && e < n) ? a.wrow[e] : zero;
  };
  auto put = [&](int k, z_t rw, z_t* buf) {
    const int64_t e = vidx(k);
    if (kCols) buf[vtid] = (e == g) ? one : ((e > g && e < n) ? zmul(scale, rw) : zero);
    else buf[vtid] = (e == g + 1) ? one : ((e >= g + 2 && e < n) ? zmul(scale, rw) : zero);
  };
  z_t raw = zero;
  if (vthr && T > 0) {
    put(forward ? 0 : T - 1, fetch(forward ? 0 : T - 1), vbuf);
    if (T > 1) raw = fetch(forward ? 1 : T - 2);
  }
  __syncthreads();
  z_t pc[8];
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) pc[c8] = zero;
  for (int j = 0; j < T; ++j) {
    const int k = forward ? j : T - 1 - j;
    const int rc = ttab[k] & 0xffff, cc = ttab[k] >> 16;
    ring.acquire(k % kRing);
    const z_t* vv = vbuf + (j & 1) * kT;
    if (vthr && j + 1 < T) {  // next tile's vector into the other buffer
      put(forward ? j + 1 : T - 2 - j, raw, vbuf + ((j + 1) & 1) * kT);
      if (j + 2 < T) raw = fetch(forward ? j + 2 : T - 3 - j);
    }
    const z_t* tl = ring.slot(k % kRing);
    z_t* rowred = swp + (j & 1) * 8 * kT;
    if (kCols) {
      const z_t v0 = vv[lane], v1 = vv[lane + 32];
      const bool seg_end = j == T - 1 || (ttab[forward ? k + 1 : k - 1] >> 16) != cc;
      const z_t* tw = tl + ring_idx(lane, 8 * warp);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        zcfma(pc[c8], tw[c8 * kRingT], v0);
        zcfma(pc[c8], tw[c8 * kRingT + 32], v1);
      }
      z_t* slot = a.P + (int64_t(cc) * a.nch + rc) * kT + 8 * warp + (lane >> 2);
      if (seg_end) {  // CTA-uniform
        const z_t tot = warp_transpose_zsum8(pc);
        if ((lane & 3) == 0) *slot = tot;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) pc[c8] = zero;
      } else if ((lane & 3) == 0) {
        *slot = zero;
      }
    } else {
      z_t r0 = zero, r1 = zero;
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        const int c = 8 * warp + c8;
        const z_t u = vv[c];
        zfma(r0, tl[ring_idx(lane, c)], u);
        zfma(r1, tl[ring_idx(lane + 32, c)], u);
      }
      rowred[warp * kT + lane] = r0;
      rowred[warp * kT + lane + 32] = r1;
    }
    __syncthreads();  // tile k fully read; partials and the next vector visible
    const int kn = forward ? k + kRing : k - kRing;  // refill the slot with the tile it serves next
    if (kn >= 0 && kn < T)
      ring.issue(k % kRing, &a.tmap, int64_t(ttab[kn] & 0xffff) * kT, int64_t(ttab[kn] >> 16) * kT);
    if (!kCols && tid < kT) {
      z_t sum = rowred[tid];
#pragma unroll
      for (int w = 1; w < 8; ++w) sum = zadd(sum, rowred[w * kT + tid]);
      a.P[(int64_t(rc) * a.nch + cc) * kT + tid] = sum;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) gebrd_panel_kernel(const __grid_constant__ GebrdArgs a) {
  GridBarrier grid(a.bar);
  extern __shared__ __align__(16) unsigned char sm[];
  Ring ring;
  unsigned char* const sm_ring = sm + ((128u - (smem_u32(sm) & 127u)) & 127u);  // TMA alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_ring + sizeof(z_t) * kRing * kTile);
  z_t* vbuf = reinterpret_cast<z_t*>(bars + 2 * kRing);  // 2 x kT: sweep vectors
  int* ttab = reinterpret_cast<int*>(vbuf + 2 * kT);       // this CTA's tiles: rc | cc << 16
  z_t* swp = reinterpret_cast<z_t*>(ttab + kTabMax);       // 2 x 8 x kT: sweep row partials
  z_t* red = swp;                          // kQ x kT (P1/P3; aliases swp)
  z_t* red2 = red + kQ * kT;               // kQ x kT
  z_t* sa = swp + 2 * 8 * kT;              // NB+1
  z_t* sb = sa + (kNB + 1);                // NB+1
  z_t* tt = sb + (kNB + 1);                // 2(NB+1)
  z_t* xs = tt + 2 * (kNB + 1);            // kT
  z_t* xc = xs + kT;                       // kT
  double* dred = reinterpret_cast<double*>(xc + kT);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = tid & (kT - 1), q = tid / kT;
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

  auto trace = [&](int i, int k) {
    if (a.trace && tid == 0 && (cta == 0 || cta == (a.nch - 1) % G)) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[((int64_t(a.p0 / kNB) * kNB + i) * 2 + (cta == 0 ? 0 : 1)) * 8 + k] = t;
    }
  };
  // panel tile grid: slabs [sp, nch)^2 (a panel never straddles a 64-slab)
  const int sp = int(a.p0 / kT), K = a.nch - sp;
  const int tq = K * K / G, tr = K * K % G;  // contiguous runs, the remainder to the first CTAs
  const int t0 = cta * tq + min(cta, tr);
  const int T = tq + (cta < tr ? 1 : 0);
  for (int k = tid; k < T; k += kThreads) {
    int rc, cc;
    gb_tile_coords(t0 + k, K, sp, rc, cc);
    ttab[k] = rc | (cc << 16);
  }
  ring.init(reinterpret_cast<z_t*>(sm_ring), bars);
  for (int k = 0; k < kRing && k < T; ++k)  // in flight during the first P1 (ttab synced by init)
    ring.issue(k, &a.tmap, int64_t(ttab[k] & 0xffff) * kT, int64_t(ttab[k] >> 16) * kT);
  for (int i = 0; i <= a.nbp; ++i) {
    const int64_t g = a.p0 + i;
    if (i < a.nbp) trace(i, 0);
    const bool last = (i == a.nbp);
    const int s0 = int(g / kT);
    // ---------------------------------------------------------------- P1 (rows)
    const bool have_prev = i > 0;  // previous column had a row reflector (g - 1 < n - 1)
    const z_t taup_prev = have_prev ? a.taup[g - 1] : zero;
    for (int c = gb_first_owned(s0, cta, G), first = 1; c < a.nch; c += G, first = 0) {
      const int64_t r = int64_t(c) * kT + rl;
      const bool valid = r < n && r >= g;
      // one memory round trip: partials, panel rows and (first slab) the small vectors
      // (all loads are issued before the first consumer)
      z_t xpart = zero, upd = zero, aold = zero, vr[kNB / kQ], xr[kNB / kQ];
      z_t pa = zero, pb = zero, pt = zero;
      if (first) {
        if (!last && tid < i) {
          pa = Y[g + int64_t(tid) * ldp];
          pb = U[g + int64_t(tid) * ldp];
        }
        if (have_prev && tid < 2 * (kNB + 1)) pt = a.t[2 * (kNB + 1) + tid];  // t3 | t4
      }
#pragma unroll
      for (int k = 0; k < kNB / kQ; ++k) {
        const int p = q + k * kQ;
        vr[k] = (valid && p < i) ? V[r + int64_t(p) * ldp] : zero;
        xr[k] = (valid && p < i - 1) ? X[r + int64_t(p) * ldp] : zero;
      }
      if (valid && q == 0 && !last) aold = a.A[r + g * lda];
      if (valid && have_prev)
        xpart = zsum_strided16(a.P + int64_t(c) * a.nch * kT + rl, kT, s0 + q, a.nch, kQ);
      if (first) {
        if (tid < kNB) {
          sa[tid] = pa;
          sb[tid] = pb;
        }
        if (tid < 2 * (kNB + 1)) tt[tid] = pt;
        __syncthreads();
      }
      if (valid) {
#pragma unroll
        for (int k = 0; k < kNB / kQ; ++k) {
          const int p = q + k * kQ;
          if (p < i) {
            const z_t vrp = vr[k];
            if (have_prev) xpart = zsub(xpart, zmul(vrp, tt[p]));
            if (p < i - 1) {
              const z_t xrp = xr[k];
              if (have_prev) xpart = zsub(xpart, zmul(xrp, tt[(kNB + 1) + p]));
              if (!last) upd = zadd(upd, zadd(zmul(vrp, zconj(sa[p])), zmul(xrp, zconj(sb[p]))));
            } else if (!last) {
              upd = zadd(upd, zmul(vrp, zconj(sa[p])));  // X(r, i-1) term added below
            }
          }
        }
      }
      red[q * kT + rl] = xpart;
      red2[q * kT + rl] = upd;
      __syncthreads();
      z_t x = zero;
      if (q == 0) {
        z_t xprev = zero;
        if (valid) {
          z_t sx = red[rl], su = red2[rl];
#pragma unroll
          for (int qq = 1; qq < kQ; ++qq) {
            sx = zadd(sx, red[qq * kT + rl]);
            su = zadd(su, red2[qq * kT + rl]);
          }
          if (have_prev) {
            xprev = zmul(taup_prev, sx);
            X[r + int64_t(i - 1) * ldp] = xprev;
          }
          if (!last) {
            x = zsub(aold, su);
            if (have_prev) x = zsub(x, zmul(xprev, zconj(sb[i - 1])));
            a.A[r + g * lda] = x;
          }
        }
        xc[rl] = xprev;
        xs[rl] = (!last && valid && r > g) ? x : zero;
        x = xs[rl];
      }
      if (last) {
        __syncthreads();
        continue;
      }
      const double nrm = block_sum(q == 0 ? zabs2(x) : 0.0, dred);
      if (tid == 0) a.normp[c] = nrm;
      {  // s12(p) = [V(:,p)^H x | X(:,p)^H x] over this slab, from the rows held in registers
        const z_t xv = xs[rl], xp = xc[rl];
        z_t pr[16];
#pragma unroll
        for (int k = 0; k < kNB / kQ; ++k) {
          const int p = q + k * kQ;
          pr[k] = zero;
          pr[8 + k] = zero;
          zcfma(pr[k], vr[k], xv);
          zcfma(pr[8 + k], (p == i - 1) ? xp : xr[k], xv);
        }
        const z_t tot = warp_transpose_zsum16(pr);
        const int idx = lane >> 1;
        if ((warp & 1) && !(lane & 1)) red[q * 16 + idx] = tot;  // rows 32..63 of the slab
        __syncthreads();
        if (!(warp & 1) && !(lane & 1)) {
          const int p = q + (idx & 7) * kQ;
          if (p < i) a.s12[int64_t(c) * 2 * kNB + (idx >> 3) * kNB + p] = zadd(tot, red[q * 16 + idx]);
        }
      }
      __syncthreads();
    }
    if (last) break;
    trace(i, 1);
    grid.sync();
    trace(i, 2);
    // ---------------------------------------------------------------- P2: column reflector + y'
    __syncthreads();  // converged warps before warp 0's butterflies (BRA.DIV fallback)
    if (warp == 0) {  // one warp per CTA (no L2 hot spot), smem broadcast
      const double v = gb_warp_sum_range(a.normp, s0, a.nch);
      if (lane == 0) {
        dred[0] = v;
        xc[0] = a.A[g + g * lda];
      }
    }
    __syncthreads();
    const double xn2 = dred[0];
    const z_t alpha = xc[0];
    double beta;
    z_t tq, scale;
    larfg_params2(alpha, xn2, beta, tq, scale);
    const bool has_cols = (g + 1 < n);
    if (has_cols) gb_sweep<true>(a, ring, ttab, vbuf, swp, T, true, g, scale);
    // off the sweep's critical path: d/tau, the reflector into the panel, t1/t2 (by the CTA
    // with the fewest tiles)
    if (cta == 0 && tid == 0) {
      a.d[g] = beta;
      a.tauq[g] = tq;
    }
    if (q == 0) {
      for (int c = gb_first_owned(s0, cta, G); c < a.nch; c += G) {
        const int64_t r = int64_t(c) * kT + rl;
        if (r < n && r >= g)
          V[r + int64_t(i) * ldp] = (r == g) ? make_double2(1.0, 0.0) : zmul(scale, a.A[r + g * lda]);
      }
    }
    // t1 / t2 on the two last CTAs (fewest tiles, no slab), one load round each
    if (cta == G - 1 || (cta == G - 2 && G >= 2)) {
      __syncthreads();  // converged warps before the shuffles
      if (cta == G - 1) gb_tsum(a.s12, 2 * kNB, 0, s0, a.nch, V + g, ldp, i, scale, t1, kNB);
      if (cta == G - 2 || G == 1) gb_tsum(a.s12, 2 * kNB, kNB, s0, a.nch, X + g, ldp, i, scale, t2, kNB);
    }
    trace(i, 3);
    grid.sync();
    trace(i, 4);
    // ---------------------------------------------------------------- P3 (columns)
    if (has_cols) {
      const int c0 = int((g + 1) / kT);
      for (int cb = gb_first_owned(c0, cta, G), first = 1; cb < a.nch; cb += G, first = 0) {
        const int64_t c = int64_t(cb) * kT + rl;
        const bool valid = c < n && c > g;
        // one memory round trip: partials, panel rows and (first slab) the small vectors
        z_t ypart = zero, wpart = zero, aold = zero, yr[kNB / kQ], ur[kNB / kQ];
        z_t pa = zero, pb = zero, pt = zero;
        if (first) {
          if (tid < i) {
            pa = V[g + int64_t(tid) * ldp];
            pb = X[g + int64_t(tid) * ldp];
          }
          if (tid < 2 * (kNB + 1)) pt = a.t[tid];  // t1 | t2
        }
#pragma unroll
        for (int k = 0; k < kNB / kQ; ++k) {
          const int p = q + k * kQ;
          yr[k] = (valid && p < i) ? Y[c + int64_t(p) * ldp] : zero;
          ur[k] = (valid && p < i) ? U[c + int64_t(p) * ldp] : zero;
        }
        if (valid && q == 0) aold = a.A[g + c * lda];
        if (valid) ypart = zsum_strided16(a.P + int64_t(cb) * a.nch * kT + rl, kT, s0 + q, a.nch, kQ);
        if (first) {
          if (tid <= kNB) {
            sa[tid] = (tid == i) ? make_double2(1.0, 0.0) : pa;
            sb[tid] = pb;
          }
          if (tid < 2 * (kNB + 1)) tt[tid] = pt;
          __syncthreads();
        }
        if (valid) {
#pragma unroll
          for (int k = 0; k < kNB / kQ; ++k) {
            const int p = q + k * kQ;
            if (p < i) {
              const z_t ycp = yr[k], ucp = ur[k];
              ypart = zsub(ypart, zadd(zmul(ycp, tt[p]), zmul(ucp, tt[(kNB + 1) + p])));
              wpart = zadd(wpart, zadd(zmul(ycp, zconj(sa[p])), zmul(ucp, zconj(sb[p]))));
            }
          }
        }
        red[q * kT + rl] = ypart;
        red2[q * kT + rl] = wpart;
        __syncthreads();
        z_t w = zero, ycur = zero;
        if (q == 0) {
          if (valid) {
            z_t sy = red[rl], sw = red2[rl];
#pragma unroll
            for (int qq = 1; qq < kQ; ++qq) {
              sy = zadd(sy, red[qq * kT + rl]);
              sw = zadd(sw, red2[qq * kT + rl]);
            }
            ycur = zmul(tq, sy);
            Y[c + int64_t(i) * ldp] = ycur;
            w = zsub(zsub(zconj(aold), sw), ycur);  // p = i term: Y(c,i) conj(V(g,i) = 1)
            a.wrow[c] = w;
          }
          xs[rl] = (valid && c >= g + 2) ? w : zero;
          xc[rl] = ycur;
          w = xs[rl];
        }
        const double nrm = block_sum(q == 0 ? zabs2(w) : 0.0, dred);
        if (tid == 0) a.normp[cb] = nrm;
        {  // s34(p) = [Y(:,p)^H w (p <= i) | U(:,p)^H w (p < i)] over this slab
          const z_t wv = xs[rl], yc = xc[rl];
          z_t pr[16];
#pragma unroll
          for (int k = 0; k < kNB / kQ; ++k) {
            const int p = q + k * kQ;
            pr[k] = zero;
            pr[8 + k] = zero;
            zcfma(pr[k], (p == i) ? yc : yr[k], wv);
            zcfma(pr[8 + k], ur[k], wv);
          }
          const z_t tot = warp_transpose_zsum16(pr);
          const int idx = lane >> 1;
          if ((warp & 1) && !(lane & 1)) red[q * 16 + idx] = tot;
          __syncthreads();
          if (!(warp & 1) && !(lane & 1)) {
            const int p = q + (idx & 7) * kQ, kind = idx >> 3;
            if (p < i || (p == i && kind == 0))
              a.s34[int64_t(cb) * 2 * (kNB + 1) + kind * (kNB + 1) + p] = zadd(tot, red[q * 16 + idx]);
          }
        }
        __syncthreads();
      }
    }
    if (q == 0) {  // reflector storage of column g (the P2 readers of A(:, g) are done)
      for (int c = gb_first_owned(s0, cta, G); c < a.nch; c += G) {
        const int64_t r = int64_t(c) * kT + rl;
        if (r < n && r > g) a.A[r + g * lda] = V[r + int64_t(i) * ldp];
      }
    }
    trace(i, 5);
    grid.sync();
    trace(i, 6);
    // ---------------------------------------------------------------- P4: row reflector + x'
    if (has_cols) {
      const int c0 = int((g + 1) / kT);
      __syncthreads();  // converged warps before warp 0's butterflies
      if (warp == 0) {
        const double v = gb_warp_sum_range(a.normp, c0, a.nch);
        if (lane == 0) {
          dred[0] = v;
          xc[0] = a.wrow[g + 1];
        }
      }
      __syncthreads();
      const double xr2 = dred[0];
      const z_t alpha2 = xc[0];
      double beta2;
      z_t tp, scale2;
      larfg_params2(alpha2, xr2, beta2, tp, scale2);
      gb_sweep<false>(a, ring, ttab, vbuf, swp, T, false, g, scale2);
      if (cta == 0 && tid == 0) {
        a.e[g] = beta2;
        a.taup[g] = tp;
      }
      if (cta == G - 1 || (cta == G - 2 && G >= 2)) {  // t3 / t4 on the two last CTAs
        __syncthreads();  // converged warps before the shuffles
        if (cta == G - 1)
          gb_tsum(a.s34, 2 * (kNB + 1), 0, c0, a.nch, Y + (g + 1), ldp, i + 1, scale2, t3, kNB + 1);
        if (cta == G - 2 || G == 1)
          gb_tsum(a.s34, 2 * (kNB + 1), kNB + 1, c0, a.nch, U + (g + 1), ldp, i, scale2, t4, kNB + 1);
      }
      if (q == 0) {
        for (int cb = gb_first_owned(c0, cta, G); cb < a.nch; cb += G) {
          const int64_t c = int64_t(cb) * kT + rl;
          if (c < n && c > g) {
            z_t u = make_double2(1.0, 0.0);
            if (c >= g + 2) {
              u = zmul(scale2, a.wrow[c]);
              a.A[g + c * lda] = u;  // row reflector storage (unconjugated)
            }
            U[c + int64_t(i) * ldp] = u;
          }
        }
      }
    }
    trace(i, 7);
    grid.sync();
  }
  ring.drain();  // no bulk copy may be in flight when the CTA exits
}

size_t gebrd_workspace_bytes(int64_t n) {
  const int64_t nch = ceil_div(n, kT);
  size_t z = 0;
  z += 4 + size_t(n) * 2 * kNB * 2; // barrier counter, VX, YU
  z += size_t(n);                   // wrow
  z += size_t(nch) * nch * kT;      // P
  z += size_t(nch) * 2 * kNB;       // s12
  z += size_t(nch) * 2 * (kNB + 1); // s34
  z += size_t(4) * (kNB + 1);       // t
  return z * sizeof(z_t) + size_t(nch) * sizeof(double) + 1024;
}

void zgebrd_upper(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tauq, z_t* taup, void* ws) {
  if (n <= 0) return;
  const int nch = int(ceil_div(n, kT));
  z_t* base = reinterpret_cast<z_t*>(ws);
  GebrdArgs a{};
  a.A = A; a.lda = lda; a.n = n; a.d = d; a.e = e; a.tauq = tauq; a.taup = taup;
  a.tmap = make_tile_map(A, lda, n);
  a.bar = reinterpret_cast<unsigned*>(base); base += 4;  // 64 bytes, zeroed with VX / YU
  a.VX = base; base += n * 2 * kNB;
  a.YU = base; base += n * 2 * kNB;
  a.wrow = base; base += n;
  a.P = base; base += int64_t(nch) * nch * kT;
  a.s12 = base; base += int64_t(nch) * 2 * kNB;
  a.s34 = base; base += int64_t(nch) * 2 * (kNB + 1);
  a.t = base; base += 4 * (kNB + 1);
  a.normp = reinterpret_cast<double*>(base);
  a.nch = nch;
  const size_t smem = (size_t(kRing) * kTile + kRing + 2 * kT + 2 * 8 * kT + 4 * (kNB + 1) + 2 * kT) *
                          sizeof(z_t) + kTabMax * sizeof(int) + 8 * sizeof(double) + 128;
  struct Occ {
    int blocks_per_sm, num_sms;
  };
  const Occ& occ = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    Occ o{0, 0};
    BSE_CUDA(cudaFuncSetAttribute(gebrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    int dev;
    BSE_CUDA(cudaGetDevice(&dev));
    BSE_CUDA(cudaDeviceGetAttribute(&o.num_sms, cudaDevAttrMultiProcessorCount, dev));
    BSE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks_per_sm, gebrd_panel_kernel,
                                                           kThreads, smem));
    return o;
  });
  const int blocks_per_sm = occ.blocks_per_sm, num_sms = occ.num_sms;
  if (blocks_per_sm < 1) throw std::runtime_error("gebrd: kernel cannot be resident");
  const z_t mone = {-1.0, 0.0}, one = {1.0, 0.0};
  const char* trace_path = getenv("BSE_GEBRD_TRACE");
  const size_t trace_n = size_t(ceil_div(n, kNB)) * kNB * 2 * 8;
  if (trace_path) BSE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.trace), trace_n * 8, s));
  for (int64_t p0 = 0; p0 < n; p0 += kNB) {
    const int nbp = int(min64(kNB, n - p0));
    BSE_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(z_t) * (4 + size_t(n) * 2 * kNB * 2), s));
    a.p0 = p0;
    a.nbp = nbp;
    const int64_t m = n - p0;
    const int64_t tiles = ceil_div(m, kT) * ceil_div(m, kT);
    int G = int(min64(int64_t(blocks_per_sm) * num_sms, tiles));
    if (panel_cta_cap() > 0) G = int(min64(G, panel_cta_cap()));  // batch lanes share the SMs
    G = max(G, 1);
    {
      const int64_t K = nch - p0 / kT;
      if (ceil_div(K * K, int64_t(G)) > kTabMax)
        throw std::runtime_error("gebrd: matrix too large for the per-CTA tile list");
    }
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
  if (trace_path) {  // developer tracing: per-column phase timestamps of two CTAs
    std::vector<unsigned long long> h(trace_n);
    BSE_CUDA(cudaMemcpyAsync(h.data(), a.trace, trace_n * 8, cudaMemcpyDeviceToHost, s));
    BSE_CUDA(cudaStreamSynchronize(s));
    BSE_CUDA(cudaFree(a.trace));
    if (FILE* f = fopen(trace_path, "w")) {
      for (size_t r = 0; r < trace_n / 8; ++r) {
        fprintf(f, "%zu,%zu", r / 2, r % 2);
        for (int k = 0; k < 8; ++k) fprintf(f, ",%llu", h[r * 8 + k]);
        fprintf(f, "\n");
      }
      fclose(f);
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
