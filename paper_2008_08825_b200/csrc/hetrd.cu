// hetrd.cu — Householder tridiagonalisation of a Hermitian matrix (lower storage) and the
// blocked back-transformation V = Q Z.
//
// Replaces the zhetrd + zunmtr halves of LAPACKE_zheevd('V','L') called at
// proj/src/backend.cpp:34. Same algorithm as LAPACK's zlatrd
// ('L') panel + zher2k trailing update, re-laid-out for B200:
//
//  * One persistent cooperative kernel per nb-column panel. Per column g two grid-wide
//    phases replace LAPACK's ~8 BLAS-2 calls (see hetrd_panel_kernel):
//      A  reflector (zlarfg, recomputed redundantly by every CTA from per-slab partial
//         norms) and the Hermitian matrix-vector product y = A22 v over the LOWER triangle
//         only: 64x64 tiles (TMA into a shared-memory ring, one contiguous run of the
//         folded tile order per CTA), each contributing A_t v to its row chunk and A_t^H v
//         to its column chunk (2.67 n^3 bytes over the reduction, the HBM-bound half of
//         zhetrd), plus per-CTA partials of v^H A22 v;
//      B  alpha from v^H A v (no extra dot reduction), W(:,g) = tau (y - V t1 - W t2) +
//         alpha v, and the next column's update with its partial norms / V^H x / W^H x.
//    All partial sums have a fixed order (bit-deterministic).
//  * The trailing update A22 -= V W^H + W V^H is one DMMA GEMM with k = 2 nb writing only
//    lower tiles.
//  * Back-transformation: all reflector blocks, their T factors and V T products are formed
//    up front (batched); each 128-reflector block then costs two DMMA GEMMs.
#include <cooperative_groups.h>

#include <cstdlib>
#include <vector>

#include "blas.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "tile_ring.cuh"

namespace cg = cooperative_groups;

namespace bseg {

namespace {
constexpr int kT = 64;         // hemv tile edge = row slab of the vector phases
constexpr int kThreads = 256;  // 4 threads per slab row
constexpr int NB = kHetrdNB;   // panel width (compile-time: fully unrolled panel loops)
constexpr int kQ = kThreads / kT;
static_assert(NB % kQ == 0 && NB <= 32, "panel width");
}  // namespace

struct alignas(64) HetrdArgs {
  z_t* A;
  int64_t lda, n;
  double* d;
  double* e;
  z_t* tau;
  z_t* VW;  // n x 2NB: [V | W]
  z_t* WV;  // n x 2NB: [W | V]
  int64_t ldp;
  z_t* Y;         // nch * nch * kT: hemv tile partials [row chunk][col chunk]
  double* normp;  // nch : partial ||x||^2 of the next reflector's tail, per slab
  z_t* s12p;      // nch x 2NB: per-slab partial W^H x | V^H x
  z_t* t12;       // 2NB : t1 = W^H v | t2 = V^H v
  double* vav;    // gridDim.x : per-CTA partials of v^H A22 v
  unsigned* bar;  // grid barrier counter, zeroed before every launch
  unsigned long long* trace;  // optional per-phase timestamps (BSE_HETRD_TRACE)
  CUtensorMap tmap;           // TMA view of A (tile_ring.cuh)
  int64_t p0;
  int nbp, nch;
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

// Warp-parallel fixed-order sums (every warp of every CTA gets bit-identical results).
// Loads are issued 8 at a time before any add, so a sum costs ~one L2 round trip.
__device__ __forceinline__ double warp_sum_range(const double* p, int lo, int hi) {
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

// First slab >= lo owned by this CTA (slab c belongs to CTA c % G); no integer division.
__device__ __forceinline__ int first_owned(int lo, int cta, int G) {
  int c = cta;
  while (c < lo) c += G;
  return c;
}

constexpr int kRing = 3;
constexpr int kTabMax = 1280;  // per-CTA tile list capacity (n <= ~40k; checked on the host)
using Ring = TileRing<kRing>;

// Tile t of a K x K lower tile triangle in "folded" column order: tile columns paired as
// (0, K-1), (1, K-2), ... (K + 1 tiles per pair, the longest column with the shortest), each
// column walked down from its diagonal tile. Contiguous runs of this order carry nearly the
// same number of diagonal tiles and column ends, whose extra work balances across the CTAs.
__device__ __forceinline__ void folded_coords(int t, int K, int& bi, int& bj) {
  const int P = t / (K + 1), r = t - P * (K + 1);
  if (r < K - P) {
    bj = P;
    bi = P + r;
  } else {
    bj = K - 1 - P;
    bi = bj + (r - (K - P));
  }
}

// One cooperative launch per nb-column panel. Per column g (index i in the panel):
//   phase A : reflector from the partial norms (zlarfg, redundantly per CTA) and the
//             Hermitian mat-vec y = A22 v over this CTA's 64x64 lower tiles (each tile adds
//             A_t v to its row chunk and A_t^H v to its column chunk) + per-CTA v^H A22 v.
//             The tiles stream through a TMA ring (tile_ring.cuh): A22 is read-only inside a
//             panel, so consecutive columns sweep the CTA's tile list in alternating directions
//             and start on the kRing tiles the previous sweep left in shared memory;
//   phase B : alpha = -1/2 |tau|^2 (v^H A v - 2 Re t1^H t2) (no separate dot reduction),
//             W(:,i) = tau (y - V t1 - W t2) + alpha v, and the NEXT column's update
//             a(:,g+1) -= V W(g+1,:)^H + W V(g+1,:)^H with its partial norms / W^H x / V^H x.
//             All of the phase's loads are issued before the first consumer (one round trip).
// => two grid barriers per column; every partial sum has a fixed order (deterministic).
// Tile entries outside the live region (rows/cols < g+1, finite panel-start data) meet zero
// vector entries or feed partials that are never read; the strict upper triangle of a
// diagonal tile (never written, may hold garbage) is excluded by selects.
__global__ void __launch_bounds__(kThreads, 1)
    hetrd_panel_kernel(const __grid_constant__ HetrdArgs a) {
  GridBarrier grid(a.bar);
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned char* const sm_ring = sm + ((128u - (smem_u32(sm) & 127u)) & 127u);  // TMA alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_ring + sizeof(z_t) * kRing * kRingT * kRingT);
  z_t* vbuf = reinterpret_cast<z_t*>(bars + 2 * kRing);  // 2 x [v rows | v cols] of a tile
  int* ttab = reinterpret_cast<int*>(vbuf + 4 * kT);       // this CTA's tiles: bi | bj << 16
  z_t* swp = reinterpret_cast<z_t*>(ttab + kTabMax);       // 2 x (8 x kT + kT): row partials | segment column sums
  z_t* wg = swp + 2 * (8 * kT + kT);       // NB : W(g+1, p)
  z_t* vg = wg + NB;                       // NB : V(g+1, p)
  z_t* xs = vg + NB;                       // kT : next column values of the slab
  z_t* wc = xs + kT;                       // kT : W(r, i) of the slab
  z_t* tt = wc + kT;                       // 2NB : t1 | t2
  z_t* zred = tt + 2 * NB;                 // 8 complex
  double* dred = reinterpret_cast<double*>(zred + 8);  // 8 doubles

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = tid & (kT - 1), q = tid / kT;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t n = a.n, lda = a.lda, ldp = a.ldp;
  z_t* V = a.VW;
  z_t* W = a.VW + int64_t(NB) * ldp;
  const z_t zero = make_double2(0.0, 0.0), one = make_double2(1.0, 0.0);

  // panel tile list: lower tiles of slabs [sp, nch) (a panel never straddles a 64-slab)
  const int sp = int((a.p0 + 1) / kT), K = a.nch - sp;
  // Tiles in folded column order, one contiguous run per CTA (the remainder to the first CTAs,
  // so the last CTA -- which also forms t1/t2 -- has the fewest): a run is a few segments
  // (consecutive tiles of one tile column), whose column sums stay in registers (see the sweep).
  const int ntiles = K * (K + 1) / 2;
  const int tq = ntiles / G, tr = ntiles % G;
  const int t0 = cta * tq + min(cta, tr);
  const int T = tq + (cta < tr ? 1 : 0);
  for (int k = tid; k < T; k += kThreads) {
    int bi, bj;
    folded_coords(t0 + k, K, bi, bj);
    ttab[k] = bi | (bj << 16);
  }
  Ring ring;
  ring.init(reinterpret_cast<z_t*>(sm_ring), bars);
  for (int k = 0; k < kRing && k < T; ++k)  // in flight during phase 0 (ttab visible: init synced)
    ring.issue(k, &a.tmap, int64_t(sp + (ttab[k] & 0xffff)) * kT, int64_t(sp + (ttab[k] >> 16)) * kT);

  // ---------------------------------------------------------------- phase 0: column p0
  {
    const int64_t g = a.p0;
    for (int c = first_owned(int(g / kT), cta, G); c < a.nch; c += G) {
      const int64_t r = int64_t(c) * kT + rl;
      z_t x = zero;
      if (q == 0 && r < n && r >= g) {
        x = a.A[r + g * lda];
        if (r == g) {
          x.y = 0.0;
          a.A[r + g * lda] = x;
          a.d[g] = x.x;
        }
      }
      const bool inx = q == 0 && r < n && r >= g + 2;
      const double nrm = block_sum(inx ? zabs2(x) : 0.0, dred);
      if (tid == 0) a.normp[c] = nrm;
    }
  }
  grid.sync();

  auto trace = [&](int i, int k) {
    const int slab_owner = (a.nch - 1) % G;  // owner of the last slab (valid to the end)
    if (a.trace && tid == 0 && (cta == 0 || cta == slab_owner)) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[((int64_t(a.p0 / NB) * NB + i) * 2 + (cta == 0 ? 0 : 1)) * 8 + k] = t;
    }
  };
  for (int i = 0; i < a.nbp; ++i) {
    const int64_t g = a.p0 + i;
    const int64_t g1 = g + 1;
    const bool has_next = (i + 1 < a.nbp);
    trace(i, 0);
    // ---------------------------------------------------------------- phase A
    const bool fwd = (i & 1) == 0;
    // Warps 4-7 own the sweep vectors (warps 0-1 finish each tile's row sums): vector thread
    // vtid < 64 holds a tile-row entry, 64 <= vtid < 128 a tile-column entry.
    const int vtid = tid - (kThreads - 2 * kT);
    const bool vthr = vtid >= 0;
    // raw A(:, g) entries of a tile's row (vtid < 64) / column (64 <= vtid < 128) chunk
    auto fetch = [&](int k) -> z_t {
      const int bi = ttab[k] & 0xffff, bj = ttab[k] >> 16;
      const int64_t e = int64_t(sp + (vtid < kT ? bi : bj)) * kT + (vtid & (kT - 1));
      return (e > g1 && e < n) ? a.A[e + g * lda] : zero;
    };
    z_t raw = zero;
    if (vthr && T > 0) raw = fetch(fwd ? 0 : T - 1);
    // one warp per CTA reduces the partial norms (avoids an L2 hot spot), smem broadcast
    if (warp == 0) {
      const double xn2w = warp_sum_range(a.normp, int(g / kT), a.nch);
      if (lane == 0) {
        dred[0] = xn2w;
        zred[0] = a.A[g1 + g * lda];  // alpha; g + 1 < n always (panels stop at n-2)
      }
    }
    __syncthreads();
    const double xn2 = dred[0];
    const z_t alpha = zred[0];
    double beta;
    z_t tau, scale;
    larfg_params(alpha, xn2, beta, tau, scale);
    if (cta == 0 && tid == 0) {
      a.e[g] = beta;
      a.tau[g] = tau;
    }
    trace(i, 1);
    // v restricted to tile k's row chunk (vtid < 64) / column chunk (64 <= vtid < 128)
    auto put_v = [&](int k, z_t rw, z_t* buf) {
      const int bi = ttab[k] & 0xffff, bj = ttab[k] >> 16;
      const int64_t e = int64_t(sp + (vtid < kT ? bi : bj)) * kT + (vtid & (kT - 1));
      buf[vtid] = (e == g1) ? one : ((e > g1 && e < n) ? zmul(scale, rw) : zero);
    };
    if (vthr && T > 0) {
      put_v(fwd ? 0 : T - 1, raw, vbuf);
      raw = (T > 1) ? fetch(fwd ? 1 : T - 2) : zero;
    }
    __syncthreads();
    // Sweep: warp w owns tile columns 8w..8w+7, lane l rows l and l+32. Each element is read
    // once for both products. Row outputs (A_t v_C) reduce across warps per tile (rowred,
    // summed by warps 0-3 after the tile's barrier, one double each). Column outputs
    // (A_t^H v_R) stay in per-lane registers over a segment -- the CTA's consecutive tiles of
    // one tile column, which share v_C -- and are reduced within the warp (transpose
    // reduction) once, at the segment's last tile. Y slots: the row part of tile (I, J) goes
    // to Y[I][J]; the column part of a whole segment to Y[J][I_last], the other tiles of the
    // segment write zeros to their Y[J][I] (a diagonal tile's two slots coincide; every slot
    // of a segment is >= J, so phase B, which sums the slots >= the current column, sees it).
    double vav = 0.0;
    // (initialised: with undefined entry values ptxas keeps them live through phase B, which
    // then serialises its batched partial-sum loads for want of registers)
    z_t pc[8], vcc[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) pc[cc] = vcc[cc] = zero;
    for (int j = 0; j < T; ++j) {
      const int k = fwd ? j : T - 1 - j;
      const int bi = ttab[k] & 0xffff, bj = ttab[k] >> 16;
      const bool diag = (bi == bj);
      const bool seg_start = j == 0 || (ttab[fwd ? k - 1 : k + 1] >> 16) != bj;
      const bool seg_end = j == T - 1 || (ttab[fwd ? k + 1 : k - 1] >> 16) != bj;
      ring.acquire(k % kRing);
      const z_t* vr = vbuf + (j & 1) * 2 * kT;  // v over tile rows
      const z_t* vc = vr + kT;                  // v over tile cols
      // reducing threads (tid < 128: row tid / 2, component tid % 2): their v entries, read
      // before the barrier (the buffer is refilled two tiles later)
      double vrd = 0.0, vcd = 0.0;
      if (tid < 2 * kT) {
        vrd = reinterpret_cast<const double*>(vr)[tid];
        vcd = reinterpret_cast<const double*>(vc)[tid];
      }
      if (seg_start) {
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          vcc[cc] = vc[8 * warp + cc];
          pc[cc] = zero;
        }
      }
      if (vthr && j + 1 < T) {  // next tile's vectors into the other buffer
        put_v(fwd ? j + 1 : T - 2 - j, raw, vbuf + ((j + 1) & 1) * 2 * kT);
        if (j + 2 < T) raw = fetch(fwd ? j + 2 : T - 3 - j);
      }
      const z_t* tl = ring.slot(k % kRing);
      const z_t v0 = vr[lane], v1 = vr[lane + 32];
      z_t r0 = zero, r1 = zero, r0b = zero, r1b = zero;  // two chains per row output
      if (!diag) {  // (CTA-uniform branch) the bulk of the sweep: no masks
        const z_t* tw = tl + ring_idx(lane, 8 * warp);
#pragma unroll
        for (int cc = 0; cc < 8; cc += 2) {
          const z_t a0 = tw[cc * kRingT], a1 = tw[cc * kRingT + 32];
          const z_t b0 = tw[(cc + 1) * kRingT], b1 = tw[(cc + 1) * kRingT + 32];
          zfma(r0, a0, vcc[cc]);
          zfma(r1, a1, vcc[cc]);
          zfma(r0b, b0, vcc[cc + 1]);
          zfma(r1b, b1, vcc[cc + 1]);
          zcfma(pc[cc], a0, v0);
          zcfma(pc[cc + 1], b0, v0);
          zcfma(pc[cc], a1, v1);
          zcfma(pc[cc + 1], b1, v1);
        }
      } else {
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const int c = 8 * warp + cc;
          const z_t a0 = tl[ring_idx(lane, c)], a1 = tl[ring_idx(lane + 32, c)];
          // diagonal tiles: lower triangle only, the Hermitian diagonal real
          const bool low0 = lane > c, low1 = lane + 32 > c;
          const z_t ac0 = low0 ? a0 : zero, ac1 = low1 ? a1 : zero;
          const z_t ar0 = low0 ? a0 : (lane == c ? make_double2(a0.x, 0.0) : zero);
          const z_t ar1 = low1 ? a1 : (lane + 32 == c ? make_double2(a1.x, 0.0) : zero);
          zfma(r0, ar0, vcc[cc]);
          zfma(r1, ar1, vcc[cc]);
          zcfma(pc[cc], ac0, v0);
          zcfma(pc[cc], ac1, v1);
        }
      }
      z_t* rowred = swp + (j & 1) * (8 * kT + kT);  // [8 warps][64 rows] | [64 cols]
      rowred[warp * kT + lane] = zadd(r0, r0b);
      rowred[warp * kT + lane + 32] = zadd(r1, r1b);
      if (seg_end) {  // CTA-uniform
        const z_t ctot = warp_transpose_zsum8(pc);
        if ((lane & 3) == 0) rowred[8 * kT + 8 * warp + (lane >> 2)] = ctot;
      }
      __syncthreads();  // tile k fully read; this tile's partials and the next vectors visible
      {
        const int kn = fwd ? k + kRing : k - kRing;  // refill the slot with the tile it serves next
        if (kn >= 0 && kn < T)
          ring.issue(k % kRing, &a.tmap, int64_t(sp + (ttab[kn] & 0xffff)) * kT,
                     int64_t(sp + (ttab[kn] >> 16)) * kT);
      }
      if (tid < 2 * kT) {
        const double* rd = reinterpret_cast<const double*>(rowred);
        double sr = rd[tid];
#pragma unroll
        for (int w = 1; w < 8; ++w) sr += rd[w * 2 * kT + tid];
        const double sc = seg_end ? rd[16 * kT + tid] : 0.0;
        const int gi = sp + bi, gj = sp + bj;
        double* Yd = reinterpret_cast<double*>(a.Y);
        if (diag) {
          Yd[(int64_t(gi) * a.nch + gi) * 2 * kT + tid] = sr + sc;
        } else {
          Yd[(int64_t(gi) * a.nch + gj) * 2 * kT + tid] = sr;
          Yd[(int64_t(gj) * a.nch + gi) * 2 * kT + tid] = sc;
        }
        // v^H (A v) contributions: rows R (A_t v_C) and, mirrored, the segment's cols C
        vav += vrd * sr + vcd * sc;
      }
    }
    {
      const double vtot = block_sum(vav, dred);
      if (tid == 0) a.vav[cta] = vtot;
    }
    // reflector vector into the panels (rows >= g+1 of the owned slabs)
    if (q == 0) {
      for (int c = first_owned(int(g1 / kT), cta, G); c < a.nch; c += G) {
        const int64_t r = int64_t(c) * kT + rl;
        if (r < n && r >= g1) {
          const z_t v = (r == g1) ? one : zmul(scale, a.A[r + g * lda]);
          V[r + int64_t(i) * ldp] = v;
          a.WV[r + int64_t(NB + i) * ldp] = v;
        }
      }
    }
    if (cta == G - 1) {  // the last CTA has the fewest tiles: t1/t2 off the critical path
      // t1 = W^H v, t2 = V^H v over rows >= g+1 (v(g+1) = 1, v(r) = scale x(r))
      const int kk = tid >> 2, part = tid & 3;  // 64 sums x 4 partial lanes
      const int p = kk & (NB - 1);
      z_t s = zero;
      if (p < i) s = zsum_strided16(a.s12p + kk, 2 * NB, int(g / kT) + part, a.nch, 4);
      warp_converge();
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 1);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 1);
      s.x += __shfl_xor_sync(0xffffffffu, s.x, 2);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, 2);
      if (part == 0 && kk < 2 * NB) {
        z_t t = zero;
        if (p < i) {
          const z_t head = kk < NB ? W[g1 + int64_t(p) * ldp] : V[g1 + int64_t(p) * ldp];
          t = zadd(zconj(head), zmul(scale, s));
        }
        a.t12[kk] = t;
      }
    }
    trace(i, 2);
    grid.sync();
    trace(i, 3);
    // ---------------------------------------------------------------- phase B
    // Mapping: 4 consecutive lanes (sq = lane & 3) share a slab row (srl = tid >> 2) and split
    // the panel columns p = sq + 4k. Cross-lane sums are shuffles, the column sums over the
    // slab rows are warp transpose-reductions plus one shared-memory exchange: two CTA
    // barriers per slab (one more on the first slab for the broadcast scalars).
    const int c0 = int(g1 / kT);
    const int srl = tid >> 2, sq = tid & 3;
    double alw = 0.0;  // alpha of W
    z_t* part = swp;   // [8 warps][4 sq][16] column-sum partials of the slab
    double* nrmw = reinterpret_cast<double*>(swp + 8 * 4 * 16);  // [8] row-norm partials
    for (int c = first_owned(c0, cta, G), first = 1; c < a.nch; c += G, first = 0) {
      const int64_t r = int64_t(c) * kT + srl;
      const bool valid = r < n && r >= g1;
      // every load of the phase is issued before the first consumer
      z_t vrr[NB / kQ], wrr[NB / kQ], vri = zero, xold = zero, ypart = zero;
      double vavr[8];
      z_t ysr[8], vgp = zero, wgp = zero, tq0 = zero, tq1 = zero;
      const z_t* yrow = a.Y + int64_t(c0) * a.nch * kT + (g1 % kT);
      if (first && warp == 0) {  // per-column scalars, summed by warp 0 after the loads
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          vavr[u] = (lane + 32 * u < G) ? a.vav[lane + 32 * u] : 0.0;
          const int m = c0 + lane + 32 * u;
          ysr[u] = (m < a.nch) ? yrow[int64_t(m) * kT] : zero;
        }
        if (lane < i) {
          vgp = V[g1 + int64_t(lane) * ldp];
          wgp = W[g1 + int64_t(lane) * ldp];
        }
        tq0 = a.t12[lane];       // t1 (zero beyond i)
        tq1 = a.t12[NB + lane];  // t2
      }
#pragma unroll
      for (int k = 0; k < NB / kQ; ++k) {
        const int p = sq + k * kQ;
        vrr[k] = (valid && p < i) ? V[r + int64_t(p) * ldp] : zero;
        wrr[k] = (valid && p < i) ? W[r + int64_t(p) * ldp] : zero;
      }
      if (valid) {
        vri = V[r + int64_t(i) * ldp];
        if (has_next) xold = a.A[r + g1 * lda];
        ypart = zsum_strided16(a.Y + int64_t(c) * a.nch * kT + srl, kT, c0 + sq, a.nch, kQ);
      }
      if (first) {
        // A CTA barrier (WARPSYNC.ALL + BAR) re-converges warp 0 before its butterflies:
        // after the lane-dependent load loops above the hardware may still see the warp as
        // diverged, and full-mask shuffles then take the WARPSYNC.COLLECTIVE fallback
        // (measured: 14k cycles for this block instead of ~600).
        __syncthreads();
        if (warp == 0) {  // row g+1 of V and W; alpha of W (same fixed order in every CTA)
          tt[lane] = tq0;
          tt[NB + lane] = tq1;
          // branch-free up to the shuffles (lane-dependent branches leave the warp diverged at
          // the butterflies, which then take the slow BRA.DIV path)
          const bool act = lane < i;
          const z_t cp = zadd(zmul(vgp, tq0), zmul(wgp, tq1));
          z_t corr = act ? cp : zero;
          double vt = act ? zcmul(tq1, tq0).x : 0.0;
          double vs = 0.0;
          z_t ysum = zero;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            vs += vavr[u];
            ysum = zadd(ysum, ysr[u]);
          }
          for (int mm = 256; c0 + mm < a.nch; mm += 32) {  // warp-uniform trip count (n > 16384)
            const int m = c0 + mm + lane;
            if (m < a.nch) ysum = zadd(ysum, yrow[int64_t(m) * kT]);
          }
          const double vw0 = warp_sum(vs);
          const z_t y = warp_zsum(ysum);
          corr = warp_zsum(corr);
          // v^H w' = v^H A v - sum_p [conj(t2_p) t1_p + conj(t1_p) t2_p]  (real)
          const double vw = vw0 - 2.0 * warp_sum(vt);
          const double alw0 = -0.5 * zabs2(tau) * vw;  // alpha of W = tau w' + alpha v (real)
          // y, corr, vw are butterfly sums: identical in every lane, so lane i forms W(g+1, i)
          // itself (no second writer of wg[i])
          const z_t tw = zmul(tau, zsub(y, corr));
          if (lane < NB) {
            vg[lane] = lane < i ? vgp : (lane == i ? one : zero);
            wg[lane] = lane < i ? wgp : (lane == i ? make_double2(tw.x + alw0, tw.y) : zero);
          }
          if (lane == 0) dred[1] = alw0;
        }
        __syncthreads();
        alw = dred[1];
      }
      z_t upd = zero;
      if (valid) {
#pragma unroll
        for (int k = 0; k < NB / kQ; ++k) {
          const int p = sq + k * kQ;
          if (p < i) {
            ypart = zsub(ypart, zadd(zmul(vrr[k], tt[p]), zmul(wrr[k], tt[NB + p])));
            upd = zadd(upd, zadd(zmul(vrr[k], zconj(wg[p])), zmul(wrr[k], zconj(vg[p]))));
          }
        }
      }
      // the 4 lanes of a row get bit-identical sums ((a+b)+(c+d) in every lane); the CTA
      // barrier re-converges the warps before the shuffles (see the first-slab block)
      __syncthreads();
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        ypart.x += __shfl_xor_sync(0xffffffffu, ypart.x, o);
        ypart.y += __shfl_xor_sync(0xffffffffu, ypart.y, o);
        upd.x += __shfl_xor_sync(0xffffffffu, upd.x, o);
        upd.y += __shfl_xor_sync(0xffffffffu, upd.y, o);
      }
      z_t xn = zero, wri = zero;
      if (valid) {
        wri = zadd(zmul(tau, ypart), zscale(vri, alw));
        if (r == g1) wri = wg[i];  // the value every CTA used for row g+1
        z_t x = zero;
        if (has_next) {
          // a(r, g+1) -= sum_{p<=i} V(r,p) conj(W(g+1,p)) + W(r,p) conj(V(g+1,p))
          x = zsub(xold, upd);
          x = zsub(x, zadd(zmul(vri, zconj(wg[i])), wri));  // p = i, V(g+1,i) = 1
          if (r == g1) x.y = 0.0;
          if (r >= g1 + 2) xn = x;
        }
        if (sq == 0) {
          W[r + int64_t(i) * ldp] = wri;
          a.WV[r + int64_t(i) * ldp] = wri;
          if (r >= g1 + 1) a.A[r + g * lda] = vri;  // reflector storage below the subdiagonal
          if (has_next) {
            if (r == g1) a.d[g1] = x.x;
            a.A[r + g1 * lda] = x;
          }
        }
      }
      if (has_next) {
        // s1[p] = sum conj(W(r,p)) x(r), s2[p] = sum conj(V(r,p)) x(r), p <= i, and ||x||^2
        z_t pr[16];
#pragma unroll
        for (int k = 0; k < NB / kQ; ++k) {
          const int p = sq + k * kQ;
          pr[k] = zero;
          pr[8 + k] = zero;
          zcfma(pr[k], (p == i) ? wri : wrr[k], xn);
          zcfma(pr[8 + k], (p == i) ? vri : vrr[k], xn);
        }
        z_t t0, t1;
        __syncthreads();  // re-converge after the lane-dependent stores above
        warp_transpose_zsum16_rows(pr, t0, t1);  // over the warp's 8 rows (lane bits 2..4)
        const int idx = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1);
        part[(warp * 4 + sq) * 16 + idx] = t0;
        part[(warp * 4 + sq) * 16 + idx + 1] = t1;
        const double nr = warp_sum(sq == 0 ? zabs2(xn) : 0.0);
        if (lane == 0) nrmw[warp] = nr;
        __syncthreads();
        if (tid < 64) {  // (sq, idx) = (tid >> 4, tid & 15): fixed-order sum over the 8 warps
          const int q2 = tid >> 4, id = tid & 15;
          z_t sum = part[q2 * 16 + id];
#pragma unroll
          for (int w = 1; w < 8; ++w) sum = zadd(sum, part[(w * 4 + q2) * 16 + id]);
          const int p = q2 + (id & 7) * kQ;
          if (p <= i) a.s12p[int64_t(c) * 2 * NB + (id >> 3) * NB + p] = sum;
        } else if (tid == 64) {
          double nsum = nrmw[0];
#pragma unroll
          for (int w = 1; w < 8; ++w) nsum += nrmw[w];
          a.normp[c] = nsum;
        }
        if (c + G < a.nch) __syncthreads();  // part / nrmw are reused by the next slab
      }
    }
    trace(i, 4);
    if (has_next) grid.sync();
    trace(i, 5);
  }
  ring.drain();  // no TMA load may be in flight when the CTA exits
}

__global__ void set_last_diag_kernel(const z_t* A, int64_t lda, int64_t n, double* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d[n - 1] = A[(n - 1) + (n - 1) * lda].x;
}

size_t hetrd_workspace_bytes(int64_t n) {
  const int64_t nch = ceil_div(n, kT);
  size_t z = 0;
  z += 4 + size_t(n) * 2 * NB * 2;  // barrier counter, VW, WV
  z += size_t(nch) * nch * kT;  // Y
  z += size_t(nch) * 2 * NB;    // s12p
  z += size_t(2 * NB);          // t12
  return z * sizeof(z_t) + size_t(nch) * sizeof(double) + 4096 * sizeof(double) + 512;
}

void zhetrd_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tau, void* ws) {
  if (n <= 0) return;
  const int nch = int(ceil_div(n, kT));
  z_t* base = reinterpret_cast<z_t*>(ws);
  HetrdArgs a{};
  a.A = A; a.lda = lda; a.n = n; a.d = d; a.e = e; a.tau = tau;
  a.tmap = make_tile_map(A, lda, n);
  a.ldp = n;
  a.bar = reinterpret_cast<unsigned*>(base); base += 4;  // 64 bytes, zeroed with VW / WV
  a.VW = base; base += n * 2 * NB;
  a.WV = base; base += n * 2 * NB;
  a.Y = base; base += int64_t(nch) * nch * kT;
  a.s12p = base; base += int64_t(nch) * 2 * NB;
  a.t12 = base; base += 2 * NB;
  a.normp = reinterpret_cast<double*>(base);
  a.vav = a.normp + nch;
  a.nch = nch;

  const size_t smem = (size_t(kRing) * kRingT * kRingT + kRing + 4 * kT + 2 * (8 * kT + kT) + 2 * NB +
                       2 * kT + 2 * NB + 8) * sizeof(z_t) + kTabMax * sizeof(int) + 8 * sizeof(double) +
                      128;
  struct Occ {
    int blocks_per_sm, num_sms;
  };
  const Occ& occ = per_device([&] {  // one-time setup per device (thread-safe: batch lanes)
    Occ o{0, 0};
    BSE_CUDA(cudaFuncSetAttribute(hetrd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    int dev;
    BSE_CUDA(cudaGetDevice(&dev));
    BSE_CUDA(cudaDeviceGetAttribute(&o.num_sms, cudaDevAttrMultiProcessorCount, dev));
    BSE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.blocks_per_sm, hetrd_panel_kernel,
                                                           kThreads, smem));
    return o;
  });
  const int blocks_per_sm = occ.blocks_per_sm, num_sms = occ.num_sms;
  if (blocks_per_sm < 1) throw std::runtime_error("hetrd: kernel cannot be resident");
  if (n == 1) {
    set_last_diag_kernel<<<1, 32, 0, s>>>(A, lda, n, d);
    BSE_LAUNCH_CHECK();
    return;
  }
  const z_t mone = {-1.0, 0.0}, one = {1.0, 0.0};
  const char* trace_path = getenv("BSE_HETRD_TRACE");
  const size_t trace_n = size_t(ceil_div(n, NB)) * NB * 2 * 8;
  if (trace_path) BSE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.trace), trace_n * 8, s));
  for (int64_t p0 = 0; p0 < n - 1; p0 += NB) {
    const int nbp = int(min64(NB, n - 1 - p0));
    BSE_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(z_t) * (4 + size_t(n) * 2 * NB * 2), s));
    a.p0 = p0;
    a.nbp = nbp;
    // shrink the grid with the trailing size (fewer CTAs => cheaper grid barriers)
    const int64_t m = n - p0;
    const int64_t tiles = ceil_div(m, kT) * (ceil_div(m, kT) + 1) / 2;
    int G = int(min64(min64(int64_t(blocks_per_sm) * num_sms, 256), tiles));  // phase B: G <= 256
    if (panel_cta_cap() > 0) G = int(min64(G, panel_cta_cap()));  // batch lanes share the SMs
    G = max(G, 1);
    {
      const int64_t K = nch - (p0 + 1) / kT;
      if (ceil_div(K * (K + 1) / 2, int64_t(G)) > kTabMax)
        throw std::runtime_error("hetrd: matrix too large for the per-CTA tile list");
    }
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
      zgemm(s, 0, 1, n - q, n - q, 2 * NB, mone, a.VW + q, n, a.WV + q, n, one, A + q + q * lda,
            lda, kGeneral, kGeneral, 1, nullptr, 0);
    }
  }
  set_last_diag_kernel<<<1, 32, 0, s>>>(A, lda, n, d);
  BSE_LAUNCH_CHECK();
  if (trace_path) {  // developer tracing: per-column phase timestamps of CTAs 0 and G-1
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

// ---------------------------------------------------------------------------------------
// Back-transformation  Z <- Q Z,  Q = H(0) H(1) ... H(n-2),  H(j) = I - tau_j v_j v_j^H with
// v_j(j+1) = 1 and v_j(j+2:n) stored in A(j+2:n, j)  (zunmtr 'L','L','N').
// Blocks of kBT reflectors, last block first:  Z <- (I - V T V^H) Z  with T from zlarft
// (forward, columnwise): three DMMA GEMMs + one small triangular kernel per block.
namespace {
constexpr int kBT = 128;  // reflectors per applied block (the K of the update GEMM)
}

// Explicit reflector matrix Vall (n x nblk*kBT, ld n): column j = v_j with explicit unit and
// zeros (padding columns j >= nref are zero):
//   mode 0 (zhetrd 'L'): v_j(j+1) = 1, v_j(r) = A(r, j)  for r > j+1
//   mode 1 (zgebrd Q)  : v_j(j)   = 1, v_j(r) = A(r, j)  for r > j
//   mode 2 (zgebrd P)  : u_j(j+1) = 1, u_j(c) = A(j, c)  for c > j+1 (row storage)
//   mode 3 (he2hb 'L') : v_j(j+kBand2) = 1, v_j(r) = A(r, j)  for r > j+kBand2 (hetrd2.cu)
__device__ __host__ __forceinline__ int reflector_offset(int mode) {
  return mode == 1 ? 0 : (mode == 3 ? kBand2 : 1);
}
__global__ void build_vall_kernel(const z_t* __restrict__ A, int64_t lda, int64_t n,
                                  int64_t nref, int64_t ncol, int mode, z_t* __restrict__ Vall) {
  const int off = reflector_offset(mode);
  const int64_t total = n * ncol;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e % n, j = e / n;
    z_t v = make_double2(0.0, 0.0);
    if (j < nref) {
      const int64_t unit = j + off;
      if (r == unit) v = make_double2(1.0, 0.0);
      else if (r > unit) v = (mode == 2) ? A[j + r * lda] : A[r + j * lda];
    }
    Vall[e] = v;
  }
}

// T factors of every block at once (zlarft forward/columnwise): one CTA per block, one
// thread per row r of T: T(r,r) = tau_r, T(r,i) = -tau_i sum_{k=r}^{i-1} T(r,k) G(k,i).
// A thread only reads its own row of T, so no barriers are needed.
__global__ void __launch_bounds__(kBT) larft_all_kernel(const z_t* __restrict__ Gall,
                                                         const z_t* __restrict__ tau,
                                                         int64_t nref, z_t* __restrict__ Tall) {
  const int b = blockIdx.x, r = threadIdx.x;
  const z_t* G = Gall + int64_t(b) * kBT * kBT;
  z_t* T = Tall + int64_t(b) * kBT * kBT;
  const int64_t j0 = int64_t(b) * kBT;
  auto tau_of = [&](int k) {
    return (j0 + k < nref) ? tau[j0 + k] : make_double2(0.0, 0.0);
  };
  for (int i = 0; i < kBT; ++i) {
    z_t v = make_double2(0.0, 0.0);
    if (i == r) {
      v = tau_of(r);
    } else if (i > r) {
      z_t s = make_double2(0.0, 0.0);
      for (int k = r; k < i; ++k) zfma(s, T[r + int64_t(k) * kBT], G[k + int64_t(i) * kBT]);
      v = zscale(zmul(tau_of(i), s), -1.0);
    }
    T[r + int64_t(i) * kBT] = v;
  }
}

size_t unmtr_workspace_bytes(int64_t n, int64_t ncols) {
  const int64_t nblk = ceil_div(max64(n, 1), kBT);
  size_t z = 0;
  z += size_t(n) * nblk * kBT * 2;       // Vall, VTall
  z += size_t(nblk) * kBT * kBT * 2;     // Gall, Tall
  z += size_t(kBT) * ncols;              // W1
  z += size_t(16) * kBT * ncols;         // split-K partials
  return z * sizeof(z_t) + 4096;
}

// Z <- H(0) H(1) ... H(nref-1) Z for the reflector family `mode`, applied in kBT-blocks from
// the last to the first as Z <- Z - (V T)(V^H Z). V, T and V T of all blocks are formed up
// front (batched, prepare_reflectors: needs only the reflectors, so the solvers run it on the
// aux stream beside the divide & conquer), and the serial part per block is two DMMA GEMMs.
void prepare_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                        int64_t lda, const z_t* tau, void* ws) {
  if (nref <= 0) return;
  const int64_t nblk = ceil_div(nref, kBT);
  const int64_t ncol = nblk * kBT;
  z_t* Vall = reinterpret_cast<z_t*>(ws);
  z_t* VTall = Vall + n * ncol;
  z_t* Gall = VTall + n * ncol;
  z_t* Tall = Gall + nblk * kBT * kBT;
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0};
  {
    const int blocks = int(min64(ceil_div(n * ncol, 256), 148 * 16));
    build_vall_kernel<<<blocks, 256, 0, s>>>(A, lda, n, nref, ncol, mode, Vall);
    BSE_LAUNCH_CHECK();
  }
  // G_b = V_b^H V_b (rows above a block are zero in Vall), all blocks in one launch
  zgemm_batched(s, 1, 0, kBT, kBT, n, one, Vall, n, n * kBT, Vall, n, n * kBT, zero, Gall, kBT,
                int64_t(kBT) * kBT, int(nblk));
  larft_all_kernel<<<unsigned(nblk), kBT, 0, s>>>(Gall, tau, nref, Tall);
  BSE_LAUNCH_CHECK();
  // (V T)_b, all blocks in one launch
  zgemm_batched(s, 0, 0, n, kBT, kBT, one, Vall, n, n * kBT, Tall, kBT, int64_t(kBT) * kBT, zero,
                VTall, n, n * kBT, int(nblk));
}

void apply_prepared_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, z_t* Z,
                               int64_t ldz, int64_t ncols, void* ws) {
  if (nref <= 0 || ncols <= 0) return;
  const int off = reflector_offset(mode);
  const int64_t nblk = ceil_div(nref, kBT);
  const int64_t ncol = nblk * kBT;
  z_t* Vall = reinterpret_cast<z_t*>(ws);
  z_t* VTall = Vall + n * ncol;
  z_t* Gall = VTall + n * ncol;
  z_t* Tall = Gall + nblk * kBT * kBT;
  z_t* W1 = Tall + nblk * kBT * kBT;
  z_t* part = W1 + int64_t(kBT) * ncols;
  const int64_t part_elems = int64_t(16) * kBT * ncols;
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0}, mone = {-1.0, 0.0};
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t j0 = b * kBT;
    const int64_t r0 = j0 + off;  // first row any reflector of the block touches
    const int64_t m = n - r0;
    if (m <= 0) continue;
    const z_t* Vb = Vall + j0 * n + r0;
    const z_t* VTb = VTall + j0 * n + r0;
    z_t* Zb = Z + r0;
    // W1 = V_b^H Z (kBT x ncols, K = m; K-split on the under-filled grid)
    zgemm(s, 1, 0, kBT, ncols, m, one, Vb, n, Zb, ldz, zero, W1, kBT, kGeneral, kGeneral, 0, part,
          part_elems);
    // Z -= (V T)_b W1
    zgemm(s, 0, 0, m, ncols, kBT, mone, VTb, n, W1, kBT, one, Zb, ldz, kGeneral, kGeneral, 0,
          nullptr, 0);
  }
}

void apply_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                      int64_t lda, const z_t* tau, z_t* Z, int64_t ldz, int64_t ncols, void* ws) {
  if (nref <= 0 || ncols <= 0) return;
  prepare_reflectors(s, mode, n, nref, A, lda, tau, ws);
  apply_prepared_reflectors(s, mode, n, nref, Z, ldz, ncols, ws);
}

void zunmtr_lower(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau, z_t* Z,
                  int64_t ldz, int64_t ncols, void* ws) {
  apply_reflectors(s, 0, n, n - 1, A, lda, tau, Z, ldz, ncols, ws);
}

}  // namespace bseg
