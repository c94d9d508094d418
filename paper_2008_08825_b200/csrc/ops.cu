// ops.cu — bandwidth-bound glue kernels of the hot path (O(n^2) HBM traffic):
//   product_pair's M1 = A+B, M2 = A-B          (proj/src/core.cpp:88)
//   lambda_from_squares / clamp_singular        (proj/src/solvers.cpp:25-45, 69-88)
//   assemble_eigenvectors + rebuild_nonpositive (proj/src/core.cpp:102-127, solvers.cpp:53-65)
//   real D&C eigenvectors -> complex, TGK vector extraction for the SVD route.
#include <cfloat>

#include "blas.h"
#include "ops.h"

namespace bseg {

namespace {
inline int grid_for(int64_t total, int threads = 256) {
  return int(min64(ceil_div(total, threads), 148 * 16));
}
}  // namespace

__global__ void zaddsub_kernel(int64_t n, const z_t* __restrict__ A, int64_t lda,
                               const z_t* __restrict__ B, int64_t ldb, z_t* __restrict__ M1,
                               z_t* __restrict__ M2, int64_t ldm) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    // the inputs are read once: streaming loads (evict-first in L2, see assemble_kernel)
    const z_t a = __ldcs(A + i + j * lda), b = __ldcs(B + i + j * ldb);
    if (M1) M1[i + j * ldm] = zadd(a, b);
    if (M2) M2[i + j * ldm] = zsub(a, b);
  }
}

void zaddsub(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
             z_t* M1, z_t* M2, int64_t ldm) {
  zaddsub_kernel<<<grid_for(n * n), 256, 0, s>>>(n, A, lda, B, ldb, M1, M2, ldm);
  BSE_LAUNCH_CHECK();
}

__global__ void real_to_complex_kernel(int64_t rows, int64_t cols, const double* __restrict__ Z,
                                       int64_t ldz, z_t* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    out[i + j * ldo] = make_double2(__ldcs(Z + i + j * ldz), 0.0);
  }
}

void real_to_complex(cudaStream_t s, int64_t rows, int64_t cols, const double* Z, int64_t ldz,
                     z_t* out, int64_t ldo) {
  real_to_complex_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, Z, ldz, out, ldo);
  BSE_LAUNCH_CHECK();
}

// Single CTA. mode 0: lambda_from_squares(d) (d ascending, solvers.cpp:25-45);
// mode 1: clamp_singular_ascending(s) with s ASCENDING on input (solvers.cpp:69-88; the
// TGK route produces ascending singular values directly).
// Outputs: lambda (n), flagged list (ascending) + count, nonpositive list + count, status
// (0 ok, 1 = spectrum has no positive entry -> ConvergenceFailure), floor.
__global__ void __launch_bounds__(1024) clamp_kernel(int64_t n, const double* __restrict__ d,
                                                     int mode, double* __restrict__ lambda,
                                                     int64_t* __restrict__ flagged,
                                                     int64_t* __restrict__ nonpos,
                                                     int64_t* __restrict__ counts,
                                                     double* __restrict__ floor_out) {
  __shared__ int64_t base_f, base_p;
  __shared__ int wf[32], wp[32];
  const double dmax = d[n - 1];
  if (!(dmax > 0.0)) {
    if (threadIdx.x == 0) {
      counts[0] = 0;
      counts[1] = 0;
      counts[2] = 1;
    }
    return;
  }
  const double fl = mode == 0 ? DBL_EPSILON * sqrt(dmax) : DBL_EPSILON * dmax;
  if (threadIdx.x == 0) {
    base_f = 0;
    base_p = 0;
    *floor_out = fl;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    bool f = false, p = false;
    if (i < n) {
      const double di = d[i];
      double lam;
      if (mode == 0) {
        lam = di > 0.0 ? sqrt(di) : 0.0;
        p = !(di > 0.0);
      } else {
        lam = di;
      }
      if (lam < fl) {
        lam = fl;
        f = true;
      } else {
        p = false;
      }
      if (!f) p = false;
      lambda[i] = lam;
    }
    const unsigned bf = __ballot_sync(0xffffffffu, f), bp = __ballot_sync(0xffffffffu, p);
    if (lane == 0) {
      wf[wid] = __popc(bf);
      wp[wid] = __popc(bp);
    }
    __syncthreads();
    int64_t of = base_f, op = base_p;
    for (int w = 0; w < wid; ++w) {
      of += wf[w];
      op += wp[w];
    }
    const unsigned lm = (1u << lane) - 1u;
    if (f) flagged[of + __popc(bf & lm)] = i;
    if (p) nonpos[op + __popc(bp & lm)] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 0; w < nw; ++w) {
        base_f += wf[w];
        base_p += wp[w];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[0] = base_f;
    counts[1] = base_p;
    counts[2] = 0;
  }
}

void clamp_spectrum(cudaStream_t s, int64_t n, const double* d, int mode, double* lambda,
                    int64_t* flagged, int64_t* nonpos, int64_t* counts, double* floor_out) {
  clamp_kernel<<<1, 1024, 0, s>>>(n, d, mode, lambda, flagged, nonpos, counts, floor_out);
  BSE_LAUNCH_CHECK();
}

// assemble_eigenvectors (core.cpp:102-127) with per-column factors (lambda1, lambda2):
//   x = v1 * (l1/l2)^(1/4), y = v2 * (l2/l1)^(1/4), V = [(x+y)/2 ; (y-x)/2]
// and the breakdown rebuild (solvers.cpp:53-65) for columns whose squared eigenvalue d_j
// came out nonpositive (nonpos_mask: d != nullptr and d[j] <= 0): q = sqrt(mag) e^{i pi/4}
// with mag = max(sqrt|d_j|, floor), x = v1 q, y = v2 / q.
__global__ void assemble_kernel(int64_t n, int64_t k, const z_t* __restrict__ V1, int64_t ld1,
                                const z_t* __restrict__ V2, int64_t ld2,
                                const double* __restrict__ l1, const double* __restrict__ l2,
                                int l2_is_one, const double* __restrict__ dsq,
                                const double* __restrict__ floor_p, z_t* __restrict__ V,
                                int64_t ldv) {
  const int64_t total = n * k;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    // last use of V1 / V2 and the solve's output V (n x 2n: 512 MB at n = 4096): streaming
    // loads and stores, so they leave L2 first and the concurrent batch lanes keep their
    // working sets (a copy-engine D2H of V slowed the lanes by 5 % through L2 eviction)
    const z_t a = __ldcs(V1 + i + j * ld1), b = __ldcs(V2 + i + j * ld2);
    z_t x, y;
    if (dsq && !(dsq[j] > 0.0)) {
      const double mag = fmax(sqrt(fabs(dsq[j])), *floor_p);
      const double r = sqrt(mag) * 0.70710678118654752440;
      const z_t q = make_double2(r, r);
      x = zmul(a, q);
      // b / q
      const double den = q.x * q.x + q.y * q.y;
      y = make_double2((b.x * q.x + b.y * q.y) / den, (b.y * q.x - b.x * q.y) / den);
    } else {
      const double lam1 = l1[j], lam2 = l2_is_one ? 1.0 : l2[j];
      const double s1 = pow(lam1 / lam2, 0.25), s2 = pow(lam2 / lam1, 0.25);
      x = zscale(a, s1);
      y = zscale(b, s2);
    }
    __stcs(V + i + j * ldv, zscale(zadd(x, y), 0.5));
    __stcs(V + (n + i) + j * ldv, zscale(zsub(y, x), 0.5));
  }
}

void assemble(cudaStream_t s, int64_t n, int64_t k, const z_t* V1, int64_t ld1, const z_t* V2,
              int64_t ld2, const double* l1, const double* l2, int l2_is_one, const double* dsq,
              const double* floor_p, z_t* V, int64_t ldv) {
  assemble_kernel<<<grid_for(n * k), 256, 0, s>>>(n, k, V1, ld1, V2, ld2, l1, l2, l2_is_one, dsq,
                                                  floor_p, V, ldv);
  BSE_LAUNCH_CHECK();
}

// Validates the assemble_eigenvectors scale factors (NonPositiveScale, core.cpp:108-116).
__global__ void check_scales_kernel(int64_t k, const double* l1, const double* l2, int* bad) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k;
       j += int64_t(gridDim.x) * blockDim.x) {
    const double a = l1[j], b = l2[j];
    if (!(a > 0.0) || !(b > 0.0) || !isfinite(a) || !isfinite(b)) atomicMin(bad, int(j));
  }
}

void check_scales(cudaStream_t s, int64_t k, const double* l1, const double* l2, int* bad) {
  check_scales_kernel<<<grid_for(k), 256, 0, s>>>(k, l1, l2, bad);
  BSE_LAUNCH_CHECK();
}

// TGK route: eigenvectors X (2n x 2n real, ld 2n, ascending eigenvalues) of the Golub–Kahan
// tridiagonal with off-diagonal (d1, e1, d2, e2, ...). The top n columns (positive
// eigenvalues sigma ascending) hold x = [v1, u1, v2, u2, ...]/sqrt(2) interleaved.
// Outputs complex Ub = sqrt(2) x_odd, Vb = sqrt(2) x_even for column j (sigma_j ascending),
// each re-normalised separately (removes the +sigma/-sigma mixing for tiny sigma).
__global__ void tgk_extract_kernel(int64_t n, const double* __restrict__ X,
                                   z_t* __restrict__ Ub, int64_t ldu, z_t* __restrict__ Vb,
                                   int64_t ldv) {
  const int64_t j = blockIdx.x;  // one CTA per singular vector pair
  const double* x = X + (n + j) * (2 * n);
  __shared__ double red[32];
  double su = 0.0, sv = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = x[2 * i], b = x[2 * i + 1];
    sv += a * a;
    su += b * b;
  }
  su = block_sum(su, red);
  sv = block_sum(sv, red);
  const double ru = su > 0.0 ? 1.0 / sqrt(su) : 0.0, rv = sv > 0.0 ? 1.0 / sqrt(sv) : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    Vb[i + j * ldv] = make_double2(x[2 * i] * rv, 0.0);
    Ub[i + j * ldu] = make_double2(x[2 * i + 1] * ru, 0.0);
  }
}

void tgk_extract(cudaStream_t s, int64_t n, const double* X, z_t* Ub, int64_t ldu, z_t* Vb,
                 int64_t ldv) {
  tgk_extract_kernel<<<unsigned(n), 256, 0, s>>>(n, X, Ub, ldu, Vb, ldv);
  BSE_LAUNCH_CHECK();
}

// TGK tridiagonal: diag 0, off-diagonal interleaving d (n) and e (n-1).
__global__ void tgk_build_kernel(int64_t n, const double* __restrict__ d,
                                 const double* __restrict__ e, double* __restrict__ td,
                                 double* __restrict__ te) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < 2 * n;
       i += int64_t(gridDim.x) * blockDim.x) {
    td[i] = 0.0;
    if (i < 2 * n - 1) te[i] = (i % 2 == 0) ? d[i / 2] : e[i / 2];
  }
}

void tgk_build(cudaStream_t s, int64_t n, const double* d, const double* e, double* td,
               double* te) {
  tgk_build_kernel<<<grid_for(2 * n), 256, 0, s>>>(n, d, e, td, te);
  BSE_LAUNCH_CHECK();
}

// Relative-accuracy refinement of the bidiagonal singular values (ascending, in place).
// The TGK divide & conquer gives sigma to absolute accuracy eps*||B||; the reference's
// zbdsqr gives high RELATIVE accuracy, which CHOL+SVD needs for its small eigenvalues
// (test_solvers.cpp:188-199). Bisection on the Golub-Kahan matrix with
// the LDL^T Sturm count is relatively accurate (Demmel-Kahan; LAPACK dbdsvdx). One warp per
// singular value does 32-way multisection inside a bracket centred on the D&C value.
__device__ __forceinline__ int tgk_count_below(int64_t n, const double* __restrict__ a2, double x,
                                               double pivmin) {
  // #eigenvalues of T_GK (zero diagonal, off-diagonal^2 a2[0..2n-2]) below x
  int c = 0;
  double q = -x;
  if (fabs(q) < pivmin) q = -pivmin;
  c += q < 0.0;
  for (int64_t k = 1; k < 2 * n; ++k) {
    q = -x - a2[k - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

__global__ void tgk_a2_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ e,
                              double scale, double* __restrict__ a2) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < 2 * n - 1;
       k += int64_t(gridDim.x) * blockDim.x) {
    const double v = ((k & 1) ? e[k >> 1] : d[k >> 1]) / scale;
    a2[k] = v * v;
  }
}

__global__ void tgk_refine_kernel(int64_t n, const double* __restrict__ a2, double scale,
                                  double bound, double* __restrict__ sig) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double pivmin = 1e-290;
  const double s0 = sig[i] / scale;
  // The divide & conquer value is accurate to O(eps * bound) absolutely, i.e. to
  // O(128 eps) relatively for s0 >= bound / 128 -- zbdsqr's own relative tolerance is
  // ~100 eps -- so only the smaller singular values are refined.
  if (s0 >= bound * (1.0 / 128.0)) return;
  const double tau = 64.0 * DBL_EPSILON * bound;
  double lo = fmax(0.0, s0 - tau), hi = s0 + tau;
  // verify the bracket: #(sigma < lo) <= i < #(sigma < hi)
  {
    int c = 0;
    if (lane == 0) c = tgk_count_below(n, a2, lo, pivmin) - int(n);
    else if (lane == 1) c = tgk_count_below(n, a2, hi, pivmin) - int(n);
    warp_converge();
    const int clo = __shfl_sync(0xffffffffu, c, 0), chi = __shfl_sync(0xffffffffu, c, 1);
    if (!(clo <= i && chi >= i + 1)) {
      lo = 0.0;
      hi = bound * (1.0 + 4.0 * DBL_EPSILON);
    }
  }
  for (int it = 0; it < 40; ++it) {
    if (hi - lo <= 2.0 * DBL_EPSILON * fmax(lo, hi) || hi - lo <= pivmin) break;
    const double x = lo + (hi - lo) * double(lane + 1) / 33.0;
    const int c = tgk_count_below(n, a2, x, pivmin) - int(n);
    const unsigned ge = __ballot_sync(0xffffffffu, c >= i + 1);  // x above sigma_i
    const int first = ge ? __ffs(ge) - 1 : 32;
    const double nlo = first == 0 ? lo : lo + (hi - lo) * double(first) / 33.0;
    const double nhi = first == 32 ? hi : lo + (hi - lo) * double(first + 1) / 33.0;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) sig[i] = 0.5 * (lo + hi) * scale;
}

__global__ void absmax_kernel(int64_t n, const double* __restrict__ d, const double* __restrict__ e,
                              double* out) {
  __shared__ double red[32];
  double m = 0.0, g = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    m = fmax(m, fabs(d[k]));
    if (k < n - 1) m = fmax(m, fabs(e[k]));
    // Gershgorin bound of T_GK: |d_k| + |e_k|, |e_{k-1}| + |d_k|
    const double l = k > 0 ? fabs(e[k - 1]) : 0.0, r = k < n - 1 ? fabs(e[k]) : 0.0;
    g = fmax(g, fabs(d[k]) + fmax(l, r));
  }
  m = warp_max(m);
  g = warp_max(g);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) mm = fmax(mm, red[w]);
    out[0] = mm > 0.0 ? mm : 1.0;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g;
  __syncthreads();
  if (threadIdx.x == 0) {
    double gg = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) gg = fmax(gg, red[w]);
    out[1] = gg;
  }
}

void tgk_refine(cudaStream_t s, int64_t n, const double* d, const double* e, double* sig,
                double* scratch) {
  if (n <= 0) return;
  // scratch: [scale, gershgorin] + a2 (2n)
  absmax_kernel<<<1, 1024, 0, s>>>(n, d, e, scratch);
  BSE_LAUNCH_CHECK();
  double h[2];
  BSE_CUDA(cudaMemcpyAsync(h, scratch, sizeof(h), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  double* a2 = scratch + 2;
  tgk_a2_kernel<<<grid_for(2 * n), 256, 0, s>>>(n, d, e, h[0], a2);
  BSE_LAUNCH_CHECK();
  const int wpb = 8;
  tgk_refine_kernel<<<unsigned(ceil_div(n, wpb)), 32 * wpb, 0, s>>>(n, a2, h[0], h[1] / h[0], sig);
  BSE_LAUNCH_CHECK();
}

// Right-scale columns by r_j = 1/sqrt(lambda_j) (CHOL+SVD, solvers.cpp:152-156).
__global__ void scale_cols_rsqrt_kernel(int64_t rows, int64_t cols, z_t* __restrict__ X,
                                        int64_t ldx, const double* __restrict__ lam) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    X[i + j * ldx] = zscale(X[i + j * ldx], 1.0 / sqrt(lam[j]));
  }
}

void scale_cols_rsqrt(cudaStream_t s, int64_t rows, int64_t cols, z_t* X, int64_t ldx,
                      const double* lam) {
  scale_cols_rsqrt_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, X, ldx, lam);
  BSE_LAUNCH_CHECK();
}

__global__ void square_vec_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = a[i] * a[i];
}

void square_vec(cudaStream_t s, int64_t n, const double* a, double* b) {
  square_vec_kernel<<<grid_for(n), 256, 0, s>>>(n, a, b);
  BSE_LAUNCH_CHECK();
}

__global__ void reverse_real_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    b[i] = a[n - 1 - i];
}

void reverse_real(cudaStream_t s, int64_t n, const double* a, double* b) {
  reverse_real_kernel<<<grid_for(n), 256, 0, s>>>(n, a, b);
  BSE_LAUNCH_CHECK();
}

// Column reversal of a complex matrix (svd's descending convention <-> ascending).
__global__ void reverse_cols_kernel(int64_t rows, int64_t cols, const z_t* __restrict__ a,
                                    int64_t lda, z_t* __restrict__ b, int64_t ldb) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    b[i + j * ldb] = a[i + (cols - 1 - j) * lda];
  }
}

void reverse_cols(cudaStream_t s, int64_t rows, int64_t cols, const z_t* a, int64_t lda, z_t* b,
                  int64_t ldb) {
  reverse_cols_kernel<<<grid_for(rows * cols), 256, 0, s>>>(rows, cols, a, lda, b, ldb);
  BSE_LAUNCH_CHECK();
}

// Hermitian deviation check & symmetrisation of from_blocks (core.cpp:45-57): partial sums
// of |m|^2 and |m - m^H|^2 per CTA (deterministic second pass on host).
__global__ void herm_dev_kernel(int64_t n, const z_t* __restrict__ M, int64_t ld,
                                double* __restrict__ part) {
  __shared__ double red[32];
  double nrm = 0.0, dev = 0.0;
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    const z_t a = M[i + j * ld], b = M[j + i * ld];
    nrm += zabs2(a);
    const z_t d = make_double2(a.x - b.x, a.y + b.y);
    dev += zabs2(d);
  }
  nrm = block_sum(nrm, red);
  dev = block_sum(dev, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = nrm;
    part[2 * blockIdx.x + 1] = dev;
  }
}

void herm_dev_partials(cudaStream_t s, int64_t n, const z_t* M, int64_t ld, double* part,
                       int nblocks) {
  herm_dev_kernel<<<nblocks, 256, 0, s>>>(n, M, ld, part);
  BSE_LAUNCH_CHECK();
}

// Diagonal of A scaled by `f` (E = lower(M1) with a halved diagonal for the X + X^H form of
// the two-sided product).
__global__ void scale_diag_kernel(int64_t n, z_t* A, int64_t lda, double f) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    A[i + i * lda] = zscale(A[i + i * lda], f);
}

void scale_diag(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double f) {
  scale_diag_kernel<<<grid_for(n), 256, 0, s>>>(n, A, lda, f);
  BSE_LAUNCH_CHECK();
}

// M(i,j) = X(i,j) + conj(X(j,i)) for i >= j (the lower triangle of X + X^H; the strict upper
// triangle of M is not written). 32x32 tile pairs (I >= J): tile (J,I) is staged transposed
// through shared memory so both reads are coalesced.
__global__ void __launch_bounds__(256) herm_lower_sum_kernel(int64_t n, const z_t* __restrict__ X,
                                                             int64_t ldx, z_t* __restrict__ M,
                                                             int64_t ldm) {
  __shared__ z_t t[32][33];
  const int64_t nt = (n + 31) / 32;
  // blockIdx.x enumerates the lower tile pairs (I >= J) row by row
  const int64_t b = blockIdx.x;
  int64_t I = int64_t((sqrt(8.0 * double(b) + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  while (I * (I + 1) / 2 > b) --I;
  const int64_t J = b - I * (I + 1) / 2;
  if (I >= nt) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // stage X(J-tile rows, I-tile cols) : element (J*32 + tx, I*32 + ty + 8k) -> t[ty+8k][tx]
  for (int k = 0; k < 4; ++k) {
    const int64_t r = J * 32 + tx, c = I * 32 + ty + 8 * k;
    t[ty + 8 * k][tx] = (r < n && c < n) ? X[r + c * ldx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int k = 0; k < 4; ++k) {
    const int64_t i = I * 32 + tx, j = J * 32 + ty + 8 * k;
    if (i < n && j < n && i >= j) {
      // conj(X(j, i)) = conj(t[i - I*32][j - J*32])
      const z_t xt = t[tx][ty + 8 * k];
      const z_t x = X[i + j * ldx];
      M[i + j * ldm] = make_double2(x.x + xt.x, x.y - xt.y);
    }
  }
}

void herm_lower_sum(cudaStream_t s, int64_t n, const z_t* X, int64_t ldx, z_t* M, int64_t ldm) {
  if (n <= 0) return;
  const int64_t nt = (n + 31) / 32;
  herm_lower_sum_kernel<<<unsigned(nt * (nt + 1) / 2), 256, 0, s>>>(n, X, ldx, M, ldm);
  BSE_LAUNCH_CHECK();
}


// ------------------------------------------------------------ TGK vectors: small-sigma block
__global__ void count_small_sigma_kernel(int64_t n, const double* __restrict__ sasc,
                                         double tau, int* k) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double lim = tau * sasc[n - 1];
  int64_t c = 0;  // sasc ascending: the first index with sigma >= lim
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sasc[mid] < lim) lo = mid + 1;
    else hi = mid;
  }
  c = lo;
  *k = int(c);
}

__device__ __forceinline__ z_t block_zsum(z_t v, double* red) {  // red: 16 doubles
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  v = warp_zsum(v);
  __syncthreads();
  if (lane == 0) {
    red[2 * wid] = v.x;
    red[2 * wid + 1] = v.y;
  }
  __syncthreads();
  z_t s = make_double2(0.0, 0.0);
  for (int w = 0; w < nw; ++w) s = zadd(s, make_double2(red[2 * w], red[2 * w + 1]));
  return s;
}

// One CTA: the b columns of X (n x b; unit length on entry to the first pass) from the last to
// the first, each against the later ones of the block (modified Gram-Schmidt, two sweeps),
// then normalised; with `replace`, a column left with less than half of its length is first
// overwritten by a fixed pseudo-random vector.
__global__ void __launch_bounds__(256) block_mgs_kernel(int64_t n, int b, z_t* X, int64_t ld,
                                                        int replace, int64_t col0) {
  __shared__ double red[16];
  for (int jj = b - 1; jj >= 0; --jj) {
    z_t* xj = X + int64_t(jj) * ld;
    for (int sweep = 0; sweep < 2; ++sweep)
      for (int i = jj + 1; i < b; ++i) {
        const z_t* xi = X + int64_t(i) * ld;
        z_t d = make_double2(0.0, 0.0);
        for (int64_t r = threadIdx.x; r < n; r += blockDim.x) zcfma(d, xi[r], xj[r]);
        d = block_zsum(d, red);
        for (int64_t r = threadIdx.x; r < n; r += blockDim.x) xj[r] = zsub(xj[r], zmul(d, xi[r]));
      }
    double n1 = 0.0;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) n1 += zabs2(xj[r]);
    n1 = block_sum(n1, red);
    // the extracted columns have unit length: one that kept less than half of it through the
    // projections (here and the caller's against the later columns) is a combination of them
    if (replace && !(n1 >= 0.25)) {
      // collapsed onto later columns: a fixed pseudo-random direction (re-projected by the
      // caller's next pass against the columns after the block, and by this kernel again)
      for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
        // (seeded by the global column index: every replaced column gets its own direction)
        uint64_t h = uint64_t(r) * 0x9E3779B97F4A7C15ull ^
                     ((uint64_t(col0 + jj) + 1) * 0x632BE59BD9B4E019ull);
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        xj[r] = make_double2(double(int64_t(h >> 11) - (int64_t(1) << 52)) * 0x1.0p-52, 0.0);
      }
      n1 = 0.0;
      for (int64_t r = threadIdx.x; r < n; r += blockDim.x) n1 += zabs2(xj[r]);
      n1 = block_sum(n1, red);
      for (int sweep = 0; sweep < 2; ++sweep)
        for (int i = jj + 1; i < b; ++i) {
          const z_t* xi = X + int64_t(i) * ld;
          z_t d = make_double2(0.0, 0.0);
          for (int64_t r = threadIdx.x; r < n; r += blockDim.x) zcfma(d, xi[r], xj[r]);
          d = block_zsum(d, red);
          for (int64_t r = threadIdx.x; r < n; r += blockDim.x) xj[r] = zsub(xj[r], zmul(d, xi[r]));
        }
      n1 = 0.0;
      for (int64_t r = threadIdx.x; r < n; r += blockDim.x) n1 += zabs2(xj[r]);
      n1 = block_sum(n1, red);
    }
    const double sc = n1 > 0.0 ? 1.0 / sqrt(n1) : 0.0;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) xj[r] = zscale(xj[r], sc);
  }
}

void tgk_reorthogonalize(cudaStream_t s, int64_t n, const double* sasc, z_t* Ub, z_t* Vb,
                         int64_t ld, z_t* ws, int* kcount) {
  if (n <= 1) return;
  constexpr double kTau = 1e-3;  // below tau sigma_max the +-sigma mirror gap 2 sigma can
                                 // cost a TGK vector its accuracy (error ~ eps ||B|| / sigma)
  constexpr int kB = 32;
  count_small_sigma_kernel<<<1, 32, 0, s>>>(n, sasc, kTau, kcount);
  BSE_LAUNCH_CHECK();
  int k = 0;
  BSE_CUDA(cudaMemcpyAsync(&k, kcount, sizeof(int), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (k <= 0) return;
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0}, mone = {-1.0, 0.0};
  for (z_t* X : {Ub, Vb}) {
    for (int64_t top = k; top > 0; top -= kB) {  // block [j0, top), largest sigma first
      const int64_t j0 = max64(0, top - kB), b = top - j0, above = n - top;
      for (int rep = 0; rep < 2; ++rep) {
        for (int t = 0; t < 2 && above > 0; ++t) {  // CGS2 against the final columns [top, n)
          zgemm(s, 1, 0, above, b, n, one, X + top * ld, ld, X + j0 * ld, ld, zero, ws, above,
                0, 0, 0, nullptr, 0);  // general shapes
          zgemm(s, 0, 0, n, b, above, mone, X + top * ld, ld, ws, above, one, X + j0 * ld, ld,
                0, 0, 0, nullptr, 0);  // general shapes
        }
        block_mgs_kernel<<<1, 256, 0, s>>>(n, int(b), X + j0 * ld, ld, rep == 0, j0);
        BSE_LAUNCH_CHECK();
      }
    }
  }
}

}  // namespace bseg
