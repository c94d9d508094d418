// verify.cu — the reference's diagnostics on the device:
//   residual                  (proj/src/verify.cpp:76-93)  out_j = ||H v_j - lambda_j v_j|| / ||H||_F
//   sigma_orthogonality_error (verify.cpp:70-74)           ||V^H Sigma V - I||_F
//   check_form1 / check_form2 (verify.cpp:46-68)           J- and Sigma-form structure predicates
//   negative_spectrum         (proj/src/solvers.cpp:223-236) (lambda, [x; y]) -> (-lambda, [y; x])
//
// Validating an n = 16384 solution on the CPU costs ~32 n^3 flops; here the products are
// DMMA GEMMs (H V as four n x k x n blocks, V^H Sigma V as two k x k x n) and every norm is a
// fixed-order two-pass reduction (bit-deterministic).
#include <cmath>

#include "blas.h"
#include "context.h"
#include "gemm.cuh"

namespace bseg {

namespace {

constexpr int kRedBlocks = 1024;  // first-pass partials of the Frobenius-type reductions

__device__ __forceinline__ double block_sum_det(double v, double* red) {
  return block_sum(v, red);  // fixed order (common.cuh)
}

// partial[b] = sum over the block-strided elements of |X(i, j)|^2, X rows x cols
__global__ void sumsq_partials_kernel(int64_t rows, int64_t cols, const z_t* X, int64_t ldx,
                                      double* partial) {
  __shared__ double red[32];
  const int64_t total = rows * cols;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    acc += zabs2(X[i + j * ldx]);
  }
  const double s = block_sum_det(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out[0] = sum of partial[0..np)
__global__ void sum_final_kernel(const double* partial, int np, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
  const double s = block_sum_det(acc, red);
  if (threadIdx.x == 0) out[0] = s;
}

// ||G - I||^2 partials, G k x k
__global__ void dev_identity_partials_kernel(int64_t k, const z_t* G, int64_t ldg,
                                             double* partial) {
  __shared__ double red[32];
  const int64_t total = k * k;
  double acc = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % k, j = e / k;
    z_t g = G[i + j * ldg];
    if (i == j) g.x -= 1.0;
    acc += zabs2(g);
  }
  const double s = block_sum_det(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// one block per column j: out[j] = sqrt(sum_i |T1 - l v_top|^2 + |-T2 - l v_bot|^2) / normh
__global__ void residual_cols_kernel(int64_t n, int64_t k, const z_t* T1, const z_t* T2,
                                     int64_t ldt, const double* lam, const z_t* V, int64_t ldv,
                                     const double* sumsq_h, double* out) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  if (j >= k) return;
  const double l = lam[j];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const z_t t = T1[i + j * ldt], x = V[i + j * ldv];
    const z_t u = T2[i + j * ldt], y = V[n + i + j * ldv];
    const z_t r1 = make_double2(t.x - l * x.x, t.y - l * x.y);
    const z_t r2 = make_double2(-u.x - l * y.x, -u.y - l * y.y);
    acc += zabs2(r1) + zabs2(r2);
  }
  const double s = block_sum_det(acc, red);
  if (threadIdx.x == 0) out[j] = sqrt(s) / sqrt(2.0 * sumsq_h[0]);  // ||H||_F^2 = 2(|A|^2+|B|^2)
}

// form predicates on m (2h x 2h): sums of |J X J - m|^2, |Sigma m^H Sigma - m|^2, |m|^2
// with X = m^H (form 1) or m^T (form 2)
__global__ void form_partials_kernel(int form, int64_t h, const z_t* M, int64_t ldm,
                                     double* partial) {
  __shared__ double red[32];
  const int64_t m = 2 * h, total = m * m;
  double aj = 0.0, as = 0.0, an = 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const z_t mij = M[i + j * ldm];
    // (J X J)(i, j) = si * sj * X(p(i), q(j)); J = [0 I; -I 0]
    const int64_t pi = i < h ? i + h : i - h, qj = j < h ? j + h : j - h;
    const double si = i < h ? 1.0 : -1.0, sj = j < h ? -1.0 : 1.0;
    const z_t mqp = M[qj + pi * ldm];  // X(p, q) = (m^H or m^T)(p, q) from m(q, p)
    const z_t x = form == 1 ? zconj(mqp) : mqp;
    const z_t zj = zscale(x, si * sj);
    // (Sigma m^H Sigma)(i, j) = s_i s_j conj(m(j, i))
    const double ti = i < h ? 1.0 : -1.0, tj = j < h ? 1.0 : -1.0;
    const z_t zs = zscale(zconj(M[j + i * ldm]), ti * tj);
    aj += zabs2(zsub(zj, mij));
    as += zabs2(zsub(zs, mij));
    an += zabs2(mij);
  }
  const double s0 = block_sum_det(aj, red);
  __syncthreads();
  const double s1 = block_sum_det(as, red);
  __syncthreads();
  const double s2 = block_sum_det(an, red);
  if (threadIdx.x == 0) {
    partial[3 * blockIdx.x + 0] = s0;
    partial[3 * blockIdx.x + 1] = s1;
    partial[3 * blockIdx.x + 2] = s2;
  }
}

__global__ void sum3_final_kernel(const double* partial, int np, double* out) {
  __shared__ double red[32];
  for (int c = 0; c < 3; ++c) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[3 * i + c];
    const double s = block_sum_det(acc, red);
    if (threadIdx.x == 0) out[c] = s;
    __syncthreads();
  }
}

__global__ void negspec_kernel(int64_t n, int64_t k, const double* lam, const z_t* V,
                               int64_t ldv, double* lam_out, z_t* Vo, int64_t ldo) {
  const int64_t rows = 2 * n, total = rows * k;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    Vo[i + j * ldo] = V[(i < n ? i + n : i - n) + j * ldv];
    if (i == 0) lam_out[j] = -lam[j];
  }
}

int grid_for(int64_t total) { return int(std::min<int64_t>((total + 255) / 256, 148 * 32)); }

int red_blocks(int64_t total) { return int(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, kRedBlocks))); }

}  // namespace

size_t residual_workspace_bytes(int64_t n, int64_t k) {
  return 2 * size_t(n) * size_t(k) * sizeof(z_t) + (2 * kRedBlocks + 8) * sizeof(double) + 1024;
}

void residual_dev(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                  int64_t ldb, int64_t k, const double* lam, const z_t* V, int64_t ldv,
                  double* out, Bump& w) {
  if (k == 0) return;
  z_t* T1 = w.take<z_t>(size_t(n) * size_t(k));
  z_t* T2 = w.take<z_t>(size_t(n) * size_t(k));
  double* part = w.take<double>(2 * kRedBlocks + 8);
  double* nh = part + 2 * kRedBlocks;
  const z_t one = {1.0, 0.0}, zero = {0.0, 0.0};
  // ||H||_F^2 = 2 ||A||^2 + 2 ||B||^2 (verify.cpp:88): partials of A then B, one final sum
  const int nb = red_blocks(n * n);
  sumsq_partials_kernel<<<nb, 256, 0, s>>>(n, n, A, lda, part);
  BSE_LAUNCH_CHECK();
  sumsq_partials_kernel<<<nb, 256, 0, s>>>(n, n, B, ldb, part + nb);
  BSE_LAUNCH_CHECK();
  sum_final_kernel<<<1, 256, 0, s>>>(part, 2 * nb, nh);
  BSE_LAUNCH_CHECK();
  // T1 = A x + B y ; T2 = B x + A y  (H v = [T1; -T2], verify.cpp:84-86)
  const z_t* X = V;
  const z_t* Y = V + n;
  zgemm(s, 0, 0, n, k, n, one, A, lda, X, ldv, zero, T1, n, kGeneral, kGeneral, 0, nullptr, 0);
  zgemm(s, 0, 0, n, k, n, one, B, ldb, Y, ldv, one, T1, n, kGeneral, kGeneral, 0, nullptr, 0);
  zgemm(s, 0, 0, n, k, n, one, B, ldb, X, ldv, zero, T2, n, kGeneral, kGeneral, 0, nullptr, 0);
  zgemm(s, 0, 0, n, k, n, one, A, lda, Y, ldv, one, T2, n, kGeneral, kGeneral, 0, nullptr, 0);
  residual_cols_kernel<<<unsigned(k), 256, 0, s>>>(n, k, T1, T2, n, lam, V, ldv, nh, out);
  BSE_LAUNCH_CHECK();
}

size_t sigma_orth_workspace_bytes(int64_t k) {
  return size_t(k) * size_t(k) * sizeof(z_t) + (kRedBlocks + 8) * sizeof(double) + 1024;
}

void sigma_orth_dev(cudaStream_t s, int64_t h, int64_t k, const z_t* V, int64_t ldv,
                    double* d_out, Bump& w) {
  z_t* G = w.take<z_t>(size_t(k) * size_t(k));
  double* part = w.take<double>(kRedBlocks + 8);
  const z_t one = {1.0, 0.0}, mone = {-1.0, 0.0}, zero = {0.0, 0.0};
  // G = V^H Sigma V = X^H X - Y^H Y (verify.cpp:72)
  zgemm(s, 1, 0, k, k, h, one, V, ldv, V, ldv, zero, G, k, kGeneral, kGeneral, 0, nullptr, 0);
  zgemm(s, 1, 0, k, k, h, mone, V + h, ldv, V + h, ldv, one, G, k, kGeneral, kGeneral, 0, nullptr,
        0);
  const int nb = red_blocks(k * k);
  dev_identity_partials_kernel<<<nb, 256, 0, s>>>(k, G, k, part);
  BSE_LAUNCH_CHECK();
  sum_final_kernel<<<1, 256, 0, s>>>(part, nb, d_out);
  BSE_LAUNCH_CHECK();
}

size_t form_workspace_bytes() { return (3 * kRedBlocks + 8) * sizeof(double) + 1024; }

// d_out[0..2] = ||J X J - m||^2, ||Sigma m^H Sigma - m||^2, ||m||^2
void form_dev(cudaStream_t s, int form, int64_t h, const z_t* M, int64_t ldm, double* d_out,
              Bump& w) {
  double* part = w.take<double>(3 * kRedBlocks + 8);
  const int nb = red_blocks(4 * h * h);
  form_partials_kernel<<<nb, 256, 0, s>>>(form, h, M, ldm, part);
  BSE_LAUNCH_CHECK();
  sum3_final_kernel<<<1, 256, 0, s>>>(part, nb, d_out);
  BSE_LAUNCH_CHECK();
}

void negative_spectrum_dev(cudaStream_t s, int64_t n, int64_t k, const double* lam, const z_t* V,
                           int64_t ldv, double* lam_out, z_t* Vo, int64_t ldo) {
  if (k == 0) return;
  negspec_kernel<<<grid_for(2 * n * k), 256, 0, s>>>(n, k, lam, V, ldv, lam_out, Vo, ldo);
  BSE_LAUNCH_CHECK();
}

}  // namespace bseg
