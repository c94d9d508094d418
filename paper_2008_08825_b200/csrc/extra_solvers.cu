// extra_solvers.cu — the reference's other two solvers and hpd_sqrt, composed from the same
// device primitives as the hot path:
//
//   SQRT      (Algorithm 1; bse::solve_sqrt, proj/src/solvers.cpp:94-117) with
//             hpd_sqrt (proj/src/backend.cpp:88-107): S = (A-B)^{1/2} from the Hermitian
//             eigendecomposition, M = S (A+B) S, lambda^2 = eig(M), V1 = S^{-1} V_M through
//             chol(S), V2 = S V_M, assembled like CHOL (same clamp / rebuild semantics).
//   REFERENCE (pencil oracle; bse::solve_reference, solvers.cpp:163-211): chol of the
//             Hermitian positive definite Sigma H = [A B; B A] (2n), K = L^{-1} Sigma L^{-H},
//             eig(K), inertia check, lambda = 1 / m over the positive half, v = L^{-H} w /
//             sqrt(m), ascending.
//
// Error payloads follow the reference: certificates of product_pair first (core.cpp:87-100),
// then NotDefinite(M2) wrapping hpd_sqrt's NotPositiveDefinite (solvers.cpp:96-101),
// NotDefinite(Full) for the Hamiltonian factor (solvers.cpp:172-177), ConvergenceFailure for
// the pencil inertia (solvers.cpp:190-196).
#include <cfloat>
#include <cmath>
#include <vector>

#include "blas.h"
#include "context.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "ops.h"

namespace bseg {

namespace {

const z_t kOne = {1.0, 0.0}, kZero = {0.0, 0.0};

// S = diag-scaled columns: X(:, j) *= sqrt(w_j)
__global__ void scale_cols_sqrt_kernel(int64_t rows, int64_t cols, z_t* X, int64_t ldx,
                                       const double* w) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    X[i + j * ldx] = zscale(X[i + j * ldx], sqrt(w[j]));
  }
}

// S <- (S + S^H) / 2 in place (pairs (i, j), i > j, handled by the lower element's thread)
__global__ void hermitize_kernel(int64_t n, z_t* S, int64_t ld) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    if (i < j) continue;
    if (i == j) {
      S[i + i * ld].y = 0.0;
      continue;
    }
    const z_t a = S[i + j * ld], b = S[j + i * ld];
    const z_t h = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));  // (a + conj(b)) / 2
    S[i + j * ld] = h;
    S[j + i * ld] = zconj(h);
  }
}

// ham = [A B; B A] (2n x 2n), Sig = diag(I, -I)
__global__ void build_ham_kernel(int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                                 z_t* H, int64_t ldh) {
  const int64_t m = 2 * n, total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const int64_t ii = i % n, jj = j % n;
    const bool diag_block = (i < n) == (j < n);
    H[i + j * ldh] = diag_block ? A[ii + jj * lda] : B[ii + jj * ldb];
  }
}

__global__ void signature_kernel(int64_t n, z_t* S, int64_t ld) {
  const int64_t m = 2 * n, total = m * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    S[i + j * ld] = make_double2(i == j ? (i < n ? 1.0 : -1.0) : 0.0, 0.0);
  }
}

// lambda(n-1-j) = 1 / m_j, V(:, n-1-j) = VW(:, j) / sqrt(m_j), m = positive eigenvalues (asc.)
__global__ void pencil_extract_kernel(int64_t n, const double* mpos, const z_t* VW, int64_t ldw,
                                      double* lam, z_t* V, int64_t ldv) {
  const int64_t rows = 2 * n, total = rows * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    const double mj = mpos[j];
    V[i + (n - 1 - j) * ldv] = zscale(VW[i + j * ldw], 1.0 / sqrt(mj));
    if (i == 0) lam[n - 1 - j] = 1.0 / mj;
  }
}

int grid_for(int64_t total) { return int(std::min<int64_t>((total + 255) / 256, 148 * 32)); }

void check_info(cudaStream_t s, const int* d_info, int code, int block, const std::string& pre,
                bool pivot_msg) {
  int h = 0;
  BSE_CUDA(cudaMemcpyAsync(&h, d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (h == 0) return;
  if (pivot_msg)
    throw DomainError{code, block, int64_t(h) - 1,
                      pre + "leading minor of order " + std::to_string(h) +
                          " is not positive definite"};
  throw DomainError{code, block, -1, pre + std::to_string(h) + ")"};
}

// product_pair certificates (core.cpp:89-99) on copies: M1 = A+B -> m1, M2 = A-B -> m2.
void product_pair_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                      int64_t ldb, z_t* m1, z_t* m2, z_t* f1, z_t* f2, Bump& w) {
  cudaStream_t s = c->stream;
  z_t* ws1 = w.take<z_t>(64 * 64);
  z_t* ws2 = w.take<z_t>(64 * 64);
  int* info = w.take<int>(2);
  zaddsub(s, n, A, lda, B, ldb, m1, m2, n);
  fork(c);
  zcopy2d(c->aux, n, n, m1, n, f1, n);
  zpotrf_lower(c->aux, n, f1, n, info + 0, ws1, false);
  zcopy2d(s, n, n, m2, n, f2, n);
  zpotrf_lower(s, n, f2, n, info + 1, ws2, false);
  join(c);
  int h[2];
  BSE_CUDA(cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (h[0] != 0)
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M1, int64_t(h[0]) - 1,
                      "A+B is not positive definite: leading minor of order " +
                          std::to_string(h[0]) + " is not positive definite"};
  if (h[1] != 0)
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, int64_t(h[1]) - 1,
                      "A-B is not positive definite: leading minor of order " +
                          std::to_string(h[1]) + " is not positive definite"};
}

}  // namespace

size_t heevd_workspace_bytes(int64_t n) {
  const size_t nn = size_t(n) * size_t(n);
  return nn * sizeof(double) + stedc_workspace_bytes(n) + tridiag_workspace_bytes(n) +
         unmtr_workspace_bytes(n, n) + size_t(n) * 48 + 8 * 256;
}

// zheevd('V','L') on the device (backend.cpp:28-45): M's lower triangle is read and
// destroyed; w ascending; Z (ldz) orthonormal vectors. Throws ConvergenceFailure.
void heevd_dev(cudaStream_t s, int64_t n, z_t* M, int64_t ldm, double* w, z_t* Z, int64_t ldz,
               Bump& b) {
  double* Zr = b.take<double>(size_t(n) * size_t(n));
  void* ws_st = b.take<char>(stedc_workspace_bytes(n));
  void* ws_ht = b.take<char>(tridiag_workspace_bytes(n));
  void* ws_um = b.take<char>(unmtr_workspace_bytes(n, n));
  double* e = b.take<double>(n);
  z_t* tau = b.take<z_t>(n);
  int* info = b.take<int>(1);
  tridiag_reduce(s, n, M, ldm, w, e, tau, ws_ht);
  dstedc(s, n, w, e, Zr, ws_st, info);
  real_to_complex(s, n, n, Zr, n, Z, ldz);
  tridiag_back(s, n, M, ldm, tau, ws_ht, Z, ldz, n, ws_um);
  check_info(s, info, BSE_ERR_CONVERGENCE_FAILURE, 0, "zheevd failed to converge (info=", false);
}

size_t hpd_sqrt_workspace_bytes(int64_t n) {
  return 2 * size_t(n) * size_t(n) * sizeof(z_t) + heevd_workspace_bytes(n) + size_t(n) * 8 + 1024;
}

// hpd_sqrt (backend.cpp:88-107): S = Q diag(sqrt(w)) Q^H, hermitized; M is not modified.
// Throws NotPositiveDefinite(i) for the first eigenvalue at or below eps * lambda_max.
void hpd_sqrt_dev(cudaStream_t s, int64_t n, const z_t* M, int64_t ldm, z_t* S, int64_t lds,
                  Bump& b) {
  z_t* Mw = b.take<z_t>(size_t(n) * size_t(n));
  z_t* Q = b.take<z_t>(size_t(n) * size_t(n));
  double* w = b.take<double>(n);
  zcopy2d(s, n, n, M, ldm, Mw, n);
  heevd_dev(s, n, Mw, n, w, Q, n, b);
  std::vector<double> hw(static_cast<size_t>(n));
  BSE_CUDA(cudaMemcpyAsync(hw.data(), w, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  const double floor = DBL_EPSILON * hw[size_t(n) - 1];
  for (int64_t i = 0; i < n; ++i) {
    if (!(hw[size_t(i)] > floor)) {
      char buf[256];
      snprintf(buf, sizeof(buf),
               "eigenvalue %g at index %lld is at or below eps*lambda_max = %g; matrix is not "
               "safely positive definite",
               hw[size_t(i)], (long long)i, floor);
      throw DomainError{BSE_ERR_NOT_POSITIVE_DEFINITE, 0, i, buf};
    }
  }
  // scaled = Q diag(sqrt(w)) in Mw ; S = scaled Q^H ; S = (S + S^H) / 2
  zcopy2d(s, n, n, Q, n, Mw, n);
  scale_cols_sqrt_kernel<<<grid_for(n * n), 256, 0, s>>>(n, n, Mw, n, w);
  BSE_LAUNCH_CHECK();
  zgemm(s, 0, 1, n, n, n, kOne, Mw, n, Q, n, kZero, S, lds, kGeneral, kGeneral, 0, nullptr, 0);
  hermitize_kernel<<<grid_for(n * n), 256, 0, s>>>(n, S, lds);
  BSE_LAUNCH_CHECK();
}

size_t solve_sqrt_workspace_bytes(int64_t n) {
  const size_t nn = size_t(n) * size_t(n);
  return 5 * nn * sizeof(z_t) + hpd_sqrt_workspace_bytes(n) + heevd_workspace_bytes(n) +
         trsm_workspace_elems(n, n, 64) * sizeof(z_t) + size_t(n) * 64 + (1 << 20);
}

void solve_sqrt_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                    double* lam, z_t* V, int64_t ldv, std::vector<int64_t>& flagged) {
  cudaStream_t s = c->stream;
  Bump w = arena(c, solve_sqrt_workspace_bytes(n));
  const size_t nn = size_t(n) * size_t(n);
  z_t* b0 = w.take<z_t>(nn);
  z_t* b1 = w.take<z_t>(nn);
  z_t* b2 = w.take<z_t>(nn);
  z_t* b3 = w.take<z_t>(nn);
  z_t* b4 = w.take<z_t>(nn);
  z_t* ws_trsm = w.take<z_t>(trsm_workspace_elems(n, n, 64));
  double* d = w.take<double>(n);
  double* l1 = w.take<double>(n);
  int64_t* flg = w.take<int64_t>(n);
  int64_t* nonpos = w.take<int64_t>(n);
  int64_t* counts = w.take<int64_t>(4);
  double* floor_p = w.take<double>(1);
  int* info = w.take<int>(1);
  z_t* ws_potrf = w.take<z_t>(64 * 64);
  const int64_t ld = n;
  // product_pair (solvers.cpp:95): M1 -> b0, M2 -> b1 (certificate factors in b2 / b3)
  product_pair_dev(c, n, A, lda, B, ldb, b0, b1, b2, b3, w);
  // S = hpd_sqrt(M2) -> b2 (solvers.cpp:96-101)
  try {
    hpd_sqrt_dev(s, n, b1, ld, b2, ld, w);
  } catch (const DomainError& e) {
    if (e.code != BSE_ERR_NOT_POSITIVE_DEFINITE) throw;
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, e.pivot,
                      "square root of A-B failed: " + e.msg};
  }
  // M = S (M1 S) -> b4 (solvers.cpp:102)
  zgemm(s, 0, 0, n, n, n, kOne, b0, ld, b2, ld, kZero, b3, ld, kGeneral, kGeneral, 0, nullptr, 0);
  zgemm(s, 0, 0, n, n, n, kOne, b2, ld, b3, ld, kZero, b4, ld, kGeneral, kGeneral, 0, nullptr, 0);
  // hermitian_eig(M) -> d, V_M in b0 (solvers.cpp:103)
  heevd_dev(s, n, b4, ld, d, b0, ld, w);
  // lambda_from_squares (solvers.cpp:104)
  clamp_spectrum(s, n, d, 0, lam, flg, nonpos, counts, floor_p);
  // V1 = S^{-1} V_M via chol(S) (solvers.cpp:106-109) -> b1 ; V2 = S V_M -> b4
  zcopy2d(s, n, n, b2, ld, b3, ld);
  zpotrf_lower(s, n, b3, ld, info, ws_potrf, false);
  check_info(s, info, BSE_ERR_NOT_POSITIVE_DEFINITE, 0, "", true);
  zcopy2d(s, n, n, b0, ld, b1, ld);
  ztrsm_lower(s, 0, 0, n, n, b3, ld, b1, ld, ws_trsm, 64);
  ztrsm_lower(s, 0, 1, n, n, b3, ld, b1, ld, ws_trsm, 64);
  zgemm(s, 0, 0, n, n, n, kOne, b2, ld, b0, ld, kZero, b4, ld, kGeneral, kGeneral, 0, nullptr, 0);
  // assemble with (lambda^2, 1) + breakdown rebuild (solvers.cpp:112-115)
  square_vec(s, n, lam, l1);
  assemble(s, n, n, b1, ld, b4, ld, l1, nullptr, 1, d, floor_p, V, ldv);
  int64_t cnt[3];
  BSE_CUDA(cudaMemcpyAsync(cnt, counts, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (cnt[2] != 0)
    throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                      "squared-problem spectrum has no positive eigenvalue"};
  flagged.resize(size_t(cnt[0]));
  if (cnt[0] > 0)
    BSE_CUDA(cudaMemcpy(flagged.data(), flg, sizeof(int64_t) * size_t(cnt[0]),
                        cudaMemcpyDeviceToHost));
  c->last = bse_phase_times{};
}

size_t solve_reference_workspace_bytes(int64_t n) {
  const size_t nn = size_t(n) * size_t(n), m = 2 * size_t(n);
  return 4 * nn * sizeof(z_t) + 3 * m * m * sizeof(z_t) + heevd_workspace_bytes(2 * n) +
         trsm_workspace_elems(2 * n, 2 * n, 64) * sizeof(z_t) + m * 16 + (1 << 20);
}

void solve_reference_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                         int64_t ldb, double* lam, z_t* V, int64_t ldv,
                         std::vector<int64_t>& flagged) {
  cudaStream_t s = c->stream;
  Bump w = arena(c, solve_reference_workspace_bytes(n));
  const size_t nn = size_t(n) * size_t(n);
  const int64_t m = 2 * n;
  const size_t mm = size_t(m) * size_t(m);
  z_t* m1 = w.take<z_t>(nn);
  z_t* m2 = w.take<z_t>(nn);
  z_t* f1 = w.take<z_t>(nn);
  z_t* f2 = w.take<z_t>(nn);
  z_t* L = w.take<z_t>(mm);
  z_t* K = w.take<z_t>(mm);
  z_t* Q = w.take<z_t>(mm);
  z_t* ws_trsm = w.take<z_t>(trsm_workspace_elems(m, m, 64));
  double* ev = w.take<double>(m);
  int* info = w.take<int>(1);
  z_t* ws_potrf = w.take<z_t>(64 * 64);
  // definiteness gate (solvers.cpp:164)
  product_pair_dev(c, n, A, lda, B, ldb, m1, m2, f1, f2, w);
  // chol(Sigma H) (solvers.cpp:167-177)
  build_ham_kernel<<<grid_for(int64_t(mm)), 256, 0, s>>>(n, A, lda, B, ldb, L, m);
  BSE_LAUNCH_CHECK();
  zpotrf_lower(s, m, L, m, info, ws_potrf, false);
  check_info(s, info, BSE_ERR_NOT_DEFINITE, BSE_BLOCK_FULL,
             "BSE Hamiltonian is not positive definite: ", true);
  // K = L^{-1} Sigma L^{-H} (solvers.cpp:179-182)
  signature_kernel<<<grid_for(int64_t(mm)), 256, 0, s>>>(n, K, m);
  BSE_LAUNCH_CHECK();
  ztrsm_lower(s, 0, 0, m, m, L, m, K, m, ws_trsm, 64);
  ztrsm_lower(s, 1, 1, m, m, L, m, K, m, ws_trsm, 64);
  heevd_dev(s, m, K, m, ev, Q, m, w);
  // inertia (solvers.cpp:184-196)
  std::vector<double> h(static_cast<size_t>(m));
  BSE_CUDA(cudaMemcpyAsync(h.data(), ev, sizeof(double) * size_t(m), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  int64_t n_pos = 0;
  for (double x : h) n_pos += (x > 0.0);
  if (n_pos != n)
    throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                      "pencil inertia is off: expected " + std::to_string(n) +
                          " positive eigenvalues, found " + std::to_string(n_pos)};
  // v = L^{-H} w / sqrt(m), lambda = 1 / m, ascending (solvers.cpp:198-210)
  z_t* W = Q + int64_t(n) * m;  // right n columns
  ztrsm_lower(s, 0, 1, m, n, L, m, W, m, ws_trsm, 64);
  pencil_extract_kernel<<<grid_for(m * n), 256, 0, s>>>(n, ev + n, W, m, lam, V, ldv);
  BSE_LAUNCH_CHECK();
  BSE_CUDA(cudaStreamSynchronize(s));
  flagged.clear();
  c->last = bse_phase_times{};
}

}  // namespace bseg
