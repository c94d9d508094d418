// solvers.cu — the two accelerated form-I BSE solvers as device pipelines.
//
//   CHOL      (Algorithm 2; bse::solve_chol, proj/src/solvers.cpp:119-135)
//   CHOL+SVD  (Algorithm 3; bse::solve_chol_svd, solvers.cpp:137-161)
//
// Orientation follows the reference: CHOL factors A-B = L L^H and forms
// M = L^H (A+B) L; CHOL+SVD forms C = L1^H L2 with L1 = chol(A+B), L2 = chol(A-B).
// product_pair's definiteness certificates (core.cpp:87-100) keep their order and error
// payloads; the certificate factor of A-B (CHOL) and both factors (CHOL+SVD) are reused
// instead of recomputed (the reference runs potrf 3x / 4x).
#include <nvtx3/nvToolsExt.h>

#include <cstdlib>
#include <cstring>

#include "blas.h"
#include "context.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "ops.h"
#include "svd.h"

namespace bseg {

namespace {

const z_t kOne = {1.0, 0.0}, kZero = {0.0, 0.0};

// Phase boundaries: CUDA events on the solve's stream (bse_phase_times) and one NVTX range
// per phase ("chol.reduce", ...; no-ops without a tool attached), so ncu can select a phase
// with --nvtx --nvtx-include "chol.reduce/".
constexpr const char* kPhaseNames[2][7] = {
    {"chol.product_pair", "chol.certify", "chol.triple", "chol.reduce", "chol.tridiag",
     "chol.backtransform", "chol.recover"},
    {"chol-svd.product_pair", "chol-svd.certify", "chol-svd.triple", "chol-svd.reduce",
     "chol-svd.tridiag", "chol-svd.backtransform", "chol-svd.recover"}};

struct PhaseClock {
  bse_ctx* c;
  const char* const* names;
  int k = 0;
  bool open = false;
  PhaseClock(bse_ctx* ctx, int method_row) : c(ctx), names(kPhaseNames[method_row]) { mark(); }
  ~PhaseClock() {
    if (open) nvtxRangePop();
  }
  void mark() {
    BSE_CUDA(cudaEventRecord(c->ev[k++], c->stream));
    if (open) nvtxRangePop();
    open = k <= 7;
    if (open) nvtxRangePushA(names[k - 1]);
  }
  float between(int a, int b) {
    float ms = 0.f;
    BSE_CUDA(cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]));
    return ms;
  }
};

}  // namespace

int64_t recover_chunk_cols(const bse_ctx* c, int64_t n, int64_t min_cols, int parts) {
  // two chunks: the first chunk's copy hides behind the second's compute; more chunks cost
  // more in narrower GEMMs / TRSM launch chains than they hide (measured 2/4/8)
  if (!c->sink_v) return n;
  const int64_t w = std::max<int64_t>(min_cols, ceil_div(ceil_div(n, parts), 64) * 64);
  return std::min<int64_t>(n, w);
}

void sink_columns(bse_ctx* c, const z_t* V, int64_t ldv, int64_t n, int64_t j0, int64_t jb) {
  if (!c->sink_v || jb <= 0) return;
  if (c->sink_k >= 16) throw std::runtime_error("too many sink chunks");
  cudaEvent_t ev = c->sink_ev[c->sink_k++];
  BSE_CUDA(cudaEventRecord(ev, c->stream));
  BSE_CUDA(cudaStreamWaitEvent(c->copy, ev, 0));
  BSE_CUDA(cudaMemcpy2DAsync(c->sink_v + 2 * j0 * c->sink_ldv, size_t(c->sink_ldv) * sizeof(z_t),
                             V + j0 * ldv, size_t(ldv) * sizeof(z_t), size_t(2 * n) * sizeof(z_t),
                             size_t(jb), cudaMemcpyDeviceToHost, c->copy));
}

bool sink_finish(bse_ctx* c) {
  if (!c->sink_v || c->sink_k == 0) return false;
  BSE_CUDA(cudaEventRecord(c->sink_ev[16], c->copy));
  BSE_CUDA(cudaStreamWaitEvent(c->stream, c->sink_ev[16], 0));
  return true;
}

namespace {

std::string pivot_msg(int info) {
  return "leading minor of order " + std::to_string(info) + " is not positive definite";
}

// product_pair certificates: potrf(M1) then potrf(M2) (core.cpp:89-99). The factors are
// returned in F1 / F2 (F1 may be null: certificate only, factored in the scratch S).
void certify(bse_ctx* c, int64_t n, z_t* F1, z_t* F2, int* info2) {
  cudaStream_t s = c->stream;
  (void)F1;
  (void)F2;
  int h[2];
  BSE_CUDA(cudaMemcpyAsync(h, info2, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (h[0] != 0)
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M1, int64_t(h[0]) - 1,
                      "A+B is not positive definite: " + pivot_msg(h[0])};
  if (h[1] != 0)
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, int64_t(h[1]) - 1,
                      "A-B is not positive definite: " + pivot_msg(h[1])};
  (void)n;
}

// Certificate of M1 = A + B for CHOL, where the factor itself is not needed (the reference
// factors it in product_pair, core.cpp:89-93, and discards it). M1 is congruent to
// M = L^H M1 L, so M1 is positive definite iff every eigenvalue of M is positive: the
// Cholesky of M1 only runs when the spectrum does not already certify it (or when M2 failed,
// to report M1 first as the reference does). Throws NotDefinite{M1} like core.cpp:91-93.
void certify_m1(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                z_t* m1, z_t* scratch, int* info0, z_t* ws) {
  cudaStream_t s = c->stream;
  zaddsub(s, n, A, lda, B, ldb, m1, scratch, n);
  zpotrf_lower(s, n, m1, n, info0, ws, false);
  int h = 0;
  BSE_CUDA(cudaMemcpyAsync(&h, info0, sizeof(int), cudaMemcpyDeviceToHost, s));
  BSE_CUDA(cudaStreamSynchronize(s));
  if (h != 0)
    throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M1, int64_t(h) - 1,
                      "A+B is not positive definite: " + pivot_msg(h)};
}

void read_flags(bse_ctx* c, int64_t n, const int64_t* d_counts, const int64_t* d_flagged,
                std::vector<int64_t>& flagged, const char* what_if_bad) {
  int64_t cnt[3];
  BSE_CUDA(cudaMemcpyAsync(cnt, d_counts, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  BSE_CUDA(cudaStreamSynchronize(c->stream));
  if (cnt[2] != 0) throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, what_if_bad};
  flagged.resize(size_t(cnt[0]));
  if (cnt[0] > 0)
    BSE_CUDA(cudaMemcpy(flagged.data(), d_flagged, sizeof(int64_t) * size_t(cnt[0]),
                        cudaMemcpyDeviceToHost));
  (void)n;
}

}  // namespace

size_t solve_workspace_bytes(int method, int64_t n) {
  const size_t nn = size_t(n) * size_t(n);
  size_t b = 0;
  if (method == BSE_METHOD_CHOL) {
    b += 4 * nn * sizeof(z_t);
    b += stedc_workspace_bytes(n) + nn * sizeof(double);
    b += tridiag_workspace_bytes(n) + unmtr_workspace_bytes(n, n);
    b += trsm_workspace_elems(n, n, 64) * sizeof(z_t);
  } else {
    b += 5 * nn * sizeof(z_t);
    const int64_t m = 2 * n;
    b += stedc_workspace_bytes(m) + size_t(m) * size_t(m) * sizeof(double);
    b += gebrd_workspace_bytes(n) + 2 * unmbr_workspace_bytes(n, n);
  }
  b += size_t(n) * 64 + (1 << 20);
  return b;
}

void solve_chol_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                    double* lam, z_t* V, int64_t ldv, std::vector<int64_t>& flagged) {
  cudaStream_t s = c->stream;
  Bump w = arena(c, solve_workspace_bytes(BSE_METHOD_CHOL, n));
  const size_t nn = size_t(n) * size_t(n);
  z_t* b0 = w.take<z_t>(nn);
  z_t* b1 = w.take<z_t>(nn);
  z_t* b2 = w.take<z_t>(nn);
  z_t* b3 = w.take<z_t>(nn);
  double* Z = w.take<double>(nn);
  void* ws_stedc = w.take<char>(stedc_workspace_bytes(n));
  void* ws_hetrd = w.take<char>(tridiag_workspace_bytes(n));
  void* ws_unmtr = w.take<char>(unmtr_workspace_bytes(n, n));
  z_t* ws_trsm = w.take<z_t>(trsm_workspace_elems(n, n, 64));
  double* d = w.take<double>(n);
  double* e = w.take<double>(n);
  z_t* tau = w.take<z_t>(n);
  int* info = w.take<int>(4);
  int64_t* flg = w.take<int64_t>(n);
  int64_t* nonpos = w.take<int64_t>(n);
  int64_t* counts = w.take<int64_t>(4);
  double* floor_p = w.take<double>(1);
  double* l1 = w.take<double>(n);
  const int64_t ld = n;

  z_t* ws_potrf2 = w.take<z_t>(64 * 64);
  PhaseClock clk(c, 0);
  // product_pair: M1 -> b0, M2 -> b1 and the factor L = chol(M2) (reused, solvers.cpp:121).
  // The certificate of M1 comes from the spectrum of M below (certify_m1).
  zaddsub(s, n, A, lda, B, ldb, b0, b1, ld);
  BSE_CUDA(cudaEventRecord(c->chol_ev, s));
  zpotrf_lower(s, n, b1, ld, info + 1, ws_trsm, false, c->la[0], c->la_ev);
  clk.mark();
  {
    int h = 0;
    BSE_CUDA(cudaMemcpyAsync(&h, info + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    BSE_CUDA(cudaStreamSynchronize(s));
    if (h != 0) {  // the reference certifies M1 first (core.cpp:89-99)
      certify_m1(c, n, A, lda, B, ldb, b2, b3, info + 0, ws_potrf2);
      throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, int64_t(h) - 1,
                        "A-B is not positive definite: " + pivot_msg(h)};
    }
    // strict certificates (bse_ctx_set_strict_certificates): the Cholesky of A+B on every
    // solve, exactly as product_pair does (core.cpp:89-93). The default certifies A+B from
    // the spectrum of L^H (A+B) L below (Sylvester's inertia: positive iff A+B is), which
    // can only differ from zpotrf's verdict when lambda_min(A+B) is within rounding of 0.
    if (c->strict_m1) certify_m1(c, n, A, lda, B, ldb, b2, b3, info + 0, ws_potrf2);
  }
  clk.mark();
  // M = L^H M1 L  (solvers.cpp:122-123), lower triangle only (zheevd reads 'L'), in the
  // Hermitian form M = X + X^H with X = L^H (E L), E = lower(M1) with a halved diagonal:
  // E L is lower x lower -> lower (n^3/6 complex MACs), L^H (E L) upper x lower (n^3/3),
  // against n^3/2 + n^3/3 for (L^H M1) L.
  scale_diag(s, n, b0, ld, 0.5);
  zgemm(s, 0, 0, n, n, n, kOne, b0, ld, b1, ld, kZero, b2, ld, kLowerOp, kLowerOp, 1, nullptr, 0);
  zgemm(s, 1, 0, n, n, n, kOne, b1, ld, b2, ld, kZero, b3, ld, kUpperOp, kLowerOp, 0, nullptr, 0);
  herm_lower_sum(s, n, b3, ld, b0, ld);
  clk.mark();
  // hermitian_eig(M) (solvers.cpp:124 -> backend.cpp:34): hetrd + D&C + back-transform
  tridiag_reduce(s, n, b0, ld, d, e, tau, ws_hetrd);
  clk.mark();
  // the back-transform's reflector blocks need only the reduction: built on the aux stream
  // while the divide & conquer runs (joined before the host sync below)
  fork(c);
  tridiag_back_prepare(c->aux, n, b0, ld, tau, ws_unmtr);
  dstedc(s, n, d, e, Z, ws_stedc, info + 2);
  join(c);
  {
    int h = 0;
    double dmin = 0.0;
    BSE_CUDA(cudaMemcpyAsync(&h, info + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
    BSE_CUDA(cudaMemcpyAsync(&dmin, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    BSE_CUDA(cudaStreamSynchronize(s));
    // M1 is certified by the spectrum when its smallest eigenvalue is positive; otherwise
    // factor it (b2, b3 are free here) and report NotDefinite{M1} as the reference would
    if (!c->strict_m1 && (h != 0 || !(dmin > 0.0)))
      certify_m1(c, n, A, lda, B, ldb, b3, b2, info + 0, ws_potrf2);
    if (h != 0)
      throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                        "zheevd failed to converge (info=" + std::to_string(h) + ")"};
  }
  clk.mark();
  real_to_complex(s, n, n, Z, n, b2, ld);
  tridiag_back(s, n, b0, ld, tau, ws_hetrd, b2, ld, n, ws_unmtr, true);
  clk.mark();
  // lambda_from_squares (solvers.cpp:125)
  clamp_spectrum(s, n, d, 0, lam, flg, nonpos, counts, floor_p);
  // l1 = lambda^2 (after clamping), l2 = 1 for the assembly below
  square_vec(s, n, lam, l1);
  // V1 = L^{-H} V_M (solvers.cpp:127) in b3 (aux stream) ; V2 = L V_M (solvers.cpp:128) in b0;
  // in column chunks when V streams to a host sink, so chunk q's copy overlaps chunk q+1
  const int64_t cw = recover_chunk_cols(c, n, 512, 2);
  for (int64_t j0 = 0; j0 < n; j0 += cw) {
    const int64_t jb = std::min<int64_t>(cw, n - j0);
    fork(c);
    zcopy2d(c->aux, n, jb, b2 + j0 * ld, ld, b3 + j0 * ld, ld);
    ztrsm_lower(c->aux, 0, 1, n, jb, b1, ld, b3 + j0 * ld, ld, ws_trsm, 64);
    zgemm(s, 0, 0, n, jb, n, kOne, b1, ld, b2 + j0 * ld, ld, kZero, b0 + j0 * ld, ld, kLowerOp,
          kGeneral, 0, nullptr, 0);
    join(c);
    // assemble with (lambda^2, 1) (solvers.cpp:130-133) + breakdown rebuild
    assemble(s, n, jb, b3 + j0 * ld, ld, b0 + j0 * ld, ld, l1 + j0, nullptr, 1, d + j0, floor_p,
             V + j0 * ldv, ldv);
    sink_columns(c, V, ldv, n, j0, jb);
  }
  clk.mark();
  read_flags(c, n, counts, flg, flagged, "squared-problem spectrum has no positive eigenvalue");
  bse_phase_times& t = c->last;
  t = bse_phase_times{};
  t.product_pair = clk.between(0, 1);
  {  // the factorisation of A-B alone (product_pair less the A+-B pass)
    float ms = 0.f;
    BSE_CUDA(cudaEventElapsedTime(&ms, c->chol_ev, c->ev[1]));
    t.cholesky = ms;
  }
  t.triple = clk.between(2, 3);
  t.reduce = clk.between(3, 4);
  t.tridiag = clk.between(4, 5);
  t.backtransform = clk.between(5, 6);
  t.recover = clk.between(6, 7);
  t.total = clk.between(0, 7);
}

void solve_chol_svd_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                        int64_t ldb, double* lam, z_t* V, int64_t ldv,
                        std::vector<int64_t>& flagged) {
  cudaStream_t s = c->stream;
  Bump w = arena(c, solve_workspace_bytes(BSE_METHOD_CHOL_SVD, n));
  const size_t nn = size_t(n) * size_t(n);
  const int64_t m2 = 2 * n;
  z_t* b0 = w.take<z_t>(nn);
  z_t* b1 = w.take<z_t>(nn);
  z_t* b2 = w.take<z_t>(nn);
  z_t* b3 = w.take<z_t>(nn);
  z_t* b4 = w.take<z_t>(nn);
  double* X = w.take<double>(size_t(m2) * size_t(m2));
  void* ws_stedc = w.take<char>(stedc_workspace_bytes(m2));
  void* ws_gebrd = w.take<char>(gebrd_workspace_bytes(n));
  void* ws_unmbr = w.take<char>(unmbr_workspace_bytes(n, n));
  void* ws_unmbr2 = w.take<char>(unmbr_workspace_bytes(n, n));
  z_t* ws_potrf2 = w.take<z_t>(64 * 64);
  double* d = w.take<double>(n);
  double* e = w.take<double>(n);
  double* td = w.take<double>(m2);
  double* te = w.take<double>(m2 + 8);
  z_t* tauq = w.take<z_t>(n);
  z_t* taup = w.take<z_t>(n);
  int* info = w.take<int>(4);
  int64_t* flg = w.take<int64_t>(n);
  int64_t* nonpos = w.take<int64_t>(n);
  int64_t* counts = w.take<int64_t>(4);
  double* floor_p = w.take<double>(1);
  double* sasc = w.take<double>(n);
  z_t* ws_potrf = w.take<z_t>(64 * 64);
  const int64_t ld = n;

  PhaseClock clk(c, 1);
  // product_pair + L1 = chol(M1), L2 = chol(M2) (solvers.cpp:138-140): b0 = L1, b1 = L2
  zaddsub(s, n, A, lda, B, ldb, b0, b1, ld);
  fork(c);
  zpotrf_lower(c->aux, n, b0, ld, info + 0, ws_potrf2, false, c->la[0], c->la_ev);
  zpotrf_lower(s, n, b1, ld, info + 1, ws_potrf, false, c->la[1], c->la_ev + 4);
  join(c);
  clk.mark();
  certify(c, n, b0, b1, info);
  clk.mark();
  // C = L1^H L2 (solvers.cpp:141): upper x lower, both triangles skipped
  zgemm(s, 1, 0, n, n, n, kOne, b0, ld, b1, ld, kZero, b2, ld, kUpperOp, kLowerOp, 0, nullptr, 0);
  clk.mark();
  // svd(C) (solvers.cpp:142): bidiagonalise, TGK divide & conquer, back-transform
  zgebrd_upper(s, n, b2, ld, d, e, tauq, taup, ws_gebrd);
  clk.mark();
  // reflector blocks of Q and P (reflectors only) on the aux stream beside the D&C
  fork(c);
  prepare_reflectors(c->aux, 1, n, n, b2, ld, tauq, ws_unmbr);
  prepare_reflectors(c->aux, 2, n, n - 1, b2, ld, taup, ws_unmbr2);
  tgk_build(s, n, d, e, td, te);
  dstedc(s, m2, td, te, X, ws_stedc, info + 2, n);  // only the positive half of the vectors
  join(c);
  clk.mark();
  // ascending singular values = top n TGK eigenvalues; vectors u (b3), v (b4)
  BSE_CUDA(cudaMemcpyAsync(sasc, td + n, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  tgk_refine(s, n, d, e, sasc, te);  // relative accuracy of the small singular values
  tgk_extract(s, n, X, b3, ld, b4, ld);
  // numerically small singular values: orthonormal U_B / V_B columns (X is free after the
  // extract; a no-op after one small count when every sigma >= 1e-3 sigma_max)
  tgk_reorthogonalize(s, n, sasc, b3, b4, ld, reinterpret_cast<z_t*>(X), info + 3);
  fork(c);
  apply_prepared_reflectors(s, 1, n, n, b3, ld, n, ws_unmbr);             // U = Q U_B
  apply_prepared_reflectors(c->aux, 2, n, n - 1, b4, ld, n, ws_unmbr2);   // V = P V_B
  join(c);
  clk.mark();
  {
    int h = 0;
    BSE_CUDA(cudaMemcpyAsync(&h, info + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
    BSE_CUDA(cudaStreamSynchronize(s));
    if (h != 0)
      throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                        "zgesvd failed to converge (" + std::to_string(h) + " superdiagonals unconverged)"};
  }
  // clamp_singular_ascending (solvers.cpp:145); s already ascending (no column reversal)
  clamp_spectrum(s, n, sasc, 1, lam, flg, nonpos, counts, floor_p);
  // V1 = L1 U diag(lam^-1/2) -> b2 ; V2 = L2 V diag(lam^-1/2) -> X (free after the extract);
  // in column chunks when V streams to a host sink
  z_t* v2 = reinterpret_cast<z_t*>(X);
  const int64_t cw = recover_chunk_cols(c, n, 512, 2);
  for (int64_t j0 = 0; j0 < n; j0 += cw) {
    const int64_t jb = std::min<int64_t>(cw, n - j0);
    zgemm(s, 0, 0, n, jb, n, kOne, b0, ld, b3 + j0 * ld, ld, kZero, b2 + j0 * ld, ld, kLowerOp,
          kGeneral, 0, nullptr, 0);
    zgemm(s, 0, 0, n, jb, n, kOne, b1, ld, b4 + j0 * ld, ld, kZero, v2 + j0 * ld, ld, kLowerOp,
          kGeneral, 0, nullptr, 0);
    scale_cols_rsqrt(s, n, jb, b2 + j0 * ld, ld, lam + j0);
    scale_cols_rsqrt(s, n, jb, v2 + j0 * ld, ld, lam + j0);
    // assemble with (lambda, lambda) -> unit scalings (solvers.cpp:158-160)
    assemble(s, n, jb, b2 + j0 * ld, ld, v2 + j0 * ld, ld, lam + j0, lam + j0, 0, nullptr,
             floor_p, V + j0 * ldv, ldv);
    sink_columns(c, V, ldv, n, j0, jb);
  }
  clk.mark();
  read_flags(c, n, counts, flg, flagged, "singular spectrum is identically zero");
  bse_phase_times& t = c->last;
  t = bse_phase_times{};
  t.product_pair = clk.between(0, 1);
  t.triple = clk.between(2, 3);
  t.reduce = clk.between(3, 4);
  t.tridiag = clk.between(4, 5);
  t.backtransform = clk.between(5, 6);
  t.recover = clk.between(6, 7);
  t.total = clk.between(0, 7);
}

}  // namespace bseg
