/*
 * bse_gpu.h — C-ABI drop-in boundary of the B200-native form-I BSE eigensolver.
 *
 * The reference (`bsesolve`, /root/reference/proj) is C++20 that calls LAPACKE/CBLAS
 * directly from proj/src/backend.cpp. This header is the FFI a C, C++, Python (ctypes)
 * or any other host binds instead: plain pointers, 64-bit sizes, column-major
 * interleaved complex128 (re, im) arrays with leading dimensions — exactly the memory
 * layout of Eigen::MatrixXcd used by the reference (types.hpp:17-18). No torch or CUDA
 * types appear in any signature.
 *
 * Every entry point returns a bse_status_code and fills *st (may be NULL) with the
 * payload of the reference's exception hierarchy (types.hpp:33-126). The C++ drop-in
 * layer (include/bse/ *.hpp) rethrows the identical exception classes.
 *
 * Host-pointer entry points copy host->device, run entirely on the GPU bound to the
 * context, and copy results back before returning (synchronous, like the reference).
 * The *_device variants take device pointers and enqueue on the context's stream; their
 * complex128 matrix operands must be 16-byte aligned (BSE_ERR_INVALID_SPEC otherwise).
 */
#ifndef BSE_GPU_H
#define BSE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSE_GPU_ABI_VERSION 1

/* Status codes: one per reference exception class (types.hpp:33-126, core.cpp:28-42). */
typedef enum bse_status_code {
  BSE_OK = 0,
  BSE_ERR_GENERIC = 1,                /* bse::Error                                  */
  BSE_ERR_DIMENSION_MISMATCH = 2,     /* bse::DimensionMismatch     types.hpp:39-42  */
  BSE_ERR_NOT_HERMITIAN = 3,          /* bse::NotHermitian          types.hpp:44-52  */
  BSE_ERR_NOT_DEFINITE = 4,           /* bse::NotDefinite{block}    types.hpp:63-71  */
  BSE_ERR_NOT_POSITIVE_DEFINITE = 5,  /* bse::NotPositiveDefinite{pivot} :73-82      */
  BSE_ERR_CONVERGENCE_FAILURE = 6,    /* bse::ConvergenceFailure    types.hpp:84-87  */
  BSE_ERR_SINGULAR_FACTOR = 7,        /* bse::SingularFactor        types.hpp:89-92  */
  BSE_ERR_NON_POSITIVE_SCALE = 8,     /* bse::NonPositiveScale      types.hpp:94-97  */
  BSE_ERR_INVALID_SPEC = 9,           /* bse::InvalidSpec           types.hpp:109-112 */
  BSE_ERR_ODD_DIMENSION = 10,         /* bse::OddDimension          types.hpp:99-102  */
  BSE_ERR_LENGTH_MISMATCH = 11,       /* bse::LengthMismatch        types.hpp:104-107 */
  BSE_ERR_CUDA = 20,                  /* device/runtime failure (no reference analogue) */
  BSE_ERR_OUT_OF_MEMORY = 21,
  BSE_ERR_NO_DEVICE = 22
} bse_status_code;

/* Block tags of NotDefinite (types.hpp:55-61). */
typedef enum bse_block { BSE_BLOCK_M1 = 0, BSE_BLOCK_M2 = 1, BSE_BLOCK_FULL = 2 } bse_block;

/* Method (types.hpp:130). Only CHOL and CHOL_SVD are accelerated. */
typedef enum bse_method {
  BSE_METHOD_SQRT = 0,
  BSE_METHOD_CHOL = 1,
  BSE_METHOD_CHOL_SVD = 2,
  BSE_METHOD_REFERENCE = 3
} bse_method;

/* backend.hpp:31-40 */
typedef enum bse_op { BSE_OP_NONE = 0, BSE_OP_ADJOINT = 1 } bse_op;
typedef enum bse_shape { BSE_SHAPE_GENERAL = 0, BSE_SHAPE_LOWER = 1, BSE_SHAPE_UPPER = 2 } bse_shape;
typedef enum bse_side { BSE_SIDE_LEFT = 0, BSE_SIDE_RIGHT = 1 } bse_side;

typedef struct bse_status {
  int32_t code;               /* bse_status_code                                        */
  int32_t block;              /* bse_block, valid for BSE_ERR_NOT_DEFINITE               */
  int64_t pivot_index;        /* zero-based, valid for BSE_ERR_NOT_POSITIVE_DEFINITE     */
  double relative_deviation;  /* valid for BSE_ERR_NOT_HERMITIAN                         */
  char message[256];          /* what() of the corresponding reference exception         */
} bse_status;

/* Per-phase device timings of the last solve (CUDA events on the context stream), ms. */
typedef struct bse_phase_times {
  double product_pair;  /* M1=A+B, M2=A-B + Cholesky certificates                       */
  double cholesky;      /* CHOL: the Cholesky factorisation of A-B alone (inside product_pair) */
  double triple;        /* CHOL: M = L^H M1 L ;  CHOL+SVD: C = L1^H L2                    */
  double reduce;        /* hetrd (CHOL) / gebrd (CHOL+SVD)                                */
  double tridiag;       /* tridiagonal divide & conquer                                   */
  double backtransform; /* unmtr / unmbr                                                  */
  double recover;       /* TRSM/TRMM + scaling + assembly                                 */
  double total;
  /* Live per-kernel timing (CUDA events on the context stream around each launch):      */
  double panel_ms;      /* sum over the reduction panel kernels (hetrd / gebrd)           */
  double panel_launches;
  double panel_bytes;   /* algorithmic HBM bytes those launches must stream               */
  double gemm_ms;       /* sum over DMMA GEMM launches of the solve                        */
  double gemm_launches;
  double gemm_flops;    /* complex-equivalent real flops of those GEMM launches (8 per      */
                        /* complex MAC executed, triangular skipping counted)               */
  double gemm_dmma_flops; /* real flops the FP64 tensor pipe executed for them (the 3M      */
                        /* kernels issue 3 real DMMA MACs per complex MAC: 6 flops)         */
} bse_phase_times;

/* ---------------------------------------------------------------- context */
typedef struct bse_ctx bse_ctx;

/* Creates a context bound to CUDA device `device` with its own stream and workspace arena. */
int bse_ctx_create(bse_ctx** ctx, int device, bse_status* st);
int bse_ctx_destroy(bse_ctx* ctx);
/* Stream the *_device entry points enqueue on (cudaStream_t, as void*). */
void* bse_ctx_stream(bse_ctx* ctx);
/* Per-phase timings of the most recent solve on this context (zeros before the first). */
int bse_ctx_last_phase_times(bse_ctx* ctx, bse_phase_times* out);
/* Number of kernels this library launched on the context (and its batch lanes) since creation. */
int64_t bse_ctx_kernel_launches(bse_ctx* ctx);
/* Enables CUDA-event timing of the panel and GEMM kernels (fills panel_ and gemm_ fields). */
int bse_ctx_set_kernel_timing(bse_ctx* ctx, int enable);
/* Frees the cached workspace arena (it is otherwise reused across calls). */
int bse_ctx_release_workspace(bse_ctx* ctx);
int bse_abi_version(void);
/* Process-wide choice of the Householder tridiagonalisation inside every Hermitian
 * eigen-decomposition (zheevd replacement, backend.cpp:34): 0 = one-stage cooperative panels
 * (default), 1 = two-stage (dense -> band -> tridiagonal, n >= 128). The initial
 * value comes from the environment variable BSE_TWO_STAGE. Returns the previous mode. */
int bse_set_tridiagonal_reduction(int mode);

/* ---------------------------------------------------------------- solvers
 * Replace bse::solve_chol (solvers.cpp:119-135), bse::solve_chol_svd (solvers.cpp:137-161)
 * and the dispatcher bse::solve (solvers.cpp:213-221). Inputs are the validated blocks of
 * a BseMatrixI (from_blocks, core.cpp:61-75, is done by the host layer).
 *   lambda         : n doubles, ascending (SpectralResult::lambda)
 *   v              : 2n x n complex, column-major, leading dimension ldv >= 2n
 *   near_singular  : capacity n; receives the flagged (clamped) indices, ascending
 *   n_near_singular: number written
 * BSE_METHOD_CHOL and BSE_METHOD_CHOL_SVD are the hot path; BSE_METHOD_SQRT (bse::solve_sqrt,
 * solvers.cpp:94-117) and BSE_METHOD_REFERENCE (the pencil oracle bse::solve_reference,
 * solvers.cpp:163-211) are composed from the same device primitives (SURVEY §8f rows f2,
 * f3). Unknown methods return BSE_ERR_INVALID_SPEC.                                       */
int bse_solve(bse_ctx* ctx, int method, int64_t n,
              const double* a, int64_t lda, const double* b, int64_t ldb,
              double* lambda, double* v, int64_t ldv,
              int64_t* near_singular, int64_t* n_near_singular, bse_status* st);

/* Same, device pointers (a, b, lambda, v on the context's device); near_singular stays a
 * host array. a, b and v must be 16-byte aligned (complex128 vectors; any cudaMalloc'd
 * pointer is), else BSE_ERR_INVALID_SPEC. Synchronous at return. */
int bse_solve_device(bse_ctx* ctx, int method, int64_t n,
                     const double* d_a, int64_t lda, const double* d_b, int64_t ldb,
                     double* d_lambda, double* d_v, int64_t ldv,
                     int64_t* near_singular, int64_t* n_near_singular, bse_status* st);

/* Batch driver: solves `batch` independent matrices with the same
 * method and shape from host buffers a[i], b[i] into lambda[i], v[i]. The upload of matrix
 * i+1 and the download of matrix i-1 run on copy streams while matrix i computes, so with
 * page-locked host buffers the PCIe traffic hides behind the solves. A page-locked v[i] is
 * written by a small streaming-copy kernel (evict-first loads, stores straight over PCIe)
 * rather than the copy engine, whose 512 MB-per-item reads pass through L2 and evict the
 * other solves' working sets; pageable outputs take cudaMemcpy. Items run on
 * bse_ctx_set_batch_lanes() lanes (default 4 solves in flight, item i on lane i % lanes).
 *   near_singular  : null or capacity batch*n (row i holds matrix i's flagged indices)
 *   n_near_singular: null or capacity batch
 *   failed_index   : null or receives the first failing item (-1 when all succeed); the
 *                    error payload in st is that item's, earlier items' outputs are valid */
int bse_solve_batched(bse_ctx* ctx, int method, int64_t n, int64_t batch,
                      const double* const* a, int64_t lda, const double* const* b, int64_t ldb,
                      double* const* lambda, double* const* v, int64_t ldv,
                      int64_t* near_singular, int64_t* n_near_singular, int64_t* failed_index,
                      bse_status* st);

/* Same over device pointers (a[i], b[i], lambda[i], v[i] on the context's device), e.g. a
 * batch already resident in HBM. Synchronous at return. */
int bse_solve_batched_device(bse_ctx* ctx, int method, int64_t n, int64_t batch,
                             const double* const* d_a, int64_t lda, const double* const* d_b,
                             int64_t ldb, double* const* d_lambda, double* const* d_v,
                             int64_t ldv, int64_t* near_singular, int64_t* n_near_singular,
                             int64_t* failed_index, bse_status* st);
/* Solves in flight per batch call, 1..8 (default 4; fewer when device memory is short: each
 * lane needs its own workspace). With L > 1 the batch runs on L contexts
 * at once (L - 1 created on first use) and each cooperative panel kernel is limited to 1/L of
 * the SMs, so one solve's latency-bound reductions overlap another's GEMM phases. */
int bse_ctx_set_batch_lanes(bse_ctx* ctx, int lanes);

/* CHOL's certificate of A+B (product_pair, core.cpp:87-100). Default (0): A-B is factored
 * (L, reused as in solvers.cpp:121) and A+B is certified by the spectrum of L^H (A+B) L,
 * which is positive iff A+B is (Sylvester's law of inertia); the Cholesky of A+B runs only
 * when that spectrum has an entry <= 0 or A-B failed, so NotDefinite{M1|M2}, its block and
 * pivot are reported as the reference reports them. The two certificates can disagree only
 * when lambda_min(A+B) is within rounding of zero. 1 = strict: the Cholesky of A+B runs on
 * every CHOL solve, as the reference's product_pair does (one extra potrf, ~5% of a solve).
 * Inherited by the context's batch lanes.                                                */
int bse_ctx_set_strict_certificates(bse_ctx* ctx, int enable);

/* ---------------------------------------------------------------- core glue (core.cpp) */
/* product_pair (core.cpp:87-100): m1 = a+b, m2 = a-b, each certified by Cholesky.     */
int bse_product_pair(bse_ctx* ctx, int64_t n, const double* a, int64_t lda,
                     const double* b, int64_t ldb, double* m1, double* m2, bse_status* st);

/* assemble_eigenvectors (core.cpp:102-127): v1, v2 n x k; lambda1, lambda2 k; v 2n x k. */
int bse_assemble_eigenvectors(bse_ctx* ctx, int64_t n, int64_t k,
                              const double* v1, int64_t ldv1, const double* v2, int64_t ldv2,
                              const double* lambda1, const double* lambda2,
                              double* v, int64_t ldv, bse_status* st);

/* The eigenvector recovery tail of bse::solve_chol / solve_sqrt (solvers.cpp:125, 130-133):
 * lambda_from_squares(d) (solvers.cpp:25-45: lambda = sqrt(d), clamped at eps*sqrt(d_max)
 * and flagged), assemble_eigenvectors with factors (lambda^2, 1) (core.cpp:102-127), then
 * rebuild_nonpositive_columns (solvers.cpp:53-65) for every d_j <= 0. v1, v2 n x k; d k
 * (ascending); lambda k; v 2n x k; near_singular capacity k. BSE_ERR_CONVERGENCE_FAILURE
 * when d_max <= 0. This is the device code the CHOL solve runs after its eigensolve,
 * exposed so the breakdown rebuild can be checked column by column against the oracle. */
int bse_assemble_from_squares(bse_ctx* ctx, int64_t n, int64_t k,
                              const double* v1, int64_t ldv1, const double* v2, int64_t ldv2,
                              const double* d, double* lambda, double* v, int64_t ldv,
                              int64_t* near_singular, int64_t* n_near_singular, bse_status* st);

/* ---------------------------------------------------------------- dense backend (backend.cpp) */
/* cholesky_lower (backend.cpp:47-62): zpotrf 'L'; strict upper of l zeroed.             */
int bse_cholesky_lower(bse_ctx* ctx, int64_t n, const double* m, int64_t ldm,
                       double* l, int64_t ldl, bse_status* st);

/* matmul (backend.cpp:131-175): c (rows x cols) = op_a(a) * op_b(b).
 * a is ar x ac, b is br x bc (as stored); triangular hints skip known-zero regions.    */
int bse_matmul(bse_ctx* ctx, int64_t ar, int64_t ac, const double* a, int64_t lda,
               int op_a, int shape_a,
               int64_t br, int64_t bc, const double* b, int64_t ldb, int op_b, int shape_b,
               double* c, int64_t ldc, bse_status* st);

/* tri_solve (backend.cpp:109-129): solves op(L) X = rhs (left) or X op(L) = rhs (right).
 * L is n x n lower; rhs is rows x cols.                                                  */
int bse_tri_solve(bse_ctx* ctx, int64_t n, const double* l, int64_t ldl,
                  int64_t rows, int64_t cols, const double* rhs, int64_t ldr,
                  int side, int op, double* x, int64_t ldx, bse_status* st);

/* hermitian_eig (backend.cpp:28-45): zheevd 'V','L' semantics — reads the LOWER triangle
 * only; values ascending; vectors orthonormal.                                           */
int bse_hermitian_eig(bse_ctx* ctx, int64_t n, const double* m, int64_t ldm,
                      double* values, double* vectors, int64_t ldv, bse_status* st);

/* svd (backend.cpp:64-86): zgesvd 'A','A' semantics; s descending; v (not v^H).         */
int bse_svd(bse_ctx* ctx, int64_t n, const double* m, int64_t ldm,
            double* u, int64_t ldu, double* s, double* v, int64_t ldv, bse_status* st);

/* hpd_sqrt (backend.cpp:88-107): s = m^{1/2} for Hermitian positive definite m (lower
 * triangle read); BSE_ERR_NOT_POSITIVE_DEFINITE (pivot_index = eigenvalue index) when an
 * eigenvalue is at or below eps * lambda_max.                                             */
int bse_hpd_sqrt(bse_ctx* ctx, int64_t n, const double* m, int64_t ldm, double* s, int64_t lds,
                 bse_status* st);

/* ---------------------------------------------------------------- diagnostics (verify.cpp)
 * device versions of the reference's checks (DMMA GEMMs + fixed-order
 * reductions, bit-deterministic). Host-pointer and *_device variants.                    */
/* residual (verify.cpp:76-93): out[j] = ||H v_j - lambda_j v_j||_2 / ||H||_F, j < k, with
 * H = [A B; -B -A]; v is 2n x k (ldv >= 2n).                                             */
int bse_residual(bse_ctx* ctx, int64_t n, const double* a, int64_t lda, const double* b,
                 int64_t ldb, int64_t k, const double* lambda, const double* v, int64_t ldv,
                 double* out, bse_status* st);
int bse_residual_device(bse_ctx* ctx, int64_t n, const double* d_a, int64_t lda,
                        const double* d_b, int64_t ldb, int64_t k, const double* d_lambda,
                        const double* d_v, int64_t ldv, double* d_out, bse_status* st);
/* sigma_orthogonality_error (verify.cpp:70-74): *out = ||V^H Sigma V - I||_F, V rows x k,
 * rows even (BSE_ERR_ODD_DIMENSION otherwise). *out is a host scalar in both variants.  */
int bse_sigma_orthogonality_error(bse_ctx* ctx, int64_t rows, int64_t k, const double* v,
                                  int64_t ldv, double* out, bse_status* st);
int bse_sigma_orthogonality_error_device(bse_ctx* ctx, int64_t rows, int64_t k,
                                         const double* d_v, int64_t ldv, double* out,
                                         bse_status* st);
/* check_form1 / check_form2 (verify.cpp:46-68): *result = 1 iff J X J = m (X = m^H for form
 * 1, m^T for form 2) and Sigma m^H Sigma = m within tol * ||m||_F; m is rows x rows.      */
int bse_check_form(bse_ctx* ctx, int form, int64_t rows, const double* m, int64_t ldm,
                   double tol, int* result, bse_status* st);
int bse_check_form_device(bse_ctx* ctx, int form, int64_t rows, const double* d_m, int64_t ldm,
                          double tol, int* result, bse_status* st);
/* negative_spectrum (solvers.cpp:223-236): lambda_out = -lambda, v_out = [v_bottom; v_top]. */
int bse_negative_spectrum(bse_ctx* ctx, int64_t n, int64_t k, const double* lambda,
                          const double* v, int64_t ldv, double* lambda_out, double* v_out,
                          int64_t ldvo, bse_status* st);
int bse_negative_spectrum_device(bse_ctx* ctx, int64_t n, int64_t k, const double* d_lambda,
                                 const double* d_v, int64_t ldv, double* d_lambda_out,
                                 double* d_v_out, int64_t ldvo, bse_status* st);

/* ---------------------------------------------------------------- input synthesis
 * Counter-based seeded generators for BASELINE.json configs (host, OpenMP). Each entry
 * (i, j) of stream s draws from splitmix64 of (seed, s, i, j), so generation is parallel
 * and reproducible bit-for-bit on any host.                                               */
/* config 1/2/4/5 family: A = diag(d) + scale*(Z+Z^H)/2, B = scale*(W+W^H)/2,
 * Z, W entries N(0,1)/sqrt(n) (real) or complex N(0,1/2)/sqrt(n) per part,
 * d ~ U[dlo, dhi]. is_complex = 0 gives zero imaginary parts.                             */
int bse_gen_dominant(int64_t n, uint64_t seed, int is_complex, double scale, double dlo,
                     double dhi, double* a, double* b);
/* reference GaussianStream (gen.cpp:8-38): splitmix64 -> mt19937_64 -> Box-Muller,
 * next_complex() pairs. Fills count complex values (2*count doubles).                   */
int bse_gen_gaussian_stream(uint64_t seed, uint64_t stream, int64_t count, double* out);
/* Counter-based standard normals / uniforms [0,1) for stream s (count doubles).        */
int bse_gen_normal(uint64_t seed, uint64_t stream, int64_t count, double* out);
int bse_gen_uniform(uint64_t seed, uint64_t stream, int64_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif /* BSE_GPU_H */
