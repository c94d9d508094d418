// hetrd.h — tridiagonalisation / back-transformation and tridiagonal divide & conquer.
#pragma once

#include "common.cuh"

namespace bseg {

constexpr int kHetrdNB = 32;
constexpr int kBand2 = 32;  // band width of the two-stage reduction (hetrd2.cu)

// A (lower) := reflectors; d (n), e (n-1) real tridiagonal; tau (n-1).
size_t hetrd_workspace_bytes(int64_t n);
void zhetrd_lower(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                  z_t* tau, void* ws);

// Z (n x ncols) <- Q Z with Q from zhetrd_lower's reflectors.
size_t unmtr_workspace_bytes(int64_t n, int64_t ncols);
void zunmtr_lower(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau, z_t* Z,
                  int64_t ldz, int64_t ncols, void* ws);

// Z <- H(0)..H(nref-1) Z ; mode 0: zhetrd 'L' reflectors, 1: zgebrd Q (columns),
// 2: zgebrd P (rows), 3: he2hb 'L' reflectors (unit at row j + kBand2). Workspace: unmtr_workspace_bytes(n, ncols).
void apply_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                      int64_t lda, const z_t* tau, z_t* Z, int64_t ldz, int64_t ncols, void* ws);
// The same in two steps: the blocks' V, T and V T (reflectors only) into ws, then the
// application to Z (same mode, n, nref and ws).
void prepare_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, const z_t* A,
                        int64_t lda, const z_t* tau, void* ws);
void apply_prepared_reflectors(cudaStream_t s, int mode, int64_t n, int64_t nref, z_t* Z,
                               int64_t ldz, int64_t ncols, void* ws);

// Two-stage tridiagonalisation (hetrd2.cu): dense lower Hermitian -> band of width kBand2
// (panel QR + DMMA her2k) -> real tridiagonal by bulge chasing. On exit A holds the stage-1
// reflectors below the band, tau1 (n) their scalars, and ws the band and the stage-2
// reflectors (keep ws until zunmtr_2stage). d (n), e (n-1) as zhetrd_lower.
size_t hetrd2_workspace_bytes(int64_t n);
void zhetrd_2stage(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                   z_t* tau1, void* ws);
// Z (n x ncols) <- Q1 Q2 Z. ws2: zhetrd_2stage's workspace; ws: unmtr_workspace_bytes with
// Q1's blocks already prepared (tridiag_back_prepare; tridiag_back does both).
void zunmtr_2stage(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau1,
                   void* ws2, z_t* Z, int64_t ldz, int64_t ncols, void* ws);
// Two-stage reduction for this n in the current mode (batch lanes, or BSE_TWO_STAGE=1/0).
bool use_two_stage(int64_t n);
int set_tridiag_mode(int mode);  // bse_set_tridiagonal_reduction; returns the previous mode
int current_tridiag_mode();      // this thread's snapshot if one is active, else the global
// Holds one reading of the mode for this thread (outermost scope wins); mode < 0: read now.
struct TridiagModeScope {
  explicit TridiagModeScope(int mode = -1);
  ~TridiagModeScope();
  TridiagModeScope(const TridiagModeScope&) = delete;
  TridiagModeScope& operator=(const TridiagModeScope&) = delete;
  bool owner;
};
// The eigen-solvers' reduction pair, one- or two-stage per use_two_stage(n) (decided in the
// calling thread; the same ws must reach tridiag_back).
size_t tridiag_workspace_bytes(int64_t n);
void tridiag_reduce(cudaStream_t s, int64_t n, z_t* A, int64_t lda, double* d, double* e,
                    z_t* tau, void* ws);
void tridiag_back(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau,
                  void* ws, z_t* Z, int64_t ldz, int64_t ncols, void* ws_unmtr,
                  bool prepared = false);
// Optional early half of tridiag_back (reflector blocks into ws_unmtr), e.g. on a second
// stream beside the tridiagonal eigensolver; then call tridiag_back(..., prepared = true).
void tridiag_back_prepare(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* tau,
                          void* ws_unmtr);

// Symmetric tridiagonal eigensolver (Cuppen divide & conquer with Gu-Eisenstat vectors).
// d (n) diagonal, e (n-1) off-diagonal (device). On exit d holds eigenvalues ascending and
// Q (n x n, ld n, real) the orthonormal eigenvectors. Returns nonzero on failure.
size_t stedc_workspace_bytes(int64_t n);
void dstedc(cudaStream_t s, int64_t n, double* d, const double* e, double* Q, void* ws,
            int* d_info,
            int64_t keep_from = 0);

}  // namespace bseg
