// context.h — per-thread solver context: device, stream, workspace arena, phase timers.
#pragma once

#include <mutex>
#include <vector>

#include "../../include/bse_gpu.h"
#include "common.cuh"

struct bse_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  bool strict_m1 = false;  // CHOL: certify A+B by its own Cholesky on every solve (see solvers.cu)  // stream-ordered staging buffers (DevBuf, batch staging)
  void* arena = nullptr;
  size_t arena_bytes = 0;
  int64_t launches = 0;
  bse_phase_times last{};
  cudaEvent_t ev[12]{};
  // second stream for independent stages (fork/join through fork_ev / join_ev)
  cudaStream_t aux = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::mutex mu;
  // live per-kernel timing (bse_ctx_set_kernel_timing)
  bool timing = false;
  std::vector<cudaEvent_t> timer_events;
  bseg::KernelTimer timer;
  // streamed eigenvector output (bse_solve into pinned host memory): the recovery stage
  // copies finished column chunks of V to sink_v on `copy` while later chunks compute
  cudaStream_t copy = nullptr;
  cudaEvent_t sink_ev[17]{};
  double* sink_v = nullptr;
  int64_t sink_ldv = 0;
  int sink_k = 0;
  // bse_solve_batched: host-to-device uploads of the next matrix run on copy_in
  cudaStream_t copy_in = nullptr;
  cudaEvent_t batch_ev[7]{};
  // batch driver: solves in flight per call (1..8) and the extra lanes' contexts
  int batch_lanes = 4;
  bse_ctx* twin[7]{};
  // look-ahead streams / events of the two concurrent Cholesky factorisations
  cudaStream_t la[2]{};
  cudaEvent_t la_ev[8]{};
  cudaEvent_t chol_ev = nullptr;  // start of the CHOL factorisation (bse_phase_times.cholesky)  // 4 per concurrent Cholesky (zpotrf_lower's look-ahead)
};

namespace bseg {

// Bump allocator over the context arena (256-byte aligned slices).
struct Bump {
  char* base;
  size_t off = 0;
  size_t cap;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    if (off > cap) throw std::runtime_error("workspace arena overflow");
    return p;
  }
};

// Ensures the arena holds at least `bytes`; returns a bump allocator over it.
Bump arena(bse_ctx* c, size_t bytes);

// aux waits for everything enqueued on the main stream so far
inline void fork(bse_ctx* c) {
  BSE_CUDA(cudaEventRecord(c->fork_ev, c->stream));
  BSE_CUDA(cudaStreamWaitEvent(c->aux, c->fork_ev, 0));
}
// main waits for everything enqueued on aux so far
inline void join(bse_ctx* c) {
  BSE_CUDA(cudaEventRecord(c->join_ev, c->aux));
  BSE_CUDA(cudaStreamWaitEvent(c->stream, c->join_ev, 0));
}

// Domain error carrying the reference exception payload (types.hpp:33-126).
struct DomainError {
  int code;
  int block;
  int64_t pivot;
  std::string msg;
};

// Column chunk width for the recovery stage: the whole matrix unless a host sink is set.
int64_t recover_chunk_cols(const bse_ctx* c, int64_t n, int64_t min_cols, int parts);
// Queues the D2H of columns [j0, j0+jb) of V (2n x n, ld ldv) to the host sink (no-op
// without a sink) on the copy stream, ordered after everything enqueued on c->stream.
void sink_columns(bse_ctx* c, const z_t* V, int64_t ldv, int64_t n, int64_t j0, int64_t jb);
// Main stream waits for the sink copies; returns true when the whole V was streamed.
bool sink_finish(bse_ctx* c);

// Solver pipelines on device pointers (solvers.cu). Throw DomainError / CudaError.
void solve_chol_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                    int64_t ldb, double* lam, z_t* V, int64_t ldv,
                    std::vector<int64_t>& flagged);
void solve_chol_svd_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                        int64_t ldb, double* lam, z_t* V, int64_t ldv,
                        std::vector<int64_t>& flagged);
size_t solve_workspace_bytes(int method, int64_t n);
// SURVEY §8f rows f2/f3 (extra_solvers.cu)
void solve_sqrt_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                    double* lam, z_t* V, int64_t ldv, std::vector<int64_t>& flagged);
void solve_reference_dev(bse_ctx* c, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                         int64_t ldb, double* lam, z_t* V, int64_t ldv,
                         std::vector<int64_t>& flagged);
size_t hpd_sqrt_workspace_bytes(int64_t n);
void hpd_sqrt_dev(cudaStream_t s, int64_t n, const z_t* M, int64_t ldm, z_t* S, int64_t lds,
                  Bump& b);

}  // namespace bseg
