// context.h — per-thread solver context: device, stream, workspace arena, phase timers.
#pragma once

#include <mutex>
#include <vector>

#include "../../include/bse_gpu.h"
#include "common.cuh"

struct bse_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
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
