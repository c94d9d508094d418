// capi.cu — the extern "C" drop-in boundary (include/bse_gpu.h).
//
// Every entry point maps the reference's C++ contract (proj/include/bse/backend.hpp,
// solvers.hpp, types.hpp) onto plain pointers + status codes. Host-pointer entry points
// stage through the context's device arena; nothing here ever computes on the CPU: when
// no CUDA device is present every compute entry point fails with BSE_ERR_NO_DEVICE.
#include <algorithm>
#include <atomic>
#include <climits>
#include <initializer_list>
#include <thread>
#include <cfloat>
#include <cstring>
#include <string>

#include "blas.h"
#include "context.h"
#include "gemm.cuh"
#include "hetrd.h"
#include "ops.h"
#include "svd.h"

using namespace bseg;

namespace bseg {  // verify.cu
size_t residual_workspace_bytes(int64_t n, int64_t k);
void residual_dev(cudaStream_t s, int64_t n, const z_t* A, int64_t lda, const z_t* B,
                  int64_t ldb, int64_t k, const double* lam, const z_t* V, int64_t ldv,
                  double* out, Bump& w);
size_t sigma_orth_workspace_bytes(int64_t k);
void sigma_orth_dev(cudaStream_t s, int64_t h, int64_t k, const z_t* V, int64_t ldv,
                    double* d_out, Bump& w);
size_t form_workspace_bytes();
void form_dev(cudaStream_t s, int form, int64_t h, const z_t* M, int64_t ldm, double* d_out,
              Bump& w);
void negative_spectrum_dev(cudaStream_t s, int64_t n, int64_t k, const double* lam, const z_t* V,
                           int64_t ldv, double* lam_out, z_t* Vo, int64_t ldo);
}  // namespace bseg

namespace bseg {

Bump arena(bse_ctx* c, size_t bytes) {
  if (c->arena_bytes < bytes) {
    if (c->arena) BSE_CUDA(cudaFree(c->arena));
    c->arena = nullptr;
    c->arena_bytes = 0;
    const size_t want = bytes + (bytes >> 4);
    cudaError_t e = cudaMalloc(&c->arena, want);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      throw CudaError(e, "workspace arena allocation");
    }
    c->arena_bytes = want;
  }
  return Bump{reinterpret_cast<char*>(c->arena), 0, c->arena_bytes};
}

}  // namespace bseg

namespace {

int set_status(bse_status* st, int code, const std::string& msg, int block = 0,
               int64_t pivot = -1, double dev = 0.0) {
  if (st) {
    st->code = code;
    st->block = block;
    st->pivot_index = pivot;
    st->relative_deviation = dev;
    std::snprintf(st->message, sizeof(st->message), "%s", msg.c_str());
  }
  return code;
}

int ok(bse_status* st) { return set_status(st, BSE_OK, ""); }

// Runs `fn` with the context bound (device, launch counter, lock) and maps exceptions.
template <typename F>
int guarded(bse_ctx* c, bse_status* st, F&& fn) {
  if (!c) return set_status(st, BSE_ERR_INVALID_SPEC, "null context");
  std::lock_guard<std::mutex> lock(c->mu);
  int64_t* prev = g_launch_counter;
  KernelTimer* prev_timer = g_timer;
  g_launch_counter = &c->launches;
  if (c->timing) {
    c->timer.pool = c->timer_events.data();
    c->timer.capacity = int(c->timer_events.size());
    c->timer.used = 0;
    g_timer = &c->timer;
  }
  struct Restore {
    int64_t* a;
    KernelTimer* b;
    ~Restore() {
      g_launch_counter = a;
      g_timer = b;
    }
  } restore{prev, prev_timer};
  const bseg::TridiagModeScope tridiag_mode;  // one reading of the reduction mode per call
  try {
    BSE_CUDA(cudaSetDevice(c->device));
    fn();
    return ok(st);
  } catch (const DomainError& e) {
    return set_status(st, e.code, e.msg, e.block, e.pivot);
  } catch (const CudaError& e) {
    const int code = e.err == cudaErrorMemoryAllocation ? BSE_ERR_OUT_OF_MEMORY : BSE_ERR_CUDA;
    return set_status(st, code, e.what());
  } catch (const std::exception& e) {
    return set_status(st, BSE_ERR_GENERIC, e.what());
  }
}

// Sums the timed launches of the last solve into c->last (after a stream sync).
void collect_timer(bse_ctx* c) {
  if (!c->timing) return;
  BSE_CUDA(cudaStreamSynchronize(c->stream));
  bse_phase_times& t = c->last;
  t.panel_ms = t.gemm_ms = t.panel_bytes = t.gemm_flops = t.gemm_dmma_flops = 0.0;
  t.panel_launches = t.gemm_launches = 0.0;
  for (int i = 0; i < c->timer.used / 2; ++i) {
    float ms = 0.f;
    BSE_CUDA(cudaEventElapsedTime(&ms, c->timer.pool[2 * i], c->timer.pool[2 * i + 1]));
    if (c->timer.kind[i] == 0) {
      t.gemm_ms += ms;
      t.gemm_flops += c->timer.work[i];
      t.gemm_dmma_flops += c->timer.work2[i];
      t.gemm_launches += 1;
    } else {
      t.panel_ms += ms;
      t.panel_bytes += c->timer.work[i];
      t.panel_launches += 1;
    }
  }
}

void h2d(bse_ctx* c, z_t* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
         int64_t cols) {
  BSE_CUDA(cudaMemcpy2DAsync(dst, size_t(ldd) * sizeof(z_t), src, size_t(lds) * sizeof(z_t),
                             size_t(rows) * sizeof(z_t), size_t(cols), cudaMemcpyHostToDevice,
                             c->stream));
}
void d2h(bse_ctx* c, double* dst, int64_t ldd, const z_t* src, int64_t lds, int64_t rows,
         int64_t cols) {
  BSE_CUDA(cudaMemcpy2DAsync(dst, size_t(ldd) * sizeof(z_t), src, size_t(lds) * sizeof(z_t),
                             size_t(rows) * sizeof(z_t), size_t(cols), cudaMemcpyDeviceToHost,
                             c->stream));
}

const z_t kOne = {1.0, 0.0}, kZero = {0.0, 0.0};

// Solve with device-resident buffers carved from a separate allocation (the solver pipeline
// owns the arena): stream-ordered allocations from the context's private memory pool (kept
// mapped between calls; bse_ctx_release_workspace trims it).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, bse_ctx* c) : s(c->stream) {
    BSE_CUDA(cudaMallocFromPoolAsync(&p, bytes, c->pool, s));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* as() { return reinterpret_cast<T*>(p); }
};

void run_solve(bse_ctx* c, int method, int64_t n, const z_t* A, int64_t lda, const z_t* B,
               int64_t ldb, double* lam, z_t* V, int64_t ldv, std::vector<int64_t>& flagged) {
  if (method == BSE_METHOD_CHOL) solve_chol_dev(c, n, A, lda, B, ldb, lam, V, ldv, flagged);
  else if (method == BSE_METHOD_CHOL_SVD) solve_chol_svd_dev(c, n, A, lda, B, ldb, lam, V, ldv, flagged);
  else if (method == BSE_METHOD_SQRT) solve_sqrt_dev(c, n, A, lda, B, ldb, lam, V, ldv, flagged);
  else if (method == BSE_METHOD_REFERENCE)
    solve_reference_dev(c, n, A, lda, B, ldb, lam, V, ldv, flagged);
  else throw DomainError{BSE_ERR_INVALID_SPEC, 0, -1, "unknown method"};
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Installs the host sink for one bse_solve call; always cleared, also on a DomainError.
struct SinkScope {
  bse_ctx* c;
  SinkScope(bse_ctx* ctx, double* v, int64_t ldv) : c(ctx) {
    c->sink_v = v;
    c->sink_ldv = ldv;
    c->sink_k = 0;
  }
  ~SinkScope() {
    if (c->sink_v && c->sink_k > 0) cudaStreamSynchronize(c->copy);
    c->sink_v = nullptr;
    c->sink_k = 0;
  }
};

// Device operands are read and written as 16-byte complex vectors.
void check_aligned16(std::initializer_list<const void*> ptrs) {
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) & 15u)
      throw DomainError{BSE_ERR_INVALID_SPEC, 0, -1,
                        "device matrix pointers must be 16-byte aligned (complex128)"};
}

void check_dims(int64_t n, int64_t lda, int64_t ldb) {
  if (n < 1) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "blocks must be at least 1x1"};
  if (lda < n || ldb < n) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "leading dimension too small"};
}

}  // namespace

extern "C" {

int bse_abi_version(void) { return BSE_GPU_ABI_VERSION; }

int bse_ctx_create(bse_ctx** out, int device, bse_status* st) {
  if (!out) return set_status(st, BSE_ERR_INVALID_SPEC, "null output pointer");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    (void)cudaGetLastError();
    return set_status(st, BSE_ERR_NO_DEVICE, "no CUDA device available");
  }
  if (device < 0 || device >= count) return set_status(st, BSE_ERR_NO_DEVICE, "device index out of range");
  bse_ctx* c = new bse_ctx();
  c->device = device;
  try {
    BSE_CUDA(cudaSetDevice(device));
    // Stream priorities: the solve's critical chains (c->stream, c->aux: Cholesky panels, the
    // reduction panels, the divide & conquer) run at the highest priority, the Cholesky
    // look-ahead streams (bulk trailing HERK updates) at the lowest, so a panel launched while
    // a bulk update fills the GPU takes the next free SMs instead of queueing behind the
    // update's remaining CTAs (BSE_STREAM_PRIORITIES=0: all equal, A/B switch).
    static const bool prio = !getenv("BSE_STREAM_PRIORITIES") || atoi(getenv("BSE_STREAM_PRIORITIES")) != 0;
    int lo_prio = 0, hi_prio = 0;
    BSE_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    if (!prio) lo_prio = hi_prio = 0;
    BSE_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_prio));
    BSE_CUDA(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, hi_prio));
    BSE_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    BSE_CUDA(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    BSE_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    BSE_CUDA(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
    for (auto& st2 : c->la)
      BSE_CUDA(cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, lo_prio));
    for (auto& ev : c->la_ev) BSE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : c->batch_ev) BSE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    // a private pool for the stream-ordered staging buffers, kept mapped between calls (the
    // process-wide default pool and its release threshold are left to the application)
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    BSE_CUDA(cudaMemPoolCreate(&c->pool, &props));
    uint64_t keep = UINT64_MAX;
    BSE_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
    for (auto& ev : c->sink_ev) BSE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : c->ev) BSE_CUDA(cudaEventCreate(&ev));
    BSE_CUDA(cudaEventCreate(&c->chol_ev));
  } catch (const CudaError& ex) {
    delete c;
    return set_status(st, BSE_ERR_CUDA, ex.what());
  }
  *out = c;
  return ok(st);
}

int bse_ctx_destroy(bse_ctx* c) {
  if (!c) return BSE_OK;
  for (auto& t : c->twin)
    if (t) bse_ctx_destroy(t);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->arena) cudaFree(c->arena);
  for (auto& ev : c->timer_events) cudaEventDestroy(ev);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
  }
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
  }
  for (auto& ev : c->sink_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->copy_in) {
    cudaStreamSynchronize(c->copy_in);
    cudaStreamDestroy(c->copy_in);
  }
  for (auto& ev : c->batch_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& st2 : c->la)
    if (st2) {
      cudaStreamSynchronize(st2);
      cudaStreamDestroy(st2);
    }
  for (auto& ev : c->la_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->chol_ev) cudaEventDestroy(c->chol_ev);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  delete c;
  return BSE_OK;
}

void* bse_ctx_stream(bse_ctx* c) { return c ? reinterpret_cast<void*>(c->stream) : nullptr; }

int bse_ctx_last_phase_times(bse_ctx* c, bse_phase_times* out) {
  if (!c || !out) return BSE_ERR_INVALID_SPEC;
  *out = c->last;
  return BSE_OK;
}

int64_t bse_ctx_kernel_launches(bse_ctx* c) {  // including the batch lanes' contexts
  if (!c) return 0;
  int64_t total = c->launches;
  for (bse_ctx* t : c->twin) total += t ? t->launches : 0;
  return total;
}

int bse_ctx_set_kernel_timing(bse_ctx* c, int enable) {
  if (!c) return BSE_ERR_INVALID_SPEC;
  std::lock_guard<std::mutex> lock(c->mu);
  cudaSetDevice(c->device);
  c->timing = enable != 0;
  if (c->timing && c->timer_events.empty()) {
    c->timer_events.resize(8192);
    for (auto& e : c->timer_events)
      if (cudaEventCreate(&e) != cudaSuccess) return BSE_ERR_CUDA;
  }
  return BSE_OK;
}

int bse_ctx_release_workspace(bse_ctx* c) {
  if (!c) return BSE_OK;
  for (bse_ctx* t : c->twin)  // the batch lanes' arenas and pools too
    if (t) bse_ctx_release_workspace(t);
  std::lock_guard<std::mutex> lock(c->mu);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->arena) cudaFree(c->arena);
  c->arena = nullptr;
  c->arena_bytes = 0;
  if (c->pool) cudaMemPoolTrimTo(c->pool, 0);
  return BSE_OK;
}

int bse_solve_device(bse_ctx* c, int method, int64_t n, const double* d_a, int64_t lda,
                     const double* d_b, int64_t ldb, double* d_lambda, double* d_v, int64_t ldv,
                     int64_t* near_singular, int64_t* n_near_singular, bse_status* st) {
  return guarded(c, st, [&] {
    check_dims(n, lda, ldb);
    if (ldv < 2 * n) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "ldv < 2n"};
    check_aligned16({d_a, d_b, d_v});
    std::vector<int64_t> flagged;
    run_solve(c, method, n, reinterpret_cast<const z_t*>(d_a), lda,
              reinterpret_cast<const z_t*>(d_b), ldb, d_lambda, reinterpret_cast<z_t*>(d_v),
              ldv, flagged);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    collect_timer(c);
    if (n_near_singular) *n_near_singular = int64_t(flagged.size());
    if (near_singular)
      for (size_t i = 0; i < flagged.size(); ++i) near_singular[i] = flagged[i];
  });
}

int bse_solve(bse_ctx* c, int method, int64_t n, const double* a, int64_t lda, const double* b,
              int64_t ldb, double* lambda, double* v, int64_t ldv, int64_t* near_singular,
              int64_t* n_near_singular, bse_status* st) {
  return guarded(c, st, [&] {
    check_dims(n, lda, ldb);
    if (ldv < 2 * n) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "ldv < 2n"};
    const size_t nn = size_t(n) * size_t(n);
    DevBuf buf(nn * 2 * sizeof(z_t) + 2 * nn * sizeof(z_t) + size_t(n) * sizeof(double) + 1024,
               c);
    z_t* dA = buf.as<z_t>();
    z_t* dB = dA + nn;
    z_t* dV = dB + nn;
    double* dL = reinterpret_cast<double*>(dV + 2 * nn);
    h2d(c, dA, n, a, lda, n, n);
    h2d(c, dB, n, b, ldb, n, n);
    std::vector<int64_t> flagged;
    // Page-locked output: the solver streams finished column chunks of V to it on the copy
    // stream while it computes the next ones. Pageable output is copied after the solve.
    SinkScope sink(c, is_pinned(v) ? v : nullptr, ldv);
    run_solve(c, method, n, dA, n, dB, n, dL, dV, 2 * n, flagged);
    collect_timer(c);
    BSE_CUDA(cudaMemcpyAsync(lambda, dL, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost,
                             c->stream));
    if (!sink_finish(c)) d2h(c, v, ldv, dV, 2 * n, 2 * n, n);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    if (n_near_singular) *n_near_singular = int64_t(flagged.size());
    if (near_singular)
      for (size_t i = 0; i < flagged.size(); ++i) near_singular[i] = flagged[i];
  });
}

}  // extern "C"

namespace {

// Items of one batch lane: every item index i with i % lanes == lane, in order.
std::vector<int64_t> lane_items(int64_t batch, int lanes, int lane) {
  std::vector<int64_t> v;
  for (int64_t i = lane; i < batch; i += lanes) v.push_back(i);
  return v;
}

struct BatchIO {  // the caller's per-item arrays (host or device pointers)
  int method;
  int64_t n, lda, ldb, ldv;
  const double* const* a;
  const double* const* b;
  double* const* lambda;
  double* const* v;
  int64_t* near_singular;
  int64_t* n_near_singular;
  bool device;  // a, b, lambda, v are device pointers (bse_solve_batched_device)
};

// First failing item over all lanes: later items of every lane are skipped once it is known.
struct BatchFail {
  std::mutex mu;
  std::atomic<int64_t> first{INT64_MAX};
  bool domain = false;
  DomainError err{};
  std::exception_ptr other;
  void record(int64_t i, const DomainError* d, std::exception_ptr e) {
    std::lock_guard<std::mutex> lk(mu);
    if (i >= first.load()) return;
    first = i;
    domain = d != nullptr;
    if (d) err = *d;
    other = d ? nullptr : e;
  }
};

void store_flags(const BatchIO& io, int64_t i, const std::vector<int64_t>& flagged) {
  if (io.n_near_singular) io.n_near_singular[i] = int64_t(flagged.size());
  if (io.near_singular)
    for (size_t f = 0; f < flagged.size(); ++f) io.near_singular[i * io.n + int64_t(f)] = flagged[f];
}

// One lane on context c. Host pointers: two slots of (A, B, V, lambda) staging, item j+1
// uploads on c->copy_in and item j-1 downloads on c->copy while item j computes on c->stream.
// Device pointers: the items are solved in place, one after the other.
void run_lane(bse_ctx* c, const BatchIO& io, const std::vector<int64_t>& items, BatchFail& fail) {
  const int64_t n = io.n;
  auto solve_item = [&](int64_t i, const z_t* A, int64_t lda, const z_t* B, int64_t ldb,
                        double* L, z_t* V, int64_t ldv) -> bool {
    std::vector<int64_t> flagged;
    if (c->timing) c->timer.used = 0;
    try {
      run_solve(c, io.method, n, A, lda, B, ldb, L, V, ldv, flagged);
    } catch (DomainError& e) {
      e.msg = "batch item " + std::to_string(i) + ": " + e.msg;
      fail.record(i, &e, nullptr);
      return false;
    }
    collect_timer(c);
    store_flags(io, i, flagged);
    return true;
  };
  if (io.device) {
    for (int64_t i : items) {
      if (i > fail.first.load()) break;
      if (!solve_item(i, reinterpret_cast<const z_t*>(io.a[i]), io.lda,
                      reinterpret_cast<const z_t*>(io.b[i]), io.ldb, io.lambda[i],
                      reinterpret_cast<z_t*>(io.v[i]), io.ldv))
        break;
    }
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    return;
  }
  const size_t nn = size_t(n) * size_t(n);
  const size_t slot = 2 * nn + 2 * nn + size_t(n) / 2 + 64;  // in z_t units
  DevBuf buf(2 * slot * sizeof(z_t), c);
  z_t *dA[2], *dB[2], *dV[2];
  double* dL[2];
  for (int k = 0; k < 2; ++k) {
    z_t* base = buf.as<z_t>() + k * slot;
    dA[k] = base;
    dB[k] = base + nn;
    dV[k] = base + 2 * nn;
    dL[k] = reinterpret_cast<double*>(base + 4 * nn);
  }
  struct Drain {  // the copy streams finish before the staging buffers are released
    bse_ctx* c;
    ~Drain() {
      cudaStreamSynchronize(c->copy_in);
      cudaStreamSynchronize(c->copy);
    }
  } drain{c};
  cudaEvent_t* in_ready = c->batch_ev;       // [2] copy_in -> compute
  cudaEvent_t* comp_done = c->batch_ev + 2;  // [2] compute -> copy_in / copy
  cudaEvent_t* out_done = c->batch_ev + 4;   // [2] copy -> compute (slot reuse)
  auto upload = [&](size_t j) {
    const int k = int(j & 1);
    const int64_t i = items[j];
    if (j >= 2) BSE_CUDA(cudaStreamWaitEvent(c->copy_in, comp_done[k], 0));
    BSE_CUDA(cudaMemcpy2DAsync(dA[k], size_t(n) * sizeof(z_t), io.a[i], size_t(io.lda) * sizeof(z_t),
                               size_t(n) * sizeof(z_t), size_t(n), cudaMemcpyHostToDevice,
                               c->copy_in));
    BSE_CUDA(cudaMemcpy2DAsync(dB[k], size_t(n) * sizeof(z_t), io.b[i], size_t(io.ldb) * sizeof(z_t),
                               size_t(n) * sizeof(z_t), size_t(n), cudaMemcpyHostToDevice,
                               c->copy_in));
    BSE_CUDA(cudaEventRecord(in_ready[k], c->copy_in));
  };
  // the staging allocation is ordered on c->stream; the copy-in stream starts after it
  BSE_CUDA(cudaEventRecord(c->batch_ev[6], c->stream));
  BSE_CUDA(cudaStreamWaitEvent(c->copy_in, c->batch_ev[6], 0));
  if (!items.empty()) upload(0);
  for (size_t j = 0; j < items.size(); ++j) {
    const int64_t i = items[j];
    if (i > fail.first.load()) break;
    const int k = int(j & 1);
    if (j + 1 < items.size()) upload(j + 1);
    BSE_CUDA(cudaStreamWaitEvent(c->stream, in_ready[k], 0));
    if (j >= 2) BSE_CUDA(cudaStreamWaitEvent(c->stream, out_done[k], 0));
    if (!solve_item(i, dA[k], n, dB[k], n, dL[k], dV[k], 2 * n)) break;
    BSE_CUDA(cudaEventRecord(comp_done[k], c->stream));
    BSE_CUDA(cudaStreamWaitEvent(c->copy, comp_done[k], 0));
    BSE_CUDA(cudaMemcpyAsync(io.lambda[i], dL[k], sizeof(double) * size_t(n),
                             cudaMemcpyDeviceToHost, c->copy));
    // the lane's last item has no later solve of its own to protect: the faster copy engine
    const bool last = j + 1 == items.size();
    if (last || !(is_pinned(io.v[i]) &&
                  zcopy2d_to_host_streaming(c->copy, 2 * n, n, dV[k], 2 * n,
                                            reinterpret_cast<z_t*>(io.v[i]), io.ldv)))
      BSE_CUDA(cudaMemcpy2DAsync(io.v[i], size_t(io.ldv) * sizeof(z_t), dV[k],
                                 size_t(2 * n) * sizeof(z_t), size_t(2 * n) * sizeof(z_t),
                                 size_t(n), cudaMemcpyDeviceToHost, c->copy));
    BSE_CUDA(cudaEventRecord(out_done[k], c->copy));
  }
  BSE_CUDA(cudaStreamSynchronize(c->copy));
  BSE_CUDA(cudaStreamSynchronize(c->stream));
}

// The batch on `lanes` contexts at once (c and its lazily created twins), one host thread
// per extra lane; each lane's cooperative panel kernels get 1/lanes of the SMs, so one lane's
// latency-bound tridiagonal / bidiagonal reductions overlap another lane's GEMM phases.
void run_batch(bse_ctx* c, const BatchIO& io, int64_t batch, int64_t* failed_index) {
  if (failed_index) *failed_index = -1;
  if (batch == 0) return;
  // lanes that fit: every extra lane needs its own solver workspace (+ staging on the host
  // path); lanes whose context already holds a large enough arena cost nothing new
  const int64_t n = io.n;
  const size_t nn = size_t(n) * size_t(n);
  size_t per_lane = io.method == BSE_METHOD_REFERENCE
                        ? 4 * solve_workspace_bytes(BSE_METHOD_CHOL_SVD, 2 * n) / 3
                        : solve_workspace_bytes(io.method == BSE_METHOD_CHOL ? BSE_METHOD_CHOL
                                                                             : BSE_METHOD_CHOL_SVD, n);
  if (!io.device) per_lane += 2 * (4 * nn + size_t(n)) * sizeof(z_t);
  size_t free_b = 0, total_b = 0;
  BSE_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int ready = 1;
  for (int l = 1; l < c->batch_lanes && c->twin[l - 1]; ++l)
    if (c->twin[l - 1]->arena_bytes >= per_lane - (io.device ? 0 : 2 * (4 * nn + size_t(n)) * sizeof(z_t)))
      ++ready;
  const int64_t fit = ready + int64_t(0.85 * double(free_b) / double(per_lane));
  const int lanes = int(std::max<int64_t>(1, std::min<int64_t>({int64_t(c->batch_lanes), batch, fit})));
  int sms = 0;
  BSE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const int prev_cap = g_panel_ctas;
  g_panel_ctas = lanes > 1 ? sms / lanes : 0;
  static const int cap_env = [] {  // developer A/B switch: panel CTAs per lane
    const char* e = getenv("BSE_PANEL_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (lanes > 1 && cap_env > 0) g_panel_ctas = cap_env;
  struct Restore {
    int v;
    ~Restore() { g_panel_ctas = v; }
  } restore{prev_cap};
  // every lane context exists before any lane thread starts: a failing create throws here,
  // with no thread running
  for (int l = 1; l < lanes; ++l) {
    if (!c->twin[l - 1]) {
      bse_status st{};
      if (bse_ctx_create(&c->twin[l - 1], c->device, &st) != BSE_OK)
        throw std::runtime_error(std::string("batch lane context: ") + st.message);
    }
  }
  BatchFail fail;
  std::vector<std::exception_ptr> lane_err(static_cast<size_t>(lanes));
  std::vector<std::thread> extra;
  extra.reserve(size_t(lanes));
  // joins every started lane thread on every exit path (a std::thread that is still joinable
  // when destroyed terminates the process, and the lanes reference this frame's locals)
  struct JoinAll {
    std::vector<std::thread>& t;
    BatchFail& f;
    ~JoinAll() {
      if (std::any_of(t.begin(), t.end(), [](const std::thread& x) { return x.joinable(); }))
        f.first.store(-1);  // an early exit: lanes stop at their next item
      for (auto& x : t)
        if (x.joinable()) x.join();
    }
  } join_all{extra, fail};
  const int cap = g_panel_ctas;             // set above from `lanes`
  const int tmode = current_tridiag_mode();  // the caller's snapshot, for every lane
  for (int l = 1; l < lanes; ++l) {
    bse_ctx* lc = c->twin[l - 1];
    lc->strict_m1 = c->strict_m1;
    extra.emplace_back([&, l, lc, cap, tmode] {
      const TridiagModeScope tridiag_mode(tmode);
      try {
        BSE_CUDA(cudaSetDevice(lc->device));
        g_launch_counter = &lc->launches;
        g_timer = nullptr;
        g_panel_ctas = cap;
        run_lane(lc, io, lane_items(batch, lanes, l), fail);
      } catch (...) {
        lane_err[size_t(l)] = std::current_exception();
      }
    });
  }
  try {
    run_lane(c, io, lane_items(batch, lanes, 0), fail);
  } catch (...) {
    lane_err[0] = std::current_exception();
  }
  for (auto& t : extra) t.join();
  for (auto& e : lane_err)
    if (e) std::rethrow_exception(e);  // CUDA / allocation failure of a lane
  if (fail.first.load() != INT64_MAX) {
    if (failed_index) *failed_index = fail.first.load();
    if (fail.domain) throw fail.err;
    std::rethrow_exception(fail.other);
  }
}

void check_batch(int64_t n, int64_t lda, int64_t ldb, int64_t ldv, int64_t batch,
                 const void* a, const void* b, const void* l, const void* v) {
  check_dims(n, lda, ldb);
  if (ldv < 2 * n) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "ldv < 2n"};
  if (batch < 0) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "negative batch"};
  if (batch > 0 && (!a || !b || !l || !v))
    throw DomainError{BSE_ERR_INVALID_SPEC, 0, -1, "null batch pointer array"};
}

}  // namespace

extern "C" {

int bse_solve_batched(bse_ctx* c, int method, int64_t n, int64_t batch, const double* const* a,
                      int64_t lda, const double* const* b, int64_t ldb, double* const* lambda,
                      double* const* v, int64_t ldv, int64_t* near_singular,
                      int64_t* n_near_singular, int64_t* failed_index, bse_status* st) {
  if (failed_index) *failed_index = -1;
  return guarded(c, st, [&] {
    check_batch(n, lda, ldb, ldv, batch, a, b, lambda, v);
    const BatchIO io{method, n, lda, ldb, ldv, a, b, lambda, v, near_singular, n_near_singular,
                     false};
    run_batch(c, io, batch, failed_index);
  });
}

int bse_solve_batched_device(bse_ctx* c, int method, int64_t n, int64_t batch,
                             const double* const* d_a, int64_t lda, const double* const* d_b,
                             int64_t ldb, double* const* d_lambda, double* const* d_v,
                             int64_t ldv, int64_t* near_singular, int64_t* n_near_singular,
                             int64_t* failed_index, bse_status* st) {
  if (failed_index) *failed_index = -1;
  return guarded(c, st, [&] {
    check_batch(n, lda, ldb, ldv, batch, d_a, d_b, d_lambda, d_v);
    for (int64_t i = 0; i < batch; ++i) check_aligned16({d_a[i], d_b[i], d_v[i]});
    const BatchIO io{method, n, lda, ldb, ldv, d_a, d_b, d_lambda, d_v, near_singular,
                     n_near_singular, true};
    run_batch(c, io, batch, failed_index);
  });
}

int bse_set_tridiagonal_reduction(int mode) { return bseg::set_tridiag_mode(mode); }

int bse_ctx_set_strict_certificates(bse_ctx* c, int enable) {
  if (!c) return BSE_ERR_INVALID_SPEC;
  std::lock_guard<std::mutex> lock(c->mu);
  c->strict_m1 = enable != 0;
  return BSE_OK;
}

int bse_ctx_set_batch_lanes(bse_ctx* c, int lanes) {
  if (!c || lanes < 1 || lanes > 8) return BSE_ERR_INVALID_SPEC;
  std::lock_guard<std::mutex> lock(c->mu);
  c->batch_lanes = lanes;
  return BSE_OK;
}

int bse_product_pair(bse_ctx* c, int64_t n, const double* a, int64_t lda, const double* b,
                     int64_t ldb, double* m1, double* m2, bse_status* st) {
  return guarded(c, st, [&] {
    check_dims(n, lda, ldb);
    const size_t nn = size_t(n) * size_t(n);
    DevBuf buf(nn * 5 * sizeof(z_t) + 64 * 64 * sizeof(z_t) + 64, c);
    z_t* dA = buf.as<z_t>();
    z_t* dB = dA + nn;
    z_t* dM1 = dB + nn;
    z_t* dM2 = dM1 + nn;
    z_t* dW = dM2 + nn;
    z_t* ws = dW + nn;
    int* info = reinterpret_cast<int*>(ws + 64 * 64);
    h2d(c, dA, n, a, lda, n, n);
    h2d(c, dB, n, b, ldb, n, n);
    zaddsub(c->stream, n, dA, n, dB, n, dM1, dM2, n);
    zcopy2d(c->stream, n, n, dM1, n, dW, n);
    zpotrf_lower(c->stream, n, dW, n, info, ws, false);
    int h[2];
    BSE_CUDA(cudaMemcpyAsync(&h[0], info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    zcopy2d(c->stream, n, n, dM2, n, dW, n);
    zpotrf_lower(c->stream, n, dW, n, info, ws, false);
    BSE_CUDA(cudaMemcpyAsync(&h[1], info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    d2h(c, m1, n, dM1, n, n, n);
    d2h(c, m2, n, dM2, n, n, n);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    if (h[0] != 0)
      throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M1, int64_t(h[0]) - 1,
                        "A+B is not positive definite: leading minor of order " +
                            std::to_string(h[0]) + " is not positive definite"};
    if (h[1] != 0)
      throw DomainError{BSE_ERR_NOT_DEFINITE, BSE_BLOCK_M2, int64_t(h[1]) - 1,
                        "A-B is not positive definite: leading minor of order " +
                            std::to_string(h[1]) + " is not positive definite"};
  });
}

int bse_assemble_eigenvectors(bse_ctx* c, int64_t n, int64_t k, const double* v1, int64_t ldv1,
                              const double* v2, int64_t ldv2, const double* lambda1,
                              const double* lambda2, double* v, int64_t ldv, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 0 || k < 0 || ldv < 2 * n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "factor shapes do not conform"};
    for (int64_t j = 0; j < k; ++j) {  // core.cpp:108-116 (validated on the host inputs)
      const double x = lambda1[j], y = lambda2[j];
      if (!(x > 0.0) || !(y > 0.0) || !std::isfinite(x) || !std::isfinite(y))
        throw DomainError{BSE_ERR_NON_POSITIVE_SCALE, 0, -1,
                          "scaling factor for column " + std::to_string(j) +
                              " is not a positive finite real"};
    }
    if (n == 0 || k == 0) return;
    const size_t nk = size_t(n) * size_t(k);
    DevBuf buf(nk * 4 * sizeof(z_t) + 2 * size_t(k) * sizeof(double) + 64, c);
    z_t* d1 = buf.as<z_t>();
    z_t* d2 = d1 + nk;
    z_t* dV = d2 + nk;
    double* l1 = reinterpret_cast<double*>(dV + 2 * nk);
    double* l2 = l1 + k;
    h2d(c, d1, n, v1, ldv1, n, k);
    h2d(c, d2, n, v2, ldv2, n, k);
    BSE_CUDA(cudaMemcpyAsync(l1, lambda1, sizeof(double) * size_t(k), cudaMemcpyHostToDevice, c->stream));
    BSE_CUDA(cudaMemcpyAsync(l2, lambda2, sizeof(double) * size_t(k), cudaMemcpyHostToDevice, c->stream));
    assemble(c->stream, n, k, d1, n, d2, n, l1, l2, 0, nullptr, l1, dV, 2 * n);
    d2h(c, v, ldv, dV, 2 * n, 2 * n, k);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_assemble_from_squares(bse_ctx* c, int64_t n, int64_t k, const double* v1,
                              int64_t ldv1, const double* v2, int64_t ldv2, const double* d,
                              double* lambda, double* v, int64_t ldv, int64_t* near_singular,
                              int64_t* n_near_singular, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 1 || k < 1 || ldv1 < n || ldv2 < n || ldv < 2 * n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "factor shapes do not conform"};
    const size_t nk = size_t(n) * size_t(k);
    DevBuf buf(nk * 4 * sizeof(z_t) + 3 * size_t(k) * sizeof(double) +
                   2 * size_t(k) * sizeof(int64_t) + 8 * sizeof(int64_t) + 64,
               c);
    z_t* d1 = buf.as<z_t>();
    z_t* d2 = d1 + nk;
    z_t* dV = d2 + nk;
    double* dd = reinterpret_cast<double*>(dV + 2 * nk);
    double* lam = dd + k;
    double* l1 = lam + k;
    int64_t* flg = reinterpret_cast<int64_t*>(l1 + k);
    int64_t* nonpos = flg + k;
    int64_t* counts = nonpos + k;
    double* floor_p = reinterpret_cast<double*>(counts + 4);
    h2d(c, d1, n, v1, ldv1, n, k);
    h2d(c, d2, n, v2, ldv2, n, k);
    BSE_CUDA(cudaMemcpyAsync(dd, d, sizeof(double) * size_t(k), cudaMemcpyHostToDevice, c->stream));
    // the same launches as the tail of solve_chol_dev (solvers.cu)
    clamp_spectrum(c->stream, k, dd, 0, lam, flg, nonpos, counts, floor_p);
    square_vec(c->stream, k, lam, l1);
    assemble(c->stream, n, k, d1, n, d2, n, l1, nullptr, 1, dd, floor_p, dV, 2 * n);
    int64_t cnt[4];
    BSE_CUDA(cudaMemcpyAsync(cnt, counts, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    if (cnt[2] != 0)
      throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                        "squared-problem spectrum has no positive eigenvalue"};
    if (near_singular && cnt[0] > 0)
      BSE_CUDA(cudaMemcpyAsync(near_singular, flg, sizeof(int64_t) * size_t(cnt[0]),
                               cudaMemcpyDeviceToHost, c->stream));
    if (n_near_singular) *n_near_singular = cnt[0];
    BSE_CUDA(cudaMemcpyAsync(lambda, lam, sizeof(double) * size_t(k), cudaMemcpyDeviceToHost,
                             c->stream));
    d2h(c, v, ldv, dV, 2 * n, 2 * n, k);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_cholesky_lower(bse_ctx* c, int64_t n, const double* m, int64_t ldm, double* l,
                       int64_t ldl, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 1 || ldm < n || ldl < n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "cholesky_lower: bad dimensions"};
    const size_t nn = size_t(n) * size_t(n);
    DevBuf buf(nn * sizeof(z_t) + 64 * 64 * sizeof(z_t) + 64, c);
    z_t* dM = buf.as<z_t>();
    z_t* ws = dM + nn;
    int* info = reinterpret_cast<int*>(ws + 64 * 64);
    h2d(c, dM, n, m, ldm, n, n);
    zpotrf_lower(c->stream, n, dM, n, info, ws, true);
    int h = 0;
    BSE_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    d2h(c, l, ldl, dM, n, n, n);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    if (h > 0)
      throw DomainError{BSE_ERR_NOT_POSITIVE_DEFINITE, 0, int64_t(h) - 1,
                        "leading minor of order " + std::to_string(h) + " is not positive definite"};
  });
}

int bse_matmul(bse_ctx* c, int64_t ar, int64_t ac, const double* a, int64_t lda, int op_a,
               int shape_a, int64_t br, int64_t bc, const double* b, int64_t ldb, int op_b,
               int shape_b, double* cmat, int64_t ldc, bse_status* st) {
  return guarded(c, st, [&] {
    const int64_t am = op_a == BSE_OP_NONE ? ar : ac, ak = op_a == BSE_OP_NONE ? ac : ar;
    const int64_t bk = op_b == BSE_OP_NONE ? br : bc, bn = op_b == BSE_OP_NONE ? bc : br;
    if (ak != bk)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1,
                        "matmul: inner dimensions differ (" + std::to_string(am) + "x" +
                            std::to_string(ak) + " times " + std::to_string(bk) + "x" +
                            std::to_string(bn) + ")"};
    const bool tri_a = shape_a != BSE_SHAPE_GENERAL, tri_b = shape_b != BSE_SHAPE_GENERAL;
    // backend.cpp:146-167: exactly one triangular operand routes to TRMM semantics
    int sa = kGeneral, sb = kGeneral;
    if (tri_a && !tri_b) {
      if (ar != ac) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "matmul (triangular operand): matrix is not square"};
      const bool lower_op = (shape_a == BSE_SHAPE_LOWER) == (op_a == BSE_OP_NONE);
      sa = lower_op ? kLowerOp : kUpperOp;
    } else if (tri_b && !tri_a) {
      if (br != bc) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "matmul (triangular operand): matrix is not square"};
      const bool lower_op = (shape_b == BSE_SHAPE_LOWER) == (op_b == BSE_OP_NONE);
      sb = lower_op ? kLowerOp : kUpperOp;
    }
    if (am == 0 || bn == 0) return;
    const size_t na = size_t(ar) * size_t(ac), nb = size_t(br) * size_t(bc),
                 ncm = size_t(am) * size_t(bn);
    DevBuf buf((na + nb + ncm) * sizeof(z_t) + 64, c);
    z_t* dA = buf.as<z_t>();
    z_t* dB = dA + na;
    z_t* dC = dB + nb;
    if (na) h2d(c, dA, ar, a, lda, ar, ac);
    if (nb) h2d(c, dB, br, b, ldb, br, bc);
    if (ak == 0) {
      BSE_CUDA(cudaMemsetAsync(dC, 0, ncm * sizeof(z_t), c->stream));
    } else {
      zgemm(c->stream, op_a, op_b, am, bn, ak, kOne, dA, ar, dB, br, kZero, dC, am, sa, sb, 0,
            nullptr, 0);
      collect_timer(c);
    }
    d2h(c, cmat, ldc, dC, am, am, bn);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_tri_solve(bse_ctx* c, int64_t n, const double* l, int64_t ldl, int64_t rows,
                  int64_t cols, const double* rhs, int64_t ldr, int side, int op, double* x,
                  int64_t ldx, bse_status* st) {
  return guarded(c, st, [&] {
    if ((side == BSE_SIDE_LEFT && rows != n) || (side == BSE_SIDE_RIGHT && cols != n))
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "tri_solve: right-hand side does not conform"};
    for (int64_t i = 0; i < n; ++i) {  // backend.cpp:114-120
      const double re = l[2 * (i + i * ldl)], im = l[2 * (i + i * ldl) + 1];
      if (std::hypot(re, im) < DBL_MIN)
        throw DomainError{BSE_ERR_SINGULAR_FACTOR, 0, -1,
                          "triangular factor has a vanishing diagonal entry at index " +
                              std::to_string(i)};
    }
    if (rows == 0 || cols == 0) return;
    const size_t nn = size_t(n) * size_t(n), nr = size_t(rows) * size_t(cols);
    const int64_t other = side == BSE_SIDE_LEFT ? cols : rows;
    DevBuf buf((nn + nr + trsm_workspace_elems(n, other, 64)) * sizeof(z_t) + 64, c);
    z_t* dL = buf.as<z_t>();
    z_t* dX = dL + nn;
    z_t* ws = dX + nr;
    h2d(c, dL, n, l, ldl, n, n);
    h2d(c, dX, rows, rhs, ldr, rows, cols);
    ztrsm_lower(c->stream, side == BSE_SIDE_LEFT ? 0 : 1, op == BSE_OP_NONE ? 0 : 1, n, other, dL,
                n, dX, rows, ws, 64);
    d2h(c, x, ldx, dX, rows, rows, cols);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_hermitian_eig(bse_ctx* c, int64_t n, const double* m, int64_t ldm, double* values,
                      double* vectors, int64_t ldv, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 1 || ldm < n || ldv < n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "hermitian_eig: bad dimensions"};
    const size_t nn = size_t(n) * size_t(n);
    const size_t bytes = nn * 2 * sizeof(z_t) + nn * sizeof(double) + stedc_workspace_bytes(n) +
                         tridiag_workspace_bytes(n) + unmtr_workspace_bytes(n, n) +
                         size_t(n) * 48 + 4096;
    Bump w = arena(c, bytes);
    z_t* dM = w.take<z_t>(nn);
    z_t* dZ = w.take<z_t>(nn);
    double* Z = w.take<double>(nn);
    void* ws_st = w.take<char>(stedc_workspace_bytes(n));
    void* ws_ht = w.take<char>(tridiag_workspace_bytes(n));
    void* ws_um = w.take<char>(unmtr_workspace_bytes(n, n));
    double* d = w.take<double>(n);
    double* e = w.take<double>(n);
    z_t* tau = w.take<z_t>(n);
    int* info = w.take<int>(2);
    h2d(c, dM, n, m, ldm, n, n);
    tridiag_reduce(c->stream, n, dM, n, d, e, tau, ws_ht);
    dstedc(c->stream, n, d, e, Z, ws_st, info);
    real_to_complex(c->stream, n, n, Z, n, dZ, n);
    tridiag_back(c->stream, n, dM, n, tau, ws_ht, dZ, n, n, ws_um);
    int h = 0;
    BSE_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaMemcpyAsync(values, d, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, c->stream));
    d2h(c, vectors, ldv, dZ, n, n, n);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    if (h != 0)
      throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1,
                        "zheevd failed to converge (info=" + std::to_string(h) + ", n=" +
                            std::to_string(n) + ")"};
  });
}

int bse_svd(bse_ctx* c, int64_t n, const double* m, int64_t ldm, double* u, int64_t ldu,
            double* s, double* v, int64_t ldv, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 1 || ldm < n || ldu < n || ldv < n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "svd: bad dimensions"};
    const size_t nn = size_t(n) * size_t(n);
    const int64_t m2 = 2 * n;
    const size_t bytes = nn * 5 * sizeof(z_t) + size_t(m2) * size_t(m2) * sizeof(double) +
                         stedc_workspace_bytes(m2) + gebrd_workspace_bytes(n) +
                         unmbr_workspace_bytes(n, n) + size_t(n) * 96 + 4096;
    Bump w = arena(c, bytes);
    z_t* dM = w.take<z_t>(nn);
    z_t* dU = w.take<z_t>(nn);
    z_t* dV = w.take<z_t>(nn);
    z_t* dU2 = w.take<z_t>(nn);
    z_t* dV2 = w.take<z_t>(nn);
    double* X = w.take<double>(size_t(m2) * size_t(m2));
    void* ws_st = w.take<char>(stedc_workspace_bytes(m2));
    void* ws_gb = w.take<char>(gebrd_workspace_bytes(n));
    void* ws_um = w.take<char>(unmbr_workspace_bytes(n, n));
    double* d = w.take<double>(n);
    double* e = w.take<double>(n);
    double* td = w.take<double>(m2);
    double* te = w.take<double>(m2 + 8);
    double* sd = w.take<double>(n);
    z_t* tq = w.take<z_t>(n);
    z_t* tp = w.take<z_t>(n);
    int* info = w.take<int>(2);
    cudaStream_t sm = c->stream;
    h2d(c, dM, n, m, ldm, n, n);
    zgebrd_upper(sm, n, dM, n, d, e, tq, tp, ws_gb);
    tgk_build(sm, n, d, e, td, te);
    dstedc(sm, m2, td, te, X, ws_st, info, n);  // only the positive half of the vectors
    tgk_extract(sm, n, X, dU, n, dV, n);
    tgk_reorthogonalize(sm, n, td + n, dU, dV, n, reinterpret_cast<z_t*>(X), info + 1);
    zunmbr_q(sm, n, dM, n, tq, dU, n, n, ws_um);
    zunmbr_p(sm, n, dM, n, tp, dV, n, n, ws_um);
    // reference convention: s descending, u/v columns to match (backend.cpp:74-84)
    tgk_refine(sm, n, d, e, td + n, te);  // relative accuracy, as zbdsqr
    reverse_real(sm, n, td + n, sd);
    reverse_cols(sm, n, n, dU, n, dU2, n);
    reverse_cols(sm, n, n, dV, n, dV2, n);
    int h = 0;
    BSE_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, sm));
    BSE_CUDA(cudaMemcpyAsync(s, sd, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, sm));
    d2h(c, u, ldu, dU2, n, n, n);
    d2h(c, v, ldv, dV2, n, n, n);
    BSE_CUDA(cudaStreamSynchronize(sm));
    if (h != 0) throw DomainError{BSE_ERR_CONVERGENCE_FAILURE, 0, -1, "zgesvd failed to converge"};
  });
}

}  // extern "C"

/* ---------------------------------------------------------------- §8f: hpd_sqrt + diagnostics */
extern "C" {

int bse_hpd_sqrt(bse_ctx* c, int64_t n, const double* m, int64_t ldm, double* out, int64_t lds,
                 bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 1 || ldm < n || lds < n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "hpd_sqrt: bad dimensions"};
    const size_t nn = size_t(n) * size_t(n);
    Bump w = arena(c, 2 * nn * sizeof(z_t) + hpd_sqrt_workspace_bytes(n) + 4096);
    z_t* dM = w.take<z_t>(nn);
    z_t* dS = w.take<z_t>(nn);
    h2d(c, dM, n, m, ldm, n, n);
    hpd_sqrt_dev(c->stream, n, dM, n, dS, n, w);
    d2h(c, out, lds, dS, n, n, n);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

static void check_residual_dims(int64_t n, int64_t lda, int64_t ldb, int64_t k, int64_t ldv) {
  if (n < 1 || lda < n || ldb < n || k < 0 || ldv < 2 * n)
    throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1,
                      "residual: result does not conform to the matrix"};
}

int bse_residual_device(bse_ctx* c, int64_t n, const double* d_a, int64_t lda,
                        const double* d_b, int64_t ldb, int64_t k, const double* d_lambda,
                        const double* d_v, int64_t ldv, double* d_out, bse_status* st) {
  return guarded(c, st, [&] {
    check_residual_dims(n, lda, ldb, k, ldv);
    check_aligned16({d_a, d_b, d_v});
    Bump w = arena(c, residual_workspace_bytes(n, k));
    residual_dev(c->stream, n, reinterpret_cast<const z_t*>(d_a), lda,
                 reinterpret_cast<const z_t*>(d_b), ldb, k, d_lambda,
                 reinterpret_cast<const z_t*>(d_v), ldv, d_out, w);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_residual(bse_ctx* c, int64_t n, const double* a, int64_t lda, const double* b,
                 int64_t ldb, int64_t k, const double* lambda, const double* v, int64_t ldv,
                 double* out, bse_status* st) {
  return guarded(c, st, [&] {
    check_residual_dims(n, lda, ldb, k, ldv);
    if (k == 0) return;
    const size_t nn = size_t(n) * size_t(n), vk = 2 * size_t(n) * size_t(k);
    Bump w = arena(c, (2 * nn + vk) * sizeof(z_t) + 2 * size_t(k) * sizeof(double) +
                          residual_workspace_bytes(n, k) + 4096);
    z_t* dA = w.take<z_t>(nn);
    z_t* dB = w.take<z_t>(nn);
    z_t* dV = w.take<z_t>(vk);
    double* dl = w.take<double>(size_t(k));
    double* dout = w.take<double>(size_t(k));
    h2d(c, dA, n, a, lda, n, n);
    h2d(c, dB, n, b, ldb, n, n);
    h2d(c, dV, 2 * n, v, ldv, 2 * n, k);
    BSE_CUDA(cudaMemcpyAsync(dl, lambda, sizeof(double) * size_t(k), cudaMemcpyHostToDevice,
                             c->stream));
    residual_dev(c->stream, n, dA, n, dB, n, k, dl, dV, 2 * n, dout, w);
    BSE_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * size_t(k), cudaMemcpyDeviceToHost,
                             c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

static int64_t half_dimension(int64_t rows, const char* who) {
  if (rows % 2 != 0)
    throw DomainError{BSE_ERR_ODD_DIMENSION, 0, -1, std::string(who) + ": row dimension must be even"};
  return rows / 2;
}

int bse_sigma_orthogonality_error_device(bse_ctx* c, int64_t rows, int64_t k, const double* d_v,
                                         int64_t ldv, double* out, bse_status* st) {
  return guarded(c, st, [&] {
    const int64_t h = half_dimension(rows, "sigma_orthogonality_error");
    if (k < 0 || ldv < rows) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "ldv < rows"};
    check_aligned16({d_v});
    *out = 0.0;
    if (k == 0) return;
    Bump w = arena(c, sigma_orth_workspace_bytes(k) + 1024);
    double* d_out = w.take<double>(1);
    sigma_orth_dev(c->stream, h, k, reinterpret_cast<const z_t*>(d_v), ldv, d_out, w);
    double sq = 0.0;
    BSE_CUDA(cudaMemcpyAsync(&sq, d_out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    *out = std::sqrt(sq);
  });
}

int bse_sigma_orthogonality_error(bse_ctx* c, int64_t rows, int64_t k, const double* v,
                                  int64_t ldv, double* out, bse_status* st) {
  return guarded(c, st, [&] {
    const int64_t h = half_dimension(rows, "sigma_orthogonality_error");
    if (k < 0 || ldv < rows) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, "ldv < rows"};
    *out = 0.0;
    if (k == 0) return;
    const size_t vk = size_t(rows) * size_t(k);
    Bump w = arena(c, vk * sizeof(z_t) + sigma_orth_workspace_bytes(k) + 4096);
    z_t* dV = w.take<z_t>(vk);
    double* d_out = w.take<double>(1);
    h2d(c, dV, rows, v, ldv, rows, k);
    sigma_orth_dev(c->stream, h, k, dV, rows, d_out, w);
    double sq = 0.0;
    BSE_CUDA(cudaMemcpyAsync(&sq, d_out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    *out = std::sqrt(sq);
  });
}

static void form_result(int form, const double* sums, double tol, int* result) {
  const double norm = std::sqrt(sums[2]);
  (void)form;
  *result = (std::sqrt(sums[0]) <= tol * norm && std::sqrt(sums[1]) <= tol * norm) ? 1 : 0;
}

int bse_check_form_device(bse_ctx* c, int form, int64_t rows, const double* d_m, int64_t ldm,
                          double tol, int* result, bse_status* st) {
  return guarded(c, st, [&] {
    const char* who = form == 2 ? "check_form2" : "check_form1";
    if (form != 1 && form != 2) throw DomainError{BSE_ERR_INVALID_SPEC, 0, -1, "form must be 1 or 2"};
    if (ldm < rows) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, std::string(who) + ": matrix must be square"};
    const int64_t h = half_dimension(rows, who);
    check_aligned16({d_m});
    Bump w = arena(c, form_workspace_bytes() + 1024);
    double* d_out = w.take<double>(4);
    form_dev(c->stream, form, h, reinterpret_cast<const z_t*>(d_m), ldm, d_out, w);
    double sums[3];
    BSE_CUDA(cudaMemcpyAsync(sums, d_out, sizeof(sums), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    form_result(form, sums, tol, result);
  });
}

int bse_check_form(bse_ctx* c, int form, int64_t rows, const double* m, int64_t ldm, double tol,
                   int* result, bse_status* st) {
  return guarded(c, st, [&] {
    const char* who = form == 2 ? "check_form2" : "check_form1";
    if (form != 1 && form != 2) throw DomainError{BSE_ERR_INVALID_SPEC, 0, -1, "form must be 1 or 2"};
    if (ldm < rows) throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1, std::string(who) + ": matrix must be square"};
    const int64_t h = half_dimension(rows, who);
    const size_t mm = size_t(rows) * size_t(rows);
    Bump w = arena(c, mm * sizeof(z_t) + form_workspace_bytes() + 4096);
    z_t* dM = w.take<z_t>(mm);
    double* d_out = w.take<double>(4);
    if (rows > 0) h2d(c, dM, rows, m, ldm, rows, rows);
    form_dev(c->stream, form, h, dM, rows, d_out, w);
    double sums[3];
    BSE_CUDA(cudaMemcpyAsync(sums, d_out, sizeof(sums), cudaMemcpyDeviceToHost, c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
    form_result(form, sums, tol, result);
  });
}

int bse_negative_spectrum_device(bse_ctx* c, int64_t n, int64_t k, const double* d_lambda,
                                 const double* d_v, int64_t ldv, double* d_lambda_out,
                                 double* d_v_out, int64_t ldvo, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 0 || k < 0 || ldv < 2 * n || ldvo < 2 * n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1,
                        "spectral result does not match the matrix dimension"};
    check_aligned16({d_v, d_v_out});
    negative_spectrum_dev(c->stream, n, k, d_lambda, reinterpret_cast<const z_t*>(d_v), ldv,
                          d_lambda_out, reinterpret_cast<z_t*>(d_v_out), ldvo);
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bse_negative_spectrum(bse_ctx* c, int64_t n, int64_t k, const double* lambda,
                          const double* v, int64_t ldv, double* lambda_out, double* v_out,
                          int64_t ldvo, bse_status* st) {
  return guarded(c, st, [&] {
    if (n < 0 || k < 0 || ldv < 2 * n || ldvo < 2 * n)
      throw DomainError{BSE_ERR_DIMENSION_MISMATCH, 0, -1,
                        "spectral result does not match the matrix dimension"};
    if (n == 0 || k == 0) return;
    const size_t vk = 2 * size_t(n) * size_t(k);
    Bump w = arena(c, 2 * vk * sizeof(z_t) + 2 * size_t(k) * sizeof(double) + 4096);
    z_t* dV = w.take<z_t>(vk);
    z_t* dO = w.take<z_t>(vk);
    double* dl = w.take<double>(size_t(k));
    double* dlo = w.take<double>(size_t(k));
    h2d(c, dV, 2 * n, v, ldv, 2 * n, k);
    BSE_CUDA(cudaMemcpyAsync(dl, lambda, sizeof(double) * size_t(k), cudaMemcpyHostToDevice,
                             c->stream));
    negative_spectrum_dev(c->stream, n, k, dl, dV, 2 * n, dlo, dO, 2 * n);
    d2h(c, v_out, ldvo, dO, 2 * n, 2 * n, k);
    BSE_CUDA(cudaMemcpyAsync(lambda_out, dlo, sizeof(double) * size_t(k), cudaMemcpyDeviceToHost,
                             c->stream));
    BSE_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
