// common.cuh — shared device/host helpers for the B200 (sm_100a) BSE eigensolver.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <stdexcept>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace bseg {

// Interleaved complex128 (re, im) — the column-major layout of Eigen::MatrixXcd that the
// reference uses (types.hpp:17-18); kept on device so no host-side repacking is needed.
using z_t = double2;

struct CudaError : std::runtime_error {
  cudaError_t err;
  CudaError(cudaError_t e, const char* what)
      : std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e)), err(e) {}
};

#define BSE_CUDA(expr)                                              \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) throw ::bseg::CudaError(_e, #expr);      \
  } while (0)

// Every kernel launch of the library goes through this counter (bse_ctx_kernel_launches).
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int n = 1) {
  if (g_launch_counter) *g_launch_counter += n;
}
#define BSE_LAUNCH_CHECK()                   \
  do {                                       \
    ::bseg::count_launch();                  \
    BSE_CUDA(cudaGetLastError());            \
  } while (0)

// Optional live per-kernel timing (enabled per context): CUDA event pairs around the
// dominant kernel classes, summed after the solve. kind 0 = DMMA GEMM, 1 = panel kernel.
struct KernelTimer {
  cudaEvent_t* pool = nullptr;
  int capacity = 0;
  int used = 0;
  int kind[4096];
  double work[4096];   // flops (GEMM, complex-equivalent: 8 per complex MAC) or algorithmic
                       // bytes (panel) of each timed launch
  double work2[4096];  // GEMM: real flops the DMMA pipe executes (6 per complex MAC in 3M)
};
extern thread_local KernelTimer* g_timer;
// Cap on the CTAs of the cooperative panel kernels (0 = every SM): the batch driver runs two
// solves at once, each panel kernel on half of the SMs, so one solve's latency-bound panels
// overlap the other's GEMM phases (set per calling thread from its context).
extern thread_local int g_panel_ctas;
// The cap in force for this thread's panel launches: the batch lane's, else the developer
// switch BSE_SOLO_PANEL_CTAS (a single solve's panels on fewer SMs, to trace a lane's panel).
int panel_cta_cap();
inline int timer_begin(cudaStream_t s, int kind, double work, double work2 = -1.0) {
  KernelTimer* t = g_timer;
  if (!t || t->used + 2 > t->capacity || t->used / 2 >= 4096) return -1;
  const int slot = t->used / 2;
  t->kind[slot] = kind;
  t->work[slot] = work;
  t->work2[slot] = work2 < 0.0 ? work : work2;
  cudaEventRecord(t->pool[t->used], s);
  t->used += 2;
  return slot;
}
inline void timer_end(cudaStream_t s, int slot) {
  if (slot < 0 || !g_timer) return;
  cudaEventRecord(g_timer->pool[2 * slot + 1], s);
}

// One-time setup per CUDA device: kernel attributes (the dynamic shared-memory limit) and
// occupancy queries are per device, so a process that runs solves on several devices (one
// context per device, or batch lanes on the same device from several host threads) sets them
// up once for each device. Every call site instantiates its own storage (the lambda's type).
constexpr int kMaxDevices = 64;
template <typename F>
const auto& per_device(F&& setup) {
  using T = decltype(setup());
  static std::once_flag once[kMaxDevices];
  static T value[kMaxDevices];
  int dev = 0;
  BSE_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("device index out of range");
  std::call_once(once[dev], [&] { value[dev] = setup(); });
  return value[dev];
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ z_t zmake(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ z_t zadd(z_t a, z_t b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ z_t zsub(z_t a, z_t b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ z_t zmul(z_t a, z_t b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ z_t zcmul(z_t a, z_t b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ z_t zconj(z_t a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ z_t zscale(z_t a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += a * b
__device__ __forceinline__ void zfma(z_t& acc, z_t a, z_t b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void zcfma(z_t& acc, z_t a, z_t b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
__device__ __forceinline__ double zabs2(z_t a) { return a.x * a.x + a.y * a.y; }

// ------------------------------------------------------------------ warp/block reductions
// Grid-wide barrier for cooperative (co-resident) launches: after a CTA barrier, thread 0
// adds 1 to a per-launch zeroed counter with a release reduction (no round trip) and polls
// it with acquire loads until every CTA of this epoch has arrived; the closing CTA barrier
// releases the block. One L2 round trip less than an arrive-with-return barrier.
struct GridBarrier {
  unsigned* ctr;
  unsigned target;
  __device__ __forceinline__ explicit GridBarrier(unsigned* c) : ctr(c), target(0) {}
  __device__ __forceinline__ void sync() {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
    __syncthreads();
  }
};

// Every warp-collective helper starts with warp_converge(): a warp that reaches a full-mask
// shuffle in a diverged state (after lane-dependent branches) otherwise takes the BRA.DIV
// fallback path, measured at ~14k cycles for a handful of shuffles in the panel kernels.
// (A plain __syncwarp() is folded away by the compiler there; the volatile bar.warp.sync
// stays, but ptxas may still turn it into a NOP when it believes the warp converged, so the
// panel kernels also put a CTA barrier -- WARPSYNC.ALL + BAR -- in front of warp-collective
// blocks that follow lane-dependent code.)
__device__ __forceinline__ void warp_converge() { asm volatile("bar.warp.sync -1;" ::: "memory"); }
__device__ __forceinline__ double warp_sum(double v) {
  warp_converge();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ z_t warp_zsum(z_t v) {
  warp_converge();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  warp_converge();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` must hold blockDim.x/32 doubles. Result broadcast to all threads.
__device__ inline double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // re-converge every warp before the butterflies (see warp_converge)
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];  // fixed order: deterministic
  return s;
}

// ------------------------------------------------------------------ async copy primitives
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte global->shared copy bypassing L1; src_bytes = 0 zero-fills (predication).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(n));
}
// 8-byte copy (cg only supports 16; use .ca for 8B).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ------------------------------------------------------------------ latency-bound reductions
// sum_k p[k * es] over k = start, start + stride, ... < hi; loads issued 16 at a time (one
// memory round trip for up to 16 terms), fixed summation order.
__device__ __forceinline__ z_t zsum_strided16(const z_t* p, int64_t es, int start, int hi,
                                               int stride) {
  z_t s[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) s[u] = make_double2(0.0, 0.0);
  for (int k0 = start; k0 < hi; k0 += 16 * stride) {
    z_t v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      v[u] = (k0 + u * stride < hi) ? p[int64_t(k0 + u * stride) * es] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 16; ++u) s[u & 3] = zadd(s[u & 3], v[u]);
  }
  return zadd(zadd(s[0], s[1]), zadd(s[2], s[3]));
}

// The same sum with loads issued 8 at a time (for call sites short of registers: a batch of 16
// that does not fit is serialised by the compiler into 16 round trips).
__device__ __forceinline__ z_t zsum_strided8(const z_t* p, int64_t es, int start, int hi,
                                             int stride) {
  z_t s[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) s[u] = make_double2(0.0, 0.0);
  for (int k0 = start; k0 < hi; k0 += 8 * stride) {
    z_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (k0 + u * stride < hi) ? p[int64_t(k0 + u * stride) * es] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u & 3] = zadd(s[u & 3], v[u]);
  }
  return zadd(zadd(s[0], s[1]), zadd(s[2], s[3]));
}

// Sums each of 16 complex values over the 32 lanes of a warp by recursive halving (16
// complex shuffles in all); on return lane l holds the total of value (l >> 1).
__device__ __forceinline__ z_t warp_transpose_zsum16(z_t (&v)[16]) {
  const int lane = threadIdx.x & 31;
  warp_converge();
#pragma unroll
  for (int st = 0; st < 4; ++st) {
    const int h = 8 >> st, o = 16 >> st;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < h) {
        const z_t keep = up ? v[h + j] : v[j];
        const z_t send = up ? v[j] : v[h + j];
        z_t r;
        r.x = __shfl_xor_sync(0xffffffffu, send.x, o);
        r.y = __shfl_xor_sync(0xffffffffu, send.y, o);
        v[j] = zadd(keep, r);
      }
    }
  }
  z_t r;
  warp_converge();
  r.x = __shfl_xor_sync(0xffffffffu, v[0].x, 1);
  r.y = __shfl_xor_sync(0xffffffffu, v[0].y, 1);
  return zadd(v[0], r);
}

// Sums each of 16 complex values over the 8 lanes of a warp that share lane bits 0..1 (the
// rows of a 4-lanes-per-row mapping), by halving over lane bits 4, 3, 2. On return a lane
// holds the totals of values idx and idx + 1, idx = 8 b4 + 4 b3 + 2 b2.
__device__ __forceinline__ void warp_transpose_zsum16_rows(z_t (&v)[16], z_t& t0, z_t& t1) {
  const int lane = threadIdx.x & 31;
  warp_converge();
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int h = 8 >> st, o = 16 >> st;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < h) {
        const z_t keep = up ? v[h + j] : v[j];
        const z_t send = up ? v[j] : v[h + j];
        z_t r;
        r.x = __shfl_xor_sync(0xffffffffu, send.x, o);
        r.y = __shfl_xor_sync(0xffffffffu, send.y, o);
        v[j] = zadd(keep, r);
      }
    }
  }
  t0 = v[0];
  t1 = v[1];
}

// Sums each of 8 complex values over the 32 lanes of a warp (9 complex shuffles in all); on
// return lanes 4j..4j+3 hold the total of value j.
__device__ __forceinline__ z_t warp_transpose_zsum8(z_t (&v)[8]) {
  const int lane = threadIdx.x & 31;
  warp_converge();
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int h = 4 >> st, o = 16 >> st;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < h) {
        const z_t keep = up ? v[h + j] : v[j];
        const z_t send = up ? v[j] : v[h + j];
        z_t r;
        r.x = __shfl_xor_sync(0xffffffffu, send.x, o);
        r.y = __shfl_xor_sync(0xffffffffu, send.y, o);
        v[j] = zadd(keep, r);
      }
    }
  }
  z_t t = v[0];
  warp_converge();
#pragma unroll
  for (int o = 2; o >= 1; o >>= 1) {
    t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
    t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
  }
  return t;
}

// ------------------------------------------------------------------ FP64 tensor core (DMMA)
// D(8x8) += A(8x4, row) * B(4x8, col); lane t holds A[t/4][t%4], B[t%4][t/4],
// C[t/4][2(t%4)], C[t/4][2(t%4)+1]. Lowers to SASS DMMA.8x8x4.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace bseg
