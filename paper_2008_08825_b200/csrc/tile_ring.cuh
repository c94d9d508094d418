// tile_ring.cuh — per-CTA shared-memory ring of 64x64 complex tiles fed by TMA
// (cp.async.bulk.tensor, completion on one mbarrier per slot).
//
// Used by the cooperative panel kernels (hetrd.cu, gebrd.cu): within one panel the trailing
// block is read-only, so each CTA streams its fixed list of tiles through kSlots slots, and a
// tile left in a slot at the end of one mat-vec sweep is reused by the next sweep without a
// reload. One thread issues one 2-D TMA box per tile; the other threads spend no instructions
// on the stream.
//
// The tensor map views the column-major complex matrix as FLOAT64 [2n x n] (lda*16-byte column
// stride) with a 128 x 64 box: a slot holds the tile column-major and dense, element (r, c) at
// c * 64 + r, every column a contiguous 1 KB run in global memory and in the slot. The kernels
// read it with lanes along r (conflict-free). Elements outside the matrix are zero-filled.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace bseg {

constexpr int kRingT = 64;  // tile edge

__device__ __forceinline__ int ring_idx(int r, int c) { return c * kRingT + r; }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Host: tensor map for a column-major complex n x n matrix (see the header comment).
CUtensorMap make_tile_map(const z_t* A, int64_t lda, int64_t n);
// The same view with a box_rows x box_cols complex box (slot layout c * box_rows + r).
CUtensorMap make_tile_map_box(const z_t* A, int64_t lda, int64_t n, int box_rows, int box_cols);

template <int kSlots>
struct TileRing {
  z_t* buf;          // kSlots * 64 * 64, 128-byte aligned
  uint64_t* bars;    // kSlots mbarriers
  uint32_t pending;  // slot s has a load not yet waited for (identical in every thread)
  uint32_t phase;    // parity of the next completion of slot s

  // All threads; ends with a CTA barrier.
  __device__ void init(z_t* b, uint64_t* br) {
    buf = b;
    bars = br;
    pending = 0;
    phase = 0;
    if (threadIdx.x == 0)
      for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    fence_proxy_async_smem();
    __syncthreads();
  }
  __device__ const z_t* slot(int s) const { return buf + s * kRingT * kRingT; }

  // All threads call (bookkeeping); thread 0 issues the box of the tile with top-left element
  // (R0, C0). The slot must be free (a CTA barrier since its last reader).
  __device__ void issue(int s, const CUtensorMap* map, int64_t R0, int64_t C0) {
    pending |= 1u << s;
    if (threadIdx.x != 0) return;
    z_t* dst = buf + s * kRingT * kRingT;
    mbar_arrive_expect_tx(&bars[s], kRingT * kRingT * 16u);
    tma_load_2d(dst, map, int(2 * R0), int(C0), &bars[s]);
  }
  // All threads: make slot s readable (waits only if a load is outstanding).
  __device__ void acquire(int s) {
    if (pending & (1u << s)) {
      mbar_wait_parity(&bars[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      pending &= ~(1u << s);
    }
  }
  __device__ void drain() {
    for (int s = 0; s < kSlots; ++s) acquire(s);
  }
};

}  // namespace bseg
