// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64 = SASS DMMA.8x8x4; sm_100 has
// no f64 tcgen05 kind) against DFMA, at 4..32 warps per SM. The SM clock during each timed
// launch is measured inside the kernel (clock64 against %globaltimer on CTA 0), so the
// result states the clock it was taken at. Prints one JSON line; bench.py reads the DMMA
// maximum from profiles/fp64_peak.json as the FP64 tensor roofline denominator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void dmma_loop(double* out, unsigned long long* clk, int iters) {
  const unsigned long long c0 = clock64(), t0 = gtimer();
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk[0] = clock64() - c0;
    clk[1] = gtimer() - t0;
  }
}

__global__ void dfma_loop(double* out, unsigned long long* clk, int iters) {
  const unsigned long long c0 = clock64(), t0 = gtimer();
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = t;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 12345.0) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk[0] = clock64() - c0;
    clk[1] = gtimer() - t0;
  }
}

int main() {
  double* out;
  unsigned long long* dclk;
  cudaMalloc(&out, 8);
  cudaMalloc(&dclk, 16);
  int sms = 0, dev = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best_dmma = 0, best_dfma = 0, mhz_dmma = 0, mhz_dfma = 0;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"runs\": [", prop.name, sms);
  bool first = true;
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int iters = 20000;
    dim3 grid(sms * 2), block(32 * warps / 2 > 1024 ? 1024 : 32 * warps / 2);
    for (int kind = 0; kind < 2; ++kind) {
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {  // the last of three back-to-back launches
        cudaEventRecord(e0);
        if (kind == 0) dmma_loop<<<grid, block>>>(out, dclk, iters);
        else dfma_loop<<<grid, block>>>(out, dclk, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      unsigned long long h[2];
      cudaMemcpy(h, dclk, 16, cudaMemcpyDeviceToHost);
      const double mhz = 1e3 * double(h[0]) / double(h[1]);
      const double flops = kind == 0 ? 2.0 * 8 * 8 * 4 * 8.0 * iters * double(grid.x) * (block.x / 32)
                                     : 2.0 * 16 * iters * double(grid.x) * block.x;
      const double tf = flops / ms / 1e9;
      if (kind == 0 && tf > best_dmma) { best_dmma = tf; mhz_dmma = mhz; }
      if (kind == 1 && tf > best_dfma) { best_dfma = tf; mhz_dfma = mhz; }
      printf("%s{\"kind\": \"%s\", \"warps_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f, "
             "\"sm_mhz\": %.0f}", first ? "" : ", ", kind == 0 ? "dmma_m8n8k4" : "dfma", warps,
             tf, ms, mhz);
      first = false;
    }
  }
  const cudaError_t err = cudaGetLastError();
  printf("], \"fp64_dmma_tflops\": %.3f, \"fp64_dmma_sm_mhz\": %.0f, \"fp64_dfma_tflops\": %.3f, "
         "\"fp64_dfma_sm_mhz\": %.0f, \"err\": \"%s\"}\n",
         best_dmma, mhz_dmma, best_dfma, mhz_dfma, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
