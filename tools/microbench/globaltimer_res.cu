#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int changes = 0; unsigned long long mind = ~0ull;
  long long c0 = clock64();
  while (changes < 100) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { if (t - prev < mind) mind = t - prev; prev = t; ++changes; }
  }
  long long c1 = clock64();
  out[0] = mind; out[1] = c1 - c0;
}
int main() { unsigned long long* d; cudaMalloc(&d, 16); k<<<1,1>>>(d); unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("globaltimer min step %llu ns, 100 changes in %llu cycles\n", h[0], h[1]); }
