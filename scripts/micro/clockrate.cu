// SM clock as seen by clock64 vs %globaltimer for a light spin kernel (sanity check of the
// per-cluster counters of the fused FFN kernel).
#include <cstdio>
__global__ void spin(unsigned long long* out, long long cycles) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long c0 = clock64();
  while (clock64() - c0 < cycles) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = c1 - c0; out[2 * blockIdx.x + 1] = g1 - g0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 16);
  unsigned long long h[296];
  for (int rep = 0; rep < 3; ++rep) {
    spin<<<148, 32>>>(d, 200000000LL);
    cudaMemcpy(h, d, 148 * 16, cudaMemcpyDeviceToHost);
    double mn = 1e9, mx = 0;
    for (int i = 0; i < 148; ++i) { double r = (double)h[2*i] / h[2*i+1] * 1e3; mn = r < mn ? r : mn; mx = r > mx ? r : mx; }
    printf("spin: clock64/globaltimer = %.0f .. %.0f MHz\n", mn, mx);
  }
  return 0;
}
