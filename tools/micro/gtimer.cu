// Resolution of %globaltimer vs clock64 on this GPU: distinct increments seen by one thread.
#include <cstdio>
#include <cstdint>
__global__ void k(uint64_t* out, int n) {
  uint64_t prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int k = 0;
  long long c0 = clock64();
  while (k < n) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[k++] = t - prev; prev = t; }
  }
  out[n] = clock64() - c0;
}
int main() {
  const int n = 64;
  uint64_t* d; cudaMalloc(&d, (n + 1) * 8);
  k<<<1, 1>>>(d, n);
  uint64_t h[n + 1];
  cudaMemcpy(h, d, (n + 1) * 8, cudaMemcpyDeviceToHost);
  uint64_t mn = ~0ull, mx = 0, sum = 0;
  for (int i = 1; i < n; ++i) { mn = h[i] < mn ? h[i] : mn; mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
  printf("globaltimer increments (ns): min %llu max %llu mean %.1f; %d increments took %llu clocks\n",
         (unsigned long long)mn, (unsigned long long)mx, (double)sum / (n - 1), n, (unsigned long long)h[n]);
  return 0;
}
