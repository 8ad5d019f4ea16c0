// Microbenchmark: cost of one grid-wide barrier in a persistent cooperative kernel
// (148 CTAs x 1024 threads): cooperative_groups grid.sync() vs a flag barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) k_cg(int n) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned target = (gen + 1) * gridDim.x;
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    while (ld_acquire(bar) < target) {}
  }
  ++gen;
  __syncthreads();
}
__global__ void __launch_bounds__(1024, 1) k_flag(int n, unsigned* bar) {
  unsigned gen = 0;
  for (int i = 0; i < n; ++i) grid_barrier(bar, gen);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  cudaMalloc(&bar, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {1024, 256}) {
    for (int n : {1, 10000}) {
      void* args[] = {&n};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("cg grid.sync  threads=%d n=%d: %.3f ms total, %.3f us/barrier (%s)\n", threads, n, ms, 1e3 * ms / n,
             cudaGetErrorString(cudaGetLastError()));
      cudaMemset(bar, 0, 64);
      void* args2[] = {&n, &bar};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_flag, sms, threads, args2, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("flag barrier  threads=%d n=%d: %.3f ms total, %.3f us/barrier (%s)\n", threads, n, ms, 1e3 * ms / n,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
