// Microbenchmark: per-iteration cost of elementwise passes inside a persistent cooperative
// kernel (148 x 1024 threads, the aol_loop_persistent mapping), n = 132,496 doubles.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(double* x, double* y, int64_t n, int iters, int vmap) {
  cg::grid_group g = cg::this_grid();
  const int sub = threadIdx.x >> 8, t = threadIdx.x & 255;
  const int slot = blockIdx.x * 4 + sub, nslots = gridDim.x * 4;
  for (int it = 0; it < iters; ++it) {
    if (MODE >= 1) {
      if (vmap) {
        for (int vb = slot; vb < 1024; vb += nslots)
          for (int64_t i = (int64_t)vb * 256 + t; i < n; i += 262144) y[i] = y[i] + 0.5 * x[i];
      } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
          y[i] = y[i] + 0.5 * x[i];
      }
    }
    if (MODE != 1) g.sync();
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 132496;
  double *x, *y;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMemset(x, 0, n * 8);
  cudaMemset(y, 0, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 5000;
  const char* names[] = {"sync only", "ew only (no sync)", "ew + sync"};
  for (int vmap = 0; vmap < 2; ++vmap)
    for (int mode = 0; mode < 3; ++mode) {
      void* args[] = {&x, &y, (void*)&n, &iters, &vmap};
      const void* f = mode == 0 ? (const void*)k<0> : mode == 1 ? (const void*)k<1> : (const void*)k<2>;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(f, sms, 1024, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("%-20s vmap=%d: %.3f us/iter (%s)\n", names[mode], vmap, 1e3 * ms / iters,
                        cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
