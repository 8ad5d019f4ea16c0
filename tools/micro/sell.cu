// Microbenchmark: CSR thread-per-row spmv vs the same rows in a sliced (SELL-32) layout, on the
// paper's CG matrix shape (27-point operator on 51^3: N 132,651, NNZ 3,442,951), fp64, L2-warm.
// Both accumulate each row left to right with separately rounded products and sums, so their
// outputs are bit-identical; the question is the L1 cost of per-lane row segments (lanes 216 B
// apart) versus lane-interleaved entries.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sell tools/micro/sell.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>

__global__ void k_csr(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                      const double* __restrict__ x, double* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int q = rp[i]; q < rp[i + 1]; ++q) acc = __dadd_rn(acc, __dmul_rn(v[q], x[ci[q]]));
  y[i] = acc;
}

// slice s = rows 32s..32s+31; entry k of lane l at base[s] + 32k + l
__global__ void k_sell(const int* __restrict__ rp, const int64_t* __restrict__ base, const int* __restrict__ sc,
                       const double* __restrict__ sv, const double* __restrict__ x, double* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int len = rp[i + 1] - rp[i];
  const int64_t b = base[i >> 5] + (i & 31);
  double acc = 0.0;
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    int c[4];
    double vv[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = sc[b + 32 * (k + u)];
      vv[u] = sv[b + 32 * (k + u)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(vv[u], xv[u]));
  }
  for (; k < len; ++k) acc = __dadd_rn(acc, __dmul_rn(sv[b + 32 * k], x[sc[b + 32 * k]]));
  y[i] = acc;
}

int main() {
  const int g = 51, n = g * g * g;
  std::vector<int> rp(n + 1), ci;
  std::vector<double> v;
  rp[0] = 0;
  for (int z = 0; z < g; ++z)
    for (int yy = 0; yy < g; ++yy)
      for (int xx = 0; xx < g; ++xx) {
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              const int a = z + dz, b = yy + dy, c = xx + dx;
              if (a < 0 || b < 0 || c < 0 || a >= g || b >= g || c >= g) continue;
              ci.push_back((a * g + b) * g + c);
              v.push_back((dz | dy | dx) ? -1.0 : 26.0);
            }
        rp[(z * g + yy) * g + xx + 1] = (int)ci.size();
      }
  const int nnz = (int)ci.size();
  const int ns = (n + 31) / 32;
  std::vector<int64_t> base(ns + 1);
  base[0] = 0;
  for (int s = 0; s < ns; ++s) {
    int mx = 0;
    for (int l = 0; l < 32 && 32 * s + l < n; ++l) mx = std::max(mx, rp[32 * s + l + 1] - rp[32 * s + l]);
    base[s + 1] = base[s] + 32LL * mx;
  }
  std::vector<int> sc(base[ns], 0);
  std::vector<double> sv(base[ns], 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < rp[i + 1] - rp[i]; ++k) {
      sc[base[i >> 5] + (i & 31) + 32 * k] = ci[rp[i] + k];
      sv[base[i >> 5] + (i & 31) + 32 * k] = v[rp[i] + k];
    }
  std::vector<double> x(n);
  for (int i = 0; i < n; ++i) x[i] = 1.0 + (i % 97) * 0.01;
  printf("n %d nnz %d sell entries %lld (%.3fx)\n", n, nnz, (long long)base[ns], (double)base[ns] / nnz);
  int *d_rp, *d_ci, *d_sc;
  int64_t* d_base;
  double *d_v, *d_sv, *d_x, *d_y1, *d_y2;
  cudaMalloc(&d_rp, (n + 1) * 4);
  cudaMalloc(&d_ci, nnz * 4);
  cudaMalloc(&d_v, nnz * 8);
  cudaMalloc(&d_sc, base[ns] * 4);
  cudaMalloc(&d_sv, base[ns] * 8);
  cudaMalloc(&d_base, (ns + 1) * 8);
  cudaMalloc(&d_x, n * 8);
  cudaMalloc(&d_y1, n * 8);
  cudaMalloc(&d_y2, n * 8);
  cudaMemcpy(d_rp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sc, sc.data(), base[ns] * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sv, sv.data(), base[ns] * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_base, base.data(), (ns + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x, x.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = (n + 255) / 256, reps = 200;
  for (int mode = 0; mode < 2; ++mode) {
    for (int w = 0; w < 5; ++w) {
      if (mode == 0) k_csr<<<blocks, 256>>>(d_rp, d_ci, d_v, d_x, d_y1, n);
      else k_sell<<<blocks, 256>>>(d_rp, d_base, d_sc, d_sv, d_x, d_y2, n);
    }
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) k_csr<<<blocks, 256>>>(d_rp, d_ci, d_v, d_x, d_y1, n);
      else k_sell<<<blocks, 256>>>(d_rp, d_base, d_sc, d_sv, d_x, d_y2, n);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.2f us per spmv (L2-warm, back to back)\n", mode ? "sell" : "csr ", 1e3 * ms / reps);
  }
  std::vector<double> y1(n), y2(n);
  cudaMemcpy(y1.data(), d_y1, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(y2.data(), d_y2, n * 8, cudaMemcpyDeviceToHost);
  printf("bitwise equal: %s\n", memcmp(y1.data(), y2.data(), n * 8) == 0 ? "yes" : "NO");
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
