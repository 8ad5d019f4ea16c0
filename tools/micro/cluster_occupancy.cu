// Probe: how many clusters of 1/2/4/8/16 CTAs (214 KB smem, 256 threads: the GEMM pair kernel's
// footprint) can be resident at once -- i.e. how many SMs a cluster size leaves usable.
#include <cstdio>
__global__ void k(int* x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 214 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 * 16 / cs * cs);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 214 * 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d SMs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
