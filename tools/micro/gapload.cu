// Microbenchmark: gather of m-float patterns at paving p = 2m (the sweep's "gaps" point) into a
// dense stream, with different global-load flavours.  Question: does the load path fetch whole
// 128 B lines (2x DRAM reads for 32/64 B runs) and which flavour fetches only the used sectors?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gapload tools/micro/gapload.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

template <int MODE>
__device__ __forceinline__ uint4 ld4(const float* p) {
  uint4 v;
  if (MODE == 0) {
    v = __ldg(reinterpret_cast<const uint4*>(p));
  } else if (MODE == 1) {
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else if (MODE == 2) {
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else if (MODE == 3) {
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else if (MODE == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  } else {
    asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  }
  return v;
}

// one thread per 16 B group; g -> (rho = g / (m/4), r = g % (m/4))
template <int MODE>
__global__ void __launch_bounds__(256) k_gap(const float* __restrict__ src, float* __restrict__ dst, int64_t ngroups,
                                             int gpp, int p) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = g / gpp, r = g - rho * gpp;
    const uint4 v = ld4<MODE>(src + rho * p + r * 4);
    *reinterpret_cast<uint4*>(dst + g * 4) = v;
  }
}


// mode 6: TMA 2-D box loads {m, R} of the strided source into a smem ring, TMA 2-D stores of the
// same boxes into the dense destination; one elected thread per CTA drives the pipeline.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGES>
__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap ms, const __grid_constant__ CUtensorMap md,
                                            int64_t ntiles, int R, int stage_bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto load = [&](int64_t k) {
    const int s = (int)(k % STAGES);
    const int64_t tile = blockIdx.x + k * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(sm + (size_t)s * stage_bytes)), "l"(&ms), "r"(0), "r"((int)(tile * R)), "r"(su32(&bar[s]))
                 : "memory");
  };
  for (int64_t k = 0; k < mine && k < STAGES; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % STAGES);
    const uint32_t par = (uint32_t)((k / STAGES) & 1);
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 ::"r"(su32(&bar[s])), "r"(par) : "memory");
    const int64_t tile = blockIdx.x + k * gridDim.x;
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(&md), "r"(0), "r"((int)(tile * R)), "r"(su32(sm + (size_t)s * stage_bytes)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage of tile k-1 once its store has read shared memory
    if (k >= 1 && k - 1 + STAGES < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k - 1 + STAGES);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_fill(uint32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}
__global__ void k_check(const uint32_t* d, int64_t T, int m, int pf, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < T * m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / m, k = i - r * m;
    if (d[i] != (uint32_t)(r * pf + k)) atomicAdd(bad, 1ull);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int PF = 4;   // paving = PF * m / 2 (1: overlap, 2: dense, 4: gaps)
template <int STAGES>
float run_tma(const float* src, float* dst, int64_t T, int m, int reps, int R, int ctas_per_sm) {
  CUtensorMap ms, md;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)T};
  cuuint64_t ss[1] = {(cuuint64_t)(PF * m / 2 * 4)}, ds[1] = {(cuuint64_t)(m * 4)};
  cuuint32_t box[2] = {(cuuint32_t)m, (cuuint32_t)R}, es[2] = {1, 1};
  auto fn = encode();
  CUresult r1 = fn(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)src, dims, ss, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = fn(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)dst, dims, ds, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("encode failed %d %d\n", (int)r1, (int)r2); return -1; }
  const int stage_bytes = m * R * 4;
  const int smem = STAGES * stage_bytes;
  cudaFuncSetAttribute(k_tma<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t ntiles = (T + R - 1) / R;
  const int grid = 148 * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_tma<STAGES><<<grid, 32, smem>>>(ms, md, ntiles, R, stage_bytes);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_tma<STAGES><<<grid, 32, smem>>>(ms, md, ntiles, R, stage_bytes);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms_ = 0;
  cudaEventElapsedTime(&ms_, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("tma kernel: %s\n", cudaGetErrorString(e)); return -1; }
  return ms_ / reps;
}

template <int MODE>
float run(const float* src, float* dst, int64_t T, int m, int reps) {
  const int gpp = m / 4;
  const int64_t ng = T * gpp;
  int grid = 148 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gap<MODE><<<grid, 256>>>(src, dst, ng, gpp, PF * m / 2);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_gap<MODE><<<grid, 256>>>(src, dst, ng, gpp, PF * m / 2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t T = argc > 1 ? atoll(argv[1]) : 100000000;
  const int only = argc > 2 ? atoi(argv[2]) : -1;
  const int reps = argc > 3 ? atoi(argv[3]) : 10;
  const int only_m = argc > 4 ? atoi(argv[4]) : 0;
  PF = argc > 5 ? atoi(argv[5]) : 4;
  for (int m : {4, 8, 16, 32, 64}) {
    if (only_m && m != only_m) continue;
    float *src, *dst;
    const size_t span = (size_t)T * PF * m / 2 + m;
    if (cudaMalloc(&src, span * 4) != cudaSuccess || cudaMalloc(&dst, (size_t)T * m * 4) != cudaSuccess) {
      printf("alloc failed\n");
      return 1;
    }
    k_fill<<<1184, 256>>>((uint32_t*)src, (int64_t)span);
    unsigned long long* bad;
    cudaMalloc(&bad, 8);
    const double bytes = ((PF >= 2 ? (double)T * m : (double)span) + (double)T * m) * 4;
    for (int mode = 0; mode < 6; ++mode) {
      if (only >= 0 && mode != only) continue;
      float ms = 0;
      switch (mode) {
        case 0: ms = run<0>(src, dst, T, m, reps); break;
        case 1: ms = run<1>(src, dst, T, m, reps); break;
        case 2: ms = run<2>(src, dst, T, m, reps); break;
        case 3: ms = run<3>(src, dst, T, m, reps); break;
        case 4: ms = run<4>(src, dst, T, m, reps); break;
        default: ms = run<5>(src, dst, T, m, reps); break;
      }
      printf("m=%d pf=%d mode=%d  %.4f ms  %.0f GB/s algorithmic\n", m, PF, mode, ms, bytes / (ms * 1e-3) / 1e9);
    }
    if (only < 0 || only == 6)
      for (int st : {4, 8, 16})
      for (int R : {16, 32, 64, 128, 256})
        for (int cps : {1, 2}) {
          if (st * m * R * 4 * cps > 200 * 1024 || m * R * 4 < 2048 || m * R * 4 > 32768) continue;
          float ms = st == 4 ? run_tma<4>(src, dst, T, m, reps, R, cps)
                   : st == 8 ? run_tma<8>(src, dst, T, m, reps, R, cps) : run_tma<16>(src, dst, T, m, reps, R, cps);
          cudaMemset(bad, 0, 8);
          k_check<<<1184, 256>>>((const uint32_t*)dst, T, m, PF * m / 2, bad);
          unsigned long long nb = 0;
          cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
          cudaMemset(dst, 0, (size_t)T * m * 4);
          printf("m=%d pf=%d mode=6 stages=%d R=%d ctas/sm=%d  %.4f ms  %.0f GB/s algorithmic  mismatches %llu\n", m, PF, st, R, cps, ms,
                 bytes / (ms * 1e-3) / 1e9, nb);
        }
    cudaFree(src);
    cudaFree(dst);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
