// Grid-wide arrival in a persistent cooperative kernel (148 CTAs x 1024 threads): variants
//  flat:      every CTA atom.add's one counter and polls it (the loop kernel's dot arrival)
//  flatflag:  atom.add on the counter; the last arriver (from the returned value) stores a flag
//             on another line; everyone polls the flag (polls do not contend with the atomics)
//  tree:      CTAs add to one of G group counters; each group's last arriver adds to the top
//             counter; the last one stores the flag; everyone polls the flag
#include <cstdio>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE, int G>
__global__ void __launch_bounds__(1024, 1) k(int n, unsigned* mem, int backoff) {
  unsigned* counter = mem;            // line 0
  unsigned* flag = mem + 32;          // line 1
  unsigned* groups = mem + 64;        // one line per group
  const int gsize = (gridDim.x + G - 1) / G;
  for (unsigned gen = 1; gen <= (unsigned)n; ++gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 0) {
        atom_add_acqrel(counter, 1);
        while (ld_acquire(counter) < gen * gridDim.x) if (backoff) __nanosleep(backoff);
      } else if (MODE == 1) {
        const unsigned old = atom_add_acqrel(counter, 1);
        if (old == gen * gridDim.x - 1) st_release(flag, gen);
        else while (ld_acquire(flag) < gen) if (backoff) __nanosleep(backoff);
      } else {
        const int g = blockIdx.x / gsize;
        const unsigned members = (unsigned)min(gsize, (int)gridDim.x - g * gsize);
        const int ngroups = (gridDim.x + gsize - 1) / gsize;
        const unsigned old = atom_add_acqrel(groups + 32 * g, 1);
        bool last = false;
        if (old == gen * members - 1) last = atom_add_acqrel(counter, 1) == gen * ngroups - 1;
        if (last) st_release(flag, gen);
        else while (ld_acquire(flag) < gen) if (backoff) __nanosleep(backoff);
      }
    }
    __syncthreads();
  }
}

template <int MODE, int G>
void run(const char* name, int sms, int n, unsigned* mem, int backoff) {
  cudaMemset(mem, 0, 64 * 1024);
  void* args[] = {&n, &mem, &backoff};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)k<MODE, G>, sms, 1024, args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-10s G=%2d backoff=%3d: %.3f us/arrival (%s)\n", name, G, backoff, 1e3 * ms / n,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* mem;
  cudaMalloc(&mem, 64 * 1024);
  const int n = 20000;
  for (int rep = 0; rep < 2; ++rep)
    for (int bo : {0, 32}) {
      run<0, 1>("flat", sms, n, mem, bo);
      run<1, 1>("flatflag", sms, n, mem, bo);
      run<2, 8>("tree", sms, n, mem, bo);
      run<2, 16>("tree", sms, n, mem, bo);
      run<2, 37>("tree", sms, n, mem, bo);
    }
  return 0;
}
