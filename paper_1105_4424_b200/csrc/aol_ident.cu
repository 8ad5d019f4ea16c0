// The reference's identity-tiler device intrinsics on B200.
//
// Semantics follow the reference executor (refexec.py:476-516) and the kernel
// bodies its code generator emits (codegen.py:126-179): element rho of every
// vector port for rho in [first, first+count).  Arithmetic is IEEE with the
// product and the sum rounded separately (numpy ufunc order), so copy/sub/scale/
// axpy/spmv_csr are bit-exact with the reference; dot_partial is a
// deterministic warp-shuffle tree (tolerance-pinned like the reference's BLAS
// dot, tests/test_refexec.py:374-389).
#include "aol_common.cuh"

namespace aol {

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <typename T> __device__ __forceinline__ T sub_rn(T a, T b);
template <> __device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

#define GRID_STRIDE(i, first, count)                                            \
  for (int64_t i = (first) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;    \
       i < (first) + (count); i += (int64_t)gridDim.x * blockDim.x)

template <typename T>
__global__ void k_sub(const T* __restrict__ x, const T* __restrict__ y, T* __restrict__ z, int64_t first,
                      int64_t count) {
  GRID_STRIDE(i, first, count) z[i] = sub_rn(x[i], y[i]);
}

template <typename T>
__global__ void k_scale(T* __restrict__ y, T a, const T* __restrict__ a_dev, int64_t first, int64_t count) {
  if (a_dev) a = *a_dev;
  GRID_STRIDE(i, first, count) y[i] = mul_rn(y[i], a);
}

template <typename T>
__global__ void k_axpy(T* __restrict__ y, const T* __restrict__ x, T a, const T* __restrict__ a_dev, int has_a,
                       int64_t first, int64_t count) {
  if (a_dev) a = *a_dev;
  if (has_a) {
    GRID_STRIDE(i, first, count) y[i] = add_rn(y[i], mul_rn(a, x[i]));
  } else {
    GRID_STRIDE(i, first, count) y[i] = add_rn(y[i], x[i]);
  }
}

template <typename T>
__global__ void k_copy(const T* __restrict__ s, T* __restrict__ d, int64_t first, int64_t count) {
  GRID_STRIDE(i, first, count) d[i] = s[i];
}

// One thread per row, entries strictly left to right (refexec.py:111-121).
template <typename T, typename I>
__global__ void k_spmv(const I* __restrict__ rowptr, const I* __restrict__ colidx, const T* __restrict__ values,
                       const T* __restrict__ x, T* __restrict__ y, int64_t first, int64_t count) {
  GRID_STRIDE(i, first, count) {
    T acc = T(0);
    const int64_t e = rowptr[i + 1];
    for (int64_t k = rowptr[i]; k < e; ++k) acc = add_rn(acc, mul_rn(values[k], x[colidx[k]]));
    y[i] = acc;
  }
}

// Deterministic two-level dot: fixed grid, each block reduces a fixed slice with
// warp shuffles, a single block then sums the block partials in index order.
constexpr int kDotBlocks = 1024;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) k_dot_blocks(const T* __restrict__ a, const T* __restrict__ b,
                                                    int64_t first, int64_t count, double* __restrict__ part) {
  double acc = 0.0;
  GRID_STRIDE(i, first, count) acc += (double)a[i] * (double)b[i];
  __shared__ double red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) k_dot_final(const double* __restrict__ part, int n, T* __restrict__ out) {
  __shared__ double red[32];
  double v = threadIdx.x < n ? part[threadIdx.x] : 0.0;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = red[threadIdx.x];
    v = warp_sum(v);
    if (threadIdx.x == 0) out[0] = (T)v;
  }
}

static double* dot_scratch(int dev) {
  static double* bufs[64] = {nullptr};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!bufs[dev]) {
    if (cudaMalloc(&bufs[dev], kDotBlocks * sizeof(double)) != cudaSuccess) bufs[dev] = nullptr;
  }
  return bufs[dev];
}

// Host scalar ops of the reference (refexec.py:462-474) as one-thread device kernels, so a
// loop body runs without host round trips.  IEEE division / sqrt are correctly rounded in
// CUDA (no fast-math), as in Python, so the results are bit-identical.
template <typename T>
__global__ void k_scalar_div(const T* num, const T* den, T* q) {
  q[0] = (T)((double)num[0] / (double)den[0]);
}
template <typename T>
__global__ void k_scalar_neg(const T* a, T* z) { z[0] = -a[0]; }
template <typename T>
__global__ void k_rel_residual(const T* num, const T* den, T* z) {
  z[0] = (T)(sqrt((double)num[0]) / sqrt((double)den[0]));
}
// dot_partial combine: total = 0.0; total += p for p in partials (refexec.py:483-486)
template <typename T>
__global__ void k_partials_sum(const T* p, int n, T* s) {
  double total = 0.0;
  for (int i = 0; i < n; ++i) total = __dadd_rn(total, (double)p[i]);
  s[0] = (T)total;
}

double* dot_scratch_for_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  return dot_scratch(dev);
}

template <typename T>
static int launch_ident_t(const aol_task& t, int64_t first, int64_t count, void* const* ports,
                          const double* scalars, cudaStream_t s) {
  const unsigned g = grid_for(count, 1024, 16);
  const bool dev_scalars = (t.flags & AOL_FLAG_DEVICE_SCALARS) != 0;
  switch (t.op) {
    case AOL_OP_COPY:
      k_copy<T><<<g, 256, 0, s>>>((const T*)ports[0], (T*)ports[1], first, count);
      break;
    case AOL_OP_SUB:
      k_sub<T><<<g, 256, 0, s>>>((const T*)ports[0], (const T*)ports[1], (T*)ports[2], first, count);
      break;
    case AOL_OP_SCALE: {
      const T* a_dev = dev_scalars ? (const T*)ports[1] : nullptr;
      if (!a_dev && (t.n_scalars < 1 || !scalars)) return fail(AOL_EINVAL, "scale needs scalar a");
      k_scale<T><<<g, 256, 0, s>>>((T*)ports[0], a_dev ? T(0) : (T)scalars[0], a_dev, first, count);
      break;
    }
    case AOL_OP_AXPY: {
      const T* a_dev = (dev_scalars && t.n_scalars > 0) ? (const T*)ports[2] : nullptr;
      k_axpy<T><<<g, 256, 0, s>>>((T*)ports[0], (const T*)ports[1],
                                  (t.n_scalars > 0 && !a_dev) ? (T)scalars[0] : T(0), a_dev,
                                  t.n_scalars > 0 ? 1 : 0, first, count);
      break;
    }
    case AOL_OP_SCALAR_DIV:
      k_scalar_div<T><<<1, 1, 0, s>>>((const T*)ports[0], (const T*)ports[1], (T*)ports[2]);
      break;
    case AOL_OP_SCALAR_NEG:
      k_scalar_neg<T><<<1, 1, 0, s>>>((const T*)ports[0], (T*)ports[1]);
      break;
    case AOL_OP_REL_RESIDUAL:
      k_rel_residual<T><<<1, 1, 0, s>>>((const T*)ports[0], (const T*)ports[1], (T*)ports[2]);
      break;
    case AOL_OP_PARTIALS_SUM:
      k_partials_sum<T><<<1, 1, 0, s>>>((const T*)ports[0], (int)count, (T*)ports[1]);
      break;
    case AOL_OP_SPMV_CSR: {
      const unsigned gs = grid_for(count, 256, 32);
      if (t.index_dtype == AOL_I64)
        k_spmv<T, int64_t><<<gs, 256, 0, s>>>((const int64_t*)ports[0], (const int64_t*)ports[1],
                                              (const T*)ports[2], (const T*)ports[3], (T*)ports[4], first, count);
      else
        k_spmv<T, int32_t><<<gs, 256, 0, s>>>((const int32_t*)ports[0], (const int32_t*)ports[1],
                                              (const T*)ports[2], (const T*)ports[3], (T*)ports[4], first, count);
      break;
    }
    case AOL_OP_DOT_PARTIAL: {
      int dev = 0;
      AOL_CUDA_CHECK(cudaGetDevice(&dev));
      double* part = dot_scratch(dev);
      if (!part) return fail(AOL_ECUDA, "cannot allocate dot scratch");
      k_dot_blocks<T><<<kDotBlocks, 256, 0, s>>>((const T*)ports[0], (const T*)ports[1], first, count, part);
      AOL_LAUNCH_CHECK("k_dot_blocks");
      k_dot_final<T><<<1, kDotBlocks, 0, s>>>(part, kDotBlocks, (T*)ports[2]);
      break;
    }
    default:
      return fail(AOL_EUNSUPPORTED, "unknown identity op");
  }
  AOL_LAUNCH_CHECK("identity op");
  return AOL_OK;
}

int launch_identity(const aol_task& t, int64_t first, int64_t count, void* const* ports, const double* scalars,
                    cudaStream_t s) {
  if (t.op == AOL_OP_COPY && (t.dtype == AOL_I32 || t.dtype == AOL_I64)) {
    const unsigned g = grid_for(count, 1024, 16);
    if (t.dtype == AOL_I32) k_copy<int32_t><<<g, 256, 0, s>>>((const int32_t*)ports[0], (int32_t*)ports[1], first, count);
    else k_copy<int64_t><<<g, 256, 0, s>>>((const int64_t*)ports[0], (int64_t*)ports[1], first, count);
    AOL_LAUNCH_CHECK("k_copy");
    return AOL_OK;
  }
  if (t.dtype == AOL_F32) return launch_ident_t<float>(t, first, count, ports, scalars, s);
  if (t.dtype == AOL_F64) return launch_ident_t<double>(t, first, count, ports, scalars, s);
  return fail(AOL_EUNSUPPORTED, "identity ops need float32/float64 values");
}

}  // namespace aol
