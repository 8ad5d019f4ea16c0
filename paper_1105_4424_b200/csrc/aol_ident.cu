// The reference's identity-tiler device intrinsics on B200.
//
// Semantics follow the reference executor (refexec.py:476-516) and the kernel
// bodies its code generator emits (codegen.py:126-179): element rho of every
// vector port for rho in [first, first+count).  Arithmetic is IEEE with the
// product and the sum rounded separately (numpy ufunc order), so copy/sub/scale/
// axpy/spmv_csr are bit-exact with the reference; dot_partial is a
// deterministic warp-shuffle tree (tolerance-pinned like the reference's BLAS
// dot, tests/test_refexec.py:374-389).
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "aol_common.cuh"
#include "aol_ident.cuh"

namespace aol {

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
  GRID_STRIDE(i, first, count) y[i] = csr_row(colidx, values, x, (int64_t)rowptr[i], (int64_t)rowptr[i + 1]);
}

// Deterministic single-pass dot: a fixed grid of kDotBlocks blocks, each reduces a fixed
// slice with warp shuffles into part[block]; the last block to finish (atomic ticket) sums
// the block partials in index order with the fixed 32 x 32 warp-shuffle tree.  One launch
// per dot instead of two; the result does not depend on block scheduling.
template <typename T>
__global__ void __launch_bounds__(256) k_dot(const T* __restrict__ a, const T* __restrict__ b, int64_t first,
                                             int64_t count, double* __restrict__ part, unsigned* __restrict__ ticket,
                                             T* __restrict__ out) {
  double acc = 0.0;
  GRID_STRIDE(i, first, count) acc = fma((double)a[i], (double)b[i], acc);
  __shared__ double red[32];
  __shared__ bool last;
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = v;
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // 8 warps x 4 groups of 32 partials: group g = part[32g .. 32g+31], lane order, then the
  // 32 group sums in order -- the same tree as one 1024-thread block.
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g = w; g < kDotBlocks / 32; g += blockDim.x >> 5) {
    double v = __ldcg(part + g * 32 + lane);
    v = warp_sum(v);
    if (lane == 0) red[g] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = red[threadIdx.x];
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      out[0] = (T)__dadd_rn(0.0, v);      // 0.0 + v: the reference's combine of one partial
      *ticket = 0;
    }
  }
}

// Several host scalar ops (refexec.py:462-474) in one one-thread launch: op k reads ports
// in0/in1 and writes port out, in program order.
struct ScalarSeq {
  int n;
  int op[kMaxScalarSeq];
  int in0[kMaxScalarSeq], in1[kMaxScalarSeq], out[kMaxScalarSeq];
  void* ports[3 * kMaxScalarSeq];
};

// kDotBlocks partials followed by the ticket counter, per (device, stream): dots on one
// stream are ordered, dots on different streams never share partials or tickets.  Zeroed
// once; the last block of every dot resets the ticket.  The cache is bounded: past
// kMaxDotScratch entries the least recently used unpinned one is freed (after its device
// is idle), and aol_release_scratch() frees every unpinned entry.  Captured device loops
// pin the scratch of their stream (the graph holds its address) until aol_loop_destroy.
struct DotScratch {
  double* p = nullptr;
  int pins = 0;
  uint64_t used = 0;
};
constexpr size_t kMaxDotScratch = 64;
static std::mutex g_scratch_mu;
static std::map<std::pair<int, cudaStream_t>, DotScratch> g_scratch;
static uint64_t g_scratch_tick = 0;

static double* dot_scratch(int dev, cudaStream_t stream, int pin_delta = 0) {
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  auto it = g_scratch.find({dev, stream});
  if (it != g_scratch.end()) {
    it->second.used = ++g_scratch_tick;
    it->second.pins += pin_delta;
    return it->second.p;
  }
  if (pin_delta < 0) return nullptr;
  if (g_scratch.size() >= kMaxDotScratch) {
    auto victim = g_scratch.end();
    for (auto v = g_scratch.begin(); v != g_scratch.end(); ++v)
      if (v->second.pins == 0 && (victim == g_scratch.end() || v->second.used < victim->second.used)) victim = v;
    if (victim != g_scratch.end()) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(victim->first.first);
      cudaDeviceSynchronize();               // no kernel still reads the victim's partials
      cudaFree(victim->second.p);
      cudaSetDevice(cur);
      g_scratch.erase(victim);
    }
  }
  double* p = nullptr;
  if (cudaMalloc(&p, (kDotBlocks + 1) * sizeof(double)) != cudaSuccess) return nullptr;
  if (cudaMemset(p, 0, (kDotBlocks + 1) * sizeof(double)) != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  DotScratch e;
  e.p = p;
  e.pins = pin_delta;
  e.used = ++g_scratch_tick;
  g_scratch[{dev, stream}] = e;
  return p;
}

int release_dot_scratch() {
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = g_scratch.begin(); it != g_scratch.end();) {
    if (it->second.pins > 0) {
      ++it;
      continue;
    }
    cudaSetDevice(it->first.first);
    cudaDeviceSynchronize();
    cudaFree(it->second.p);
    it = g_scratch.erase(it);
  }
  cudaSetDevice(cur);
  return (int)g_scratch.size();
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

template <typename T>
__global__ void k_scalar_seq(ScalarSeq q) {
  for (int k = 0; k < q.n; ++k) {
    const T* a = (const T*)q.ports[q.in0[k]];
    const T* b = q.in1[k] >= 0 ? (const T*)q.ports[q.in1[k]] : nullptr;
    T* z = (T*)q.ports[q.out[k]];
    switch (q.op[k]) {
      case AOL_OP_SCALAR_DIV: z[0] = (T)((double)a[0] / (double)b[0]); break;
      case AOL_OP_SCALAR_NEG: z[0] = -a[0]; break;
      case AOL_OP_REL_RESIDUAL: z[0] = (T)(sqrt((double)a[0]) / sqrt((double)b[0])); break;
      default: break;
    }
  }
}

double* dot_scratch_for_stream(cudaStream_t stream, int pin_delta) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  return dot_scratch(dev, stream, pin_delta);
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
      double* part = dot_scratch(dev, s);
      if (!part) return fail(AOL_ECUDA, "cannot allocate dot scratch");
      k_dot<T><<<kDotBlocks, 256, 0, s>>>((const T*)ports[0], (const T*)ports[1], first, count, part,
                                          reinterpret_cast<unsigned*>(part + kDotBlocks), (T*)ports[2]);
      break;
    }
    case AOL_OP_SCALAR_SEQ: {
      // count = number of ops; scalars = (op, in0, in1, out) per op; in1 = -1 when unused
      if (count < 1 || count > kMaxScalarSeq || !scalars)
        return fail(AOL_EINVAL, "scalar_seq needs 1..8 ops and their (op, in0, in1, out) program");
      ScalarSeq q{};
      q.n = (int)count;
      int np = 0;
      for (int k = 0; k < q.n; ++k) {
        q.op[k] = (int)scalars[4 * k];
        q.in0[k] = (int)scalars[4 * k + 1];
        q.in1[k] = (int)scalars[4 * k + 2];
        q.out[k] = (int)scalars[4 * k + 3];
        const bool two = q.op[k] != AOL_OP_SCALAR_NEG;
        if (q.op[k] < AOL_OP_SCALAR_DIV || q.op[k] > AOL_OP_REL_RESIDUAL)
          return fail(AOL_EINVAL, "scalar_seq: op must be div, neg or rel_residual");
        if (q.in0[k] < 0 || q.out[k] < 0 || (two && q.in1[k] < 0))
          return fail(AOL_EINVAL, "scalar_seq: bad port index");
        np = std::max(np, std::max(q.in0[k], std::max(q.in1[k], q.out[k])) + 1);
      }
      if (np > 3 * kMaxScalarSeq) return fail(AOL_EINVAL, "scalar_seq: too many ports");
      for (int i = 0; i < np; ++i) {
        if (!ports[i]) return fail(AOL_EINVAL, "scalar_seq: null port");
        q.ports[i] = ports[i];
      }
      k_scalar_seq<T><<<1, 1, 0, s>>>(q);
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
