// Device helpers shared by the identity-op kernels (aol_ident.cu) and the persistent
// LoopStep interpreter (aol_loopk.cu): IEEE ops with the product and the sum rounded
// separately (numpy ufunc order), and the fixed dot reduction tree.
#pragma once

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

// One CSR row, strictly left to right with the product and the sum rounded separately
// (refexec.py:111-121).  The entries are consumed in batches of 8: every colidx/values load
// of a batch, then every x gather, then the 8 dependent adds — the loads of a batch are in
// flight together instead of one L2 round trip per entry, and the add order is unchanged.
template <typename T, typename I>
__device__ __forceinline__ T csr_row(const I* colidx, const T* values, const T* x, int64_t q, int64_t e) {
  T acc = T(0);
  for (; q + 8 <= e; q += 8) {
    I c[8];
    T v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      c[u] = colidx[q + u];
      v[u] = values[q + u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  if (q + 4 <= e) {
    I c[4];
    T v[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = colidx[q + u];
      v[u] = values[q + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    q += 4;
  }
  for (; q < e; ++q) acc = add_rn(acc, mul_rn(values[q], x[colidx[q]]));
  return acc;
}

constexpr int kDotBlocks = 1024;
constexpr int kMaxScalarSeq = 8;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace aol
