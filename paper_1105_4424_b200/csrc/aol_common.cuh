// Shared device/host helpers of libaolb200.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/aol_b200.h"

namespace aol {

// ---------------------------------------------------------------- errors ----
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);
// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr if unavailable);
// cast to PFN_cuTensorMapEncodeTiled_v12000 (cudaTypedefs.h)
void* tensor_map_encoder();

#define AOL_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::aol::cuda_fail(_e, #expr); \
  } while (0)

#define AOL_LAUNCH_CHECK(what)                                  \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::aol::cuda_fail(_e, what);   \
    ::aol::count_launch();                                      \
  } while (0)

constexpr int kNumSMs = 148;

// ------------------------------------------------------------ fast divmod ----
// Division of a 32-bit unsigned value by a runtime-constant divisor using the
// round-up magic-number method (one __umulhi + shift).
struct FastDiv32 {
  uint32_t d, mul, shr;
  __host__ __device__ FastDiv32() : d(1), mul(0), shr(0) {}
  __host__ explicit FastDiv32(uint32_t divisor) : d(divisor) {
    if (divisor == 1) { mul = 0; shr = 0; return; }
    uint32_t l = 0;
    while ((1ull << l) < divisor) ++l;
    uint64_t m = ((1ull << 32) * ((1ull << l) - divisor)) / divisor + 1;
    mul = (uint32_t)m;
    shr = l;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
    uint32_t t = __umulhi(n, mul);
    return (t + ((n - t) >> 1)) >> (shr - 1);
  }
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// --------------------------------------------------------- device tiler ----
// Kernel-parameter form of an aol_tiler.  origin_red = origin mod array;
// fit_red[d][k] = fitting mod array (both non-negative).  rep_div / pat_div
// are the unravel divisors (32-bit fast path when every index fits).
struct DevTiler {
  int a, q, p, small;           // ranks; small = repetition and pattern totals < 2^31
  int cheap;                    // every raw coordinate lies in [-2 s_d, 3 s_d): mod by compare/subtract
  int fits32;                   // small && cheap && every raw coordinate and offset fits in int32
  int64_t s[AOL_MAX_RANK];      // array shape
  int64_t st[AOL_MAX_RANK];     // row-major array strides
  int64_t o[AOL_MAX_RANK];      // origin reduced mod s
  int64_t P[AOL_MAX_RANK][AOL_MAX_RANK];
  int64_t F[AOL_MAX_RANK][AOL_MAX_RANK];
  int64_t rep[AOL_MAX_RANK];
  int64_t pat[AOL_MAX_RANK];
  FastDiv32 rep_div[AOL_MAX_RANK];
  FastDiv32 pat_div[AOL_MAX_RANK];
};

__device__ __forceinline__ int64_t emod(int64_t v, int64_t m) {
  int64_t r = v % m;
  return r < 0 ? r + m : r;
}

// unravel x over dims[0..n) row-major (last fastest) into c[]
__device__ __forceinline__ void unravel(const DevTiler& t, bool rep_side, int64_t x,
                                        int64_t c[AOL_MAX_RANK]) {
  const int n = rep_side ? t.q : t.p;
#pragma unroll
  for (int d = AOL_MAX_RANK - 1; d >= 0; --d) {
    if (d >= n) { c[d] = 0; continue; }
    if (d == 0) { c[0] = x; break; }
    if (t.small) {
      uint32_t qv, rv;
      (rep_side ? t.rep_div[d] : t.pat_div[d]).divmod((uint32_t)x, qv, rv);
      c[d] = rv;
      x = qv;
    } else {
      const int64_t dim = rep_side ? t.rep[d] : t.pat[d];
      c[d] = x % dim;
      x /= dim;
    }
  }
}

// Flat offset of (rho, iota): the generic, always-correct restatement of
// SURVEY.md Appendix A with one Euclidean mod per array dimension.
__device__ __forceinline__ int64_t tiler_offset(const DevTiler& t, int64_t rho, int64_t iota) {
  int64_t r[AOL_MAX_RANK], i[AOL_MAX_RANK];
  unravel(t, true, rho, r);
  unravel(t, false, iota, i);
  int64_t off = 0;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    if (d >= t.a) break;
    int64_t e = t.o[d];
#pragma unroll
    for (int j = 0; j < AOL_MAX_RANK; ++j)
      if (j < t.q) e += t.P[d][j] * r[j];
#pragma unroll
    for (int k = 0; k < AOL_MAX_RANK; ++k)
      if (k < t.p) e += t.F[d][k] * i[k];
    if (t.cheap) {                                  // at most two wraps either way
      const int64_t sd = t.s[d];
      if (e >= sd) {
        e -= sd;
        if (e >= sd) e -= sd;
      } else if (e < 0) {
        e += sd;
        if (e < 0) e += sd;
      }
      off += e * t.st[d];
    } else {
      off += emod(e, t.s[d]) * t.st[d];
    }
  }
  return off;
}

// 32-bit form of tiler_offset (DevTiler::fits32): the same Appendix-A arithmetic in int32 --
// one IMAD per term instead of a 64-bit multiply sequence; the generic kernels are integer-bound.
template <int A, int Q, int P>
__device__ __forceinline__ int32_t tiler_offset32(const DevTiler& t, uint32_t rho, uint32_t iota) {
  int32_t r[Q > 0 ? Q : 1], i[P > 0 ? P : 1];
#pragma unroll
  for (int j = Q - 1; j >= 1; --j) {
    uint32_t qv, rv;
    t.rep_div[j].divmod(rho, qv, rv);
    r[j] = (int32_t)rv;
    rho = qv;
  }
  r[0] = (int32_t)rho;
#pragma unroll
  for (int k = P - 1; k >= 1; --k) {
    uint32_t qv, rv;
    t.pat_div[k].divmod(iota, qv, rv);
    i[k] = (int32_t)rv;
    iota = qv;
  }
  i[0] = (int32_t)iota;
  int32_t off = 0;
#pragma unroll
  for (int d = 0; d < A; ++d) {
    int32_t e = (int32_t)t.o[d];
#pragma unroll
    for (int j = 0; j < Q; ++j) e += (int32_t)t.P[d][j] * r[j];
#pragma unroll
    for (int k = 0; k < P; ++k) e += (int32_t)t.F[d][k] * i[k];
    const int32_t sd = (int32_t)t.s[d];
    if (e >= sd) {
      e -= sd;
      if (e >= sd) e -= sd;
    } else if (e < 0) {
      e += sd;
      if (e < 0) e += sd;
    }
    off += e * (int32_t)t.st[d];
  }
  return off;
}

// Per-repetition base coordinates reduced into [0, s_d).
__device__ __forceinline__ void tiler_base(const DevTiler& t, int64_t rho, int64_t base[AOL_MAX_RANK]) {
  int64_t r[AOL_MAX_RANK];
  unravel(t, true, rho, r);
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    if (d >= t.a) { base[d] = 0; continue; }
    int64_t e = t.o[d];
#pragma unroll
    for (int j = 0; j < AOL_MAX_RANK; ++j)
      if (j < t.q) e += t.P[d][j] * r[j];
    base[d] = emod(e, t.s[d]);
  }
}

// ------------------------------------------------------------ host side ----
// Checked conversion of an aol_tiler into its kernel form.
int make_dev_tiler(const aol_tiler& in, DevTiler& out);
int64_t tiler_rep_total(const aol_tiler& t);
int64_t tiler_pat_total(const aol_tiler& t);
int64_t tiler_arr_total(const aol_tiler& t);

// Affine analysis (no wrap over the full box): off = c0 + sum A_j r_j + sum B_k i_k.
struct Affine {
  bool ok;
  int64_t c0;
  int64_t A[AOL_MAX_RANK];
  int64_t B[AOL_MAX_RANK];
};
Affine tiler_affine(const aol_tiler& t);

size_t dtype_size(int dtype);

inline unsigned grid_for(int64_t work, int per_block, int max_waves = 64) {
  int64_t g = (work + per_block - 1) / per_block;
  int64_t cap = (int64_t)kNumSMs * max_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace aol
