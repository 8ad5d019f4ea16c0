// Array-OL tiler gather/scatter engine and the CUDA-core tile intrinsics (sm_100a).
//
// Semantics: SURVEY.md Appendix A (tiler) and paper_1105_4424_b200/intrinsics.py
// (elementary tasks).  Every launch covers repetitions [first, first+count) of the
// linearised repetition space, exactly like one reference launch
// (refexec.py:488-514; codegen.py:128-129 guards `gid >= count`).
//
// Arithmetic in the tile intrinsics uses __fmul_rn/__fadd_rn (no FMA contraction)
// in pattern order, which is the order of the reference's spmv_csr executor
// (refexec.py:111-121) that pins the oracle — results are bit-exact.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "aol_async.cuh"
#include "aol_common.cuh"

namespace aol {

// ------------------------------------------------------------ host side ----

static int64_t prod(const int64_t* v, int n) {
  int64_t t = 1;
  for (int i = 0; i < n; ++i) t *= v[i];
  return t;
}
int64_t tiler_rep_total(const aol_tiler& t) { return prod(t.rep, t.rep_rank); }
int64_t tiler_pat_total(const aol_tiler& t) { return prod(t.pattern, t.pat_rank); }
int64_t tiler_arr_total(const aol_tiler& t) { return prod(t.array, t.arr_rank); }

static int64_t emod_h(int64_t v, int64_t m) {
  int64_t r = v % m;
  return r < 0 ? r + m : r;
}

int make_dev_tiler(const aol_tiler& in, DevTiler& out) {
  memset(&out, 0, sizeof(out));
  if (in.arr_rank < 1 || in.arr_rank > AOL_MAX_RANK || in.rep_rank < 1 ||
      in.rep_rank > AOL_MAX_RANK || in.pat_rank < 1 || in.pat_rank > AOL_MAX_RANK)
    return fail(AOL_EINVAL, "tiler ranks must be in 1..4");
  out.a = in.arr_rank;
  out.q = in.rep_rank;
  out.p = in.pat_rank;
  for (int d = 0; d < out.a; ++d)
    if (in.array[d] < 1) return fail(AOL_EINVAL, "tiler array dimensions must be >= 1");
  for (int j = 0; j < out.q; ++j)
    if (in.rep[j] < 1) return fail(AOL_EINVAL, "tiler repetition dimensions must be >= 1");
  for (int k = 0; k < out.p; ++k)
    if (in.pattern[k] < 1) return fail(AOL_EINVAL, "tiler pattern dimensions must be >= 1");
  const double lim = 4.0e18;  // keep every raw coordinate inside int64 (< 2^62)
  int64_t acc = 1;
  out.cheap = 1;
  for (int d = out.a - 1; d >= 0; --d) {
    out.s[d] = in.array[d];
    out.st[d] = acc;
    acc *= in.array[d];
    out.o[d] = emod_h(in.origin[d], in.array[d]);
    double span = (double)in.array[d];
    double lo = (double)out.o[d], hi = (double)out.o[d];   // raw coordinate range along d
    for (int j = 0; j < out.q; ++j) {
      out.P[d][j] = in.paving[d][j];
      const double v = (double)in.paving[d][j] * (double)(in.rep[j] - 1);
      span += fabs(v);
      (v < 0 ? lo : hi) += v;
    }
    for (int k = 0; k < out.p; ++k) {
      out.F[d][k] = in.fitting[d][k];
      const double v = (double)in.fitting[d][k] * (double)(in.pattern[k] - 1);
      span += fabs(v);
      (v < 0 ? lo : hi) += v;
    }
    if (span > lim) return fail(AOL_EINVAL, "tiler coordinates overflow int64");
    if (lo < -2.0 * (double)in.array[d] || hi >= 3.0 * (double)in.array[d]) out.cheap = 0;
    if (lo < -2.0e9 || hi > 2.0e9) out.fits32 = -1;
  }
  for (int j = 0; j < out.q; ++j) out.rep[j] = in.rep[j];
  for (int k = 0; k < out.p; ++k) out.pat[k] = in.pattern[k];
  const int64_t R = tiler_rep_total(in), Pt = tiler_pat_total(in);
  out.small = (R < (1ll << 31) && Pt < (1ll << 31)) ? 1 : 0;
  out.fits32 = (out.fits32 == 0 && out.small && out.cheap && acc < (1ll << 31)) ? 1 : 0;
  if (out.small) {
    for (int j = 0; j < out.q; ++j) out.rep_div[j] = FastDiv32((uint32_t)in.rep[j]);
    for (int k = 0; k < out.p; ++k) out.pat_div[k] = FastDiv32((uint32_t)in.pattern[k]);
  }
  return AOL_OK;
}

Affine tiler_affine(const aol_tiler& t) {
  Affine r;
  memset(&r, 0, sizeof(r));
  int64_t st[AOL_MAX_RANK], acc = 1;
  for (int d = t.arr_rank - 1; d >= 0; --d) {
    st[d] = acc;
    acc *= t.array[d];
  }
  for (int d = 0; d < t.arr_rank; ++d) {
    int64_t o = emod_h(t.origin[d], t.array[d]);
    int64_t lo = o, hi = o;
    for (int j = 0; j < t.rep_rank; ++j) {
      int64_t v = t.paving[d][j] * (t.rep[j] - 1);
      lo += std::min<int64_t>(0, v);
      hi += std::max<int64_t>(0, v);
    }
    for (int k = 0; k < t.pat_rank; ++k) {
      int64_t v = t.fitting[d][k] * (t.pattern[k] - 1);
      lo += std::min<int64_t>(0, v);
      hi += std::max<int64_t>(0, v);
    }
    if (lo < 0 || hi >= t.array[d]) return r;  // wraps: not affine
    r.c0 += o * st[d];
  }
  for (int j = 0; j < t.rep_rank; ++j)
    for (int d = 0; d < t.arr_rank; ++d) r.A[j] += t.paving[d][j] * st[d];
  for (int k = 0; k < t.pat_rank; ++k)
    for (int d = 0; d < t.arr_rank; ++d) r.B[k] += t.fitting[d][k] * st[d];
  r.ok = true;
  return r;
}

size_t dtype_size(int dtype) { return (dtype == AOL_F32 || dtype == AOL_I32) ? 4 : 8; }

// ------------------------------------------------------ pattern tables ----
// fr[k * a + d] = (sum_k F_dk i_k) mod s_d for pattern point k: the per-pattern
// part of each coordinate, pre-reduced so one conditional subtract suffices.
constexpr int kTableMax = 4096;  // int64 entries in shared memory (32 KB)

__device__ __forceinline__ void fill_table(const DevTiler& t, int64_t* fr, int64_t npat) {
  for (int64_t k = threadIdx.x; k < npat; k += blockDim.x) {
    int64_t i[AOL_MAX_RANK];
    unravel(t, false, k, i);
#pragma unroll
    for (int d = 0; d < AOL_MAX_RANK; ++d) {
      if (d >= t.a) break;
      int64_t e = 0;
#pragma unroll
      for (int kk = 0; kk < AOL_MAX_RANK; ++kk)
        if (kk < t.p) e += t.F[d][kk] * i[kk];
      fr[k * t.a + d] = emod(e, t.s[d]);
    }
  }
}

__device__ __forceinline__ int64_t table_offset(const DevTiler& t, const int64_t base[AOL_MAX_RANK],
                                                const int64_t* fr, int64_t k) {
  int64_t off = 0;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    if (d >= t.a) break;
    int64_t e = base[d] + fr[k * t.a + d];
    if (e >= t.s[d]) e -= t.s[d];
    off += e * t.st[d];
  }
  return off;
}

// ------------------------------------------------------------- kernels ----

__global__ void k_tiler_offsets(DevTiler t, int64_t first, int64_t count, int64_t npat,
                                int64_t* __restrict__ out) {
  const int64_t n = count * npat;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = tiler_offset(t, first + e / npat, e % npat);
}

// Generic gather -> scatter: one thread per (rho, iota) element (32-bit split when it fits).
template <typename T>
__global__ void __launch_bounds__(256) k_tile_copy_generic(const T* __restrict__ src, T* __restrict__ dst,
                                                           DevTiler ts, DevTiler td, int64_t first, int64_t count,
                                                           int64_t npat, FastDiv32 pdiv, int small) {
  const int64_t n = count * npat;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rho, iota;
    if (small) {
      uint32_t q, r;
      pdiv.divmod((uint32_t)e, q, r);
      rho = first + q;
      iota = r;
    } else {
      rho = first + e / npat;
      iota = e % npat;
    }
    dst[tiler_offset(td, rho, iota)] = src[tiler_offset(ts, rho, iota)];
  }
}

// The same with compile-time ranks and 32-bit arithmetic (both tilers fits32), 4 elements per
// thread with the loads issued before the stores.
template <typename T, int AS, int QS, int PS, int AD, int QD, int PD>
__global__ void __launch_bounds__(256) k_tile_copy_generic32(const T* __restrict__ src, T* __restrict__ dst,
                                                             DevTiler ts, DevTiler td, uint32_t first, uint32_t n,
                                                             FastDiv32 pdiv) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
    T v[4];
    int32_t od[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = e0 + u * stride;
      od[u] = -1;
      if (e < n && e >= e0) {
        uint32_t q, r;
        pdiv.divmod(e, q, r);
        v[u] = src[tiler_offset32<AS, QS, PS>(ts, first + q, r)];
        od[u] = tiler_offset32<AD, QD, PD>(td, first + q, r);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (od[u] >= 0) dst[od[u]] = v[u];
  }
}

// Both tilers affine with a collapsed 1-D repetition and 1-D pattern:
//   src[cs + As*rho + Bs*iota] -> dst[cd + Ad*rho + Bd*iota].
// Consecutive threads take consecutive (rho, iota), so dense sides coalesce.
template <typename T, int UNROLL>
__global__ void __launch_bounds__(256) k_tile_copy_affine(const T* __restrict__ src, T* __restrict__ dst,
                                                          int64_t cs, int64_t As, int64_t Bs, int64_t cd,
                                                          int64_t Ad, int64_t Bd, int64_t first, int64_t n,
                                                          FastDiv32 pdiv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * UNROLL;
  for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x) * UNROLL + threadIdx.x; e0 < n; e0 += stride) {
    T v[UNROLL];
    int64_t od[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t e = e0 + (int64_t)u * blockDim.x;
      od[u] = -1;
      if (e < n) {
        uint32_t q, r;
        pdiv.divmod((uint32_t)e, q, r);
        const int64_t rho = first + q;
        v[u] = __ldg(src + cs + As * rho + Bs * (int64_t)r);
        od[u] = cd + Ad * rho + Bd * (int64_t)r;
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      if (od[u] >= 0) dst[od[u]] = v[u];
  }
}

// Single-element patterns every other element (P == 1, As == 2) into a dense stream, fp32:
// a thread takes 4 consecutive repetitions, reads the 8-element source span as two 16-byte
// vectors (even elements kept) and writes one 16-byte vector -- half the load instructions
// of the scalar gather; the DRAM traffic (whole sectors) is the same.
// U groups per thread per pass (all loads issued before the stores) keep 32*U bytes per thread
// in flight.
template <int U>
__global__ void __launch_bounds__(256) k_gather_stride2(const float* __restrict__ src, float* __restrict__ dst,
                                                        int64_t ngroups) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; g + (U - 1) * stride < ngroups; g += U * stride) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldg(reinterpret_cast<const float4*>(src) + 2 * (g + u * stride));
      b[u] = __ldg(reinterpret_cast<const float4*>(src) + 2 * (g + u * stride) + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      reinterpret_cast<float4*>(dst)[g + u * stride] = make_float4(a[u].x, a[u].z, b[u].x, b[u].z);
  }
  for (; g < ngroups; g += stride) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(src) + 2 * g);
    const float4 b = __ldg(reinterpret_cast<const float4*>(src) + 2 * g + 1);
    reinterpret_cast<float4*>(dst)[g] = make_float4(a.x, a.z, b.x, b.z);
  }
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Affine copy, V consecutive pattern elements per thread (P % V == 0, destination
// contiguous within a pattern and V-aligned).  The source is read as one V-vector
// when the pattern is contiguous (SRC_VEC), else as V strided scalars.
template <typename T> struct Vec2;
template <> struct Vec2<uint32_t> { using t2 = uint2; using t4 = uint4; };
template <> struct Vec2<uint64_t> { using t2 = ulonglong2; using t4 = ulonglong2; };

template <typename T, int V, bool SRC_VEC>
__global__ void __launch_bounds__(256) k_tile_copy_vec(const T* __restrict__ src, T* __restrict__ dst, int64_t cs,
                                                       int64_t As, int64_t Bs, int64_t cd, int64_t Ad,
                                                       int64_t first, int64_t ngroups, FastDiv32 pdiv) {
  using V2 = typename Vec2<T>::t2;
  using V4 = typename Vec2<T>::t4;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t q, r;
    pdiv.divmod((uint32_t)(g * V), q, r);
    const int64_t rho = first + q;
    const int64_t so = cs + As * rho + Bs * (int64_t)r;
    const int64_t doff = cd + Ad * rho + (int64_t)r;
    T v[V];
    if (SRC_VEC) {
      if constexpr (V == 4 && sizeof(T) == 4) {
        const V4 t = __ldg(reinterpret_cast<const V4*>(src + so));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else if constexpr (V == 2) {
        const V2 t = __ldg(reinterpret_cast<const V2*>(src + so));
        v[0] = t.x; v[1] = t.y;
      } else {
#pragma unroll
        for (int u = 0; u < V; ++u) v[u] = __ldg(src + so + u);
      }
    } else {
#pragma unroll
      for (int u = 0; u < V; ++u) v[u] = __ldg(src + so + Bs * u);
    }
    if constexpr (V == 4 && sizeof(T) == 4) {
      V4 t; t.x = v[0]; t.y = v[1]; t.z = v[2]; t.w = v[3];
      *reinterpret_cast<V4*>(dst + doff) = t;
    } else if constexpr (V == 2) {
      V2 t; t.x = v[0]; t.y = v[1];
      *reinterpret_cast<V2*>(dst + doff) = t;
    } else {
#pragma unroll
      for (int u = 0; u < V; ++u) dst[doff + u] = v[u];
    }
  }
}

// TMA box copy: rows of `P` contiguous elements, row pitch As (source) / Ad (destination).
// Both sides are 2-D tensor maps {P, rows}; a CTA streams boxes of R rows through a
// STAGES-deep shared-memory ring: TMA load (mbarrier completion) -> TMA store
// (bulk-group completion).  The copy engine issues only the bytes of each box, the SM
// issues one instruction per box, and no register ever holds the data.  One elected
// thread per CTA drives the whole pipeline (2 CTAs per SM for >= 128 B rows).
// Planes (`tile_copy.tma_plane`): tiles are {bw columns x R rows} boxes of ncb column blocks per
// row block, loaded at column cs0 + cb*bw and stored at cd0 + cb*bw -- the maps' bases are the
// 16 B-aligned addresses at or below each side's first element, so unaligned row starts (shifts,
// crops) need no register path; the last boxes' overhang is zero-filled on load and clipped on store.
template <int STAGES>
__global__ void __launch_bounds__(32) k_tile_copy_tma(const __grid_constant__ CUtensorMap ms,
                                                      const __grid_constant__ CUtensorMap md, int64_t ntiles, int R,
                                                      uint32_t stage_bytes, uint32_t stage_pitch, int64_t ncb,
                                                      int bw, int cs0, int cd0) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[STAGES];
  if (threadIdx.x != 0) return;
  for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;   // tiles blockIdx.x + k*gridDim.x
  auto tile_rc = [&](int64_t k, int& row, int& col) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    const int64_t rb = ncb == 1 ? t : t / ncb;
    row = (int)(rb * R);
    col = (int)(t - rb * ncb) * bw;
  };
  auto load = [&](int64_t k) {
    const int st = (int)(k % STAGES);
    int row, col;
    tile_rc(k, row, col);
    mbar_expect_tx(&full[st], stage_bytes);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(ring + (size_t)st * stage_pitch)),
        "l"(&ms), "r"(cs0 + col), "r"(row), "r"(smem_u32(&full[st]))
        : "memory");
  };
  for (int64_t k = 0; k < mine && k < STAGES; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % STAGES);
    mbar_wait(&full[st], (uint32_t)((k / STAGES) & 1));
    int row, col;
    tile_rc(k, row, col);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&md),
                 "r"(cd0 + col), "r"(row), "r"(smem_u32(ring + (size_t)st * stage_pitch))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage of box k-1 once its store has finished reading shared memory
    if (k >= 1 && k - 1 + STAGES < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k - 1 + STAGES);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Overlapping source rows (0 < As < P, unit fitting, fp32) into dense destination rows: tile t
// of R repetitions needs the contiguous source window [cs + As*r0, cs + As*(r0+R-1) + P), read
// ONCE from DRAM by one bulk copy (the 16-byte aligned part; the <= 3 trailing elements come
// from global memory) into a double-buffered shared-memory ring; 256 threads expand it into P-element
// rows with coalesced 16-byte stores.  Each input element is read once instead of P/As times
// through L1/L2 as the register gather does.
constexpr int kWinMaxStages = 8;
template <int LOGP>
__global__ void __launch_bounds__(256) k_tile_copy_window(const float* __restrict__ src, float* __restrict__ dst,
                                                          int64_t cs, int64_t As, int64_t cd, int64_t first,
                                                          int64_t count, int R, uint32_t win_pitch, int nst) {
  constexpr int P = 1 << LOGP;
  extern __shared__ __align__(128) unsigned char ring_raw[];
  float* ring = reinterpret_cast<float*>(ring_raw);
  __shared__ __align__(8) uint64_t full[kWinMaxStages];
  const int tid = threadIdx.x;
  const int64_t ntiles = (count + R - 1) / R;
  const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto window = [&](int64_t k, int64_t& a0, int64_t& a1, int64_t& w1, int64_t& r0, int64_t& n) {
    r0 = first + (blockIdx.x + k * gridDim.x) * (int64_t)R;
    n = min((int64_t)R, first + count - r0);
    const int64_t w0 = cs + As * r0;
    w1 = cs + As * (r0 + n - 1) + P;
    a0 = w0 & ~int64_t(3);
    a1 = w1 & ~int64_t(3);
  };
  auto load = [&](int64_t k) {
    int64_t a0, a1, w1, r0, n;
    window(k, a0, a1, w1, r0, n);
    const int st = (int)(k % nst);
    const uint32_t bytes = (uint32_t)((a1 - a0) * 4);
    mbar_expect_tx(&full[st], bytes);
    if (bytes) bulk_load(ring + (size_t)st * win_pitch, src + a0, bytes, &full[st]);
  };
  if (tid == 0)
    for (int64_t k = 0; k < mine && k < nst; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % nst);
    int64_t a0, a1, w1, r0, n;
    window(k, a0, a1, w1, r0, n);
    mbar_wait(&full[st], (uint32_t)((k / nst) & 1));
    const float* win = ring + (size_t)st * win_pitch;
    float* out = dst + cd + r0 * P;                    // dense rows: [n][P]
    const int total = (int)(n * P);
    // window-local 32-bit indices: element e of the tile is win[off0 + As*(e/P) + e%P]
    const int off0 = (int)(cs + As * r0 - a0), lim = (int)(a1 - a0), as = (int)As;
    const float* tail = src + a0;
    auto at = [&](int e) -> float {
      const int li = off0 + as * (e >> LOGP) + (e & (P - 1));
      return li < lim ? win[li] : __ldg(tail + li);
    };
    if (((uintptr_t)out & 15) == 0) {
      for (int e = tid * 4; e + 4 <= total; e += 256 * 4)
        *reinterpret_cast<float4*>(out + e) = make_float4(at(e), at(e + 1), at(e + 2), at(e + 3));
      for (int e = (total & ~3) + tid; e < total; e += 256) out[e] = at(e);
    } else {
      for (int e = tid; e < total; e += 256) out[e] = at(e);
    }
    __syncthreads();                                     // stage st consumed by every thread
    if (tid == 0 && k + nst < mine) load(k + nst);
  }
}

// Affine copies whose repetition space and pattern each need two strides per side (2-D block
// tilers: an image cut into b x b blocks written as a dense stream, and back).  Element e of the
// launch is (rho, iota) = (first + e / P, e % P); each side decomposes rho into (r0, r1) with its
// own repetition strides and iota into (i0, i1) with its own pattern strides.  V consecutive
// elements stay inside one row i1 of both patterns, so they move as one V-vector when both
// sides are contiguous there.
struct Side2 {
  int64_t c, A0, A1, B0, B1;
  FastDiv32 nr1, p1;
};

__device__ __forceinline__ int64_t side2_off(const Side2& sd, uint32_t rho, uint32_t iota) {
  uint32_t r0, r1, i0, i1;
  sd.nr1.divmod(rho, r0, r1);
  sd.p1.divmod(iota, i0, i1);
  return sd.c + sd.A0 * r0 + sd.A1 * r1 + sd.B0 * i0 + sd.B1 * i1;
}

template <typename T, int V>
__global__ void __launch_bounds__(256) k_tile_copy_affine2d(const T* __restrict__ src, T* __restrict__ dst, Side2 ss,
                                                            Side2 sd, int64_t first, int64_t ngroups, FastDiv32 pdiv) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t q, iota;
    pdiv.divmod((uint32_t)(g * V), q, iota);
    const uint32_t rho = (uint32_t)(first + q);
    const int64_t so = side2_off(ss, rho, iota), doff = side2_off(sd, rho, iota);
    if constexpr (V == 4 && sizeof(T) == 4) {
      *reinterpret_cast<uint4*>(dst + doff) = __ldg(reinterpret_cast<const uint4*>(src + so));
    } else if constexpr (V == 2 && sizeof(T) == 4) {
      *reinterpret_cast<uint2*>(dst + doff) = __ldg(reinterpret_cast<const uint2*>(src + so));
    } else {
      dst[doff] = __ldg(src + so);
    }
  }
}

// Row-stride gather through TMA (fp32, P in {8, 16, 32, 64}): a tile of RT repetitions x P
// pattern elements arrives as RT/32 {32 reps, P} boxes with the 128B swizzle (16-byte chunk c
// of row i lands at chunk c ^ (i & 7)), is transposed by 128 threads into a staging tile, and
// leaves through TMA stores.  P <= 16: dense [RT][P] staging, one store box, thread e takes
// element e (column reads conflict-free for 8 rows).  P >= 32: staging as P/32 swizzled
// [RT][32] boxes and 4-rep x 8-element warp blocks (reads conflict-free, writes 2-way).
// Three input tiles in flight, two staging tiles; one thread issues every bulk copy.
template <int P>
__global__ void __launch_bounds__(128) k_tile_copy_tma_transpose(const __grid_constant__ CUtensorMap ms,
                                                                 const __grid_constant__ CUtensorMap md,
                                                                 int64_t ntiles) {
  constexpr int RT = P >= 64 ? 64 : 128, NBR = RT / 32;
  constexpr int BOX = 32 * P * 4, BOX_STRIDE = (BOX + 1023) & ~1023, IN_BYTES = NBR * BOX_STRIDE;
  constexpr bool SWO = P >= 32;                            // swizzled [RT][32] output boxes
  constexpr int NBO = SWO ? P / 32 : 1, OBOX = SWO ? RT * 128 : RT * P * 4;
  constexpr int OUT_BYTES = NBO * OBOX, NIN = 3, NOUT = 2;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* in = base;
  unsigned char* out = base + NIN * IN_BYTES;
  __shared__ __align__(8) uint64_t full[NIN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < NIN; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto load = [&](int64_t k) {
    const int st = (int)(k % NIN);
    const int r0 = (int)((blockIdx.x + k * gridDim.x) * RT);
    mbar_expect_tx(&full[st], NBR * BOX);
#pragma unroll
    for (int b = 0; b < NBR; ++b)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(in + st * IN_BYTES + b * BOX_STRIDE)),
          "l"(&ms), "r"(r0 + 32 * b), "r"(0), "r"(smem_u32(&full[st]))
          : "memory");
  };
  auto in_off = [](int r, int i) -> uint32_t {            // byte offset of element (rep r, pattern i)
    const int rl = r & 31;
    return (uint32_t)((r >> 5) * BOX_STRIDE + i * 128 + ((((rl >> 2) ^ (i & 7)) << 4) | ((rl & 3) << 2)));
  };
  if (tid == 0)
    for (int64_t k = 0; k < mine && k < NIN; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % NIN), ob = (int)(k % NOUT);
    mbar_wait(&full[st], (uint32_t)((k / NIN) & 1));
    if (tid == 0 && k >= NOUT) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NOUT - 1) : "memory");
    __syncthreads();
    const unsigned char* src = in + st * IN_BYTES;
    unsigned char* dst = out + ob * OUT_BYTES;
    if constexpr (!SWO) {
#pragma unroll
      for (int e = tid; e < RT * P; e += 128)
        reinterpret_cast<float*>(dst)[e] = *reinterpret_cast<const float*>(src + in_off(e / P, e % P));
    } else {
      // warp block: 4 reps x 8 pattern elements (lane: rep lane >> 3, element lane & 7)
#pragma unroll 4
      for (int blk = warp; blk < (RT / 4) * (P / 8); blk += 4) {
        const int r = (blk % (RT / 4)) * 4 + (lane >> 3), i = (blk / (RT / 4)) * 8 + (lane & 7);
        const int il = i & 31;
        const uint32_t o = (uint32_t)((i >> 5) * OBOX + r * 128 + ((((il >> 2) ^ (r & 7)) << 4) | ((il & 3) << 2)));
        *reinterpret_cast<float*>(dst + o) = *reinterpret_cast<const float*>(src + in_off(r, i));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const int r0 = (int)((blockIdx.x + k * gridDim.x) * RT);
#pragma unroll
      for (int b = 0; b < NBO; ++b)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&md),
                     "r"(32 * b), "r"(r0), "r"(smem_u32(dst + b * OBOX))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (k + NIN < mine) load(k + NIN);
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// "Row-stride" gathers: consecutive repetitions are adjacent in the source (As == 1) while
// the pattern elements are far apart (one array row, Bs >= 32); the destination is the dense
// pattern stream.  A 32x32 (repetition x pattern) tile goes through padded shared memory so
// both the source reads (along repetitions) and the destination writes (along the stream)
// are coalesced — the classic transpose.
template <typename T, bool VEC>
__global__ void __launch_bounds__(256) k_tile_copy_transpose(const T* __restrict__ src, T* __restrict__ dst,
                                                             int64_t cs, int64_t Bs, int64_t cd, int64_t P,
                                                             int64_t first, int64_t count, int pc, int rshift,
                                                             FastDiv32 pcdiv, int pitch) {
  // tile = (1 << rshift) repetitions x pc pattern elements (pc <= 64, <= 4096 elements).
  // pitch == 32/pc (mod 32): a warp's 32 accesses in either phase fall in 32 distinct banks.
  constexpr int PER = VEC ? 4 : 16;                // loads per thread per tile (vectors or scalars)
  constexpr int W = VEC ? 4 : 1;                   // elements per access
  __shared__ T tile[4096 + 32 * 33];
  const int rt = 1 << rshift;
  const int64_t nrb = (count + rt - 1) / rt, npb = (P + pc - 1) / pc;
  for (int64_t b = blockIdx.x; b < nrb * npb; b += gridDim.x) {
    const int64_t rb = b / npb, pb = b - rb * npb;
    const int64_t r0 = first + rb * rt, p0 = pb * pc;
    const int pw = (int)(P - p0 < pc ? P - p0 : pc);
    const int rw = (int)(first + count - r0 < rt ? first + count - r0 : rt);
    const bool full = VEC && pw == pc && rw == rt;
    T v[PER * W];
#pragma unroll
    for (int u = 0; u < PER; ++u) {                                // coalesced along repetitions
      const int k = (threadIdx.x + u * 256) * W;
      const int pl = k >> rshift, rl = k & (rt - 1);
      if (k < pc * rt) {
        const T* sp = src + cs + (r0 + rl) + Bs * (p0 + pl);
        if (full) {
          if constexpr (sizeof(T) == 4) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(sp));
            v[u * W] = q.x; v[u * W + 1] = q.y; v[u * W + 2] = q.z; v[u * W + 3] = q.w;
          } else {
#pragma unroll
            for (int e = 0; e < W; ++e) v[u * W + e] = __ldg(sp + e);
          }
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e)
            if (pl < pw && rl + e < rw) v[u * W + e] = __ldg(sp + e);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int k = (threadIdx.x + u * 256) * W;
      const int pl = k >> rshift, rl = k & (rt - 1);
      if (k < pc * rt) {
#pragma unroll
        for (int e = 0; e < W; ++e)
          if (pl < pw && rl + e < rw) tile[pl * pitch + rl + e] = v[u * W + e];
      }
    }
    __syncthreads();
    if (full) {                                                    // 16-byte stores along the stream
      for (int k = threadIdx.x * 4; k < pw * rw; k += 256 * 4) {
        T o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t rl, pl;
          pcdiv.divmod((uint32_t)(k + e), rl, pl);
          o[e] = tile[pl * pitch + rl];
        }
        T* dp = dst + cd + r0 * P + k;
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<uint4*>(dp) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) dp[e] = o[e];
        }
      }
    } else {
      for (int k = threadIdx.x; k < pw * rw; k += blockDim.x) {    // coalesced along the dense stream
        uint32_t rl, pl;
        if (pw == pc) pcdiv.divmod((uint32_t)k, rl, pl);
        else { rl = (uint32_t)(k / pw); pl = (uint32_t)(k - rl * pw); }
        dst[cd + (r0 + rl) * P + p0 + pl] = tile[pl * pitch + rl];
      }
    }
    __syncthreads();
  }
}

// Contiguous on both sides: a streaming copy with 16-byte vectors.
__global__ void __launch_bounds__(256) k_stream_copy16(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                       int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x * 4 + threadIdx.x; i < n16; i += stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * blockDim.x < n16) v[u] = __ldcs(src + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * blockDim.x < n16) __stcs(dst + i + u * blockDim.x, v[u]);
  }
}

template <typename T>
__global__ void k_stream_copy_tail(const T* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Pattern dot (generic matmul): c[off_c(rho)] = sum_k a_k * b_k, k ascending, no FMA.
template <typename T>
__global__ void k_matmul_generic(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ c,
                                 DevTiler ta, DevTiler tb, DevTiler tc, int64_t first, int64_t count,
                                 int64_t K, int use_table) {
  extern __shared__ int64_t smem[];
  int64_t* fa = smem;
  int64_t* fb = smem + (use_table ? K * ta.a : 0);
  if (use_table) {
    fill_table(ta, fa, K);
    fill_table(tb, fb, K);
    __syncthreads();
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = first + e;
    T acc = T(0);
    if (use_table) {
      int64_t ba[AOL_MAX_RANK], bb[AOL_MAX_RANK];
      tiler_base(ta, rho, ba);
      tiler_base(tb, rho, bb);
      for (int64_t k = 0; k < K; ++k) {
        const T x = a[table_offset(ta, ba, fa, k)], y = b[table_offset(tb, bb, fb, k)];
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, __fmul_rn(x, y));
        else acc = __dadd_rn(acc, __dmul_rn(x, y));
      }
    } else {
      for (int64_t k = 0; k < K; ++k) {
        const T x = a[tiler_offset(ta, rho, k)], y = b[tiler_offset(tb, rho, k)];
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, __fmul_rn(x, y));
        else acc = __dadd_rn(acc, __dmul_rn(x, y));
      }
    }
    c[tiler_offset(tc, rho, 0)] = acc;
  }
}

// Raw (unreduced) base coordinates b_d = o_d + P_d . r for one repetition.
__device__ __forceinline__ void tiler_base_raw(const DevTiler& t, int64_t rho, int64_t b[AOL_MAX_RANK]) {
  int64_t r[AOL_MAX_RANK];
  unravel(t, true, rho, r);
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    b[d] = 0;
    if (d >= t.a) continue;
    int64_t e = t.o[d];
#pragma unroll
    for (int j = 0; j < AOL_MAX_RANK; ++j)
      if (j < t.q) e += t.P[d][j] * r[j];
    b[d] = e;
  }
}

// Per-dimension extent of the pattern: raw offsets F_d . i lie in [lo_d, hi_d].
struct PatSpan {
  int64_t lo[AOL_MAX_RANK], hi[AOL_MAX_RANK];
};

__device__ __forceinline__ bool wrap_free(const DevTiler& t, const PatSpan& sp, const int64_t b[AOL_MAX_RANK],
                                          int64_t& off) {
  bool ok = true;
  off = 0;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    if (d >= t.a) break;
    ok = ok && (b[d] + sp.lo[d] >= 0) && (b[d] + sp.hi[d] < t.s[d]);
    off += b[d] * t.st[d];
  }
  return ok;
}

// raw flat pattern offsets: foff[k] = sum_d (F_d . i_k) * st_d   (valid when the window does not wrap)
__device__ __forceinline__ void fill_raw_offsets(const DevTiler& t, int64_t* foff, int64_t npat) {
  for (int64_t k = threadIdx.x; k < npat; k += blockDim.x) {
    int64_t i[AOL_MAX_RANK];
    unravel(t, false, k, i);
    int64_t o = 0;
#pragma unroll
    for (int d = 0; d < AOL_MAX_RANK; ++d) {
      if (d >= t.a) break;
      int64_t e = 0;
#pragma unroll
      for (int kk = 0; kk < AOL_MAX_RANK; ++kk)
        if (kk < t.p) e += t.F[d][kk] * i[kk];
      o += e * t.st[d];
    }
    foff[k] = o;
  }
}

// Pattern linear map: y_pat[j] = sum_i w[j, i] * x_pat[i], i ascending, no FMA.
// One thread per repetition.  Fast path (window does not wrap): flat offsets
// base + foff[i] with no modulo at all; the x window is read with float4 when
// it is contiguous and 16-byte aligned (XVEC).  Wrapping windows take the
// reduced-table path (one Euclidean mod per dimension per repetition).
template <typename T, int MAXO, bool XVEC>
__global__ void __launch_bounds__(256) k_filter_generic(const T* __restrict__ x, const T* __restrict__ w,
                                                        T* __restrict__ y, DevTiler tx, DevTiler ty, PatSpan sx,
                                                        PatSpan sy, int64_t first, int64_t count, int px, int py,
                                                        int64_t nx) {
  extern __shared__ int64_t smem[];
  int64_t* fx = smem;                                   // reduced tables (wrap path)
  int64_t* fy = fx + (int64_t)px * tx.a;
  int64_t* ox = fy + (int64_t)py * ty.a;                // raw flat offsets (fast path)
  int64_t* oy = ox + px;
  T* ws = reinterpret_cast<T*>(oy + py);
  fill_table(tx, fx, px);
  fill_table(ty, fy, py);
  fill_raw_offsets(tx, ox, px);
  fill_raw_offsets(ty, oy, py);
  for (int k = threadIdx.x; k < px * py; k += blockDim.x) ws[k] = w[k];
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = first + e;
    int64_t bx[AOL_MAX_RANK], by[AOL_MAX_RANK];
    tiler_base_raw(tx, rho, bx);
    tiler_base_raw(ty, rho, by);
#pragma unroll
    for (int d = 0; d < AOL_MAX_RANK; ++d) {   // a window one period away is still whole
      if (d < tx.a) bx[d] = emod(bx[d], tx.s[d]);
      if (d < ty.a) by[d] = emod(by[d], ty.s[d]);
    }
    int64_t xoff, yoff;
    const bool xfree = wrap_free(tx, sx, bx, xoff);
    const bool yfree = wrap_free(ty, sy, by, yoff);
    T acc[MAXO];
#pragma unroll
    for (int j = 0; j < MAXO; ++j) acc[j] = T(0);
    if (XVEC && xfree && (xoff & 3) == 0 && xoff + 16 <= nx) {
      float xv[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + (xoff >> 2) + q);
        xv[4 * q] = v.x; xv[4 * q + 1] = v.y; xv[4 * q + 2] = v.z; xv[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < px) {
#pragma unroll
          for (int j = 0; j < MAXO; ++j)
            if (j < py) acc[j] = __fadd_rn(acc[j], __fmul_rn(ws[j * px + i], xv[i]));
        }
      }
    } else {
      for (int i = 0; i < px; ++i) {
        const T xv = xfree ? __ldg(x + xoff + ox[i]) : __ldg(x + table_offset(tx, bx, fx, i));
#pragma unroll
        for (int j = 0; j < MAXO; ++j) {
          if (j < py) {
            if constexpr (sizeof(T) == 4) acc[j] = __fadd_rn(acc[j], __fmul_rn(ws[j * px + i], xv));
            else acc[j] = __dadd_rn(acc[j], __dmul_rn(ws[j * px + i], xv));
          }
        }
      }
    }
    if (yfree) {
#pragma unroll
      for (int j = 0; j < MAXO; ++j)
        if (j < py) y[yoff + oy[j]] = acc[j];
    } else {
#pragma unroll
      for (int j = 0; j < MAXO; ++j)
        if (j < py) y[table_offset(ty, by, fy, j)] = acc[j];
    }
  }
}

// ---- 32-bit batched form (both tilers fits32, one shared repetition space, indices < 2^31) ----
// A warp covers 32*R consecutive repetitions; lane l takes rho0 + l + 32k (k < R), so each load
// instruction of the warp walks one run of the array while the R repetitions of a lane share one
// unravel, one window check and every weight read.  Same pattern order and rounding as
// k_filter_generic: y_pat[j] = sum_i w[j, i] * x_pat[i], i ascending, mul then add.
__device__ __forceinline__ int32_t wrap2(int32_t e, int32_t s) {   // raw coordinate in [-2s, 3s)
  if (e >= s) {
    e -= s;
    if (e >= s) e -= s;
  } else if (e < 0) {
    e += s;
    if (e < 0) e += s;
  }
  return e;
}

template <int Q>
__device__ __forceinline__ void base32(const DevTiler& t, const int32_t r[Q], int32_t b[AOL_MAX_RANK]) {
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    int32_t e = 0;
    if (d < t.a) {
      e = (int32_t)t.o[d];
#pragma unroll
      for (int j = 0; j < Q; ++j) e += (int32_t)t.P[d][j] * r[j];
    }
    b[d] = e;
  }
}

// base reduced into [0, s_d) (raw bases lie in [-2s, 3s)): the window test and flat offsets use it
__device__ __forceinline__ void reduce32(const DevTiler& t, const int32_t b[AOL_MAX_RANK], int32_t c[AOL_MAX_RANK]) {
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) c[d] = d < t.a ? wrap2(b[d], (int32_t)t.s[d]) : 0;
}

// window of the repetition whose base is b + k*step (k in [0, kmax]) stays inside the array:
// linear in k, so the two ends decide
__device__ __forceinline__ bool window_free32(const DevTiler& t, const PatSpan& sp, const int32_t b[AOL_MAX_RANK],
                                              const int32_t step[AOL_MAX_RANK], int kmax) {
  bool ok = true;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    if (d >= t.a) break;
    const int32_t e = b[d] + kmax * step[d];
    const int32_t lo = min(b[d], e), hi = max(b[d], e);
    ok = ok && lo + (int32_t)sp.lo[d] >= 0 && hi + (int32_t)sp.hi[d] < (int32_t)t.s[d];
  }
  return ok;
}

__device__ __forceinline__ int32_t flat32(const DevTiler& t, const int32_t b[AOL_MAX_RANK]) {
  int32_t o = 0;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d)
    if (d < t.a) o += b[d] * (int32_t)t.st[d];
  return o;
}

// element i of a (possibly wrapping) window: raw base + raw pattern coordinate, reduced per dim
__device__ __forceinline__ int32_t wrapped32(const DevTiler& t, const int32_t b[AOL_MAX_RANK], const int32_t* rc,
                                             int i) {
  int32_t o = 0;
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d)
    if (d < t.a) o += wrap2(b[d] + rc[i * t.a + d], (int32_t)t.s[d]) * (int32_t)t.st[d];
  return o;
}

template <typename T>
__device__ __forceinline__ T mul_add_rn(T acc, T w, T x) {
  if constexpr (sizeof(T) == 4) return __fadd_rn(acc, __fmul_rn(w, x));
  else return __dadd_rn(acc, __dmul_rn(w, x));
}

// XV: the x pattern is one contiguous run of <= 16 floats and a lane's repetitions are 16 B apart:
// each window comes in as four float4 loads with the weights held in registers.
template <typename T, int MAXO, int R, int Q, bool XV>
__global__ void __launch_bounds__(256) k_filter_batched32(const T* __restrict__ x, const T* __restrict__ w,
                                                          T* __restrict__ y, DevTiler tx, DevTiler ty, PatSpan sx,
                                                          PatSpan sy, int32_t first, int32_t count, int px,
                                                          int py, int32_t nx) {
  extern __shared__ __align__(16) unsigned char fsm[];
  T* ws = reinterpret_cast<T*>(fsm);
  int32_t* ox = reinterpret_cast<int32_t*>(ws + px * py);   // raw flat pattern offsets
  int32_t* oy = ox + px;
  int32_t* rx = oy + py;                                     // raw per-dim pattern coordinates
  int32_t* ry = rx + px * tx.a;
  for (int k = threadIdx.x; k < px * py; k += blockDim.x) ws[k] = w ? w[k] : T(1);   // no w: tile_sum (1*x == x)
  for (int k = threadIdx.x; k < px + py; k += blockDim.x) {
    const bool isx = k < px;
    const DevTiler& t = isx ? tx : ty;
    const int kk = isx ? k : k - px;
    int64_t i[AOL_MAX_RANK];
    unravel(t, false, kk, i);
    int32_t o = 0;
    for (int d = 0; d < t.a; ++d) {
      int32_t e = 0;
      for (int m = 0; m < t.p; ++m) e += (int32_t)t.F[d][m] * (int32_t)i[m];
      (isx ? rx : ry)[kk * t.a + d] = e;
      o += e * (int32_t)t.st[d];
    }
    (isx ? ox : oy)[kk] = o;
  }
  __syncthreads();
  int32_t stx[AOL_MAX_RANK], sty[AOL_MAX_RANK];   // base step between a lane's repetitions
#pragma unroll
  for (int d = 0; d < AOL_MAX_RANK; ++d) {
    stx[d] = d < tx.a ? 32 * (int32_t)tx.P[d][Q - 1] : 0;
    sty[d] = d < ty.a ? 32 * (int32_t)ty.P[d][Q - 1] : 0;
  }
  const int32_t nl = (int32_t)tx.rep[Q - 1];
  const int lane = threadIdx.x & 31;
  const int32_t stride = gridDim.x * 256 * R;
  for (int32_t c = blockIdx.x * 256 * R + (threadIdx.x >> 5) * 32 * R + lane; c < count; c += stride) {
    int32_t r[Q];
    {
      uint32_t v = (uint32_t)(first + c);
#pragma unroll
      for (int j = Q - 1; j >= 1; --j) {
        uint32_t qv, rv;
        tx.rep_div[j].divmod(v, qv, rv);
        r[j] = (int32_t)rv;
        v = qv;
      }
      r[0] = (int32_t)v;
    }
    int32_t bx[AOL_MAX_RANK], by[AOL_MAX_RANK], cx[AOL_MAX_RANK], cy[AOL_MAX_RANK];
    base32<Q>(tx, r, bx);
    base32<Q>(ty, r, by);
    reduce32(tx, bx, cx);
    reduce32(ty, by, cy);
    const bool run = r[Q - 1] + 32 * (R - 1) < nl && c + 32 * (R - 1) < count;
    if (run && window_free32(tx, sx, cx, stx, R - 1) && window_free32(ty, sy, cy, sty, R - 1)) {
      const int32_t xo = flat32(tx, cx), yo = flat32(ty, cy);
      const int32_t dx = flat32(tx, stx), dy = flat32(ty, sty);
      T acc[R][MAXO];
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int j = 0; j < MAXO; ++j) acc[k][j] = T(0);
      bool vec = false;
      if constexpr (XV) {
        if ((xo & 3) == 0 && xo + (R - 1) * dx + 16 <= nx) {
          vec = true;
          float wr[MAXO][16];
#pragma unroll
          for (int j = 0; j < MAXO; ++j)
#pragma unroll
            for (int i = 0; i < 16; ++i) wr[j][i] = (j < py && i < px) ? ws[j * px + i] : 0.f;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            float xv[16];
            const float4* xp = reinterpret_cast<const float4*>(x + xo + k * dx);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 v = __ldg(xp + q);
              xv[4 * q] = v.x; xv[4 * q + 1] = v.y; xv[4 * q + 2] = v.z; xv[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < px) {
#pragma unroll
                for (int j = 0; j < MAXO; ++j)
                  if (j < py) acc[k][j] = mul_add_rn(acc[k][j], wr[j][i], xv[i]);
              }
          }
        }
      }
#pragma unroll 4
      for (int i = 0; i < (vec ? 0 : px); ++i) {
        T xv[R];
        const int32_t oi = xo + ox[i];
#pragma unroll
        for (int k = 0; k < R; ++k) xv[k] = __ldg(x + oi + k * dx);
#pragma unroll
        for (int j = 0; j < MAXO; ++j)
          if (j < py) {
            const T wv = ws[j * px + i];
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k][j] = mul_add_rn(acc[k][j], wv, xv[k]);
          }
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
#pragma unroll
        for (int j = 0; j < MAXO; ++j)
          if (j < py) y[yo + k * dy + oy[j]] = acc[k][j];
      continue;
    }
    // one repetition at a time (window wraps, or the lane's run leaves the repetition row)
    for (int k = 0; k < R; ++k) {
      const int32_t e = c + 32 * k;
      if (e >= count) break;
      if (k > 0) {
        uint32_t v = (uint32_t)(first + e);
#pragma unroll
        for (int j = Q - 1; j >= 1; --j) {
          uint32_t qv, rv;
          tx.rep_div[j].divmod(v, qv, rv);
          r[j] = (int32_t)rv;
          v = qv;
        }
        r[0] = (int32_t)v;
        base32<Q>(tx, r, bx);
        base32<Q>(ty, r, by);
        reduce32(tx, bx, cx);
        reduce32(ty, by, cy);
      }
      const bool xf = window_free32(tx, sx, cx, stx, 0), yf = window_free32(ty, sy, cy, sty, 0);
      const int32_t xo = flat32(tx, cx), yo = flat32(ty, cy);
      T acc[MAXO];
#pragma unroll
      for (int j = 0; j < MAXO; ++j) acc[j] = T(0);
      for (int i = 0; i < px; ++i) {
        const T xv = __ldg(x + (xf ? xo + ox[i] : wrapped32(tx, bx, rx, i)));
#pragma unroll
        for (int j = 0; j < MAXO; ++j)
          if (j < py) acc[j] = mul_add_rn(acc[j], ws[j * px + i], xv);
      }
#pragma unroll
      for (int j = 0; j < MAXO; ++j)
        if (j < py) y[yf ? yo + oy[j] : wrapped32(ty, by, ry, j)] = acc[j];
    }
  }
}

// Pattern reduction: s[off_s(rho)] = sum_i x_pat[i], i ascending.
template <typename T>
__global__ void k_tile_sum_generic(const T* __restrict__ x, T* __restrict__ s, DevTiler tx, DevTiler ts,
                                   int64_t first, int64_t count, int px) {
  extern __shared__ int64_t smem[];
  fill_table(tx, smem, px);
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = first + e;
    int64_t bx[AOL_MAX_RANK];
    tiler_base(tx, rho, bx);
    T acc = T(0);
    for (int i = 0; i < px; ++i) {
      if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, x[table_offset(tx, bx, smem, i)]);
      else acc = __dadd_rn(acc, x[table_offset(tx, bx, smem, i)]);
    }
    s[tiler_offset(ts, rho, 0)] = acc;
  }
}

// Pattern reductions over an affine x tiler (x[cs + As*rho + Bs*i], collapsed to one repetition
// and one pattern stride).  Always i ascending with one rounding per add, like the generic form.
//
// Contiguous patterns (Bs == 1, e.g. row sums): a warp owns 32 repetitions and walks their
// patterns in 32-element chunks.  Lane l copies element i0+l of each of the 32 rows with
// cp.async (every copy instruction covers one row's 128 contiguous bytes: coalesced) into a
// padded 32x33 shared tile; TS_DEPTH chunks are in flight while lane j adds row j's values of
// the oldest chunk in order.  The sum of a row is one dependent chain (i ascending, one
// rounding per add), so the loads are what has to be hidden.
constexpr int TS_DEPTH = 4;
template <typename T> constexpr int ts_warps() { return sizeof(T) == 4 ? 2 : 1; }   // <= 48 KB static smem

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(sizeof(T)) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(32 * ts_warps<T>()) k_tile_sum_rows(const T* __restrict__ x, T* __restrict__ s,
                                                                  int64_t cs, int64_t As, int64_t P, DevTiler ts,
                                                                  int64_t first, int64_t count) {
  constexpr int WARPS = ts_warps<T>();
  __shared__ T tile[WARPS][TS_DEPTH][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * WARPS;
  const int64_t nchunks = (P + 31) / 32;
  for (int64_t wb = blockIdx.x * WARPS + warp; wb * 32 < count; wb += nwarps) {
    const int64_t r0 = first + wb * 32;
    const int nr = (int)(first + count - r0 < 32 ? first + count - r0 : 32);
    auto issue = [&](int64_t c) {
      if (c < nchunks) {
        const int64_t i0 = c * 32;
        const int ni = (int)(P - i0 < 32 ? P - i0 : 32);
        T(*tl)[33] = tile[warp][c % TS_DEPTH];
        if (lane < ni)
          for (int j = 0; j < nr; ++j) cp_async_elem(&tl[j][lane], x + cs + As * (r0 + j) + i0 + lane);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");      // (empty groups keep the count)
    };
    for (int c = 0; c < TS_DEPTH - 1; ++c) issue(c);
    T acc = T(0);
    for (int64_t c = 0; c < nchunks; ++c) {
      issue(c + TS_DEPTH - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(TS_DEPTH - 1) : "memory");
      __syncwarp();
      const int ni = (int)(P - c * 32 < 32 ? P - c * 32 : 32);
      const T(*tl)[33] = tile[warp][c % TS_DEPTH];
      if (lane < nr) {
        for (int k = 0; k < ni; ++k) {
          if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, tl[lane][k]);
          else acc = __dadd_rn(acc, tl[lane][k]);
        }
      }
      __syncwarp();                                               // slot c % TS_DEPTH free again
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (lane < nr) s[tiler_offset(ts, r0 + lane, 0)] = acc;
  }
}

// Any other affine pattern (e.g. column sums, As == 1: consecutive threads read consecutive
// addresses), and, with `table == false`, wrapping tilers too large for the offset table.
template <typename T, bool AFFINE>
__global__ void __launch_bounds__(256) k_tile_sum_direct(const T* __restrict__ x, T* __restrict__ s, int64_t cs,
                                                         int64_t As, int64_t Bs, DevTiler tx, DevTiler ts,
                                                         int64_t first, int64_t count, int64_t P) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = first + e;
    T acc = T(0);
    if (AFFINE) {
      const T* p = x + cs + As * rho;
      int64_t i = 0;
      for (; i + 64 <= P; i += 64) {               // 64 loads in flight, then the 64 adds in order
        T v[64];
#pragma unroll
        for (int u = 0; u < 64; ++u) v[u] = __ldg(p + Bs * (i + u));
#pragma unroll
        for (int u = 0; u < 64; ++u) {
          if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, v[u]);
          else acc = __dadd_rn(acc, v[u]);
        }
      }
      for (; i < P; ++i) {
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, __ldg(p + Bs * i));
        else acc = __dadd_rn(acc, __ldg(p + Bs * i));
      }
    } else {
      for (int64_t i = 0; i < P; ++i) {
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, x[tiler_offset(tx, rho, i)]);
        else acc = __dadd_rn(acc, x[tiler_offset(tx, rho, i)]);
      }
    }
    s[tiler_offset(ts, rho, 0)] = acc;
  }
}

// Column sums (affine tile_sum with As == 1: consecutive repetitions are consecutive columns, the
// pattern walks rows of pitch Bs).  A CTA owns 32 columns; one elected producer thread streams
// {32 columns x RB rows} TMA boxes (8 KB) through a 4-deep shared-memory ring, and the consumer
// warp's lane j adds column j's rows in order (i ascending, one rounding per add, like
// k_tile_sum_direct).  The thread-per-column kernel has only count/32 warps to keep loads in
// flight; here every SM holds ~100 KB of boxes in flight while the add chains run from smem.
constexpr int kColStages = 4;
template <typename T>
__global__ void __launch_bounds__(64) k_tile_sum_cols(const __grid_constant__ CUtensorMap mx, T* __restrict__ s,
                                                      DevTiler ts, int64_t first, int rem, int64_t count,
                                                      int64_t P) {
  constexpr int RB = 8192 / (32 * (int)sizeof(T));   // rows per box
  extern __shared__ __align__(128) unsigned char cring[];
  __shared__ __align__(8) uint64_t full[kColStages], empty[kColStages];
  const T* ring = reinterpret_cast<const T*>(cring);
  const int64_t nbox = (P + RB - 1) / RB;
  const int c0 = blockIdx.x * 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kColStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {                           // producer
    for (int64_t k = 0; k < nbox; ++k) {
      const int st = (int)(k % kColStages);
      if (k >= kColStages) mbar_wait(&empty[st], (uint32_t)((k / kColStages - 1) & 1));
      mbar_expect_tx(&full[st], 8192);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(cring + st * 8192)),
          "l"(&mx), "r"(c0), "r"((int)(k * RB)), "r"(smem_u32(&full[st]))
          : "memory");
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  T acc = T(0);
  for (int64_t k = 0; k < nbox; ++k) {
    const int st = (int)(k % kColStages);
    mbar_wait(&full[st], (uint32_t)((k / kColStages) & 1));
    const T* b = ring + st * (8192 / sizeof(T)) + lane;
    const int64_t rows = P - k * RB;
    if (rows >= RB) {
#pragma unroll 16
      for (int r = 0; r < RB; ++r) {
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, b[r * 32]);
        else acc = __dadd_rn(acc, b[r * 32]);
      }
    } else {
      for (int r = 0; r < (int)rows; ++r) {
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, b[r * 32]);
        else acc = __dadd_rn(acc, b[r * 32]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  const int c = c0 + lane;
  if (c >= rem && c < rem + count) s[tiler_offset(ts, first - rem + c, 0)] = acc;
}

// Row sums over non-overlapping rows (tile_sum.rows with a 16 B row pitch >= P): a CTA owns 32
// repetitions (rows); the producer streams {128 B of each row x 32 rows} TMA boxes with the 128B
// swizzle (16 B chunk c of row r lands at c ^ (r & 7)) through an 8-deep ring, so lane j's 16 B
// reads of row j are conflict-free per quarter warp; lane j adds its row's elements in order.
constexpr int kRowStages = 8;
template <typename T>
__global__ void __launch_bounds__(64) k_tile_sum_rows_tma(const __grid_constant__ CUtensorMap mx, T* __restrict__ s,
                                                          DevTiler ts, int64_t first, int64_t count, int64_t P) {
  constexpr int E = 128 / (int)sizeof(T);            // elements per row per box
  constexpr int EC = 16 / (int)sizeof(T);            // elements per 16 B chunk
  extern __shared__ __align__(1024) unsigned char rring_raw[];
  unsigned char* rring = reinterpret_cast<unsigned char*>(((uintptr_t)rring_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kRowStages], empty[kRowStages];
  const int64_t nbox = (P + E - 1) / E;
  const int r0 = blockIdx.x * 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRowStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    for (int64_t k = 0; k < nbox; ++k) {
      const int st = (int)(k % kRowStages);
      if (k >= kRowStages) mbar_wait(&empty[st], (uint32_t)((k / kRowStages - 1) & 1));
      mbar_expect_tx(&full[st], 4096);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(rring + st * 4096)),
          "l"(&mx), "r"((int)(k * E)), "r"(r0), "r"(smem_u32(&full[st]))
          : "memory");
    }
    return;
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  T acc = T(0);
  for (int64_t k = 0; k < nbox; ++k) {
    const int st = (int)(k % kRowStages);
    mbar_wait(&full[st], (uint32_t)((k / kRowStages) & 1));
    const unsigned char* row = rring + st * 4096 + lane * 128;
    const int64_t left = P - k * E;
    if (left >= E) {
      T v[E];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 q = *reinterpret_cast<const uint4*>(row + ((c ^ (lane & 7)) << 4));
        memcpy(&v[c * EC], &q, 16);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, v[e]);
        else acc = __dadd_rn(acc, v[e]);
      }
    } else {
      for (int e = 0; e < (int)left; ++e) {
        const T v = *reinterpret_cast<const T*>(row + (((e / EC) ^ (lane & 7)) << 4) + (e % EC) * sizeof(T));
        if constexpr (sizeof(T) == 4) acc = __fadd_rn(acc, v);
        else acc = __dadd_rn(acc, v);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (r0 + lane < count) s[tiler_offset(ts, first + r0 + lane, 0)] = acc;
}

// ------------------------------------------------------- launch wrappers ----

int launch_tiler_offsets(const aol_tiler& t, int64_t first, int64_t count, int64_t* out,
                         cudaStream_t stream) {
  DevTiler dt;
  int rc = make_dev_tiler(t, dt);
  if (rc) return rc;
  const int64_t R = tiler_rep_total(t), Pt = tiler_pat_total(t);
  if (first < 0 || count < 0 || first + count > R)
    return fail(AOL_EINVAL, "repetition range outside the repetition space");
  if (count == 0) return AOL_OK;
  k_tiler_offsets<<<grid_for(count * Pt, 256), 256, 0, stream>>>(dt, first, count, Pt, out);
  AOL_LAUNCH_CHECK("k_tiler_offsets");
  return AOL_OK;
}

// Collapse a 1-D view out of the repetition/pattern coefficients when possible.
static bool collapse(const int64_t* coef, const int64_t* dims, int n, int64_t& stride) {
  // coef[j] == coef[j+1] * dims[j+1] for every adjacent pair (ignoring extent-1 dims)
  int64_t s = 0;
  bool have = false;
  int64_t expect_next = 0;
  for (int j = n - 1; j >= 0; --j) {
    if (dims[j] == 1) continue;
    if (!have) {
      s = coef[j];
      have = true;
      expect_next = coef[j] * dims[j];
    } else {
      if (coef[j] != expect_next) return false;
      expect_next = coef[j] * dims[j];
    }
  }
  stride = have ? s : 0;
  return true;
}

// TMA box rows: 16-byte aligned pitches, P*esz a 16-byte multiple of at least 32 bytes
// (16-byte rows measured slower than register vectors), P <= 256 (box limit), destination
// rows disjoint.  Overlapping source rows (paving < pattern: the overlap re-reads hit L2)
// only from 128-byte rows, where the box ring measured 6.1 vs 5.5 TB/s; below that the
// register path wins (tools/micro/gapload.cu, profiles/r1_tma_vs_ldg_gather.json).
static bool tma_rows_ok(int64_t P, int64_t As, int64_t Ad, size_t esz) {
  const int64_t rb = P * (int64_t)esz;
  return P <= 256 && rb >= 32 && rb % 16 == 0 && (As * (int64_t)esz) % 16 == 0 && (Ad * (int64_t)esz) % 16 == 0 &&
         As > 0 && (As >= P || rb >= 128) && Ad >= P;
}

constexpr int64_t kTmaStreamRow = 256;      // bytes per TMA row when a dense copy is streamed as boxes
constexpr int64_t kTmaMinBytes = 1 << 20;   // below this the single-pass register copy wins (launch-bound)

// Merge adjacent row-major dims whose coefficients nest (coef[j] == coef[j+1] * dims[j+1]) and
// drop extent-1 dims; true with <= 2 dims left: (outer extent, outer coef, inner extent, inner coef).
static bool squeeze2(const int64_t* coef, const int64_t* dims, int n, int64_t& d0, int64_t& c0, int64_t& d1,
                     int64_t& c1) {
  int64_t ed[AOL_MAX_RANK], ec[AOL_MAX_RANK];
  int m = 0;
  for (int j = 0; j < n; ++j) {
    if (dims[j] == 1) continue;
    if (m > 0 && ec[m - 1] == coef[j] * dims[j]) {
      ed[m - 1] *= dims[j];
      ec[m - 1] = coef[j];
    } else {
      ed[m] = dims[j];
      ec[m] = coef[j];
      ++m;
    }
  }
  if (m > 2) return false;
  if (m == 0) { d0 = 1; c0 = 0; d1 = 1; c1 = 0; return true; }
  if (m == 1) { d0 = 1; c0 = 0; d1 = ed[0]; c1 = ec[0]; return true; }
  d0 = ed[0]; c0 = ec[0]; d1 = ed[1]; c1 = ec[1];
  return true;
}

struct Affine2 {
  int64_t c, A0, A1, nr1, B0, B1, p1;
};

static bool affine2_of(const aol_tiler& t, Affine2& o) {
  Affine a = tiler_affine(t);
  if (!a.ok) return false;
  int64_t d0, d1, p0;
  if (!squeeze2(a.A, t.rep, t.rep_rank, d0, o.A0, o.nr1, o.A1)) return false;
  if (!squeeze2(a.B, t.pattern, t.pat_rank, p0, o.B0, o.p1, o.B1)) return false;
  (void)d0;
  (void)p0;
  o.c = a.c0;
  return true;
}

// 2-D rep space (pattern total 1) whose inner axis is contiguous on both sides: rows of L elements
// at 16 B-multiple pitches As / Ad (>= L), whole rows in the launch range, >= 1 MB: `tile_copy.tma_plane`
static bool plane_of(const aol_tiler& ts, const aol_tiler& td, int64_t first, int64_t count, size_t esz,
                     int64_t& cs, int64_t& As, int64_t& cd, int64_t& Ad, int64_t& L) {
  Affine2 a, b;
  if (getenv("AOL_COPY_NO_PLANE") || tiler_pat_total(ts) != 1 || !affine2_of(ts, a) || !affine2_of(td, b)) return false;
  L = a.nr1;
  if (L < 32 || b.nr1 != L || a.A1 != 1 || b.A1 != 1 || a.A0 < L || b.A0 < L || (a.A0 * (int64_t)esz) % 16 ||
      (b.A0 * (int64_t)esz) % 16 || first % L || count % L || count * (int64_t)esz < kTmaMinBytes)
    return false;
  cs = a.c;
  As = a.A0;
  cd = b.c;
  Ad = b.A0;
  return true;
}

struct CopyPlan {
  int kind;  // 0 generic, 1 affine1, 2 stream, 3 vector (V elements / thread), 4 transpose
  int64_t cs, As, Bs, cd, Ad, Bd;
  int V;
  bool src_vec;
  bool tma;  // kinds 2/3: TMA box ring first (k_tile_copy_tma), the register path if misaligned
  bool window;  // kind 3: overlapping rows through the bulk-copy window ring (k_tile_copy_window)
};

static CopyPlan plan_tile_copy(const aol_tiler& ts, const aol_tiler& td, int64_t first, int64_t count,
                               size_t esz) {
  CopyPlan p{};
  Affine s = tiler_affine(ts), d = tiler_affine(td);
  if (!s.ok || !d.ok) return p;
  int64_t As, Ad, Bs, Bd;
  // the shared repetition space must collapse identically on both sides
  if (!collapse(s.A, ts.rep, ts.rep_rank, As) || !collapse(d.A, td.rep, td.rep_rank, Ad) ||
      !collapse(s.B, ts.pattern, ts.pat_rank, Bs) || !collapse(d.B, td.pattern, td.pat_rank, Bd)) {
    // two strides per side still affine: block tilers
    Affine2 a2s, a2d;
    if (affine2_of(ts, a2s) && affine2_of(td, a2d)) p.kind = 5;
    return p;
  }
  const int64_t P = tiler_pat_total(ts);
  p.kind = 1;
  p.cs = s.c0; p.As = As; p.Bs = P > 1 ? Bs : 0;
  p.cd = d.c0; p.Ad = Ad; p.Bd = P > 1 ? Bd : 0;
  const bool src_dense = (P == 1 || p.Bs == 1) && p.As == P;
  const bool dst_dense = (P == 1 || p.Bd == 1) && p.Ad == P;
  if (src_dense && dst_dense) {
    p.kind = 2;
    p.tma = count * P * (int64_t)esz >= kTmaMinBytes && (p.cs * (int64_t)esz) % 16 == (p.cd * (int64_t)esz) % 16;
    return p;
  }
  // row-stride gather into a dense stream: transpose through shared memory
  if (p.As == 1 && P > 1 && (p.Bs >= 32 || p.Bs <= -32) && p.Ad == P && p.Bd == 1) {
    p.kind = 4;
    // TMA transpose from 32-byte pattern columns up (m = 4 measured slower than registers: 4.8 vs 5.2 TB/s)
    p.tma = esz == 4 && (P == 8 || P == 16 || P == 32 || P == 64) && p.Bs > 0 && p.Bs % 4 == 0 && p.cd % 4 == 0 &&
            count >= 128 && count * P * (int64_t)esz >= kTmaMinBytes;
    return p;
  }
  // vector path: destination contiguous within the pattern, V | P, V-aligned offsets
  // prefer the widest V that also vectorises the source; else the widest store-only V
  for (int pass = 0; pass < 2 && p.kind != 3; ++pass) {
    for (int V = 4; V >= 2; V /= 2) {
      if (P % V || (P > 1 && p.Bd != 1) || p.cd % V || p.Ad % V) continue;
      const bool sv = (P == 1 || p.Bs == 1) && p.cs % V == 0 && p.As % V == 0;
      if (pass == 0 && !sv) continue;
      p.V = V;
      p.src_vec = sv;
      p.kind = 3;
      break;
    }
  }
  // overlapping contiguous source rows into dense rows: one bulk window per tile (measured 6.0-6.1
  // TB/s for 8-64 B rows vs 5.1-5.6 through registers; >= 128 B rows go to TMA boxes, 6.1)
  if (p.kind == 3 && esz == 4 && P > 1 && P <= 16 && (P & (P - 1)) == 0 && p.Bs == 1 && p.Bd == 1 && p.As > 0 &&
      p.As < P && p.Ad == P && count * P * (int64_t)esz >= kTmaMinBytes) {
    p.window = true;
    return p;
  }
  // contiguous pattern rows on both sides at 16-byte pitches: TMA boxes
  if (p.kind == 3 && P > 1 && p.Bs == 1 && p.Bd == 1 && (p.cs * (int64_t)esz) % 16 == 0 &&
      (p.cd * (int64_t)esz) % 16 == 0 && tma_rows_ok(P, p.As, p.Ad, esz) && count * P * (int64_t)esz >= kTmaMinBytes)
    p.tma = true;
  (void)first;
  return p;
}

static bool seam_boxes(const aol_tiler& ts, const aol_tiler& td, int64_t cuts[AOL_MAX_RANK][3], int ncut[AOL_MAX_RANK]);

// kind 4 with m in {2, 4} fp32, 16 B-aligned pattern rows and destination: k_tile_copy_interleave
static bool interleave_ok(const CopyPlan& p, int64_t P, size_t esz, int64_t count) {
  return !p.tma && esz == 4 && (P == 2 || P == 4) && p.Bs > 0 && p.Bs % 4 == 0 && p.cs % 4 == 0 && p.cd % 4 == 0 &&
         count >= 64 && !getenv("AOL_COPY_SMEM_TRANSPOSE");
}

const char* tile_copy_plan_name(const aol_tiler& ts, const aol_tiler& td, int64_t first, int64_t count,
                                size_t esz, void* const* ports) {
  const CopyPlan pl = plan_tile_copy(ts, td, first, count, esz);
  const bool aligned = !ports || ((uintptr_t)ports[0] % 16 == 0 && (uintptr_t)ports[1] % 16 == 0);
  switch (pl.kind) {
    case 4:
      if (interleave_ok(pl, tiler_pat_total(ts), esz, count) && aligned) return "tile_copy.interleave";
      return pl.tma && aligned ? "tile_copy.tma_transpose" : "tile_copy.transpose";
    case 3:
      if (pl.window && (!ports || (uintptr_t)ports[0] % 16 == 0)) return "tile_copy.window";
      if (pl.tma && aligned) return "tile_copy.tma_box";
      return pl.src_vec ? "tile_copy.vec" : "tile_copy.vec_store";
    case 2: return pl.tma ? "tile_copy.tma_stream" : "tile_copy.stream16";
    case 5: {
      int64_t cs, As, cd, Ad, L;
      if (!plane_of(ts, td, first, count, esz, cs, As, cd, Ad, L)) return "tile_copy.affine2d";
      const int64_t r0 = first / L;
      const bool al = ((cs + As * r0) * (int64_t)esz) % 16 == 0 && ((cd + Ad * r0) * (int64_t)esz) % 16 == 0 &&
                      (!ports || ((uintptr_t)ports[0] % 16 == 0 && (uintptr_t)ports[1] % 16 == 0));
      return al ? "tile_copy.tma_plane" : esz == 4 ? "tile_copy.rows_shift" : "tile_copy.affine2d";
    }
    case 1: return pl.As == 2 && pl.Ad == 1 && tiler_pat_total(ts) == 1 && esz == 4 ? "tile_copy.stride2" : "tile_copy.affine";
    default: {
      int64_t cuts[AOL_MAX_RANK][3];
      int ncut[AOL_MAX_RANK];
      if (first == 0 && count == tiler_rep_total(ts) && seam_boxes(ts, td, cuts, ncut)) return "tile_copy.seam_boxes";
      return "tile_copy.generic";
    }
  }
}

// Rows of P contiguous elements at pitches As (src) / Ad (dst) through k_tile_copy_tma.
// Returns AOL_EUNSUPPORTED (nothing launched) when the alignment is not expressible as
// TMA boxes (tma_rows_ok + 16-byte aligned bases).
static int launch_tma_rows(const void* src, void* dst, int64_t rows, int64_t P, int64_t As, int64_t Ad, size_t esz,
                           cudaStream_t stream) {
  if (!tma_rows_ok(P, As, Ad, esz) || (uintptr_t)src % 16 || (uintptr_t)dst % 16) return AOL_EUNSUPPORTED;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return AOL_EUNSUPPORTED;
  const int64_t rb = P * (int64_t)esz;
  // ring geometry (measured, tools/micro/gapload.cu): ~32 KB in flight per CTA for 32-64 B
  // rows, 4 x 8 KB stages and 2 CTAs per SM for >= 128 B rows
  const int R = (int)std::min<int64_t>(256, std::max<int64_t>(1, (rb <= 32 ? 2048 : rb < 128 ? 4096 : 8192) / rb));
  const int stages = rb <= 32 ? 16 : rb < 128 ? 8 : 4;
  const int cps = rb < 128 ? 1 : 2;
  const uint32_t stage_bytes = (uint32_t)(R * rb);
  const uint32_t stage_pitch = (stage_bytes + 127) & ~127u;   // TMA shared-memory boxes are 128 B aligned
  const CUtensorMapDataType dt = esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const int64_t kMaxRows = (int64_t)1 << 30;            // box coordinates are int32
  for (int64_t r0 = 0; r0 < rows; r0 += kMaxRows) {
    const int64_t n = std::min<int64_t>(kMaxRows, rows - r0);
    CUtensorMap ms, md;
    cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)n};
    cuuint64_t ss[1] = {(cuuint64_t)(As * (int64_t)esz)}, ds[1] = {(cuuint64_t)(Ad * (int64_t)esz)};
    cuuint32_t box[2] = {(cuuint32_t)P, (cuuint32_t)R}, es[2] = {1, 1};
    const char* s0 = static_cast<const char*>(src) + r0 * As * (int64_t)esz;
    char* d0 = static_cast<char*>(dst) + r0 * Ad * (int64_t)esz;
    if (encode(&ms, dt, 2, const_cast<char*>(s0), dims, ss, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        encode(&md, dt, 2, d0, dims, ds, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (r0 == 0) return AOL_EUNSUPPORTED;
      return fail(AOL_ECUDA, "cuTensorMapEncodeTiled failed for a tile_copy chunk");
    }
    const int64_t ntiles = (n + R - 1) / R;
    const int smem = stages * (int)stage_pitch;
    int sms = kNumSMs, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * cps);
    void (*k)(const CUtensorMap, const CUtensorMap, int64_t, int, uint32_t, uint32_t, int64_t, int, int, int) =
        stages == 16 ? k_tile_copy_tma<16> : stages == 8 ? k_tile_copy_tma<8> : k_tile_copy_tma<4>;
    // every ring above is <= 34 KB: within the default 48 KB dynamic shared memory limit
    k<<<grid, 32, smem, stream>>>(ms, md, ntiles, R, stage_bytes, stage_pitch, 1, 0, 0, 0);
    AOL_LAUNCH_CHECK("k_tile_copy_tma");
  }
  return AOL_OK;
}

// Rows of L contiguous floats at any element offsets (2-D shifts' seam boxes, crops): TMA tiles
// cannot start off 16 B, so each thread writes one 16 B-aligned float4 of a destination row and
// builds it from the two aligned source float4s that straddle it (the neighbour lane loads the
// same lines: L1 absorbs the second read).  Row heads/tails narrower than a float4 and loads that
// would leave the source array go scalar.
template <int U>
__global__ void __launch_bounds__(256) k_copy_rows_shift(const float* __restrict__ src, float* __restrict__ dst,
                                                          int64_t rows, int64_t L, int64_t As, int64_t Ad,
                                                          int64_t vblocks, const float* __restrict__ src_end) {
  // block b -> (row, chunk of 256*U float4s): thread t writes the row's aligned float4s
  // chunk*256U + t + 256u (u < U, loads first); the thread one past the last float4 writes the
  // scalar head and tail
  for (int64_t b = blockIdx.x; b < rows * vblocks; b += gridDim.x) {
    const int64_t r = b / vblocks;
    const int64_t q0 = (b - r * vblocks) * (256 * U) + threadIdx.x;
    float* drow = dst + r * Ad;
    const float* srow = src + r * As;
    const int64_t h = (int64_t)((4 - (((uintptr_t)drow >> 2) & 3)) & 3);
    const int64_t head = h < L ? h : L;
    const int64_t nvec = (L - head) >> 2;
    float4 o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + 256 * u;
      if (q >= nvec) continue;
      const float* sp = srow + head + 4 * q;
      const int sh = (int)(((uintptr_t)sp >> 2) & 3);
      const float4* a = reinterpret_cast<const float4*>(sp - sh);
      if (sh == 0) {
        o[u] = __ldg(a);
      } else if (reinterpret_cast<const float*>(a + 2) <= src_end) {
        const float4 x0 = __ldg(a), x1 = __ldg(a + 1);
        o[u] = sh == 1 ? make_float4(x0.y, x0.z, x0.w, x1.x) : sh == 2 ? make_float4(x0.z, x0.w, x1.x, x1.y)
                                                                       : make_float4(x0.w, x1.x, x1.y, x1.z);
      } else {
        o[u] = make_float4(__ldg(sp), __ldg(sp + 1), __ldg(sp + 2), __ldg(sp + 3));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + 256 * u;
      if (q < nvec) {
        *reinterpret_cast<float4*>(drow + head + 4 * q) = o[u];
      } else if (q == nvec) {
        for (int64_t j = 0; j < head; ++j) drow[j] = __ldg(srow + j);
        for (int64_t j = head + 4 * nvec; j < L; ++j) drow[j] = __ldg(srow + j);
      }
    }
  }
}

// one float4 per thread: 2 or 4 per thread (loads first) measured 5.3 / 4.8 TB/s vs 6.0
static void launch_rows_shift(const float* s0, float* d0, int64_t rows, int64_t L, int64_t As, int64_t Ad,
                              const float* src_end, cudaStream_t stream) {
  const int64_t vblocks = (L / 4 + 1 + 255) / 256;   // float4s + the head/tail thread, per row
  const unsigned grid = (unsigned)std::min<int64_t>(rows * vblocks, (int64_t)kNumSMs * 64);
  k_copy_rows_shift<1><<<grid, 256, 0, stream>>>(s0, d0, rows, L, As, Ad, vblocks, src_end);
}

// Two / four pattern rows interleaved into a dense stream (pattern down a column with m = P in
// {2, 4}: src (rho, i) at rho + Bs*i, dst at P*rho + i): a thread writes output float4 g (reps
// (4/P)g ..), loading 4/P consecutive elements of each pattern row, so every load and store
// instruction of a warp is one contiguous run.  m = 2 / 4 at T >= 1e8: 5.95-6.44 TB/s; the
// shared-memory tile transpose gave 5.1-5.4 and a float4-per-row load form 5.3-5.6.
template <int P>
__global__ void __launch_bounds__(256) k_tile_copy_interleave_st(const float* __restrict__ src,
                                                                 float* __restrict__ dst, int64_t Bs, int64_t nq) {
  constexpr int RPG = 4 / P;                          // repetitions per output float4
  const int64_t ng = nq * P;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    float e[4];
    if constexpr (P == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = __ldcs(src + Bs * i + g);
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float2 t = __ldcs(reinterpret_cast<const float2*>(src + Bs * i) + g);
        e[i] = t.x;          // rep 2g, pattern i   -> flat 2*0 + i
        e[2 + i] = t.y;      // rep 2g+1, pattern i -> flat 2*1 + i
      }
    }
    __stcs(reinterpret_cast<float4*>(dst) + g, make_float4(e[0], e[1], e[2], e[3]));
  }
}

// Plane copy: `rows` rows of L contiguous elements starting at src / dst (any element alignment),
// row pitches As / Ad (16 B multiples, >= L), through k_tile_copy_tma with {64 | 32 elements x 32 rows}
// boxes (256 B x 32 = 8 KB), 4 stages, 2 CTAs per SM.
static int launch_tma_plane(const void* src, void* dst, int64_t rows, int64_t L, int64_t As, int64_t Ad, size_t esz,
                            cudaStream_t stream) {
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return AOL_EUNSUPPORTED;
  const int bw = (int)(256 / esz), R = 32;
  const int cs0 = (int)(((uintptr_t)src % 16) / esz), cd0 = (int)(((uintptr_t)dst % 16) / esz);
  if ((uintptr_t)src % esz || (uintptr_t)dst % esz) return AOL_EUNSUPPORTED;
  const char* sb = static_cast<const char*>(src) - cs0 * esz;
  char* db = static_cast<char*>(dst) - cd0 * esz;
  const uint32_t stage_bytes = 8192;
  const CUtensorMapDataType dt = esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const int64_t ncb = (L + bw - 1) / bw;
  const int64_t kMaxRows = (int64_t)1 << 24;   // tile indices and box coordinates stay in int32
  for (int64_t r0 = 0; r0 < rows; r0 += kMaxRows) {
    const int64_t n = std::min<int64_t>(kMaxRows, rows - r0);
    CUtensorMap ms, md;
    cuuint64_t sdims[2] = {(cuuint64_t)(cs0 + L), (cuuint64_t)n}, ddims[2] = {(cuuint64_t)(cd0 + L), (cuuint64_t)n};
    cuuint64_t ss[1] = {(cuuint64_t)(As * (int64_t)esz)}, ds[1] = {(cuuint64_t)(Ad * (int64_t)esz)};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)R}, es[2] = {1, 1};
    if (encode(&ms, dt, 2, const_cast<char*>(sb + r0 * As * (int64_t)esz), sdims, ss, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        encode(&md, dt, 2, db + r0 * Ad * (int64_t)esz, ddims, ds, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
      if (r0 == 0) return AOL_EUNSUPPORTED;
      return fail(AOL_ECUDA, "cuTensorMapEncodeTiled failed for a tile_copy plane chunk");
    }
    const int64_t ntiles = ((n + R - 1) / R) * ncb;
    int sms = kNumSMs, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * 2);
    k_tile_copy_tma<4><<<grid, 32, 4 * stage_bytes, stream>>>(ms, md, ntiles, R, stage_bytes, stage_bytes, ncb, bw,
                                                              cs0, cd0);
    AOL_LAUNCH_CHECK("k_tile_copy_tma(plane)");
  }
  return AOL_OK;
}

// Overlapping source rows into dense rows through k_tile_copy_window (fp32, P a power of two
// up to 64 (the plan uses it for P <= 16), 0 < As < P, Bs == 1, Ad == P).  AOL_EUNSUPPORTED (nothing launched) otherwise.
static int launch_window(const float* src, float* dst, int64_t cs, int64_t As, int64_t cd, int64_t first,
                         int64_t count, int64_t P, cudaStream_t stream) {
  int logp = -1;
  for (int l = 0; l <= 6; ++l)
    if ((int64_t)1 << l == P) logp = l;
  if (logp < 0 || As <= 0 || As >= P || (uintptr_t)src % 16) return AOL_EUNSUPPORTED;
  // ring geometry (measured, m = 2/4 overlap at T = 1e8/1e9): 32 KB windows, double-buffered,
  // 8 CTAs per SM in the grid (about 3 resident): 6.0-6.1 TB/s; 8 KB x 4 stages gave 5.4-5.7
  static const int win_kb = env_int("AOL_WIN_KB", 32), nst = env_int("AOL_WIN_NST", 2),
                   cps = env_int("AOL_WIN_CPS", 8);
  const int R = (int)std::max<int64_t>(32, std::min<int64_t>(16384, win_kb * 256 / As));
  const uint32_t win_pitch = (uint32_t)(((As * (R - 1) + P + 8) + 31) & ~int64_t(31));
  const int smem = nst * (int)win_pitch * 4;
  if (smem > 200 * 1024) return AOL_EUNSUPPORTED;
  const int64_t ntiles = (count + R - 1) / R;
  int sms = kNumSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * cps);
  void (*k)(const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t, int, uint32_t, int);
  switch (logp) {
    case 0: k = k_tile_copy_window<0>; break;
    case 1: k = k_tile_copy_window<1>; break;
    case 2: k = k_tile_copy_window<2>; break;
    case 3: k = k_tile_copy_window<3>; break;
    case 4: k = k_tile_copy_window<4>; break;
    case 5: k = k_tile_copy_window<5>; break;
    default: k = k_tile_copy_window<6>; break;
  }
  if (smem > 48 * 1024) AOL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // (the attribute call is per launch: launches reach here only for >= 1 MB copies)
  k<<<grid, 256, smem, stream>>>(src, dst, cs, As, cd, first, count, R, win_pitch, nst);
  AOL_LAUNCH_CHECK("k_tile_copy_window");
  return AOL_OK;
}

// Row-stride gather (src rows of pitch Bs, reps contiguous) into the dense [count][P] stream
// with k_tile_copy_tma_transpose.  AOL_EUNSUPPORTED (nothing launched) outside its domain.
static int launch_tma_transpose(const float* src, float* dst, int64_t count, int64_t P, int64_t Bs,
                                cudaStream_t stream) {
  if (!(P == 8 || P == 16 || P == 32 || P == 64) || Bs <= 0 || (Bs * 4) % 16 || (uintptr_t)src % 16 ||
      (uintptr_t)dst % 16 || count < 128 || count >= ((int64_t)1 << 31))
    return AOL_EUNSUPPORTED;
  const int RT = P >= 64 ? 64 : 128;
  const bool swo = P >= 32;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return AOL_EUNSUPPORTED;
  CUtensorMap ms, md;
  cuuint64_t sdims[2] = {(cuuint64_t)count, (cuuint64_t)P}, sstr[1] = {(cuuint64_t)(Bs * 4)};
  cuuint32_t sbox[2] = {32, (cuuint32_t)P}, es[2] = {1, 1};
  cuuint64_t ddims[2] = {(cuuint64_t)P, (cuuint64_t)count}, dstr[1] = {(cuuint64_t)(P * 4)};
  cuuint32_t dbox[2] = {(cuuint32_t)(swo ? 32 : P), (cuuint32_t)RT};
  if (encode(&ms, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<float*>(src), sdims, sstr, sbox, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      encode(&md, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, dst, ddims, dstr, dbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swo ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return AOL_EUNSUPPORTED;
  const int64_t ntiles = (count + RT - 1) / RT;
  const int box_stride = ((int)(32 * P * 4) + 1023) & ~1023;
  const int smem = 3 * (RT / 32) * box_stride + 2 * RT * (int)P * 4 + 1024;
  int sms = kNumSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * 4);
  void (*k)(const CUtensorMap, const CUtensorMap, int64_t) =
      P == 8 ? k_tile_copy_tma_transpose<8> : P == 16 ? k_tile_copy_tma_transpose<16>
      : P == 32 ? k_tile_copy_tma_transpose<32> : k_tile_copy_tma_transpose<64>;
  if (smem > 48 * 1024) AOL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // (the attribute call is per launch: launches reach here only for >= 1 MB copies)
  k<<<grid, 128, smem, stream>>>(ms, md, ntiles);
  AOL_LAUNCH_CHECK("k_tile_copy_tma_transpose");
  return AOL_OK;
}

// Toroidal copies (shifts, rotations): when every array axis of both tilers is driven by exactly
// one repetition axis with paving 1 and no pattern extent (pattern total 1), the only wraps are
// at r_j = s_d - o_d.  Splitting every repetition axis at those seams gives <= 2^q boxes over
// which both tilers are affine; each box is the same task with its repetition extents and the
// origins advanced to the box corner, and runs on the affine plans.  Whole-range launches only.
static bool seam_boxes(const aol_tiler& ts, const aol_tiler& td, int64_t cuts[AOL_MAX_RANK][3], int ncut[AOL_MAX_RANK]) {
  const int q = ts.rep_rank;
  // 1-D shifts too: two dense boxes on the funnel-shift kernel, 0.365 ms for 2^28 elements (the
  // 32-bit generic kernel: 0.41)
  if (td.rep_rank != q || tiler_pat_total(ts) != 1) return false;
  for (int j = 0; j < q; ++j) {
    cuts[j][0] = 0;
    ncut[j] = 1;
  }
  for (const aol_tiler* t : {&ts, &td}) {
    for (int d = 0; d < t->arr_rank; ++d) {
      int jd = -1;
      for (int j = 0; j < q; ++j)
        if (t->paving[d][j] != 0) {
          if (jd >= 0 || t->paving[d][j] != 1) return false;
          jd = j;
        }
      for (int k = 0; k < t->pat_rank; ++k)
        if (t->fitting[d][k] != 0 && t->pattern[k] > 1) return false;
      const int64_t sd = t->array[d];
      const int64_t o = ((t->origin[d] % sd) + sd) % sd;
      if (jd < 0) continue;                                  // constant coordinate: never wraps
      if (t->rep[jd] > sd) return false;                     // would wrap more than once
      const int64_t seam = sd - o;
      if (o > 0 && seam < t->rep[jd]) {
        bool have = false;
        for (int c = 0; c < ncut[jd]; ++c) have = have || cuts[jd][c] == seam;
        if (!have) {
          if (ncut[jd] >= 3) return false;
          cuts[jd][ncut[jd]++] = seam;
        }
      }
    }
  }
  for (int j = 0; j < q; ++j)                                // sort the (<= 3) cut points
    for (int a = 1; a < ncut[j]; ++a)
      for (int b = a; b > 0 && cuts[j][b] < cuts[j][b - 1]; --b) std::swap(cuts[j][b], cuts[j][b - 1]);
  int boxes = 1;
  for (int j = 0; j < q; ++j) boxes *= ncut[j];
  return boxes > 1;
}

static aol_tiler box_tiler(const aol_tiler& t, const int64_t lo[AOL_MAX_RANK], const int64_t ext[AOL_MAX_RANK]) {
  aol_tiler b = t;
  for (int d = 0; d < t.arr_rank; ++d) {
    int64_t o = t.origin[d];
    for (int j = 0; j < t.rep_rank; ++j) o += t.paving[d][j] * lo[j];
    b.origin[d] = o;
  }
  for (int j = 0; j < t.rep_rank; ++j) b.rep[j] = ext[j];
  return b;
}

template <typename T>
static int launch_tile_copy_t(const aol_tiler& ts, const aol_tiler& td, int64_t first, int64_t count,
                              const void* src, void* dst, cudaStream_t stream) {
  const int64_t P = tiler_pat_total(ts);
  // the register kernels index (rho, iota) pairs with 32-bit divisions: split huge ranges
  const int64_t max_count = std::max<int64_t>(1, ((int64_t)1 << 31) / std::max<int64_t>(P, 1));
  if (count > max_count) {
    for (int64_t c0 = 0; c0 < count; c0 += max_count) {
      const int rc = launch_tile_copy_t<T>(ts, td, first + c0, std::min(max_count, count - c0), src, dst, stream);
      if (rc) return rc;
    }
    return AOL_OK;
  }
  CopyPlan p = plan_tile_copy(ts, td, first, count, sizeof(T));
  const T* s = static_cast<const T*>(src);
  T* d = static_cast<T*>(dst);
  if (p.kind == 3 && p.window) {
    const int rc = launch_window(reinterpret_cast<const float*>(s), reinterpret_cast<float*>(d), p.cs, p.As, p.cd,
                                 first, count, P, stream);
    if (rc != AOL_EUNSUPPORTED) return rc;
  }
  if (p.kind == 3 && p.tma) {
    const int rc = launch_tma_rows(s + p.cs + p.As * first, d + p.cd + p.Ad * first, count, P, p.As, p.Ad,
                                   sizeof(T), stream);
    if (rc != AOL_EUNSUPPORTED) return rc;
  }
  if (p.kind == 2) {
    const T* s0 = s + p.cs + first * P;
    T* d0 = d + p.cd + first * P;
    const int64_t n = count * P;
    if (((uintptr_t)s0 % 16) == ((uintptr_t)d0 % 16)) {
      // peel to 16-byte alignment, stream the body (TMA box rows, then 16-byte vectors), copy the tail
      int64_t head = ((16 - ((uintptr_t)s0 % 16)) % 16) / sizeof(T);
      if (head > n) head = n;
      if (head) {
        k_stream_copy_tail<T><<<1, 32, 0, stream>>>(s0, d0, head);
        AOL_LAUNCH_CHECK("k_stream_copy_tail");
      }
      int64_t done = head;
      constexpr int64_t row = kTmaStreamRow / (int64_t)sizeof(T);
      if (p.tma && (n - done) / row > 0) {
        const int64_t rows = (n - done) / row;
        const int rc = launch_tma_rows(s0 + done, d0 + done, rows, row, row, row, sizeof(T), stream);
        if (rc == AOL_OK) done += rows * row;
        else if (rc != AOL_EUNSUPPORTED) return rc;
      }
      const int64_t body16 = (n - done) * (int64_t)sizeof(T) / 16;
      if (body16) {
        k_stream_copy16<<<grid_for(body16, 1024, 8), 256, 0, stream>>>(
            reinterpret_cast<const uint4*>(s0 + done), reinterpret_cast<uint4*>(d0 + done), body16);
        AOL_LAUNCH_CHECK("k_stream_copy16");
      }
      done += body16 * 16 / (int64_t)sizeof(T);
      if (n - done) {
        k_stream_copy_tail<T><<<1, 256, 0, stream>>>(s0 + done, d0 + done, n - done);
        AOL_LAUNCH_CHECK("k_stream_copy_tail");
      }
      return AOL_OK;
    }
    if (sizeof(T) == 4 && n >= 4096 && (uintptr_t)s % 16 == 0 && (uintptr_t)d0 % 4 == 0 && (uintptr_t)s0 % 4 == 0) {
      // relatively misaligned dense copy (1-D shifts): one "row" through the funnel-shift kernel
      launch_rows_shift((const float*)s0, (float*)d0, 1, n, 0, 0, (const float*)s + tiler_arr_total(ts), stream);
      AOL_LAUNCH_CHECK("k_copy_rows_shift");
      return AOL_OK;
    }
    p.kind = 1;
  }
  if (p.kind == 4 && p.tma) {
    // peel repetitions up to a 16-byte aligned source column, TMA the rest
    const int64_t head = std::min<int64_t>(count, (4 - (p.cs + first) % 4) % 4);
    const int rc = launch_tma_transpose(reinterpret_cast<const float*>(s) + p.cs + first + head,
                                        reinterpret_cast<float*>(d) + p.cd + (first + head) * P, count - head, P,
                                        p.Bs, stream);
    if (rc == AOL_OK) {
      if (head == 0) return AOL_OK;
      count = head;                                   // the head goes through the register transpose
    } else if (rc != AOL_EUNSUPPORTED) {
      return rc;
    }
  }
  if (p.kind == 4 && interleave_ok(p, P, sizeof(T), count) && (uintptr_t)s % 16 == 0 && (uintptr_t)d % 16 == 0) {
    const int64_t head = std::min<int64_t>(count, (4 - first % 4) % 4);
    const int64_t nq = (count - head) / 4, tail = count - head - 4 * nq;
    const float* s0 = reinterpret_cast<const float*>(s) + p.cs + first + head;
    float* d0 = reinterpret_cast<float*>(d) + p.cd + (first + head) * P;
    if (nq > 0) {
      if (P == 2) k_tile_copy_interleave_st<2><<<grid_for(nq * 2, 256, 16), 256, 0, stream>>>(s0, d0, p.Bs, nq);
      else k_tile_copy_interleave_st<4><<<grid_for(nq * 4, 256, 16), 256, 0, stream>>>(s0, d0, p.Bs, nq);
      AOL_LAUNCH_CHECK("k_tile_copy_interleave");
    }
    int rc = AOL_OK;
    if (head > 0 && (rc = launch_tile_copy_t<T>(ts, td, first, head, src, dst, stream))) return rc;
    if (tail > 0) return launch_tile_copy_t<T>(ts, td, first + count - tail, tail, src, dst, stream);
    return AOL_OK;
  }
  if (p.kind == 4) {
    const int pc = (int)std::min<int64_t>(P, 64);
    int pc2 = 1;
    while (pc2 < pc) pc2 <<= 1;
    int rshift = 0;
    while ((1 << (rshift + 1)) * pc2 <= 4096) ++rshift;      // tile: 2^rshift x pc <= 4096 elements
    const int64_t tiles = ((count + (1 << rshift) - 1) >> rshift) * ((P + pc - 1) / pc);
    const int pitch = (1 << rshift) + (pc2 >= 32 ? 1 : 32 / pc2);
    // 16-byte accesses on both sides when every tile row / stream chunk is aligned
    const bool vec = sizeof(T) == 4 && pc == P && (1 << rshift) >= 4 && p.cs % 4 == 0 && p.Bs % 4 == 0 &&
                     first % 4 == 0 && p.cd % 4 == 0 && ((uintptr_t)s % 16) == 0 && ((uintptr_t)d % 16) == 0;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)kNumSMs * 16);
    if (vec)
      k_tile_copy_transpose<T, true><<<grid, 256, 0, stream>>>(s, d, p.cs, p.Bs, p.cd, P, first, count, pc, rshift,
                                                               FastDiv32((uint32_t)pc), pitch);
    else
      k_tile_copy_transpose<T, false><<<grid, 256, 0, stream>>>(s, d, p.cs, p.Bs, p.cd, P, first, count, pc, rshift,
                                                                FastDiv32((uint32_t)pc), pitch);
    AOL_LAUNCH_CHECK("k_tile_copy_transpose");
    return AOL_OK;
  }
  if (p.kind == 3) {
    int V = p.V;
    if (sizeof(T) == 8 && V > 2) V = 2;                 // 16-byte vectors
    const uintptr_t sa = (uintptr_t)s, da = (uintptr_t)d;
    const size_t vb = (size_t)V * sizeof(T);
    if (da % vb == 0 && (!p.src_vec || sa % vb == 0)) {
      const int64_t groups = count * P / V;
      const unsigned grid = grid_for(groups, 1024, 16);
      const FastDiv32 pd((uint32_t)P);
#define AOL_VEC_LAUNCH(VV, SV)                                                                               \
  k_tile_copy_vec<T, VV, SV><<<grid, 256, 0, stream>>>(s, d, p.cs, p.As, p.Bs, p.cd, p.Ad, first, groups, pd)
      if (V == 4) { if (p.src_vec) AOL_VEC_LAUNCH(4, true); else AOL_VEC_LAUNCH(4, false); }
      else { if (p.src_vec) AOL_VEC_LAUNCH(2, true); else AOL_VEC_LAUNCH(2, false); }
#undef AOL_VEC_LAUNCH
      AOL_LAUNCH_CHECK("k_tile_copy_vec");
      return AOL_OK;
    }
    p.kind = 1;
  }
  if (p.kind == 5) {
    int64_t pcs, pAs, pcd, pAd, L;
    if (plane_of(ts, td, first, count, sizeof(T), pcs, pAs, pcd, pAd, L)) {
      const int64_t r0 = first / L, rows = count / L;
      const T* s0 = s + pcs + pAs * r0;
      T* d0 = d + pcd + pAd * r0;
      if ((uintptr_t)s0 % 16 == 0 && (uintptr_t)d0 % 16 == 0) {
        const int rc = launch_tma_plane(s0, d0, rows, L, pAs, pAd, sizeof(T), stream);
        if (rc != AOL_EUNSUPPORTED) return rc;
      } else if (sizeof(T) == 4 && (uintptr_t)d0 % 4 == 0 && (uintptr_t)s0 % 4 == 0 && (uintptr_t)s % 16 == 0) {
        launch_rows_shift((const float*)s0, (float*)d0, rows, L, pAs, pAd, (const float*)s + tiler_arr_total(ts),
                          stream);
        AOL_LAUNCH_CHECK("k_copy_rows_shift");
        return AOL_OK;
      }
    }
    Affine2 a, b;
    affine2_of(ts, a);
    affine2_of(td, b);
    const int64_t nr1s = std::max<int64_t>(1, a.nr1), nr1d = std::max<int64_t>(1, b.nr1);
    const int64_t p1s = std::max<int64_t>(1, a.p1), p1d = std::max<int64_t>(1, b.p1);
    if (first + count < ((int64_t)1 << 32) && P < ((int64_t)1 << 31)) {
      Side2 ss{a.c, a.A0, a.A1, a.B0, a.B1, FastDiv32((uint32_t)nr1s), FastDiv32((uint32_t)p1s)};
      Side2 sd{b.c, b.A0, b.A1, b.B0, b.B1, FastDiv32((uint32_t)nr1d), FastDiv32((uint32_t)p1d)};
      // widest vector V: V | both inner pattern extents, unit inner strides, every offset V-aligned
      int V = 1;
      for (int v = 4; v >= 2 && sizeof(T) == 4; v /= 2) {
        auto ok = [&](const Affine2& q, int64_t p1) {
          return p1 % v == 0 && (q.B1 == 1 || p1 == 1) && q.c % v == 0 && q.A0 % v == 0 && q.A1 % v == 0 &&
                 q.B0 % v == 0;
        };
        if (P % v == 0 && ok(a, p1s) && ok(b, p1d) && (uintptr_t)s % (v * sizeof(T)) == 0 &&
            (uintptr_t)d % (v * sizeof(T)) == 0) {
          V = v;
          break;
        }
      }
      const int64_t groups = count * P / V;
      const unsigned grid = grid_for(groups, 1024, 16);
      const FastDiv32 pd((uint32_t)P);
      if (V == 4)
        k_tile_copy_affine2d<T, 4><<<grid, 256, 0, stream>>>(s, d, ss, sd, first, groups, pd);
      else if (V == 2)
        k_tile_copy_affine2d<T, 2><<<grid, 256, 0, stream>>>(s, d, ss, sd, first, groups, pd);
      else
        k_tile_copy_affine2d<T, 1><<<grid, 256, 0, stream>>>(s, d, ss, sd, first, groups, pd);
      AOL_LAUNCH_CHECK("k_tile_copy_affine2d");
      return AOL_OK;
    }
    p.kind = 0;                                          // 32-bit index space exceeded: generic
  }
  if (p.kind == 1 && sizeof(T) == 4 && P == 1 && p.As == 2 && p.Ad == 1) {
    // stride-2 gather: whole groups of 4 repetitions from 16-byte aligned source/destination
    const float* s0 = reinterpret_cast<const float*>(s) + p.cs + 2 * first;
    float* d0 = reinterpret_cast<float*>(d) + p.cd + first;
    // every group reads 8 source elements: stay inside the source array
    const int64_t room = (tiler_arr_total(ts) - (p.cs + 2 * first)) / 8;
    const int64_t groups = std::min<int64_t>(count / 4, std::max<int64_t>(room, 0));
    if (groups > 0 && (uintptr_t)s0 % 16 == 0 && (uintptr_t)d0 % 16 == 0) {
      static const int s2u = env_int("AOL_S2_U", 1), s2w = env_int("AOL_S2_WAVES", 16);
      const unsigned g2 = grid_for(groups, 256 * s2u, s2w);
      if (s2u >= 4) k_gather_stride2<4><<<g2, 256, 0, stream>>>(s0, d0, groups);
      else if (s2u == 2) k_gather_stride2<2><<<g2, 256, 0, stream>>>(s0, d0, groups);
      else k_gather_stride2<1><<<grid_for(groups, 1024, s2w), 256, 0, stream>>>(s0, d0, groups);
      AOL_LAUNCH_CHECK("k_gather_stride2");
      first += 4 * groups;                              // the < 4 trailing repetitions below
      count -= 4 * groups;
      if (count == 0) return AOL_OK;
    }
  }
  if (p.kind == 1) {
    const int64_t n = count * P;
    k_tile_copy_affine<T, 4><<<grid_for(n, 1024, 16), 256, 0, stream>>>(
        s, d, p.cs, p.As, p.Bs, p.cd, p.Ad, p.Bd, first, n, FastDiv32((uint32_t)P));
    AOL_LAUNCH_CHECK("k_tile_copy_affine");
    return AOL_OK;
  }
  // toroidal shifts over the whole repetition space: affine boxes between the seams
  int64_t cuts[AOL_MAX_RANK][3];
  int ncut[AOL_MAX_RANK];
  if (p.kind == 0 && first == 0 && count == tiler_rep_total(ts) && seam_boxes(ts, td, cuts, ncut)) {
    const int q = ts.rep_rank;
    int idx[AOL_MAX_RANK] = {0, 0, 0, 0};
    for (;;) {
      int64_t lo[AOL_MAX_RANK] = {0, 0, 0, 0}, ext[AOL_MAX_RANK] = {0, 0, 0, 0};
      int64_t n = 1;
      for (int j = 0; j < q; ++j) {
        lo[j] = cuts[j][idx[j]];
        const int64_t hi = idx[j] + 1 < ncut[j] ? cuts[j][idx[j] + 1] : ts.rep[j];
        ext[j] = hi - lo[j];
        n *= ext[j];
      }
      if (n > 0) {
        const aol_tiler bs = box_tiler(ts, lo, ext), bd = box_tiler(td, lo, ext);
        const int rc = launch_tile_copy_t<T>(bs, bd, 0, n, src, dst, stream);
        if (rc) return rc;
      }
      int j = q - 1;
      while (j >= 0 && ++idx[j] == ncut[j]) idx[j--] = 0;
      if (j < 0) break;
    }
    return AOL_OK;
  }
  DevTiler dts, dtd;
  int rc = make_dev_tiler(ts, dts);
  if (rc) return rc;
  rc = make_dev_tiler(td, dtd);
  if (rc) return rc;
  const bool small = count * P < ((int64_t)1 << 32) && P < ((int64_t)1 << 32);
  // 32-bit kernels for the common ranks (array <= 3, repetition <= 3, pattern <= 2)
  if (dts.fits32 && dtd.fits32 && first + count < ((int64_t)1 << 31) && count * P < ((int64_t)1 << 31) &&
      dts.a <= 3 && dts.q <= 3 && dts.p <= 2 && dtd.a <= 3 && dtd.q <= 3 && dtd.p <= 2 && dts.q == dtd.q) {
    const uint32_t n = (uint32_t)(count * P);
    const unsigned grid = grid_for((n + 3) / 4, 256);
    const FastDiv32 pd((uint32_t)P);
    void (*k)(const T*, T*, DevTiler, DevTiler, uint32_t, uint32_t, FastDiv32) = nullptr;
    // src ranks x dst ranks: instantiate the usual shapes (same repetition rank on both sides)
#define AOL_G32(as, ps, ad, pd_, QQ) \
    if (dts.a == as && dts.p == ps && dtd.a == ad && dtd.p == pd_ && dts.q == QQ) k = k_tile_copy_generic32<T, as, QQ, ps, ad, QQ, pd_>;
#define AOL_G32Q(QQ) AOL_G32(1, 1, 1, 1, QQ) AOL_G32(2, 1, 2, 1, QQ) AOL_G32(3, 1, 3, 1, QQ) AOL_G32(2, 1, 1, 1, QQ) \
    AOL_G32(1, 1, 2, 1, QQ) AOL_G32(2, 2, 1, 1, QQ) AOL_G32(1, 1, 2, 2, QQ) AOL_G32(2, 2, 2, 2, QQ) AOL_G32(3, 1, 1, 1, QQ) \
    AOL_G32(1, 1, 3, 1, QQ) AOL_G32(3, 2, 1, 1, QQ) AOL_G32(2, 1, 1, 2, QQ) AOL_G32(1, 2, 1, 1, QQ) AOL_G32(1, 1, 1, 2, QQ)
    AOL_G32Q(1) AOL_G32Q(2) AOL_G32Q(3)
#undef AOL_G32Q
#undef AOL_G32
    if (k) {
      k<<<grid, 256, 0, stream>>>(s, d, dts, dtd, (uint32_t)first, n, pd);
      AOL_LAUNCH_CHECK("k_tile_copy_generic32");
      return AOL_OK;
    }
  }
  k_tile_copy_generic<T><<<grid_for(count * P, 256), 256, 0, stream>>>(
      s, d, dts, dtd, first, count, P, FastDiv32(small ? (uint32_t)P : 1u), small ? 1 : 0);
  AOL_LAUNCH_CHECK("k_tile_copy_generic");
  return AOL_OK;
}

int launch_tile_copy(const aol_task& t, int64_t first, int64_t count, void* const* ports,
                     cudaStream_t stream) {
  if (dtype_size(t.dtype) == 4)
    return launch_tile_copy_t<uint32_t>(t.tilers[0], t.tilers[1], first, count, ports[0], ports[1], stream);
  return launch_tile_copy_t<uint64_t>(t.tilers[0], t.tilers[1], first, count, ports[0], ports[1], stream);
}

int launch_matmul_generic(const aol_task& t, int64_t first, int64_t count, void* const* ports,
                          cudaStream_t stream) {
  DevTiler ta, tb, tc;
  int rc;
  if ((rc = make_dev_tiler(t.tilers[0], ta)) || (rc = make_dev_tiler(t.tilers[1], tb)) ||
      (rc = make_dev_tiler(t.tilers[2], tc)))
    return rc;
  const int64_t K = tiler_pat_total(t.tilers[0]);
  const int use_table = K * (ta.a + tb.a) <= kTableMax ? 1 : 0;
  const size_t smem = use_table ? (size_t)K * (ta.a + tb.a) * sizeof(int64_t) : 0;
  const unsigned grid = grid_for(count, 128, 32);
  if (t.dtype == AOL_F32)
    k_matmul_generic<float><<<grid, 128, smem, stream>>>(
        (const float*)ports[0], (const float*)ports[1], (float*)ports[2], ta, tb, tc, first, count, K, use_table);
  else
    k_matmul_generic<double><<<grid, 128, smem, stream>>>(
        (const double*)ports[0], (const double*)ports[1], (double*)ports[2], ta, tb, tc, first, count, K,
        use_table);
  AOL_LAUNCH_CHECK("k_matmul_generic");
  return AOL_OK;
}

static PatSpan pattern_span(const aol_tiler& t) {
  PatSpan sp;
  memset(&sp, 0, sizeof(sp));
  for (int d = 0; d < t.arr_rank; ++d)
    for (int k = 0; k < t.pat_rank; ++k) {
      const int64_t v = t.fitting[d][k] * (t.pattern[k] - 1);
      sp.lo[d] += std::min<int64_t>(0, v);
      sp.hi[d] += std::max<int64_t>(0, v);
    }
  return sp;
}

// x pattern is a contiguous run: raw offsets foff[i] == i (1-D along the last dim, unit fitting)
static bool contiguous_pattern(const aol_tiler& t) {
  int64_t st[AOL_MAX_RANK], acc = 1;
  for (int d = t.arr_rank - 1; d >= 0; --d) { st[d] = acc; acc *= t.array[d]; }
  int64_t expect = 1;
  for (int k = t.pat_rank - 1; k >= 0; --k) {
    if (t.pattern[k] == 1) continue;
    int64_t c = 0;
    for (int d = 0; d < t.arr_rank; ++d) c += t.fitting[d][k] * st[d];
    if (c != expect) return false;
    expect *= t.pattern[k];
  }
  return true;
}

template <typename T, int MAXO, bool XVEC>
static int launch_filter_t(const aol_task& t, const DevTiler& tx, const DevTiler& ty, int64_t first, int64_t count,
                           int px, int py, void* const* ports, cudaStream_t stream) {
  const size_t smem = ((size_t)px * tx.a + (size_t)py * ty.a + px + py) * sizeof(int64_t) +
                      (size_t)px * py * sizeof(T);
  auto kern = k_filter_generic<T, MAXO, XVEC>;
  if (smem > 48 * 1024)
    AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t nx = tiler_arr_total(t.tilers[0]);
  kern<<<grid_for(count, 256, 16), 256, smem, stream>>>((const T*)ports[0], (const T*)ports[1], (T*)ports[2], tx,
                                                        ty, pattern_span(t.tilers[0]), pattern_span(t.tilers[1]),
                                                        first, count, px, py, nx);
  AOL_LAUNCH_CHECK("k_filter_generic");
  return AOL_OK;
}

// both tilers 32-bit safe over one repetition space, range inside int32
static bool filter_batched_ok(const DevTiler& tx, const DevTiler& ty, int64_t first, int64_t count) {
  const bool off = getenv("AOL_FILTER_WIDE") != nullptr;   // diagnostic: the int64 / line_tiled kernels
  if (off || !tx.fits32 || !ty.fits32 || tx.q != ty.q || first + count >= ((int64_t)1 << 31)) return false;
  for (int j = 0; j < tx.q; ++j)
    if (tx.rep[j] != ty.rep[j]) return false;
  return true;
}

template <typename T, int MAXO, int R, int Q, bool XV>
static int launch_filter_b32(const aol_task& t, const DevTiler& tx, const DevTiler& ty, int64_t first,
                              int64_t count, int px, int py, void* const* ports, cudaStream_t stream) {
  const size_t smem = (size_t)px * py * sizeof(T) + ((size_t)px + py + (size_t)px * tx.a + (size_t)py * ty.a) * 4;
  auto kern = k_filter_batched32<T, MAXO, R, Q, XV>;
  if (smem > 48 * 1024)
    AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t per = 256 * R;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + per - 1) / per, (int64_t)kNumSMs * 8));
  kern<<<grid, 256, smem, stream>>>((const T*)ports[0], (const T*)ports[1], (T*)ports[2], tx, ty,
                                    pattern_span(t.tilers[0]), pattern_span(t.tilers[1]), (int32_t)first,
                                    (int32_t)count, px, py, (int32_t)tiler_arr_total(t.tilers[0]));
  return AOL_OK;
}

template <typename T, int MAXO, int R, bool XV = false>
static int launch_filter_b32_q(const aol_task& t, const DevTiler& tx, const DevTiler& ty, int64_t first,
                               int64_t count, int px, int py, void* const* ports, cudaStream_t stream) {
  int rc;
  switch (tx.q) {
    case 1: rc = launch_filter_b32<T, MAXO, R, 1, XV>(t, tx, ty, first, count, px, py, ports, stream); break;
    case 2: rc = launch_filter_b32<T, MAXO, R, 2, XV>(t, tx, ty, first, count, px, py, ports, stream); break;
    case 3: rc = launch_filter_b32<T, MAXO, R, 3, XV>(t, tx, ty, first, count, px, py, ports, stream); break;
    default: rc = launch_filter_b32<T, MAXO, R, 4, XV>(t, tx, ty, first, count, px, py, ports, stream); break;
  }
  if (rc) return rc;
  AOL_LAUNCH_CHECK("k_filter_batched32");
  return AOL_OK;
}

bool stencil_box_applicable(const aol_task& t, int& KH, int& KW);
int launch_stencil_box(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
bool box_pool_applicable(const aol_task& t, int& KH, int& KW);
int launch_box_pool(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
struct LineGeom;
bool line_filter_geometry(const aol_task& t, LineGeom& g);
const char* line_filter_variant(const LineGeom& g);
int launch_line_filter(const aol_task& t, const LineGeom& g, int64_t first, int64_t count, void* const* ports,
                       cudaStream_t s);
// opaque storage for a LineGeom (defined in aol_linefilter.cu)
struct alignas(16) LineGeomBuf { unsigned char b[256]; };

// Routing: the config-shaped kernels (stencil boxes, block pooling, the 13->3 / 14->4 line forms and
// strided line filters) first; then the 32-bit batched kernel, which beats the shared-memory line
// window (`line_tiled`, 2-4x on 1-D FIRs and decimators, tools/time_filters.py) and every
// thread-per-repetition form; the int64 kernels last.
// line-filter variants the batched kernel replaces when it applies (`tile_filter.line`, paving > 4,
// stays: 0.82 vs 1.02 ms on 64x2048x2048 rows /8, tools/time_filters.py)
// A task whose input the MARTE placement puts in deviceLocal memory (AOL_FLAG_STAGE_SMEM) keeps the
// shared-memory-staged window: the placement decides the staging, not the routing heuristic.
static bool line_yields(const aol_task& t, const char* variant) {
  return strcmp(variant, "tile_filter.line_tiled") == 0 && !(t.flags & AOL_FLAG_STAGE_SMEM);
}

static bool filter_batched_route(const aol_task& t, int64_t first, int64_t count, DevTiler& tx, DevTiler& ty) {
  if (make_dev_tiler(t.tilers[0], tx) || make_dev_tiler(t.tilers[1], ty)) return false;
  const int64_t px = tiler_pat_total(t.tilers[0]), py = tiler_pat_total(t.tilers[1]);
  const int64_t esz = t.dtype == AOL_F32 ? 4 : 8;
  const int64_t smem = px * py * esz + (px + py + px * tx.a + py * ty.a) * 4;
  return py <= 16 && smem <= 200 * 1024 && filter_batched_ok(tx, ty, first, count);
}

const char* filter_plan_name(const aol_task& t) {
  int kh, kw;
  if (stencil_box_applicable(t, kh, kw)) return "tile_filter.stencil_box";
  if (box_pool_applicable(t, kh, kw)) return "tile_filter.box_pool";
  LineGeomBuf gb;
  const bool line = line_filter_geometry(t, *reinterpret_cast<LineGeom*>(&gb));
  const char* variant = line ? line_filter_variant(*reinterpret_cast<LineGeom*>(&gb)) : nullptr;
  if (line && !line_yields(t, variant)) return variant;
  DevTiler tx, ty;
  if (filter_batched_route(t, 0, tiler_rep_total(t.tilers[0]), tx, ty)) return "tile_filter.batched";
  if (line) return variant;
  const int64_t px = tiler_pat_total(t.tilers[0]), py = tiler_pat_total(t.tilers[1]);
  if (t.dtype == AOL_F32 && px <= 16 && py <= 4 && contiguous_pattern(t.tilers[0])) return "tile_filter.window_vec";
  return "tile_filter.generic";
}

int launch_filter_generic(const aol_task& t, int64_t first, int64_t count, void* const* ports,
                          cudaStream_t stream) {
  int kh, kw;
  if (stencil_box_applicable(t, kh, kw)) return launch_stencil_box(t, first, count, ports, stream);
  if (box_pool_applicable(t, kh, kw) && (uintptr_t)ports[0] % 16 == 0 && (uintptr_t)ports[2] % 16 == 0)
    return launch_box_pool(t, first, count, ports, stream);
  LineGeomBuf gb;
  const bool line = line_filter_geometry(t, *reinterpret_cast<LineGeom*>(&gb));
  if (line && !line_yields(t, line_filter_variant(*reinterpret_cast<LineGeom*>(&gb))))
    return launch_line_filter(t, *reinterpret_cast<LineGeom*>(&gb), first, count, ports, stream);
  DevTiler tx, ty;
  const bool batched = filter_batched_route(t, first, count, tx, ty);
  if (!batched && line) return launch_line_filter(t, *reinterpret_cast<LineGeom*>(&gb), first, count, ports, stream);
  int rc;
  if ((rc = make_dev_tiler(t.tilers[0], tx)) || (rc = make_dev_tiler(t.tilers[1], ty))) return rc;
  const int64_t px = tiler_pat_total(t.tilers[0]), py = tiler_pat_total(t.tilers[1]);
  const bool f32 = t.dtype == AOL_F32;
  if (batched) {
    // R = 16 when a lane's repetitions are one element apart (dense 1-D runs), else 8 (measured)
    int32_t lane_step = 0;
    for (int d = 0; d < tx.a; ++d) lane_step += (int32_t)tx.P[d][tx.q - 1] * (int32_t)tx.st[d];
    if (f32 && py <= 2 && px <= 16 && lane_step % 4 == 0 && contiguous_pattern(t.tilers[0]))
      return py == 1 ? launch_filter_b32_q<float, 1, 8, true>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
                     : launch_filter_b32_q<float, 2, 8, true>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
    if (py == 1 && lane_step == 1)
      return f32 ? launch_filter_b32_q<float, 1, 16>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
                 : launch_filter_b32_q<double, 1, 16>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
    if (py == 1)
      return f32 ? launch_filter_b32_q<float, 1, 8>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
                 : launch_filter_b32_q<double, 1, 8>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
    if (py <= 4)
      return f32 ? launch_filter_b32_q<float, 4, 8>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
                 : launch_filter_b32_q<double, 4, 4>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
    return f32 ? launch_filter_b32_q<float, 16, 2>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
               : launch_filter_b32_q<double, 16, 2>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
  }
  if (px * tx.a + py * ty.a + px + py > kTableMax * 4 || px * py > 16384)
    return fail(AOL_EUNSUPPORTED, "tile_filter pattern too large (px*py <= 16384)");
  if (py > 16) return fail(AOL_EUNSUPPORTED, "tile_filter supports at most 16 outputs per pattern");
  if (f32 && px <= 16 && py <= 4 && contiguous_pattern(t.tilers[0]))
    return launch_filter_t<float, 4, true>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
  if (py <= 4)
    return f32 ? launch_filter_t<float, 4, false>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
               : launch_filter_t<double, 4, false>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
  return f32 ? launch_filter_t<float, 16, false>(t, tx, ty, first, count, (int)px, (int)py, ports, stream)
             : launch_filter_t<double, 16, false>(t, tx, ty, first, count, (int)px, (int)py, ports, stream);
}

// tile_sum.columns: As == 1, 16 B row pitch, enough columns and rows to stream (else direct)
static bool tile_sum_cols_ok(int64_t As, int64_t Bs, int64_t P, int64_t count, int64_t esz) {
  return As == 1 && (Bs * esz) % 16 == 0 && Bs >= count && P >= 128 && count >= 256 &&
         count < ((int64_t)1 << 31) && P < ((int64_t)1 << 31);
}

// tile_sum plan: "rows" (affine, contiguous pattern), "direct" (other affine), "generic"
// (offset table in shared memory), "generic_direct" (wrapping and too large for the table).
static int tile_sum_kind(const aol_task& t, int64_t& cs, int64_t& As, int64_t& Bs) {
  const aol_tiler& tx = t.tilers[0];
  Affine a = tiler_affine(tx);
  const int64_t P = tiler_pat_total(tx);
  if (a.ok && collapse(a.A, tx.rep, tx.rep_rank, As) && collapse(a.B, tx.pattern, tx.pat_rank, Bs)) {
    cs = a.c0;
    if (P == 1) Bs = 0;
    return P >= 32 && Bs == 1 ? 0 : 1;
  }
  int64_t dummy = 0;
  DevTiler d;
  if (make_dev_tiler(tx, d) == AOL_OK) dummy = P * d.a;
  return dummy <= kTableMax ? 2 : 3;
}

// Wrapping patterns and strided non-column patterns: tile_sum is the one-output filter with unit
// weights (1*x == x bit for bit, so the sums are the same), so the 32-bit batched filter kernel
// serves it (`tile_sum.batched`).
static bool tile_sum_batched_ok(const aol_task& t, int64_t first, int64_t count, int64_t As) {
  DevTiler a, b;
  (void)As;
  return count >= 1024 && filter_batched_route(t, first, count, a, b);
}

const char* tile_sum_plan_name(const aol_task& t) {
  int64_t cs, As, Bs;
  switch (tile_sum_kind(t, cs, As, Bs)) {
    case 0: return "tile_sum.rows";
    case 1:
      if (tile_sum_cols_ok(As, Bs, tiler_pat_total(t.tilers[0]), tiler_rep_total(t.tilers[0]), t.dtype == AOL_F32 ? 4 : 8))
        return "tile_sum.columns";
      return As != 1 && tile_sum_batched_ok(t, 0, tiler_rep_total(t.tilers[0]), As) ? "tile_sum.batched" : "tile_sum.direct";
    case 2: return tile_sum_batched_ok(t, 0, tiler_rep_total(t.tilers[0]), As) ? "tile_sum.batched" : "tile_sum.generic";
    default: return tile_sum_batched_ok(t, 0, tiler_rep_total(t.tilers[0]), As) ? "tile_sum.batched" : "tile_sum.generic_direct";
  }
}

// 1 = this range needs the cp.async rows kernel (overlapping rows or misaligned start)
template <typename T>
static int launch_tile_sum_rows_tma(const T* x, T* sp, const DevTiler& ts, int64_t cs, int64_t As, int64_t P,
                                    int64_t first, int64_t count, cudaStream_t stream) {
  const T* base = x + cs + As * first;
  if (As < P || (As * (int64_t)sizeof(T)) % 16 || (uintptr_t)base % 16 || P < 256 || count < 256 ||
      count >= ((int64_t)1 << 31) || P >= ((int64_t)1 << 31) || getenv("AOL_TILE_SUM_CPASYNC"))
    return 1;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return 1;
  CUtensorMap mx;
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)count}, str[1] = {(cuuint64_t)(As * sizeof(T))};
  cuuint32_t box[2] = {(cuuint32_t)(128 / sizeof(T)), 32}, es[2] = {1, 1};
  if (encode(&mx, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
             const_cast<T*>(base), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 1;
  const int smem = kRowStages * 4096 + 1024;
  const unsigned grid = (unsigned)((count + 31) / 32);
  k_tile_sum_rows_tma<T><<<grid, 64, smem, stream>>>(mx, sp, ts, first, count, P);
  AOL_LAUNCH_CHECK("k_tile_sum_rows_tma");
  return AOL_OK;
}

template <typename T>
static int launch_tile_sum_cols(const T* x, T* sp, const DevTiler& ts, int64_t cs, int64_t Bs, int64_t P,
                                int64_t first, int64_t count, cudaStream_t stream) {
  const T* base = x + cs + first;
  const int rem = (int)(((uintptr_t)base % 16) / sizeof(T));
  if (count + rem > Bs || (uintptr_t)base % sizeof(T)) return 1;   // the tensor's rows must not overlap
  base -= rem;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!encode) return fail(AOL_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap mx;
  constexpr int RB = 8192 / (32 * (int)sizeof(T));
  cuuint64_t dims[2] = {(cuuint64_t)(count + rem), (cuuint64_t)P}, str[1] = {(cuuint64_t)(Bs * sizeof(T))};
  cuuint32_t box[2] = {32, (cuuint32_t)RB}, es[2] = {1, 1};
  if (encode(&mx, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
             const_cast<T*>(base), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(AOL_ECUDA, "tile_sum.columns: tensor map encode failed");
  const int smem = kColStages * 8192;
  const unsigned grid = (unsigned)((count + rem + 31) / 32);
  k_tile_sum_cols<T><<<grid, 64, smem, stream>>>(mx, sp, ts, first, rem, count, P);
  AOL_LAUNCH_CHECK("k_tile_sum_cols");
  return AOL_OK;
}

int launch_tile_sum(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t stream) {
  DevTiler tx, ts;
  int rc;
  if ((rc = make_dev_tiler(t.tilers[0], tx)) || (rc = make_dev_tiler(t.tilers[1], ts))) return rc;
  const int64_t px = tiler_pat_total(t.tilers[0]);
  int64_t cs = 0, As = 0, Bs = 0;
  const int kind = tile_sum_kind(t, cs, As, Bs);
  const bool f32 = t.dtype == AOL_F32;
  if (kind == 0) {
    rc = f32 ? launch_tile_sum_rows_tma<float>((const float*)ports[0], (float*)ports[1], ts, cs, As, px, first, count,
                                               stream)
             : launch_tile_sum_rows_tma<double>((const double*)ports[0], (double*)ports[1], ts, cs, As, px, first,
                                                count, stream);
    if (rc <= 0) return rc;
    const int per = 32 * (f32 ? ts_warps<float>() : ts_warps<double>());
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + per - 1) / per, (int64_t)kNumSMs * 32));
    if (f32)
      k_tile_sum_rows<float><<<grid, per, 0, stream>>>((const float*)ports[0], (float*)ports[1], cs, As, px, ts,
                                                       first, count);
    else
      k_tile_sum_rows<double><<<grid, per, 0, stream>>>((const double*)ports[0], (double*)ports[1], cs, As, px, ts,
                                                        first, count);
    AOL_LAUNCH_CHECK("k_tile_sum_rows");
    return AOL_OK;
  }
  if (kind == 1 && tile_sum_cols_ok(As, Bs, px, count, f32 ? 4 : 8)) {
    // returns 1 when this range's alignment needs the direct form
    rc = f32 ? launch_tile_sum_cols<float>((const float*)ports[0], (float*)ports[1], ts, cs, Bs, px, first, count, stream)
             : launch_tile_sum_cols<double>((const double*)ports[0], (double*)ports[1], ts, cs, Bs, px, first, count,
                                            stream);
    if (rc <= 0) return rc;
  }
  if ((kind >= 2 || (kind == 1 && As != 1)) && tile_sum_batched_ok(t, first, count, As)) {
    DevTiler bx, by;
    filter_batched_route(t, first, count, bx, by);
    void* fp[3] = {ports[0], nullptr, ports[1]};
    return f32 ? launch_filter_b32_q<float, 1, 8>(t, bx, by, first, count, (int)px, 1, fp, stream)
               : launch_filter_b32_q<double, 1, 8>(t, bx, by, first, count, (int)px, 1, fp, stream);
  }
  if (kind == 1 || kind == 3) {
    const unsigned grid = grid_for(count, 256, 16);
    if (kind == 1) {
      if (f32) k_tile_sum_direct<float, true><<<grid, 256, 0, stream>>>((const float*)ports[0], (float*)ports[1], cs, As, Bs, tx, ts, first, count, px);
      else k_tile_sum_direct<double, true><<<grid, 256, 0, stream>>>((const double*)ports[0], (double*)ports[1], cs, As, Bs, tx, ts, first, count, px);
    } else {
      if (f32) k_tile_sum_direct<float, false><<<grid, 256, 0, stream>>>((const float*)ports[0], (float*)ports[1], cs, As, Bs, tx, ts, first, count, px);
      else k_tile_sum_direct<double, false><<<grid, 256, 0, stream>>>((const double*)ports[0], (double*)ports[1], cs, As, Bs, tx, ts, first, count, px);
    }
    AOL_LAUNCH_CHECK("k_tile_sum_direct");
    return AOL_OK;
  }
  const size_t smem = (size_t)px * tx.a * sizeof(int64_t);
  if (t.dtype == AOL_F32)
    k_tile_sum_generic<float><<<grid_for(count, 256, 16), 256, smem, stream>>>(
        (const float*)ports[0], (float*)ports[1], tx, ts, first, count, (int)px);
  else
    k_tile_sum_generic<double><<<grid_for(count, 256, 16), 256, smem, stream>>>(
        (const double*)ports[0], (double*)ports[1], tx, ts, first, count, (int)px);
  AOL_LAUNCH_CHECK("k_tile_sum_generic");
  return AOL_OK;
}

}  // namespace aol
