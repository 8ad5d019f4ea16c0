// Line filters: the tile_filter class of the Array-OL downscaler (config C3).
//
// Recognised when both tilers (x: input, y: output) have
//   * the same array rank a, repetition rank a, identity paving and zero origin on
//     every axis except one "line" axis dp, where repetitions step by s_x / s_y;
//   * repetition extent == array extent on every non-line axis;
//   * a 1-D pattern along dp with unit fitting (x may wrap around the line, y may not).
// The arrays then factor as [outer, line, inner] (outer = product of the axes
// before dp, inner = product after), and repetition rho = ((o*NL) + l)*inner + i.
//     y[o, l*s_y + oy + j, i] = sum_t w[j, t] * x[o, (l*s_x + ox + t) mod S_x, i]
// accumulated in pattern order with __fmul_rn / __fadd_rn (bit-exact vs the oracle).
//
// inner == 1 (horizontal filter, e.g. 13 taps paving 8): the window is a contiguous
// run read with float4 when aligned and not wrapping.  inner > 1 (vertical filter,
// e.g. 14 taps paving 9): consecutive threads take consecutive i, so every tap is a
// coalesced row read and every output a coalesced row write.
#include <cstdlib>
#include <cstring>

#include "aol_async.cuh"
#include "aol_common.cuh"

namespace aol {

struct LineGeom {
  int64_t outer, inner, NL;
  int64_t Sx, Sy;          // line extents in x / y
  int64_t sx, sy;          // paving steps along the line
  int64_t ox, oy;          // origins along the line (reduced)
  int px, py;
  int small;               // rho fits 32 bits: fast divisions
  FastDiv32 div_inner, div_nl;
};

bool line_filter_geometry(const aol_task& t, LineGeom& g) {
  const aol_tiler &tx = t.tilers[0], &ty = t.tilers[1];
  if (t.dtype != AOL_F32) return false;
  const int a = tx.arr_rank;
  if (ty.arr_rank != a || tx.rep_rank != a || ty.rep_rank != a) return false;
  // line axis: the only axis with non-zero fitting in x
  int dp = -1, kx = -1, ky = -1;
  for (int k = 0; k < tx.pat_rank; ++k) {
    if (tx.pattern[k] == 1) continue;
    if (kx >= 0) return false;
    kx = k;
  }
  for (int k = 0; k < ty.pat_rank; ++k) {
    if (ty.pattern[k] == 1) continue;
    if (ky >= 0) return false;
    ky = k;
  }
  if (kx < 0) return false;
  for (int d = 0; d < a; ++d)
    if (tx.fitting[d][kx] != 0) {
      if (dp >= 0 || tx.fitting[d][kx] != 1) return false;
      dp = d;
    }
  if (dp < 0) return false;
  if (ky >= 0)
    for (int d = 0; d < a; ++d)
      if (ty.fitting[d][ky] != (d == dp ? 1 : 0)) return false;
  for (int d = 0; d < a; ++d) {
    for (int j = 0; j < a; ++j) {
      const int64_t wantx = (d == j) ? (d == dp ? tx.paving[d][d] : 1) : 0;
      const int64_t wanty = (d == j) ? (d == dp ? ty.paving[d][d] : 1) : 0;
      if (tx.paving[d][j] != wantx || ty.paving[d][j] != wanty) return false;
    }
    if (d != dp) {
      if (tx.rep[d] != tx.array[d] || ty.array[d] != tx.array[d] || ty.rep[d] != tx.rep[d]) return false;
      if (tx.origin[d] % tx.array[d] != 0 || ty.origin[d] % ty.array[d] != 0) return false;
    }
  }
  if (tx.paving[dp][dp] <= 0 || ty.paving[dp][dp] <= 0) return false;
  memset(&g, 0, sizeof(g));
  g.outer = 1;
  g.inner = 1;
  for (int d = 0; d < dp; ++d) g.outer *= tx.array[d];
  for (int d = dp + 1; d < a; ++d) g.inner *= tx.array[d];
  g.NL = tx.rep[dp];
  g.Sx = tx.array[dp];
  g.Sy = ty.array[dp];
  g.sx = tx.paving[dp][dp];
  g.sy = ty.paving[dp][dp];
  g.ox = ((tx.origin[dp] % g.Sx) + g.Sx) % g.Sx;
  g.oy = ((ty.origin[dp] % g.Sy) + g.Sy) % g.Sy;
  g.px = (int)tx.pattern[kx];
  g.py = ky >= 0 ? (int)ty.pattern[ky] : 1;
  if (g.px > 32 || g.py > 8 || g.px > g.Sx) return false;
  // y must not wrap
  if (g.oy + g.sy * (g.NL - 1) + g.py - 1 >= g.Sy) return false;
  const int64_t R = g.outer * g.NL * g.inner;
  g.small = R < (1ll << 31) && g.inner < (1ll << 31) && g.NL < (1ll << 31);
  if (g.small) {
    g.div_inner = FastDiv32((uint32_t)g.inner);
    g.div_nl = FastDiv32((uint32_t)g.NL);
  }
  return true;
}

template <int PX, int PY, typename IDX>
__global__ void __launch_bounds__(256) k_line_filter(const float* __restrict__ x, const float* __restrict__ w,
                                                     float* __restrict__ y, LineGeom g, int64_t first,
                                                     int64_t count) {
  constexpr int MAXP = PX > 0 ? PX : 32;
  constexpr int MAXO = PY > 0 ? PY : 8;
  const int px = PX > 0 ? PX : g.px;
  const int py = PY > 0 ? PY : g.py;
  __shared__ float ws[32 * 8];
  for (int k = threadIdx.x; k < px * py; k += blockDim.x) ws[k] = w[k];
  __syncthreads();
  const IDX inner = (IDX)g.inner;
  const IDX SxI = (IDX)(g.Sx * g.inner), SyI = (IDX)(g.Sy * g.inner);
  const IDX Sx = (IDX)g.Sx;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = first + e;
    IDX i, l, o;
    if (g.small) {
      uint32_t q, r, q2, r2;
      g.div_inner.divmod((uint32_t)rho, q, r);
      g.div_nl.divmod(q, q2, r2);
      i = (IDX)r; l = (IDX)r2; o = (IDX)q2;
    } else {
      i = (IDX)(rho % g.inner);
      const int64_t q = rho / g.inner;
      l = (IDX)(q % g.NL);
      o = (IDX)(q / g.NL);
    }
    IDX row = l * (IDX)g.sx + (IDX)g.ox;
    if (row >= Sx) row %= Sx;
    const float* xb = x + (o * SxI + i);
    float xv[MAXP];
    if (row + (IDX)px <= Sx) {                       // window does not wrap
      if (g.inner == 1 && MAXP <= 16 && row + 16 <= Sx && ((((uintptr_t)(xb + row)) & 15) == 0)) {
        const float4* p = reinterpret_cast<const float4*>(xb + row);
#pragma unroll
        for (int q = 0; q < (MAXP + 3) / 4; ++q) {
          const float4 v = __ldg(p + q);
          if (4 * q < MAXP) xv[4 * q] = v.x;
          if (4 * q + 1 < MAXP) xv[4 * q + 1] = v.y;
          if (4 * q + 2 < MAXP) xv[4 * q + 2] = v.z;
          if (4 * q + 3 < MAXP) xv[4 * q + 3] = v.w;
        }
      } else {
        const float* xp = xb + row * inner;
#pragma unroll
        for (int t = 0; t < MAXP; ++t) {
          if (t < px) {
            xv[t] = __ldg(xp);
            xp += inner;
          }
        }
      }
    } else {                                          // wraps around the line: rare
#pragma unroll
      for (int t = 0; t < MAXP; ++t) {
        if (t < px) {
          xv[t] = __ldg(xb + row * inner);
          if (++row == Sx) row = 0;
        }
      }
    }
    float* yp = y + (o * SyI + (l * (IDX)g.sy + (IDX)g.oy) * inner + i);
#pragma unroll
    for (int j = 0; j < MAXO; ++j) {
      if (j < py) {
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < MAXP; ++t)
          if (t < px) acc = __fadd_rn(acc, __fmul_rn(ws[j * px + t], xv[t]));
        *yp = acc;
        yp += inner;
      }
    }
  }
}

// Vertical strips (inner > 1): one thread computes REPS consecutive line repetitions of one
// (outer, inner) column.  Their windows overlap (px > sx), so the (REPS-1)*sx + px rows are
// loaded once into registers; every output is still summed over its own taps in order.
template <int PX, int PY, int SX, int REPS>
__global__ void __launch_bounds__(256, (REPS <= 2 ? 4 : 3)) k_line_filter_vstrip(const float* __restrict__ x, const float* __restrict__ w,
                                                            float* __restrict__ y, LineGeom g, int64_t first,
                                                            int64_t last, int64_t o_lo, int64_t ngroups) {
  constexpr int NRW = (REPS - 1) * SX + PX;
  __shared__ float ws[PX * PY];
  for (int k = threadIdx.x; k < PX * PY; k += blockDim.x) ws[k] = w[k];
  __syncthreads();
  const uint32_t inner = (uint32_t)g.inner;
  const int64_t NLG = (g.NL + REPS - 1) / REPS;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ngroups;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % g.inner;
    const int64_t q = e / g.inner;
    const int64_t lg = q % NLG, o = o_lo + q / NLG;
    const int64_t l0 = lg * REPS;
    const int64_t rho0 = (o * g.NL + l0) * g.inner + i;
    const int64_t rhoN = (o * g.NL + min(l0 + REPS, g.NL) - 1) * g.inner + i;
    if (rhoN < first || rho0 > last) continue;
    uint32_t row = (uint32_t)((l0 * SX + g.ox) % g.Sx);
    const float* xb = x + (uint64_t)o * (uint64_t)(g.Sx * g.inner) + i;
    float xw[NRW];
#pragma unroll
    for (int t = 0; t < NRW; ++t) {
      xw[t] = __ldg(xb + (uint64_t)row * inner);
      if (++row == (uint32_t)g.Sx) row = 0;
    }
    float* yb = y + (uint64_t)o * (uint64_t)(g.Sy * g.inner) + i;
#pragma unroll
    for (int u = 0; u < REPS; ++u) {
      const int64_t l = l0 + u;
      const int64_t rho = rho0 + (int64_t)u * g.inner;
      if (l >= g.NL || rho < first || rho > last) continue;
      float* yp = yb + (uint64_t)(l * g.sy + g.oy) * inner;
#pragma unroll
      for (int j = 0; j < PY; ++j) {
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < PX; ++t) acc = __fadd_rn(acc, __fmul_rn(ws[j * PX + t], xw[u * SX + t]));
        yp[(uint64_t)j * inner] = acc;
      }
    }
  }
}

static_assert(sizeof(LineGeom) <= 256, "LineGeomBuf in aol_tile.cu must hold a LineGeom");

static bool hline_stream_ok(const LineGeom& g);
static bool hline_stream_any_ok(const LineGeom& g);
static bool vline_stream_ok(const LineGeom& g);
static int launch_line_stream(const LineGeom& lg, int64_t first, int64_t count, const float* x, const float* w,
                              float* y, cudaStream_t s);

// Generic horizontal line filter (inner == 1: 1-D FIRs and decimating FIRs with paving <= 4,
// any px <= 32 / py <= 8): a CTA takes up to 8192 consecutive repetitions of one line, loads
// their whole input window [ox + sx*l0, ox + sx*(l0+n-1) + px) once with coalesced loads into
// shared memory (padded one float per 32 so strided window starts hit distinct banks), then
// each thread forms its repetitions' py outputs from it, taps in pattern order with
// __fmul_rn / __fadd_rn (bit-exact).  Replaces one thread per repetition re-reading
// overlapping windows through L1 (1-D FIR, 8 taps, 2^27 elements: 2.18 -> 0.75 ms).  Wider
// pavings keep the thread-per-repetition kernel, which measured faster there.
constexpr int LT_THREADS = 256, LT_WIN = 8192;          // window floats per tile (32 KB + padding)

__device__ __forceinline__ int lt_pad(int k) { return k + (k >> 5); }

__global__ void __launch_bounds__(LT_THREADS) k_line_tiled(const float* __restrict__ x, const float* __restrict__ w,
                                                           float* __restrict__ y, LineGeom g, int TL,
                                                           int64_t first, int64_t last, int64_t tile0,
                                                           int64_t ntiles) {
  __shared__ float win[LT_WIN + LT_WIN / 32 + 1];
  __shared__ float ws[32 * 8];
  const int px = g.px, py = g.py;
  for (int k = threadIdx.x; k < px * py; k += LT_THREADS) ws[k] = w[k];
  const int64_t tpl = (g.NL + TL - 1) / TL;                 // tiles per line
  for (int64_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
    const int64_t tile = tile0 + tt;
    const int64_t o = tile / tpl, l0 = (tile - o * tpl) * TL;
    const int n = (int)(g.NL - l0 < TL ? g.NL - l0 : TL);
    const int64_t rho0 = o * g.NL + l0;
    // clip to the launch range
    const int a = (int)(first > rho0 ? first - rho0 : 0);
    const int b = (int)(last < rho0 + n - 1 ? last - rho0 + 1 : n);
    __syncthreads();                                        // previous tile's window consumed
    if (a < b) {
      const int64_t c0 = (g.ox + g.sx * (l0 + a)) % g.Sx;
      const int wl = (int)(g.sx * (b - 1 - a) + px);
      const float* xr = x + o * g.Sx;
      for (int k = threadIdx.x; k < wl; k += LT_THREADS) {
        int64_t c = c0 + k;
        if (c >= g.Sx) c %= g.Sx;
        win[lt_pad(k)] = __ldg(xr + c);
      }
    }
    __syncthreads();
    if (a < b) {
      float* yr = y + o * g.Sy + g.oy;
      for (int r = a + threadIdx.x; r < b; r += LT_THREADS) {
        const int base = (int)(g.sx * (r - a));
        float* yp = yr + (l0 + r) * g.sy;
        for (int j = 0; j < py; ++j) {
          float acc = 0.0f;
          for (int t = 0; t < px; ++t) acc = __fadd_rn(acc, __fmul_rn(ws[j * px + t], win[lt_pad(base + t)]));
          yp[j] = acc;
        }
      }
    }
  }
}

static bool line_tiled_ok(const LineGeom& g) {
  return g.inner == 1 && g.sx >= 1 && g.sx <= 4 && !(g.px == 13 && g.py == 3) && !(g.px == 14 && g.py == 4);
}

static int launch_line_tiled(const LineGeom& g, int64_t first, int64_t count, const float* x, const float* w,
                             float* y, cudaStream_t s) {
  const int TL = (int)std::min<int64_t>(LT_WIN, (LT_WIN - g.px) / g.sx + 1);
  const int64_t last = first + count - 1;
  const int64_t tpl = (g.NL + TL - 1) / TL;
  const int64_t o_lo = first / g.NL, o_hi = last / g.NL;
  const int64_t t_lo = o_lo * tpl + (first - o_lo * g.NL) / TL;
  const int64_t t_hi = o_hi * tpl + (last - o_hi * g.NL) / TL;
  const int64_t ntiles = t_hi - t_lo + 1;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)kNumSMs * 8);
  k_line_tiled<<<grid, LT_THREADS, 0, s>>>(x, w, y, g, TL, first, last, t_lo, ntiles);
  AOL_LAUNCH_CHECK("k_line_tiled");
  return AOL_OK;
}

const char* line_filter_variant(const LineGeom& g) {
  if (hline_stream_ok(g)) return "tile_filter.line_13x3_stream";
  if (hline_stream_any_ok(g)) return "tile_filter.line_stream";
  if (vline_stream_ok(g)) return "tile_filter.line_14x4_stream";
  if (g.px == 13 && g.py == 3) return "tile_filter.line_13x3";
  if (g.px == 14 && g.py == 4 && g.inner > 1 && g.sx == 9) return "tile_filter.line_14x4_vstrip";
  if (g.px == 14 && g.py == 4) return "tile_filter.line_14x4";
  if (line_tiled_ok(g)) return "tile_filter.line_tiled";
  return "tile_filter.line";
}

int launch_line_filter(const aol_task& t, const LineGeom& g, int64_t first, int64_t count, void* const* ports,
                       cudaStream_t s) {
  const float* x = static_cast<const float*>(ports[0]);
  const float* w = static_cast<const float*>(ports[1]);
  float* y = static_cast<float*>(ports[2]);
  if (count > 0 && (hline_stream_ok(g) || hline_stream_any_ok(g) || vline_stream_ok(g)))
    return launch_line_stream(g, first, count, x, w, y, s);
  const unsigned grid = grid_for(count, 256, 8);
  // 32-bit offsets whenever both arrays fit (every in-range offset < 2^32)
  const bool idx32 = g.outer * g.Sx * g.inner < (1ll << 32) && g.outer * g.Sy * g.inner < (1ll << 32);
  if (idx32 && g.inner > 1 && g.px == 14 && g.py == 4 && g.sx == 9 && g.Sx * g.inner < (1ll << 32)) {
    static const int reps_env = getenv("AOL_VSTRIP_REPS") ? atoi(getenv("AOL_VSTRIP_REPS")) : 0;
    const int REPS = reps_env >= 2 && reps_env <= 4 ? reps_env : 4;
    const int64_t last = first + count - 1;
    const int64_t NLG = (g.NL + REPS - 1) / REPS;
    // repetition groups intersecting [first, last]
    const int64_t o_lo = first / (g.NL * g.inner), o_hi = last / (g.NL * g.inner);
    const int64_t ngroups = (o_hi - o_lo + 1) * NLG * g.inner;
    const unsigned grid = grid_for(ngroups, 256, 8);
    if (REPS == 2)
      k_line_filter_vstrip<14, 4, 9, 2><<<grid, 256, 0, s>>>(x, w, y, g, first, last, o_lo, ngroups);
    else if (REPS == 3)
      k_line_filter_vstrip<14, 4, 9, 3><<<grid, 256, 0, s>>>(x, w, y, g, first, last, o_lo, ngroups);
    else
      k_line_filter_vstrip<14, 4, 9, 4><<<grid, 256, 0, s>>>(x, w, y, g, first, last, o_lo, ngroups);
    AOL_LAUNCH_CHECK("k_line_filter_vstrip");
    return AOL_OK;
  }
  if (line_tiled_ok(g)) return launch_line_tiled(g, first, count, x, w, y, s);
  if (idx32) {
    if (g.px == 13 && g.py == 3)
      k_line_filter<13, 3, uint32_t><<<grid, 256, 0, s>>>(x, w, y, g, first, count);
    else if (g.px == 14 && g.py == 4)
      k_line_filter<14, 4, uint32_t><<<grid, 256, 0, s>>>(x, w, y, g, first, count);
    else
      k_line_filter<0, 0, uint32_t><<<grid, 256, 0, s>>>(x, w, y, g, first, count);
  } else {
    k_line_filter<0, 0, int64_t><<<grid, 256, 0, s>>>(x, w, y, g, first, count);
  }
  AOL_LAUNCH_CHECK("k_line_filter");
  (void)t;
  return AOL_OK;
}

}  // namespace aol

namespace aol {

// -----------------------------------------------------------------------------
// Task fusion: a horizontal line filter (inner == 1) feeding a vertical line filter
// through an intermediate array that only the second task reads — the Array-OL
// downscaler (config C3).  The fused kernel computes, per tile of the consumer's
// repetition space, the intermediate rows the tile needs into shared memory (same
// tap order, same __fmul_rn/__fadd_rn, so the values are bit-identical to the
// unfused intermediate) and applies the consumer filter from shared memory.  The
// intermediate never touches HBM: x is read once (+ (px_v - sx_v)/(TV*sx_v) halo
// rows) and y written once.
// -----------------------------------------------------------------------------
constexpr int FZ_TV = 8;       // consumer line repetitions per tile
constexpr int FZ_HR = 32;      // producer repetitions per intermediate row per tile
constexpr int FZ_THREADS = 256;

struct FusedGeom {
  LineGeom h, v;
  int64_t R;                   // rows of the intermediate (= v.Sx)
  int64_t Wm;                  // columns of the intermediate (= h.Sy = v.inner)
  int64_t W;                   // x line length (= h.Sx)
  int NR;                      // intermediate rows per tile
  int TI;                      // intermediate columns per tile (FZ_HR * h.sy)
  int64_t tiles_i, tiles_l;
};

bool fused_line_geometry(const aol_task& th, const aol_task& tv, FusedGeom& f) {
  if (!line_filter_geometry(th, f.h) || !line_filter_geometry(tv, f.v)) return false;
  const LineGeom &h = f.h, &v = f.v;
  if (h.inner != 1 || v.inner != h.Sy || h.outer != v.outer * v.Sx) return false;
  // the producer writes every intermediate element exactly once (dense, no origin)
  if (h.oy != 0 || h.sy != h.py || h.NL * h.sy != h.Sy) return false;
  if (h.px > 16 || v.px > 16 || h.py > 8 || v.py > 8) return false;
  // the intermediate array of the producer's output tiler must be the consumer's x array
  const aol_tiler &hy = th.tilers[1], &vx = tv.tilers[0];
  if (hy.arr_rank != vx.arr_rank) return false;
  for (int d = 0; d < hy.arr_rank; ++d)
    if (hy.array[d] != vx.array[d]) return false;
  f.R = v.Sx;
  f.Wm = h.Sy;
  f.W = h.Sx;
  f.NR = (int)((FZ_TV - 1) * v.sx + v.px);
  f.TI = FZ_HR * (int)h.sy;
  if ((int64_t)f.NR * f.TI * 4 > 96 * 1024) return false;
  f.tiles_i = (f.Wm + f.TI - 1) / f.TI;
  f.tiles_l = (v.NL + FZ_TV - 1) / FZ_TV;
  return f.R * f.W * v.outer < (1ll << 32);   // 32-bit x offsets
}

// Tile form: a CTA owns (frame, FZ_TV consecutive consumer line repetitions, TI intermediate
// columns).  Phase 1 computes the NR = (FZ_TV-1)*sx_v + px_v intermediate rows of the tile
// into shared memory (producer taps in order, two producer repetitions per thread per
// iteration so 8 window loads are in flight); phase 2 applies the consumer filter from
// shared memory.  Every value is formed in the unfused order -> bit-identical results.
template <int PXH, int PYH, int PXV, int PYV>
__global__ void __launch_bounds__(FZ_THREADS, 3) k_fused_line_filters(const float* __restrict__ x,
                                                                      const float* __restrict__ wh,
                                                                      const float* __restrict__ wv,
                                                                      float* __restrict__ y, FusedGeom g,
                                                                      int64_t first, int64_t last, int64_t tile0,
                                                                      int64_t ntiles) {
  extern __shared__ float mt[];                     // [NR][TI] intermediate tile
  __shared__ float swh[PXH * PYH], swv[PXV * PYV];
  for (int k = threadIdx.x; k < PXH * PYH; k += blockDim.x) swh[k] = wh[k];
  for (int k = threadIdx.x; k < PXV * PYV; k += blockDim.x) swv[k] = wv[k];
  const LineGeom &h = g.h, &v = g.v;
  const uint32_t R = (uint32_t)g.R, W = (uint32_t)g.W, TI = (uint32_t)g.TI;
  const int items = g.NR * FZ_HR;
  for (int64_t tt = tile0 + blockIdx.x; tt < tile0 + ntiles; tt += gridDim.x) {
    const uint32_t ib = (uint32_t)(tt % g.tiles_i);
    const int64_t q = tt / g.tiles_i;
    const uint32_t lb = (uint32_t)(q % g.tiles_l);
    const uint32_t fr = (uint32_t)(q / g.tiles_l);
    const uint32_t lv0 = lb * FZ_TV;
    const uint32_t i0 = ib * TI;
    const uint32_t lh0 = i0 / (uint32_t)h.sy;
    const uint32_t row0 = lv0 * (uint32_t)v.sx + (uint32_t)v.ox;
    __syncthreads();                                // weights ready / previous tile consumed
    for (int it = threadIdx.x; it < items; it += 2 * FZ_THREADS) {
      float xv[2][16];
      uint32_t dst[2];
      bool ok[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int item = it + u * FZ_THREADS;
        const uint32_t k = (uint32_t)item / FZ_HR, hh = (uint32_t)item % FZ_HR;
        const uint32_t lh = lh0 + hh;
        ok[u] = item < items && lh < (uint32_t)h.NL;
        dst[u] = k * TI + hh * PYH;
        if (!ok[u]) continue;
        uint32_t r = row0 + k;
        while (r >= R) r -= R;
        const uint32_t xrow = (fr * R + r) * W;
        uint32_t col = lh * (uint32_t)h.sx + (uint32_t)h.ox;
        if (col >= W) col %= W;
        if (col + 16 <= W && ((xrow + col) & 3) == 0) {
          const float4* p = reinterpret_cast<const float4*>(x + xrow + col);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4 t4 = __ldg(p + e);
            xv[u][4 * e] = t4.x; xv[u][4 * e + 1] = t4.y; xv[u][4 * e + 2] = t4.z; xv[u][4 * e + 3] = t4.w;
          }
        } else {
          uint32_t c = col;
#pragma unroll
          for (int t = 0; t < PXH; ++t) {
            xv[u][t] = __ldg(x + xrow + c);
            if (++c == W) c = 0;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int j = 0; j < PYH; ++j) {
          float acc = 0.0f;
#pragma unroll
          for (int t = 0; t < PXH; ++t) acc = __fadd_rn(acc, __fmul_rn(swh[j * PXH + t], xv[u][t]));
          mt[dst[u] + j] = acc;
        }
      }
    }
    __syncthreads();
    for (int item = threadIdx.x; item < FZ_TV * (int)TI; item += blockDim.x) {
      const uint32_t l = (uint32_t)item / TI, c = (uint32_t)item % TI;
      const int64_t lv = lv0 + l, i = i0 + c;
      if (lv >= v.NL || i >= g.Wm) continue;
      const int64_t rho = ((int64_t)fr * v.NL + lv) * g.Wm + i;
      if (rho < first || rho > last) continue;
      float* yp = y + ((int64_t)fr * v.Sy + lv * v.sy + v.oy) * g.Wm + i;
      const float* mp = mt + (l * (uint32_t)v.sx) * TI + c;
#pragma unroll
      for (int j = 0; j < PYV; ++j) {
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < PXV; ++t) acc = __fadd_rn(acc, __fmul_rn(swv[j * PXV + t], mp[t * TI]));
        yp[(int64_t)j * g.Wm] = acc;
      }
    }
  }
}

// -----------------------------------------------------------------------------
// Streaming form (the default when the geometry allows): a persistent CTA per SM owns a
// contiguous run of consumer line repetitions.  One producer warp streams whole x rows
// (W floats + a 32-byte wrap halo = x[row][0..7]) into an NST-stage shared-memory ring
// with cp.async.bulk, completion on mbarriers.  Each consumer thread owns one producer
// repetition lh of the row (window x[8lh .. 8lh+12]), computes its PYH intermediate values
// for the row and folds them straight into register accumulators of the consumer filter
// for its PYH columns -- "current" rep (tap t = s mod SXV) and "previous" rep (tap
// t + SXV while t < PXV - SXV).  Rows arrive in tap order, so every output is the unfused
// sum in the unfused order (bit-identical), and the intermediate never exists anywhere.
// x is read once (+ (PXV - SXV) rows per CTA run and per frame), y written once.
// -----------------------------------------------------------------------------
constexpr int FS_NST = 8;

// (a0, a1) += (p0, p1) with one packed add (each lane IEEE round-to-nearest, like
// __fadd_rn).  The products stay scalar __fmul_rn: ptxas contracts a packed mul.rn.f32x2
// feeding a packed add into FFMA2 (one rounding), which would break bit-exactness.
__device__ __forceinline__ void add2_rn(float& a0, float& a1, float p0, float p1) {
  asm("{\n\t.reg .b64 ra, rp;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rp, {%2, %3};\n\t"
      "add.rn.f32x2 ra, ra, rp;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(p0), "f"(p1));
}

struct StreamGeom {
  int64_t F, R, W;               // x: [F, R, W]
  int64_t NLh, NLv, Wm, Sy;      // producer reps per row, consumer reps per frame, y row length, y rows
  int64_t first, last;           // consumer repetition range (rho, inclusive)
};

// VONLY: the consumer alone (unfused vertical filter): the ring holds rows of its input
// (width W = Wm, no halo) and a thread's PYH "producer outputs" are the row's columns
// PYH*lh .. PYH*lh + PYH-1, read from shared memory instead of computed.
template <int PXH, int SXH, int PYH, int PXV, int SXV, int PYV, bool VONLY = false>
__global__ void __launch_bounds__(512, 1) k_fused_stream(const float* __restrict__ x, const float* __restrict__ wh,
                                                          const float* __restrict__ wv, float* __restrict__ y,
                                                          StreamGeom g, int n_consumer_warps) {
  static_assert(PXV > SXV && PXV - SXV <= SXV, "consumer windows overlap by less than one paving step");
  extern __shared__ __align__(128) unsigned char fs_smem[];
  const int RS = (int)g.W + (VONLY ? 0 : 8);                     // floats per stage (row + halo)
  float* stages = reinterpret_cast<float*>(fs_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(fs_smem + (size_t)FS_NST * RS * 4);
  uint64_t* empty = full + FS_NST;
  __shared__ float swv[PXV * PYV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < PXV * PYV; k += blockDim.x) swv[k] = wv[k];
  if (threadIdx.x == 0) {
    for (int i = 0; i < FS_NST; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, n_consumer_warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's consumer repetitions [v0, v1) in (frame * NLv + lv) units
  const int64_t v_lo = g.first / g.Wm, v_hi = g.last / g.Wm + 1;
  const int64_t nv = v_hi - v_lo;
  const int64_t v0 = v_lo + nv * blockIdx.x / gridDim.x, v1 = v_lo + nv * (blockIdx.x + 1) / gridDim.x;
  const uint32_t row_bytes = (uint32_t)g.W * 4;

  if (warp == n_consumer_warps) {                                 // producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t v = v0; v < v1;) {
        const int64_t f = v / g.NLv, ra = v % g.NLv;
        const int64_t rb = (v1 - f * g.NLv < g.NLv) ? v1 - f * g.NLv : g.NLv;
        const int64_t nrows = (rb - ra) * SXV + (PXV - SXV);
        for (int64_t sidx = 0; sidx < nrows; ++sidx) {
          const int64_t row = (ra * SXV + sidx) % g.R;
          const float* src = x + (f * g.R + row) * g.W;
          mbar_wait(empty + stage, phase ^ 1);
          mbar_expect_tx(full + stage, row_bytes + (VONLY ? 0 : 32));
          float* dst = stages + (size_t)stage * RS;
          bulk_load(dst, src, row_bytes, full + stage);
          if (!VONLY) bulk_load(dst + g.W, src, 32, full + stage);   // wrap halo: x[row][0..7]
          if (++stage == FS_NST) {
            stage = 0;
            phase ^= 1;
          }
        }
        v = f * g.NLv + rb;
      }
    }
    return;
  }

  // consumers: thread lh owns producer repetition lh (threads past NLh compute on a clamped
  // window and never store)
  const int lh = threadIdx.x;
  const bool active = lh < g.NLh;
  // window (fused) / column group (VONLY) byte offset in a row
  const uint32_t win = (uint32_t)((VONLY ? PYH : SXH) * (active ? lh : 0)) * 4;
  const int64_t left = g.Wm - (int64_t)PYH * lh;
  const int ncol = VONLY ? (left < PYH ? (int)(left > 0 ? left : 0) : PYH) : PYH;   // columns this thread stores
  float whr[PYH][PXH];
  if (!VONLY) {
#pragma unroll
    for (int j = 0; j < PYH; ++j)
#pragma unroll
      for (int t = 0; t < PXH; ++t) whr[j][t] = wh[j * PXH + t];
  }
  const uint32_t stage0 = smem_u32(stages);
  const uint32_t stage_bytes = (uint32_t)RS * 4;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t v = v0; v < v1;) {
    const int64_t f = v / g.NLv, ra = v % g.NLv;
    const int64_t rb = (v1 - f * g.NLv < g.NLv) ? v1 - f * g.NLv : g.NLv;
    const int nrep = (int)(rb - ra);
    // this frame segment's outputs lie wholly inside [first, last]?
    const bool whole = (f * g.NLv + ra) * g.Wm >= g.first && (f * g.NLv + rb) * g.Wm - 1 <= g.last;
    float cur[PYH][PYV], prev[PYH][PYV];
    for (int u = 0; u <= nrep; ++u) {               // u == nrep: the tail rows of rep nrep-1 only
#pragma unroll
      for (int t = 0; t < SXV; ++t) {
        if (u == nrep && t >= PXV - SXV) break;
        mbar_wait(full + stage, phase);
        float xw[16];
        const uint32_t a = stage0 + (uint32_t)stage * stage_bytes + win;
        if (VONLY) {
#pragma unroll
          for (int c = 0; c < PYH; ++c)
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xw[c]) : "r"(a + 4 * c));
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float4 q;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                         : "r"(a + 16 * e));
            xw[4 * e] = q.x; xw[4 * e + 1] = q.y; xw[4 * e + 2] = q.z; xw[4 * e + 3] = q.w;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stage);
        if (++stage == FS_NST) {
          stage = 0;
          phase ^= 1;
        }
        if (t == 0) {                               // rep u starts, rep u-1 continues
#pragma unroll
          for (int c = 0; c < PYH; ++c)
#pragma unroll
            for (int j = 0; j < PYV; ++j) {
              prev[c][j] = cur[c][j];
              cur[c][j] = 0.0f;
            }
        }
        float hv[PYH];                              // the producer's outputs, unfused order
        if (VONLY) {
#pragma unroll
          for (int c = 0; c < PYH; ++c) hv[c] = xw[c];
        } else {
#pragma unroll
          for (int c = 0; c < PYH; ++c) hv[c] = 0.0f;
#pragma unroll
          for (int k = 0; k < PXH; ++k) {
#pragma unroll
            for (int c = 0; c + 1 < PYH; c += 2)
              add2_rn(hv[c], hv[c + 1], __fmul_rn(whr[c][k], xw[k]), __fmul_rn(whr[c + 1][k], xw[k]));
            if (PYH % 2) hv[PYH - 1] = __fadd_rn(hv[PYH - 1], __fmul_rn(whr[PYH - 1][k], xw[k]));
          }
        }
        static_assert(PYV % 2 == 0, "consumer outputs are accumulated in pairs");
        if (u < nrep) {
#pragma unroll
          for (int j = 0; j < PYV; j += 2) {
            const float w0 = swv[j * PXV + t], w1 = swv[(j + 1) * PXV + t];
#pragma unroll
            for (int c = 0; c < PYH; ++c) add2_rn(cur[c][j], cur[c][j + 1], __fmul_rn(w0, hv[c]), __fmul_rn(w1, hv[c]));
          }
        }
        if (t < PXV - SXV && u >= 1) {
#pragma unroll
          for (int j = 0; j < PYV; j += 2) {
            const float w0 = swv[j * PXV + t + SXV], w1 = swv[(j + 1) * PXV + t + SXV];
#pragma unroll
            for (int c = 0; c < PYH; ++c)
              add2_rn(prev[c][j], prev[c][j + 1], __fmul_rn(w0, hv[c]), __fmul_rn(w1, hv[c]));
          }
          if (t == PXV - SXV - 1 && active) {       // rep u-1 complete: store it
            const int64_t lv = ra + u - 1;
            float* yp = y + (f * g.Sy + lv * PYV) * g.Wm + (int64_t)lh * PYH;
            if (whole && ncol == PYH) {
#pragma unroll
              for (int j = 0; j < PYV; ++j)
#pragma unroll
                for (int c = 0; c < PYH; ++c) yp[(int64_t)j * g.Wm + c] = prev[c][j];
            } else {
              const int64_t rho0 = (f * g.NLv + lv) * g.Wm + (int64_t)lh * PYH;
#pragma unroll
              for (int j = 0; j < PYV; ++j)
#pragma unroll
                for (int c = 0; c < PYH; ++c)
                  if (c < ncol && rho0 + c >= g.first && rho0 + c <= g.last) yp[(int64_t)j * g.Wm + c] = prev[c][j];
            }
          }
        }
      }
    }
    v = f * g.NLv + rb;
  }
}

static int launch_fused_stream(const FusedGeom& fg, int64_t first, int64_t count, const float* x, const float* wh,
                               const float* wv, float* y, cudaStream_t s) {
  const LineGeom &h = fg.h, &v = fg.v;
  StreamGeom g;
  g.F = v.outer;
  g.R = fg.R;
  g.W = fg.W;
  g.NLh = h.NL;
  g.NLv = v.NL;
  g.Wm = fg.Wm;
  g.Sy = v.Sy;
  g.first = first;
  g.last = first + count - 1;
  const int cw = (int)((h.NL + 31) / 32);
  const size_t smem = (size_t)FS_NST * (g.W + 8) * 4 + 2 * FS_NST * sizeof(uint64_t);
  auto kern = k_fused_stream<13, 8, 3, 14, 9, 4>;
  AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0;
  AOL_CUDA_CHECK(cudaGetDevice(&dev));
  AOL_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t nv = g.last / g.Wm - g.first / g.Wm + 1;
  const int grid = (int)(nv < sms ? nv : sms);
  kern<<<grid, (cw + 1) * 32, smem, s>>>(x, wh, wv, y, g, cw);
  AOL_LAUNCH_CHECK("k_fused_stream");
  return AOL_OK;
}

// Streaming horizontal line filter (inner == 1, the unfused H task): whole x rows (+ the
// 32-byte wrap halo) through the same bulk-copy ring; thread lh computes the PY outputs of
// repetition lh from a 16-float shared-memory window in k_line_filter's tap order.
// PX == 0 / SX == 0: taps (<= 16) and paving (a multiple of 4, >= 8) given at run time
// (`tile_filter.line_stream`: strided 1-D line filters other than the config's 13 -> 3).
template <int PX, int SX, int PY>
__global__ void __launch_bounds__(512, 1) k_hline_stream(const float* __restrict__ x, const float* __restrict__ w,
                                                         float* __restrict__ y, StreamGeom g, int n_consumer_warps,
                                                         int px_rt, int sx_rt) {
  constexpr int PXM = PX > 0 ? PX : 16;
  const int px = PX > 0 ? PX : px_rt;
  const int sx = SX > 0 ? SX : sx_rt;
  extern __shared__ __align__(128) unsigned char fs_smem[];
  const int RS = (int)g.W + 8;
  float* stages = reinterpret_cast<float*>(fs_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(fs_smem + (size_t)FS_NST * RS * 4);
  uint64_t* empty = full + FS_NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < FS_NST; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, n_consumer_warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t o_lo = g.first / g.NLh, o_hi = g.last / g.NLh + 1, no = o_hi - o_lo;
  const int64_t r0 = o_lo + no * blockIdx.x / gridDim.x, r1 = o_lo + no * (blockIdx.x + 1) / gridDim.x;
  const uint32_t row_bytes = (uint32_t)g.W * 4;
  if (warp == n_consumer_warps) {                                 // producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t o = r0; o < r1; ++o) {
        const float* src = x + o * g.W;
        mbar_wait(empty + stage, phase ^ 1);
        mbar_expect_tx(full + stage, row_bytes + 32);
        float* dst = stages + (size_t)stage * RS;
        bulk_load(dst, src, row_bytes, full + stage);
        bulk_load(dst + g.W, src, 32, full + stage);
        if (++stage == FS_NST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int lh = threadIdx.x;
  const bool active = lh < g.NLh;
  const uint32_t win = (uint32_t)(sx * (active ? lh : 0)) * 4;
  float wr[PY][PXM];
#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int t = 0; t < PXM; ++t) wr[j][t] = t < px ? w[j * px + t] : 0.0f;
  const uint32_t stage0 = smem_u32(stages), stage_bytes = (uint32_t)RS * 4;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t o = r0; o < r1; ++o) {
    mbar_wait(full + stage, phase);
    float xw[16];
    const uint32_t a = stage0 + (uint32_t)stage * stage_bytes + win;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float4 q;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                   : "r"(a + 16 * e));
      xw[4 * e] = q.x; xw[4 * e + 1] = q.y; xw[4 * e + 2] = q.z; xw[4 * e + 3] = q.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stage);
    if (++stage == FS_NST) {
      stage = 0;
      phase ^= 1;
    }
    float hv[PY];
#pragma unroll
    for (int c = 0; c < PY; ++c) hv[c] = 0.0f;
#pragma unroll
    for (int k = 0; k < PXM; ++k) {
      if (PX == 0 && k >= px) break;
#pragma unroll
      for (int c = 0; c + 1 < PY; c += 2)
        add2_rn(hv[c], hv[c + 1], __fmul_rn(wr[c][k], xw[k]), __fmul_rn(wr[c + 1][k], xw[k]));
      if (PY % 2) hv[PY - 1] = __fadd_rn(hv[PY - 1], __fmul_rn(wr[PY - 1][k], xw[k]));
    }
    const int64_t rho = o * g.NLh + lh;
    if (active && rho >= g.first && rho <= g.last) {
      float* yp = y + o * g.Wm + (int64_t)lh * PY;
#pragma unroll
      for (int c = 0; c < PY; ++c) yp[c] = hv[c];
    }
  }
}

// the unfused streaming forms (H: 13 taps paving 8 -> 3; V: 14 taps paving 9 -> 4)
static bool hline_stream_ok(const LineGeom& g) {
  if (getenv("AOL_LINE_CLASSIC")) return false;
  return g.inner == 1 && g.px == 13 && g.sx == 8 && g.py == 3 && g.sy == 3 && g.ox == 0 && g.oy == 0 &&
         g.NL * g.sx == g.Sx && g.NL * g.sy == g.Sy && g.Sx % 4 == 0 && g.NL <= 15 * 32 &&
         (size_t)FS_NST * (g.Sx + 8) * 4 + 256 <= 200 * 1024;
}

// other strided 1-D line filters through the same ring: 16 B-aligned windows of <= 16 taps whose
// overhang past the row end fits the 8-float wrap halo
static bool hline_stream_any_ok(const LineGeom& g) {
  if (getenv("AOL_LINE_CLASSIC") || hline_stream_ok(g)) return false;
  return g.inner == 1 && g.sx % 4 == 0 && g.sx >= 8 && g.px <= 16 && g.px <= g.sx + 8 && g.py >= 1 && g.py <= 4 &&
         g.sy == g.py && g.ox == 0 && g.oy == 0 && g.NL * g.sx == g.Sx && g.NL * g.sy == g.Sy && g.Sx % 4 == 0 &&
         g.NL <= 15 * 32 && (size_t)FS_NST * (g.Sx + 8) * 4 + 256 <= 200 * 1024;
}

static bool vline_stream_ok(const LineGeom& g) {
  if (getenv("AOL_LINE_CLASSIC")) return false;
  return g.inner > 1 && g.px == 14 && g.sx == 9 && g.py == 4 && g.sy == 4 && g.ox == 0 && g.oy == 0 &&
         g.inner % 4 == 0 && (g.inner + 2) / 3 <= 15 * 32 && (size_t)FS_NST * g.inner * 4 + 256 <= 200 * 1024;
}

static int launch_line_stream(const LineGeom& lg, int64_t first, int64_t count, const float* x, const float* w,
                              float* y, cudaStream_t s) {
  StreamGeom g;
  g.first = first;
  g.last = first + count - 1;
  int dev = 0, sms = 0;
  AOL_CUDA_CHECK(cudaGetDevice(&dev));
  AOL_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (lg.inner == 1) {
    g.F = lg.outer;
    g.R = 1;
    g.W = lg.Sx;
    g.NLh = lg.NL;
    g.NLv = 1;
    g.Wm = lg.Sy;
    g.Sy = lg.Sy;
    const int cw = (int)((lg.NL + 31) / 32);
    const size_t smem = (size_t)FS_NST * (g.W + 8) * 4 + 2 * FS_NST * sizeof(uint64_t);
    auto kern = hline_stream_ok(lg) ? k_hline_stream<13, 8, 3>
                : lg.py == 1 ? k_hline_stream<0, 0, 1> : lg.py == 2 ? k_hline_stream<0, 0, 2>
                : lg.py == 3 ? k_hline_stream<0, 0, 3> : k_hline_stream<0, 0, 4>;
    AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t rows = g.last / g.NLh - g.first / g.NLh + 1;
    kern<<<(int)(rows < sms ? rows : sms), (cw + 1) * 32, smem, s>>>(x, w, y, g, cw, lg.px, (int)lg.sx);
    AOL_LAUNCH_CHECK("k_hline_stream");
    return AOL_OK;
  }
  g.F = lg.outer;
  g.R = lg.Sx;
  g.W = lg.inner;
  g.NLh = (lg.inner + 2) / 3;
  g.NLv = lg.NL;
  g.Wm = lg.inner;
  g.Sy = lg.Sy;
  const int cw = (int)((g.NLh + 31) / 32);
  const size_t smem = (size_t)FS_NST * g.W * 4 + 2 * FS_NST * sizeof(uint64_t);
  auto kern = k_fused_stream<13, 8, 3, 14, 9, 4, true>;
  AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t nv = g.last / g.Wm - g.first / g.Wm + 1;
  kern<<<(int)(nv < sms ? nv : sms), (cw + 1) * 32, smem, s>>>(x, nullptr, w, y, g, cw);
  AOL_LAUNCH_CHECK("k_vline_stream");
  return AOL_OK;
}

// streaming form applies: 13x3 paving 8 -> 14x4 paving 9, full rows, no origins, x rows
// 16-byte aligned and a ring of FS_NST rows fitting in shared memory
static bool fused_stream_ok(const FusedGeom& fg) {
  const LineGeom &h = fg.h, &v = fg.v;
  if (getenv("AOL_FUSED_TILE")) return false;
  return h.px == 13 && h.sx == 8 && h.py == 3 && h.sy == 3 && h.ox == 0 && h.NL * h.sx == fg.W &&
         v.px == 14 && v.sx == 9 && v.py == 4 && v.sy == 4 && v.ox == 0 && v.oy == 0 && fg.W % 4 == 0 &&
         h.NL <= 15 * 32 && (size_t)FS_NST * (fg.W + 8) * 4 + 256 <= 200 * 1024;
}

int launch_fused_line_filters(const aol_task& th, const aol_task& tv, int64_t first, int64_t count,
                              void* const* ph, void* const* pv, cudaStream_t s) {
  FusedGeom g;
  if (!fused_line_geometry(th, tv, g)) return fail(AOL_EUNSUPPORTED, "task pair is not a fusable line-filter chain");
  if (!(g.h.px == 13 && g.h.py == 3 && g.v.px == 14 && g.v.py == 4))
    return fail(AOL_EUNSUPPORTED, "fused line filters are instantiated for 13x3 -> 14x4");
  if (count <= 0) return AOL_OK;
  if (fused_stream_ok(g))
    return launch_fused_stream(g, first, count, static_cast<const float*>(ph[0]), static_cast<const float*>(ph[1]),
                               static_cast<const float*>(pv[1]), static_cast<float*>(pv[2]), s);
  const int64_t last = first + count - 1;
  const int64_t per_frame = g.v.NL * g.Wm;
  const int64_t f_lo = first / per_frame, f_hi = last / per_frame;
  const int64_t tiles_per_frame = g.tiles_i * g.tiles_l;
  const int64_t tile0 = f_lo * tiles_per_frame, ntiles = (f_hi - f_lo + 1) * tiles_per_frame;
  const size_t smem = (size_t)g.NR * g.TI * sizeof(float);
  auto kern = k_fused_line_filters<13, 3, 14, 4>;
  if (smem > 48 * 1024)
    AOL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = ntiles < (int64_t)kNumSMs * 16 ? ntiles : (int64_t)kNumSMs * 16;
  kern<<<(unsigned)grid, FZ_THREADS, smem, s>>>(static_cast<const float*>(ph[0]), static_cast<const float*>(ph[1]),
                                                static_cast<const float*>(pv[1]), static_cast<float*>(pv[2]), g, first,
                                                last, tile0, ntiles);
  AOL_LAUNCH_CHECK("k_fused_line_filters");
  return AOL_OK;
}

}  // namespace aol
