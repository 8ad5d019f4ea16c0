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
#include <cstring>

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

static_assert(sizeof(LineGeom) <= 256, "LineGeomBuf in aol_tile.cu must hold a LineGeom");

const char* line_filter_variant(const LineGeom& g) {
  if (g.px == 13 && g.py == 3) return "tile_filter.line_13x3";
  if (g.px == 14 && g.py == 4) return "tile_filter.line_14x4";
  return "tile_filter.line";
}

int launch_line_filter(const aol_task& t, const LineGeom& g, int64_t first, int64_t count, void* const* ports,
                       cudaStream_t s) {
  const float* x = static_cast<const float*>(ports[0]);
  const float* w = static_cast<const float*>(ports[1]);
  float* y = static_cast<float*>(ports[2]);
  const unsigned grid = grid_for(count, 256, 8);
  // 32-bit offsets whenever both arrays fit (every in-range offset < 2^32)
  const bool idx32 = g.outer * g.Sx * g.inner < (1ll << 32) && g.outer * g.Sy * g.inner < (1ll << 32);
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
