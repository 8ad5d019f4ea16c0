// 2-D box-pattern filter with toroidal (modulo) wrap — config C4, the `stencil` task.
//
// Recognised when the x tiler is a KHxKW box (fitting = I2, paving = I2, any
// origin) over an [H, W] array with repetition space [H, W], and the y tiler is
// the identity [H, W] -> pattern [1].  Output (r, c) =
//     sum_{di, dj} w[di*KW + dj] * x[(r + o_r + di) mod H][(c + o_c + dj) mod W]
// accumulated in pattern order (di, dj) row-major with __fmul_rn / __fadd_rn —
// the oracle's order, so results are bit-exact.
//
// Register tiling: a thread owns a 4-row x 4-column output block; it loads the
// (4+KH-1) input rows once as float4 (+ KW-1 neighbour columns), so each input
// element is fetched ~1.1 times from L1 instead of KH*KW times.  Rows wrap by a
// per-row modulo computed once; columns wrap only in the two neighbour loads.
#include <cstdlib>

#include "aol_common.cuh"

namespace aol {

constexpr int ST_TX = 32, ST_TY = 4;       // threads
constexpr int ST_RPT = 8, ST_CPT = 4;      // outputs per thread: rows, cols
constexpr int ST_ROWS = ST_TY * ST_RPT;    // 32 output rows per CTA
constexpr int ST_COLS = ST_TX * ST_CPT;    // 128 output cols per CTA

template <int KH, int KW>
__global__ void __launch_bounds__(ST_TX* ST_TY) k_stencil_box(const float* __restrict__ x, const float* __restrict__ w,
                                                              float* __restrict__ y, int H, int W, int orow,
                                                              int ocol, int64_t first, int64_t last) {
  static_assert(KW == 3, "column neighbour scheme assumes KW == 3");
  __shared__ float ws[KH * KW];
  if (threadIdx.x + threadIdx.y * ST_TX < KH * KW) ws[threadIdx.x + threadIdx.y * ST_TX] = w[threadIdx.x + threadIdx.y * ST_TX];
  __syncthreads();
  const int r0 = blockIdx.y * ST_ROWS + threadIdx.y * ST_RPT;
  const int c0 = blockIdx.x * ST_COLS + threadIdx.x * ST_CPT;
  if (r0 >= H || c0 >= W) return;
  // input column of the window centre (dj = 1) for output column c0, wrapped
  const int cin = (int)(((int64_t)c0 + ocol + 1) % W);
  const int cl = cin == 0 ? W - 1 : cin - 1;        // left neighbour of the float4
  const int cr = (cin + ST_CPT) % W;                 // right neighbour
  const bool vec = (cin % 4 == 0) && (cin + ST_CPT <= W) && (W % 4 == 0);
  float acc[ST_RPT][ST_CPT];
#pragma unroll
  for (int i = 0; i < ST_RPT; ++i)
#pragma unroll
    for (int j = 0; j < ST_CPT; ++j) acc[i][j] = 0.0f;
  // load the whole (ST_RPT + KH - 1) x (ST_CPT + 2) input block first: every load is
  // independent, so a thread keeps ~3*(ST_RPT+KH-1) requests in flight
  float v[ST_RPT + KH - 1][ST_CPT + 2];
#pragma unroll
  for (int rr = 0; rr < ST_RPT + KH - 1; ++rr) {
    int row = r0 + orow + rr;
    if (row >= H) row -= H;
    if (row >= H) row %= H;
    const float* xr = x + (int64_t)row * W;
    v[rr][0] = __ldg(xr + cl);
    if (vec) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(xr + cin));
      v[rr][1] = q.x; v[rr][2] = q.y; v[rr][3] = q.z; v[rr][4] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < ST_CPT; ++j) v[rr][1 + j] = __ldg(xr + (cin + j) % W);
    }
    v[rr][ST_CPT + 1] = __ldg(xr + cr);
  }
#pragma unroll
  for (int i = 0; i < ST_RPT; ++i)
#pragma unroll
    for (int di = 0; di < KH; ++di)
#pragma unroll
      for (int j = 0; j < ST_CPT; ++j)
#pragma unroll
        for (int dj = 0; dj < KW; ++dj)
          acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(ws[di * KW + dj], v[i + di][j + dj]));
  // accumulation order per output: di-major, dj-minor = the pattern's row-major order
#pragma unroll
  for (int i = 0; i < ST_RPT; ++i) {
    const int r = r0 + i;
    if (r >= H) break;
    float* yr = y + (int64_t)r * W;
    const int64_t lin = (int64_t)r * W + c0;
    if (lin >= first && lin + ST_CPT - 1 <= last && c0 + ST_CPT <= W && (W % 4 == 0)) {
      *reinterpret_cast<float4*>(yr + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < ST_CPT; ++j)
        if (c0 + j < W && lin + j >= first && lin + j <= last) yr[c0 + j] = acc[i][j];
    }
  }
}

// (a0, a1) += (p0, p1), one packed IEEE round-to-nearest add per lane (products stay
// scalar __fmul_rn: ptxas would contract a packed mul into the packed add).
__device__ __forceinline__ void st_add2(float& a0, float& a1, float p0, float p1) {
  asm("{\n\t.reg .b64 ra, rp;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rp, {%2, %3};\n\t"
      "add.rn.f32x2 ra, ra, rp;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(p0), "f"(p1));
}

// Fast form (the common case: W % 4 == 0 and the window centre column of every float4 is
// 16-byte aligned): a thread owns 4 columns and slides a KH-row register window down
// SV_RPT output rows -- each input row is loaded once per strip (float4 + two neighbour
// scalars), the KH-1 halo rows once per SV_RPT rows.  Same tap order as k_stencil_box.
constexpr int SV_TX = 128, SV_RPT = 16;

template <int KH>
__global__ void __launch_bounds__(SV_TX) k_stencil_slide(const float* __restrict__ x, const float* __restrict__ w,
                                                         float* __restrict__ y, int H, int W, int orow, int ocol,
                                                         int rows, int64_t first, int64_t last) {
  float wr[KH * 3];
#pragma unroll
  for (int k = 0; k < KH * 3; ++k) wr[k] = __ldg(w + k);
  const int c0 = (blockIdx.x * SV_TX + threadIdx.x) * 4;
  const int r0 = blockIdx.y * SV_RPT;
  if (c0 >= W || r0 >= rows) return;
  int cin = c0 + ocol + 1;                              // window centre of column c0 (dj = 1)
  if (cin >= W) cin -= W;
  const int cl = cin == 0 ? W - 1 : cin - 1;
  const int cr = cin + 4 == W ? 0 : cin + 4;
  int row = r0 + orow;                                  // input row of tap di = 0
  if (row >= H) row -= H;
  // every window load is issued before any arithmetic: (SV_RPT + KH - 1) rows x 3 requests
  // in flight per thread
  float v[SV_RPT + KH - 1][6];
#pragma unroll
  for (int rr = 0; rr < SV_RPT + KH - 1; ++rr) {
    const float* xr = x + (size_t)row * (size_t)W;
    const float4 q = __ldg(reinterpret_cast<const float4*>(xr + cin));
    v[rr][0] = __ldg(xr + cl);
    v[rr][1] = q.x; v[rr][2] = q.y; v[rr][3] = q.z; v[rr][4] = q.w;
    v[rr][5] = __ldg(xr + cr);
    if (++row == H) row = 0;
  }
  const bool whole = (int64_t)r0 * W + c0 >= first && (int64_t)(r0 + SV_RPT - 1) * W + c0 + 3 <= last &&
                     r0 + SV_RPT <= rows;
#pragma unroll
  for (int i = 0; i < SV_RPT; ++i) {
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
    for (int di = 0; di < KH; ++di) {
      const float* vr = v[i + di];
#pragma unroll
      for (int dj = 0; dj < 3; ++dj) {
        const float wt = wr[di * 3 + dj];
        st_add2(a0, a1, __fmul_rn(wt, vr[dj]), __fmul_rn(wt, vr[dj + 1]));
        st_add2(a2, a3, __fmul_rn(wt, vr[dj + 2]), __fmul_rn(wt, vr[dj + 3]));
      }
    }
    const int r = r0 + i;
    float* yr = y + (size_t)r * (size_t)W + c0;
    if (whole) {
      *reinterpret_cast<float4*>(yr) = make_float4(a0, a1, a2, a3);
    } else if (r < rows) {
      const int64_t lin = (int64_t)r * W + c0;
      const float a[4] = {a0, a1, a2, a3};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lin + j >= first && lin + j <= last) yr[j] = a[j];
    }
  }
}

// Wider windows (KW = 5 or 7, any KH in {3, 5, 7}; the window centre column 16-byte aligned):
// a thread still owns 4 columns, but each input row arrives as three float4s -- the aligned
// quads left of, at and right of the centre -- of which the KW/2 innermost neighbours on
// each side are kept.  RPT output rows per thread with every window load issued before any
// arithmetic; the same tap order (di-major, dj-minor) and rounding as every other form.
template <int KH, int KW, int RPT>
__global__ void __launch_bounds__(SV_TX) k_stencil_slide_wide(const float* __restrict__ x,
                                                              const float* __restrict__ w, float* __restrict__ y,
                                                              int H, int W, int orow, int ocol, int rows,
                                                              int64_t first, int64_t last) {
  constexpr int HW = KW / 2;
  static_assert(KW % 2 == 1 && HW >= 1 && HW <= 4, "odd window widths 3..9");
  float wr[KH * KW];
#pragma unroll
  for (int k = 0; k < KH * KW; ++k) wr[k] = __ldg(w + k);
  const int c0 = (blockIdx.x * SV_TX + threadIdx.x) * 4;
  const int r0 = blockIdx.y * RPT;
  if (c0 >= W || r0 >= rows) return;
  const int cin = (int)(((int64_t)c0 + ocol + HW) % W);   // window centre of column c0, aligned
  const int cl4 = cin >= 4 ? cin - 4 : cin - 4 + W;        // aligned quads either side
  const int cr4 = cin + 4 >= W ? cin + 4 - W : cin + 4;
  int row = (int)(((int64_t)r0 + orow) % H);
  float v[RPT + KH - 1][4 + 2 * HW];
#pragma unroll
  for (int rr = 0; rr < RPT + KH - 1; ++rr) {
    const float* xr = x + (size_t)row * (size_t)W;
    const float4 l = __ldg(reinterpret_cast<const float4*>(xr + cl4));
    const float4 c = __ldg(reinterpret_cast<const float4*>(xr + cin));
    const float4 r = __ldg(reinterpret_cast<const float4*>(xr + cr4));
    const float lq[4] = {l.x, l.y, l.z, l.w}, rq[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int k = 0; k < HW; ++k) {
      v[rr][k] = lq[4 - HW + k];
      v[rr][HW + 4 + k] = rq[k];
    }
    v[rr][HW] = c.x; v[rr][HW + 1] = c.y; v[rr][HW + 2] = c.z; v[rr][HW + 3] = c.w;
    if (++row == H) row = 0;
  }
  const bool whole = (int64_t)r0 * W + c0 >= first && (int64_t)(r0 + RPT - 1) * W + c0 + 3 <= last &&
                     r0 + RPT <= rows;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
    for (int di = 0; di < KH; ++di) {
      const float* vr = v[i + di];
#pragma unroll
      for (int dj = 0; dj < KW; ++dj) {
        const float wt = wr[di * KW + dj];
        st_add2(a0, a1, __fmul_rn(wt, vr[dj]), __fmul_rn(wt, vr[dj + 1]));
        st_add2(a2, a3, __fmul_rn(wt, vr[dj + 2]), __fmul_rn(wt, vr[dj + 3]));
      }
    }
    const int r = r0 + i;
    float* yr = y + (size_t)r * (size_t)W + c0;
    if (whole) {
      *reinterpret_cast<float4*>(yr) = make_float4(a0, a1, a2, a3);
    } else if (r < rows) {
      const int64_t lin = (int64_t)r * W + c0;
      const float a[4] = {a0, a1, a2, a3};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lin + j >= first && lin + j <= last) yr[j] = a[j];
    }
  }
}

// Recognise the box-stencil tiler pair; returns false when the generic kernel must run.
bool stencil_box_applicable(const aol_task& t, int& KH, int& KW) {
  const aol_tiler &tx = t.tilers[0], &ty = t.tilers[1];
  if (t.dtype != AOL_F32) return false;
  if (tx.arr_rank != 2 || tx.rep_rank != 2 || tx.pat_rank != 2) return false;
  if (ty.arr_rank != 2 || ty.rep_rank != 2) return false;
  if (tx.array[0] != tx.rep[0] || tx.array[1] != tx.rep[1]) return false;
  if (ty.array[0] != tx.array[0] || ty.array[1] != tx.array[1]) return false;
  if (tx.paving[0][0] != 1 || tx.paving[0][1] != 0 || tx.paving[1][0] != 0 || tx.paving[1][1] != 1) return false;
  if (tx.fitting[0][0] != 1 || tx.fitting[0][1] != 0 || tx.fitting[1][0] != 0 || tx.fitting[1][1] != 1) return false;
  if (ty.paving[0][0] != 1 || ty.paving[0][1] != 0 || ty.paving[1][0] != 0 || ty.paving[1][1] != 1) return false;
  for (int k = 0; k < ty.pat_rank; ++k)
    if (ty.pattern[k] != 1) return false;
  if (ty.origin[0] % ty.array[0] != 0 || ty.origin[1] % ty.array[1] != 0) return false;
  KH = (int)tx.pattern[0];
  KW = (int)tx.pattern[1];
  if (!(KH == 3 || KH == 5 || KH == 7) || !(KW == 3 || KW == 5 || KW == 7)) return false;
  if (tx.array[0] >= (1ll << 31) || tx.array[1] >= (1ll << 31)) return false;
  if (KW != 3) {                     // wide windows: only the aligned quad form exists
    const int64_t W = tx.array[1];
    const int64_t oc = ((tx.origin[1] % W) + W) % W;
    if (W % 4 || (oc + KW / 2) % W % 4 || W < 8) return false;
  }
  return true;
}

int launch_stencil_box(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s) {
  int KH, KW;
  if (!stencil_box_applicable(t, KH, KW)) return fail(AOL_EUNSUPPORTED, "not a box stencil");
  const aol_tiler& tx = t.tilers[0];
  const int H = (int)tx.array[0], W = (int)tx.array[1];
  auto emod = [](int64_t v, int64_t m) { int64_t r = v % m; return r < 0 ? r + m : r; };
  const int orow = (int)emod(tx.origin[0], H), ocol = (int)emod(tx.origin[1], W);
  const int64_t last = first + count - 1;
  const int rlo = (int)(first / W), rhi = (int)(last / W);
  dim3 block(ST_TX, ST_TY);
  dim3 grid((W + ST_COLS - 1) / ST_COLS, (rhi - rlo + ST_ROWS) / ST_ROWS);
  // launch over rows [rlo, rhi]: shift the row origin so blockIdx.y = 0 starts at rlo
  const float* x = static_cast<const float*>(ports[0]);
  const float* w = static_cast<const float*>(ports[1]);
  float* y = static_cast<float*>(ports[2]) + (int64_t)rlo * W;
  const int orow_shift = (int)emod((int64_t)orow + rlo, H);
  const int64_t f2 = first - (int64_t)rlo * W, l2 = last - (int64_t)rlo * W;
  const int Hrows = rhi - rlo + 1;
  // rows are addressed relative to rlo for the output; the input row is (r + rlo + orow) mod H
  const int cshift = (int)emod((int64_t)ocol + 1, W);
  if (KW != 3) {
    // (applicability guaranteed W % 4 == 0 and an aligned window centre)
    constexpr int RPT = 8;                 // measured: 16 rows per thread is slower (registers)
    dim3 g3((W / 4 + SV_TX - 1) / SV_TX, (Hrows + RPT - 1) / RPT);
    void (*k)(const float*, const float*, float*, int, int, int, int, int, int64_t, int64_t) =
        KW == 5 ? (KH == 3 ? k_stencil_slide_wide<3, 5, RPT> : KH == 5 ? k_stencil_slide_wide<5, 5, RPT>
                                                                        : k_stencil_slide_wide<7, 5, RPT>)
                : (KH == 3 ? k_stencil_slide_wide<3, 7, RPT> : KH == 5 ? k_stencil_slide_wide<5, 7, RPT>
                                                                        : k_stencil_slide_wide<7, 7, RPT>);
    k<<<g3, SV_TX, 0, s>>>(x, w, y, H, W, orow_shift, ocol, Hrows, f2, l2);
    AOL_LAUNCH_CHECK("k_stencil_slide_wide");
    return AOL_OK;
  }
  if (W % 4 == 0 && cshift % 4 == 0 && !getenv("AOL_STENCIL_BOX") && KH != 7) {
    dim3 g2((W / 4 + SV_TX - 1) / SV_TX, (Hrows + SV_RPT - 1) / SV_RPT);
    if (KH == 3)
      k_stencil_slide<3><<<g2, SV_TX, 0, s>>>(x, w, y, H, W, orow_shift, ocol, Hrows, f2, l2);
    else
      k_stencil_slide<5><<<g2, SV_TX, 0, s>>>(x, w, y, H, W, orow_shift, ocol, Hrows, f2, l2);
    AOL_LAUNCH_CHECK("k_stencil_slide");
    return AOL_OK;
  }
  if (KH == 3)
    k_stencil_box<3, 3><<<grid, block, 0, s>>>(x, w, y, H, W, orow_shift, ocol, f2, l2);
  else if (KH == 5)
    k_stencil_box<5, 3><<<grid, block, 0, s>>>(x, w, y, H, W, orow_shift, ocol, f2, l2);
  else
    k_stencil_box<7, 3><<<grid, block, 0, s>>>(x, w, y, H, W, orow_shift, ocol, f2, l2);
  (void)Hrows;
  AOL_LAUNCH_CHECK("k_stencil_box");
  return AOL_OK;
}

// Block pooling / decimating 2-D filters: x tiler = a KH x KW box (fitting I2) paved by its
// own size (paving diag(KH, KW)), origin 0, over [H, W] with repetition space [H/KH, W/KW];
// y the identity over [H/KH, W/KW].  Output (r, c) = sum_{di, dj} w[di*KW + dj] *
// x[r*KH + di][c*KW + dj], taps row-major (bit-exact).  A thread owns 4 consecutive outputs
// of one row: KH input rows x 4*KW contiguous floats as float4s, one float4 store.
template <int KH, int KW>
__global__ void __launch_bounds__(256) k_box_pool(const float* __restrict__ x, const float* __restrict__ w,
                                                  float* __restrict__ y, int64_t Ho, int64_t Wo, int64_t W,
                                                  int64_t first, int64_t last) {
  float wr[KH * KW];
#pragma unroll
  for (int k = 0; k < KH * KW; ++k) wr[k] = __ldg(w + k);
  const int64_t q0 = first / 4, q1 = last / 4;                    // quads of outputs in range
  const int64_t wq = Wo / 4;                                      // quads per output row (Wo % 4 == 0)
  for (int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= q1;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / wq, c0 = (q - r * wq) * 4;
    float v[KH][4 * KW];
#pragma unroll
    for (int di = 0; di < KH; ++di) {
      const float4* xr = reinterpret_cast<const float4*>(x + (r * KH + di) * W + c0 * KW);
#pragma unroll
      for (int e = 0; e < KW; ++e) {
        const float4 t4 = __ldg(xr + e);
        v[di][4 * e] = t4.x; v[di][4 * e + 1] = t4.y; v[di][4 * e + 2] = t4.z; v[di][4 * e + 3] = t4.w;
      }
    }
    float a[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float acc = 0.0f;
#pragma unroll
      for (int di = 0; di < KH; ++di)
#pragma unroll
        for (int dj = 0; dj < KW; ++dj) acc = __fadd_rn(acc, __fmul_rn(wr[di * KW + dj], v[di][j * KW + dj]));
      a[j] = acc;
    }
    const int64_t lin = r * Wo + c0;
    float* yp = y + lin;
    if (lin >= first && lin + 3 <= last) {
      *reinterpret_cast<float4*>(yp) = make_float4(a[0], a[1], a[2], a[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (lin + j >= first && lin + j <= last) yp[j] = a[j];
    }
  }
}

bool box_pool_applicable(const aol_task& t, int& KH, int& KW) {
  const aol_tiler &tx = t.tilers[0], &ty = t.tilers[1];
  if (t.dtype != AOL_F32) return false;
  if (tx.arr_rank != 2 || tx.rep_rank != 2 || tx.pat_rank != 2 || ty.arr_rank != 2 || ty.rep_rank != 2) return false;
  KH = (int)tx.pattern[0];
  KW = (int)tx.pattern[1];
  if (KH < 1 || KH > 4 || KW < 1 || KW > 4 || KH * KW < 2) return false;
  if (tx.paving[0][0] != KH || tx.paving[0][1] != 0 || tx.paving[1][0] != 0 || tx.paving[1][1] != KW) return false;
  if (tx.fitting[0][0] != 1 || tx.fitting[0][1] != 0 || tx.fitting[1][0] != 0 || tx.fitting[1][1] != 1) return false;
  if (tx.origin[0] % tx.array[0] != 0 || tx.origin[1] % tx.array[1] != 0) return false;
  const int64_t Ho = tx.rep[0], Wo = tx.rep[1];
  if (tx.array[0] != Ho * KH || tx.array[1] != Wo * KW) return false;
  if (ty.array[0] != Ho || ty.array[1] != Wo || ty.rep[0] != Ho || ty.rep[1] != Wo) return false;
  if (ty.paving[0][0] != 1 || ty.paving[0][1] != 0 || ty.paving[1][0] != 0 || ty.paving[1][1] != 1) return false;
  for (int k = 0; k < ty.pat_rank; ++k)
    if (ty.pattern[k] != 1) return false;
  if (ty.origin[0] % ty.array[0] != 0 || ty.origin[1] % ty.array[1] != 0) return false;
  return Wo % 4 == 0;                                    // float4 quads of outputs, 16 B input rows
}

int launch_box_pool(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s) {
  int KH, KW;
  if (!box_pool_applicable(t, KH, KW)) return fail(AOL_EUNSUPPORTED, "not a block pooling filter");
  const aol_tiler& tx = t.tilers[0];
  const float* x = static_cast<const float*>(ports[0]);
  const float* w = static_cast<const float*>(ports[1]);
  float* y = static_cast<float*>(ports[2]);
  if ((uintptr_t)x % 16 || (uintptr_t)y % 16) return fail(AOL_EUNSUPPORTED, "unaligned pooling ports");
  const int64_t Ho = tx.rep[0], Wo = tx.rep[1], W = tx.array[1];
  const int64_t last = first + count - 1;
  const int64_t quads = last / 4 - first / 4 + 1;
  const unsigned grid = (unsigned)std::min<int64_t>((quads + 255) / 256, (int64_t)kNumSMs * 16);
  void (*k)(const float*, const float*, float*, int64_t, int64_t, int64_t, int64_t, int64_t) = nullptr;
#define AOL_POOL(a, b) if (KH == a && KW == b) k = k_box_pool<a, b>;
  AOL_POOL(1, 2) AOL_POOL(1, 3) AOL_POOL(1, 4) AOL_POOL(2, 1) AOL_POOL(2, 2) AOL_POOL(2, 3) AOL_POOL(2, 4)
  AOL_POOL(3, 1) AOL_POOL(3, 2) AOL_POOL(3, 3) AOL_POOL(3, 4) AOL_POOL(4, 1) AOL_POOL(4, 2) AOL_POOL(4, 3)
  AOL_POOL(4, 4)
#undef AOL_POOL
  k<<<grid, 256, 0, s>>>(x, w, y, Ho, Wo, W, first, last);
  AOL_LAUNCH_CHECK("k_box_pool");
  return AOL_OK;
}

}  // namespace aol
