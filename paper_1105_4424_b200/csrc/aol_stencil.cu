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
  if (KW != 3 || !(KH == 3 || KH == 5)) return false;
  if (tx.array[0] >= (1ll << 31) || tx.array[1] >= (1ll << 31)) return false;
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
  if (KH == 3)
    k_stencil_box<3, 3><<<grid, block, 0, s>>>(x, w, y, H, W, orow_shift, ocol, f2, l2);
  else
    k_stencil_box<5, 3><<<grid, block, 0, s>>>(x, w, y, H, W, orow_shift, ocol, f2, l2);
  (void)Hrows;
  AOL_LAUNCH_CHECK("k_stencil_box");
  return AOL_OK;
}

}  // namespace aol
