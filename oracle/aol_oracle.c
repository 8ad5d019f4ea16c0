/*
 * CPU ORACLE (C restatement) — TEST INFRASTRUCTURE ONLY.
 *
 * Same semantics as oracle/aol_oracle.py (whose header lists the reference
 * file:line it restates): the Array-OL tiler index function (SURVEY.md
 * Appendix A) and the tile intrinsics, accumulating in pattern order with
 * the product and the sum rounded separately (the order of the reference's
 * spmv_csr executor, refexec.py:111-121).  Built with -ffp-contract=off so
 * the compiler never fuses a*b+c.  Used only by tests/ (large-size checks)
 * and by bench.py's CPU-baseline / `--impl reference` legs; never by the
 * product package.  OpenMP parallelises over repetitions (results do not
 * depend on the thread count).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define R4 4

typedef struct orc_tiler {
  int32_t arr_rank, rep_rank, pat_rank, reserved;
  int64_t array[R4], rep[R4], pattern[R4], origin[R4];
  int64_t paving[R4][R4], fitting[R4][R4];
} orc_tiler;

static int64_t emod(int64_t v, int64_t m) {
  int64_t r = v % m;
  return r < 0 ? r + m : r;
}

static int64_t total(const int64_t* v, int n) {
  int64_t t = 1;
  for (int i = 0; i < n; ++i) t *= v[i];
  return t;
}

/* off(rho, iota): unravel rho over rep and iota over pattern (row-major), then
 * e_d = (o_d + P_d.r + F_d.i) mod s_d and off = sum_d e_d * stride_d. */
static int64_t offset(const orc_tiler* t, int64_t rho, int64_t iota) {
  int64_t r[R4] = {0}, i[R4] = {0};
  for (int j = t->rep_rank - 1; j >= 0; --j) {
    r[j] = rho % t->rep[j];
    rho /= t->rep[j];
  }
  for (int k = t->pat_rank - 1; k >= 0; --k) {
    i[k] = iota % t->pattern[k];
    iota /= t->pattern[k];
  }
  int64_t off = 0, stride = 1;
  for (int d = t->arr_rank - 1; d >= 0; --d) {
    int64_t e = t->origin[d];
    for (int j = 0; j < t->rep_rank; ++j) e += t->paving[d][j] * r[j];
    for (int k = 0; k < t->pat_rank; ++k) e += t->fitting[d][k] * i[k];
    off += emod(e, t->array[d]) * stride;
    stride *= t->array[d];
  }
  return off;
}

int orc_threads(void) {
#ifdef _OPENMP
  int n = 1;
#pragma omp parallel
  {
#pragma omp single
    n = omp_get_num_threads();
  }
  return n;
#else
  return 1;
#endif
}

void orc_tiler_offsets(const orc_tiler* t, int64_t first, int64_t count, int64_t* out) {
  const int64_t P = total(t->pattern, t->pat_rank);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e)
    for (int64_t k = 0; k < P; ++k) out[e * P + k] = offset(t, first + e, k);
}

/* element size 4 or 8: bit moves */
void orc_tile_copy(const void* src, void* dst, int esize, const orc_tiler* ts, const orc_tiler* td, int64_t first,
                   int64_t count) {
  const int64_t P = total(ts->pattern, ts->pat_rank);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e)
    for (int64_t k = 0; k < P; ++k) {
      const int64_t so = offset(ts, first + e, k), dof = offset(td, first + e, k);
      if (esize == 4) ((uint32_t*)dst)[dof] = ((const uint32_t*)src)[so];
      else ((uint64_t*)dst)[dof] = ((const uint64_t*)src)[so];
    }
}

void orc_matmul_f32(const float* a, const float* b, float* c, const orc_tiler* ta, const orc_tiler* tb,
                    const orc_tiler* tc, int64_t first, int64_t count) {
  const int64_t K = total(ta->pattern, ta->pat_rank);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e) {
    float acc = 0.0f;
    for (int64_t k = 0; k < K; ++k) {
      const float p = a[offset(ta, first + e, k)] * b[offset(tb, first + e, k)];
      acc = acc + p;
    }
    c[offset(tc, first + e, 0)] = acc;
  }
}

/* Canonical row-major GEMM rows [row_lo, row_hi): the same k-ascending,
 * mul-then-add order as orc_matmul_f32, vectorised across the columns. */
void orc_gemm_rows_f32(const float* A, const float* B, float* C, int64_t N, int64_t K, int64_t row_lo,
                       int64_t row_hi) {
#pragma omp parallel for schedule(static)
  for (int64_t i = row_lo; i < row_hi; ++i) {
    float* crow = C + i * N;
    for (int64_t j = 0; j < N; ++j) crow[j] = 0.0f;
    for (int64_t k = 0; k < K; ++k) {
      const float aik = A[i * K + k];
      const float* brow = B + k * N;
      for (int64_t j = 0; j < N; ++j) {
        const float p = aik * brow[j];
        crow[j] = crow[j] + p;
      }
    }
  }
}

void orc_filter_f32(const float* x, const float* w, float* y, const orc_tiler* tx, const orc_tiler* ty,
                    int64_t first, int64_t count) {
  const int64_t px = total(tx->pattern, tx->pat_rank), py = total(ty->pattern, ty->pat_rank);
#pragma omp parallel
  {
    float* xs = (float*)malloc(sizeof(float) * (size_t)px);
#pragma omp for schedule(static)
    for (int64_t e = 0; e < count; ++e) {
      for (int64_t i = 0; i < px; ++i) xs[i] = x[offset(tx, first + e, i)];
      for (int64_t j = 0; j < py; ++j) {
        float acc = 0.0f;
        for (int64_t i = 0; i < px; ++i) {
          const float p = w[j * px + i] * xs[i];
          acc = acc + p;
        }
        y[offset(ty, first + e, j)] = acc;
      }
    }
    free(xs);
  }
}

/* Toroidal 3x3 stencil rows [row_lo, row_hi) of an H x W grid, pattern order
 * (di, dj) row-major from (-1,-1): the stencil task of config C4 written out. */
void orc_stencil3x3_rows_f32(const float* x, const float* w, float* y, int64_t H, int64_t W, int64_t row_lo,
                             int64_t row_hi) {
#pragma omp parallel for schedule(static)
  for (int64_t r = row_lo; r < row_hi; ++r) {
    for (int64_t c = 0; c < W; ++c) {
      float acc = 0.0f;
      for (int di = 0; di < 3; ++di) {
        const int64_t rr = emod(r + di - 1, H);
        for (int dj = 0; dj < 3; ++dj) {
          const int64_t cc = emod(c + dj - 1, W);
          const float p = w[di * 3 + dj] * x[rr * W + cc];
          acc = acc + p;
        }
      }
      y[r * W + c] = acc;
    }
  }
}
