// extern "C" surface of libaolb200.so (include/aol_b200.h): validation + kernel dispatch.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "aol_common.cuh"

namespace aol {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return AOL_ECUDA;
}
void count_launch(int n) { g_launches += n; }

// defined in the kernel translation units
int launch_tiler_offsets(const aol_tiler& t, int64_t first, int64_t count, int64_t* out, cudaStream_t s);
int launch_tile_copy(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
const char* tile_sum_plan_name(const aol_task& t);
const char* tile_copy_plan_name(const aol_tiler& ts, const aol_tiler& td, int64_t first, int64_t count,
                                size_t esz, void* const* ports);
int launch_matmul_generic(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
int launch_filter_generic(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
const char* filter_plan_name(const aol_task& t);
int launch_tile_sum(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
int launch_identity(const aol_task& t, int64_t first, int64_t count, void* const* ports, const double* scalars,
                    cudaStream_t s);
bool gemm_tf32_applicable(const aol_task& t, void* const* ports);
bool gemm_batched_applicable(const aol_task& t, void* const* ports);
bool recognise_gemm_strides(const aol_task& t);
int launch_gemm_exact(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
int launch_gemm_exact_batched(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
bool gemm_exact_batched_applicable(const aol_task& t);
int launch_gemm_batched(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
int launch_fused_line_filters(const aol_task& th, const aol_task& tv, int64_t first, int64_t count,
                              void* const* ph, void* const* pv, cudaStream_t s);
int launch_gemm_tf32(const aol_task& t, int64_t first, int64_t count, void* const* ports, cudaStream_t s);
int release_dot_scratch();
int release_loop_scratch();
int release_gemm_scratch();

static int tilers_needed(int op) {
  switch (op) {
    case AOL_OP_TILE_COPY: return 2;
    case AOL_OP_MATMUL: return 3;
    case AOL_OP_TILE_FILTER: return 2;
    case AOL_OP_TILE_SUM: return 2;
    default: return 0;
  }
}

static int validate(const aol_task* t) {
  if (!t) return fail(AOL_EINVAL, "null task");
  if (t->dtype < AOL_F32 || t->dtype > AOL_I64) return fail(AOL_EINVAL, "bad dtype");
  const int need = tilers_needed(t->op);
  const bool ident = t->op >= AOL_OP_COPY && t->op <= AOL_OP_SCALAR_SEQ;
  if (!ident && need == 0) return fail(AOL_EUNSUPPORTED, "unknown op " + std::to_string(t->op));
  if (t->n_tilers != need) return fail(AOL_EINVAL, "op needs " + std::to_string(need) + " tilers");
  if (need) {
    DevTiler tmp;
    int64_t R = -1;
    for (int i = 0; i < need; ++i) {
      int rc = make_dev_tiler(t->tilers[i], tmp);
      if (rc) return rc;
      const int64_t r = tiler_rep_total(t->tilers[i]);
      if (R >= 0 && r != R) return fail(AOL_EINVAL, "tilers disagree on the repetition space");
      R = r;
    }
    const bool flt = t->dtype == AOL_F32 || t->dtype == AOL_F64;
    if (t->op != AOL_OP_TILE_COPY && !flt) return fail(AOL_EUNSUPPORTED, "op needs float32/float64 ports");
    const int64_t p0 = tiler_pat_total(t->tilers[0]), p1 = tiler_pat_total(t->tilers[1]);
    if (t->op == AOL_OP_TILE_COPY && p0 != p1) return fail(AOL_EINVAL, "src/dst pattern sizes differ");
    if (t->op == AOL_OP_MATMUL && (p0 != p1 || tiler_pat_total(t->tilers[2]) != 1))
      return fail(AOL_EINVAL, "matmul needs equal a/b patterns and a single-element c pattern");
    if (t->op == AOL_OP_TILE_SUM && p1 != 1) return fail(AOL_EINVAL, "tile_sum needs a single-element s pattern");
  }
  return AOL_OK;
}

static int64_t task_rep_total(const aol_task* t) {
  return tilers_needed(t->op) ? tiler_rep_total(t->tilers[0]) : -1;
}

static const char* plan_name(const aol_task* t, int64_t first, int64_t count, void* const* ports) {
  switch (t->op) {
    case AOL_OP_TILE_COPY:
      return tile_copy_plan_name(t->tilers[0], t->tilers[1], first, count, dtype_size(t->dtype), ports);
    case AOL_OP_MATMUL:
      if (ports && gemm_tf32_applicable(*t, ports))
        return t->precision == AOL_PREC_3XTF32 ? "matmul.tcgen05_3xtf32" : "matmul.tcgen05_tf32";
      if (ports && gemm_batched_applicable(*t, ports))
        return t->precision == AOL_PREC_3XTF32 ? "matmul.tcgen05_3xtf32_batched" : "matmul.tcgen05_tf32_batched";
      if (recognise_gemm_strides(*t)) return "matmul.exact_tiled";
      return gemm_exact_batched_applicable(*t) ? "matmul.exact_tiled_batched" : "matmul.generic_exact";
    case AOL_OP_TILE_FILTER: return filter_plan_name(*t);
    case AOL_OP_TILE_SUM: return tile_sum_plan_name(*t);
    default: return "identity";
  }
}

}  // namespace aol

using namespace aol;

extern "C" {

int aol_abi_version(void) { return AOL_ABI_VERSION; }

const char* aol_last_error(void) { return g_last_error.c_str(); }

int aol_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  int sm100 = 0;
  for (int d = 0; d < c; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major == 10) ++sm100;
  }
  if (n) *n = sm100;
  if (!sm100) return fail(AOL_ENODEV, "no sm_100 device visible");
  return AOL_OK;
}

int aol_validate(const aol_task* task) { return validate(task); }

// Ports every launch of `t` dereferences (aol_op's port lists; device scalars appended after the
// vectors); 0 where the count is data-dependent (scalar_seq).
static int required_ports(const aol_task* t) {
  const int dev_scalar = (t->flags & AOL_FLAG_DEVICE_SCALARS) && t->n_scalars > 0 ? 1 : 0;
  switch (t->op) {
    case AOL_OP_COPY: return 2;
    case AOL_OP_SUB: return 3;
    case AOL_OP_SCALE: return 1 + dev_scalar;
    case AOL_OP_AXPY: return 2 + dev_scalar;
    case AOL_OP_SPMV_CSR: return 5;
    case AOL_OP_DOT_PARTIAL: return 3;
    case AOL_OP_SCALAR_DIV: return 3;
    case AOL_OP_SCALAR_NEG: return 2;
    case AOL_OP_REL_RESIDUAL: return 3;
    case AOL_OP_PARTIALS_SUM: return 2;
    case AOL_OP_TILE_COPY: return 2;
    case AOL_OP_MATMUL: return 3;
    case AOL_OP_TILE_FILTER: return 3;
    case AOL_OP_TILE_SUM: return 2;
    default: return 0;
  }
}

int aol_launch(const aol_task* t, int64_t first, int64_t count, void* const* ports, const double* scalars,
               void* stream) {
  int rc = validate(t);
  if (rc) return rc;
  if (first < 0 || count < 0) return fail(AOL_EINVAL, "negative repetition range");
  const int64_t R = task_rep_total(t);
  if (R >= 0 && first + count > R) return fail(AOL_EINVAL, "repetition range outside the repetition space");
  if (!ports) return fail(AOL_EINVAL, "null port array");
  if (count == 0) return AOL_OK;
  for (int p = 0, n = required_ports(t); p < n; ++p)      // a null port would fault the kernel
    if (!ports[p]) return fail(AOL_EINVAL, "null port " + std::to_string(p));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (t->op) {
    case AOL_OP_TILE_COPY: return launch_tile_copy(*t, first, count, ports, s);
    case AOL_OP_MATMUL:
      if (gemm_tf32_applicable(*t, ports)) return launch_gemm_tf32(*t, first, count, ports, s);
      if (gemm_batched_applicable(*t, ports)) return launch_gemm_batched(*t, first, count, ports, s);
      {
        const int rc = launch_gemm_exact(*t, first, count, ports, s);   // canonical GEMM, exact order
        if (rc != AOL_EUNSUPPORTED) return rc;
        const int rb = launch_gemm_exact_batched(*t, first, count, ports, s);
        if (rb != AOL_EUNSUPPORTED) return rb;
      }
      return launch_matmul_generic(*t, first, count, ports, s);
    case AOL_OP_TILE_FILTER: return launch_filter_generic(*t, first, count, ports, s);
    case AOL_OP_TILE_SUM: return launch_tile_sum(*t, first, count, ports, s);
    default: return launch_identity(*t, first, count, ports, scalars, s);
  }
}

int aol_plan_name(const aol_task* t, int64_t first, int64_t count, void* const* ports, char* buf, int buflen) {
  int rc = validate(t);
  if (rc) return rc;
  if (!buf || buflen < 1) return fail(AOL_EINVAL, "bad buffer");
  snprintf(buf, (size_t)buflen, "%s", plan_name(t, first, count, ports));
  return AOL_OK;
}

int aol_tiler_offsets(const aol_tiler* tiler, int64_t first, int64_t count, int64_t* out_dev, void* stream) {
  if (!tiler || !out_dev) return fail(AOL_EINVAL, "null argument");
  return launch_tiler_offsets(*tiler, first, count, out_dev, static_cast<cudaStream_t>(stream));
}

int64_t aol_launch_counter(void) { return g_launches.load(); }

int aol_release_scratch(void) {
  release_dot_scratch();
  release_loop_scratch();
  release_gemm_scratch();
  return AOL_OK;
}

int aol_launch_fused2(const aol_task* producer, const aol_task* consumer, int64_t first, int64_t count,
                      void* const* producer_ports, void* const* consumer_ports, void* stream) {
  int rc = validate(producer);
  if (rc) return rc;
  if ((rc = validate(consumer))) return rc;
  if (producer->op != AOL_OP_TILE_FILTER || consumer->op != AOL_OP_TILE_FILTER)
    return fail(AOL_EUNSUPPORTED, "fusion is implemented for tile_filter -> tile_filter chains");
  if (first < 0 || count < 0 || first + count > task_rep_total(consumer))
    return fail(AOL_EINVAL, "repetition range outside the consumer's repetition space");
  if (!producer_ports || !consumer_ports) return fail(AOL_EINVAL, "null port array");
  return launch_fused_line_filters(*producer, *consumer, first, count, producer_ports, consumer_ports,
                                   static_cast<cudaStream_t>(stream));
}

}  // extern "C"
