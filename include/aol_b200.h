/*
 * aol_b200.h — C ABI of libaolb200.so, the B200 (sm_100a) Array-OL repetitive-task engine.
 *
 * This is the drop-in boundary below the Python host mirror
 * (paper_1105_4424_b200/executor.py).  It replaces the body of the
 * reference's per-device launch loop, i.e. what
 *     gmodelc.refexec.execute_schedule -> run_device -> "for launch in step.launches"
 * does at /root/reference/pkg/src/gmodelc/refexec.py:476-516, and it follows the
 * kernel parameter convention the reference's code generator emits for the
 * same launch (codegen.py:105-123: `first, count`, then the ports in
 * IntrinsicSpec order, host-resident scalar inputs by value).
 *
 * Plain C types only: no torch or C++ types cross this boundary.
 *  - Ownership: the caller owns every port buffer (device pointers) and every
 *    stream; the library never frees caller memory.  The library owns only
 *    per-process tensor-map/attribute caches and its thread-local error text.
 *  - Errors: functions return AOL_OK (0) or a negative aol_status; the message
 *    of the last failure on the calling thread is returned by aol_last_error().
 *    Validation failures are reported before anything is launched.
 *  - Threading: launches are asynchronous on the caller's stream; the library
 *    keeps no mutable global state besides lazily-initialised caches guarded
 *    by a mutex.
 */
#ifndef AOL_B200_H
#define AOL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AOL_ABI_VERSION 2
#define AOL_MAX_RANK 4      /* array / repetition / pattern rank limit */
#define AOL_MAX_TILERS 4    /* tiled ports per task */
#define AOL_MAX_PORTS 8

typedef enum aol_status {
  AOL_OK = 0,
  AOL_EINVAL = -1,        /* malformed task / tiler / arguments */
  AOL_ECUDA = -2,         /* CUDA runtime or driver failure */
  AOL_EUNSUPPORTED = -3,  /* op/dtype combination not implemented */
  AOL_ENODEV = -4         /* no sm_100 device visible */
} aol_status;

typedef enum aol_dtype { AOL_F32 = 0, AOL_F64 = 1, AOL_I32 = 2, AOL_I64 = 3 } aol_dtype;

/* Elementary tasks.  1..15: the reference's identity-tiler device intrinsics
 * (intrinsics.py:51-83); 16..: Array-OL tile intrinsics. */
typedef enum aol_op {
  AOL_OP_COPY = 1,        /* ports: src, dst                            dst[i] = src[i]        */
  AOL_OP_SUB = 2,         /* ports: x, y, z                             z[i] = x[i] - y[i]     */
  AOL_OP_SCALE = 3,       /* ports: y;     scalars: a                   y[i] *= a              */
  AOL_OP_AXPY = 4,        /* ports: y, x;  scalars: a (if n_scalars=1)  y[i] += a*x[i] | x[i]  */
  AOL_OP_SPMV_CSR = 5,    /* ports: rowptr, colidx, values, x, y        row-wise, left to right */
  AOL_OP_DOT_PARTIAL = 6, /* ports: a, b, partial (1 element, device)   partial = sum a[i]*b[i] */
  AOL_OP_SCALAR_DIV = 7,  /* ports: num, den, q (1 element each)        q = num / den  (host op div) */
  AOL_OP_SCALAR_NEG = 8,  /* ports: a, z                                z = -a         (host op neg) */
  AOL_OP_REL_RESIDUAL = 9,/* ports: num, den, z                         z = sqrt(num)/sqrt(den)      */
  AOL_OP_PARTIALS_SUM = 10,/* ports: partials (count elements), s       s = ((p0 + p1) + p2) ... fp64,
                              ascending device order (refexec.py:483-486); first must be 0 */
  AOL_OP_SCALAR_SEQ = 11, /* ports: the scalars used; count = n ops (1..8); scalars: per op
                              (op 7|8|9, in0, in1 (-1 for neg), out) as port indices — several
                              host scalar ops in program order in ONE launch */
  AOL_OP_TILE_COPY = 16,  /* ports: src, dst           tilers: src, dst                        */
  AOL_OP_MATMUL = 17,     /* ports: a, b, c            tilers: a, b, c   c = sum_k a_k * b_k   */
  AOL_OP_TILE_FILTER = 18,/* ports: x, w, y            tilers: x, y      y_j = sum_i w_ji x_i  */
  AOL_OP_TILE_SUM = 19    /* ports: x, s               tilers: x, s      s = sum_i x_i         */
} aol_op;

/* flags: scalar inputs (scale/axpy `a`) are read from a device pointer appended after
 * the vector ports instead of `scalars` — lets a whole loop body run without host
 * round trips (CUDA-graph capture of LoopStep bodies). */
#define AOL_FLAG_DEVICE_SCALARS 1
/* flags: the task's tiled input is placed in deviceLocal memory by the MARTE allocation
 * (memmap.py:65-133 -> placement.py): kernels with a shared-memory-staged form take it
 * (tile_filter: the per-tile smem window `line_tiled` instead of the register-window
 * batched kernel).  Results are identical; only the staging changes. */
#define AOL_FLAG_STAGE_SMEM 2

typedef enum aol_precision {
  AOL_PREC_DEFAULT = 0,   /* matmul: TF32 tensor cores; everything else: exact order */
  AOL_PREC_TF32 = 1,      /* matmul on tcgen05 kind::tf32 (tolerance stated in DESIGN.md) */
  AOL_PREC_3XTF32 = 2,    /* matmul on tcgen05, hi/lo split, 3 products, K-chunked accumulation with
                             round-to-nearest adds: 8.1e-7 normwise vs fp64 at 8192^3 (cuBLAS SIMT fp32:
                             1.6e-6); stated bound (2^-20 + 2^-21 sqrt(K)) |A||B| per element */
  AOL_PREC_EXACT = 3      /* CUDA cores, pattern order, no FMA: bit-exact vs the oracle */
} aol_precision;

/* e(r,i) = (origin + paving.r + fitting.i) mod array   (component-wise, Euclidean)
 * off    = row-major flat offset of e in `array`.
 * r = row-major unravel of the repetition index over rep[0..rep_rank),
 * i = row-major unravel of the pattern index over pattern[0..pat_rank). */
typedef struct aol_tiler {
  int32_t arr_rank, rep_rank, pat_rank, reserved;
  int64_t array[AOL_MAX_RANK];
  int64_t rep[AOL_MAX_RANK];
  int64_t pattern[AOL_MAX_RANK];
  int64_t origin[AOL_MAX_RANK];
  int64_t paving[AOL_MAX_RANK][AOL_MAX_RANK];   /* [array dim][repetition dim] */
  int64_t fitting[AOL_MAX_RANK][AOL_MAX_RANK];  /* [array dim][pattern dim]    */
} aol_tiler;

typedef struct aol_task {
  int32_t op;              /* aol_op */
  int32_t dtype;           /* aol_dtype of the value ports */
  int32_t index_dtype;     /* AOL_I32 / AOL_I64: spmv rowptr/colidx */
  int32_t precision;       /* aol_precision */
  int32_t n_tilers;        /* tiled ports, in IntrinsicSpec port order */
  int32_t n_scalars;       /* host-resident scalar inputs passed by value */
  int32_t flags;           /* AOL_FLAG_* */
  int32_t reserved;
  aol_tiler tilers[AOL_MAX_TILERS];
} aol_task;

/* ABI version of the loaded library (== AOL_ABI_VERSION). */
int aol_abi_version(void);

/* Message of the last failure on this thread ("" if none). */
const char* aol_last_error(void);

/* Number of visible sm_100 devices; fails with AOL_ENODEV if none. */
int aol_device_count(int* n);

/* Validate a task without launching (same checks aol_launch performs). */
int aol_validate(const aol_task* task);

/* One launch of a repetitive task over repetitions [first, first+count) on the
 * current device, asynchronously on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  `ports` are device pointers in IntrinsicSpec order
 * (intrinsics.py:51-83 for reference ops); `scalars` are host scalar inputs.
 * Replaces one iteration of refexec.py:488-514 / one clEnqueueNDRangeKernel of
 * the generated host code (codegen.py:456-457). */
int aol_launch(const aol_task* task, int64_t first, int64_t count,
               void* const* ports, const double* scalars, void* stream);

/* Kernel variant aol_launch would pick for this task (diagnostics / tests):
 * writes a NUL-terminated name into buf. */
int aol_plan_name(const aol_task* task, int64_t first, int64_t count,
                  void* const* ports, char* buf, int buflen);

/* Debug / parity: flat offsets off(r, i) for r in [first, first+count) computed
 * on the GPU into out_dev[(r-first)*pattern_total + i] (int64, device memory). */
int aol_tiler_offsets(const aol_tiler* tiler, int64_t first, int64_t count,
                      int64_t* out_dev, void* stream);

/* Number of kernels this library has launched in this process (evidence counter). */
int64_t aol_launch_counter(void);

/* Free the library's cached device scratch: the per-(device, stream) dot_partial partials
 * (bounded LRU cache of 64 entries) and the persistent loop's per-device block.  Waits for
 * each owning device to go idle first; scratch pinned by a live aol_loop graph is kept.
 * The next launch that needs scratch allocates it again.  No reference counterpart. */
int aol_release_scratch(void);

/* Fused output gather over peer memory (the output array that crosses
 * shards is assembled at the root by the producing kernels themselves).  The root exports
 * its output buffer; every other rank maps it and passes the mapped pointer as the output
 * port of its launches, so the kernels' stores travel over NVLink into the root's array.
 * Replaces the reference's host-side gather of per-device results (refexec.py:545-547);
 * no OpenCL counterpart.
 *   aol_ipc_export: 64-byte CUDA IPC handle of the allocation holding dev_ptr, and dev_ptr's
 *                   byte offset in that allocation
 *   aol_ipc_import: map a handle exported by another process (peer access enabled lazily);
 *                   *dev_ptr = mapped base + offset
 *   aol_ipc_close:  unmap (by the pointer aol_ipc_import returned) */
int aol_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset);
int aol_ipc_import(const void* handle64, int64_t offset, void** dev_ptr);
int aol_ipc_close(void* dev_ptr);

/* Strided 2-D asynchronous copy, host <-> device either way (cudaMemcpy2DAsync, direction from
 * the pointers; pinned host memory): `height` rows of `width_bytes`, row pitches in bytes.  The
 * streamed MatMul moves column blocks of row-major B and C with it, so C blocks can be computed
 * and downloaded while B is still uploading.  No reference counterpart (refexec copies whole
 * arrays, refexec.py:392-398, :545-547). */
int aol_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes, int64_t height,
                 void* stream);

/* Task fusion: run `consumer` over its repetitions [first, first+count) computing
 * the part of `producer`'s output it reads on the fly, in shared memory, instead of
 * reading a materialised intermediate array (bit-identical results; the
 * intermediate is not written).  The executor calls it for two consecutive
 * DeviceSteps whose connecting port group only they use; returns
 * AOL_EUNSUPPORTED (nothing launched) when the pair is not fusable — currently a
 * horizontal 13->3 line filter feeding a vertical 14->4 line filter, the Array-OL
 * downscaler.  No reference counterpart (the reference runs steps one by one,
 * refexec.py:518-541). */
int aol_launch_fused2(const aol_task* producer, const aol_task* consumer, int64_t first, int64_t count,
                      void* const* producer_ports, void* const* consumer_ports, void* stream);

/* Device-side LoopStep (refexec.py:525-541): one CUDA graph holding a conditional WHILE
 * node.  aol_loop_begin starts capturing `stream` (a non-default cudaStream_t) into the
 * node's body; the caller then enqueues one loop iteration with aol_launch on that stream
 * (device-resident scalars, AOL_FLAG_DEVICE_SCALARS, AOL_OP_SCALAR_*, AOL_OP_PARTIALS_SUM);
 * aol_loop_end appends the check (iterations += 1; stop when *relres_dev <= tol or after
 * max_iter iterations) and instantiates.  aol_loop_run executes the whole loop with no host
 * round trip per iteration and returns the bookkeeping of ExecutionResult (refexec.py:367-372).
 * No reference counterpart beyond the interpreter loop itself. */
typedef struct aol_loop aol_loop;
int aol_loop_begin(void* stream, const void* relres_dev, int relres_dtype, double tol, int64_t max_iter,
                   aol_loop** loop);
int aol_loop_end(aol_loop* loop);
int aol_loop_run(aol_loop* loop, void* stream, int64_t* iterations, double* final_relres, int* converged);
int aol_loop_destroy(aol_loop* loop);

/* A LoopStep body as ONE persistent cooperative kernel (no launch and no host round trip
 * per iteration).  `ops` is the body in schedule order, one entry per
 * KernelLaunch / host scalar op; `port` holds indices into `ports` in the aol_launch port
 * order (scale/axpy: the scalar `a` after the vectors).  All ops share `dtype` (f32/f64);
 * spmv index arrays are `index_dtype`.  Runs until scalar port `relres_port` <= tol or
 * max_iter iterations, like refexec.py:525-541, with results bit-identical to launching
 * the same ops one by one.  Returns AOL_EUNSUPPORTED (nothing launched) for bodies
 * outside its op set (copy/sub/scale/axpy/spmv_csr/dot_partial/div/neg/rel_residual),
 * > 128 ops, > 96 op groups or > 32 ports; callers then fall back to aol_loop_begin/end/run. */
typedef struct aol_loop_op {
  int32_t op;
  int32_t n_scalars;       /* axpy: 1 -> y += a*x, 0 -> y += x */
  int32_t part, n_parts;   /* dot_partial: launch index in its step, launches in the step */
  int64_t first, count;    /* the launch range (ignored for scalar ops) */
  int32_t port[6];
} aol_loop_op;

int aol_loop_persistent(const aol_loop_op* ops, int n_ops, void* const* ports, int n_ports, int dtype,
                        int index_dtype, int relres_port, double tol, int64_t max_iter, void* stream,
                        int64_t* iterations, double* final_relres, int* converged);

#ifdef __cplusplus
}
#endif

#endif /* AOL_B200_H */
