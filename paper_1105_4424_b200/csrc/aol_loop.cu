// Device-side LoopStep (refexec.py:525-541) as ONE CUDA graph: a conditional WHILE node
// whose body is the captured loop body followed by a one-thread check kernel.  The check
// kernel counts the iteration, records relres and clears the condition when
// relres <= tol or the iteration bound is reached — the reference's do-while, with no
// host round trip per iteration.
#include <cuda_runtime.h>

#include <new>

#include "aol_common.cuh"

namespace aol {

double* dot_scratch_for_stream(cudaStream_t stream, int pin_delta);

struct LoopState {
  int64_t iterations;
  double relres;
  int converged;
};

template <typename T>
__global__ void k_loop_check(cudaGraphConditionalHandle h, const T* relres, double tol, int64_t max_iter,
                             LoopState* st) {
  const int64_t n = ++st->iterations;
  const double r = (double)relres[0];
  st->relres = r;
  unsigned int more = 1;
  if (r <= tol) {
    st->converged = 1;
    more = 0;
  } else if (n >= max_iter) {
    more = 0;
  }
  cudaGraphSetConditional(h, more);
}

}  // namespace aol

struct aol_loop {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t stream = nullptr;
  const void* relres = nullptr;
  int relres_dtype = AOL_F64;
  double tol = 0;
  int64_t max_iter = 0;
  aol::LoopState* state = nullptr;
  int device = 0;
};

using namespace aol;

extern "C" {

int aol_loop_begin(void* stream, const void* relres_dev, int relres_dtype, double tol, int64_t max_iter,
                   aol_loop** out) {
  if (!stream || !relres_dev || !out || max_iter < 1) return fail(AOL_EINVAL, "aol_loop_begin: bad arguments");
  if (relres_dtype != AOL_F32 && relres_dtype != AOL_F64) return fail(AOL_EINVAL, "relres must be float32/float64");
  // dots captured on this stream use its scratch: allocate it now (no cudaMalloc during
  // capture) and pin it for the graph's lifetime (aol_loop_destroy unpins)
  if (!dot_scratch_for_stream(static_cast<cudaStream_t>(stream), 1)) return fail(AOL_ECUDA, "cannot allocate dot scratch");
  aol_loop* L = new (std::nothrow) aol_loop();
  if (!L) return fail(AOL_ECUDA, "out of host memory");
  L->stream = static_cast<cudaStream_t>(stream);
  cudaGetDevice(&L->device);
  L->relres = relres_dev;
  L->relres_dtype = relres_dtype;
  L->tol = tol;
  L->max_iter = max_iter;
  cudaError_t e = cudaMalloc(&L->state, sizeof(LoopState));
  if (e == cudaSuccess) e = cudaGraphCreate(&L->graph, 0);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = L->handle;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, L->graph, nullptr, 0, &p);
  if (e == cudaSuccess) {
    L->body = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(L->stream, L->body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  }
  if (e != cudaSuccess) {
    if (L->graph) cudaGraphDestroy(L->graph);
    if (L->state) cudaFree(L->state);
    dot_scratch_for_stream(L->stream, -1);
    delete L;
    return cuda_fail(e, "aol_loop_begin");
  }
  *out = L;
  return AOL_OK;
}

int aol_loop_end(aol_loop* L) {
  if (!L) return fail(AOL_EINVAL, "null loop");
  if (L->relres_dtype == AOL_F64)
    k_loop_check<double><<<1, 1, 0, L->stream>>>(L->handle, (const double*)L->relres, L->tol, L->max_iter, L->state);
  else
    k_loop_check<float><<<1, 1, 0, L->stream>>>(L->handle, (const float*)L->relres, L->tol, L->max_iter, L->state);
  cudaError_t e = cudaGetLastError();
  cudaGraph_t captured = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(L->stream, &captured);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&L->exec, L->graph, 0);
  if (e != cudaSuccess) return cuda_fail(e, "aol_loop_end");
  count_launch();
  return AOL_OK;
}

int aol_loop_run(aol_loop* L, void* stream, int64_t* iterations, double* final_relres, int* converged) {
  if (!L || !L->exec) return fail(AOL_EINVAL, "loop not instantiated");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : L->stream;
  AOL_CUDA_CHECK(cudaMemsetAsync(L->state, 0, sizeof(LoopState), s));
  AOL_CUDA_CHECK(cudaGraphLaunch(L->exec, s));
  LoopState h;
  AOL_CUDA_CHECK(cudaMemcpyAsync(&h, L->state, sizeof(h), cudaMemcpyDeviceToHost, s));
  AOL_CUDA_CHECK(cudaStreamSynchronize(s));
  count_launch();
  if (iterations) *iterations = h.iterations;
  if (final_relres) *final_relres = h.relres;
  if (converged) *converged = h.converged;
  return AOL_OK;
}

int aol_loop_destroy(aol_loop* L) {
  if (!L) return AOL_OK;
  if (L->exec) cudaGraphExecDestroy(L->exec);
  if (L->graph) cudaGraphDestroy(L->graph);
  if (L->state) cudaFree(L->state);
  int cur = 0;
  cudaGetDevice(&cur);
  if (L->device != cur) cudaSetDevice(L->device);
  dot_scratch_for_stream(L->stream, -1);
  if (L->device != cur) cudaSetDevice(cur);
  delete L;
  return AOL_OK;
}

}  // extern "C"
