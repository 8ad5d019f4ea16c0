// CUDA IPC for the fused output gather: every rank's kernels store the
// output ranges they produce straight into the root's buffer through a peer mapping
// (NVLink on a multi-GPU box), so the gather costs no separate phase.
//
//   aol_ipc_export: handle of the cudaMalloc allocation holding `ptr` + ptr's byte offset
//                   in it (torch's caching allocator hands out pieces of larger segments;
//                   the base comes from cuMemGetAddressRange)
//   aol_ipc_import: open a handle exported by another process (peer access enabled lazily)
//                   and return base + offset
//   aol_ipc_close:  close a mapping made by aol_ipc_import (by the pointer it returned)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "aol_b200.h"
#include "aol_common.cuh"

namespace aol {

typedef CUresult (*PFN_addr_range)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_addr_range addr_range_fn() {
  static PFN_addr_range fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_addr_range>(p);
  });
  return fn;
}

// An allocation is opened once per process and reference-counted: the same handle imported
// again (a new executor over the root's cached allocation) reuses the mapping.
struct IpcMap {
  void* base;
  int refs;
};
static std::mutex g_ipc_mu;
static std::map<std::string, IpcMap> g_ipc_open;   // handle bytes -> mapping
static std::map<void*, std::string> g_ipc_ptrs;    // pointer handed out -> handle bytes (one per import)
static std::map<void*, int> g_ipc_ptr_refs;

}  // namespace aol

extern "C" {

int aol_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset) {
  using namespace aol;
  if (!dev_ptr || !handle64 || !offset) return fail(AOL_EINVAL, "null argument");
  auto fn = addr_range_fn();
  if (!fn) return fail(AOL_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return fail(AOL_EINVAL, "pointer is not inside a device allocation");
  cudaIpcMemHandle_t h;
  AOL_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
  return AOL_OK;
}

int aol_ipc_import(const void* handle64, int64_t offset, void** dev_ptr) {
  using namespace aol;
  if (!handle64 || !dev_ptr || offset < 0) return fail(AOL_EINVAL, "bad argument");
  const std::string key(static_cast<const char*>(handle64), 64);
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  auto it = g_ipc_open.find(key);
  if (it == g_ipc_open.end()) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    void* base = nullptr;
    AOL_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    it = g_ipc_open.emplace(key, IpcMap{base, 0}).first;
  }
  it->second.refs += 1;
  void* p = static_cast<char*>(it->second.base) + offset;
  g_ipc_ptrs[p] = key;
  g_ipc_ptr_refs[p] += 1;
  *dev_ptr = p;
  return AOL_OK;
}

int aol_ipc_close(void* dev_ptr) {
  using namespace aol;
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  auto pit = g_ipc_ptrs.find(dev_ptr);
  if (pit == g_ipc_ptrs.end()) return fail(AOL_EINVAL, "pointer was not returned by aol_ipc_import");
  const std::string key = pit->second;
  if (--g_ipc_ptr_refs[dev_ptr] == 0) {
    g_ipc_ptr_refs.erase(dev_ptr);
    g_ipc_ptrs.erase(pit);
  }
  auto it = g_ipc_open.find(key);
  if (it != g_ipc_open.end() && --it->second.refs == 0) {
    void* base = it->second.base;
    g_ipc_open.erase(it);
    AOL_CUDA_CHECK(cudaIpcCloseMemHandle(base));
  }
  return AOL_OK;
}

// Strided (2-D) asynchronous copy between host and device memory in either direction
// (cudaMemcpy2DAsync, direction from the pointers): the GEMM's 2-D streamed path moves column
// blocks of row-major B and C with it.  Pinned host memory for an asynchronous copy.
int aol_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes, int64_t height,
                 void* stream) {
  using namespace aol;
  if (!dst || !src || width_bytes < 0 || height < 0 || dpitch < width_bytes || spitch < width_bytes)
    return fail(AOL_EINVAL, "bad 2-D copy geometry");
  if (width_bytes == 0 || height == 0) return AOL_OK;
  AOL_CUDA_CHECK(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes, (size_t)height,
                                   cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return AOL_OK;
}

}  // extern "C"
