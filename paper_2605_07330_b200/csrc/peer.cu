// peer.cu — CUDA IPC / copy-engine plumbing for the NVLink bucket transfer
// (include/sparsesync_peer.h). Host code only.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include "../../include/sparsesync_peer.h"

namespace {
inline int ck(cudaError_t e) { return e == cudaSuccess ? SYNC_OK : SYNC_ERR_CUDA; }

// cuMemGetAddressRange through the runtime's driver entry point (no link-time dependency on libcuda).
typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
GetRangeFn get_range() {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GetRangeFn)p;
  }
  return fn;
}
}  // namespace

extern "C" {

int sync_peer_mem_export(const void* d_ptr, uint8_t* out_handle, uint64_t* offset, uint64_t* alloc_bytes) {
  if (!d_ptr || !out_handle || !offset) return SYNC_ERR_ARG;
  CUdeviceptr base = 0;
  size_t size = 0;
  GetRangeFn range = get_range();
  if (!range || range(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) return SYNC_ERR_CUDA;
  cudaIpcMemHandle_t h;
  int st = ck(cudaIpcGetMemHandle(&h, (void*)base));
  if (st) return st;
  static_assert(sizeof(h) == SYNC_PEER_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  memcpy(out_handle, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)d_ptr - base);
  if (alloc_bytes) *alloc_bytes = size;
  return SYNC_OK;
}

int sync_peer_mem_open(const uint8_t* handle, void** d_base) {
  if (!handle || !d_base) return SYNC_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return ck(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
}

int sync_peer_mem_close(void* d_base) { return d_base ? ck(cudaIpcCloseMemHandle(d_base)) : SYNC_ERR_ARG; }

int sync_peer_event_create(void** ev, uint8_t* out_handle) {
  if (!ev || !out_handle) return SYNC_ERR_ARG;
  cudaEvent_t e;
  int st = ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
  if (st) return st;
  cudaIpcEventHandle_t h;
  static_assert(sizeof(h) == SYNC_PEER_HANDLE_BYTES, "cudaIpcEventHandle_t size");
  st = ck(cudaIpcGetEventHandle(&h, e));
  if (st) {
    cudaEventDestroy(e);
    return st;
  }
  memcpy(out_handle, &h, sizeof(h));
  *ev = (void*)e;
  return SYNC_OK;
}

int sync_peer_event_open(const uint8_t* handle, void** ev) {
  if (!handle || !ev) return SYNC_ERR_ARG;
  cudaIpcEventHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaEvent_t e;
  int st = ck(cudaIpcOpenEventHandle(&e, h));
  if (!st) *ev = (void*)e;
  return st;
}

int sync_peer_event_record(void* ev, sync_stream_t stream) {
  return ev ? ck(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream)) : SYNC_ERR_ARG;
}

int sync_peer_stream_wait(sync_stream_t stream, void* ev) {
  return ev ? ck(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0)) : SYNC_ERR_ARG;
}

int sync_peer_event_destroy(void* ev) { return ev ? ck(cudaEventDestroy((cudaEvent_t)ev)) : SYNC_ERR_ARG; }

int sync_peer_copy(void* d_dst, const void* d_src, uint64_t bytes, sync_stream_t stream) {
  if (!bytes) return SYNC_OK;
  if (!d_dst || !d_src) return SYNC_ERR_ARG;
  return ck(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
}

}  // extern "C"
