// capi_ipc.cu — device arenas shareable across processes (CUDA IPC), for the SMC engine's
// peer stores: K6 on rank r writes the outputs whose ancestors it owns straight into the owner
// rank's buffers over NVLink (SURVEY.md §8(e) option B).
#include <cstring>

#include "capi_internal.cuh"
#include "../../include/cuppl_gpu.h"

using namespace cuppl;

extern "C" {

int cuppl_arena_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return set_error(CUPPL_E_ARGUMENT, "arena: bad arguments");
  return cuda_status(cudaMalloc(ptr, bytes), "cudaMalloc");
}

int cuppl_arena_free(void* ptr) { return cuda_status(cudaFree(ptr), "cudaFree"); }

int cuppl_ipc_handle(const void* arena, void* handle_out) {
  if (!arena || !handle_out) return set_error(CUPPL_E_ARGUMENT, "ipc: NULL argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(arena));
  if (e != cudaSuccess) return cuda_status(e, "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  return CUPPL_OK;
}

int cuppl_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return set_error(CUPPL_E_ARGUMENT, "ipc: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int cuppl_ipc_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); }

}  // extern "C"
