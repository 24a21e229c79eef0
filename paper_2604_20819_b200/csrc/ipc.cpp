// CUDA IPC plumbing for the peer-memory multi-GPU exchange (include/cqs.h).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <string>

#include "cqs_internal.h"

using namespace cqs;

static PFN_cuMemGetAddressRange_v3020 addr_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  }
  return fn;
}

extern "C" cqs_status cqs_ipc_handle(const void* dev_ptr, void* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(CQS_E_INVALID, "cqs_ipc_handle: NULL argument");
  auto fn = addr_range_fn();
  if (!fn) return fail(CQS_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, CUdeviceptr(reinterpret_cast<uintptr_t>(dev_ptr))) != CUDA_SUCCESS)
    return fail(CQS_E_CUDA, "cqs_ipc_handle: pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *offset = uint64_t(reinterpret_cast<uintptr_t>(dev_ptr) - uintptr_t(base));
  return CQS_OK;
}

extern "C" cqs_status cqs_ipc_open(const void* handle, void** base) {
  if (!handle || !base) return fail(CQS_E_INVALID, "cqs_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return CQS_OK;
}

extern "C" cqs_status cqs_ipc_close(void* base) {
  if (!base) return fail(CQS_E_INVALID, "cqs_ipc_close: NULL");
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(CQS_E_CUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
  return CQS_OK;
}
