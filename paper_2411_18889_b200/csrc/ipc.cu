// Multi-process peer memory for the fused-halo diffusion transport.
//
// One process per GPU: each rank exports the CUDA IPC handle of the allocation
// holding its slab, the neighbours map it (peer access over NVLink/NVSwitch,
// enabled lazily by the driver), and the boundary-plane stencil launches read
// their halo planes straight out of the neighbour's field -- the halo
// exchange is fused into the stencil kernel's loads; there is no NCCL call and
// no staging copy. Handles carry the offset of the pointer inside its
// allocation because torch's caching allocator sub-allocates segments.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"

namespace {

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRangeFn get_range() {
  static GetRangeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<GetRangeFn>(nullptr);
    return reinterpret_cast<GetRangeFn>(p);
  }();
  return fn;
}

}  // namespace

extern "C" {

size_t b2_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int b2_ipc_export(const void* dptr, void* handle, size_t* offset) {
  if (!dptr || !handle || !offset) return B2_EINVAL;
  GetRangeFn range = get_range();
  if (!range) return B2_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) return B2_EINVAL;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return static_cast<int>(e);
  std::memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<uintptr_t>(dptr) - static_cast<uintptr_t>(base);
  return B2_OK;
}

int b2_ipc_import(const void* handle, size_t offset, void** dptr) {
  if (!handle || !dptr) return B2_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return static_cast<int>(e);
  *dptr = static_cast<char*>(base) + offset;
  return B2_OK;
}

int b2_ipc_close(void* dptr, size_t offset) {
  if (!dptr) return B2_EINVAL;
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(dptr) - offset);
  return e == cudaSuccess ? B2_OK : static_cast<int>(e);
}

}  // extern "C"
