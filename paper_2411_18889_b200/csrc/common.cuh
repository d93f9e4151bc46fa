// Shared helpers for the solomon_b200 sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "solomon_b200.h"

namespace b2 {

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B2_OK : static_cast<int>(e);
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Cached per-device attributes (queried once per device).
struct DeviceInfo {
  int sms = 0;
  int smem_optin = 0;
};
const DeviceInfo& device_info();

}  // namespace b2
