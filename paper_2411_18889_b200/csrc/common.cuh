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

// Opt the kernel `fn` into the full dynamic shared memory of the current device,
// once per (device, kernel) -- the attribute is per context. Thread-safe.
void allow_max_dynamic_smem(const void* fn);

// Watchdog of the device-side polls (runtime.cu): where a waiting kernel records
// that it gave up, and how long it may wait. A launch argument of every polling
// kernel; built on the host per launch from the current device and the
// b2_set_poll_timeout_ms setting.
struct Watch {
  unsigned int* fault;  // per-device word: first fault code, 0 = none
  unsigned long long timeout_ns;
};
Watch make_watch();
// fault codes (which kernel gave up), reported by b2_fault_status / b2_fault_kernel
constexpr unsigned int kFaultLeapfrogSmall = 1, kFaultResident = 2, kFaultSlabEdges = 3, kFaultHalo2 = 4,
                       kFaultForceRing = 5;

// ---- Device helpers shared by the persistent kernels (k_leapfrog_small,
// k_diffusion_resident): 16-byte words a producer CTA publishes and a consumer
// CTA polls. A .b128 access is single-copy atomic (PTX memory model; libcu++'s
// 16-byte cuda::atomic load/store compile to the same LDG/STG.E.128.STRONG.GPU),
// so a word carrying its own step tag needs no fence or flag.
#ifdef __CUDACC__
__device__ __forceinline__ uint4 ld_relaxed_b128(const uint4* p) {
  unsigned long long lo, hi;
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(lo), "=l"(hi)
               : "l"(p)
               : "memory");
  return make_uint4(static_cast<unsigned>(lo), static_cast<unsigned>(lo >> 32), static_cast<unsigned>(hi),
                    static_cast<unsigned>(hi >> 32));
}
__device__ __forceinline__ void st_relaxed_b128(uint4* p, uint4 v) {
  const unsigned long long lo = (static_cast<unsigned long long>(v.y) << 32) | v.x;
  const unsigned long long hi = (static_cast<unsigned long long>(v.w) << 32) | v.z;
  asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.gpu.global.b128 [%0], t; }" ::"l"(p), "l"(lo),
               "l"(hi)
               : "memory");
}
// System-scope twins for words another GPU writes over NVLink (peer mailboxes).
__device__ __forceinline__ uint4 ld_relaxed_sys_b128(const uint4* p) {
  unsigned long long lo, hi;
  asm volatile("{ .reg .b128 t; ld.relaxed.sys.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(lo), "=l"(hi)
               : "l"(p)
               : "memory");
  return make_uint4(static_cast<unsigned>(lo), static_cast<unsigned>(lo >> 32), static_cast<unsigned>(hi),
                    static_cast<unsigned>(hi >> 32));
}
__device__ __forceinline__ void st_relaxed_sys_b128(uint4* p, uint4 v) {
  const unsigned long long lo = (static_cast<unsigned long long>(v.y) << 32) | v.x;
  const unsigned long long hi = (static_cast<unsigned long long>(v.w) << 32) | v.z;
  asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.sys.global.b128 [%0], t; }" ::"l"(p), "l"(lo),
               "l"(hi)
               : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One poll iteration's verdict: true = stop waiting. Gives up when another
// poller on this device already recorded a fault (so one dead peer ends every
// wait within one poll, not one timeout each), or when this wait, begun at t0,
// exceeded the limit -- then it records `code` (first fault wins). The caller
// leaves its loops and exits normally: no __trap, the context stays usable.
__device__ __forceinline__ bool poll_expired(const Watch& w, unsigned long long t0, unsigned int code) {
  if (w.fault && *reinterpret_cast<volatile unsigned int*>(w.fault)) return true;
  if (globaltimer_ns() - t0 <= w.timeout_ns) return false;
  if (w.fault) atomicCAS(w.fault, 0u, code);
  return true;
}
// The same without the early exit on a standing fault: for waits whose giving up would
// corrupt data rather than merely skip work (a ring slot still being read).
__device__ __forceinline__ bool poll_timed_out(const Watch& w, unsigned long long t0, unsigned int code) {
  if (globaltimer_ns() - t0 <= w.timeout_ns) return false;
  if (w.fault) atomicCAS(w.fault, 0u, code);
  return true;
}
#endif

}  // namespace b2
