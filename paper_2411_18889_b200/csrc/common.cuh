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
// test hook (b2_debug_withhold_publish): the CTA of the persistent small-N leapfrog that never
// announces its positions, so the watchdog path can be exercised; -1 = none
int debug_withhold();
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
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_u32_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
// ---- PTX helpers: mbarrier + bulk async copy (sm_90+/sm_100a) -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// generic-proxy writes to global (acquired from other SMs) before a bulk copy reads them
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

#endif

}  // namespace b2
