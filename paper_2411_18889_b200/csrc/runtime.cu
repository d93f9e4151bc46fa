// Library runtime shared by every kernel file: cached device attributes, the
// dynamic-shared-memory opt-in, error strings, and the watchdog of the
// device-side polls (DESIGN.md §6 "Failure detection").
//
// Polling kernels (k_leapfrog_small, k_diffusion_resident, the p2p slab halo
// kernels) wait in the GPU for 16-byte words another CTA or another GPU
// publishes. If a word never arrives (a dead or stalled peer), the waiting
// kernel must neither hang the GPU nor kill the context: it records a fault
// code in a per-device word, every other poll on the device sees the word and
// gives up too, the kernels exit normally, and the host turns the word into an
// error (b2_fault_status -> B2_ETIMEOUT, SolomonError in Python). The context
// stays usable. The wait limit is a launch argument: b2_set_poll_timeout_ms or
// SOLOMON_POLL_TIMEOUT_S (default 120 s -- longer than any host stall a
// healthy run has, e.g. a checkpoint write or first-use plan timing).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace b2 {

__device__ unsigned int g_fault[4];  // [0]: first fault code on this device (0 = none)

constexpr int kMaxDevices = 64;

const DeviceInfo& device_info() {
  static DeviceInfo infos[kMaxDevices];
  static bool ready[kMaxDevices] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!ready[dev]) {
    cudaDeviceGetAttribute(&infos[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&infos[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    ready[dev] = true;
  }
  return infos[dev];
}

void allow_max_dynamic_smem(const void* fn) {
  static std::mutex mu;
  static std::vector<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : done)
    if (d.first == dev && d.second == fn) return;
  // the opt-in limit covers static + dynamic shared memory
  cudaFuncAttributes fa{};
  const size_t stat = cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? fa.sharedSizeBytes : 0;
  const int dyn = device_info().smem_optin - static_cast<int>(stat);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess)
    cudaGetLastError();  // a later launch reports a real problem; never leave a sticky error here
  done.emplace_back(dev, fn);
}

static std::atomic<long long> g_timeout_ms{[] {
  const char* e = std::getenv("SOLOMON_POLL_TIMEOUT_S");
  const double s = e ? std::atof(e) : 120.0;
  return static_cast<long long>((s > 0 ? s : 120.0) * 1000.0);
}()};

static unsigned int* fault_ptr() {
  static unsigned int* ptrs[kMaxDevices] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!ptrs[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_fault) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ptrs[dev] = static_cast<unsigned int*>(p);
  }
  return ptrs[dev];
}

Watch make_watch() {
  Watch w;
  w.fault = fault_ptr();
  w.timeout_ns = static_cast<unsigned long long>(g_timeout_ms.load()) * 1000000ull;
  return w;
}

}  // namespace b2

using namespace b2;

namespace b2 {
static std::atomic<int> g_withhold{-1};
int debug_withhold() { return g_withhold.load(); }
}  // namespace b2

extern "C" {

int b2_debug_withhold_publish(int cta) {
  b2::g_withhold.store(cta < 0 ? -1 : cta);
  return B2_OK;
}

int b2_set_poll_timeout_ms(long long ms) {
  if (ms <= 0) return B2_EINVAL;
  g_timeout_ms.store(ms);
  return B2_OK;
}

long long b2_poll_timeout_ms(void) { return g_timeout_ms.load(); }

int b2_fault_status(void* stream, int clear, int* which) {
  if (which) *which = 0;
  cudaError_t e = cudaStreamSynchronize(as_stream(stream));
  if (e != cudaSuccess) return static_cast<int>(e);
  unsigned int* p = fault_ptr();
  if (!p) return launch_status();
  unsigned int code = 0;
  if ((e = cudaMemcpy(&code, p, sizeof(code), cudaMemcpyDeviceToHost)) != cudaSuccess) return static_cast<int>(e);
  if (code && clear) {
    const unsigned int zero = 0;
    if ((e = cudaMemcpy(p, &zero, sizeof(zero), cudaMemcpyHostToDevice)) != cudaSuccess) return static_cast<int>(e);
  }
  if (which) *which = static_cast<int>(code);
  return code ? B2_ETIMEOUT : B2_OK;
}

const char* b2_error_string(int code) {
  switch (code) {
    case B2_OK: return "ok";
    case B2_EINVAL: return "invalid argument";
    case B2_EALIGN: return "pointer not 16-byte aligned";
    case B2_ESPACE: return "workspace too small";
    case B2_ENOMEM: return "out of device memory";
    case B2_ETIMEOUT: return "a device-side wait for a peer's data timed out (see b2_fault_status)";
    case B2_ENOTSUP: return "no kernel for this shape on this path";
    default: return code > 0 ? cudaGetErrorString(static_cast<cudaError_t>(code)) : "unknown error";
  }
}

const char* b2_fault_kernel(int which) {
  switch (which) {
    case 0: return "none";
    case kFaultLeapfrogSmall: return "k_leapfrog_small (position words of another CTA)";
    case kFaultResident: return "k_diffusion_resident (face words of another brick)";
    case kFaultSlabEdges: return "k_diffusion_slab_edges (a neighbour rank's halo rows)";
    case kFaultHalo2: return "k_diffusion_slab_halo2 (a neighbour rank's two halo planes)";
    case kFaultForceRing: return "k_force_fast (a ring slot of the in-kernel chunk reduction)";
    default: return "unknown kernel";
  }
}

const char* b2_version(void) { return "solomon_b200 0.2.0 (sm_100a)"; }

}  // extern "C"
