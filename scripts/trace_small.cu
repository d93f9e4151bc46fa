// Phase timeline of k_leapfrog_small (tuning probe, not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSOLOMON_B200_BUILD -Iinclude \
//        -Ipaper_2411_18889_b200/csrc scripts/trace_small.cu -o scripts/trace_small && scripts/trace_small [n] [steps]
//
// Builds the kernel with B2_SMALL_TRACE (globaltimer stamps per CTA and step) and
// prints the mean duration of: gather (incl. waiting for other CTAs' positions),
// force + reduce, kick/drift/publish, and the whole step.
#define B2_SMALL_TRACE
#include "../paper_2411_18889_b200/csrc/nbody_small.cu"

#include <cstdio>
#include <vector>

namespace b2 {
const DeviceInfo& device_info() {
  static DeviceInfo d;
  if (!d.sms) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  }
  return d;
}
void allow_max_dynamic_smem(const void* fn) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, device_info().smem_optin);
}
Watch make_watch() { return Watch{nullptr, 4000000000ull}; }
}  // namespace b2

int main(int argc, char** argv) {
  using namespace b2;
  const int n = argc > 1 ? std::atoi(argv[1]) : 4096;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 40;
  std::vector<float4> h(n);
  for (int i = 0; i < n; ++i) {
    const float u = (i * 0.618034f) - static_cast<int>(i * 0.618034f);
    h[i] = make_float4(u - 0.5f, ((i * 7) % 101) / 101.f - 0.5f, ((i * 13) % 97) / 97.f - 0.5f, 1.f / n);
  }
  float4 *pos, *vel, *acc;
  cudaMalloc(&pos, n * 16);
  cudaMalloc(&vel, n * 16);
  cudaMalloc(&acc, n * 16);
  cudaMemset(vel, 0, n * 16);
  uint4* pub;
  cudaMalloc(&pub, 2 * n * 16);
  const int nch = nchunks_for(n, 0);
  const int sms = device_info().sms;
  const int I = 2 * kSmallPairs * ((n + 2 * kSmallPairs * sms - 1) / (2 * kSmallPairs * sms));
  const int ctas = (n + I - 1) / I;
  const size_t smem = (static_cast<size_t>(n) + nch + static_cast<size_t>(nch) * I) * 16 + n * 4;
  unsigned long long* trace;
  cudaMalloc(&trace, static_cast<size_t>(ctas) * steps * 4 * 8);
  cudaFuncSetAttribute(k_leapfrog_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 200; ++rep) {
    cudaMemcpy(pos, h.data(), n * 16, cudaMemcpyHostToDevice);
    cudaMemset(pub, 0, 2 * n * 16);
    SmallArgs a{n, pos, vel, acc, pub, 1.f / 4096, 1.f / 128, 1.f / 256, steps, B2_INIT_ACC, chunk_size(n, 0), nch,
                I, Watch{nullptr, 4000000000ull}, trace};
    void* args[] = {&a};
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_leapfrog_small<false>), ctas,
                                                  kSmallThreads, args, smem, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      std::printf("launch failed: %s\n", cudaGetErrorString(err));
      return 1;
    }
    std::vector<unsigned long long> t(static_cast<size_t>(ctas) * steps * 4);
    cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
    double ph[4] = {};
    long cnt = 0;
    for (int b = 0; b < ctas; ++b)
      for (int s = 3; s + 1 < steps; ++s) {
        const unsigned long long* q = &t[(static_cast<size_t>(b) * steps + s) * 4];
        ph[0] += q[1] - q[0];
        ph[1] += q[2] - q[1];
        ph[2] += q[3] - q[2];
        ph[3] += q[4] - q[0];
        ++cnt;
      }
    if (rep % 50 != 49) continue;
    std::printf("n=%d ctas=%d nch=%d: %.2f us/step (events, incl. init force)  gather %.0f  force %.0f  "
                "kick+publish %.0f  step %.0f ns\n",
                n, ctas, nch, ms * 1e3 / steps, ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt);
  }
  return 0;
}
