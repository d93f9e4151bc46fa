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
#include <algorithm>
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
int debug_withhold() { return -1; }
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
  float4* pub;
  cudaMalloc(&pub, small_workspace_bytes(n));
  const int nch = nchunks_for(n, 0);
  const int sms = device_info().sms;
  SmallShape sh;
  if (!small_shape(n, nch, sms, &sh)) {
    std::printf("n=%d: outside the persistent path\n", n);
    return 1;
  }
  const int ctas = sh.ctas;
  const size_t smem = small_smem_bytes(n, nch, sh.I);
  unsigned long long* trace;
  const size_t tw = static_cast<size_t>(ctas) * steps * 32;
  cudaMalloc(&trace, tw * 8);
  const void* fn = reinterpret_cast<const void*>(small_kernel<false>(sh.NP));
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nw = std::min(8, sh.threads / 32);
  for (int rep = 0; rep < 100; ++rep) {
    cudaMemcpy(pos, h.data(), n * 16, cudaMemcpyHostToDevice);
    cudaMemset(pub, 0, small_workspace_bytes(n));
    cudaMemset(trace, 0, tw * 8);
    SmallArgs a{n, pos, vel, acc, pub, reinterpret_cast<unsigned int*>(pub + 2 * n), 1.f / 4096, 1.f / 128,
                1.f / 256, steps, B2_INIT_ACC, chunk_size(n, 0), nch, sh.I, sh.G, Watch{nullptr, 4000000000ull}, -1,
                trace};
    void* args[] = {&a};
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel(fn, ctas, sh.threads, args, smem, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      std::printf("launch failed: %s\n", cudaGetErrorString(err));
      return 1;
    }
    if (rep != 99) continue;
    std::vector<unsigned long long> t(tw);
    cudaMemcpy(t.data(), trace, tw * 8, cudaMemcpyDeviceToHost);
    auto T = [&](int b, int st, int k) { return static_cast<double>(t[(static_cast<size_t>(b) * steps + st) * 32 + k]); };
    // per step s (steady state): phases of CTA b, and the exchange of state s+2 (announced in
    // step s, gathered in step s+1)
    double bar0 = 0, reduce = 0, announce = 0, flag_lat_first = 0, flag_lat_last = 0, data = 0, force = 0,
           force_skew = 0, fbar = 0, stepd = 0, ann_skew = 0;
    long cnt = 0, sc = 0;
    for (int st = 3; st + 2 < steps; ++st) {
      double amin = 1e30, amax = 0, fmin = 1e30, fmax = 0;
      for (int b = 0; b < ctas; ++b) {
        amin = std::min(amin, T(b, st, 4));
        amax = std::max(amax, T(b, st, 4));
        for (int w = 0; w < nw; ++w) {
          fmin = std::min(fmin, T(b, st + 1, 8 + w));
          fmax = std::max(fmax, T(b, st + 1, 8 + w));
        }
      }
      ann_skew += amax - amin;
      flag_lat_first += fmin - amax;
      flag_lat_last += fmax - amax;
      ++sc;
      for (int b = 0; b < ctas; ++b) {
        bar0 += T(b, st, 1) - T(b, st, 0);
        reduce += T(b, st, 3) - T(b, st, 2);
        announce += T(b, st, 4) - T(b, st, 3);
        double wmax = 0, wmin = 1e30, dsum = 0, fsum = 0;
        for (int w = 0; w < nw; ++w) {
          dsum += T(b, st, 16 + w) - T(b, st, 8 + w);
          fsum += T(b, st, 24 + w) - T(b, st, 16 + w);
          wmax = std::max(wmax, T(b, st, 24 + w));
          wmin = std::min(wmin, T(b, st, 24 + w));
        }
        data += dsum / nw;
        force += fsum / nw;
        force_skew += wmax - wmin;
        fbar += T(b, st, 2) - wmax;
        stepd += T(b, st + 1, 0) - T(b, st, 0);
        ++cnt;
      }
    }
    std::printf("n=%d ctas=%d threads=%d nch=%d NP=%d: %.2f us/step (events)\n", n, ctas, sh.threads, nch, sh.NP,
                ms * 1e3 / steps);
    std::printf("  step %.0f ns | top barrier %.0f | producer probes: last publish -> first/last warp %.0f / %.0f "
                "(announce skew %.0f) | slice read %.0f | force task %.0f (warp skew %.0f, barrier after %.0f) | "
                "reduce %.0f | update+publish %.0f\n",
                stepd / cnt, bar0 / cnt, flag_lat_first / sc, flag_lat_last / sc, ann_skew / sc, data / cnt,
                force / cnt, force_skew / cnt, fbar / cnt, reduce / cnt, announce / cnt);
  }
  return 0;
}
