// Phase timeline of k_diffusion_resident (tuning probe, not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_2411_18889_b200/csrc \
//        scripts/trace_resident.cu -o scripts/trace_resident && scripts/trace_resident [n] [steps]
//
// Builds the kernel with B2_RESIDENT_TRACE (globaltimer stamps per brick and step)
// and prints the mean duration of each phase: halo pull (incl. waiting for
// the neighbours' tagged faces), march, face export, and
// the whole step.
#define B2_RESIDENT_TRACE
#include "../paper_2411_18889_b200/csrc/diffusion_resident.cu"

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
  const int n = argc > 1 ? std::atoi(argv[1]) : 128;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 60;
  const size_t cells = static_cast<size_t>(n) * n * n;
  std::vector<float> h(cells);
  for (size_t i = 0; i < cells; ++i) h[i] = static_cast<float>((i * 2654435761u) % 1000) / 1000.f;
  float *f, *fn;
  cudaMalloc(&f, cells * 4);
  cudaMalloc(&fn, cells * 4);
  cudaMemcpy(f, h.data(), cells * 4, cudaMemcpyHostToDevice);
  ResPlan p;
  if (!resident_plan_for(n, n, n, p)) {
    std::printf("no plan\n");
    return 1;
  }
  const int nb = p.nbi * p.nbj;
  const int face_cap = std::max(p.BI, p.BJ) * ((n + 2) / 3);
  const size_t mbytes = static_cast<size_t>(nb) * 8 * face_cap * sizeof(uint4);
  uint4* mbox;
  unsigned long long* trace;
  cudaMalloc(&mbox, mbytes);
  cudaMalloc(&trace, static_cast<size_t>(nb) * steps * 4 * 8);
  cudaFuncSetAttribute(k_diffusion_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const float dx = 1.f / n;
  const Coefs c = make_coefs(dx, dx, dx, 0.1f * dx * dx, 1.f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(mbox, 0, mbytes);
    ResArgs a{f, fn, n, n, n, steps, p.BI, p.BJ, p.nbj, mbox, face_cap, c, Watch{nullptr, 4000000000ull}, trace};
    void* args[] = {&a};
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_diffusion_resident), nb,
                                                  kResidentThreads, args, p.smem, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      std::printf("launch failed: %s\n", cudaGetErrorString(err));
      return 1;
    }
    std::vector<unsigned long long> t(static_cast<size_t>(nb) * steps * 4);
    cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
    double ph[4] = {};
    long cnt = 0;
    for (int bb = 0; bb < nb; ++bb)
      for (int s = 5; s + 1 < steps; ++s) {
        const unsigned long long* q = &t[(static_cast<size_t>(bb) * steps + s) * 4];
        const unsigned long long* qn = q + 4;
        ph[0] += q[1] - q[0];
        ph[1] += q[2] - q[1];
        ph[2] += qn[0] - q[2];
        ph[3] += qn[0] - q[0];
        ++cnt;
      }
    std::printf("n=%d BI=%d BJ=%d bricks=%d: %.2f us/step (events)  pull %.0f  march %.0f  export %.0f  "
                "step %.0f ns\n",
                n, p.BI, p.BJ, nb, ms * 1e3 / steps, ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt);
  }
  return 0;
}
