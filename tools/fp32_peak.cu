// FP32 / packed-FP32 / MUFU throughput microbenchmark for the n-body roofline.
// Measures the chip's sustained FP32 FMA rate (scalar FFMA and packed FFMA2) and
// the MUFU.RSQ rate, so roofline.peak for calc_acc is a measured number.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1234.5f) out[0] = s;
}

template <int CH>
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 acc[CH];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(acc[c], av, bv);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  if (s == 1234.5f) out[0] = s;
}

template <int CH>
__global__ void k_rsqrt(float* out, int iters) {
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 1.0f + threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float r;
        asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(acc[c]));
        acc[c] = r;
      }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1234.5f) out[0] = s;
}

template <typename K>
static float time_it(K launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  float* d; CK(cudaMalloc(&d, 16));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  const double lanes = double(threads) * blocks;
  {
    float ms = time_it([&] { k_ffma<8><<<blocks, threads>>>(d, iters, 0.9999f, 1e-4f); }, 5);
    double flops = lanes * iters * 8 * 8 * 2;
    printf("{\"test\":\"ffma\",\"ms\":%.3f,\"tflops\":%.2f}\n", ms, flops / ms / 1e9);
  }
  {
    float ms = time_it([&] { k_ffma2<8><<<blocks, threads>>>(d, iters, 0.9999f, 1e-4f); }, 5);
    double flops = lanes * iters * 8 * 8 * 4;
    printf("{\"test\":\"ffma2\",\"ms\":%.3f,\"tflops\":%.2f}\n", ms, flops / ms / 1e9);
  }
  {
    float ms = time_it([&] { k_rsqrt<8><<<blocks, threads>>>(d, iters / 4); }, 5);
    double ops = lanes * (iters / 4) * 8 * 8;
    printf("{\"test\":\"mufu_rsqrt\",\"ms\":%.3f,\"gops\":%.1f,\"per_sm_per_clk_at_1965\":%.2f}\n", ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / 1.965e9);
  }
  CK(cudaGetLastError());
  return 0;
}
