// Diagnostics library (libsolomon_probe.so, NOT part of the product ABI):
// measures the FP32 FMA roofline the n-body kernel is judged against. The
// n-body path is FP32 CUDA-core work; MEASURED_PEAKS.json records only HBM and
// bf16 tensor peaks, so bench.py measures the FP32 peak live on the same GPU
// with a packed-FFMA2 throughput kernel (148 SMs x 128 lanes x 2 flop x clock).
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) k_ffma2_peak(float* out, int iters, float a, float b) {
  float2 acc[CH];
  const float2 av = make_float2(a, a), bv = make_float2(b, b);
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

extern "C" double solomon_probe_fp32_tflops(int reps) {
  float* d = nullptr;
  if (cudaMalloc(&d, 16) != cudaSuccess) return -1.0;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma2_peak<8><<<blocks, threads>>>(d, iters, 0.9999f, 1e-4f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    k_ffma2_peak<8><<<blocks, threads>>>(d, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  const double flops = double(threads) * blocks * iters * 8 * 8 * 4;  // 2 lanes x 2 flop per FFMA2
  return flops / (best * 1e-3) / 1e12;
}

// Operand-pattern probes for the n-body FMA-pipe ceiling:
// mode 0: FFMA2 acc = fma(x_c, y_c, acc)  -- 3 distinct register pairs per op
// mode 1: FFMA2 acc = fma(x_c, y,   acc)  -- one operand shared across ops
// mode 2: FFMA  acc = fma(x_c, y_c, acc)  -- scalar, 3 distinct registers
// mode 3: FFMA2 acc = fma(x_c, x_c, acc)  -- 2 distinct pairs
template <int MODE>
__global__ void __launch_bounds__(256) k_pattern(float* out, int iters, const float* seed) {
  constexpr int CH = 8;
  float2 acc[CH], x[CH], y[CH];
  float sacc[CH], sx[CH], sy[CH];
  const float s0 = seed[threadIdx.x & 31];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const float a = seed[(threadIdx.x + 3 * c + 1) & 31], b = seed[(threadIdx.x + 5 * c + 2) & 31];
    const float q = seed[(threadIdx.x + 7 * c + 3) & 31], r = seed[(threadIdx.x + 11 * c + 4) & 31];
    acc[c] = make_float2(s0 + a, s0 - b);
    x[c] = make_float2(a, b);
    y[c] = make_float2(q, r);
    sacc[c] = s0 + b;
    sx[c] = a;
    sy[c] = q;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (MODE == 0) acc[c] = __ffma2_rn(x[c], y[c], acc[c]);
        if (MODE == 1) acc[c] = __ffma2_rn(x[c], y[0], acc[c]);
        if (MODE == 2) sacc[c] = fmaf(sx[c], sy[c], sacc[c]);
        if (MODE == 3) acc[c] = __ffma2_rn(x[c], x[c], acc[c]);
      }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y + sacc[c];
  if (s == 1234.5f) out[0] = s;
}

extern "C" double solomon_probe_pattern_tflops(int mode) {
  float *d = nullptr, *seed = nullptr;
  cudaMalloc(&d, 16);
  cudaMalloc(&seed, 32 * sizeof(float));
  cudaMemset(seed, 0, 32 * sizeof(float));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256, blocks = sms * 8, iters = 2048;
  auto launch = [&] {
    switch (mode) {
      case 0: k_pattern<0><<<blocks, threads>>>(d, iters, seed); break;
      case 1: k_pattern<1><<<blocks, threads>>>(d, iters, seed); break;
      case 2: k_pattern<2><<<blocks, threads>>>(d, iters, seed); break;
      default: k_pattern<3><<<blocks, threads>>>(d, iters, seed); break;
    }
  };
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(d);
  cudaFree(seed);
  const double lanes = (mode == 2) ? 1.0 : 2.0;
  return double(threads) * blocks * iters * 8 * 8 * lanes * 2 / (best * 1e-3) / 1e12;
}
