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
        if (MODE == 4) acc[c] = __fadd2_rn(acc[c], x[c]);
        if (MODE == 5) acc[c] = __fmul2_rn(acc[c], x[c]);
        if (MODE == 6) acc[c] = __ffma2_rn(acc[c], make_float2(s0, s0), x[c]);
        if (MODE == 7) acc[c] = __fadd2_rn(acc[c], make_float2(s0, s0));
        if (MODE == 8) acc[c] = __fmul2_rn(acc[c], make_float2(s0, s0));
        if (MODE == 9) acc[c] = __ffma2_rn(acc[c], make_float2(s0, s0), make_float2(s0, s0));
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
      case 3: k_pattern<3><<<blocks, threads>>>(d, iters, seed); break;
      case 4: k_pattern<4><<<blocks, threads>>>(d, iters, seed); break;
      case 5: k_pattern<5><<<blocks, threads>>>(d, iters, seed); break;
      case 6: k_pattern<6><<<blocks, threads>>>(d, iters, seed); break;
      case 7: k_pattern<7><<<blocks, threads>>>(d, iters, seed); break;
      case 8: k_pattern<8><<<blocks, threads>>>(d, iters, seed); break;
      default: k_pattern<9><<<blocks, threads>>>(d, iters, seed); break;
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
  const double flop = (mode == 4 || mode == 5 || mode == 7 || mode == 8) ? 1.0 : 2.0;  // add/mul count 1
  return double(threads) * blocks * iters * 8 * 8 * lanes * flop / (best * 1e-3) / 1e12;
}

// n-body inner-loop probes: j-particles from __constant__ (uniform datapath)
// vs shared memory, same 12 i-particles per thread (6 packed pairs).
__constant__ float4 c_j[4096];

__device__ __forceinline__ float rsq_(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int SRC>  // 0: constant, 1: shared (duplicated pairs)
__global__ void __launch_bounds__(256, 1) k_nbody_probe(const float4* __restrict__ gj, int reps, float eps2,
                                                        float4* out) {
  constexpr int P = 6;
  __shared__ float4 sj[2 * 1024];
  float2 nx[P], ny[P], nz[P], ax[P], ay[P], az[P];
  for (int p = 0; p < P; ++p) {
    const float f = 0.001f * (threadIdx.x + 256 * p + blockIdx.x);
    nx[p] = make_float2(-f, -f - 0.1f);
    ny[p] = make_float2(f * 0.5f, f * 0.3f);
    nz[p] = make_float2(-f * 0.7f, f * 0.2f);
    ax[p] = ay[p] = az[p] = make_float2(0.f, 0.f);
  }
  if (SRC == 1) {
    for (int j = threadIdx.x; j < 1024; j += 256) {
      const float4 q = gj[j];
      sj[2 * j] = make_float4(q.x, q.x, q.y, q.y);
      sj[2 * j + 1] = make_float4(q.z, q.z, q.w, q.w);
    }
    __syncthreads();
  }
  const float2 e2 = make_float2(eps2, eps2);
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int j = 0; j < 1024; ++j) {
      float2 X, Y, Z, M;
      if (SRC == 0) {
        const float4 q = c_j[j];
        X = make_float2(q.x, q.x);
        Y = make_float2(q.y, q.y);
        Z = make_float2(q.z, q.z);
        M = make_float2(q.w, q.w);
      } else {
        const float4 A = sj[2 * j], B = sj[2 * j + 1];
        X = make_float2(A.x, A.y);
        Y = make_float2(A.z, A.w);
        Z = make_float2(B.x, B.y);
        M = make_float2(B.z, B.w);
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float2 rx = __fadd2_rn(X, nx[p]);
        const float2 ry = __fadd2_rn(Y, ny[p]);
        const float2 rz = __fadd2_rn(Z, nz[p]);
        float2 r2 = __ffma2_rn(rx, rx, e2);
        r2 = __ffma2_rn(ry, ry, r2);
        r2 = __ffma2_rn(rz, rz, r2);
        float2 w = make_float2(rsq_(r2.x), rsq_(r2.y));
        w = __fmul2_rn(w, __fmul2_rn(w, w));
        w = __fmul2_rn(w, M);
        ax[p] = __ffma2_rn(rx, w, ax[p]);
        ay[p] = __ffma2_rn(ry, w, ay[p]);
        az[p] = __ffma2_rn(rz, w, az[p]);
      }
    }
  }
  float s = 0.f;
  for (int p = 0; p < P; ++p) s += ax[p].x + ax[p].y + ay[p].x + ay[p].y + az[p].x + az[p].y;
  out[blockIdx.x * 256 + threadIdx.x] = make_float4(s, 0, 0, 0);
}

// Returns achieved "20-flop" TFLOP/s of the inner loop.
extern "C" double solomon_probe_nbody_inner(int src) {
  float4 h[4096];
  for (int j = 0; j < 4096; ++j) h[j] = make_float4(0.01f * (j % 97), 0.02f * (j % 89), -0.013f * (j % 83), 1e-3f);
  cudaMemcpyToSymbol(c_j, h, sizeof(h));
  float4 *gj = nullptr, *out = nullptr;
  cudaMalloc(&gj, sizeof(h));
  cudaMemcpy(gj, h, sizeof(h), cudaMemcpyHostToDevice);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 2, reps = 64;
  cudaMalloc(&out, sizeof(float4) * 256 * blocks);
  auto launch = [&] {
    if (src == 0)
      k_nbody_probe<0><<<blocks, 256>>>(gj, reps, 1e-4f, out);
    else
      k_nbody_probe<1><<<blocks, 256>>>(gj, reps, 1e-4f, out);
  };
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(gj);
  cudaFree(out);
  const double inter = double(blocks) * 256 * 12 * 1024.0 * reps;
  return 20.0 * inter / (ms * 1e-3) / 1e12;
}
