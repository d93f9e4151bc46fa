// Shared pieces of the n-body kernels (nbody.cu, nbody_small.cu): chunking of the
// j-sum (depends on Nj only, so sharded and unsharded runs sum in the same order),
// MUFU helpers and the packed-FP32 interaction of listing_nbody.c:9-20.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace b2 {

constexpr int kChunkAlign = 64;    // j-chunk sizes are multiples of this
constexpr int kTargetChunks = 64;  // j-chunks per force evaluation (fast path)

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---------------------------------------------------------------------------
// K1 fast: packed-FP32 tile kernel.
// grid.x = n_itiles * nchunks; block = BLOCK threads; out = partials[c][Ni].
// One j against the thread's P = IPT/2 packed i-pairs, written stage by stage
// across the pairs (breadth-first) so every dependent FP32 op has P-1
// independent ones in front of it -- the fixed-latency FFMA2 chain of
// listing_nbody.c:14 otherwise leaves the FMA pipe idle (ncu "stall wait").
template <int P, bool POT>
__device__ __forceinline__ void interact_bf(const float2 X, const float2 Y, const float2 Z, const float2 M,
                                            const float2 (&nx)[P], const float2 (&ny)[P], const float2 (&nz)[P],
                                            const float2 e2, float2 (&ax)[P], float2 (&ay)[P], float2 (&az)[P],
                                            float2 (&ap)[P]) {
  float2 rx[P], ry[P], rz[P], r2[P], w[P];
#pragma unroll
  for (int p = 0; p < P; ++p) rx[p] = __fadd2_rn(X, nx[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) ry[p] = __fadd2_rn(Y, ny[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) rz[p] = __fadd2_rn(Z, nz[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) r2[p] = __ffma2_rn(rx[p], rx[p], e2);
#pragma unroll
  for (int p = 0; p < P; ++p) r2[p] = __ffma2_rn(ry[p], ry[p], r2[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) r2[p] = __ffma2_rn(rz[p], rz[p], r2[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) w[p] = make_float2(rsqrt_approx(r2[p].x), rsqrt_approx(r2[p].y));
  float2 w2[P];
#pragma unroll
  for (int p = 0; p < P; ++p) w2[p] = __fmul2_rn(w[p], w[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) w[p] = __fmul2_rn(w[p], w2[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) w[p] = __fmul2_rn(w[p], M);
#pragma unroll
  for (int p = 0; p < P; ++p) ax[p] = __ffma2_rn(rx[p], w[p], ax[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) ay[p] = __ffma2_rn(ry[p], w[p], ay[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) az[p] = __ffma2_rn(rz[p], w[p], az[p]);
  if (POT) {
#pragma unroll
    for (int p = 0; p < P; ++p) ap[p] = __ffma2_rn(r2[p], w[p], ap[p]);
  }
}

// j-chunk size, a function of Nj only (so sharded and unsharded runs sum in the same
// order). Large Nj: ~64 chunks, 64-aligned (the tile kernel's waves and ring). Nj up to
// kFineChunkNj: ~128 chunks, 32-aligned -- the persistent small-N leapfrog's parallelism
// is (own particles / 2) x chunks per SM, and 128 chunks give it 8 warps x 7 packed pairs
// at N = 4096 (64 chunks left it at 14 warps x 2 pairs, ~55% of the FMA pipe). Up to
// kAlign32Nj: ~64 chunks, 32-aligned, so that its 4 pair groups x chunks fill 8 warps
// evenly (9472: 60 chunks of 160 instead of 50 of 192, which left 7 warps on 4 schedulers).
constexpr int kFineChunkNj = 4736, kAlign32Nj = 9472;
constexpr int kFineChunks = 128, kFineAlign = 32;
inline int chunk_size(int Nj, int flags) {
  if (flags & B2_EXACT) return Nj;
  const int target = Nj <= kFineChunkNj ? kFineChunks : kTargetChunks;
  const int align = Nj <= kAlign32Nj ? kFineAlign : kChunkAlign;
  int c = (Nj + target - 1) / target;
  c = (c + align - 1) / align * align;
  return std::max(c, align);
}

inline int nchunks_for(int Nj, int flags) {
  if (Nj <= 0) return 0;
  const int c = chunk_size(Nj, flags);
  return (Nj + c - 1) / c;
}

// The persistent small-N path of b2_leapfrog (nbody_small.cu); false = not applicable,
// nothing launched.
size_t small_workspace_bytes(int n);
bool launch_leapfrog_small(int n, float4* pos, float4* vel, float4* acc, float eps, float dt, int nsteps, int flags,
                           void* workspace, size_t workspace_bytes, cudaStream_t s);

}  // namespace b2
