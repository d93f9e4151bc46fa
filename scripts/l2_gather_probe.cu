// Probe (tuning, not library): how long do 147 CTAs take to each read the same 64 KiB of
// 16-byte position words from L2 into shared memory -- the per-step gather of the
// persistent small-N leapfrog (k_leapfrog_small)? Variants: per-warp LDG.128 slices (16
// words per lane), the same with the slice order rotated per CTA, one cp.async.bulk per
// warp slice, and TMA multicast of 1/C of the words to all CTAs of a cluster of C.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/l2_gather_probe.cu -o scripts/l2_gather_probe
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

constexpr int N = 4096;
constexpr int THREADS = 256;
constexpr int REPS = 64;

__device__ __forceinline__ unsigned long long gclock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// mode 0: warp w reads words [512w, 512w+512) with __ldcg; mode 1: slice (w + blockIdx) % 8
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) k_ldg(const uint4* __restrict__ src, unsigned long long* out) {
  extern __shared__ uint4 sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long acc = 0;
  for (int r = 0; r < REPS; ++r) {
    __syncthreads();
    const unsigned long long t0 = gclock();
    const int sl = MODE == 1 ? (w + blockIdx.x) & 7 : w;
    const uint4* s = src + (r & 1) * N + sl * 512;
    uint4 q[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) q[k] = __ldcg(s + lane + 32 * k);
#pragma unroll
    for (int k = 0; k < 16; ++k) sm[sl * 512 + lane + 32 * k] = q[k];
    __syncthreads();
    acc += gclock() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / REPS;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase)
      : "memory");
}

// mode 2: one 8 KiB cp.async.bulk per warp slice (lane 0 issues), all 8 on one mbarrier
__global__ void __launch_bounds__(THREADS, 1) k_bulk(const uint4* __restrict__ src, unsigned long long* out) {
  extern __shared__ uint4 sm[];
  __shared__ alignas(8) uint64_t bar;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned long long acc = 0;
  for (int r = 0; r < REPS; ++r) {
    __syncthreads();
    const unsigned long long t0 = gclock();
    if (threadIdx.x == 0) mbar_expect(&bar, N * 16);
    __syncthreads();
    if (lane == 0) {
      const uint4* s = src + (r & 1) * N + w * 512;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (unsigned)__cvta_generic_to_shared(sm + w * 512)),
          "l"(s), "r"(512 * 16), "r"((unsigned)__cvta_generic_to_shared(&bar))
          : "memory");
    }
    mbar_wait(&bar, r & 1);
    acc += gclock() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / REPS;
}

// mode 3: clusters of C; CTA rank k of a cluster multicasts words [k N/C, (k+1) N/C) to all
// C CTAs (one bulk copy per warp of its share)
template <int C>
__global__ void __launch_bounds__(THREADS, 1) k_mcast(const uint4* __restrict__ src, unsigned long long* out) {
  extern __shared__ uint4 sm[];
  __shared__ alignas(8) uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cl.sync();
  unsigned long long acc = 0;
  constexpr int share = N / C, per_warp = share / 8;
  for (int r = 0; r < REPS; ++r) {
    cl.sync();  // every CTA's barrier armed for this round before anyone's copy lands
    const unsigned long long t0 = gclock();
    if (threadIdx.x == 0) mbar_expect(&bar, N * 16);
    cl.sync();
    if (lane == 0) {
      const int off = rank * share + w * per_warp;
      const uint4* s = src + (r & 1) * N + off;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
          "%4;" ::"r"((unsigned)__cvta_generic_to_shared(sm + off)),
          "l"(s), "r"(per_warp * 16), "r"((unsigned)__cvta_generic_to_shared(&bar)), "h"((unsigned short)((1 << C) - 1))
          : "memory");
    }
    mbar_wait(&bar, r & 1);
    acc += gclock() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / REPS;
}

// mode 4: the leapfrog's exchange pattern. Per round CTA b publishes its 28 words {x, y, z,
// tag} (plain stores, then a release of its ready word), each warp acquires the ready words
// of its slice's producers, reads the slice (__ldcg) and stores it to shared memory
// (P[j + j / chunk] with the mass from M[j], DIV = 1) or straight (DIV = 0). out: mean ns
// of [ready seen -> slice in shared memory] and of the whole round.
__device__ __forceinline__ uint4 ld_b128(const uint4* p) {
  unsigned long long lo, hi;
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(lo), "=l"(hi)
               : "l"(p)
               : "memory");
  return make_uint4(static_cast<unsigned>(lo), static_cast<unsigned>(lo >> 32), static_cast<unsigned>(hi),
                    static_cast<unsigned>(hi >> 32));
}
__device__ __forceinline__ uint4 ld_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// DIV: 0 __ldcg, 1 __ldcg + div, 2 ld.relaxed.b128, 3 ld.relaxed.v4
template <int DIV>
__global__ void __launch_bounds__(THREADS, 1) k_xchg(uint4* pub, unsigned int* ready, int chunk,
                                                     unsigned long long* out) {
  extern __shared__ float4 P4[];
  float* M = reinterpret_cast<float*>(P4 + N + 256);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int I = 28, i0 = blockIdx.x * I;
  for (int j = threadIdx.x; j < N; j += THREADS) M[j] = 1.f;
  __syncthreads();
  unsigned long long acc_read = 0, acc_round = 0;
  for (int r = 1; r <= REPS; ++r) {
    __syncthreads();
    const unsigned long long t0 = gclock();
    if (threadIdx.x < I && i0 + threadIdx.x < N)
      __stcg(pub + (r & 1) * N + i0 + threadIdx.x, make_uint4(1, 2, 3, r));
    if (threadIdx.x < 32) {
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + 32 * blockIdx.x), "r"(r) : "memory");
    }
    const int wj0 = w * 512, wj1 = wj0 + 512;
    for (int b = wj0 / I + lane; b <= (wj1 - 1) / I; b += 32) {
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + 32 * b) : "memory");
      } while (v < (unsigned)r);
    }
    __syncwarp();
    const unsigned long long t1 = gclock();
    const uint4* src = pub + (r & 1) * N;
    uint4 q[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      q[k] = DIV == 2 ? ld_b128(src + wj0 + lane + 32 * k)
                      : DIV == 3 ? ld_v4(src + wj0 + lane + 32 * k) : __ldcg(src + wj0 + lane + 32 * k);
    int bad = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int j = wj0 + lane + 32 * k;
      bad |= q[k].w != (unsigned)r;
      if (DIV == 1)
        P4[j + j / chunk] = make_float4(__uint_as_float(q[k].x), __uint_as_float(q[k].y), __uint_as_float(q[k].z), M[j]);
      else
        P4[j] = make_float4(__uint_as_float(q[k].x), __uint_as_float(q[k].y), __uint_as_float(q[k].z), 1.f);
    }
    __syncwarp();
    const unsigned long long t2 = gclock();
    if (bad) out[512 + blockIdx.x] = 1;
    acc_read += t2 - t1;
    __syncthreads();
    acc_round += gclock() - t0;
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x] = acc_read / REPS;
    out[128 + 256 + blockIdx.x] = acc_round / REPS;
  }
}

static void report(const char* name, unsigned long long* d, int ctas) {
  unsigned long long h[256];
  cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
  double s = 0, mx = 0;
  for (int i = 0; i < ctas; ++i) {
    s += h[i];
    mx = h[i] > mx ? h[i] : mx;
  }
  std::printf("%-28s ctas=%d  mean %.0f ns  max %.0f ns per 64 KiB gather (incl. 2 barriers)\n", name, ctas, s / ctas, mx);
}

int main() {
  uint4* src;
  cudaMalloc(&src, 2 * N * 16);
  cudaMemset(src, 0, 2 * N * 16);
  unsigned long long* out;
  cudaMalloc(&out, 256 * 8);
  const int smem = N * 16;
  cudaFuncSetAttribute(k_ldg<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_ldg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ctas : {1, 147}) {
    k_ldg<0><<<ctas, THREADS, smem>>>(src, out);
    cudaDeviceSynchronize();
    report("ldg per-warp slice", out, ctas);
    k_ldg<1><<<ctas, THREADS, smem>>>(src, out);
    cudaDeviceSynchronize();
    report("ldg rotated slices", out, ctas);
    k_bulk<<<ctas, THREADS, smem>>>(src, out);
    cudaDeviceSynchronize();
    report("bulk copy per warp", out, ctas);
  }
  {
    uint4* pub;
    unsigned int* ready;
    cudaMalloc(&pub, 2 * N * 16);
    cudaMalloc(&ready, 148 * 128);
    unsigned long long* o2;
    cudaMalloc(&o2, 1024 * 8);
    const int sm2 = (N + 256) * 16 + N * 4;
    for (int div : {0, 1, 2, 3}) {
      auto kern = div == 0 ? k_xchg<0> : div == 1 ? k_xchg<1> : div == 2 ? k_xchg<2> : k_xchg<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
      cudaMemset(pub, 0, 2 * N * 16);
      cudaMemset(ready, 0, 148 * 128);
      cudaMemset(o2, 0, 1024 * 8);
      void* args[] = {&pub, &ready, (void*)nullptr, &o2};
      int chunk = 32;
      args[2] = &chunk;
      cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, 147, THREADS, args, sm2, 0);
      cudaDeviceSynchronize();
      unsigned long long h[1024];
      cudaMemcpy(h, o2, sizeof h, cudaMemcpyDeviceToHost);
      double rd = 0, rnd = 0;
      int bad = 0;
      for (int b = 0; b < 147; ++b) {
        rd += h[b];
        rnd += h[384 + b];
        bad += h[512 + b] != 0;
      }
      std::printf("exchange (div=%d, %s): ready -> slice in smem %.0f ns, round %.0f ns, CTAs with stale words %d\n", div,
                  cudaGetErrorString(e), rd / 147, rnd / 147, bad);
    }
  }
  auto mc = [&](auto kern, int C, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int ctas : {C, 148 / C * C}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ctas);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const uint4*)src, out);
      cudaError_t e2 = cudaDeviceSynchronize();
      if (e != cudaSuccess || e2 != cudaSuccess) {
        std::printf("%s C=%d ctas=%d failed: %s / %s (max active clusters %d)\n", name, C, ctas, cudaGetErrorString(e),
                    cudaGetErrorString(e2), ncl);
        cudaGetLastError();
        continue;
      }
      char nm[64];
      std::snprintf(nm, sizeof nm, "%s C=%d (max clusters %d)", name, C, ncl);
      report(nm, out, ctas);
    }
  };
  mc(k_mcast<2>, 2, "multicast");
  mc(k_mcast<4>, 4, "multicast");
  mc(k_mcast<8>, 8, "multicast");
  mc(k_mcast<16>, 16, "multicast");
  return 0;
}
