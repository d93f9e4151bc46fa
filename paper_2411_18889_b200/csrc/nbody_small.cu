// K2' -- the whole small-N leapfrog run in one persistent launch (b2_leapfrog for
// n <= 32 x SMs). Reference force law: pkg/tests/fixtures/listing_nbody.c:1-27 via
// interact_bf (nbody_common.cuh); bit-identical to the two-kernel path of nbody.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "nbody_common.cuh"

namespace b2 {

// ---------------------------------------------------------------------------
// K2' small-N leapfrog: the whole KDK run in ONE persistent launch (BASELINE
// configs[0]: N=4096, where the two-kernel step is ~20 us of launch gaps,
// under-filled force tiles and a latency-bound reduce for ~6 us of arithmetic).
//
// One CTA per I <= 32 i-particles (I/2 packed pairs; I sized so the grid spans
// every SM: 28 at N=4096 -> 147 CTAs), all CTAs co-resident
// (cooperative launch). Each step every CTA gathers ALL positions into shared
// memory, computes its i-particles' forces chunk by chunk, reduces the chunk
// partials and applies the kicks and drift. Positions travel between CTAs as
// self-validating 16-byte words {x, y, z, step tag} (masses never change, so
// the tag takes .w's place; each CTA keeps the masses it gathers in registers):
// a .b128 store/load is single-copy atomic, so consumers poll the data itself
// -- no grid barrier, no fence. A word that never arrives ends the run through
// the watchdog (poll_expired, runtime.cu) instead of hanging. Two tag parities suffice: a CTA publishes step
// s+2's positions only after gathering every CTA's step s+1 positions, which
// each CTA publishes only after it finished reading step s's.
//
// Bit-identical to the two-kernel path (b2_calc_acc_partials + b2_kdk_update):
// same j-chunks (chunk_size depends on N only), each chunk summed in j order
// with the same packed-FP32 interaction, partials summed c = 0, 1, ... and the
// same FMA kick/drift sequence.
constexpr int kSmallThreads = 512;
// Force-phase shape (swept with scripts/trace_small.cu at N=4096: 2 pairs x
// unroll 2 over 147 CTAs 10.5 us/force; unroll 1: 11.3; 4 pairs over 128 CTAs: 11.5).
#ifndef B2_SMALL_UNROLL
#define B2_SMALL_UNROLL 2
#endif
constexpr int kSmallUnroll = B2_SMALL_UNROLL;
#ifndef B2_SMALL_PAIRS
#define B2_SMALL_PAIRS 2
#endif
constexpr int kSmallPairs = B2_SMALL_PAIRS;  // packed i-pairs per thread in the force phase
#ifndef B2_SMALL_RBATCH
#define B2_SMALL_RBATCH 8  // chunk partials loaded per batch in the in-order reduce
#endif
constexpr int kSmallImax = 32;     // i-particles per CTA (at most; a multiple of 4)
constexpr int kSmallGather = 10;   // positions gathered per thread: n <= 10 * 512

struct SmallArgs {
  int n;
  float4* pos;
  float4* vel;
  float4* acc;
  uint4* pub;  // [2][n] tagged positions, zeroed before launch
  float eps2, dt, h;
  int nsteps, flags;  // B2_POTENTIAL | B2_INIT_ACC
  int chunk, nch;
  int I;  // i-particles per CTA: 4 * ceil(n / (4 * SMs)) <= 32, so the grid spans every SM
  Watch watch;  // a position word that never arrives ends the run (runtime.cu), no trap
#ifdef B2_SMALL_TRACE
  unsigned long long* trace;  // [cta][step][4] globaltimer stamps (scripts/trace_small.cu)
#endif
};
#ifdef B2_SMALL_TRACE
#define B2_STRACE(k) \
  if (tid == 0) a.trace[(static_cast<size_t>(blockIdx.x) * a.nsteps + st) * 4 + (k)] = globaltimer_ns()
#else
#define B2_STRACE(k)
#endif


template <bool POT>
__global__ void __launch_bounds__(kSmallThreads, 1) k_leapfrog_small(const SmallArgs a) {
  extern __shared__ float4 sm4[];
  const int n = a.n, tid = threadIdx.x;
  float4* P = sm4;                   // positions {x, y, z, m} of the current state, j at j + j / chunk
  const int IB = a.I;                // i-particles per CTA (the last CTA may own fewer)
  float4* part = sm4 + n + a.nch;    // [nch][IB] chunk partials of this CTA's i
  float* M = reinterpret_cast<float*>(part + a.nch * IB);  // [n] masses (constant)
  const int i0 = blockIdx.x * IB;
  const int I = min(IB, n - i0);

  // state 0: every position straight from pos (nobody writes pos before the end)
  for (int j = tid; j < n; j += kSmallThreads) {
    const float4 q = a.pos[j];
    P[j + j / a.chunk] = q;
    M[j] = q.w;
  }
  // own particle (threads tid < I): i = i0 + tid
  float4 x = make_float4(0.f, 0.f, 0.f, 0.f), v = x, acc = x;
  if (tid < I) {
    x = a.pos[i0 + tid];
    v = a.vel[i0 + tid];
    if (!(a.flags & B2_INIT_ACC)) acc = a.acc[i0 + tid];  // else computed below (acc may be uninitialised)
  }
  const float2 e2 = make_float2(a.eps2, a.eps2);
  __syncthreads();

  // forces on this CTA's i from the positions in P -> acc (threads tid < I).
  // Task = (group g of 2 packed pairs = 4 i, chunk c): thread tid -> g = tid % 8,
  // c = tid / 8, so nch <= 64 chunks (kTargetChunks) need one task per thread; a
  // warp reads 4 chunks' j at a time, P padded by one float4 per chunk so those
  // four addresses fall in different banks.
  auto force = [&]() {
    constexpr int NP = kSmallPairs;
    const int G = IB / (2 * NP), H = IB / 2;  // groups of NP pairs; pair p of group g = (i0+NP*g+p, i0+H+NP*g+p)
    const int g = tid % G, c = tid / G;
    if (c < a.nch) {
      float2 nx[NP], ny[NP], nz[NP], ax[NP], ay[NP], az[NP], ap[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int ia = min(i0 + NP * g + p, n - 1), ib = min(i0 + H + NP * g + p, n - 1);
        const float4 pa = P[ia + ia / a.chunk], pb = P[ib + ib / a.chunk];
        nx[p] = make_float2(-pa.x, -pb.x);
        ny[p] = make_float2(-pa.y, -pb.y);
        nz[p] = make_float2(-pa.z, -pb.z);
        ax[p] = ay[p] = az[p] = ap[p] = make_float2(0.f, 0.f);
      }
      const float4* q = P + c * (a.chunk + 1);
      const int len = min(a.chunk, n - c * a.chunk);
      float4 pj = q[0];
#pragma unroll kSmallUnroll
      for (int jj = 0; jj < len; ++jj) {
        const float4 pn = q[jj + 1];  // next j one iteration ahead (the padding slot makes q[len] readable)
        interact_bf<NP, POT>(make_float2(pj.x, pj.x), make_float2(pj.y, pj.y), make_float2(pj.z, pj.z),
                             make_float2(pj.w, pj.w), nx, ny, nz, e2, ax, ay, az, ap);
        pj = pn;
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        part[c * IB + NP * g + p] = make_float4(ax[p].x, ay[p].x, az[p].x, POT ? ap[p].x : 0.f);
        part[c * IB + H + NP * g + p] = make_float4(ax[p].y, ay[p].y, az[p].y, POT ? ap[p].y : 0.f);
      }
    }
    __syncthreads();
    if (tid < I) {  // fixed order c = 0, 1, ..., as k_kdk_update
      float4 s = part[tid];
      int cc = 1;
#if B2_SMALL_RBATCH > 1
      for (; cc + B2_SMALL_RBATCH <= a.nch; cc += B2_SMALL_RBATCH) {  // loads in flight together, adds in order
        float4 q[B2_SMALL_RBATCH];
#pragma unroll
        for (int u = 0; u < B2_SMALL_RBATCH; ++u) q[u] = part[(cc + u) * IB + tid];
#pragma unroll
        for (int u = 0; u < B2_SMALL_RBATCH; ++u) {
          s.x = __fadd_rn(s.x, q[u].x);
          s.y = __fadd_rn(s.y, q[u].y);
          s.z = __fadd_rn(s.z, q[u].z);
          s.w = __fadd_rn(s.w, q[u].w);
        }
      }
#endif
      for (; cc < a.nch; ++cc) {
        const float4 p = part[cc * IB + tid];
        s.x = __fadd_rn(s.x, p.x);
        s.y = __fadd_rn(s.y, p.y);
        s.z = __fadd_rn(s.z, p.z);
        s.w = __fadd_rn(s.w, p.w);
      }
      acc = s;
    }
  };
  auto kick_drift = [&](float h_begin) {  // B2_KDK_KICK_DRIFT
    v.x = __fmaf_rn(acc.x, h_begin, v.x);
    v.y = __fmaf_rn(acc.y, h_begin, v.y);
    v.z = __fmaf_rn(acc.z, h_begin, v.z);
    x.x = __fmaf_rn(v.x, a.dt, x.x);
    x.y = __fmaf_rn(v.y, a.dt, x.y);
    x.z = __fmaf_rn(v.z, a.dt, x.z);
  };
  auto publish = [&](int state) {
    if (tid < I)
      st_relaxed_b128(a.pub + static_cast<size_t>(state & 1) * n + i0 + tid,
                      make_uint4(__float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z),
                                 static_cast<unsigned int>(state)));
  };
  auto gather = [&](int state) {
    const uint4* src = a.pub + static_cast<size_t>(state & 1) * n;
    const unsigned int want = static_cast<unsigned int>(state);
    const unsigned long long t0 = globaltimer_ns();
    bool dead = false;
#pragma unroll
    for (int k0 = 0; k0 < kSmallGather; k0 += kSmallGather / 2) {  // two batches of in-flight loads
      constexpr int B = kSmallGather / 2;
      uint4 w[B];
      unsigned int todo = 0;
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int j = tid + (k0 + k) * kSmallThreads;
        if (j < n) {
          w[k] = ld_relaxed_b128(src + j);
          todo |= 1u << k;
        }
      }
      while (todo) {
#pragma unroll
        for (int k = 0; k < B; ++k) {
          if (!(todo >> k & 1)) continue;
          const int j = tid + (k0 + k) * kSmallThreads;
          if (w[k].w == want) {
            P[j + j / a.chunk] =
                make_float4(__uint_as_float(w[k].x), __uint_as_float(w[k].y), __uint_as_float(w[k].z), M[j]);
            todo &= ~(1u << k);
          } else {
            w[k] = ld_relaxed_b128(src + j);
          }
        }
        if (todo && poll_expired(a.watch, t0, kFaultLeapfrogSmall)) {  // a CTA never published: give up
          dead = true;
          break;
        }
      }
    }
    // barrier + CTA-wide vote (no static shared memory: the dynamic allocation may use it all);
    // false: leave without writing pos / vel / acc (b2_fault_status reports it)
    return !__syncthreads_or(dead);
  };

  const float h = a.h;
  if (a.flags & B2_INIT_ACC) force();
  if (a.nsteps > 0) {
    if (tid < I) kick_drift(h);  // opening kick + drift of step 0
    publish(1);
    for (int st = 0; st < a.nsteps; ++st) {
      B2_STRACE(0);
      __syncthreads();  // everyone is done reading P
      if (!gather(st + 1)) return;
      B2_STRACE(1);
      force();
      B2_STRACE(2);
      if (tid < I) {
        v.x = __fmaf_rn(acc.x, h, v.x);  // closing kick (B2_KDK_KICK_END)
        v.y = __fmaf_rn(acc.y, h, v.y);
        v.z = __fmaf_rn(acc.z, h, v.z);
        if (st + 1 < a.nsteps) kick_drift(h);
      }
      if (st + 1 < a.nsteps) publish(st + 2);
      B2_STRACE(3);
    }
  }
  if (tid < I) {
    a.pos[i0 + tid] = x;
    a.vel[i0 + tid] = v;
    a.acc[i0 + tid] = acc;
  }
}

// The persistent small-N path of b2_leapfrog (k_leapfrog_small), when it applies:
// fast arithmetic, n <= 32 x SMs, >= 2 j-chunks, tasks/gathers within the
// per-thread budgets, shared memory fits, and the workspace holds the [2][n]
// tagged-position buffer. Returns false (nothing launched) otherwise.
bool launch_leapfrog_small(int n, float4* pos, float4* vel, float4* acc, float eps, float dt, int nsteps,
                                  int flags, void* workspace, size_t workspace_bytes, cudaStream_t s) {
  static const int enabled = [] {
    const char* e = std::getenv("SOLOMON_NBODY_PERSISTENT");
    return e ? std::atoi(e) : 1;
  }();
  if (!enabled || (flags & B2_EXACT)) return false;
  const int nch = nchunks_for(n, flags & B2_POTENTIAL);
  const DeviceInfo& di = device_info();
  const int I = 2 * kSmallPairs * ((n + 2 * kSmallPairs * di.sms - 1) / (2 * kSmallPairs * di.sms));
  const int ctas = (n + I - 1) / I;
  const size_t smem = (static_cast<size_t>(n) + nch + static_cast<size_t>(nch) * I) * sizeof(float4) +
                      static_cast<size_t>(n) * sizeof(float);
  if (nch < 2 || I > kSmallImax || ctas > di.sms || n > kSmallGather * kSmallThreads || (I / (2 * kSmallPairs)) * nch > kSmallThreads ||
      smem > static_cast<size_t>(di.smem_optin) ||
      workspace_bytes < 2 * static_cast<size_t>(n) * sizeof(uint4))
    return false;
  const bool pot = flags & B2_POTENTIAL;
  const void* fn = pot ? reinterpret_cast<const void*>(k_leapfrog_small<true>)
                       : reinterpret_cast<const void*>(k_leapfrog_small<false>);
  allow_max_dynamic_smem(fn);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSmallThreads, smem) != cudaSuccess ||
      per_sm * di.sms < ctas) {
    cudaGetLastError();
    return false;
  }
  uint4* pub = static_cast<uint4*>(workspace);
  if (cudaMemsetAsync(pub, 0, 2 * static_cast<size_t>(n) * sizeof(uint4), s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  SmallArgs args{n, pos, vel, acc, pub, eps * eps, dt, 0.5f * dt, nsteps, flags & (B2_POTENTIAL | B2_INIT_ACC),
                 chunk_size(n, flags & B2_POTENTIAL), nch, I, make_watch()};
  void* argv[] = {&args};
  if (cudaLaunchCooperativeKernel(fn, ctas, kSmallThreads, argv, smem, s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

}  // namespace b2
