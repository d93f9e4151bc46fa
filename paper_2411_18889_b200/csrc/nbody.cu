// K1: direct-summation softened gravity (calc_acc) and K2: fused leapfrog
// update, hand-written for sm_100a.
//
// Reference: pkg/tests/fixtures/listing_nbody.c:1-27 (= PAPER.md:467-493).
//   for i < Ni:                 (parallel, :2-3)
//     pi = ipos[i]; pi.w = eps^2                                  (:4-5)
//     for j < Nj:               (sequential, :7-8)
//       r  = pj - pi                                              (:11-13)
//       r2 = fma(rz,rz, fma(ry,ry, fma(rx,rx, eps^2)))            (:14)
//       w  = 1/sqrt(r2); w *= w*w; w *= m_j                       (:15-17)
//       a += r*w  (3 FMA); [pot: a.w = fma(r2, w, a.w)]           (:18-23)
//
// Fast kernel design: FP32 CUDA-core work (not a contraction,
// so no tensor cores). Each thread owns IPT=16 i-particles as 8 packed pairs
// (default variant 0: 128 threads, 2 CTAs/SM) and evaluates every interaction
// with Blackwell's packed FP32 instructions (FADD2/FFMA2/FMUL2 -- 12 issue
// slots per 2 interactions instead of 24) plus MUFU.RSQ. j-particles stream
// through shared memory in BLOCK-sized tiles, double-buffered; one LDS.128 per
// j feeds the packed ops as scalar-broadcast operands (SCHED 2; the older
// pre-duplicated {x,x,y,y},{z,z,m,m} layout survives as SCHED 0/1 variants).
// Nj is cut into fixed chunks whose size
// depends on Nj only; each (i-tile, j-chunk) is one CTA of work, giving >50
// waves at N=2^20 (no tail), and per-chunk partial sums are combined in a
// fixed order by the K2 update kernel (deterministic, shard-invariant).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "nbody_common.cuh"

namespace b2 {

// shared constants, helpers and interact_bf: nbody_common.cuh

// Depth-first form (one pair at a time), kept as a tuning variant.
template <int P, bool POT>
__device__ __forceinline__ void interact_df(const float2 X, const float2 Y, const float2 Z, const float2 M,
                                            const float2 (&nx)[P], const float2 (&ny)[P], const float2 (&nz)[P],
                                            const float2 e2, float2 (&ax)[P], float2 (&ay)[P], float2 (&az)[P],
                                            float2 (&ap)[P]) {
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const float2 rx = __fadd2_rn(X, nx[p]);
    const float2 ry = __fadd2_rn(Y, ny[p]);
    const float2 rz = __fadd2_rn(Z, nz[p]);
    float2 r2 = __ffma2_rn(rx, rx, e2);
    r2 = __ffma2_rn(ry, ry, r2);
    r2 = __ffma2_rn(rz, rz, r2);
    float2 w = make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
    w = __fmul2_rn(w, __fmul2_rn(w, w));
    w = __fmul2_rn(w, M);
    ax[p] = __ffma2_rn(rx, w, ax[p]);
    ay[p] = __ffma2_rn(ry, w, ay[p]);
    az[p] = __ffma2_rn(rz, w, az[p]);
    if (POT) ap[p] = __ffma2_rn(r2, w, ap[p]);
  }
}

// Pairs [0, P-ALT) on the reference formula (rsqrt, cube, mass), pairs
// [P-ALT, P) on s = ex2(fma(-1.5, lg2(r2), lg2(m_j))).
template <int P, int ALT, bool POT>
__device__ __forceinline__ void interact_mixed(const float2 X, const float2 Y, const float2 Z, const float2 M,
                                               const float LM, const float2 (&nx)[P], const float2 (&ny)[P],
                                               const float2 (&nz)[P], const float2 e2, float2 (&ax)[P],
                                               float2 (&ay)[P], float2 (&az)[P], float2 (&ap)[P]) {
  const float2 lm = make_float2(LM, LM);
  const float2 k15 = make_float2(-1.5f, -1.5f);
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const float2 rx = __fadd2_rn(X, nx[p]);
    const float2 ry = __fadd2_rn(Y, ny[p]);
    const float2 rz = __fadd2_rn(Z, nz[p]);
    float2 r2 = __ffma2_rn(rx, rx, e2);
    r2 = __ffma2_rn(ry, ry, r2);
    r2 = __ffma2_rn(rz, rz, r2);
    float2 w;
    if (p < P - ALT) {
      w = make_float2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
      w = __fmul2_rn(w, __fmul2_rn(w, w));
      w = __fmul2_rn(w, M);
    } else {
      const float2 l = make_float2(lg2_approx(r2.x), lg2_approx(r2.y));
      const float2 y = __ffma2_rn(l, k15, lm);
      w = make_float2(ex2_approx(y.x), ex2_approx(y.y));
    }
    ax[p] = __ffma2_rn(rx, w, ax[p]);
    ay[p] = __ffma2_rn(ry, w, ay[p]);
    az[p] = __ffma2_rn(rz, w, az[p]);
    if (POT) ap[p] = __ffma2_rn(r2, w, ap[p]);
  }
}

// In-kernel, in-order reduction of the j-chunk partials (Fused.ring set).
// The grid is ordered chunk-minor (blockIdx = itile * nch + chunk), so the nch CTAs of one
// i-tile run at about the same time. Each writes its partial tile into ring slot
// itile % R of a ring of R tiles x nch x BLOCK*IPT float4 and arrives on the slot's
// counter; the LAST arriving CTA sums the slot's partials in the fixed order c = 0, 1,
// ..., nch-1 -- the order k_kdk_update uses, so the bits are those of the two-kernel path
// -- writes acc, drops the slot's lines from L2 without write-back (discard.global.L2) and
// opens the slot for i-tile itile + R. A CTA waits for its slot only if the reduction of
// i-tile itile - R (R * nch = 2048 CTAs earlier in launch order, ~7 waves at N = 2^20) has
// not finished -- which in-order CTA dispatch never lets happen; the watchdog bounds the
// wait regardless. The work item comes from blockIdx, not a ticket counter: a value loaded
// from shared memory is not provably warp-uniform, which moved the j loop off the uniform
// datapath (1.9% slower, measured). Scratch: R * nch * tile * 16 B (64 MiB at nch = 64)
// instead of nch * Ni * 16 B (1 GiB at N = 2^20, 4 GiB at 2^22), and the partials never
// reach HBM (ncu: 22 MB of DRAM traffic per launch at N = 2^20, was 1.18 GB).
struct Fused {
  float4* ring;         // [R][nch][tile] partial tiles
  unsigned int* ctrl;   // [0..R) arrivals per slot, [R .. 2R) i-tiles that went through each slot
  float4* acc;          // [Ni] result
  int R;                // ring slots
  Watch watch;
};
constexpr int kRingSlots = 32;         // of the largest tile (2048 i); smaller tiles get more
constexpr int kMaxRingSlots = 1024;    // control words: arrivals + gates per slot
constexpr size_t kRingCtrlBytes = 2 * kMaxRingSlots * sizeof(unsigned int);  // zeroed per launch

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// The fused force kernel's ring protocol, out of line on purpose: inlined, the extra code
// perturbed ptxas's schedule of the j loop (register banks, operand-reuse flags) and cost
// 1.2-2.5% at N = 2^20 (measured); as calls it costs two calls per CTA. ring_wait: wait
// until the i-tile's ring slot is free (i-tile itile - R reduced). ring_finish: arrive on
// the slot; the last chunk CTA sums the slot's partials in the fixed order c = 0..nch-1 (as
// k_kdk_update), writes acc, discards the slot's L2 lines and opens the slot for itile + R.
__device__ __noinline__ void ring_wait(const Fused& fz, int itile) {
  if (threadIdx.x == 0) {
    const unsigned int want = static_cast<unsigned int>(itile / fz.R);
    const unsigned int* gate = fz.ctrl + fz.R + itile % fz.R;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_u32(gate) != want)
      if (poll_timed_out(fz.watch, t0, kFaultForceRing)) break;
  }
  __syncthreads();
}

template <int BLOCK, int kIPT>
__device__ __noinline__ void ring_finish(const Fused& fz, int nch, int itile, int Ni) {
  constexpr int TILE = BLOCK * kIPT;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int slot = itile % fz.R;
  unsigned int* arrive = fz.ctrl + slot;
  unsigned int* gate = fz.ctrl + fz.R + slot;
  const float4* __restrict__ tile = fz.ring + static_cast<size_t>(slot) * nch * TILE;
  __syncthreads();
  if (tid == 0) {
    __threadfence();  // publish this CTA's partials before arriving
    s_last = atomicAdd(arrive, 1u) == static_cast<unsigned int>(nch - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();  // acquire side: the other chunks' partials are visible
  // fixed summation order c = 0, 1, ..., nch-1 (as k_kdk_update): batches of loads in flight
#pragma unroll 1
  for (int e = 0; e < kIPT; ++e) {
    const int il = tid + e * BLOCK;
    const float4* __restrict__ col = tile + il;
    float4 a = __ldcg(col);
    constexpr int B = 16;
    for (int c0 = 1; c0 < nch; c0 += B) {
      float4 q[B];
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (c0 + b < nch) q[b] = __ldcg(col + static_cast<size_t>(c0 + b) * TILE);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (c0 + b < nch) {
          a.x = __fadd_rn(a.x, q[b].x);
          a.y = __fadd_rn(a.y, q[b].y);
          a.z = __fadd_rn(a.z, q[b].z);
          a.w = __fadd_rn(a.w, q[b].w);
        }
      }
    }
    const int i = itile * TILE + il;
    if (i < Ni) fz.acc[i] = a;
  }
  __syncthreads();  // every read of the slot is done
  // drop the slot's lines from L2 without writing them back: the partials never reach HBM
  for (size_t l = tid; l < static_cast<size_t>(nch) * TILE / 8; l += BLOCK) discard_l2_line(tile + 8 * l);
  __syncthreads();
  if (tid == 0) {
    *arrive = 0u;
    st_release_u32(gate, static_cast<unsigned int>(itile / fz.R + 1));  // open the slot for itile + R
  }
}

// SCHED: 0 depth-first / 1 breadth-first source order (ptxas mostly reschedules).
// SCHED 2: j-values kept NON-duplicated in shared memory and fed to the packed
// ops as scalar-broadcast operands (FADD2 R, R.F32x2, R.F32): one LDS.128 per j
// and one fewer register-pair read per FADD2/FMUL2 -- the register file read
// bandwidth, not the FMA datapath, is what caps this loop (probe: FFMA2 with
// three distinct register pairs runs at 52% of peak).
//
// ALT > 0 moves the last ALT pairs of every thread onto a second formula that
// trades FMA-pipe work for MUFU work: m r^-3 = ex2(fma(-1.5, lg2(r2), lg2(m)))
// -- 2 MUFU + 1 FFMA2 per pair instead of 1 MUFU + 3 FMUL2 -- so the FP32
// pipe (the binding one) and the MUFU pipe (58% busy) are balanced.
template <int BLOCK, int kIPT, int MINB, int UNR, int SCHED, int ALT, bool POT>
__global__ void __launch_bounds__(BLOCK, MINB)
    k_force_fast(const float4* __restrict__ ipos, int Ni, const float4* __restrict__ jpos, int Nj,
                 int jchunk, int n_itiles, float eps2, float4* __restrict__ out, const Fused fz) {
  constexpr int P = kIPT / 2;
  constexpr int DUP = SCHED >= 2 ? 1 : 2;  // float4 slots per j in shared memory
  static_assert(ALT == 0 || DUP == 1, "ALT path uses scalar-broadcast j");
  __shared__ float4 sj[2][DUP * BLOCK];
  __shared__ float slm[2][ALT > 0 ? BLOCK : 1];
  const int tid = threadIdx.x;
  const int nch = gridDim.x / n_itiles;
  // fz.ring set: in-kernel reduction; null: partials out. One kernel serves both modes -- a
  // separate fused instantiation scheduled the j loop differently and ran 1.2-2.5% slower.
  const bool fused = fz.ring != nullptr;
  // fused: chunk-minor, the chunks of an i-tile run together (what the ring needs); partials:
  // i-tile-minor, the CTAs running together share their j-chunk (mid N, small CTAs)
  const int itile = fused ? blockIdx.x / nch : blockIdx.x % n_itiles;
  const int chunk = fused ? blockIdx.x % nch : blockIdx.x / n_itiles;
  const int ibase = itile * (BLOCK * kIPT) + tid;
  if (fused) ring_wait(fz, itile);  // ring slot free? (i-tile itile - R reduced: never waits in practice)

  float2 nx[P], ny[P], nz[P];
  float2 ax[P], ay[P], az[P], ap[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int ia = min(ibase + (2 * p) * BLOCK, Ni - 1);
    const int ib = min(ibase + (2 * p + 1) * BLOCK, Ni - 1);
    const float4 a = __ldg(ipos + ia), b = __ldg(ipos + ib);
    // r = pj - pi computed as pj + (-pi): identical in IEEE arithmetic.
    nx[p] = make_float2(-a.x, -b.x);
    ny[p] = make_float2(-a.y, -b.y);
    nz[p] = make_float2(-a.z, -b.z);
    ax[p] = ay[p] = az[p] = ap[p] = make_float2(0.f, 0.f);
  }
  const float2 e2 = make_float2(eps2, eps2);

  const int j0 = chunk * jchunk;
  const int j1 = min(j0 + jchunk, Nj);
  const int ntiles = (j1 - j0 + BLOCK - 1) / BLOCK;

  // Padding j (beyond j1) gets m = 0 far away (1e18 on every axis): r2 ~ 3e36 stays
  // finite, w = rsqrt(r2)^3 * 0 = 0, so it adds exactly +0 -- also for eps = 0 and an
  // i-particle at the origin, where a padding j AT the origin would give inf * 0 = NaN.
  auto fetch = [&](int t) -> float4 {
    const int j = j0 + t * BLOCK + tid;
    return j < j1 ? __ldg(jpos + j) : make_float4(1e18f, 1e18f, 1e18f, 0.f);
  };
  auto stash = [&](int buf, float4 pj) {
    if (DUP == 1) {
      sj[buf][tid] = pj;
      if (ALT > 0) slm[buf][tid] = lg2_approx(pj.w);  // -inf for m = 0: contributes 0
    } else {
      sj[buf][2 * tid + 0] = make_float4(pj.x, pj.x, pj.y, pj.y);
      sj[buf][2 * tid + 1] = make_float4(pj.z, pj.z, pj.w, pj.w);
    }
  };

  stash(0, fetch(0));
  __syncthreads();

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    float4 next;
    const bool more = (t + 1) < ntiles;
    if (more) next = fetch(t + 1);

    const float4* __restrict__ s = sj[buf];
#pragma unroll UNR
    for (int jj = 0; jj < BLOCK; ++jj) {
      float2 X, Y, Z, M;
      float LM = 0.f;
      if (ALT > 0) LM = slm[buf][jj];
      if (DUP == 1) {
        const float4 q = s[jj];
        X = make_float2(q.x, q.x);
        Y = make_float2(q.y, q.y);
        Z = make_float2(q.z, q.z);
        M = make_float2(q.w, q.w);
      } else {
        const float4 A = s[2 * jj + 0];
        const float4 B = s[2 * jj + 1];
        X = make_float2(A.x, A.y);
        Y = make_float2(A.z, A.w);
        Z = make_float2(B.x, B.y);
        M = make_float2(B.z, B.w);
      }
      if (ALT > 0)
        interact_mixed<P, ALT, POT>(X, Y, Z, M, LM, nx, ny, nz, e2, ax, ay, az, ap);
      else if (SCHED >= 1)
        interact_bf<P, POT>(X, Y, Z, M, nx, ny, nz, e2, ax, ay, az, ap);
      else
        interact_df<P, POT>(X, Y, Z, M, nx, ny, nz, e2, ax, ay, az, ap);
    }
    if (more) stash(buf ^ 1, next);
    __syncthreads();
  }

  // partials: [chunk][Ni] (unfused), or this chunk's row of the i-tile's ring slot (fused) --
  // the same store code either way (it shares the register allocation of the j loop)
  constexpr int TILE = BLOCK * kIPT;
  float4* __restrict__ o = fused ? fz.ring + (static_cast<size_t>(itile % fz.R) * nch + chunk) * TILE -
                                       static_cast<size_t>(itile) * TILE
                                 : out + static_cast<size_t>(chunk) * Ni;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int ia = ibase + (2 * p) * BLOCK;
    const int ib = ibase + (2 * p + 1) * BLOCK;
    if (ia < Ni) o[ia] = make_float4(ax[p].x, ay[p].x, az[p].x, POT ? ap[p].x : 0.f);
    if (ib < Ni) o[ib] = make_float4(ax[p].y, ay[p].y, az[p].y, POT ? ap[p].y : 0.f);
  }
  if (fused) ring_finish<BLOCK, kIPT>(fz, nch, itile, Ni);  // the last chunk CTA of the i-tile reduces the slot
}


// ---------------------------------------------------------------------------
// K1 exact: the reference's arithmetic, bit for bit (IEEE sqrt and divide,
// explicit roundings so nvcc cannot contract, sequential j). One i per thread.
template <bool POT>
__global__ void __launch_bounds__(128)
    k_force_exact(const float4* __restrict__ ipos, int Ni, const float4* __restrict__ jpos, int Nj, float eps2,
                  float4* __restrict__ out) {
  constexpr int T = 128;
  __shared__ float4 sj[T];
  const int i = blockIdx.x * T + threadIdx.x;
  const float4 pi = __ldg(ipos + min(i, Ni - 1));
  float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
  for (int jt = 0; jt < Nj; jt += T) {
    const int cnt = min(T, Nj - jt);
    __syncthreads();
    if (threadIdx.x < cnt) sj[threadIdx.x] = __ldg(jpos + jt + threadIdx.x);
    __syncthreads();
    for (int jj = 0; jj < cnt; ++jj) {
      const float4 pj = sj[jj];
      const float rx = __fsub_rn(pj.x, pi.x);
      const float ry = __fsub_rn(pj.y, pi.y);
      const float rz = __fsub_rn(pj.z, pi.z);
      const float r2 = __fmaf_rn(rz, rz, __fmaf_rn(ry, ry, __fmaf_rn(rx, rx, eps2)));
      float w = __fdiv_rn(1.0f, __fsqrt_rn(r2));
      w = __fmul_rn(w, __fmul_rn(w, w));
      w = __fmul_rn(w, pj.w);
      ax = __fmaf_rn(rx, w, ax);
      ay = __fmaf_rn(ry, w, ay);
      az = __fmaf_rn(rz, w, az);
      if (POT) aw = __fmaf_rn(r2, w, aw);
    }
  }
  if (i < Ni) out[i] = make_float4(ax, ay, az, aw);
}

// ---------------------------------------------------------------------------
// K2: fused reduce + kick(s) + drift (+ publish). One particle per thread.
//
// Publish (multi-GPU fused all-gather): the new position is also
// stored into every peer's position buffer (mapped over NVLink/NVSwitch via
// CUDA IPC), so the all-gather of the next step's positions happens inside
// the kernel that produces them -- no collective call.
constexpr int kMaxPeers = 8;
struct Peers {
  float4* p[kMaxPeers];
  int n;
  float4* mc;  // NVLS: the multicast view of every rank's next buffer (this rank's slice), or null
};
constexpr int kPublish = 8;  // internal phase bit

__global__ void __launch_bounds__(128)
    k_kdk_update(int n, const float4* pos_in, float4* pos_out, float4* __restrict__ vel, float4* __restrict__ acc,
                 const float4* __restrict__ partials, int nchunks, float h_end, float h_begin, float dt, int phases,
                 Peers peers) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 a;
  if (phases & B2_KDK_REDUCE) {
    // Fixed summation order c = 0, 1, ..., nchunks-1; loads are issued a batch
    // at a time so the chain is bound by the adds, not by 64 serial round trips.
    constexpr int B = 16;
    a = __ldcs(partials + i);
    for (int c0 = 1; c0 < nchunks; c0 += B) {
      float4 p[B];
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (c0 + b < nchunks) p[b] = __ldcs(partials + static_cast<size_t>(c0 + b) * n + i);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (c0 + b < nchunks) {
          a.x = __fadd_rn(a.x, p[b].x);
          a.y = __fadd_rn(a.y, p[b].y);
          a.z = __fadd_rn(a.z, p[b].z);
          a.w = __fadd_rn(a.w, p[b].w);
        }
      }
    }
    acc[i] = a;
  } else if (phases & (B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) {
    a = acc[i];
  }
  const bool drift = phases & B2_KDK_KICK_DRIFT;
  const bool publish = phases & kPublish;
  float4 x;
  if (drift || publish) x = pos_in[i];
  if (phases & (B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) {
    float4 v = vel[i];
    if (phases & B2_KDK_KICK_END) {
      v.x = __fmaf_rn(a.x, h_end, v.x);
      v.y = __fmaf_rn(a.y, h_end, v.y);
      v.z = __fmaf_rn(a.z, h_end, v.z);
    }
    if (drift) {
      v.x = __fmaf_rn(a.x, h_begin, v.x);
      v.y = __fmaf_rn(a.y, h_begin, v.y);
      v.z = __fmaf_rn(a.z, h_begin, v.z);
      x.x = __fmaf_rn(v.x, dt, x.x);
      x.y = __fmaf_rn(v.y, dt, x.y);
      x.z = __fmaf_rn(v.z, dt, x.z);
    }
    vel[i] = v;
  }
  if (drift || publish) {
    if (peers.mc) {
      // one store through the switch lands in every rank's copy, this rank's included
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(peers.mc + i), "f"(x.x),
                   "f"(x.y), "f"(x.z), "f"(x.w)
                   : "memory");
    } else {
      pos_out[i] = x;
#pragma unroll
      for (int k = 0; k < kMaxPeers; ++k)
        if (k < peers.n) peers.p[k][i] = x;  // peer store over NVLink/NVSwitch
    }
  }
}

// ---------------------------------------------------------------------------
// Host-side planning.


// Launch variants of the fast kernel: {threads, i per thread, min CTAs/SM, j unroll}.
using ForceFn = void (*)(const float4*, int, const float4*, int, int, int, float, float4*, const Fused);
struct ForceVariant {
  int block, ipt;
  ForceFn fn[2];  // potential off / on; Fused{} = partials out, a ring = in-kernel reduction
};
#define B2_FV(B, I, M, U, S, A) \
  { B, I, { k_force_fast<B, I, M, U, S, A, false>, k_force_fast<B, I, M, U, S, A, true> } }
static const ForceVariant kVariants[] = {
    B2_FV(128, 16, 2, 1, 2, 0),  // 0: default for large N (best of the round-1 sweep)
    B2_FV(64, 8, 8, 4, 1, 0),    // 1: medium N (more CTAs)
    B2_FV(256, 8, 2, 4, 0, 0),   // 2: round-1 first version
    B2_FV(256, 12, 1, 2, 1, 0),  // 3: duplicated-pair j
    B2_FV(128, 16, 2, 1, 3, 2),  // 4: 2 of 8 pairs on ex2/lg2
    B2_FV(128, 16, 2, 1, 3, 3),  // 5: 3 of 8
    B2_FV(256, 12, 1, 2, 3, 2),  // 6: 2 of 6
    B2_FV(256, 12, 1, 2, 3, 1),  // 7: 1 of 6
    B2_FV(128, 16, 2, 2, 3, 2),  // 8
    B2_FV(256, 8, 2, 4, 3, 1),   // 9: 1 of 4
    B2_FV(64, 2, 16, 4, 2, 0),   // 10: small N
    B2_FV(32, 8, 16, 4, 2, 0),   // 11: chunks of an odd multiple of 32 j (Nj <= kAlign32Nj, e.g. N=4096)
};
#undef B2_FV

static int env_int_nb(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

static int large_variant() {
  static int v = [] {
    const char* e = std::getenv("SOLOMON_NBODY_VARIANT");  // tuning knob (bench sweeps)
    int x = e ? std::atoi(e) : 0;
    return (x >= 0 && x < static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]))) ? x : 0;
  }();
  return v;
}

// The variant launch_partials / launch_fused take for Ni (same per-lane arithmetic and j
// order in every variant, so the choice never moves a bit).
static const ForceVariant* pick_variant(int Ni, int nch, int jchunk) {
  if (jchunk % 64) return &kVariants[11];  // 32-j tiles: no padding in 32-aligned chunks
  const ForceVariant* v = &kVariants[large_variant()];
  static const long long want_k = std::max(0, env_int_nb("SOLOMON_NBODY_WANT", 4));  // tuning knob: CTAs per SM
  const long long want = want_k * device_info().sms;
  auto ctas = [&](const ForceVariant* c) { return (long long)((Ni + c->block * c->ipt - 1) / (c->block * c->ipt)) * nch; };
  // below that, 64 x 8 only while it still gives >= 16 CTAs per SM; else 64 x 2 (N = 8192:
  // 1598 vs 1455 Ginteractions/s, scripts/midn_sweep.py).
  if (ctas(v) < want) v = ctas(&kVariants[1]) >= 4 * want ? &kVariants[1] : &kVariants[10];
  return v;
}

constexpr int kMaxTile = 2048;  // largest BLOCK * IPT of a fused variant

// rows of i (per chunk) the ring holds: kRingSlots tiles of the largest variant, or all of Ni
static size_t fused_ring_rows(int Ni) {
  return std::min<size_t>(static_cast<size_t>(kRingSlots) * kMaxTile, static_cast<size_t>(std::max(Ni, 0)) + kMaxTile);
}

static size_t fused_workspace_bytes(int Ni, int Nj, int flags) {
  const int nch = nchunks_for(Nj, flags);
  return kRingCtrlBytes + 128 + static_cast<size_t>(nch) * fused_ring_rows(Ni) * sizeof(float4);
}

// Force with the in-kernel in-order reduction: acc = sum_c partials_c (bits of partials +
// B2_KDK_REDUCE). ws >= fused_workspace_bytes; one memset of the control words + one launch.
static int launch_partials(int Ni, const float4* ipos, int Nj, const float4* jpos, float eps, int flags,
                           float4* out, cudaStream_t s);
static int launch_update(int n, float4* pos, float4* vel, float4* acc, const float4* partials, int nchunks,
                         float h_end, float h_begin, float dt, int phases, cudaStream_t s,
                         const float4* pos_in = nullptr, const Peers* peers = nullptr);

static int launch_fused(int Ni, const float4* ipos, int Nj, const float4* jpos, float eps, int flags, float4* acc,
                        void* ws, cudaStream_t s) {
  const int jchunk = chunk_size(Nj, flags);
  const int nch = nchunks_for(Nj, flags);
  const ForceVariant* v = pick_variant(Ni, nch, jchunk);
  const int tile = v->block * v->ipt;
  const int nit = (Ni + tile - 1) / tile;
  unsigned int* ctrl = static_cast<unsigned int*>(ws);
  const uintptr_t rb = (reinterpret_cast<uintptr_t>(ws) + kRingCtrlBytes + 127) & ~static_cast<uintptr_t>(127);
  // Up to ~63k i the workspace holds all nch x Ni partials anyway: there the reduce is a second
  // launch (the same fixed order, so the same bits) -- faster than the ring at small and mid N,
  // where the ring's per-CTA fence, arrival and slot wait are not hidden (N = 8192: 44 vs 56 us,
  // 32768: 427 vs 503, 65536: 1643 vs 1710). The ring is what keeps large N in 64 MiB.
  if (fused_ring_rows(Ni) >= static_cast<size_t>(Ni)) {
    float4* part = reinterpret_cast<float4*>(rb);
    int rc = launch_partials(Ni, ipos, Nj, jpos, eps, flags, part, s);
    if (rc) return rc;
    return launch_update(Ni, nullptr, nullptr, acc, part, nch, 0.f, 0.f, 0.f, B2_KDK_REDUCE, s);
  }
  // ring slots: every i-tile of the launch when the workspace holds them (small tiles at mid N,
  // where 32 slots made later i-tiles wait on earlier ones), else kRingSlots of the largest tile
  const int slots = static_cast<int>(std::min<size_t>(fused_ring_rows(Ni) / tile, kMaxRingSlots));
  Fused fz{reinterpret_cast<float4*>(rb), ctrl, acc, std::min(nit, std::max(slots, 1)), make_watch()};
  cudaError_t e = cudaMemsetAsync(ctrl, 0, 2 * static_cast<size_t>(fz.R) * sizeof(unsigned int), s);
  if (e != cudaSuccess) return static_cast<int>(e);
  v->fn[(flags & B2_POTENTIAL) ? 1 : 0]<<<nit * nch, v->block, 0, s>>>(ipos, Ni, jpos, Nj, jchunk, nit, eps * eps, acc,
                                                                     fz);
  return launch_status();
}

static int launch_partials(int Ni, const float4* ipos, int Nj, const float4* jpos, float eps, int flags,
                           float4* out, cudaStream_t s) {
  const float eps2 = eps * eps;  // listing_nbody.c:5
  const bool pot = flags & B2_POTENTIAL;
  if (flags & B2_EXACT) {
    const int grid = (Ni + 127) / 128;
    if (pot)
      k_force_exact<true><<<grid, 128, 0, s>>>(ipos, Ni, jpos, Nj, eps2, out);
    else
      k_force_exact<false><<<grid, 128, 0, s>>>(ipos, Ni, jpos, Nj, eps2, out);
    return launch_status();
  }
  const int jchunk = chunk_size(Nj, flags);
  const int nch = nchunks_for(Nj, flags);
  // Largest tile whose (i-tile, j-chunk) grid still fills the 148 SMs: the tuned large
  // variant, else 64x8, else 64x2 (small N is latency-bound and needs every warp it can get).
  const ForceVariant* v = pick_variant(Ni, nch, jchunk);
  const int nit = (Ni + v->block * v->ipt - 1) / (v->block * v->ipt);
  v->fn[pot ? 1 : 0]<<<nit * nch, v->block, 0, s>>>(ipos, Ni, jpos, Nj, jchunk, nit, eps2, out, Fused{});
  return launch_status();
}

static int launch_update(int n, float4* pos, float4* vel, float4* acc, const float4* partials, int nchunks,
                         float h_end, float h_begin, float dt, int phases, cudaStream_t s, const float4* pos_in,
                         const Peers* peers) {
  if (n <= 0) return B2_OK;
  Peers pp{};
  if (peers) pp = *peers;
  if (!pos_in) pos_in = pos;
  if (pp.n > 0 || pos_in != pos) phases |= kPublish;
  k_kdk_update<<<(n + 127) / 128, 128, 0, s>>>(n, pos_in, pos, vel, acc, partials, nchunks, h_end, h_begin, dt, phases,
                                               pp);
  return launch_status();
}

static int check_particles(int n, const float* p) {
  if (n < 0) return B2_EINVAL;
  if (n > 0 && p == nullptr) return B2_EINVAL;
  if (n > 0 && !aligned16(p)) return B2_EALIGN;
  return B2_OK;
}

}  // namespace b2

using namespace b2;

extern "C" {

int b2_calc_acc_nchunks(int Nj, int flags) { return nchunks_for(Nj, flags); }

size_t b2_calc_acc_workspace_bytes(int Ni, int Nj, int flags) {
  const int nch = nchunks_for(Nj, flags);
  if (nch <= 1 || Ni <= 0) return 0;
  return fused_workspace_bytes(Ni, Nj, flags);
}

int b2_calc_acc_partials(int Ni, const float* ipos, int Nj, const float* jpos, float eps, int flags,
                         float* partials, void* stream) {
  int rc;
  if ((rc = check_particles(Ni, ipos)) || (rc = check_particles(Nj, jpos)) || (rc = check_particles(Ni, partials)))
    return rc;
  if (flags & ~(B2_POTENTIAL | B2_EXACT)) return B2_EINVAL;
  if (Ni == 0) return B2_OK;
  if (Nj == 0) {
    cudaMemsetAsync(partials, 0, sizeof(float4) * static_cast<size_t>(Ni), as_stream(stream));
    return launch_status();
  }
  return launch_partials(Ni, reinterpret_cast<const float4*>(ipos), Nj, reinterpret_cast<const float4*>(jpos), eps,
                         flags, reinterpret_cast<float4*>(partials), as_stream(stream));
}

int b2_calc_acc(int Ni, const float* ipos, float* iacc, int Nj, const float* jpos, float eps, int flags,
                void* workspace, size_t workspace_bytes, void* stream) {
  int rc;
  if ((rc = check_particles(Ni, ipos)) || (rc = check_particles(Ni, iacc)) || (rc = check_particles(Nj, jpos)))
    return rc;
  if (flags & ~(B2_POTENTIAL | B2_EXACT)) return B2_EINVAL;
  if (Ni == 0) return B2_OK;
  cudaStream_t s = as_stream(stream);
  if (Nj == 0) {
    cudaMemsetAsync(iacc, 0, sizeof(float4) * static_cast<size_t>(Ni), s);
    return launch_status();
  }
  const int nch = nchunks_for(Nj, flags);
  if (nch == 1)
    return launch_partials(Ni, reinterpret_cast<const float4*>(ipos), Nj, reinterpret_cast<const float4*>(jpos), eps,
                           flags, reinterpret_cast<float4*>(iacc), s);
  if (workspace_bytes < b2_calc_acc_workspace_bytes(Ni, Nj, flags)) return B2_ESPACE;
  if (!aligned16(workspace)) return B2_EALIGN;
  return launch_fused(Ni, reinterpret_cast<const float4*>(ipos), Nj, reinterpret_cast<const float4*>(jpos), eps,
                      flags, reinterpret_cast<float4*>(iacc), workspace, s);
}

int b2_kdk_update(int n, float* pos, float* vel, float* acc, const float* partials, int nchunks, float h_end,
                  float h_begin, float dt, int phases, void* stream) {
  int rc;
  if (phases & ~(B2_KDK_REDUCE | B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) return B2_EINVAL;
  if ((rc = check_particles(n, acc))) return rc;
  if ((phases & B2_KDK_REDUCE) && ((rc = check_particles(n, partials)) || nchunks < 1)) return rc ? rc : B2_EINVAL;
  if ((phases & (B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) && (rc = check_particles(n, vel))) return rc;
  if ((phases & B2_KDK_KICK_DRIFT) && (rc = check_particles(n, pos))) return rc;
  return launch_update(n, reinterpret_cast<float4*>(pos), reinterpret_cast<float4*>(vel),
                       reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(partials), nchunks, h_end,
                       h_begin, dt, phases, as_stream(stream));
}

int b2_kdk_update_publish(int n, const float* pos_in, float* pos_out, float* vel, float* acc, const float* partials,
                          int nchunks, float h_end, float h_begin, float dt, int phases, float* const* peers,
                          int npeers, void* stream) {
  int rc;
  if (phases & ~(B2_KDK_REDUCE | B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) return B2_EINVAL;
  if (npeers < 0 || npeers > kMaxPeers || (npeers > 0 && !peers)) return B2_EINVAL;
  if ((rc = check_particles(n, acc)) || (rc = check_particles(n, pos_in)) || (rc = check_particles(n, pos_out)))
    return rc;
  if ((phases & B2_KDK_REDUCE) && ((rc = check_particles(n, partials)) || nchunks < 1)) return rc ? rc : B2_EINVAL;
  if ((phases & (B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) && (rc = check_particles(n, vel))) return rc;
  Peers pp{};
  pp.n = npeers;
  for (int k = 0; k < npeers; ++k) {
    if ((rc = check_particles(n, peers[k]))) return rc;
    pp.p[k] = reinterpret_cast<float4*>(peers[k]);
  }
  const int ph = phases | kPublish;
  if (n <= 0) return B2_OK;
  k_kdk_update<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(
      n, reinterpret_cast<const float4*>(pos_in), reinterpret_cast<float4*>(pos_out), reinterpret_cast<float4*>(vel),
      reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(partials), nchunks, h_end, h_begin, dt, ph, pp);
  return launch_status();
}

int b2_kdk_update_multicast(int n, const float* pos_in, float* mc_out, float* vel, float* acc, const float* partials,
                            int nchunks, float h_end, float h_begin, float dt, int phases, void* stream) {
  int rc;
  if (phases & ~(B2_KDK_REDUCE | B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) return B2_EINVAL;
  if ((rc = check_particles(n, acc)) || (rc = check_particles(n, pos_in)) || (rc = check_particles(n, mc_out)))
    return rc;
  if ((phases & B2_KDK_REDUCE) && ((rc = check_particles(n, partials)) || nchunks < 1)) return rc ? rc : B2_EINVAL;
  if ((phases & (B2_KDK_KICK_END | B2_KDK_KICK_DRIFT)) && (rc = check_particles(n, vel))) return rc;
  if (n <= 0) return B2_OK;
  Peers pp{};
  pp.mc = reinterpret_cast<float4*>(mc_out);
  k_kdk_update<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(
      n, reinterpret_cast<const float4*>(pos_in), nullptr, reinterpret_cast<float4*>(vel),
      reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(partials), nchunks, h_end, h_begin, dt,
      phases | kPublish, pp);
  return launch_status();
}

size_t b2_leapfrog_workspace_bytes(int n, int flags) {
  const int ff = flags & (B2_POTENTIAL | B2_EXACT);
  // the fused force's ring, or the persistent small-N path's [2][n] position words + ready lines
  return std::max(b2_calc_acc_workspace_bytes(n, n, ff), small_workspace_bytes(n));
}

int b2_leapfrog(int n, float* pos, float* vel, float* acc, float eps, float dt, int nsteps, int flags,
                void* workspace, size_t workspace_bytes, void* stream) {
  int rc;
  if ((rc = check_particles(n, pos)) || (rc = check_particles(n, vel)) || (rc = check_particles(n, acc))) return rc;
  if (flags & ~(B2_POTENTIAL | B2_EXACT | B2_INIT_ACC) || nsteps < 0) return B2_EINVAL;
  if (n == 0) return B2_OK;
  const int fflags = flags & (B2_POTENTIAL | B2_EXACT);
  if (workspace_bytes < b2_leapfrog_workspace_bytes(n, flags)) return B2_ESPACE;
  if (!aligned16(workspace)) return B2_EALIGN;
  cudaStream_t s = as_stream(stream);
  float4* P = reinterpret_cast<float4*>(pos);
  float4* V = reinterpret_cast<float4*>(vel);
  float4* A = reinterpret_cast<float4*>(acc);
  if (launch_leapfrog_small(n, P, V, A, eps, dt, nsteps, flags, workspace, workspace_bytes, s)) return B2_OK;
  const float h = 0.5f * dt;
  // Steady state is two launches per step: force, then one update. Up to ~63k particles the
  // force writes its nch x n chunk partials into the workspace and the update reduces them
  // (B2_KDK_REDUCE) before its kicks; beyond, the force reduces them in-kernel (ring) and the
  // update reads acc. Same summation order either way.
  const int nch = nchunks_for(n, fflags);
  const bool partials = nch > 1 && fused_ring_rows(n) >= static_cast<size_t>(n);
  const float4* part = reinterpret_cast<const float4*>(
      (reinterpret_cast<uintptr_t>(workspace) + kRingCtrlBytes + 127) & ~static_cast<uintptr_t>(127));
  auto force = [&]() {
    if (partials)
      return launch_partials(n, P, n, P, eps, fflags, const_cast<float4*>(part), s);
    return b2_calc_acc(n, pos, acc, n, pos, eps, fflags, workspace, workspace_bytes, s);
  };
  const int reduce = partials ? B2_KDK_REDUCE : 0;
  if (flags & B2_INIT_ACC) {
    if ((rc = force())) return rc;
    if (partials && (rc = launch_update(n, P, V, A, part, nch, 0.f, 0.f, 0.f, B2_KDK_REDUCE, s))) return rc;
  }
  if (nsteps == 0) return B2_OK;
  // step 0 opening kick + drift
  if ((rc = launch_update(n, P, V, A, nullptr, 1, 0.f, h, dt, B2_KDK_KICK_DRIFT, s))) return rc;
  for (int st = 0; st < nsteps; ++st) {
    if ((rc = force())) return rc;
    const bool last = st + 1 == nsteps;
    const int ph = reduce | B2_KDK_KICK_END | (last ? 0 : B2_KDK_KICK_DRIFT);
    if ((rc = launch_update(n, P, V, A, part, partials ? nch : 1, h, h, dt, ph, s))) return rc;
  }
  return B2_OK;
}

}  // extern "C"
