// K2' -- the whole small-N leapfrog run in one persistent launch (b2_leapfrog for
// n <= 64 x SMs). Reference force law: pkg/tests/fixtures/listing_nbody.c:1-27 via
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
// under-filled force tiles and a latency-bound reduce for ~5.5 us of arithmetic).
//
// One CTA per I = 2H <= 64 own particles (I sized so the grid spans every SM: 28 at
// N=4096 -> 147 CTAs, 56 at N=8192), all CTAs co-resident (cooperative launch). Own particle pairs
// are (i0 + p, i0 + H + p), p < H -- the packed FFMA2 lanes. Force task = (group g of
// NP pairs, j-chunk c): thread tid -> g = tid % G, c = tid / G, so a CTA runs
// G x nch threads (N=4096: 2 groups of 7 pairs x 128 chunks of 32 j = 256 threads, 8
// warps, 7 independent pairs each -- the shape of the large tile kernel's 8 warps x 8
// pairs; N=8192: 4 groups of 7 pairs x 64 chunks of 128 j).
//
// Exchange (scripts/trace_small.cu, scripts/l2_gather_probe.cu): positions {x, y, z, m}
// go to a [2][n] global buffer (state parity); after its particles' stores, warp 0 of each
// CTA does one release-add on one of 8 arrival counters (CTA b -> counter b % 8). A step
// starts when warp 0 has acquired every counter's full count (lanes 0-7, one counter each)
// -- every CTA published the state -- and each WARP then pulls only the chunks its lanes
// compute with bulk copies (cp.async.bulk, one per chunk into its padded slot) completed on
// the warp's own mbarrier. A count that never completes ends the run through the watchdog
// (poll_expired, runtime.cu) instead of hanging. Measured against the alternatives: polling
// self-validating tagged words per warp (no fence, no counter) let the CTAs drift up to
// 3-4 us apart and each warp waited for the latest of its ~19 producers (13.5 us/step);
// step-wide counters keep the CTAs within ~0.3 us (11.3 us/step with LDG slices; the bulk
// copies take the slice read from 1.9 to ~0.8 us). Two parities suffice: a CTA writes state
// s+2 only after every CTA announced s+1, which each does only after its force of step s --
// after its bulk copies of state s completed.
//
// Bit-identical to the two-kernel path (b2_calc_acc_partials + b2_kdk_update):
// same j-chunks (chunk_size depends on N only), each chunk summed in j order
// with the same packed-FP32 interaction, partials summed c = 0, 1, ... and the
// same FMA kick/drift sequence.
constexpr int kSmallMaxThreads = 256;
#ifndef B2_SMALL_UNROLL
#define B2_SMALL_UNROLL 2
#endif
constexpr int kSmallUnroll = B2_SMALL_UNROLL;  // j-loop unroll of the force task
#ifndef B2_SMALL_IMAX
#define B2_SMALL_IMAX 64
#endif
constexpr int kSmallImax = B2_SMALL_IMAX;  // own particles per CTA (at most; even)
constexpr int kSmallMaxNP = 8;   // packed pairs per thread

struct SmallArgs {
  int n;
  float4* pos;
  float4* vel;
  float4* acc;
  float4* pub;  // [2][n] published positions {x, y, z, m} by state parity
  unsigned int* arrive;  // [8][32]: publishes of CTAs b with b % 8 == k in word 32 k, zeroed
  float eps2, dt, h;
  int nsteps, flags;  // B2_POTENTIAL | B2_INIT_ACC
  int chunk, nch;
  int I;  // own particles per CTA: 2 * ceil(n / (2 * SMs)) <= 32, so the grid spans every SM
  int G;  // pair groups per CTA (threads = G * nch, rounded up to a warp)
  Watch watch;  // a position word that never arrives ends the run (runtime.cu), no trap
  int withhold;  // test hook: this CTA never announces (b2_debug_withhold_publish), -1 = none
#ifdef B2_SMALL_TRACE
  unsigned long long* trace;  // [cta][step][32] globaltimer stamps (scripts/trace_small.cu)
#endif
};
#ifdef B2_SMALL_TRACE
// slots: 0 before / 1 after the step's first barrier, 2 after the force barrier, 3 after the
// reduce, 4 after the kick/drift/publish; 8 + w / 16 + w / 24 + w: warp w after the counters'
// barrier / slice copied / force task done
#define B2_STRACE_IF(cond, k) \
  if (cond) a.trace[(static_cast<size_t>(blockIdx.x) * a.nsteps + st) * 32 + (k)] = globaltimer_ns()
#else
#define B2_STRACE_IF(cond, k)
#endif
#define B2_STRACE(k) B2_STRACE_IF(tid == 0, k)
#define B2_WTRACE(k) B2_STRACE_IF(lane == 0 && w < 8, (k) + w)

// shared memory (float4 units unless noted): P [n + nch + 1] positions {x, y, z, m}, j at
// j + j / chunk (one pad slot per chunk: the 8 lanes of an LDS.128 phase read 4-8 chunks at
// distinct bank groups); own, ownv, owna [I] own positions, velocities, accelerations; part
// [4 I][S] floats: the chunk partials transposed -- row 4 t + k holds component k of own
// particle t for every chunk, so the in-order reduce of a row reads consecutive words four
// chunks per LDS.128 (S = roundup(nch, 32) + 4 words: 32-chunk blocks never leave the row,
// and S % 32 == 4 puts the 8 rows of an LDS.128 phase on distinct banks); wbar [8] the
// warps' bulk-copy mbarriers.
__host__ __device__ inline int small_part_stride(int nch) { return (nch + 31) / 32 * 32 + 4; }
inline size_t small_smem_bytes(int n, int nch, int I) {
  return (static_cast<size_t>(n) + nch + 1 + 3 * static_cast<size_t>(I)) * sizeof(float4) +
         3 * static_cast<size_t>((I / 2 + 1) & ~1) * sizeof(float2) +
         4 * static_cast<size_t>(I) * small_part_stride(nch) * sizeof(float) + 8 * sizeof(uint64_t);
}

template <int NP, bool POT>
__global__ void __launch_bounds__(kSmallMaxThreads, 1) k_leapfrog_small(const SmallArgs a) {
  extern __shared__ float4 sm4[];
  const int n = a.n, tid = threadIdx.x, lane = tid & 31;
  const int chunk = a.chunk, nch = a.nch, IB = a.I, H = IB / 2, G = a.G;
  float4* P = sm4;
  float4* own = P + n + nch + 1;
  float4* ownv = own + IB;
  float4* owna = ownv + IB;
  float2* negp = reinterpret_cast<float2*>(owna + IB);  // [3][H] (-x, -y, -z of pair p's two lanes)
  const int S = small_part_stride(nch);
  float* part = reinterpret_cast<float*>(negp + 3 * ((H + 1) & ~1));  // [4 IB][S]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(part + 4 * IB * S);  // [8]
  const int i0 = blockIdx.x * IB;
  const int I = min(IB, n - i0);

  // this thread's force task and this warp's j-range (the chunks its lanes own)
  const int g = tid % G, c = tid / G;
  const int w = tid >> 5;
  const int wc0 = min(nch, (32 * w) / G), wc1 = min(nch, (32 * w + 32) / G);
  const int wj0 = wc0 * chunk, wj1 = min(n, wc1 * chunk);

  // state 0: every position straight from pos (nobody writes pos before the end)
  for (int j = tid; j < n; j += blockDim.x) P[j + j / chunk] = a.pos[j];
  if (lane == 0 && w < 8) mbar_init(&wbar[w], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // own particles i = i0 + t, t < I: x in own[], v in ownv[], acc in owna[] -- shared memory,
  // not registers, so the force phase has the whole register file for its pairs
  for (int t = tid; t < I; t += blockDim.x) {
    own[t] = a.pos[i0 + t];
    ownv[t] = a.vel[i0 + t];
    if (!(a.flags & B2_INIT_ACC)) owna[t] = a.acc[i0 + t];  // else computed below (acc may be uninitialised)
  }
  // negated pair coordinates of own particle t (lane t / H of pair t % H)
  auto set_neg = [&](int t, const float4 x) {
    float* nf = reinterpret_cast<float*>(negp) + 2 * (t % H) + t / H;
    nf[0] = -x.x;
    nf[2 * H] = -x.y;
    nf[4 * H] = -x.z;
  };
  // (pairs past the last CTA's particles take its last particle: computed, never stored)
  for (int t = tid; t < 2 * H; t += blockDim.x) set_neg(t, a.pos[i0 + min(t, I - 1)]);
  const float2 e2 = make_float2(a.eps2, a.eps2);
  __syncthreads();

  // chunk partials of this thread's task (g, c) from P and own -> part
  auto force_task = [&]() {
    if (c >= nch) return;
    float2 nx[NP], ny[NP], nz[NP], ax[NP], ay[NP], az[NP], ap[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int pa = min(g * NP + p, H - 1);
      nx[p] = negp[pa];
      ny[p] = negp[H + pa];
      nz[p] = negp[2 * H + pa];
      ax[p] = ay[p] = az[p] = ap[p] = make_float2(0.f, 0.f);
    }
    const float4* q = P + c * (chunk + 1);
    const int len = min(chunk, n - c * chunk);
#ifndef B2_SMALL_PREFETCH
#define B2_SMALL_PREFETCH 0  // 1: next j loaded one iteration ahead (measured slower: 7.15 vs 6.95 us)
#endif
#if B2_SMALL_PREFETCH
    float4 pj = *q++;
    const float4* const qend = q + len;
#pragma unroll 1
    for (; q != qend; ++q) {
      const float4 pn = *q;  // next j one iteration ahead (the pad slot makes q[len] readable)
      interact_bf<NP, POT>(make_float2(pj.x, pj.x), make_float2(pj.y, pj.y), make_float2(pj.z, pj.z),
                           make_float2(pj.w, pj.w), nx, ny, nz, e2, ax, ay, az, ap);
      pj = pn;
    }
#else
    const float4* const qend = q + len;
#pragma unroll kSmallUnroll
    for (; q != qend; ++q) {
      const float4 pj = *q;
      interact_bf<NP, POT>(make_float2(pj.x, pj.x), make_float2(pj.y, pj.y), make_float2(pj.z, pj.z),
                           make_float2(pj.w, pj.w), nx, ny, nz, e2, ax, ay, az, ap);
    }
#endif
    float* o = part + c;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int pa = g * NP + p;
      if (pa < H) {
        float* ra = o + 4 * pa * S;
        float* rb = o + 4 * (H + pa) * S;
        ra[0] = ax[p].x, ra[S] = ay[p].x, ra[2 * S] = az[p].x, ra[3 * S] = POT ? ap[p].x : 0.f;
        rb[0] = ax[p].y, rb[S] = ay[p].y, rb[2 * S] = az[p].y, rb[3 * S] = POT ? ap[p].y : 0.f;
      }
    }
  };
  // one COMPONENT of own particle t's acc: the chunk partials summed in the fixed order c = 0,
  // 1, ... (as k_kdk_update). Thread r < 4 I sums row r of part (component r % 4 of particle
  // r / 4): 32 chunks per block as 8 LDS.128 at immediate offsets, the next block's loads in
  // flight while this block's adds run -- the 127 dependent adds are the chain.
  auto reduce_component = [&](int r) {
    const float4* row = reinterpret_cast<const float4*>(part + r * S);
    float4 cur[8], nxt[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) cur[u] = row[u];
    float s = cur[0].x;
    int c0 = 0;
#pragma unroll 1
    for (; c0 + 32 < nch; c0 += 32) {  // full blocks (the row holds roundup(nch, 32) words)
#pragma unroll
      for (int u = 0; u < 8; ++u) nxt[u] = row[(c0 + 32) / 4 + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + 4 * u > 0) s = __fadd_rn(s, cur[u].x);
        s = __fadd_rn(s, cur[u].y);
        s = __fadd_rn(s, cur[u].z);
        s = __fadd_rn(s, cur[u].w);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // the last block: chunks c0 .. nch-1
      const int c = c0 + 4 * u;
      if (c > 0 && c < nch) s = __fadd_rn(s, cur[u].x);
      if (c + 1 < nch) s = __fadd_rn(s, cur[u].y);
      if (c + 2 < nch) s = __fadd_rn(s, cur[u].z);
      if (c + 3 < nch) s = __fadd_rn(s, cur[u].w);
    }
    reinterpret_cast<float*>(owna)[r] = s;
  };
  // the first 4 I threads reduce (acc -> owna), then threads t < I kick / drift / publish
  auto reduce_all = [&]() {
    const int nr = 4 * I, nb = (nr + 31) & ~31;
    if (tid < nb) {
      if (tid < nr) reduce_component(tid);
      asm volatile("bar.sync 1, %0;" ::"r"(nb) : "memory");  // named barrier: the reducing warps only
    }
  };
  // own particle t: closing kick (B2_KDK_KICK_END) [-> kick + drift (B2_KDK_KICK_DRIFT) ->
  // publish state `pub_state`]
  auto update = [&](int t, bool kick_end, int pub_state) {
    const float4 acc = owna[t];
    float4 v = ownv[t], x = own[t];
    const float h = a.h;
    if (kick_end) {
      v.x = __fmaf_rn(acc.x, h, v.x);
      v.y = __fmaf_rn(acc.y, h, v.y);
      v.z = __fmaf_rn(acc.z, h, v.z);
    }
    if (pub_state > 0) {
      v.x = __fmaf_rn(acc.x, h, v.x);
      v.y = __fmaf_rn(acc.y, h, v.y);
      v.z = __fmaf_rn(acc.z, h, v.z);
      x.x = __fmaf_rn(v.x, a.dt, x.x);
      x.y = __fmaf_rn(v.y, a.dt, x.y);
      x.z = __fmaf_rn(v.z, a.dt, x.z);
      own[t] = x;
      set_neg(t, x);
      a.pub[static_cast<size_t>(pub_state & 1) * n + i0 + t] = x;  // ordered by announce()'s release
    }
    ownv[t] = v;
  };
  // after the CTA's particles t < I were published: one arrival on the CTA's counter (release:
  // the words are visible to whoever acquires the count)
#ifndef B2_SMALL_WARPSYNC
#define B2_SMALL_WARPSYNC 1
#endif
  // counter of CTA b: b % 8 (step-wide wait), or the contiguous group b * 8 / ctas (per-warp wait)
  auto counter_of = [&](int b) { return B2_SMALL_WARPSYNC ? b * 8 / static_cast<int>(gridDim.x) : b & 7; };
  auto counter_size = [&](int k) {  // CTAs on counter k
    const int C = gridDim.x;
    return B2_SMALL_WARPSYNC ? ((k + 1) * C + 7) / 8 - (k * C + 7) / 8 : (C - k + 7) / 8;
  };
  // (after threads t < I stored their positions; called by the warps holding them: I <= 64)
  const int pubw = (I + 31) >> 5;  // warps that publish
  auto announce = [&]() {
    if (pubw > 1)
      asm volatile("bar.sync 2, %0;" ::"r"(32 * pubw) : "memory");
    else
      __syncwarp();
    if (tid == 0 && static_cast<int>(blockIdx.x) != a.withhold) {
#ifdef B2_PROBE_NOFENCE  // timing probe only: the arrival WITHOUT release -- incorrect
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(a.arrive + 32 * counter_of(blockIdx.x)), "r"(1u)
                   : "memory");
#else
      red_release_add_u32(a.arrive + 32 * counter_of(blockIdx.x), 1u);
#endif
    }
  };
  // this warp: wait until the CTAs on the counters of its slice's producers published `state`
  auto slice_published = [&](int state) -> bool {
    bool ok = true;
    if (wc0 < wc1) {
      const int k0 = counter_of(wj0 / IB), k1 = counter_of((wj1 - 1) / IB);
      if (lane <= k1 - k0) {
        const int k = k0 + lane;
        const unsigned int want = static_cast<unsigned int>(counter_size(k)) * state;
        const unsigned long long t0 = globaltimer_ns();
        for (unsigned int it = 1; ld_acquire_u32_gpu(a.arrive + 32 * k) < want; ++it)
          if (!(it & 31) && poll_expired(a.watch, t0, kFaultLeapfrogSmall)) {
            ok = false;
            break;
          }
      }
    }
    return __all_sync(0xffffffffu, ok);
  };
  // warp 0: wait until every CTA published state `state` (lane k < 8 acquires counter k);
  // false = the watchdog gave up
  auto all_published = [&](int state) -> bool {
    bool ok = true;
    if (lane < 8) {
      const unsigned int want = static_cast<unsigned int>(counter_size(lane)) * state;
      const unsigned long long t0 = globaltimer_ns();
      // the watchdog every 32nd poll: its own load would double each poll's round trip
      for (unsigned int k = 1; ld_acquire_u32_gpu(a.arrive + 32 * lane) < want; ++k)
        if (!(k & 31) && poll_expired(a.watch, t0, kFaultLeapfrogSmall)) {
          ok = false;
          break;
        }
    }
    return __all_sync(0xffffffffu, ok);
  };
  // this warp's chunks of state `state` into their P slots: one bulk copy per chunk (lanes in
  // parallel), all on the warp's mbarrier (phase = step parity). After the CTA barrier that
  // followed warp 0's acquire of the counters.
  auto fetch_slice = [&](int state, int st) {
    if (wc0 >= wc1) return;
    if (lane == 0) mbar_expect_tx(&wbar[w], static_cast<uint32_t>(wj1 - wj0) * sizeof(float4));
    __syncwarp();
    fence_proxy_async_global();  // the acquired generic stores, now read by the async proxy
    fence_proxy_async();         // the slots' earlier generic reads, now overwritten by it
    const float4* src = a.pub + static_cast<size_t>(state & 1) * n;
    for (int cc = wc0 + lane; cc < wc1; cc += 32) {
      const int j0 = cc * chunk;
      bulk_g2s(P + cc * (chunk + 1), src + j0, static_cast<uint32_t>(min(chunk, n - j0)) * sizeof(float4), &wbar[w]);
    }
    mbar_wait(&wbar[w], static_cast<uint32_t>(st & 1));
  };

  if (a.flags & B2_INIT_ACC) {
    force_task();
    __syncthreads();
    reduce_all();
  }
  if (a.nsteps > 0) {
    // opening kick + drift of step 0, publish state 1 (owna: written above by the same warps,
    // ordered by the named barrier; or loaded before the first barrier)
    if (tid < I) update(tid, false, 1);
    if (tid < 32 * pubw) announce();
    for (int st = 0; st < a.nsteps; ++st) {
      B2_STRACE(0);
      __syncthreads();  // own[] holds this state; every read of part[] (reduce) is done
      // every CTA published state st+1 (barrier + CTA-wide vote: no static shared memory, the
      // dynamic allocation may use it all); a watchdog expiry leaves without writing pos / vel /
      // acc (b2_fault_status reports it)
#if B2_SMALL_WARPSYNC
      const bool ok = slice_published(st + 1);
      B2_STRACE(1);
      B2_WTRACE(8);
      if (ok) {
        fetch_slice(st + 1, st);
        B2_WTRACE(16);
        force_task();
      }
      B2_WTRACE(24);
      if (__syncthreads_or(!ok)) return;
#else
      if (__syncthreads_or(tid < 32 && !all_published(st + 1))) return;
      B2_STRACE(1);
      B2_WTRACE(8);
      fetch_slice(st + 1, st);
      B2_WTRACE(16);
      force_task();
      B2_WTRACE(24);
      __syncthreads();
#endif
      B2_STRACE(2);
      reduce_all();
      B2_STRACE(3);
      if (tid < I) update(tid, true, st + 1 < a.nsteps ? st + 2 : 0);
      if (tid < 32 * pubw && st + 1 < a.nsteps) announce();
      B2_STRACE(4);
    }
  }
  __syncthreads();
  for (int t = tid; t < I; t += blockDim.x) {
    a.pos[i0 + t] = own[t];
    a.vel[i0 + t] = ownv[t];
    a.acc[i0 + t] = owna[t];
  }
}

// the persistent path's workspace: [2][n] published positions + 8 arrival-counter lines
size_t small_workspace_bytes(int n) { return 2 * static_cast<size_t>(std::max(n, 0)) * sizeof(float4) + 1024; }

using SmallFn = void (*)(const SmallArgs);
template <bool POT>
static SmallFn small_kernel(int np) {
  switch (np) {
    case 1: return k_leapfrog_small<1, POT>;
    case 2: return k_leapfrog_small<2, POT>;
    case 3: return k_leapfrog_small<3, POT>;
    case 4: return k_leapfrog_small<4, POT>;
    case 5: return k_leapfrog_small<5, POT>;
    case 6: return k_leapfrog_small<6, POT>;
    case 7: return k_leapfrog_small<7, POT>;
    default: return k_leapfrog_small<8, POT>;
  }
}

// Launch shape of the persistent small-N path for n on this device: own particles per CTA,
// pair groups, pairs per thread, threads, CTAs. False when n is outside its range.
struct SmallShape {
  int I, G, NP, threads, ctas;
};
static bool small_shape(int n, int nch, int sms, SmallShape* s) {
  if (n <= 0 || nch < 2) return false;
  s->I = 2 * ((n + 2 * sms - 1) / (2 * sms));
  if (s->I > kSmallImax) return false;
  const int H = s->I / 2;
  // pair groups: 1, 2 or 4 (a warp's lanes must map to whole chunks: G divides 32)
  s->G = H <= kSmallMaxNP ? 1 : H <= 2 * kSmallMaxNP ? 2 : 4;
  s->NP = (H + s->G - 1) / s->G;
  s->threads = (std::max(s->G * nch, 4 * s->I) + 31) / 32 * 32;  // force tasks; the 4 I reduce rows
  s->ctas = (n + s->I - 1) / s->I;
  return s->threads <= kSmallMaxThreads && s->ctas <= sms && 32 % s->G == 0;
}

// The persistent small-N path of b2_leapfrog (k_leapfrog_small), when it applies:
// fast arithmetic, n <= 64 x SMs, >= 2 j-chunks, tasks within one CTA, shared memory
// fits, and the workspace holds small_workspace_bytes(n). Returns false
// (nothing launched) otherwise.
bool launch_leapfrog_small(int n, float4* pos, float4* vel, float4* acc, float eps, float dt, int nsteps,
                                  int flags, void* workspace, size_t workspace_bytes, cudaStream_t s) {
  static const int enabled = [] {
    const char* e = std::getenv("SOLOMON_NBODY_PERSISTENT");
    return e ? std::atoi(e) : 1;
  }();
  if (!enabled || (flags & B2_EXACT)) return false;
  const int nch = nchunks_for(n, flags & B2_POTENTIAL);
  const DeviceInfo& di = device_info();
  SmallShape sh;
  if (!small_shape(n, nch, di.sms, &sh)) return false;
  const size_t smem = small_smem_bytes(n, nch, sh.I);
  if (smem > static_cast<size_t>(di.smem_optin) || workspace_bytes < small_workspace_bytes(n)) return false;
  const bool pot = flags & B2_POTENTIAL;
  const void* fn = reinterpret_cast<const void*>(pot ? small_kernel<true>(sh.NP) : small_kernel<false>(sh.NP));
  allow_max_dynamic_smem(fn);
  // co-residency of the whole grid (cooperative launch), cached per shape and device: the
  // occupancy query costs microseconds of host time on a ~200 us run
  struct Fit {
    const void* fn;
    int threads, dev;
    size_t smem;
    bool ok;
  };
  static thread_local Fit last{nullptr, 0, -1, 0, false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (last.fn != fn || last.threads != sh.threads || last.smem != smem || last.dev != dev) {
    int per_sm = 0;
    const bool ok = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, sh.threads, smem) == cudaSuccess &&
                    per_sm * di.sms >= sh.ctas;
    cudaGetLastError();
    last = Fit{fn, sh.threads, dev, smem, ok};
  }
  if (!last.ok) return false;
  float4* pub = static_cast<float4*>(workspace);
  // only the counters need zeroing (the positions are written before they are read)
  if (cudaMemsetAsync(pub + 2 * static_cast<size_t>(n), 0, 1024, s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  SmallArgs args{n, pos, vel, acc, pub, reinterpret_cast<unsigned int*>(pub + 2 * static_cast<size_t>(n)), eps * eps, dt, 0.5f * dt, nsteps, flags & (B2_POTENTIAL | B2_INIT_ACC),
                 chunk_size(n, flags & B2_POTENTIAL), nch, sh.I, sh.G, make_watch(), debug_withhold()};
  void* argv[] = {&args};
  if (cudaLaunchCooperativeKernel(fn, sh.ctas, sh.threads, argv, smem, s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

}  // namespace b2
