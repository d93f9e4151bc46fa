// K3'' -- the shared-memory-resident diffusion time loop (all steps of a grid that
// fits the SMs' shared memory in one persistent launch), for b2_diffusion3d_run.
// Reference arithmetic: pkg/tests/fixtures/listing_diffusion.c:5-25 via cell4
// (diffusion_common.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <mutex>

#include "diffusion_common.cuh"

namespace b2 {

// ---------------------------------------------------------------------------
// Shared-memory-resident time loop for grids that fit the chip's aggregate
// shared memory (configs[1]: 128^3 = 8 MiB over 128 SMs). Per-step launches and
// grid-wide barriers both leave a 128^3 step at ~6.5 us, bound by dependent L2
// round trips, not by bandwidth. Here the field never leaves the SMs:
//
//  * one persistent CTA per brick of BI planes x BJ rows x all nz (cooperative
//    launch => co-resident); the brick lives in shared memory for all steps,
//    ping-ponging between two copies; each thread marches one float4 column
//    along i (old i-1 / i in registers);
//  * bricks exchange only their boundary faces, as self-validating 16-byte
//    words {v0, v1, v2, step tag} in a per-brick mailbox (face x step parity).
//    A .b128 access is single-copy atomic (the PTX memory model; libcu++'s
//    16-byte cuda::atomic uses the same instruction), so a consumer polls the
//    data itself: no fence, no flag, no grid barrier -- the step-to-step
//    critical path is one L2 store->load latency;
//  * f is read at step 0 (own cells and halos); the final state is written
//    once, to buffer nsteps & 1 (b2_diffusion3d_run's ping-pong contract; the
//    other buffer is untouched).
//
// A producer cannot lap a consumer: exporting step s+2's faces needs the
// consumer's step s+1 faces, which the consumer exports only after it pulled
// step s+1's -- so two mailbox parities suffice. A face that never arrives ends the run
// through the watchdog (poll_expired, runtime.cu). Same arithmetic and clamps as
// k_diffusion_direct: bit-identical to single steps.
struct ResArgs {
  float* f;
  float* fn;
  int nx, ny, nz;
  int nsteps;
  int BI, BJ, nbj;
  uint4* mbox;   // [brick][face 0..3][parity][face_cap] 16-byte words, zeroed before launch
  int face_cap;  // words per face: max(BI, BJ) rows x ceil(nz / 3)
  Coefs c;
  Watch watch;  // a face that never arrives ends the run (runtime.cu), no trap
#ifdef B2_RESIDENT_TRACE
  unsigned long long* trace;  // [brick][step][4] globaltimer stamps (scripts/trace_resident.cu)
#endif
};
#ifdef B2_RESIDENT_TRACE
#define B2_TRACE(k) \
  if (tid == 0) a.trace[(static_cast<size_t>(b) * a.nsteps + s) * 4 + (k)] = globaltimer_ns()
#else
#define B2_TRACE(k)
#endif


constexpr int kResidentThreads = 512;
constexpr int kResidentUnits = 6;  // max halo words per thread per step

__global__ void __launch_bounds__(kResidentThreads, 1) k_diffusion_resident(const ResArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int nz = a.nz, nz4 = nz >> 2, ny = a.ny, nx = a.nx;
  const int BJ = a.BJ, nbj = a.nbj;
  const int b = blockIdx.x;
  const int i0 = (b / nbj) * a.BI, j0 = (b % nbj) * BJ;
  const int PI = min(a.BI, nx - i0), PJ = min(BJ, ny - j0);  // planes / rows owned
  const size_t plane = static_cast<size_t>(ny) * nz;
  const int planef = (BJ + 2) * nz;  // smem plane q = own plane q-1, row r = own row r-1
  const int buff = (a.BI + 2) * planef;
  const bool has_im = i0 > 0, has_ip = i0 + PI < nx, has_jm = j0 > 0, has_jp = j0 + PJ < ny;
  const int tid = threadIdx.x;
  const int per_plane = PJ * nz4;  // float4 cells of one own plane
  const int cap = a.face_cap;      // mailbox of face d of brick bb, parity p: a.mbox + ((bb*4 + d)*2 + p)*cap

  float* cur = sm;
  float* nxt = sm + buff;
  auto at = [&](int q, int r) { return q * planef + r * nz; };  // float offset inside a buffer

  // own cells, state 0
  for (int u = tid; u < PI * per_plane; u += blockDim.x) {
    const int l = u / per_plane, v = u - l * per_plane, jj = v / nz4, c4 = v - jj * nz4;
    *reinterpret_cast<float4*>(cur + at(l + 1, jj + 1) + 4 * c4) = __ldg(reinterpret_cast<const float4*>(
        a.f + static_cast<size_t>(i0 + l) * plane + static_cast<size_t>(j0 + jj) * nz) + c4);
  }

  // this thread's column (row jj, float4 column c4)
  const int jj = tid / nz4, c4 = tid - (tid / nz4) * nz4;
  const bool mine = tid < per_plane;
  const int rjp = jj + 1 < PJ ? jj + 2 : (has_jp ? PJ + 1 : jj + 1);  // smem rows; clamp = own row
  const int rjm = jj > 0 ? jj : (has_jm ? 0 : jj + 1);
  const int djp = (rjp - (jj + 1)) * nz, djm = (rjm - (jj + 1)) * nz;
  const Coefs c = a.c;

  // Halo / face words: 3 consecutive-k values of one row (rows padded to
  // n3 = ceil(nz/3) words). A brick's face toward neighbour X has exactly the
  // shape of X's face toward it, so one word numbering serves both directions:
  //   [i-lo: PJ rows][i-hi: PJ rows][j-lo: PI planes][j-hi: PI planes], present faces only.
  const int n3 = (nz + 2) / 3, rem = nz - 3 * (n3 - 1);  // values in a row's last word (1..3)
  const int n_iu = PJ * n3, n_ju = PI * n3;
  const int nu = (has_im + has_ip) * n_iu + (has_jm + has_jp) * n_ju;
  auto locate = [&](int u, int& seg, int& row, int& t) {  // word -> face, row (or plane), word in row
    seg = 0;
    if (has_im) {
      if (u < n_iu) goto found;
      u -= n_iu;
    }
    seg = 1;
    if (has_ip) {
      if (u < n_iu) goto found;
      u -= n_iu;
    }
    seg = 2;
    if (has_jm) {
      if (u < n_ju) goto found;
      u -= n_ju;
    }
    seg = 3;
  found:
    row = u / n3;
    t = u - row * n3;
  };
  auto halo_slot = [&](int seg, int row) {  // smem row receiving a neighbour's face row
    return seg < 2 ? at(seg == 0 ? 0 : PI + 1, row + 1) : at(row + 1, seg == 2 ? 0 : PJ + 1);
  };
  // Per-thread word descriptors, fixed for the launch (parity 0 / buffer 0 offsets):
  //   pull: neighbour's mailbox word -> my halo slot;  export: my own cells -> my mailbox word.
  // (smem offsets < 2^16 floats: pull_dst and exp_src share one register)
  int pull_src[kResidentUnits], exp_dst[kResidentUnits];
  unsigned int smem_off[kResidentUnits];  // pull_dst | exp_src << 16
  unsigned int short_words = 0;  // bit w: word w holds `rem` < 3 values
#pragma unroll
  for (int w = 0; w < kResidentUnits; ++w) {
    const int u = tid + w * kResidentThreads;
    pull_src[w] = exp_dst[w] = 0;
    smem_off[w] = 0;
    if (u < nu) {
      int seg, row, t;
      locate(u, seg, row, t);
      const int within = row * n3 + t;
      const int nb = seg == 0 ? b - nbj : seg == 1 ? b + nbj : seg == 2 ? b - 1 : b + 1;
      pull_src[w] = (nb * 8 + 2 * (seg ^ 1)) * cap + within;  // the neighbour's face pointing back at me
      exp_dst[w] = (b * 8 + 2 * seg) * cap + within;
      const int pull_dst = halo_slot(seg, row) + 3 * t;
      const int exp_src = (seg < 2 ? at(seg == 0 ? 1 : PI, row + 1) : at(row + 1, seg == 2 ? 1 : PJ)) + 3 * t;
      smem_off[w] = static_cast<unsigned int>(pull_dst) | (static_cast<unsigned int>(exp_src) << 16);
      if (t == n3 - 1 && rem < 3) short_words |= 1u << w;
    }
  }

  for (int s = 0; s < a.nsteps; ++s) {
    B2_TRACE(0);
    bool dead = false;  // this thread gave up waiting for a face
    // ---- pull the halo of state s into cur ----
    if (s == 0) {
      for (int u = tid; u < nu; u += blockDim.x) {
        int seg, row, t;
        locate(u, seg, row, t);
        const size_t src = seg < 2 ? static_cast<size_t>(seg == 0 ? i0 - 1 : i0 + PI) * plane +
                                         static_cast<size_t>(j0 + row) * nz
                                   : static_cast<size_t>(i0 + row) * plane +
                                         static_cast<size_t>(seg == 2 ? j0 - 1 : j0 + PJ) * nz;
        const int cnt = t == n3 - 1 ? rem : 3;
        for (int e = 0; e < cnt; ++e) cur[halo_slot(seg, row) + 3 * t + e] = a.f[src + 3 * t + e];
      }
    } else {
      const unsigned int want = static_cast<unsigned int>(s);
      const uint4* mb = a.mbox + (s & 1) * cap;
      uint4 v[kResidentUnits];
      unsigned int todo = 0;
#pragma unroll
      for (int w = 0; w < kResidentUnits; ++w) {
        if (tid + w * kResidentThreads < nu) {
          v[w] = ld_relaxed_b128(mb + pull_src[w]);
          todo |= 1u << w;
        }
      }
      const unsigned long long t0 = globaltimer_ns();
      while (todo) {
#pragma unroll
        for (int w = 0; w < kResidentUnits; ++w) {
          if (!(todo >> w & 1)) continue;
          if (v[w].w == want) {
            float* d = cur + (smem_off[w] & 0xffffu);
            d[0] = __uint_as_float(v[w].x);
            if (!(short_words >> w & 1) || rem > 1) d[1] = __uint_as_float(v[w].y);
            if (!(short_words >> w & 1)) d[2] = __uint_as_float(v[w].z);
            todo &= ~(1u << w);
          } else {
            v[w] = ld_relaxed_b128(mb + pull_src[w]);  // not there yet: poll again
          }
        }
        // A neighbour never arrived: give up instead of hanging the GPU (the watchdog
        // records it; b2_fault_status reports it). (A poll back-off of 64-1000 ns was
        // measured slower: the lines are not contended.)
        if (todo && poll_expired(a.watch, t0, kFaultResident)) {
          dead = true;
          break;
        }
      }
    }
    // barrier + CTA-wide vote (no static shared memory next to the full dynamic allocation)
    if (__syncthreads_or(dead)) return;  // uniform: f / fn left as they were
    B2_TRACE(1);
    // ---- march this thread's column: cur (state s) -> nxt (state s+1); smem only ----
    // (Computing the brick's shell first and exporting it before the interior was
    // measured slower on B200: 3.96 vs 3.67 us/step at 128^3.)
    if (mine) {
      const float* __restrict__ pc = cur + at(1, jj + 1) + 4 * c4;
      float* __restrict__ pn = nxt + at(1, jj + 1) + 4 * c4;
      float4 fc = *reinterpret_cast<const float4*>(pc);
      float4 fim = has_im ? *reinterpret_cast<const float4*>(pc - planef) : fc;  // IMAX(i-1, 0)
#pragma unroll 2
      for (int l = 0; l < PI; ++l) {
        const float4 fip = (l + 1 < PI || has_ip) ? *reinterpret_cast<const float4*>(pc + planef) : fc;  // IMIN
        const float4 fjp = *reinterpret_cast<const float4*>(pc + djp);
        const float4 fjm = *reinterpret_cast<const float4*>(pc + djm);
        // (k neighbours by warp shuffle instead of these two loads measured slower: 2.2 vs 1.7 us/step)
        const float kl = c4 > 0 ? pc[-1] : fc.x;        // IMAX(k-1, 0)
        const float kr = c4 + 1 < nz4 ? pc[4] : fc.w;  // IMIN(k+1, nz-1)
        *reinterpret_cast<float4*>(pn) = cell4(c, fc, fip, fim, fjp, fjm, kl, kr);
        fim = fc;
        fc = fip;
        pc += planef;
        pn += planef;
      }
    }
    __syncthreads();  // nxt complete
    B2_TRACE(2);
    // ---- export my faces of state s+1: every thread, 16-byte tagged words ----
    {
      const unsigned int tag = static_cast<unsigned int>(s + 1);
      uint4* mb = a.mbox + ((s + 1) & 1) * cap;
#pragma unroll
      for (int w = 0; w < kResidentUnits; ++w) {
        if (tid + w * kResidentThreads < nu) {
          const float* q = nxt + (smem_off[w] >> 16);
          const bool full = !(short_words >> w & 1);
          st_relaxed_b128(mb + exp_dst[w], make_uint4(__float_as_uint(q[0]),
                                                      full || rem > 1 ? __float_as_uint(q[1]) : 0u,
                                                      full ? __float_as_uint(q[2]) : 0u, tag));
        }
      }
    }
    float* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  if (a.nsteps == 0) return;
  float* Z = (a.nsteps & 1) ? a.fn : a.f;
  for (int u = tid; u < PI * per_plane; u += blockDim.x) {
    const int l = u / per_plane, v = u - l * per_plane, r = v / nz4, k4 = v - r * nz4;
    reinterpret_cast<float4*>(Z + static_cast<size_t>(i0 + l) * plane + static_cast<size_t>(j0 + r) * nz)[k4] =
        *reinterpret_cast<const float4*>(cur + at(l + 1, r + 1) + 4 * k4);
  }
}

// Brick plan for k_diffusion_resident: at most one brick per SM, two copies of
// the brick plus its halo in one SM's shared memory, one float4 column per
// thread (BJ*nz/4 <= 512), at most kResidentUnits halo units per thread. Fewest
// planes per brick wins (each plane is one cell on every thread's march).
struct ResPlan {
  int BI = 0, BJ = 0, nbi = 0, nbj = 0;
  size_t smem = 0;
};

static bool resident_plan_for(int nx, int ny, int nz, ResPlan& p) {
  if (nz % 4 != 0 || nz / 4 > kResidentThreads) return false;
  const int nz4 = nz / 4;
  const DeviceInfo& di = device_info();
  const size_t cap = static_cast<size_t>(di.smem_optin > 0 ? di.smem_optin : 227 * 1024);
  for (int BJ = 1; BJ * nz4 <= kResidentThreads; BJ *= 2) {
    const int bj = std::min(BJ, ny);
    const int nbj = (ny + bj - 1) / bj;
    if (nbj <= di.sms) {
      const int per = di.sms / nbj;
      const int BI = (nx + per - 1) / per;
      const int nbi = (nx + BI - 1) / BI;
      const size_t smem = 2 * static_cast<size_t>(BI + 2) * (bj + 2) * nz * sizeof(float);
      const long long halo_units = (2LL * bj + 2LL * BI) * ((nz + 2) / 3);
      if (smem <= cap && smem / 2 / sizeof(float) < 65536 &&
          halo_units <= static_cast<long long>(kResidentUnits) * kResidentThreads &&
          (!p.BI || BI < p.BI || (BI == p.BI && bj > p.BJ))) {
        p.BI = BI;
        p.BJ = bj;
        p.nbi = nbi;
        p.nbj = nbj;
        p.smem = smem;
      }
    }
    if (bj == ny) break;
  }
  return p.BI > 0;
}

// Per-device mailbox for k_diffusion_resident, sized by plan_resident (b2_diffusion3d_plan:
// allocation and the wait for earlier users happen there, never in the stream-ordered
// run). Launches on one device are chained through an event (each waits for the
// previous one to finish with the mailbox), so concurrent runs on different streams
// stay safe.
struct Mailbox {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaEvent_t done = nullptr;
  bool used = false;
};
static std::mutex g_mbox_mu;
static Mailbox g_boxes[64];

static size_t resident_mailbox_bytes(const ResPlan& p, int nz) {
  const int face_cap = std::max(p.BI, p.BJ) * ((nz + 2) / 3);
  return static_cast<size_t>(p.nbi) * p.nbj * 4 * 2 * face_cap * sizeof(uint4);
}

int plan_resident(int nx, int ny, int nz) {
  ResPlan p;
  if (!resident_plan_for(nx, ny, nz, p)) return B2_OK;  // not a resident shape: nothing to set up
  const size_t bytes = resident_mailbox_bytes(p, nz);
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mbox_mu);
  Mailbox& mb = g_boxes[dev];
  cudaError_t e;
  if (!mb.done && (e = cudaEventCreateWithFlags(&mb.done, cudaEventDisableTiming)) != cudaSuccess) {
    mb.done = nullptr;
    return static_cast<int>(e);
  }
  if (mb.bytes >= bytes) return B2_OK;
  if (mb.ptr) {
    cudaEventSynchronize(mb.done);  // the last run that used the old mailbox is done with it
    cudaFree(mb.ptr);
  }
  mb.ptr = nullptr;
  mb.bytes = 0;
  mb.used = false;
  if ((e = cudaMalloc(&mb.ptr, bytes)) != cudaSuccess) {
    cudaGetLastError();
    mb.ptr = nullptr;
    return static_cast<int>(e);
  }
  mb.bytes = bytes;
  return B2_OK;
}

bool launch_resident(int nx, int ny, int nz, const Coefs& c, float* f, float* fn, int nsteps, cudaStream_t s) {
  ResPlan p;
  if (!resident_plan_for(nx, ny, nz, p)) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;  // the event chain below is not capturable; per-step path instead
  }
  const int nbricks = p.nbi * p.nbj;
  allow_max_dynamic_smem(reinterpret_cast<const void*>(k_diffusion_resident));
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mbox_mu);
  Mailbox& mb = g_boxes[dev];
  const size_t bytes = resident_mailbox_bytes(p, nz);
  if (!mb.ptr || mb.bytes < bytes) return false;  // not planned for this shape (b2_diffusion3d_plan)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_diffusion_resident, kResidentThreads, p.smem) !=
          cudaSuccess ||
      per_sm * device_info().sms < nbricks) {
    cudaGetLastError();
    return false;
  }
  const int face_cap = std::max(p.BI, p.BJ) * ((nz + 2) / 3);
  if (mb.used) cudaStreamWaitEvent(s, mb.done, 0);
  cudaMemsetAsync(mb.ptr, 0, bytes, s);  // no stale tags
  ResArgs a{f, fn, nx, ny, nz, nsteps, p.BI, p.BJ, p.nbj, static_cast<uint4*>(mb.ptr), face_cap, c, make_watch()};
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_diffusion_resident), nbricks, kResidentThreads,
                                  args, p.smem, s) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaEventRecord(mb.done, s);
  mb.used = true;
  return true;
}

}  // namespace b2
