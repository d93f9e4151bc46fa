// K4 -- the fused slab-halo exchange of the multi-GPU diffusion path
// (SlabDiffusion, transport="p2p"). Slabs along i, the slowest
// axis of INDEX (listing_diffusion.c:1); a rank's two edge planes need one
// plane from each neighbour per step (the IMAX/IMIN(i+-1) terms of :15-16).
//
// One kernel per step computes both edge planes of the slab and moves the
// halo itself, over peer memory with no collective, no event and no host
// barrier:
//   * every rank owns a mailbox per side: [2 step parities][ny rows][ceil(nz/2)]
//     16-byte words {v0, tag, v1, tag}, tag = state index + 1. Each 8-byte half
//     carries its own tag, so a word is ready when both tags match even if the
//     fabric splits the 16-byte peer store into 8-byte pieces (the only
//     atomicity relied on across NVLink; NCCL's LL protocol makes the same
//     assumption). A word carries its own readiness: no flag, no fence;
//   * the edge kernel polls its own mailbox for the neighbour's plane of
//     state s (rows of this CTA only), computes its edge rows of state s+1 and
//     stores them, tagged, straight into the neighbour's mailbox (NVLink /
//     NVSwitch peer stores; the pointer is a CUDA-IPC mapping);
//   * a row that never arrives (dead or stalled peer) ends the wait after the
//     poll timeout through the watchdog (poll_expired, runtime.cu): the kernel
//     exits normally and b2_fault_status reports B2_ETIMEOUT -- no trap, the
//     context survives;
//   * a producer cannot lap a consumer: its state s+2 rows need the consumer's
//     state s+1 rows, which the consumer pushes only after it has read state s
//     (same row tiling on every rank), so two parities suffice.
// The interior planes are an ordinary b2_diffusion3d_slab launch. Arithmetic
// and clamps are those of the single-device step (cell4): bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>

#include "diffusion_common.cuh"

namespace b2 {

constexpr int kEdgeThreads = 256;

struct EdgeArgs {
  const float* f;
  float* fn;
  int nx, ny, nz;
  int TJ;             // rows per CTA
  const uint4* in_lo;  // my mailbox, side fed by rank-1 (null: global i = 0, clamp)
  const uint4* in_hi;  // my mailbox, side fed by rank+1 (null: global i = nx-1, clamp)
  uint4* out_lo;       // rank-1's mailbox side fed by me (null: no neighbour)
  uint4* out_hi;       // rank+1's mailbox side fed by me
  int step;            // computes state step+1 from state step
  int push_only;       // setup: publish this rank's edge planes of state `step`
  Coefs c;
  Watch watch;         // a neighbour that never pushes ends the step (runtime.cu), no trap
};

__global__ void __launch_bounds__(kEdgeThreads) k_diffusion_slab_edges(const EdgeArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int nz = a.nz, nz4 = nz >> 2, ny = a.ny, nx = a.nx, TJ = a.TJ;
  const int n2 = (nz + 1) / 2;  // words per row: two values each
  const int side = blockIdx.y;  // 0: plane 0 (halo from rank-1), 1: plane nx-1 (halo from rank+1)
  const int p = side ? nx - 1 : 0;
  const size_t plane = static_cast<size_t>(ny) * nz;
  const float* fp = a.f + static_cast<size_t>(p) * plane;
  const uint4* in = side ? a.in_hi : a.in_lo;
  uint4* out = side ? a.out_hi : a.out_lo;
  const int j0 = blockIdx.x * TJ, rows = min(TJ, ny - j0);
  const int tid = threadIdx.x;
  auto word = [&](int parity, int j, int t) { return (static_cast<size_t>(parity) * ny + j) * n2 + t; };
  auto push = [&](const float* rowsrc, size_t rstride, int state) {  // rows j0.. of state `state` -> out
    const unsigned int tag = static_cast<unsigned int>(state + 1);
    for (int w = tid; w < rows * n2; w += blockDim.x) {
      const int r = w / n2, t = w - r * n2, k = 2 * t;
      const float* src = rowsrc + r * rstride + k;
      const uint4 v = make_uint4(__float_as_uint(src[0]), tag, k + 1 < nz ? __float_as_uint(src[1]) : 0u, tag);
      st_relaxed_sys_b128(out + word(state & 1, j0 + r, t), v);  // peer GPU memory: system scope
    }
  };
  if (a.push_only) {
    if (out) push(fp + static_cast<size_t>(j0) * nz, nz, a.step);
    return;
  }
  float* halo = sm;            // [TJ][nz] the neighbour's plane of state `step`, rows j0..
  float* res = sm + TJ * nz;   // [TJ][nz] this CTA's new edge rows (state step+1)
  bool gave_up = false;  // this thread's wait expired (voted CTA-wide below)
  if (in) {
    const unsigned int want = static_cast<unsigned int>(a.step + 1);
    const unsigned long long t0 = globaltimer_ns();
    for (int w = tid; w < rows * n2; w += blockDim.x) {
      const int r = w / n2, t = w - r * n2, k = 2 * t;
      const uint4* src = in + word(a.step & 1, j0 + r, t);
      uint4 v = ld_relaxed_sys_b128(src);  // written by a peer GPU: system scope
      bool dead = false;
      while (v.y != want || v.w != want) {  // the neighbour's row (both halves) is not there yet
        if ((dead = poll_expired(a.watch, t0, kFaultSlabEdges))) break;  // a dead peer: give up, no hang
        __nanosleep(64);
        v = ld_relaxed_sys_b128(src);
      }
      if (dead) {
        gave_up = true;
        break;
      }
      float* d = halo + r * nz + k;
      d[0] = __uint_as_float(v.x);
      if (k + 1 < nz) d[1] = __uint_as_float(v.z);
    }
  }
  if (__syncthreads_or(gave_up)) return;  // uniform: no edge planes, nothing pushed (b2_fault_status reports it)
  const float* fo = a.f + static_cast<size_t>(side ? nx - 2 : 1) * plane;  // the in-slab i neighbour
  for (int u = tid; u < rows * nz4; u += blockDim.x) {
    const int r = u / nz4, c4 = u - r * nz4, j = j0 + r;
    const float* row = fp + static_cast<size_t>(j) * nz;
    const float4 fc = reinterpret_cast<const float4*>(row)[c4];
    const float4 fh = in ? *reinterpret_cast<const float4*>(halo + r * nz + 4 * c4) : fc;  // IMAX/IMIN(i+-1) clamp
    const float4 fs = reinterpret_cast<const float4*>(fo + static_cast<size_t>(j) * nz)[c4];
    const float4 fjp = reinterpret_cast<const float4*>(fp + static_cast<size_t>(min(j + 1, ny - 1)) * nz)[c4];
    const float4 fjm = reinterpret_cast<const float4*>(fp + static_cast<size_t>(max(j - 1, 0)) * nz)[c4];
    const float kl = c4 > 0 ? row[4 * c4 - 1] : fc.x;        // IMAX(k-1, 0)
    const float kr = c4 + 1 < nz4 ? row[4 * c4 + 4] : fc.w;  // IMIN(k+1, nz-1)
    const float4 o = side ? cell4(a.c, fc, fh, fs, fjp, fjm, kl, kr)   // fip = halo, fim = plane nx-2
                          : cell4(a.c, fc, fs, fh, fjp, fjm, kl, kr);  // fip = plane 1, fim = halo
    reinterpret_cast<float4*>(a.fn + static_cast<size_t>(p) * plane + static_cast<size_t>(j) * nz)[c4] = o;
    *reinterpret_cast<float4*>(res + r * nz + 4 * c4) = o;
  }
  __syncthreads();
  if (out) push(res, nz, a.step + 1);
}

// ---------------------------------------------------------------------------
// Two-plane halo exchange for SlabDiffusion.run (two steps per exchange):
// between two-step passes each rank ships its two edge planes of the current state to
// each neighbour and takes the neighbours' into the halo planes of its halo-extended
// slab [lo_h halo | nx_local own | hi_h halo] (lo_h, hi_h = 2, or 0 at a global end,
// where the pass's own clamp applies). Same self-validating words as above, one
// 8-byte half per value pair: {v, tag, v, tag}, tag = exchange index + 1, two
// exchange parities. Phase 0 pushes (no waiting); phase 1 polls its own mailbox and
// writes the halo planes. Two launches, so every push of a rank is issued before any
// of its CTAs waits: no cross-rank cycle whatever the residency.
struct Xchg2Args {
  float* f;
  int ny, nz, TJ;
  int lo_h, nxl;
  const uint4* in_lo;  // my mailbox sides, fed by rank-1 / rank+1 (null: global end)
  const uint4* in_hi;
  uint4* out_lo;  // the neighbours' sides fed by me (null: no neighbour)
  uint4* out_hi;
  int xchg, phase;
  Watch watch;
};

__global__ void __launch_bounds__(kEdgeThreads) k_diffusion_slab_halo2(const Xchg2Args a) {
  const int ny = a.ny, nz = a.nz, n2 = (nz + 1) / 2;
  const int side = blockIdx.y;
  const int j0 = blockIdx.x * a.TJ, rows = min(a.TJ, ny - j0);
  const size_t plane = static_cast<size_t>(ny) * nz;
  const int parity = a.xchg & 1;
  const unsigned int tag = static_cast<unsigned int>(a.xchg + 1);
  auto word = [&](int p, int j, int t) { return ((static_cast<size_t>(parity) * 2 + p) * ny + j) * n2 + t; };
  const int per_plane = rows * n2;
  if (a.phase == 0) {
    uint4* out = side ? a.out_hi : a.out_lo;
    if (!out) return;
    const int first = side ? a.lo_h + a.nxl - 2 : a.lo_h;  // my two planes next to that neighbour
    for (int w = threadIdx.x; w < 2 * per_plane; w += blockDim.x) {
      const int p = w / per_plane, rem = w - p * per_plane, r = rem / n2, t = rem - r * n2, k = 2 * t;
      const float* src = a.f + static_cast<size_t>(first + p) * plane + static_cast<size_t>(j0 + r) * nz + k;
      st_relaxed_sys_b128(out + word(p, j0 + r, t),
                          make_uint4(__float_as_uint(src[0]), tag, k + 1 < nz ? __float_as_uint(src[1]) : 0u, tag));
    }
    return;
  }
  const uint4* in = side ? a.in_hi : a.in_lo;
  if (!in) return;
  const int dst0 = side ? a.lo_h + a.nxl : 0;  // my halo planes on that side
  const unsigned long long t0 = globaltimer_ns();
  for (int w = threadIdx.x; w < 2 * per_plane; w += blockDim.x) {
    const int p = w / per_plane, rem = w - p * per_plane, r = rem / n2, t = rem - r * n2, k = 2 * t;
    const uint4* src = in + word(p, j0 + r, t);
    uint4 v = ld_relaxed_sys_b128(src);
    while (v.y != tag || v.w != tag) {
      if (poll_expired(a.watch, t0, kFaultHalo2)) return;  // a dead peer: give up (watchdog), no hang
      __nanosleep(64);
      v = ld_relaxed_sys_b128(src);
    }
    float* d = a.f + static_cast<size_t>(dst0 + p) * plane + static_cast<size_t>(j0 + r) * nz + k;
    d[0] = __uint_as_float(v.x);
    if (k + 1 < nz) d[1] = __uint_as_float(v.z);
  }
}

}  // namespace b2

using namespace b2;

extern "C" {

size_t b2_diffusion3d_mailbox_bytes(int ny, int nz) {
  if (ny <= 0 || nz <= 0) return 0;
  return 2ull * static_cast<size_t>(ny) * ((nz + 1) / 2) * sizeof(uint4);  // one side: 2 parities
}

int b2_diffusion3d_slab_edges(int nx_local, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                              const float* f, float* fn, const void* in_lo, const void* in_hi, void* out_lo,
                              void* out_hi, int step, int push_only, void* stream) {
  if (nx_local < 2 || ny <= 0 || nz <= 0 || nz % 4 || !f || !fn || f == fn || step < 0) return B2_EINVAL;
  if (!aligned16(f) || !aligned16(fn) || !aligned16(in_lo) || !aligned16(in_hi) || !aligned16(out_lo) ||
      !aligned16(out_hi))
    return B2_EALIGN;
  const int nz4 = nz / 4;
  const int TJ = std::max(1, std::min(ny, kEdgeThreads / std::max(1, std::min(nz4, kEdgeThreads))));
  const size_t smem = 2ull * TJ * nz * sizeof(float);
  if (smem > static_cast<size_t>(device_info().smem_optin)) return B2_EINVAL;
  if (smem > 48 * 1024) allow_max_dynamic_smem(reinterpret_cast<const void*>(k_diffusion_slab_edges));
  EdgeArgs a{f,
             fn,
             nx_local,
             ny,
             nz,
             TJ,
             static_cast<const uint4*>(in_lo),
             static_cast<const uint4*>(in_hi),
             static_cast<uint4*>(out_lo),
             static_cast<uint4*>(out_hi),
             step,
             push_only,
             make_coefs(dx, dy, dz, dt, kappa),
             make_watch()};
  const dim3 grid((ny + TJ - 1) / TJ, 2);
  k_diffusion_slab_edges<<<grid, kEdgeThreads, push_only ? 0 : smem, as_stream(stream)>>>(a);
  return launch_status();
}

size_t b2_diffusion3d_mailbox2_bytes(int ny, int nz) {
  if (ny <= 0 || nz <= 0) return 0;
  return 4ull * static_cast<size_t>(ny) * ((nz + 1) / 2) * sizeof(uint4);  // one side: 2 parities x 2 planes
}

int b2_diffusion3d_slab_halo2(int nx_ext, int ny, int nz, int lo_h, int nx_local, float* f, const void* in_lo,
                              const void* in_hi, void* out_lo, void* out_hi, int xchg, int phase, void* stream) {
  const int hi_h = nx_ext - lo_h - nx_local;
  if (nx_local < 2 || ny <= 0 || nz <= 0 || !f || xchg < 0 || (phase != 0 && phase != 1) ||
      (lo_h != 0 && lo_h != 2) || (hi_h != 0 && hi_h != 2) || (in_lo && lo_h != 2) || (in_hi && hi_h != 2))
    return B2_EINVAL;
  if (!aligned16(in_lo) || !aligned16(in_hi) || !aligned16(out_lo) || !aligned16(out_hi)) return B2_EALIGN;
  const int n2 = (nz + 1) / 2;
  const int TJ = std::max(1, std::min(ny, 2048 / (2 * n2)));
  Xchg2Args a{f,
              ny,
              nz,
              TJ,
              lo_h,
              nx_local,
              static_cast<const uint4*>(in_lo),
              static_cast<const uint4*>(in_hi),
              static_cast<uint4*>(out_lo),
              static_cast<uint4*>(out_hi),
              xchg,
              phase,
              make_watch()};
  k_diffusion_slab_halo2<<<dim3((ny + TJ - 1) / TJ, 2), kEdgeThreads, 0, as_stream(stream)>>>(a);
  return launch_status();
}

}  // extern "C"
