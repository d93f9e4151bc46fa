// K3: one explicit 7-point diffusion step (diffusion3d), hand-written for sm_100a.
//
// Reference: pkg/tests/fixtures/listing_diffusion.c:1-25 (= PAPER.md:553-578).
//   INDEX(nx,ny,nz,i,j,k) = k + nz*(j + ny*i)        (:1)  k fastest, i slowest
//   ce=cw=kappa*dt/dx^2, cn=cs=kappa*dt/dy^2, ct=cb=kappa*dt/dz^2, cc=1-sum (:6-9)
//   fn = cc*f + ce*f[i+1] + cw*f[i-1] + cn*f[j+1] + cs*f[j-1] + ct*f[k+1] + cb*f[k-1]
//   with neighbour indices clamped to the grid (:15-20).
//
// Design: HBM-bound (8 B/cell algorithmic). Each CTA owns a
// tile of TJ full-width rows (j0..j0+TJ-1, all k) and marches along i (the
// slowest, plane-contiguous axis) over a range of planes. A tile-plane plus
// its j-1/j+1 halo rows is ONE contiguous run of (TJ+2)*nz floats, so it is
// fetched with a single cp.async.bulk (UBLKCP, the TMA bulk-copy engine) into
// an NST-deep shared-memory ring completed on mbarriers. Each thread keeps the
// f[i-1] and f[i] values of its cells in registers, reads f[i+1] and the
// in-plane neighbours from shared memory, and streams fn out with 16-byte
// stores -- every f value crosses HBM once. The clamp of :15-20 is applied in
// the kernel (TMA does not clamp). The arithmetic is the reference's as g++
// -O3 contracts it: v = ce*f_ip; v = fma(cc, f, v); then
// fma(cw,f_im), fma(cn,f_jp), fma(cs,f_jm), fma(ct,f_kp), fma(cb,f_km) --
// bit-identical to the reference build.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "diffusion_common.cuh"

namespace b2 {

// ---------------------------------------------------------------------------
// Marching kernel. Template S = float4 cells per thread per plane (registers).
// Runtime: TJ rows per tile (TJ*nz/4 <= 256*S), NST pipeline stages.
constexpr int kMarchThreads = 256;

struct MarchArgs {
  const float* f;        // local planes [0, nx)
  const float* halo_lo;  // plane -1 or null (clamp)
  const float* halo_hi;  // plane nx or null (clamp)
  float* fn;
  int nx, ny, nz;
  int TJ, n_jtiles;
  int i_begin, i_end, IC;  // output planes [i_begin, i_end), IC planes per CTA
  int nst;
  Coefs c;
};

template <int S>
__global__ void __launch_bounds__(kMarchThreads, (S <= 2 ? 4 : 2)) k_diffusion_march(const MarchArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nz = a.nz, ny = a.ny, nx = a.nx;
  const int nz4 = nz >> 2;
  const int TJ = a.TJ, NST = a.nst;
  const size_t plane = static_cast<size_t>(ny) * nz;
  const int stage_floats = (TJ + 2) * nz;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  float* stages = reinterpret_cast<float*>(smem_raw + 128);

  const int jt = blockIdx.x % a.n_jtiles;
  const int ic = blockIdx.x / a.n_jtiles;
  const int j0 = jt * TJ;
  const int rows = min(TJ, ny - j0);
  const int i0 = a.i_begin + ic * a.IC;
  const int i1 = min(i0 + a.IC, a.i_end);
  if (i0 >= i1) return;  // uniform per CTA
  const int L = (i1 - i0) + 2;  // planes to fetch: i0-1 .. i1

  const int jlo = max(j0 - 1, 0);
  const int jhi = min(j0 + rows, ny - 1);  // inclusive
  const uint32_t bytes = static_cast<uint32_t>((jhi - jlo + 1) * nz * sizeof(float));
  const int dst_row = jlo - (j0 - 1);  // buffer row q <-> global row j0-1+q

  auto plane_src = [&](int p) -> const float* {
    if (p < 0) return a.halo_lo ? a.halo_lo : a.f;  // IMAX(i-1, 0)
    if (p >= nx) return a.halo_hi ? a.halo_hi : a.f + static_cast<size_t>(nx - 1) * plane;  // IMIN(i+1, nx-1)
    return a.f + static_cast<size_t>(p) * plane;
  };
  auto issue = [&](int q) {  // fetch plane i0-1+q into stage q % NST
    const int st = q % NST;
    uint64_t* bar = bars + st;
    mbar_expect_tx(bar, bytes);
    bulk_g2s(stages + static_cast<size_t>(st) * stage_floats + dst_row * nz,
             plane_src(i0 - 1 + q) + static_cast<size_t>(jlo) * nz, bytes, bar);
  };

  if (threadIdx.x == 0) {
    for (int st = 0; st < NST; ++st) mbar_init(bars + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int pre = min(NST, L);
    for (int q = 0; q < pre; ++q) issue(q);
  }
  __syncthreads();

  // Per-thread cell positions within the tile.
  int srow[S], scol[S];
  bool sval[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int pos = threadIdx.x + s * kMarchThreads;
    srow[s] = pos / nz4;
    scol[s] = pos - srow[s] * nz4;
    sval[s] = srow[s] < rows;
  }

  auto stage_ptr = [&](int q) -> const float* { return stages + static_cast<size_t>(q % NST) * stage_floats; };
  auto wait_q = [&](int q) { mbar_wait(bars + (q % NST), (q / NST) & 1); };
  auto own = [&](const float* buf, int s) -> float4 {
    return *reinterpret_cast<const float4*>(buf + (srow[s] + 1) * nz + 4 * scol[s]);
  };

  float4 fim[S], fc[S];
  // q = 0: plane i0-1 -> f[i-1] registers; release its stage.
  wait_q(0);
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (sval[s]) fim[s] = own(stage_ptr(0), s);
  __syncthreads();
  if (threadIdx.x == 0 && NST < L) {
    fence_proxy_async();
    issue(NST);
  }
  // q = 1: plane i0 -> f[i] registers (stage kept for the in-plane neighbours).
  wait_q(1);
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (sval[s]) fc[s] = own(stage_ptr(1), s);

  const Coefs c = a.c;
  for (int q = 1; q + 1 < L; ++q) {
    const int p = i0 + q - 1;  // output plane
    const float* cur = stage_ptr(q);
    wait_q(q + 1);
    const float* nxt = stage_ptr(q + 1);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (!sval[s]) continue;
      const int r = srow[s], c4 = scol[s];
      const int j = j0 + r;
      const float4 fip = own(nxt, s);
      const int rjp = min(j + 1, ny - 1) - (j0 - 1);
      const int rjm = max(j - 1, 0) - (j0 - 1);
      const float4 fjp = *reinterpret_cast<const float4*>(cur + rjp * nz + 4 * c4);
      const float4 fjm = *reinterpret_cast<const float4*>(cur + rjm * nz + 4 * c4);
      const float* rowp = cur + (r + 1) * nz;
      const float4 fcv = fc[s];
      const float kl = c4 > 0 ? rowp[4 * c4 - 1] : fcv.x;         // IMAX(k-1, 0)
      const float kr = c4 + 1 < nz4 ? rowp[4 * c4 + 4] : fcv.w;   // IMIN(k+1, nz-1)
      const float4 fm = fim[s];
      const float4 o = cell4(c, fcv, fip, fm, fjp, fjm, kl, kr);
      st_stream(reinterpret_cast<float4*>(a.fn + static_cast<size_t>(p) * plane + static_cast<size_t>(j) * nz) + c4, o);
      fim[s] = fcv;
      fc[s] = fip;
    }
    __syncthreads();  // everyone is done with stage q
    if (threadIdx.x == 0 && q + NST < L) {
      fence_proxy_async();
      issue(q + NST);
    }
  }
}


// ---------------------------------------------------------------------------
// Generic kernel for shapes the marching kernel does not take (nz % 4 != 0,
// unaligned pointers). One thread per cell, 64-bit offsets.
__global__ void __launch_bounds__(256)
    k_diffusion_generic(const float* __restrict__ f, const float* __restrict__ halo_lo,
                        const float* __restrict__ halo_hi, float* __restrict__ fn, int nx, int ny, int nz, int i_begin,
                        int i_end, Coefs c) {
  const size_t plane = static_cast<size_t>(ny) * nz;
  const size_t total = static_cast<size_t>(i_end - i_begin) * plane;
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int i = i_begin + static_cast<int>(t / plane);
    const size_t r = t % plane;
    const int j = static_cast<int>(r / nz);
    const int k = static_cast<int>(r % nz);
    const float* P = f + static_cast<size_t>(i) * plane;
    const float* Pm = i > 0 ? P - plane : (halo_lo ? halo_lo : P);
    const float* Pp = i < nx - 1 ? P + plane : (halo_hi ? halo_hi : P);
    const size_t jk = static_cast<size_t>(j) * nz + k;
    const float fc = P[jk];
    const float fjp = P[static_cast<size_t>(min(j + 1, ny - 1)) * nz + k];
    const float fjm = P[static_cast<size_t>(max(j - 1, 0)) * nz + k];
    const float fkp = P[static_cast<size_t>(j) * nz + min(k + 1, nz - 1)];
    const float fkm = P[static_cast<size_t>(j) * nz + max(k - 1, 0)];
    fn[static_cast<size_t>(i) * plane + jk] = cell(c, fc, Pp[jk], Pm[jk], fjp, fjm, fkp, fkm);
  }
}

// ---------------------------------------------------------------------------
// Direct kernel for L2-resident grids (configs[1]: 128^3 = 2 x 8 MiB): one
// thread per 4 consecutive k cells, every neighbour straight from L1/L2 with
// 16-byte loads. No staging pipeline to fill, so short steps are not
// latency-bound on the march kernel's prologue. Requires nz % 4 == 0 and
// 16-byte aligned f / fn; same arithmetic (bit-identical).
__global__ void __launch_bounds__(256)
    k_diffusion_direct(const float* __restrict__ f, const float* __restrict__ halo_lo,
                       const float* __restrict__ halo_hi, float* __restrict__ fn, int nx, int ny, int nz,
                       int i_begin, int i_end, Coefs c) {
  const int nz4 = nz >> 2;
  const size_t plane = static_cast<size_t>(ny) * nz;
  const size_t total = static_cast<size_t>(i_end - i_begin) * ny * nz4;
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int c4 = static_cast<int>(t % nz4);
    const size_t r = t / nz4;
    const int j = static_cast<int>(r % ny);
    const int i = i_begin + static_cast<int>(r / ny);
    const float* P = f + static_cast<size_t>(i) * plane;
    const float* Pm = i > 0 ? P - plane : (halo_lo ? halo_lo : P);
    const float* Pp = i < nx - 1 ? P + plane : (halo_hi ? halo_hi : P);
    const size_t jk = static_cast<size_t>(j) * nz + 4 * c4;
    const float4 fc = __ldg(reinterpret_cast<const float4*>(P + jk));
    const float4 fip = __ldg(reinterpret_cast<const float4*>(Pp + jk));
    const float4 fim = __ldg(reinterpret_cast<const float4*>(Pm + jk));
    const float4 fjp = __ldg(reinterpret_cast<const float4*>(P + static_cast<size_t>(min(j + 1, ny - 1)) * nz + 4 * c4));
    const float4 fjm = __ldg(reinterpret_cast<const float4*>(P + static_cast<size_t>(max(j - 1, 0)) * nz + 4 * c4));
    const float kl = c4 > 0 ? __ldg(P + jk - 1) : fc.x;
    const float kr = c4 + 1 < nz4 ? __ldg(P + jk + 4) : fc.w;
    const float4 o = cell4(c, fc, fip, fim, fjp, fjm, kl, kr);
    *reinterpret_cast<float4*>(fn + static_cast<size_t>(i) * plane + jk) = o;
  }
}

// Multi-step persistent variant for L2-resident grids (SURVEY.md §8f row 1:
// device-resident time loop): one cooperative launch runs nsteps steps with a
// grid-wide barrier between them, so a 128^3 step costs its L2 traffic, not a
// kernel launch. Ping-pongs a <-> b; same arithmetic as k_diffusion_direct.
__global__ void __launch_bounds__(256)
    k_diffusion_multi(float* a, float* b, int nx, int ny, int nz, int nsteps, Coefs c) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nz4 = nz >> 2;
  const size_t plane = static_cast<size_t>(ny) * nz;
  const size_t total = static_cast<size_t>(nx) * ny * nz4;
  for (int st = 0; st < nsteps; ++st) {
    const float* f = (st & 1) ? b : a;
    float* fn = (st & 1) ? a : b;
    for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<size_t>(gridDim.x) * blockDim.x) {
      const int c4 = static_cast<int>(t % nz4);
      const size_t r = t / nz4;
      const int j = static_cast<int>(r % ny);
      const int i = static_cast<int>(r / ny);
      const float* P = f + static_cast<size_t>(i) * plane;
      const float* Pm = i > 0 ? P - plane : P;
      const float* Pp = i < nx - 1 ? P + plane : P;
      const size_t jk = static_cast<size_t>(j) * nz + 4 * c4;
      // plain (coherent) loads: f was written by other CTAs earlier in this launch
      const float4 fc = *reinterpret_cast<const float4*>(P + jk);
      const float4 fip = *reinterpret_cast<const float4*>(Pp + jk);
      const float4 fim = *reinterpret_cast<const float4*>(Pm + jk);
      const float4 fjp = *reinterpret_cast<const float4*>(P + static_cast<size_t>(min(j + 1, ny - 1)) * nz + 4 * c4);
      const float4 fjm = *reinterpret_cast<const float4*>(P + static_cast<size_t>(max(j - 1, 0)) * nz + 4 * c4);
      const float kl = c4 > 0 ? P[jk - 1] : fc.x;
      const float kr = c4 + 1 < nz4 ? P[jk + 4] : fc.w;
      const float4 o = cell4(c, fc, fip, fim, fjp, fjm, kl, kr);
      *reinterpret_cast<float4*>(fn + static_cast<size_t>(i) * plane + jk) = o;
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// Host planning.
struct MarchPlan {
  int S = 0, TJ = 0, nst = 0, n_jtiles = 0, IC = 0, grid = 0;
  size_t smem = 0;
};


static bool plan_march(int nx_out, int ny, int nz, MarchPlan& mp) {
  if (nz % 4 != 0 || nz < 4) return false;
  const int nz4 = nz / 4;
  const DeviceInfo& di = device_info();
  static const int occ = std::max(1, env_int("SOLOMON_DIFF_OCC", 2));
  static const int max_nst = std::max(2, env_int("SOLOMON_DIFF_NST", 3));  // 3 beat 2 and 4 (round-1 sweep)
  static const int force_s = env_int("SOLOMON_DIFF_S", 0);
  static const int force_splits = env_int("SOLOMON_DIFF_SPLITS", 0);
  // Choose S (cells/thread/4) so the stages of `occ` CTAs fit one SM's shared memory.
  static const int kS[] = {4, 8, 2, 1};
  for (int S : kS) {
    if (force_s && S != force_s) continue;
    int TJ = (kMarchThreads * S) / nz4;
    if (TJ < 1) continue;
    TJ = std::min(TJ, ny);
    const size_t stage = static_cast<size_t>(TJ + 2) * nz * sizeof(float);
    const size_t budget = (228 * 1024) / occ - 1024 - 128;
    int nst = static_cast<int>(std::min<size_t>(max_nst, budget / stage));
    if (nst < 2) continue;
    mp.S = S;
    mp.TJ = TJ;
    mp.nst = nst;
    mp.smem = 128 + stage * nst;
    break;
  }
  if (!mp.S) return false;
  mp.n_jtiles = (ny + mp.TJ - 1) / mp.TJ;
  // Single co-resident wave when possible: split i so that n_jtiles * splits
  // fills the residency; neighbours then march in lock step and share halo
  // rows/planes through L2.
  const int resident = occ * di.sms;
  int splits = force_splits ? force_splits : std::max(1, resident / mp.n_jtiles);
  splits = std::min(splits, std::max(1, nx_out / 4));
  mp.IC = (nx_out + splits - 1) / splits;
  mp.grid = mp.n_jtiles * ((nx_out + mp.IC - 1) / mp.IC);
  return true;
}

static int launch_march(const MarchPlan& mp, int nx, int ny, int nz, const Coefs& c, const float* f, const float* lo,
                        const float* hi, float* fn, int i_begin, int i_end, cudaStream_t s) {
  MarchArgs a{f, lo, hi, fn, nx, ny, nz, mp.TJ, mp.n_jtiles, i_begin, i_end, mp.IC, mp.nst, c};
  switch (mp.S) {
#define B2_MARCH_CASE(SV)                                                       \
  case SV: {                                                                    \
    allow_max_dynamic_smem(reinterpret_cast<const void*>(k_diffusion_march<SV>)); \
    k_diffusion_march<SV><<<mp.grid, kMarchThreads, mp.smem, s>>>(a);           \
    break;                                                                      \
  }
    B2_MARCH_CASE(1)
    B2_MARCH_CASE(2)
    B2_MARCH_CASE(4)
    B2_MARCH_CASE(8)
#undef B2_MARCH_CASE
    default:
      return B2_EINVAL;
  }
  return launch_status();
}

// A plan with S cells per thread, `occ` CTAs per SM of shared memory and `splits` i-splits
// (0: fill one wave of occ x SMs).
static bool plan_march_with(int nx_out, int ny, int nz, int S, int occ, int splits_req, MarchPlan& mp) {
  if (nz % 4 != 0 || nz < 4) return false;
  const int nz4 = nz / 4;
  int TJ = std::min((kMarchThreads * S) / nz4, ny);
  if (TJ < 1) return false;
  static const int max_nst = std::max(2, env_int("SOLOMON_DIFF_NST", 3));
  const size_t stage = static_cast<size_t>(TJ + 2) * nz * sizeof(float);
  const int nst = static_cast<int>(std::min<size_t>(max_nst, ((228 * 1024) / occ - 1024 - 128) / stage));
  if (nst < 2) return false;
  mp = MarchPlan{};
  mp.S = S, mp.TJ = TJ, mp.nst = nst, mp.smem = 128 + stage * nst;
  mp.n_jtiles = (ny + TJ - 1) / TJ;
  int splits = splits_req ? splits_req : std::max(1, occ * device_info().sms / mp.n_jtiles);
  splits = std::min(splits, std::max(1, nx_out / 4));
  mp.IC = (nx_out + splits - 1) / splits;
  mp.grid = mp.n_jtiles * ((nx_out + mp.IC - 1) / mp.IC);
  return true;
}

// Tuned single-step plans, per (output planes, ny, nz, device). b2_diffusion3d_plan times
// the default plan and a few alternatives (2 or 4 cells per thread at the occupancy their
// launch bounds allow, a few i-split counts) on the caller's buffers (f read, fn's planes
// [i_begin, i_end) written) and keeps the fastest: rows whose width leaves the default
// wave under-filled (768 floats: 569 GLUPS) reach ~790. Same bits for every plan. The
// stream-ordered calls only look the plan up (no timing, no host synchronisation) and
// take the model's default for shapes nobody planned.
static std::mutex g_march_mu;
static std::map<std::tuple<int, int, int, int>, MarchPlan> g_march_cache;

static bool march_tuning_enabled() {
  static const bool tune = env_int("SOLOMON_DIFF_AUTOTUNE", 1) && !env_int("SOLOMON_DIFF_S", 0) &&
                           !env_int("SOLOMON_DIFF_SPLITS", 0) && !std::getenv("SOLOMON_DIFF_OCC");
  return tune;
}

static bool plan_march_lookup(int nx_out, int ny, int nz, MarchPlan& best) {
  if (!plan_march(nx_out, ny, nz, best)) return false;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_march_mu);
  auto it = g_march_cache.find(std::make_tuple(nx_out, ny, nz, dev));
  if (it != g_march_cache.end()) best = it->second;
  return true;
}

// Host-synchronising; skipped (model pick kept) under stream capture, for thin slabs,
// when a SOLOMON_DIFF_{S,SPLITS,OCC} knob forces a plan, or with SOLOMON_DIFF_AUTOTUNE=0.
static int plan_march_tune(int nx, int ny, int nz, const Coefs& c, const float* f, float* fn, int i_begin,
                           int i_end, cudaStream_t s) {
  const int nx_out = i_end - i_begin;
  MarchPlan best;
  if (!plan_march(nx_out, ny, nz, best) || !march_tuning_enabled() || nx_out < 8) return B2_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(nx_out, ny, nz, dev);
  {
    std::lock_guard<std::mutex> lk(g_march_mu);
    if (g_march_cache.count(key)) return B2_OK;
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return B2_OK;
  }
  std::vector<MarchPlan> cand{best};
  for (const int S : {2, 4}) {
    for (const int splits : {0, 2, 3, 4}) {
      MarchPlan q;
      if (!plan_march_with(nx_out, ny, nz, S, S <= 2 ? 4 : 2, splits, q)) continue;
      bool dup = false;
      for (const MarchPlan& p : cand) dup |= p.S == q.S && p.TJ == q.TJ && p.IC == q.IC && p.nst == q.nst;
      if (!dup) cand.push_back(q);
    }
  }
  cudaEvent_t ev[2];
  cudaError_t e;
  if ((e = cudaEventCreate(&ev[0])) != cudaSuccess) return static_cast<int>(e);
  if ((e = cudaEventCreate(&ev[1])) != cudaSuccess) {
    cudaEventDestroy(ev[0]);
    return static_cast<int>(e);
  }
  float best_ms = 1e30f;
  for (const MarchPlan& p : cand) {
    if (launch_march(p, nx, ny, nz, c, f, nullptr, nullptr, fn, i_begin, i_end, s)) continue;  // warm-up
    cudaEventRecord(ev[0], s);
    for (int r = 0; r < 2; ++r) launch_march(p, nx, ny, nz, c, f, nullptr, nullptr, fn, i_begin, i_end, s);
    cudaEventRecord(ev[1], s);
    float ms = 0.f;
    if (cudaEventSynchronize(ev[1]) != cudaSuccess || cudaEventElapsedTime(&ms, ev[0], ev[1]) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (ms < best_ms) {
      best_ms = ms;
      best = p;
    }
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  std::lock_guard<std::mutex> lk(g_march_mu);
  g_march_cache[key] = best;
  return launch_status();
}

static int launch_step(int nx, int ny, int nz, const Coefs& c, const float* f, const float* lo, const float* hi,
                       float* fn, int i_begin, int i_end, cudaStream_t s) {
  if (i_end <= i_begin) return B2_OK;
  MarchPlan mp;
  const bool ok_align = aligned16(f) && aligned16(fn) && (!lo || aligned16(lo)) && (!hi || aligned16(hi));
  // Grids whose two fields sit comfortably in L2 take the direct kernel.
  static const long long direct_max = env_int("SOLOMON_DIFF_DIRECT_MAXCELLS", 1 << 22);
  const long long cells = static_cast<long long>(i_end - i_begin) * ny * nz;
  // ...and so do thin boundary launches of a slab: their halo planes may live in
  // a peer GPU's memory (fused halo transport), read here with plain loads.
  const bool thin_halo = (i_end - i_begin) <= 2 && (lo || hi);
  if (ok_align && nz % 4 == 0 && (cells <= direct_max || thin_halo)) {
    const long long work = cells / 4;
    const int grid = static_cast<int>(std::min<long long>((work + 255) / 256, 148LL * 16));
    k_diffusion_direct<<<grid, 256, 0, s>>>(f, lo, hi, fn, nx, ny, nz, i_begin, i_end, c);
    return launch_status();
  }
  if (ok_align && plan_march_lookup(i_end - i_begin, ny, nz, mp))
    return launch_march(mp, nx, ny, nz, c, f, lo, hi, fn, i_begin, i_end, s);
  const size_t total = static_cast<size_t>(i_end - i_begin) * ny * nz;
  const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 64));
  k_diffusion_generic<<<grid, 256, 0, s>>>(f, lo, hi, fn, nx, ny, nz, i_begin, i_end, c);
  return launch_status();
}

static int check_grid(int nx, int ny, int nz, const float* f, const float* fn) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || !f || !fn) return B2_EINVAL;
  if (f == fn) return B2_EINVAL;  // restrict: listing_diffusion.c:5
  return B2_OK;
}

}  // namespace b2

using namespace b2;

extern "C" {

int b2_diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa, const float* f,
                   float* fn, void* stream) {
  if (int rc = check_grid(nx, ny, nz, f, fn)) return rc;
  return launch_step(nx, ny, nz, make_coefs(dx, dy, dz, dt, kappa), f, nullptr, nullptr, fn, 0, nx,
                     as_stream(stream));
}

int b2_diffusion3d_slab(int nx_local, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                        const float* f, const float* halo_lo, const float* halo_hi, float* fn, int i_begin, int i_end,
                        void* stream) {
  if (int rc = check_grid(nx_local, ny, nz, f, fn)) return rc;
  if (i_begin < 0 || i_end > nx_local || i_begin > i_end) return B2_EINVAL;
  return launch_step(nx_local, ny, nz, make_coefs(dx, dy, dz, dt, kappa), f, halo_lo, halo_hi, fn, i_begin, i_end,
                     as_stream(stream));
}

int b2_diffusion3d_plan(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa, const float* f,
                        float* fn, int nsteps, void* stream) {
  if (int rc = check_grid(nx, ny, nz, f, fn)) return rc;
  if (nsteps < 0) return B2_EINVAL;
  const Coefs c = make_coefs(dx, dy, dz, dt, kappa);
  cudaStream_t s = as_stream(stream);
  const bool aligned = nz % 4 == 0 && aligned16(f) && aligned16(fn);
  if (!aligned) return B2_OK;  // the generic kernel has no plan
  static const long long direct_max = env_int("SOLOMON_DIFF_DIRECT_MAXCELLS", 1 << 22);
  const long long cells = static_cast<long long>(nx) * ny * nz;
  int rc;
  if (cells > direct_max) {
    // whole-grid steps, and the interior planes [1, nx-1) of a slab (SlabDiffusion.step)
    if ((rc = plan_march_tune(nx, ny, nz, c, f, fn, 0, nx, s))) return rc;
    if (nx > 2 && (rc = plan_march_tune(nx, ny, nz, c, f, fn, 1, nx - 1, s))) return rc;
  }
  if (nsteps >= 2) {
    if ((rc = plan_resident(nx, ny, nz))) return rc;
    if (env_int("SOLOMON_DIFF_TEMPORAL", 1) && (rc = plan_tb2_tune(nx, ny, nz, c, f, fn, s))) return rc;
  }
  return B2_OK;
}

int b2_diffusion3d_run(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa, float* f,
                       float* fn, int nsteps, int* result_in_fn, void* stream) {
  if (int rc = check_grid(nx, ny, nz, f, fn)) return rc;
  if (nsteps < 0) return B2_EINVAL;
  const Coefs c = make_coefs(dx, dy, dz, dt, kappa);
  cudaStream_t s = as_stream(stream);
  if (result_in_fn) *result_in_fn = nsteps & 1;
  static const long long direct_max = env_int("SOLOMON_DIFF_DIRECT_MAXCELLS", 1 << 22);
  static const int use_multi = env_int("SOLOMON_DIFF_MULTI", 1);
  // Large grids: two steps per HBM pass (k_diffusion_tb2) where the planner finds a
  // tile shape worth it (512^3: 1235 vs 790 GLUPS effective);
  // SOLOMON_DIFF_TEMPORAL=0 forces one step per pass.
  static const int use_tb = env_int("SOLOMON_DIFF_TEMPORAL", 1);
  static const int use_resident = env_int("SOLOMON_DIFF_RESIDENT", 1);
  const long long cells = static_cast<long long>(nx) * ny * nz;
  const bool aligned = nz % 4 == 0 && aligned16(f) && aligned16(fn);
  if (use_resident && nsteps > 1 && aligned && launch_resident(nx, ny, nz, c, f, fn, nsteps, s)) return B2_OK;
  if (use_multi && nsteps > 1 && aligned && cells <= direct_max) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_diffusion_multi, 256, 0);
    const long long work = (cells / 4 + 255) / 256;
    const int grid = static_cast<int>(std::min<long long>(work, static_cast<long long>(per_sm) * device_info().sms));
    if (grid > 0) {
      int nxv = nx, nyv = ny, nzv = nz, ns = nsteps;
      Coefs cv = c;
      void* args[] = {&f, &fn, &nxv, &nyv, &nzv, &ns, &cv};
      cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_diffusion_multi), grid, 256, args,
                                                  0, s);
      if (e == cudaSuccess) return B2_OK;
      cudaGetLastError();  // fall through to per-step launches
    }
  }
  float* a = f;
  float* b = fn;
  int done = 0;
  TB2Plan tb;
  if (use_tb && nsteps >= 2 && aligned && plan_tb2_lookup(nx, ny, nz, tb)) {
    for (; done + 2 <= nsteps; done += 2) {
      if (int rc = launch_tb2(tb, nx, ny, nz, c, a, b, s)) return rc;
      std::swap(a, b);
    }
  }
  for (; done < nsteps; ++done) {
    if (int rc = launch_step(nx, ny, nz, c, a, nullptr, nullptr, b, 0, nx, s)) return rc;
    std::swap(a, b);
  }
  if (result_in_fn) *result_in_fn = a == fn;
  return B2_OK;
}

int b2_diffusion3d_run2_planes(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                               const float* f, float* fn, int p0, int p1, int p2, int p3, void* stream) {
  if (int rc = check_grid(nx, ny, nz, f, fn)) return rc;
  if (p0 < 0 || p1 > nx || p0 > p1 || p2 < 0 || p3 > nx || p2 > p3 || (p2 < p3 && p0 < p1 && p2 < p1 && p0 < p3))
    return B2_EINVAL;
  TB2Plan tb;
  if (nz % 4 != 0 || !aligned16(f) || !aligned16(fn) || !plan_tb2_lookup(nx, ny, nz, tb)) return B2_ENOTSUP;
  if (p0 == p1 && p2 == p3) return B2_OK;
  if (p0 == p1) std::swap(p0, p2), std::swap(p1, p3);
  return launch_tb2(tb, nx, ny, nz, make_coefs(dx, dy, dz, dt, kappa), f, fn, as_stream(stream), p0, p1, p2, p3);
}

}  // extern "C"

