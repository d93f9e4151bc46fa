// K3' -- two explicit diffusion steps per HBM pass (temporal blocking), for the
// device-resident time loop b2_diffusion3d_run on large grids. Reference arithmetic:
// pkg/tests/fixtures/listing_diffusion.c:5-25 via cell4 (diffusion_common.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "diffusion_common.cuh"

namespace b2 {

// ---------------------------------------------------------------------------
// Two steps per HBM pass (temporal blocking) for the device-resident time loop
// (b2_diffusion3d_run), warp-specialised. A CTA owns output rows [j0, j0+TJ)
// of step 2 over planes [i0, i1) and marches along i as a three-role pipeline
// coupled only by mbarriers (no CTA-wide barrier in the loop):
//
//   producer warp  -- cp.async.bulk of input rows j0-2 .. j0-2+R-1 of each plane
//                     into an NST-deep ring (full/empty mbarriers). Rows outside
//                     the grid are filled with copies of the edge row, so the
//                     j clamp of listing_diffusion.c:17-18 is in the data;
//   step-1 warps   -- step 1 on rows j0-1 .. (one row each side recomputed, as
//                     the neighbour tile does) into an NS1-deep ring of step-1
//                     planes; the edge rows are also stored into the row just
//                     outside the grid (the clamp for step 2);
//   step-2 warps   -- step 2 on rows [j0, j0+TJ) from the step-1 ring, one plane
//                     behind, streamed to fn with evict-first stores.
//
// Each compute thread owns one float4 column and S consecutive rows, with the
// i-1 / i values in registers: the in-plane j neighbours are its own registers
// except at its block ends, so a cell costs one LDS.128 (i+1), two LDS.32 (k+-1)
// and the stencil FMAs (cell4k). f is read once and f'' written once: 8 B of HBM
// per two cell-updates. Arithmetic and clamps as two single steps: bit-identical.
struct TB2Args {
  const float* f;
  float* fn;
  int nx, ny, nz;
  int TJ, n_jtiles, IC, nst, ns1;
  int R, R1;  // rows per input-ring slot / per step-1 slot
  int i_lo, i_hi;  // output planes [i_lo, i_hi): the whole grid, or a slab's interior / edges
  int i_lo2, i_hi2, splits1;  // i-splits >= splits1 cover a second range (a slab's two edges, one launch)
  Coefs c;
};

constexpr int kTBWarps1 = 8, kTBWarps2 = 8;
constexpr int kTBThreads = 32 * (1 + kTBWarps1 + kTBWarps2);
// Every active compute thread arrives on the ring mbarriers itself (release of its own
// shared-memory accesses): measured as fast as one elected lane per warp after
// __syncwarp, and clean under compute-sanitizer racecheck.

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int S1, int S2>
__global__ void __launch_bounds__(kTBThreads, 1) k_diffusion_tb2(const TB2Args a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nz = a.nz, nz4 = nz >> 2, ny = a.ny, nx = a.nx;
  const int TJ = a.TJ;
  constexpr int NST = kTBStages, NS1 = kTBStages;
  const size_t plane = static_cast<size_t>(ny) * nz;
  const int in_floats = a.R * nz;   // ring row r <-> global row j0 - 2 + r
  const int s1_floats = a.R1 * nz;  // s1 row r <-> global row j0 - 1 + r

  uint64_t* full_in = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty_in = full_in + NST;
  uint64_t* full_s1 = empty_in + NST;
  uint64_t* empty_s1 = full_s1 + NS1;
  float* in_ring = reinterpret_cast<float*>(smem_raw + 256);
  float* s1_ring = in_ring + static_cast<size_t>(NST) * in_floats;

  const int jt = blockIdx.x % a.n_jtiles, ic = blockIdx.x / a.n_jtiles;
  const int j0 = jt * TJ, rows = min(TJ, ny - j0);
  const bool second = ic >= a.splits1;
  const int i0 = second ? a.i_lo2 + (ic - a.splits1) * a.IC : a.i_lo + ic * a.IC;
  const int i1 = min(i0 + a.IC, second ? a.i_hi2 : a.i_hi);
  if (i0 >= i1) return;                                               // uniform per CTA
  const int qlo = max(i0 - 1, 0), qhi = min(i1, nx - 1);              // step-1 planes
  const int lo_in = max(qlo - 1, 0), hi_in = min(qhi + 1, nx - 1);    // input planes
  const int L = hi_in - lo_in + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // active threads per compute role: whole row blocks of nz4 threads (nz4 % 32 == 0)
  const int act1 = (32 * kTBWarps1 / nz4) * nz4, act2 = (32 * kTBWarps2 / nz4) * nz4;

  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) {
      mbar_init(full_in + k, 1);
      mbar_init(empty_in + k, act1);
    }
    for (int k = 0; k < NS1; ++k) {
      mbar_init(full_s1 + k, act1);
      mbar_init(empty_s1 + k, act2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // ---- producer ----
    if (lane == 0) {
      const int R = a.R;
      const int gfirst = max(j0 - 2, 0), glast = min(j0 - 2 + R - 1, ny - 1);
      const uint32_t row_bytes = static_cast<uint32_t>(nz * sizeof(float));
      const uint32_t main_bytes = static_cast<uint32_t>(glast - gfirst + 1) * row_bytes;
      const int n_top = gfirst - (j0 - 2), n_bot = (j0 - 2 + R - 1) - glast;  // rows outside the grid
      const uint32_t bytes = main_bytes + static_cast<uint32_t>(n_top + n_bot) * row_bytes;
      for (int t = 0; t < L; ++t) {
        const int st = t % NST;
        if (t >= NST) mbar_wait(empty_in + st, ((t / NST) - 1) & 1);
        fence_proxy_async();  // generic reads of the slot before the async-proxy refill
        mbar_expect_tx(full_in + st, bytes);
        float* slot = in_ring + static_cast<size_t>(st) * in_floats;
        const float* src = a.f + static_cast<size_t>(lo_in + t) * plane;
        bulk_g2s(slot + n_top * nz, src + static_cast<size_t>(gfirst) * nz, main_bytes, full_in + st);
        for (int r = 0; r < n_top; ++r) bulk_g2s(slot + r * nz, src, row_bytes, full_in + st);  // IMAX(j-1, 0)
        for (int r = 0; r < n_bot; ++r)                                                         // IMIN(j+1, ny-1)
          bulk_g2s(slot + (R - 1 - r) * nz, src + static_cast<size_t>(ny - 1) * nz, row_bytes, full_in + st);
      }
    }
    return;
  }

  const Coefs c = a.c;
  auto s1_slot = [&](int q) { return s1_ring + static_cast<size_t>((q - qlo) % NS1) * s1_floats; };
  auto wait_s1 = [&](int q) { const int t = q - qlo; mbar_wait(full_s1 + t % NS1, (t / NS1) & 1); };

  if (warp <= kTBWarps1) {  // ---- step 1: s1 rows r = 0 .. <-> global j0-1+r (ring row r+1) ----
    const int tid = threadIdx.x - 32;
    if (tid >= act1) return;  // whole idle warps when 256 is not a multiple of the row width
    auto in_slot = [&](int pl) { return in_ring + static_cast<size_t>((pl - lo_in) % NST) * in_floats; };
    auto wait_in = [&](int pl) { const int t = pl - lo_in; mbar_wait(full_in + t % NST, (t / NST) & 1); };
    const int c4 = tid % nz4, r0 = (tid / nz4) * S1;
    const bool kfirst = c4 == 0, klast = c4 + 1 == nz4;
    unsigned int real = 0, dup_up = 0, dup_dn = 0;  // bit k: row inside the grid / also store at row-1 / row+1
#pragma unroll
    for (int k = 0; k < S1; ++k) {
      const int g = j0 - 1 + r0 + k;
      if (g >= 0 && g < ny) real |= 1u << k;
      if (g == 0 && r0 + k >= 1) dup_up |= 1u << k;               // s1 row for g = -1 := s1(g = 0)
      if (g == ny - 1 && r0 + k + 1 < a.R1) dup_dn |= 1u << k;    // s1 row for g = ny := s1(g = ny-1)
    }
    const int base = (r0 + 1) * nz + 4 * c4;  // ring offset of row r0; s1 offset of row r0 is base - nz
    float4 xp[S1], xc[S1];
    if (qlo > 0) {
      wait_in(qlo - 1);
      const float* b = in_slot(qlo - 1) + base;
#pragma unroll
      for (int k = 0; k < S1; ++k) xp[k] = *reinterpret_cast<const float4*>(b + k * nz);
    }
    wait_in(qlo);
    {
      const float* b = in_slot(qlo) + base;
#pragma unroll
      for (int k = 0; k < S1; ++k) {
        xc[k] = *reinterpret_cast<const float4*>(b + k * nz);
        if (qlo == 0) xp[k] = xc[k];  // IMAX(i-1, 0)
      }
    }
    if (qlo > 0) mbar_arrive(empty_in + (qlo - 1 - lo_in) % NST);
    // One step-1 plane; EDGE: this thread's rows include rows outside the grid or edge
    // duplicates to store (tiles at j = 0 / ny-1 only) -- interior threads take the
    // unpredicated copy (+4% at 512^3).
    auto plane1 = [&](auto edge_tag, int q) {
      constexpr bool EDGE = decltype(edge_tag)::value;
      const bool has_next = q + 1 <= nx - 1;
      if (has_next) wait_in(q + 1);
      const int t1 = q - qlo;
      if (t1 >= NS1) mbar_wait(empty_s1 + t1 % NS1, ((t1 / NS1) - 1) & 1);
      const float* __restrict__ cur = in_slot(q) + base;
      const float* __restrict__ nxt = has_next ? in_slot(q + 1) + base : cur;  // IMIN(i+1, nx-1)
      float* __restrict__ out = s1_slot(q) + base - nz;
#pragma unroll
      for (int k = 0; k < S1; ++k) {
        const float* rowp = cur + k * nz;
        const float4 xn = *reinterpret_cast<const float4*>(nxt + k * nz);
        const float4 fjp = k + 1 < S1 ? xc[k + 1] : *reinterpret_cast<const float4*>(rowp + nz);
        const float4 fjm = k > 0 ? xp[k - 1] : *reinterpret_cast<const float4*>(rowp - nz);  // xp[k-1]: old xc[k-1]
        const float kl = kfirst ? xc[k].x : rowp[-1];  // IMAX(k-1, 0)
        const float kr = klast ? xc[k].w : rowp[4];    // IMIN(k+1, nz-1)
        const float4 o = cell4k(c, xc[k], xn, xp[k], fjp, fjm, kl, kr);
        float* dst = out + k * nz;
        if (!EDGE || (real >> k & 1)) *reinterpret_cast<float4*>(dst) = o;
        if (EDGE && (dup_up >> k & 1)) *reinterpret_cast<float4*>(dst - nz) = o;
        if (EDGE && (dup_dn >> k & 1)) *reinterpret_cast<float4*>(dst + nz) = o;
        xp[k] = xc[k];
        xc[k] = xn;
      }
      mbar_arrive(full_s1 + t1 % NS1);
      mbar_arrive(empty_in + (q - lo_in) % NST);
    };
    // warp-uniform (a warp is one row block): rows outside the grid or edge duplicates
    const bool edge = real != (1u << S1) - 1 || dup_up || dup_dn;
    if (edge) {
      for (int q = qlo; q <= qhi; ++q) plane1(std::true_type{}, q);
    } else {
      for (int q = qlo; q <= qhi; ++q) plane1(std::false_type{}, q);
    }
    return;
  }

  // ---- step 2: output rows j0 + r2 (s1 row r2 + 1) ----
  const int tid = threadIdx.x - 32 * (1 + kTBWarps1);
  if (tid >= act2) return;
  const int c4 = tid % nz4, r0 = (tid / nz4) * S2;
  const bool kfirst = c4 == 0, klast = c4 + 1 == nz4;
  unsigned int comp = 0;
#pragma unroll
  for (int k = 0; k < S2; ++k)
    if (r0 + k < rows) comp |= 1u << k;
  const int base = (r0 + 1) * nz + 4 * c4;  // s1 offset of row r0
  float4 ya[S2], yb[S2];
  if (i0 > 0) {
    wait_s1(i0 - 1);
    const float* b = s1_slot(i0 - 1) + base;
#pragma unroll
    for (int k = 0; k < S2; ++k) ya[k] = *reinterpret_cast<const float4*>(b + k * nz);
  }
  wait_s1(i0);
  {
    const float* b = s1_slot(i0) + base;
#pragma unroll
    for (int k = 0; k < S2; ++k) {
      yb[k] = *reinterpret_cast<const float4*>(b + k * nz);
      if (i0 == 0) ya[k] = yb[k];  // IMAX(i-1, 0) on step-1 values
    }
  }
  if (i0 > 0) {
    mbar_arrive(empty_s1 + (i0 - 1 - qlo) % NS1);
  }
  for (int p = i0; p < i1; ++p) {
    const bool has_next = p + 1 <= nx - 1;
    if (has_next) wait_s1(p + 1);
    const float* __restrict__ cur = s1_slot(p) + base;
    const float* __restrict__ nxt = has_next ? s1_slot(p + 1) + base : cur;  // IMIN(i+1, nx-1)
    // output row g = j0 + r0 + k = j0 - 1 + (s1 row): fn offset = s1 offset + (j0 - 1) * nz
    float* dst = a.fn + static_cast<ptrdiff_t>(p) * static_cast<ptrdiff_t>(plane) +
                 static_cast<ptrdiff_t>(j0 - 1) * nz + base;
#pragma unroll
    for (int k = 0; k < S2; ++k) {
      const float* rowp = cur + k * nz;
      const float4 yn = *reinterpret_cast<const float4*>(nxt + k * nz);
      const float4 fjp = k + 1 < S2 ? yb[k + 1] : *reinterpret_cast<const float4*>(rowp + nz);
      const float4 fjm = k > 0 ? ya[k - 1] : *reinterpret_cast<const float4*>(rowp - nz);  // ya[k-1]: old yb[k-1]
      const float kl = kfirst ? yb[k].x : rowp[-1];
      const float kr = klast ? yb[k].w : rowp[4];
      if (comp >> k & 1) st_stream(reinterpret_cast<float4*>(dst + k * nz), cell4k(c, yb[k], yn, ya[k], fjp, fjm, kl, kr));
      ya[k] = yb[k];
      yb[k] = yn;
    }
    mbar_arrive(empty_s1 + (p - qlo) % NS1);
  }
}

// Temporal-blocked (2 steps per pass) plan for k_diffusion_tb2: one CTA per SM
// (~170 KB of rings), TJ output rows per tile chosen so that j-tiles x i-splits
// fill the SMs in one wave while keeping the recomputed halo rows (2 of TJ+2)
// small; S1/S2 = float4 cells per step-1/step-2 thread must match an
// instantiation below.

static bool tb2_instantiated(int S1, int S2) {
  return (S1 == 2 && (S2 == 1 || S2 == 2)) || (S1 == 3 && (S2 == 2 || S2 == 3)) ||
         (S1 == 4 && (S2 == 3 || S2 == 4)) || (S1 == 5 && (S2 == 3 || S2 == 4)) ||
         (S1 == 6 && (S2 == 4 || S2 == 5 || S2 == 6));
}

// Every admissible (tile height, i-split) plan with its model score, best first.
static std::vector<std::pair<double, TB2Plan>> tb2_candidates(int nx, int ny, int nz) {
  std::vector<std::pair<double, TB2Plan>> out;
  if (nz % 4 != 0 || nx < 2) return out;
  const int nz4 = nz / 4;
  // whole warps per row (a warp never spans two row blocks); rows wider than a role's threads
  // do not fit, and threads past the last full row block idle
  if (nz4 % 32 != 0 || nz4 > 32 * kTBWarps1 || nz4 > 32 * kTBWarps2) return out;
  const int blocks1 = 32 * kTBWarps1 / nz4, blocks2 = 32 * kTBWarps2 / nz4;
  const DeviceInfo& di = device_info();
  const size_t cap = static_cast<size_t>(di.smem_optin > 0 ? di.smem_optin : 227 * 1024);
  static const int force_tj = env_int("SOLOMON_DIFF_TB_TJ", 0);  // tuning knob (scripts/tb.sh sweeps)
  for (int TJ = 1; TJ <= std::min(ny, 32); ++TJ) {
    if (force_tj && TJ != force_tj) continue;
    TB2Plan p;
    p.TJ = TJ;
    p.S1 = (TJ + 2 + blocks1 - 1) / blocks1;
    p.S2 = (TJ + blocks2 - 1) / blocks2;
    // TJ < 5 recomputes too many halo rows -- except where one row block spans the row
    // (rows of 768-1024 floats: 6 step-1 rows per thread) and TJ = 4 is the tallest tile.
    if (!tb2_instantiated(p.S1, p.S2) || TJ < (force_tj ? 1 : blocks1 == 1 ? 4 : 5)) continue;
    p.R1 = std::max(blocks1 * p.S1, blocks2 * p.S2 + 2);  // step-1 rows written / read (one past the last)
    p.R = blocks1 * p.S1 + 2;                             // input rows read by step 1
    p.smem = 256 + (static_cast<size_t>(p.nst) * p.R + static_cast<size_t>(p.ns1) * p.R1) * nz * sizeof(float);
    if (p.smem > cap) continue;
    p.n_jtiles = (ny + TJ - 1) / TJ;
    // i-splits: enough CTAs to fill the SMs, and a split count that avoids a ragged last wave
    // (each split re-reads 2 planes and recomputes 2 step-1 planes).
    const int max_splits = std::max(1, std::min(16, nx / 8));
    static const int force_splits = env_int("SOLOMON_DIFF_TB_SPLITS", 0);  // tuning knob
    for (int splits = 1; splits <= max_splits; ++splits) {
      if (force_splits && splits != force_splits) continue;
      TB2Plan q = p;
      q.IC = (nx + splits - 1) / splits;
      q.grid = q.n_jtiles * ((nx + q.IC - 1) / q.IC);
      const double waves = std::ceil(static_cast<double>(q.grid) / di.sms);
      const double util = q.grid / (waves * di.sms);
      const double score = util * TJ / (TJ + 2.0) * static_cast<double>(q.IC) / (q.IC + 2.0);
      out.emplace_back(score, q);
    }
  }
  // best score first; ties keep the smaller tile / fewer splits (enumeration order)
  std::stable_sort(out.begin(), out.end(),
                   [](const std::pair<double, TB2Plan>& x, const std::pair<double, TB2Plan>& y) {
                     return x.first > y.first + 1e-9;
                   });
  return out;
}

static void tb2_report(const char* what, int nx, int ny, int nz, const TB2Plan& p, double v) {
  static const bool verbose = env_int("SOLOMON_DIFF_TB_VERBOSE", 0) != 0;
  if (verbose)
    std::fprintf(stderr, "tb2 plan %dx%dx%d: TJ=%d S=%d,%d IC=%d grid=%d smem=%zu %s=%.4f\n", nx, ny, nz, p.TJ, p.S1,
                 p.S2, p.IC, p.grid, p.smem, what, v);
}

bool plan_tb2(int nx, int ny, int nz, TB2Plan& best) {
  const auto c = tb2_candidates(nx, ny, nz);
  if (c.empty()) return false;
  best = c.front().second;
  tb2_report("score", nx, ny, nz, best, c.front().first);
  return true;
}

// Tuned plans per (nx, ny, nz, device). b2_diffusion3d_plan times the model's best few
// plans on the caller's own buffers (f read, fn written: fn is scratch until the run
// writes it) and keeps the fastest. Every plan gives the same bits, so the choice only
// moves time. The stream-ordered run only looks the plan up (no timing, no host
// synchronisation) and takes the model's pick for shapes nobody planned.
static std::mutex g_tb2_mu;
static std::map<std::tuple<int, int, int, int>, TB2Plan> g_tb2_cache;

bool plan_tb2_lookup(int nx, int ny, int nz, TB2Plan& best) {
  if (!plan_tb2(nx, ny, nz, best)) return false;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_tb2_mu);
  auto it = g_tb2_cache.find(std::make_tuple(nx, ny, nz, dev));
  if (it != g_tb2_cache.end()) best = it->second;
  return true;
}

// Host-synchronising, hence skipped while the stream is being captured;
// SOLOMON_DIFF_AUTOTUNE=0 keeps the model's pick.
int plan_tb2_tune(int nx, int ny, int nz, const Coefs& c, const float* f, float* fn, cudaStream_t s) {
  static const int autotune = env_int("SOLOMON_DIFF_AUTOTUNE", 1);
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(nx, ny, nz, dev);
  {
    std::lock_guard<std::mutex> lk(g_tb2_mu);
    if (g_tb2_cache.count(key)) return B2_OK;
  }
  const auto cand = tb2_candidates(nx, ny, nz);
  if (cand.empty()) return B2_OK;
  TB2Plan best = cand.front().second;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!autotune || cand.size() == 1 || cudaStreamIsCapturing(s, &cap) != cudaSuccess ||
      cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return B2_OK;  // model pick, not cached: a later uncaptured plan call may still tune
  }
  // the model's best few plans, each timed in three interleaved rounds (two launches after a
  // warm-up), the minimum per plan kept: a single round was within the noise between plans
  constexpr int kCandidates = 4, kRounds = 3;
  cudaEvent_t ev[2];
  cudaError_t e;
  if ((e = cudaEventCreate(&ev[0])) != cudaSuccess) return static_cast<int>(e);
  if ((e = cudaEventCreate(&ev[1])) != cudaSuccess) {
    cudaEventDestroy(ev[0]);
    return static_cast<int>(e);
  }
  const size_t nc = std::min(cand.size(), static_cast<size_t>(kCandidates));
  std::vector<float> tmin(nc, 1e30f);
  for (int round = 0; round < kRounds; ++round) {
    for (size_t i = 0; i < nc; ++i) {
      const TB2Plan& p = cand[i].second;
      if (launch_tb2(p, nx, ny, nz, c, f, fn, s)) continue;  // warm-up (smem opt-in, caches)
      cudaEventRecord(ev[0], s);
      for (int r = 0; r < 2; ++r) launch_tb2(p, nx, ny, nz, c, f, fn, s);
      cudaEventRecord(ev[1], s);
      float ms = 0.f;
      if (cudaEventSynchronize(ev[1]) != cudaSuccess || cudaEventElapsedTime(&ms, ev[0], ev[1]) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      tmin[i] = std::min(tmin[i], ms / 2);
    }
  }
  float best_ms = 1e30f;
  for (size_t i = 0; i < nc; ++i) {
    tb2_report("ms", nx, ny, nz, cand[i].second, tmin[i]);
    if (tmin[i] < best_ms) {
      best_ms = tmin[i];
      best = cand[i].second;
    }
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  std::lock_guard<std::mutex> lk(g_tb2_mu);
  g_tb2_cache[key] = best;
  return launch_status();
}

template <int S1, int S2>
static void launch_tb2_t(const TB2Plan& p, const TB2Args& a, cudaStream_t s) {
  allow_max_dynamic_smem(reinterpret_cast<const void*>(k_diffusion_tb2<S1, S2>));
  k_diffusion_tb2<S1, S2><<<p.grid, kTBThreads, p.smem, s>>>(a);
}

int launch_tb2(const TB2Plan& p, int nx, int ny, int nz, const Coefs& c, const float* f, float* fn,
                      cudaStream_t s, int i_lo, int i_hi, int i_lo2, int i_hi2) {
  if (i_hi < 0) i_hi = nx;
  TB2Plan q = p;
  int splits1 = (nx + p.IC - 1) / p.IC;
  if (i_lo != 0 || i_hi != nx || i_hi2 > i_lo2) {  // plane ranges: the plan's i-split length, re-spread
    const int len = i_hi - i_lo, len2 = std::max(i_hi2 - i_lo2, 0);
    const int longest = std::max(len, len2);
    if (longest <= 0) return B2_OK;
    const int splits = (longest + p.IC - 1) / p.IC;
    q.IC = (longest + splits - 1) / splits;
    splits1 = len > 0 ? (len + q.IC - 1) / q.IC : 0;
    q.grid = q.n_jtiles * (splits1 + (len2 + q.IC - 1) / q.IC);
  }
  TB2Args a{f, fn, nx, ny, nz, q.TJ, q.n_jtiles, q.IC, q.nst, q.ns1, q.R, q.R1, i_lo, i_hi, i_lo2, i_hi2, splits1, c};
#define B2_TB2_CASE(A, B) \
  if (q.S1 == A && q.S2 == B) launch_tb2_t<A, B>(q, a, s); else
  B2_TB2_CASE(2, 1) B2_TB2_CASE(2, 2) B2_TB2_CASE(3, 2) B2_TB2_CASE(3, 3) B2_TB2_CASE(4, 3) B2_TB2_CASE(4, 4)
  B2_TB2_CASE(5, 3) B2_TB2_CASE(5, 4) B2_TB2_CASE(6, 4) B2_TB2_CASE(6, 5) B2_TB2_CASE(6, 6) return B2_EINVAL;
#undef B2_TB2_CASE
  return launch_status();
}

}  // namespace b2
