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
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace b2 {

struct Coefs {
  float cc, ce, cn, ct;
};

// listing_diffusion.c:6-9, evaluated in the same order as the reference build.
static Coefs make_coefs(float dx, float dy, float dz, float dt, float kappa) {
  volatile float kd = kappa * dt;  // volatile: keep every FP32 rounding on the host too
  volatile float ce = kd / (dx * dx);
  volatile float cn = kd / (dy * dy);
  volatile float ct = kd / (dz * dz);
  volatile float s = ce + ce;
  s = s + cn;
  s = s + cn;
  s = s + ct;
  s = s + ct;
  Coefs c;
  c.cc = 1.0f - s;
  c.ce = ce;
  c.cn = cn;
  c.ct = ct;
  return c;
}

__device__ __forceinline__ float cell(const Coefs& c, float fc, float fip, float fim, float fjp, float fjm, float fkp,
                                      float fkm) {
  float v = __fmul_rn(c.ce, fip);
  v = __fmaf_rn(c.cc, fc, v);
  v = __fmaf_rn(c.ce, fim, v);  // cw = ce
  v = __fmaf_rn(c.cn, fjp, v);
  v = __fmaf_rn(c.cn, fjm, v);  // cs = cn
  v = __fmaf_rn(c.ct, fkp, v);
  v = __fmaf_rn(c.ct, fkm, v);  // cb = ct
  return v;
}

// Four consecutive-k cells at once with packed FP32 (FFMA2/FMUL2: per-lane IEEE
// fma/mul, so identical to four cell() calls) -- halves the FP32 issue slots of
// the stencil arithmetic. kl = f[k0-1] (clamped), kr = f[k0+4] (clamped).
__device__ __forceinline__ float4 cell4(const Coefs& c, float4 fc, float4 fip, float4 fim, float4 fjp, float4 fjm,
                                        float kl, float kr) {
  const float2 ce = make_float2(c.ce, c.ce), cc = make_float2(c.cc, c.cc);
  const float2 cn = make_float2(c.cn, c.cn), ct = make_float2(c.ct, c.ct);
  float2 lo = __fmul2_rn(ce, make_float2(fip.x, fip.y));
  float2 hi = __fmul2_rn(ce, make_float2(fip.z, fip.w));
  lo = __ffma2_rn(cc, make_float2(fc.x, fc.y), lo);
  hi = __ffma2_rn(cc, make_float2(fc.z, fc.w), hi);
  lo = __ffma2_rn(ce, make_float2(fim.x, fim.y), lo);
  hi = __ffma2_rn(ce, make_float2(fim.z, fim.w), hi);
  lo = __ffma2_rn(cn, make_float2(fjp.x, fjp.y), lo);
  hi = __ffma2_rn(cn, make_float2(fjp.z, fjp.w), hi);
  lo = __ffma2_rn(cn, make_float2(fjm.x, fjm.y), lo);
  hi = __ffma2_rn(cn, make_float2(fjm.z, fjm.w), hi);
  lo = __ffma2_rn(ct, make_float2(fc.y, fc.z), lo);  // f[k+1]
  hi = __ffma2_rn(ct, make_float2(fc.w, kr), hi);
  lo = __ffma2_rn(ct, make_float2(kl, fc.x), lo);    // f[k-1]
  hi = __ffma2_rn(ct, make_float2(fc.y, fc.z), hi);
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// ---- PTX helpers: mbarrier + bulk async copy (sm_90+/sm_100a) -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }

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
// and the 14 packed-FP32 ops. f is read once and f'' written once: 8 B of HBM
// per two cell-updates. Arithmetic and clamps as two single steps: bit-identical.
struct TB2Args {
  const float* f;
  float* fn;
  int nx, ny, nz;
  int TJ, n_jtiles, IC, nst, ns1;
  int R, R1;  // rows per input-ring slot / per step-1 slot
  Coefs c;
};

constexpr int kTBWarps1 = 8, kTBWarps2 = 8;
constexpr int kTBThreads = 32 * (1 + kTBWarps1 + kTBWarps2);
constexpr int kTBStages = 4;  // input-ring and step-1-ring depth (powers of two: slot math is masks)
// Every compute thread arrives on the ring mbarriers itself (release of its own
// shared-memory accesses): measured as fast as one elected lane per warp after
// __syncwarp, and clean under compute-sanitizer racecheck.
constexpr int kTBArrive = 32;

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
  const int i0 = ic * a.IC, i1 = min(i0 + a.IC, nx);
  if (i0 >= i1) return;                                               // uniform per CTA
  const int qlo = max(i0 - 1, 0), qhi = min(i1, nx - 1);              // step-1 planes
  const int lo_in = max(qlo - 1, 0), hi_in = min(qhi + 1, nx - 1);    // input planes
  const int L = hi_in - lo_in + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int k = 0; k < NST; ++k) {
      mbar_init(full_in + k, 1);
      mbar_init(empty_in + k, kTBArrive * kTBWarps1);
    }
    for (int k = 0; k < NS1; ++k) {
      mbar_init(full_s1 + k, kTBArrive * kTBWarps1);
      mbar_init(empty_s1 + k, kTBArrive * kTBWarps2);
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
    for (int q = qlo; q <= qhi; ++q) {
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
        const float4 o = cell4(c, xc[k], xn, xp[k], fjp, fjm, kl, kr);
        float* dst = out + k * nz;
        if (real >> k & 1) *reinterpret_cast<float4*>(dst) = o;
        if (dup_up >> k & 1) *reinterpret_cast<float4*>(dst - nz) = o;
        if (dup_dn >> k & 1) *reinterpret_cast<float4*>(dst + nz) = o;
        xp[k] = xc[k];
        xc[k] = xn;
      }
      mbar_arrive(full_s1 + t1 % NS1);
      mbar_arrive(empty_in + (q - lo_in) % NST);
    }
    return;
  }

  // ---- step 2: output rows j0 + r2 (s1 row r2 + 1) ----
  const int tid = threadIdx.x - 32 * (1 + kTBWarps1);
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
      if (comp >> k & 1) st_stream(reinterpret_cast<float4*>(dst + k * nz), cell4(c, yb[k], yn, ya[k], fjp, fjm, kl, kr));
      ya[k] = yb[k];
      yb[k] = yn;
    }
    mbar_arrive(empty_s1 + (p - qlo) % NS1);
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
// step s+1's -- so two mailbox parities suffice. Same arithmetic and clamps as
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
        // A neighbour never arrived: fail loudly instead of hanging the GPU. (A poll
        // back-off of 64-1000 ns was measured slower: the lines are not contended.)
        if (todo && globaltimer_ns() - t0 > 4000000000ull) __trap();
      }
    }
    __syncthreads();
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

// ---------------------------------------------------------------------------
// Host planning.
struct MarchPlan {
  int S = 0, TJ = 0, nst = 0, n_jtiles = 0, IC = 0, grid = 0;
  size_t smem = 0;
};

static int env_int(const char* name, int dflt) {  // tuning knobs for bench sweeps
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

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

// Temporal-blocked (2 steps per pass) plan for k_diffusion_tb2: one CTA per SM
// (~170 KB of rings), TJ output rows per tile chosen so that j-tiles x i-splits
// fill the SMs in one wave while keeping the recomputed halo rows (2 of TJ+2)
// small; S1/S2 = float4 cells per step-1/step-2 thread must match an
// instantiation below.
struct TB2Plan {
  int TJ = 0, S1 = 0, S2 = 0, nst = kTBStages, ns1 = kTBStages, n_jtiles = 0, IC = 0, grid = 0, R = 0, R1 = 0;
  size_t smem = 0;
};

static bool tb2_instantiated(int S1, int S2) {
  return (S1 == 2 && (S2 == 1 || S2 == 2)) || (S1 == 3 && (S2 == 2 || S2 == 3)) ||
         (S1 == 4 && (S2 == 3 || S2 == 4)) || (S1 == 5 && (S2 == 3 || S2 == 4)) || (S1 == 6 && (S2 == 5 || S2 == 6));
}

static bool plan_tb2(int nx, int ny, int nz, TB2Plan& best) {
  if (nz % 4 != 0 || nx < 2) return false;
  const int nz4 = nz / 4;
  if ((32 * kTBWarps1) % nz4 != 0 || (32 * kTBWarps2) % nz4 != 0 || nz4 < 32) return false;  // row blocks, full warps
  const int blocks1 = 32 * kTBWarps1 / nz4, blocks2 = 32 * kTBWarps2 / nz4;
  const DeviceInfo& di = device_info();
  const size_t cap = static_cast<size_t>(di.smem_optin > 0 ? di.smem_optin : 227 * 1024);
  static const int force_tj = env_int("SOLOMON_DIFF_TB_TJ", 0);  // tuning knob (scripts/tb.sh sweeps)
  double best_score = -1.0;
  for (int TJ = 1; TJ <= std::min(ny, 32); ++TJ) {
    if (force_tj && TJ != force_tj) continue;
    TB2Plan p;
    p.TJ = TJ;
    p.S1 = (TJ + 2 + blocks1 - 1) / blocks1;
    p.S2 = (TJ + blocks2 - 1) / blocks2;
    if (!tb2_instantiated(p.S1, p.S2) || TJ < 5) continue;  // TJ < 5: recomputed halo rows cost more than they save
    p.R1 = std::max(blocks1 * p.S1, blocks2 * p.S2 + 2);  // step-1 rows written / read (one past the last)
    p.R = blocks1 * p.S1 + 2;                             // input rows read by step 1
    p.smem = 256 + (static_cast<size_t>(p.nst) * p.R + static_cast<size_t>(p.ns1) * p.R1) * nz * sizeof(float);
    if (p.smem > cap) continue;
    p.n_jtiles = (ny + TJ - 1) / TJ;
    const int splits = std::max(1, std::min(di.sms / p.n_jtiles, std::max(1, nx / 8)));
    p.IC = (nx + splits - 1) / splits;
    p.grid = p.n_jtiles * ((nx + p.IC - 1) / p.IC);
    const double waves = std::ceil(static_cast<double>(p.grid) / di.sms);
    const double util = p.grid / (waves * di.sms);
    const double score = util * TJ / (TJ + 2.0) * static_cast<double>(p.IC) / (p.IC + 2.0);
    if (score > best_score) {
      best_score = score;
      best = p;
    }
  }
  return best_score > 0;
}

template <int S1, int S2>
static void launch_tb2_t(const TB2Plan& p, const TB2Args& a, cudaStream_t s) {
  static bool set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!set[dev]) {  // per device: the opt-in is a per-context function attribute
    cudaFuncSetAttribute(k_diffusion_tb2<S1, S2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    set[dev] = true;
  }
  k_diffusion_tb2<S1, S2><<<p.grid, kTBThreads, p.smem, s>>>(a);
}

static int launch_tb2(const TB2Plan& p, int nx, int ny, int nz, const Coefs& c, const float* f, float* fn,
                      cudaStream_t s) {
  TB2Args a{f, fn, nx, ny, nz, p.TJ, p.n_jtiles, p.IC, p.nst, p.ns1, p.R, p.R1, c};
#define B2_TB2_CASE(A, B) \
  if (p.S1 == A && p.S2 == B) launch_tb2_t<A, B>(p, a, s); else
  B2_TB2_CASE(2, 1) B2_TB2_CASE(2, 2) B2_TB2_CASE(3, 2) B2_TB2_CASE(3, 3) B2_TB2_CASE(4, 3) B2_TB2_CASE(4, 4)
  B2_TB2_CASE(5, 3) B2_TB2_CASE(5, 4) B2_TB2_CASE(6, 5) B2_TB2_CASE(6, 6) return B2_EINVAL;
#undef B2_TB2_CASE
  return launch_status();
}

// Brick plan for k_diffusion_resident: at most one brick per SM, two copies of
// the brick plus its halo in one SM's shared memory, one float4 column per
// thread (BJ*nz/4 <= 512), at most kResidentUnits halo units per thread. Fewest
// planes per brick wins (each plane is one cell on every thread's march).
struct ResPlan {
  int BI = 0, BJ = 0, nbi = 0, nbj = 0;
  size_t smem = 0;
};

static bool plan_resident(int nx, int ny, int nz, ResPlan& p) {
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

// Per-device mailbox for k_diffusion_resident, grown on demand. Launches on one
// device are chained through an event (each waits for the previous one to
// finish with the mailbox), so concurrent runs on different streams stay safe.
struct Mailbox {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaEvent_t done = nullptr;
  bool used = false;
};

static bool launch_resident(int nx, int ny, int nz, const Coefs& c, float* f, float* fn, int nsteps,
                            cudaStream_t s) {
  ResPlan p;
  if (!plan_resident(nx, ny, nz, p)) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;  // the event chain below is not capturable; per-step path instead
  }
  const int nbricks = p.nbi * p.nbj;
  static std::mutex mu;
  static Mailbox boxes[64];
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!attr[dev]) {
    cudaFuncSetAttribute(k_diffusion_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr[dev] = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_diffusion_resident, kResidentThreads, p.smem) !=
          cudaSuccess ||
      per_sm * device_info().sms < nbricks) {
    cudaGetLastError();
    return false;
  }
  const int face_cap = std::max(p.BI, p.BJ) * ((nz + 2) / 3);
  const size_t bytes = static_cast<size_t>(nbricks) * 4 * 2 * face_cap * sizeof(uint4);
  Mailbox& mb = boxes[dev];
  if (!mb.done && cudaEventCreateWithFlags(&mb.done, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (mb.bytes < bytes) {
    if (mb.ptr) {
      cudaEventSynchronize(mb.done);
      cudaFree(mb.ptr);
    }
    mb.ptr = nullptr;
    mb.bytes = 0;
    if (cudaMalloc(&mb.ptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    mb.bytes = bytes;
  }
  if (mb.used) cudaStreamWaitEvent(s, mb.done, 0);
  cudaMemsetAsync(mb.ptr, 0, bytes, s);  // no stale tags
  ResArgs a{f, fn, nx, ny, nz, nsteps, p.BI, p.BJ, p.nbj, static_cast<uint4*>(mb.ptr), face_cap, c};
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
  if (ok_align && plan_march(i_end - i_begin, ny, nz, mp)) {
    MarchArgs a{f, lo, hi, fn, nx, ny, nz, mp.TJ, mp.n_jtiles, i_begin, i_end, mp.IC, mp.nst, c};
    switch (mp.S) {
#define B2_MARCH_CASE(SV)                                                                                     \
  case SV: {                                                                                                  \
    static bool attr_set[64] = {};                                                                            \
    int dev_ = 0;                                                                                             \
    cudaGetDevice(&dev_);                                                                                     \
    if (!attr_set[dev_]) {                                                                                    \
      cudaFuncSetAttribute(k_diffusion_march<SV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); \
      attr_set[dev_] = true;                                                                                  \
    }                                                                                                         \
    k_diffusion_march<SV><<<mp.grid, kMarchThreads, mp.smem, s>>>(a);                                         \
    break;                                                                                                    \
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
  if (use_tb && nsteps >= 2 && aligned && plan_tb2(nx, ny, nz, tb)) {
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

}  // extern "C"
