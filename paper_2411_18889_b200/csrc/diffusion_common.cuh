// Shared pieces of the diffusion kernels: the reference arithmetic and coefficients
// (listing_diffusion.c:6-21), PTX helpers (mbarrier, bulk async copy), and the entry
// points the time-loop dispatcher in diffusion.cu calls into diffusion_tb2.cu and
// diffusion_resident.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace b2 {

struct Coefs {
  float cc, ce, cn, ct;
};

// listing_diffusion.c:6-9, evaluated in the same order as the reference build.
inline Coefs make_coefs(float dx, float dy, float dz, float dt, float kappa) {
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

// cell4 with the k-direction terms as scalar FMAs on the halves of the packed
// accumulators (same per-element operation order, so the same bits): the
// k-neighbour pairs (f.y, f.z), (f.w, kr), (kl, f.x) straddle register pairs and
// cost MOVs to build for FFMA2.
__device__ __forceinline__ float4 cell4k(const Coefs& c, float4 fc, float4 fip, float4 fim, float4 fjp, float4 fjm,
                                         float kl, float kr) {
  const float2 ce = make_float2(c.ce, c.ce), cc = make_float2(c.cc, c.cc);
  const float2 cn = make_float2(c.cn, c.cn);
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
  float4 o;
  o.x = __fmaf_rn(c.ct, kl, __fmaf_rn(c.ct, fc.y, lo.x));  // f[k+1] then f[k-1]
  o.y = __fmaf_rn(c.ct, fc.x, __fmaf_rn(c.ct, fc.z, lo.y));
  o.z = __fmaf_rn(c.ct, fc.y, __fmaf_rn(c.ct, fc.w, hi.x));
  o.w = __fmaf_rn(c.ct, fc.z, __fmaf_rn(c.ct, kr, hi.y));
  return o;
}

// PTX helpers (mbarrier, bulk async copy): common.cuh

__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }

inline int env_int(const char* name, int dflt) {  // tuning knobs for bench sweeps
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// ---- two steps per HBM pass (diffusion_tb2.cu) ----
constexpr int kTBStages = 4;  // input-ring and step-1-ring depth (powers of two: slot math is masks)
struct TB2Plan {
  int TJ = 0, S1 = 0, S2 = 0, nst = kTBStages, ns1 = kTBStages, n_jtiles = 0, IC = 0, grid = 0, R = 0, R1 = 0;
  size_t smem = 0;
};
bool plan_tb2(int nx, int ny, int nz, TB2Plan& best);
bool plan_tb2_lookup(int nx, int ny, int nz, TB2Plan& best);  // tuned plan if planned, else the model's pick
int plan_tb2_tune(int nx, int ny, int nz, const Coefs& c, const float* f, float* fn, cudaStream_t s);
// two steps; output planes [i_lo, i_hi) (default: all) and [i_lo2, i_hi2) of fn only,
// inputs clamped at 0 / nx-1
int launch_tb2(const TB2Plan& p, int nx, int ny, int nz, const Coefs& c, const float* f, float* fn, cudaStream_t s,
               int i_lo = 0, int i_hi = -1, int i_lo2 = 0, int i_hi2 = 0);

// ---- shared-memory-resident time loop (diffusion_resident.cu) ----
// Launches all nsteps for grids that fit the SMs' shared memory; false if not applicable
// or the device's mailbox was not sized for the shape by plan_resident (b2_diffusion3d_plan).
bool launch_resident(int nx, int ny, int nz, const Coefs& c, float* f, float* fn, int nsteps, cudaStream_t s);
int plan_resident(int nx, int ny, int nz);  // (re)allocates the mailbox; host-synchronising

}  // namespace b2
