// TEST INFRASTRUCTURE ONLY. Wraps the reference's own fallback-lowered listings
// (generated into oracle/_ref/ by oracle/build_ref.py; never committed) with the
// prelude they assume and C entry points for ctypes.
//
//   listing_nbody.c:1      void calc_acc(const int Ni, float4*, float4*, const int Nj, float4*, const float eps)
//   listing_nbody.c:21-23  #ifdef CALCULATE_POTENTIAL  -> built twice, with and without
//   listing_diffusion.c:5  void diffusion3d(int nx, ..., const float *restrict f, float *restrict fn)
#include <cmath>

struct float4 {
  float x, y, z, w;
};
#define restrict __restrict__

#define calc_acc ref_impl_calc_acc
#include "nbody_fallback.cpp"
#undef calc_acc

#define CALCULATE_POTENTIAL
#define calc_acc ref_impl_calc_acc_pot
#include "nbody_fallback.cpp"
#undef calc_acc
#undef CALCULATE_POTENTIAL

#include "diffusion_fallback.cpp"

extern "C" {
void ref_calc_acc(int Ni, float* ipos, float* iacc, int Nj, float* jpos, float eps, int potential) {
  float4* ip = reinterpret_cast<float4*>(ipos);
  float4* ia = reinterpret_cast<float4*>(iacc);
  float4* jp = reinterpret_cast<float4*>(jpos);
  if (potential)
    ref_impl_calc_acc_pot(Ni, ip, ia, Nj, jp, eps);
  else
    ref_impl_calc_acc(Ni, ip, ia, Nj, jp, eps);
}

void ref_diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                     const float* f, float* fn) {
  diffusion3d(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn);
}
}
