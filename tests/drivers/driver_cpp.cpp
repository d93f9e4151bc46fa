// A C++ caller written the way the paper's drivers call the listings
// (pkg/tests/fixtures/listing_nbody.c:1, listing_diffusion.c:5): its OWN
// `struct float4`, the reference call sites unchanged, linked against
// libsolomon_b200 instead of the transpiled listing.
//
//   driver_cpp IN OUT   -- IN: int32 N, nx, ny, nz; float eps, dx, dy, dz, dt, kappa;
//                          float4[N] pos; float[nx*ny*nz] f.
//                          OUT: float4[N] acc (calc_acc), float4[N] acc (calc_acc_exact),
//                          float4[N] acc+pot (calc_acc_potential), float[...] fn (diffusion3d).
// Exit 0 on success, 3 if the library reported an error (b2_last_error).
#include <cstdio>
#include <cstdlib>
#include <vector>

struct float4 {  // the listing's float4 (listing_nbody.c:4-5), not CUDA's
  float x, y, z, w;
};

#include "solomon_b200.h"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  FILE* in = std::fopen(argv[1], "rb");
  if (!in) return 2;
  int dims[4];
  float par[6];
  if (std::fread(dims, sizeof(int), 4, in) != 4 || std::fread(par, sizeof(float), 6, in) != 6) return 2;
  const int N = dims[0], nx = dims[1], ny = dims[2], nz = dims[3];
  const size_t cells = static_cast<size_t>(nx) * ny * nz;
  std::vector<float4> pos(N), acc(N), acc_exact(N), acc_pot(N);
  std::vector<float> f(cells), fn(cells);
  if (std::fread(pos.data(), sizeof(float4), N, in) != static_cast<size_t>(N) ||
      std::fread(f.data(), sizeof(float), cells, in) != cells)
    return 2;
  std::fclose(in);

  const float eps = par[0];
  calc_acc(N, pos.data(), acc.data(), N, pos.data(), eps);  // listing_nbody.c:1, unchanged
  int rc = b2_last_error();
  calc_acc_exact(N, pos.data(), acc_exact.data(), N, pos.data(), eps);
  rc = rc ? rc : b2_last_error();
  calc_acc_potential(N, pos.data(), acc_pot.data(), N, pos.data(), eps);  // -DCALCULATE_POTENTIAL
  rc = rc ? rc : b2_last_error();
  diffusion3d(nx, ny, nz, par[1], par[2], par[3], par[4], par[5], f.data(), fn.data());  // listing_diffusion.c:5
  rc = rc ? rc : b2_last_error();
  if (rc) {
    std::fprintf(stderr, "driver_cpp: %s\n", b2_error_string(rc));
    return 3;
  }
  FILE* out = std::fopen(argv[2], "wb");
  if (!out) return 2;
  std::fwrite(acc.data(), sizeof(float4), N, out);
  std::fwrite(acc_exact.data(), sizeof(float4), N, out);
  std::fwrite(acc_pot.data(), sizeof(float4), N, out);
  std::fwrite(fn.data(), sizeof(float), cells, out);
  std::fclose(out);
  return 0;
}
