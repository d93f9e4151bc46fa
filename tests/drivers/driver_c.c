/* The same driver in C99: the caller's own float4 typedef is made the header's
 * parameter type with SOLOMON_FLOAT4_TYPE, so the listing's call sites
 * (listing_nbody.c:1, listing_diffusion.c:5) compile unchanged and warning-free.
 * Same file formats and exit codes as driver_cpp.cpp. */
#include <stdio.h>
#include <stdlib.h>

typedef struct {
  float x, y, z, w;
} float4;
#define SOLOMON_FLOAT4_TYPE float4
#include "solomon_b200.h"

int main(int argc, char **argv) {
  if (argc != 3) return 2;
  FILE *in = fopen(argv[1], "rb");
  if (!in) return 2;
  int dims[4];
  float par[6];
  if (fread(dims, sizeof(int), 4, in) != 4 || fread(par, sizeof(float), 6, in) != 6) return 2;
  const int N = dims[0], nx = dims[1], ny = dims[2], nz = dims[3];
  const size_t cells = (size_t)nx * ny * nz;
  float4 *pos = malloc(sizeof(float4) * N), *acc = malloc(sizeof(float4) * N);
  float4 *acc_exact = malloc(sizeof(float4) * N), *acc_pot = malloc(sizeof(float4) * N);
  float *f = malloc(sizeof(float) * cells), *fn = malloc(sizeof(float) * cells);
  if (fread(pos, sizeof(float4), N, in) != (size_t)N || fread(f, sizeof(float), cells, in) != cells) return 2;
  fclose(in);

  const float eps = par[0];
  int rc;
  calc_acc(N, pos, acc, N, pos, eps);
  rc = b2_last_error();
  calc_acc_exact(N, pos, acc_exact, N, pos, eps);
  rc = rc ? rc : b2_last_error();
  calc_acc_potential(N, pos, acc_pot, N, pos, eps);
  rc = rc ? rc : b2_last_error();
  diffusion3d(nx, ny, nz, par[1], par[2], par[3], par[4], par[5], f, fn);
  rc = rc ? rc : b2_last_error();
  if (rc) {
    fprintf(stderr, "driver_c: %s\n", b2_error_string(rc));
    return 3;
  }
  FILE *out = fopen(argv[2], "wb");
  if (!out) return 2;
  fwrite(acc, sizeof(float4), N, out);
  fwrite(acc_exact, sizeof(float4), N, out);
  fwrite(acc_pot, sizeof(float4), N, out);
  fwrite(fn, sizeof(float), cells, out);
  fclose(out);
  free(pos), free(acc), free(acc_exact), free(acc_pot), free(f), free(fn);
  return 0;
}
