// Drop-in layer: the reference's exact C signatures on top of the b2_* API.
//
//   calc_acc     -- pkg/tests/fixtures/listing_nbody.c:1
//   diffusion3d  -- pkg/tests/fixtures/listing_diffusion.c:5
//
// The reference functions are synchronous and take whatever pointers the
// backend implies: host memory under the fallback (host OpenMP) lowering,
// device-present memory under OpenACC `present(f, fn)` (listing_diffusion.c:10,
// conformance.rows:756). These entry points accept both: device/managed
// pointers are used in place; host pointers are staged through a cached
// device buffer. Either way the call returns when the result is in the
// caller's buffer. Errors (the reference has none -- bad sizes are UB there)
// are reported on stderr and through b2_last_error().
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace b2 {

static thread_local int g_last_error = B2_OK;

// Per-device staging arena for host-pointer calls (grown on demand, never shrunk),
// one lock per device: concurrent drop-in calls on different GPUs do not serialise.
// The arena stream is a BLOCKING stream: it is ordered after work the caller queued
// on the legacy default stream (torch's default stream) and vice versa, like the
// reference's synchronous present(f, fn) call (listing_diffusion.c:10).
struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
};

constexpr int kMaxDev = 64;
static std::mutex g_arena_mu[kMaxDev];
static Arena g_arena[kMaxDev];

static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// 0 on success, else the cudaError_t of the failed stream creation / allocation.
static int arena_get(int dev, size_t bytes, void** out, cudaStream_t* s) {
  Arena& a = g_arena[dev];
  cudaError_t e;
  if (!a.stream && (e = cudaStreamCreateWithFlags(&a.stream, cudaStreamDefault)) != cudaSuccess) {
    a.stream = nullptr;
    return static_cast<int>(e);
  }
  if (a.bytes < bytes) {
    if (a.ptr) cudaFree(a.ptr);
    a.ptr = nullptr;
    a.bytes = 0;
    if ((e = cudaMalloc(&a.ptr, bytes)) != cudaSuccess) {
      cudaGetLastError();
      return static_cast<int>(e);
    }
    a.bytes = bytes;
  }
  *s = a.stream;
  *out = a.ptr;
  return B2_OK;
}

// Copy-in / copy-out streams and per-chunk events for the pipelined host path.
constexpr int kMaxChunks = 16;
struct Pipe {
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t ev_in[kMaxChunks], ev_comp[kMaxChunks];
};
static Pipe g_pipe[64];

static Pipe& pipe_get(int dev) {
  Pipe& p = g_pipe[dev];
  if (!p.in) {
    cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p.out, cudaStreamNonBlocking);
    for (int c = 0; c < kMaxChunks; ++c) {
      cudaEventCreateWithFlags(&p.ev_in[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&p.ev_comp[c], cudaEventDisableTiming);
    }
  }
  return p;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();  // clear: plain host pointers may report an error on old drivers
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

static size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

static int report(const char* fn, int rc) {
  g_last_error = rc;
  if (rc != B2_OK) std::fprintf(stderr, "solomon_b200: %s failed: %s (%d)\n", fn, b2_error_string(rc), rc);
  return rc;
}

static int calc_acc_dropin(int Ni, void* ipos, void* iacc, int Nj, void* jpos, float eps, int flags) {
  if (Ni < 0 || Nj < 0 || (Ni > 0 && (!ipos || !iacc)) || (Nj > 0 && !jpos)) return B2_EINVAL;
  if (Ni == 0) return B2_OK;
  const bool dev = is_device_ptr(ipos) && is_device_ptr(iacc) && (Nj == 0 || is_device_ptr(jpos));
  const size_t ws = b2_calc_acc_workspace_bytes(Ni, Nj, flags);
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_arena_mu[d]);
  cudaStream_t s;
  int rc;
  if (dev) {
    void* w = nullptr;
    if ((rc = arena_get(d, ws ? ws : 256, &w, &s))) return rc;
    if ((rc = b2_calc_acc(Ni, static_cast<float*>(ipos), static_cast<float*>(iacc), Nj, static_cast<float*>(jpos),
                          eps, flags, w, ws, s)))
      return rc;
    cudaError_t e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? B2_OK : static_cast<int>(e);
  }
  const size_t bi = align_up(sizeof(float4) * static_cast<size_t>(Ni));
  const size_t bj = align_up(sizeof(float4) * static_cast<size_t>(Nj));
  const bool same = ipos == jpos && Ni == Nj;
  const size_t total = bi /*ipos*/ + bi /*iacc*/ + (same ? 0 : bj) + align_up(ws);
  void* basev = nullptr;
  if ((rc = arena_get(d, total, &basev, &s))) return rc;
  char* base = static_cast<char*>(basev);
  float* d_i = reinterpret_cast<float*>(base);
  float* d_a = reinterpret_cast<float*>(base + bi);
  float* d_j = same ? d_i : reinterpret_cast<float*>(base + 2 * bi);
  void* d_w = base + 2 * bi + (same ? 0 : bj);
  cudaMemcpyAsync(d_i, ipos, sizeof(float4) * static_cast<size_t>(Ni), cudaMemcpyDefault, s);
  if (!same && Nj) cudaMemcpyAsync(d_j, jpos, sizeof(float4) * static_cast<size_t>(Nj), cudaMemcpyDefault, s);
  if ((rc = b2_calc_acc(Ni, d_i, d_a, Nj, d_j, eps, flags, d_w, ws, s))) return rc;
  cudaMemcpyAsync(iacc, d_a, sizeof(float4) * static_cast<size_t>(Ni), cudaMemcpyDefault, s);
  cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? B2_OK : static_cast<int>(e);
}

static int diffusion_dropin(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                            const float* f, float* fn) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || !f || !fn || f == fn) return B2_EINVAL;
  const size_t n = static_cast<size_t>(nx) * ny * nz;
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_arena_mu[d]);
  cudaStream_t s;
  void* basev = nullptr;
  int rc;
  if (is_device_ptr(f) && is_device_ptr(fn)) {
    if ((rc = arena_get(d, 256, &basev, &s))) return rc;
    // synchronous call: time the step's tile plans once per shape (b2_diffusion3d_plan)
    if ((rc = b2_diffusion3d_plan(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn, 1, s))) return rc;
    if ((rc = b2_diffusion3d(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn, s))) return rc;
    cudaError_t e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? B2_OK : static_cast<int>(e);
  }
  const size_t b = align_up(n * sizeof(float));
  if ((rc = arena_get(d, 2 * b, &basev, &s))) return rc;
  char* base = static_cast<char*>(basev);
  float* d_f = reinterpret_cast<float*>(base);
  float* d_fn = reinterpret_cast<float*>(base + b);
  // Host buffers: pipeline the step over plane chunks so the H2D copy of chunk
  // c+1, the stencil on chunk c and the D2H copy of chunk c-1 overlap (two copy
  // engines + SMs). Output planes [lo, hi) need input planes lo-1..hi, i.e. the
  // chunk itself and the first plane of the next one.
  Pipe& P = pipe_get(d);
  const size_t plane = static_cast<size_t>(ny) * nz;
  const int K = std::max(1, std::min(kMaxChunks, nx / 16));
  auto lo_of = [&](int c) { return static_cast<int>(static_cast<long long>(c) * nx / K); };
  for (int c = 0; c < K; ++c) {
    const int lo = lo_of(c), hi = lo_of(c + 1);
    cudaMemcpyAsync(d_f + lo * plane, f + lo * plane, (hi - lo) * plane * sizeof(float), cudaMemcpyDefault, P.in);
    cudaEventRecord(P.ev_in[c], P.in);
  }
  for (int c = 0; c < K; ++c) {
    cudaStreamWaitEvent(s, P.ev_in[c], 0);
    if (c + 1 < K) cudaStreamWaitEvent(s, P.ev_in[c + 1], 0);
    if ((rc = b2_diffusion3d_slab(nx, ny, nz, dx, dy, dz, dt, kappa, d_f, nullptr, nullptr, d_fn, lo_of(c),
                                  lo_of(c + 1), s)))
      return rc;
    cudaEventRecord(P.ev_comp[c], s);
  }
  for (int c = 0; c < K; ++c) {
    const int lo = lo_of(c), hi = lo_of(c + 1);
    cudaStreamWaitEvent(P.out, P.ev_comp[c], 0);
    cudaMemcpyAsync(fn + lo * plane, d_fn + lo * plane, (hi - lo) * plane * sizeof(float), cudaMemcpyDefault, P.out);
  }
  cudaError_t e = cudaStreamSynchronize(P.out);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? B2_OK : static_cast<int>(e);
}

}  // namespace b2

using namespace b2;

extern "C" {

void calc_acc(const int Ni, solomon_float4* ipos, solomon_float4* iacc, const int Nj, solomon_float4* jpos,
              const float eps) {
  report("calc_acc", calc_acc_dropin(Ni, ipos, iacc, Nj, jpos, eps, 0));
}

void calc_acc_potential(const int Ni, solomon_float4* ipos, solomon_float4* iacc, const int Nj, solomon_float4* jpos,
                        const float eps) {
  report("calc_acc_potential", calc_acc_dropin(Ni, ipos, iacc, Nj, jpos, eps, B2_POTENTIAL));
}

void diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa, const float* f,
                 float* fn) {
  report("diffusion3d", diffusion_dropin(nx, ny, nz, dx, dy, dz, dt, kappa, f, fn));
}

void calc_acc_exact(const int Ni, solomon_float4* ipos, solomon_float4* iacc, const int Nj, solomon_float4* jpos,
                    const float eps) {
  report("calc_acc_exact", calc_acc_dropin(Ni, ipos, iacc, Nj, jpos, eps, B2_EXACT));
}

void calc_acc_potential_exact(const int Ni, solomon_float4* ipos, solomon_float4* iacc, const int Nj,
                              solomon_float4* jpos, const float eps) {
  report("calc_acc_potential_exact", calc_acc_dropin(Ni, ipos, iacc, Nj, jpos, eps, B2_POTENTIAL | B2_EXACT));
}

int b2_last_error(void) { return g_last_error; }

}  // extern "C"
