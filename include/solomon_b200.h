/*
 * solomon_b200 -- B200 (sm_100a) drop-in for the two offloaded kernels of
 * arXiv 2411.18889 (Miki & Hanawa, "Solomon"): the direct-summation N-body
 * force `calc_acc` and the 7-point 3D diffusion step `diffusion3d`, plus the
 * leapfrog (KDK) integrator the north star adds.
 *
 * Two layers, both plain C ABI (no CUDA or torch types in any signature):
 *
 * 1. Drop-in entry points with the reference's EXACT signatures. They accept
 *    host pointers (the reference's fallback/OpenMP calling convention:
 *    staged through device memory, synchronous on return) or device pointers
 *    (the OpenACC `present(...)` convention: computed in place, synchronous).
 *
 * 2. Stream-ordered `b2_*` API on device pointers: no allocation, no host
 *    synchronisation, returns 0 or an error code; scratch space is
 *    caller-owned (`*_workspace_bytes`). The exceptions are named set-up and
 *    query calls: b2_diffusion3d_plan (times tile plans and sizes the resident
 *    mailbox; plans are cached per shape and device, so later calls read that
 *    process-wide cache), b2_fault_status, and the b2_ipc_* mappings.
 *
 * Layouts are the reference's: particles are AoS float4 {x, y, z, m}
 * (listing_nbody.c:1,4-5,9); accelerations float4 {ax, ay, az, pot|0}
 * (listing_nbody.c:6,25); grids are float[nx*ny*nz] with
 * INDEX = k + nz*(j + ny*i), k fastest (listing_diffusion.c:1).
 */
#ifndef SOLOMON_B200_H
#define SOLOMON_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The particle type of listing_nbody.c:1, a 16-byte {x, y, z, w}. A C caller
 * whose driver defines its own float4 (the listing assumes one) can make it the
 * parameter type with `#define SOLOMON_FLOAT4_TYPE float4` before including
 * this header; C++ callers need nothing (see the overloads at the end). */
#if defined(SOLOMON_FLOAT4_TYPE)
typedef SOLOMON_FLOAT4_TYPE solomon_float4;
#elif defined(__VECTOR_TYPES_H__) || defined(__CUDACC__)
typedef float4 solomon_float4;
#else
typedef struct solomon_float4 {
  float x, y, z, w;
} solomon_float4;
#endif

/* ---- return codes of the b2_* API --------------------------------------- */
#define B2_OK 0
#define B2_EINVAL (-1)  /* bad size / null pointer / unsupported flag        */
#define B2_EALIGN (-2)  /* pointer not 16-byte aligned                       */
#define B2_ESPACE (-3)  /* workspace too small                               */
#define B2_ENOMEM (-4)  /* (unused since 0.2: allocation failures report the
                           cudaError_t of the failed cudaMalloc)             */
#define B2_ETIMEOUT (-5) /* a device-side wait for data another CTA or GPU
                            publishes gave up (b2_fault_status)              */
#define B2_ENOTSUP (-6) /* no kernel for this shape on this path (e.g. no
                            two-steps-per-pass plan: b2_diffusion3d_run2_planes) */
/* positive values are cudaError_t codes from the launch / copy / allocation */

/* ---- b2_calc_acc flags --------------------------------------------------- */
#define B2_POTENTIAL 1 /* also accumulate .w += m_j/sqrt(r2): listing_nbody.c:21-23 */
#define B2_EXACT 2     /* IEEE 1/sqrt and the reference's sequential j order:
                          bit-identical to the reference's -O3 fallback build  */

/* =========================================================================
 * 1. Drop-in entry points (reference signatures)
 * ========================================================================= */

/* Replaces `void calc_acc(const int Ni, float4 *ipos, float4 *iacc,
 *                         const int Nj, float4 *jpos, const float eps)`
 * -- pkg/tests/fixtures/listing_nbody.c:1. Host or device
 * pointers; synchronous. Fast path (rsqrt.approx, j-chunked sums): results
 * agree with the reference to FP32 tolerance. */
void calc_acc(const int Ni, solomon_float4 *ipos, solomon_float4 *iacc, const int Nj,
              solomon_float4 *jpos, const float eps);

/* The same listing built with -DCALCULATE_POTENTIAL (listing_nbody.c:21-23). */
void calc_acc_potential(const int Ni, solomon_float4 *ipos, solomon_float4 *iacc, const int Nj,
                        solomon_float4 *jpos, const float eps);

/* The same two with the reference's arithmetic bit for bit (B2_EXACT: IEEE
 * 1/sqrt, sequential j): identical to the listing's -O3 fallback build. */
void calc_acc_exact(const int Ni, solomon_float4 *ipos, solomon_float4 *iacc, const int Nj,
                    solomon_float4 *jpos, const float eps);
void calc_acc_potential_exact(const int Ni, solomon_float4 *ipos, solomon_float4 *iacc, const int Nj,
                              solomon_float4 *jpos, const float eps);

/* Replaces `void diffusion3d(int nx, int ny, int nz, float dx, float dy,
 *   float dz, float dt, float kappa, const float *restrict f, float *restrict fn)`
 * -- pkg/tests/fixtures/listing_diffusion.c:5. Host or device
 * pointers; synchronous; bit-identical to the reference's -O3 build. */
void diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                 const float *f, float *fn);

/* Status of the last drop-in call on this thread (the reference's functions
 * are void; this is how the drop-in reports failures -- also on stderr). */
int b2_last_error(void);
const char *b2_error_string(int code);
const char *b2_version(void);

/* --- Failure detection of the device-side waits ---------------------------
 * Some kernels wait in the GPU for 16-byte words that another CTA
 * (b2_leapfrog's persistent small-N path, b2_diffusion3d_run's resident path)
 * or another GPU (the p2p slab halo: b2_diffusion3d_slab_edges,
 * b2_diffusion3d_slab_halo2) publishes. A wait that exceeds the poll timeout
 * does not hang or trap: the kernel records a fault code in a per-device word,
 * every other waiting kernel on that device gives up at its next poll, and all
 * of them exit normally (their outputs are then undefined). The CUDA context
 * stays usable. */
int b2_set_poll_timeout_ms(long long ms); /* default SOLOMON_POLL_TIMEOUT_S or 120 s;
                                             applies to later launches            */
long long b2_poll_timeout_ms(void);
/* Synchronises `stream` (NULL: the legacy default stream), then reports the
 * current device's fault word: B2_OK, or B2_ETIMEOUT with *which (if not NULL)
 * set to the kernel that gave up first (b2_fault_kernel names it). clear = 1
 * resets the word. Host-synchronising: call it at a checkpoint of a run, not
 * per step. */
int b2_fault_status(void *stream, int clear, int *which);
const char *b2_fault_kernel(int which);
/* Test hook: CTA `cta` of b2_leapfrog's persistent small-N path never announces
 * its positions in later launches (-1: none), so the other CTAs' waits expire --
 * exercises the watchdog path (tests/test_faults_gpu.py). */
int b2_debug_withhold_publish(int cta);

/* =========================================================================
 * 2. Stream-ordered API (device pointers; `stream` is a cudaStream_t or NULL)
 * ========================================================================= */

/* --- N-body force (listing_nbody.c:1-27) --- */

/* Number of j-chunks the fast path splits Nj into. Depends on Nj and flags
 * only, so a sharded run (different Ni) sums in the same order as an
 * unsharded one. 1 for B2_EXACT. */
int b2_calc_acc_nchunks(int Nj, int flags);

/* Scratch bytes b2_calc_acc needs (0 when nchunks == 1): all nchunks x Ni
 * partials up to ~63k i (summed by a second launch), beyond that a ring of 32
 * i-tiles the force kernel sums in place -- at most ~64 MiB at 64 chunks
 * (N = 2^20 and 2^22 alike). Same bits either way. */
size_t b2_calc_acc_workspace_bytes(int Ni, int Nj, int flags);

/* iacc[i] = sum_j m_j (r_j - r_i) / (|r_j - r_i|^2 + eps^2)^{3/2}, i < Ni. */
int b2_calc_acc(int Ni, const float *ipos, float *iacc, int Nj, const float *jpos, float eps,
                int flags, void *workspace, size_t workspace_bytes, void *stream);

/* Per-chunk partial sums: partials[c*Ni + i], c < b2_calc_acc_nchunks(Nj, flags).
 * The building block the fused leapfrog update consumes. */
int b2_calc_acc_partials(int Ni, const float *ipos, int Nj, const float *jpos, float eps, int flags,
                         float *partials, void *stream);

/* --- Leapfrog kick-drift-kick (no reference counterpart) --- */

#define B2_KDK_REDUCE 1     /* acc = sum_c partials[c]  (fixed order c = 0..nchunks-1) */
#define B2_KDK_KICK_END 2   /* vel.xyz = fma(acc, h_end, vel)   closing half-kick        */
#define B2_KDK_KICK_DRIFT 4 /* vel.xyz = fma(acc, h_begin, vel); pos.xyz = fma(vel, dt, pos) */

/* Fused per-particle update; phases run in the order listed above. */
int b2_kdk_update(int n, float *pos, float *vel, float *acc, const float *partials, int nchunks,
                  float h_end, float h_begin, float dt, int phases, void *stream);

/* Multi-GPU variant (fused all-gather): reads positions from pos_in, writes
 * the updated (or, without B2_KDK_KICK_DRIFT, unchanged) positions to pos_out
 * AND to each of the npeers (<= 8) peer buffers -- device addresses mapped
 * with b2_ipc_import, i.e. other GPUs' position arrays over NVLink/NVSwitch. */
int b2_kdk_update_publish(int n, const float *pos_in, float *pos_out, float *vel, float *acc,
                          const float *partials, int nchunks, float h_end, float h_begin, float dt,
                          int phases, float *const *peers, int npeers, void *stream);

/* NVLS variant (NVSwitch multicast all-gather): the updated positions are stored
 * ONCE through mc_out -- the multicast view (b2_mc_bind) of every rank's position
 * buffer at this rank's slice -- and land in every rank's copy, this one's included. */
int b2_kdk_update_multicast(int n, const float *pos_in, float *mc_out, float *vel, float *acc,
                            const float *partials, int nchunks, float h_end, float h_begin, float dt,
                            int phases, void *stream);

/* Whole single-device leapfrog: nsteps KDK steps of the self-gravitating
 * system pos[n] (acc must hold a(pos) on entry unless B2_INIT_ACC is set;
 * holds a(pos) on exit). Small systems (n <= 64 x SMs, fast arithmetic) run
 * every step in one persistent launch; otherwise two launches per step. Both
 * give the same bits. */
#define B2_INIT_ACC 4
int b2_leapfrog(int n, float *pos, float *vel, float *acc, float eps, float dt, int nsteps, int flags,
                void *workspace, size_t workspace_bytes, void *stream);
size_t b2_leapfrog_workspace_bytes(int n, int flags);

/* --- 3D diffusion (listing_diffusion.c:1-25) --- */

/* One explicit step fn = L(f) over the whole grid; f != fn. Uses the tile
 * plan b2_diffusion3d_plan chose for the shape on this device, else the
 * model's default (same bits either way). */
int b2_diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                   const float *f, float *fn, void *stream);

/* Set-up call (the ONE place the diffusion path may allocate or synchronise):
 * times a few tile plans of the single step (whole grid and the interior
 * planes [1, nx-1) of a slab) and, with nsteps >= 2, of the two-steps-per-pass
 * kernel on f (read) and fn (written: scratch), keeps the fastest per shape and
 * device, and sizes the library-owned mailbox of b2_diffusion3d_run's resident
 * path. Host-synchronising; tuning is skipped under stream capture and with
 * SOLOMON_DIFF_AUTOTUNE=0. Optional: unplanned shapes run on the model's plans
 * (and without the resident path), with identical bits. */
int b2_diffusion3d_plan(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                        const float *f, float *fn, int nsteps, void *stream);

/* Slab variant for i-decomposition: f holds this rank's
 * nx_local planes; halo_lo / halo_hi are the neighbour planes i = -1 and
 * i = nx_local (ny*nz floats each) or NULL at a global boundary (clamp, as
 * IMAX(i-1,0) / IMIN(i+1,nx-1)). Computes output planes [i_begin, i_end). */
int b2_diffusion3d_slab(int nx_local, int ny, int nz, float dx, float dy, float dz, float dt,
                        float kappa, const float *f, const float *halo_lo, const float *halo_hi,
                        float *fn, int i_begin, int i_end, void *stream);

/* Fused slab-halo exchange for i-decomposed multi-GPU diffusion.
 * Computes planes 0 and nx_local-1 of fn (state step+1) from f (state step)
 * and the neighbours' edge planes, and publishes this rank's new edge planes.
 * Halos travel through per-rank mailboxes of 16-byte words {value, tag, value,
 * tag} (one side = b2_diffusion3d_mailbox_bytes(ny, nz)): in_lo / in_hi are this rank's sides
 * fed by rank-1 / rank+1 (NULL at a global boundary: clamp), out_lo / out_hi
 * the neighbours' sides fed by this rank (peer pointers from b2_ipc_import;
 * NULL: no neighbour). Mailboxes must be zeroed before the first push.
 * push_only = 1 publishes the edge planes of state `step` (call once per run
 * before the first step). No host synchronisation: the kernel polls its
 * mailbox for rows tagged with the expected state. Planes 1..nx_local-2 are a
 * b2_diffusion3d_slab(..., halo_lo = halo_hi = NULL, 1, nx_local-1) launch. */
size_t b2_diffusion3d_mailbox_bytes(int ny, int nz);
int b2_diffusion3d_slab_edges(int nx_local, int ny, int nz, float dx, float dy, float dz, float dt,
                              float kappa, const float *f, float *fn, const void *in_lo,
                              const void *in_hi, void *out_lo, void *out_hi, int step,
                              int push_only, void *stream);

/* Two-plane halo exchange for two steps per exchange (SlabDiffusion.run,
 * DESIGN.md §6). f is this rank's halo-extended slab of nx_ext = lo_h +
 * nx_local + hi_h planes (lo_h / hi_h = 2 with a neighbour on that side, 0 at
 * a global end). phase 0 pushes this rank's two edge planes of the current
 * state into the neighbours' mailboxes (out_lo / out_hi: peer pointers from
 * b2_ipc_import, b2_diffusion3d_mailbox2_bytes(ny, nz) bytes per side);
 * phase 1 waits in the GPU for the neighbours' planes in this rank's own
 * mailbox (in_lo / in_hi) and writes them into the halo planes. xchg counts
 * exchanges from 0 (mailboxes zeroed once before the first). Launch phase 0
 * then phase 1 on the same stream. */
size_t b2_diffusion3d_mailbox2_bytes(int ny, int nz);
int b2_diffusion3d_slab_halo2(int nx_ext, int ny, int nz, int lo_h, int nx_local, float *f,
                              const void *in_lo, const void *in_hi, void *out_lo, void *out_hi,
                              int xchg, int phase, void *stream);

/* nsteps device-resident steps ping-ponging f <-> fn (no host sync, no
 * allocation). Grids that fit the chip's shared memory (e.g. 128^3) run all
 * steps in one persistent launch with the field resident in shared memory
 * (bricks exchanging faces through the library-owned mailbox that
 * b2_diffusion3d_plan(..., nsteps >= 2, ...) sized; unplanned: the next path);
 * other L2-resident grids in one cooperative launch; large grids two steps
 * per HBM pass where the planner finds a worthwhile tile
 * (SOLOMON_DIFF_TEMPORAL=0: one step per pass), with the tile plan
 * b2_diffusion3d_plan timed if it ran. All paths are bit-identical to nsteps
 * single steps. *result_in_fn (if not NULL) is set to 1 when the final field
 * is in fn, 0 when it is in f; the other buffer is scratch. */
int b2_diffusion3d_run(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                       float *f, float *fn, int nsteps, int *result_in_fn, void *stream);

/* Two steps f -> fn written ONLY to fn's planes [p0, p1) and [p2, p3) (disjoint;
 * either may be empty; the rest of fn is untouched), reading f's planes within two
 * of them, clamped at 0 / nx-1 -- the same bits as those planes of
 * b2_diffusion3d_run(..., 2, ...). For slabs that overlap a halo exchange with the
 * pass: the planes that need no halo first, then the two next to each halo (one
 * launch for both) once it arrived. Uses the two-steps-per-pass kernel; B2_ENOTSUP
 * when the shape has no plan for it (empty ranges only ask). */
int b2_diffusion3d_run2_planes(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                               const float *f, float *fn, int p0, int p1, int p2, int p3, void *stream);

/* --- NVLS multicast buffers (NVSwitch) --------------------------
 * One multicast object spans the ranks' GPUs. Rank 0: b2_mc_create (adds its
 * device, exports a b2_mc_handle_bytes() fabric handle to send to the others); every
 * other rank: b2_mc_add_device; after ALL ranks added their device (host barrier):
 * b2_mc_bind maps this rank's copy (uc) and the multicast view (mc) of `bytes` (a
 * multiple of b2_mc_granular_bytes). Stores through mc reach every rank's copy. */
int b2_mc_supported(int device); /* 1: the GPU supports multicast AND this process can
                                    create an object (reaches the NVSwitch fabric) */
size_t b2_mc_handle_bytes(void);
int b2_mc_granular_bytes(size_t bytes, int ndev, size_t *out);
int b2_mc_create(size_t bytes, int ndev, int device, void *handle, void **binding);
int b2_mc_add_device(const void *handle, int device, void **binding);
int b2_mc_bind(void *binding, size_t bytes, void **uc_ptr, void **mc_ptr);
int b2_mc_release(void *binding);

/* --- Peer memory across processes (multi-GPU fused halo) --- */

/* Size of an exported handle (a cudaIpcMemHandle_t, 64 bytes). */
size_t b2_ipc_handle_bytes(void);
/* Export the allocation holding dptr: handle (b2_ipc_handle_bytes() bytes) and
 * dptr's offset inside that allocation. */
int b2_ipc_export(const void *dptr, void *handle, size_t *offset);
/* Map a peer's exported allocation into this process (peer access enabled on
 * demand) and return the address of the exported pointer. */
int b2_ipc_import(const void *handle, size_t offset, void **dptr);
int b2_ipc_close(void *dptr, size_t offset);

#ifdef __cplusplus
}

/* C++ callers: the listing's call sites compile unchanged with the caller's own
 * 16-byte float4 (listing_nbody.c:1 takes `float4 *`; a driver that defines
 * `struct float4 {float x, y, z, w;}` binds here, the pointers are passed on). */
#include <type_traits>
#define SOLOMON_B200_F4_OVERLOAD(name)                                                              \
  template <class F4, class = typename std::enable_if<sizeof(F4) == 16 &&                           \
                                                      !std::is_same<F4, solomon_float4>::value>::type> \
  inline void name(const int Ni, F4 *ipos, F4 *iacc, const int Nj, F4 *jpos, const float eps) {     \
    name(Ni, reinterpret_cast<solomon_float4 *>(ipos), reinterpret_cast<solomon_float4 *>(iacc), Nj,  \
         reinterpret_cast<solomon_float4 *>(jpos), eps);                                            \
  }
SOLOMON_B200_F4_OVERLOAD(calc_acc)
SOLOMON_B200_F4_OVERLOAD(calc_acc_potential)
SOLOMON_B200_F4_OVERLOAD(calc_acc_exact)
SOLOMON_B200_F4_OVERLOAD(calc_acc_potential_exact)
#undef SOLOMON_B200_F4_OVERLOAD
#endif

#endif /* SOLOMON_B200_H */
