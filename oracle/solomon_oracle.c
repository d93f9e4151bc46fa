/*
 * CPU restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * this library; the product package (paper_2411_18889_b200) never does. It is
 * the checker, never the thing measured or shipped.
 *
 * Every function restates a reference listing operation-for-operation so the
 * result is bit-identical to the reference's own fallback build
 * (oracle/_ref/libref_ieee_*.so, built by oracle/build_ref.py from the
 * reference sources) -- tests/test_oracle.py pins that, and pins both against
 * the committed golden vectors in tests/golden/.
 *
 * Compiled with -ffp-contract=off: every fused multiply-add below is explicit,
 * matching the contraction GCC -O3 applies to the reference listings (checked
 * by disassembly of libref_ieee_native.so).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* ---------------------------------------------------------------------------
 * calc_acc -- pkg/tests/fixtures/listing_nbody.c:1-27 (= PAPER.md:467-493)
 * ipos/jpos/iacc: float4[N] AoS {x, y, z, w}; jpos.w = mass.
 */
void oracle_calc_acc(int Ni, const float *ipos, float *iacc, int Nj, const float *jpos, float eps,
                     int potential) {
  const float eps2 = eps * eps; /* listing_nbody.c:5  pi.w = eps * eps */
#pragma omp parallel for schedule(static)
  for (int i = 0; i < Ni; i++) { /* :3 parallel i-loop */
    const float pix = ipos[4 * (size_t)i + 0];
    const float piy = ipos[4 * (size_t)i + 1];
    const float piz = ipos[4 * (size_t)i + 2];
    float ax = 0.0f, ay = 0.0f, az = 0.0f, aw = 0.0f; /* :6 */
    for (int j = 0; j < Nj; j++) {                    /* :8 sequential j-loop, self term included */
      const float *pj = jpos + 4 * (size_t)j;
      const float rx = pj[0] - pix; /* :11-13 */
      const float ry = pj[1] - piy;
      const float rz = pj[2] - piz;
      const float r2 = fmaf(rz, rz, fmaf(ry, ry, fmaf(rx, rx, eps2))); /* :14 */
      float w = 1.0f / sqrtf(r2);                                       /* :15 */
      w *= w * w;                                                       /* :16 */
      w *= pj[3];                                                       /* :17 */
      ax = fmaf(rx, w, ax);                                             /* :18-20 */
      ay = fmaf(ry, w, ay);
      az = fmaf(rz, w, az);
      if (potential) aw = fmaf(r2, w, aw); /* :21-23 CALCULATE_POTENTIAL */
    }
    iacc[4 * (size_t)i + 0] = ax; /* :25 */
    iacc[4 * (size_t)i + 1] = ay;
    iacc[4 * (size_t)i + 2] = az;
    iacc[4 * (size_t)i + 3] = aw;
  }
}

/* ---------------------------------------------------------------------------
 * diffusion3d -- pkg/tests/fixtures/listing_diffusion.c:1-25 (= PAPER.md:553-578)
 * INDEX(nx,ny,nz,i,j,k) = k + nz*(j + ny*i)  (:1): k fastest, i slowest.
 * Clamped neighbours IMIN/IMAX (:2-3, :15-20). 64-bit offsets (the reference's
 * int INDEX overflows past 1290^3; identical results below that).
 */
void oracle_diffusion_coeffs(float dx, float dy, float dz, float dt, float kappa, float c[4]) {
  const float kd = kappa * dt;
  const float ce = kd / (dx * dx); /* :6  cw = ce */
  const float cn = kd / (dy * dy); /* :7  cs = cn */
  const float ct = kd / (dz * dz); /* :8  cb = ct */
  const float cc = 1.0f - (((((ce + ce) + cn) + cn) + ct) + ct); /* :9 */
  c[0] = cc;
  c[1] = ce;
  c[2] = cn;
  c[3] = ct;
}

void oracle_diffusion3d(int nx, int ny, int nz, float dx, float dy, float dz, float dt, float kappa,
                        const float *f, float *fn) {
  float c[4];
  oracle_diffusion_coeffs(dx, dy, dz, dt, kappa, c);
  const float cc = c[0], ce = c[1], cw = c[1], cn = c[2], cs = c[2], ct = c[3], cb = c[3];
  const size_t sy = (size_t)nz, sx = (size_t)nz * (size_t)ny;
#pragma omp parallel for collapse(2) schedule(static)
  for (int i = 0; i < nx; i++) {
    for (int j = 0; j < ny; j++) {
      const int ip = i + 1 < nx - 1 ? i + 1 : nx - 1; /* IMIN(i + 1, nx - 1) */
      const int im = i - 1 > 0 ? i - 1 : 0;           /* IMAX(i - 1, 0) */
      const int jp = j + 1 < ny - 1 ? j + 1 : ny - 1;
      const int jm = j - 1 > 0 ? j - 1 : 0;
      for (int k = 0; k < nz; k++) {
        const int kp = k + 1 < nz - 1 ? k + 1 : nz - 1;
        const int km = k - 1 > 0 ? k - 1 : 0;
        const size_t ix = (size_t)k + sy * (size_t)j + sx * (size_t)i;
        /* :21 as g++ -O3 contracts it: the first sum
         * cc*f + ce*f_ip becomes fma(cc, f, ce*f_ip); then five more FMAs
         * left to right. */
        float v = ce * f[(size_t)k + sy * j + sx * ip];
        v = fmaf(cc, f[ix], v);
        v = fmaf(cw, f[(size_t)k + sy * j + sx * im], v);
        v = fmaf(cn, f[(size_t)k + sy * jp + sx * i], v);
        v = fmaf(cs, f[(size_t)k + sy * jm + sx * i], v);
        v = fmaf(ct, f[(size_t)kp + sy * j + sx * i], v);
        v = fmaf(cb, f[(size_t)km + sy * j + sx * i], v);
        fn[ix] = v;
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * Leapfrog kick-drift-kick -- NO reference counterpart (north star only,
 * SURVEY.md §8a row a7). Spec, per particle, FP32, explicit FMA:
 *   kick : v = fma(a, h, v)            (h = dt/2, xyz only)
 *   drift: x = fma(v, dt, x)           (xyz only; x.w = mass untouched)
 * One step = kick, drift, a = calc_acc(x), kick.
 */
void oracle_kick(int n, float *vel, const float *acc, float h) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; i++)
    for (int d = 0; d < 3; d++) vel[4 * (size_t)i + d] = fmaf(acc[4 * (size_t)i + d], h, vel[4 * (size_t)i + d]);
}

void oracle_drift(int n, float *pos, const float *vel, float dt) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; i++)
    for (int d = 0; d < 3; d++) pos[4 * (size_t)i + d] = fmaf(vel[4 * (size_t)i + d], dt, pos[4 * (size_t)i + d]);
}

/* nsteps KDK steps of the whole system; acc holds a(x) on entry and exit. */
void oracle_leapfrog(int n, float *pos, float *vel, float *acc, float eps, float dt, int nsteps, int potential) {
  const float h = 0.5f * dt;
  for (int s = 0; s < nsteps; s++) {
    oracle_kick(n, vel, acc, h);
    oracle_drift(n, pos, vel, dt);
    oracle_calc_acc(n, pos, acc, n, pos, eps, potential);
    oracle_kick(n, vel, acc, h);
  }
}

/* ---------------------------------------------------------------------------
 * Chunked force + fused update: restates the STRUCTURE of the fast GPU path
 * (csrc/nbody.cu) with the reference's per-pair arithmetic, so the multi-rank
 * exchange logic (paper_2411_18889_b200/distributed.py) can be checked on CPU.
 * partials[c*Ni + i] = sum over j in chunk c (sequential from 0).
 */
void oracle_calc_acc_partials(int Ni, const float *ipos, int Nj, const float *jpos, float eps, int potential,
                              int chunk, float *partials) {
  const int nch = (Nj + chunk - 1) / chunk;
  for (int c = 0; c < nch; c++) {
    const int j0 = c * chunk;
    const int cnt = (Nj - j0) < chunk ? (Nj - j0) : chunk;
    oracle_calc_acc(Ni, ipos, partials + 4 * (size_t)c * Ni, cnt, jpos + 4 * (size_t)j0, eps, potential);
  }
}

/* Phases as b2_kdk_update (include/solomon_b200.h): 1 reduce, 2 closing kick, 4 opening kick + drift. */
void oracle_kdk_update(int n, float *pos, float *vel, float *acc, const float *partials, int nchunks, float h_end,
                       float h_begin, float dt, int phases) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; i++) {
    float a[4];
    if (phases & 1) {
      for (int d = 0; d < 4; d++) a[d] = partials[4 * (size_t)i + d];
      for (int c = 1; c < nchunks; c++)
        for (int d = 0; d < 4; d++) a[d] = a[d] + partials[4 * ((size_t)c * n + i) + d];
      for (int d = 0; d < 4; d++) acc[4 * (size_t)i + d] = a[d];
    } else {
      for (int d = 0; d < 4; d++) a[d] = acc[4 * (size_t)i + d];
    }
    if (phases & 2)
      for (int d = 0; d < 3; d++) vel[4 * (size_t)i + d] = fmaf(a[d], h_end, vel[4 * (size_t)i + d]);
    if (phases & 4) {
      for (int d = 0; d < 3; d++) vel[4 * (size_t)i + d] = fmaf(a[d], h_begin, vel[4 * (size_t)i + d]);
      for (int d = 0; d < 3; d++) pos[4 * (size_t)i + d] = fmaf(vel[4 * (size_t)i + d], dt, pos[4 * (size_t)i + d]);
    }
  }
}

/* ---------------------------------------------------------------------------
 * FP64 yardstick for calc_acc (NOT a restatement): the same force law in double
 * precision with an exact 1/sqrt, used by the tests and bench.py to measure how far
 * an FP32 result is from the exact sum. At N = 2^22 the reference's own sequential
 * FP32 j-sum (listing_nbody.c:8-24) is 3.5e-4 (relative L2) away from it, so a
 * large-N parity check judges an implementation by its distance to this, next to the
 * reference's distance. out: double[4*Ni].
 */
void oracle_calc_acc_f64(int Ni, const float *ipos, double *out, int Nj, const float *jpos, float eps) {
  const double eps2 = (double)eps * (double)eps;
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < Ni; i++) {
    const double pix = ipos[4 * (size_t)i + 0], piy = ipos[4 * (size_t)i + 1], piz = ipos[4 * (size_t)i + 2];
    double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
    for (int j = 0; j < Nj; j++) {
      const float *pj = jpos + 4 * (size_t)j;
      const double rx = pj[0] - pix, ry = pj[1] - piy, rz = pj[2] - piz;
      const double r2 = rx * rx + ry * ry + rz * rz + eps2;
      const double w1 = 1.0 / sqrt(r2);
      const double w = pj[3] * w1 * w1 * w1;
      ax += rx * w;
      ay += ry * w;
      az += rz * w;
      aw += pj[3] * w1;
    }
    out[4 * (size_t)i + 0] = ax;
    out[4 * (size_t)i + 1] = ay;
    out[4 * (size_t)i + 2] = az;
    out[4 * (size_t)i + 3] = aw;
  }
}
