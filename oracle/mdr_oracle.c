/*
 * mdr_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's hot path, used as the parity checker by tests/, smoke() and the
 * CPU arm of bench.py.  It is never linked into, or called by, the product.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the golden vectors of the reference's own tests (RNG stream, half
 *       conversions, reduce4 / reduce7 / block-reduce frozen examples, the
 *       single-well stationarity, the ADADELTA first step), and
 *   (2) the reference itself, compiled in place into oracle/_ref by
 *       oracle/Makefile, on seeded random inputs (bit-for-bit).
 * Built with -O2 -ffp-contract=off like the reference (CMakeLists.txt:24);
 * double/float operations below are written in the reference's evaluation
 * order so results agree to the last bit.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mdr.h"
#include "crmath.h"

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ RNG */
/* rng.cpp:11-56 — splitmix64 finalizer over a counter, keyed by
 * mix64(seed ^ mix64(fnv1a64(label))). */
static uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key, ctr;
} orc_rng;

static orc_rng orc_rng_make(uint64_t seed, const char* label) {
  uint64_t h = 0xcbf29ce484222325ull; /* FNV-1a 64 offset basis */
  for (const unsigned char* p = (const unsigned char*)label; *p; ++p)
    h = (h ^ *p) * 0x100000001b3ull;
  orc_rng r;
  r.key = orc_mix64(seed ^ orc_mix64(h));
  r.ctr = 0;
  return r;
}

static uint64_t orc_u64(orc_rng* r) {
  r->ctr += 1; /* pre-increment: draw n uses counter n (rng.cpp:34-37) */
  return orc_mix64(r->key + r->ctr * 0x9e3779b97f4a7c15ull);
}
static double orc_unit(orc_rng* r) { return (double)(orc_u64(r) >> 11) * 0x1p-53; }
static double orc_uniform(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_unit(r); }
static double orc_normal(orc_rng* r) { /* rng.cpp:47-52, exactly two draws */
  const double u1 = (double)((orc_u64(r) >> 11) + 1) * 0x1p-53;
  const double u2 = orc_unit(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * ORC_PI * u2);
}
/* The same draw with correctly rounded log / cos (grid mode, crmath.h). */
static double orc_normal_cr(orc_rng* r) {
  const double u1 = (double)((orc_u64(r) >> 11) + 1) * 0x1p-53;
  const double u2 = orc_unit(r);
  return sqrt(-2.0 * cr_log(u1)) * cr_cos(2.0 * ORC_PI * u2);
}
static uint64_t orc_index(orc_rng* r, uint64_t n) { return n == 0 ? 0 : orc_u64(r) % n; }

void orc_rng_draws(uint64_t seed, const char* label, uint64_t n, uint64_t* out) {
  orc_rng r = orc_rng_make(seed, label);
  for (uint64_t i = 0; i < n; ++i) out[i] = orc_u64(&r);
}

void orc_rng_normals(uint64_t seed, const char* label, uint64_t n, double* out) {
  orc_rng r = orc_rng_make(seed, label);
  for (uint64_t i = 0; i < n; ++i) out[i] = orc_normal(&r);
}

/* ------------------------------------------------------------ binary16 */
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* half.cpp:8-54: RNE, subnormals kept, overflow to inf, NaN -> 0x7E00.
 * Restated via the "magic add" formulation: scale into the half grid,
 * let the binary32 adder round, read the bits back. */
static uint16_t orc_f2h(float v) {
  const uint32_t x = f2u(v);
  const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  const uint32_t mag = x & 0x7fffffffu;
  if (mag > 0x7f800000u) return 0x7e00;                  /* NaN */
  if (mag >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u); /* >= 65520 -> inf */
  if (mag < 0x38800000u) {
    /* below the smallest normal half (2^-14): result is k * 2^-24 with k
     * the RNE rounding of |v| * 2^24; adding 0.5 (2^-1) aligns the binary32
     * ulp to 2^-24 so the hardware add performs exactly that rounding. */
    const float t = u2f(mag) + 0.5f;
    return (uint16_t)(sign | (uint16_t)(f2u(t) - 0x3f000000u));
  }
  /* normal range: keep 10 mantissa bits, RNE on the 13 dropped ones */
  const uint32_t odd = (mag >> 13) & 1u;
  const uint32_t r = (mag + 0x0fffu + odd) >> 13; /* may carry into exponent */
  return (uint16_t)(sign | (uint16_t)(r - (112u << 10)));
}

/* half.cpp:56-74: exact widening. */
static float orc_h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  if (e == 0x1f) return m ? u2f(0x7fc00000u) : u2f(sign | 0x7f800000u);
  if (e == 0) return u2f(sign | f2u((float)m * 0x1p-24f));
  return u2f(sign | ((e + 112u) << 23) | (m << 13));
}

void orc_f32_to_half(const float* in, size_t n, uint16_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_f2h(in[i]);
}
void orc_half_to_f32(const uint16_t* in, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_h2f(in[i]);
}
static float orc_hround(float v) { return orc_h2f(orc_f2h(v)); }

/* ------------------------------------------------------------- MMA unit */
/* mma.cpp:41-64: d = (sum_k ascending a*b in fp32) + c, one half rounding
 * in Half mode.  a, b, c, d row-major 16x16. */
static void orc_mma_f(const float* a, const float* b, const float* c, int half_mode, float* d) {
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) {
      float acc = 0.0f;
      for (int k = 0; k < 16; ++k) acc += a[i * 16 + k] * b[k * 16 + j];
      const float r = acc + c[i * 16 + j];
      d[i * 16 + j] = half_mode ? orc_hround(r) : r;
    }
}

int orc_mma(const uint16_t* a, const uint16_t* b, const float* c, int accum, float* d) {
  float af[256], bf[256];
  for (int i = 0; i < 256; ++i) {
    af[i] = orc_h2f(a[i]);
    bf[i] = orc_h2f(b[i]);
  }
  orc_mma_f(af, bf, c, accum == MDR_ACCUM_HALF, d);
  return MDR_OK;
}

/* ------------------------------------------------------- reduce4 / 7 */
static void zero_stats(mdr_sync_stats* s) { if (s) memset(s, 0, sizeof *s); }
static void add_stats(mdr_sync_stats* a, const mdr_sync_stats* b) {
  a->block_syncs += b->block_syncs;
  a->warp_shuffles += b->warp_shuffles;
  a->atomic_adds += b->atomic_adds;
  a->memory_fences += b->memory_fences;
  a->mma_ops += b->mma_ops;
  a->shared_mem_bytes += b->shared_mem_bytes;
  a->precision_conversions += b->precision_conversions;
}

/* reduce4 reduce.cpp:80-111.  Chunk of <=64 vectors packed column-major
 * (pack_vectors reduce.cpp:36-51): element (row i, col k) of A is component
 * i%4 of vector 4k + i/4.  V += A*P (P all ones, reduce.cpp:12-21); then
 * W = Q*half(V) (Q(i,j) = [i==j mod 4], reduce.cpp:23-34). */
int orc_reduce4(const float* vecs, int n, int accum, float* out, mdr_sync_stats* st) {
  if (n < 1) return MDR_ERR_SIZE;
  const int half_mode = accum == MDR_ACCUM_HALF;
  const int chunks = (n + 63) / 64;
  static float ones[256], q[256];
  for (int i = 0; i < 256; ++i) {
    ones[i] = 1.0f;
    q[i] = ((i / 16) % 4 == (i % 16) % 4) ? 1.0f : 0.0f;
  }
  float v[256] = {0}, a[256], vop[256], w[256], zero[256] = {0};
  for (int c = 0; c < chunks; ++c) {
    for (int i = 0; i < 256; ++i) a[i] = 0.0f;
    for (int j = 0; j < 64 && c * 64 + j < n; ++j)
      for (int comp = 0; comp < 4; ++comp) {
        const int flat = 4 * j + comp;               /* column-major staging */
        const int row = flat % 16, col = flat / 16;
        a[row * 16 + col] = orc_hround(vecs[4 * (c * 64 + j) + comp]);
      }
    float nv[256];
    orc_mma_f(a, ones, v, half_mode, nv);
    memcpy(v, nv, sizeof v);
  }
  for (int i = 0; i < 256; ++i) vop[i] = orc_hround(v[i]); /* accum_to_operand */
  orc_mma_f(q, vop, zero, half_mode, w);
  out[0] = w[0 * 16];
  out[1] = w[1 * 16];
  out[2] = w[2 * 16];
  out[3] = w[3 * 16];
  if (st) {
    zero_stats(st);
    st->block_syncs = 2;
    st->shared_mem_bytes = (uint64_t)chunks * 64 * 4 * 2;
    st->precision_conversions = 4ull * (uint64_t)n + (half_mode ? 4u : 256u);
    st->mma_ops = (uint64_t)chunks + 1;
  }
  return MDR_OK;
}

/* baseline_warp_reduce reduce.cpp:113-134: lockstep shuffle-down tree. */
int orc_warp_reduce(const float* lanes, int n, float* out, mdr_sync_stats* st) {
  if (n != 32) return MDR_ERR_SIZE;
  float v[32];
  memcpy(v, lanes, sizeof v);
  for (int off = 16; off >= 1; off /= 2)
    for (int i = 0; i + off < 32; ++i) v[i] = v[i] + v[i + off]; /* i<j reads old v[j]: j>i */
  *out = v[0];
  if (st) {
    zero_stats(st);
    st->warp_shuffles = 160;
  }
  return MDR_OK;
}

static int block_ok(int threads) { return threads >= 32 && threads <= 1024 && threads % 32 == 0; }

/* baseline_block_reduce reduce.cpp:136-163. */
int orc_block_reduce(const float* values, int n, int threads, float* out, mdr_sync_stats* st) {
  if (!block_ok(threads)) return MDR_ERR_BLOCK_SIZE;
  if (n != threads) return MDR_ERR_SIZE;
  float acc = 0.0f, w;
  for (int k = 0; k < threads / 32; ++k) {
    orc_warp_reduce(values + 32 * k, 32, &w, NULL);
    acc += w;
  }
  *out = acc;
  if (st) {
    zero_stats(st);
    st->block_syncs = 3;
    st->memory_fences = 2;
    st->shared_mem_bytes = 4;
    st->atomic_adds = (uint64_t)(threads / 32);
    st->warp_shuffles = 160ull * (uint64_t)(threads / 32);
  }
  return MDR_OK;
}

/* reduce7 reduce.cpp:165-209; recs n x {e,gx,gy,gz,tx,ty,tz}. */
int orc_reduce7(const float* recs, int n, int method, int accum, float* out, mdr_sync_stats* st) {
  mdr_sync_stats tot, one;
  zero_stats(&tot);
  if (method == MDR_METHOD_BASELINE) {
    if (!block_ok(n)) return MDR_ERR_BLOCK_SIZE;
    float* col = (float*)malloc(sizeof(float) * (size_t)n);
    for (int c = 0; c < 7; ++c) {
      for (int i = 0; i < n; ++i) col[i] = recs[7 * i + c];
      orc_block_reduce(col, n, n, &out[c], &one);
      add_stats(&tot, &one);
    }
    free(col);
  } else {
    if (n < 64) return MDR_ERR_BLOCK_SIZE;
    float* g = (float*)malloc(sizeof(float) * 4 * (size_t)n);
    float* t = (float*)malloc(sizeof(float) * 4 * (size_t)n);
    for (int i = 0; i < n; ++i) {
      const float* r = recs + 7 * i;
      g[4 * i] = r[1]; g[4 * i + 1] = r[2]; g[4 * i + 2] = r[3]; g[4 * i + 3] = r[0];
      t[4 * i] = r[4]; t[4 * i + 1] = r[5]; t[4 * i + 2] = r[6]; t[4 * i + 3] = 0.0f;
    }
    float rg[4], rt[4];
    orc_reduce4(g, n, accum, rg, &one);
    add_stats(&tot, &one);
    orc_reduce4(t, n, accum, rt, &one);
    add_stats(&tot, &one);
    out[0] = rg[3]; out[1] = rg[0]; out[2] = rg[1]; out[3] = rg[2];
    out[4] = rt[0]; out[5] = rt[1]; out[6] = rt[2];
    free(g);
    free(t);
  }
  if (st) *st = tot;
  return MDR_OK;
}

/* simulate_block (Vec4 form) simblock.cpp:436-463. */
int orc_simulate_block4(const float* vecs, int n, int method, int accum, float* out, mdr_sync_stats* st) {
  const int lo = method == MDR_METHOD_TCU ? 64 : 32;
  if (n < lo || n > 1024 || n % 32) return MDR_ERR_BLOCK_SIZE;
  if (method == MDR_METHOD_TCU) return orc_reduce4(vecs, n, accum, out, st);
  mdr_sync_stats tot, one;
  zero_stats(&tot);
  float* col = (float*)malloc(sizeof(float) * (size_t)n);
  for (int c = 0; c < 4; ++c) {
    for (int i = 0; i < n; ++i) col[i] = vecs[4 * i + c];
    orc_block_reduce(col, n, n, &out[c], &one);
    add_stats(&tot, &one);
  }
  free(col);
  if (st) *st = tot;
  return MDR_OK;
}

/* ------------------------------------------------------------- scoring */
typedef struct { double v[3]; } v3;
typedef struct { double m[3][3]; } m3; /* rows */

static double dot3(v3 a, v3 b) { return a.v[0] * b.v[0] + a.v[1] * b.v[1] + a.v[2] * b.v[2]; }
static v3 cross3(v3 a, v3 b) {
  v3 r = {{a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
           a.v[0] * b.v[1] - a.v[1] * b.v[0]}};
  return r;
}
static v3 add3(v3 a, v3 b) { v3 r = {{a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]}}; return r; }
static v3 sub3(v3 a, v3 b) { v3 r = {{a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]}}; return r; }
static v3 scl3(double s, v3 a) { v3 r = {{s * a.v[0], s * a.v[1], s * a.v[2]}}; return r; }
static v3 mv3(const m3* m, v3 x) {
  v3 r;
  for (int i = 0; i < 3; ++i) {
    v3 row = {{m->m[i][0], m->m[i][1], m->m[i][2]}};
    r.v[i] = dot3(row, x);
  }
  return r;
}
static m3 mm3(const m3* a, const m3* b) { /* docking.cpp:36-44 */
  m3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[i][j] = a->m[i][0] * b->m[0][j] + a->m[i][1] * b->m[1][j] + a->m[i][2] * b->m[2][j];
  return r;
}
static m3 rz(double a) {
  const double c = cos(a), s = sin(a);
  m3 r = {{{c, -s, 0.0}, {s, c, 0.0}, {0.0, 0.0, 1.0}}};
  return r;
}
static m3 ry(double a) {
  const double c = cos(a), s = sin(a);
  m3 r = {{{c, 0.0, s}, {0.0, 1.0, 0.0}, {-s, 0.0, c}}};
  return r;
}

/* torsion_axis docking.cpp:181-189 */
static v3 orc_torsion_axis(int k) {
  const double az = 2.399963229728653 * k + 0.3;
  const double zc = 0.5 + 0.35 * sin(0.9 * k + 0.4);
  v3 v = {{0.8 * cos(az), 0.8 * sin(az), zc}};
  const double n = sqrt(dot3(v, v));
  v3 r = {{v.v[0] / n, v.v[1] / n, v.v[2] / n}};
  return r;
}

void orc_torsion_axis_out(int k, double* out3) {
  v3 a = orc_torsion_axis(k);
  out3[0] = a.v[0]; out3[1] = a.v[1]; out3[2] = a.v[2];
}

static double wrap(double a) { /* docking.cpp:62-64 */
  return a - 2.0 * ORC_PI * floor((a + ORC_PI) / (2.0 * ORC_PI));
}
static void normalize_angles(double* g, int dim) { /* docking.cpp:172-179 */
  for (int d = 3; d < dim; ++d) g[d] = wrap(g[d]);
}

typedef struct {
  m3 R;
  v3 ax_phi, ax_theta, ax_alpha;
  v3* tors_world; /* n_rot */
} frame_t;

static m3 rz_cr(double a) { /* rz with correctly rounded trig (grid mode) */
  double s, c;
  cr_sincos(a, &s, &c);
  m3 r = {{{c, -s, 0.0}, {s, c, 0.0}, {0.0, 0.0, 1.0}}};
  return r;
}
static m3 ry_cr(double a) {
  double s, c;
  cr_sincos(a, &s, &c);
  m3 r = {{{c, 0.0, s}, {0.0, 1.0, 0.0}, {-s, 0.0, c}}};
  return r;
}

/* build_frame docking.cpp:78-91; cr: correctly rounded trig (grid mode) */
static void build_frame_x(const mdr_instance* in, const double* g, frame_t* f, int cr) {
  const m3 a = cr ? rz_cr(g[3]) : rz(g[3]), b = cr ? ry_cr(g[4]) : ry(g[4]), c = cr ? rz_cr(g[5]) : rz(g[5]);
  const m3 ab = mm3(&a, &b);
  f->R = mm3(&ab, &c);
  v3 ez = {{0.0, 0.0, 1.0}}, ey = {{0.0, 1.0, 0.0}};
  f->ax_phi = ez;
  f->ax_theta = mv3(&a, ey);
  f->ax_alpha = mv3(&ab, ez);
  for (int k = 0; k < in->n_rot; ++k) f->tors_world[k] = mv3(&f->R, orc_torsion_axis(k));
}
static void build_frame(const mdr_instance* in, const double* g, frame_t* f) { build_frame_x(in, g, f, 0); }

typedef struct {
  double e;
  v3 grad, torque;
} partial_t;

/* evaluate_atoms docking.cpp:95-128 */
static void evaluate_atoms(const mdr_instance* in, const double* g, const frame_t* f, partial_t* out) {
  const v3 t = {{g[0], g[1], g[2]}};
  for (int i = 0; i < in->n_atoms; ++i) {
    const double* at = in->atom_xyzw + 4 * i;
    v3 local = {{at[0], at[1], at[2]}};
    const int k = in->atom_torsion[i];
    if (k >= 0) { /* rotate_axis docking.cpp:57-60 */
      const v3 ax = orc_torsion_axis(k);
      const double ang = g[6 + k], c = cos(ang), s = sin(ang);
      local = add3(add3(scl3(c, local), scl3(s, cross3(ax, local))),
                   scl3((1.0 - c) * dot3(ax, local), ax));
    }
    const v3 world = add3(t, mv3(&f->R, local));
    partial_t p;
    memset(&p, 0, sizeof p);
    for (int j = 0; j < in->n_sites; ++j) {
      const double* s = in->site_xyzdd + 5 * j;
      const v3 sp = {{s[0], s[1], s[2]}};
      const double d0 = s[4];
      const v3 delta = sub3(world, sp);
      const double c2 = 0.5625 * d0 * d0;
      const double u = dot3(delta, delta) + c2;
      const double rho2 = (d0 * d0 + c2) / u;
      const double rho6 = rho2 * rho2 * rho2;
      const double rho12 = rho6 * rho6;
      const double we = at[3] * s[3];
      p.e += we * (rho12 - 2.0 * rho6);
      const double scale = -12.0 * we * (rho12 - rho6) / u;
      p.grad = add3(p.grad, scl3(scale, delta));
    }
    p.torque = cross3(sub3(world, t), p.grad);
    out[i] = p;
  }
}

static float dot3f(const float* a, const float* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static int partition_ok(int partition, int method) {
  const int lo = method == MDR_METHOD_TCU ? 64 : 32;
  return partition >= lo && partition <= 1024 && partition % 32 == 0;
}

/* score docking.cpp:191-233 */
int orc_score(const mdr_instance* in, const double* g, int method, int accum, int partition,
              float* energy, float* grad, float* torque, mdr_sync_stats* st) {
  if (!partition_ok(partition, method)) return MDR_ERR_BLOCK_SIZE;
  frame_t f;
  v3 tw[64];
  if (in->n_rot > 64) return MDR_ERR_SIZE;
  f.tors_world = tw;
  build_frame(in, g, &f);
  partial_t* p = (partial_t*)malloc(sizeof(partial_t) * (size_t)(in->n_atoms > 0 ? in->n_atoms : 1));
  evaluate_atoms(in, g, &f, p);
  float* slots = (float*)calloc((size_t)partition * 7, sizeof(float));
  for (int i = 0; i < in->n_atoms; ++i) { /* round-robin, docking.cpp:202-213 */
    float* s = slots + 7 * (i % partition);
    s[0] += (float)p[i].e;
    s[1] += (float)p[i].grad.v[0];
    s[2] += (float)p[i].grad.v[1];
    s[3] += (float)p[i].grad.v[2];
    s[4] += (float)p[i].torque.v[0];
    s[5] += (float)p[i].torque.v[1];
    s[6] += (float)p[i].torque.v[2];
  }
  float sums[7];
  const int rc = orc_reduce7(slots, partition, method, accum, sums, st);
  free(slots);
  free(p);
  if (rc) return rc;
  *energy = sums[0];
  const float tq[3] = {sums[4], sums[5], sums[6]};
  torque[0] = tq[0]; torque[1] = tq[1]; torque[2] = tq[2];
  grad[0] = sums[1]; grad[1] = sums[2]; grad[2] = sums[3];
  const v3* axes[3] = {&f.ax_phi, &f.ax_theta, &f.ax_alpha};
  for (int a = 0; a < 3; ++a) {
    const float af[3] = {(float)axes[a]->v[0], (float)axes[a]->v[1], (float)axes[a]->v[2]};
    grad[3 + a] = dot3f(af, tq);
  }
  for (int k = 0; k < in->n_rot; ++k) {
    const float af[3] = {(float)tw[k].v[0], (float)tw[k].v[1], (float)tw[k].v[2]};
    grad[6 + k] = dot3f(af, tq);
  }
  return MDR_OK;
}

/* score_reference docking.cpp:235-270 */
int orc_score_reference(const mdr_instance* in, const double* g, double* energy, double* grad,
                        double* torque) {
  frame_t f;
  v3 tw[64];
  if (in->n_rot > 64) return MDR_ERR_SIZE;
  f.tors_world = tw;
  build_frame(in, g, &f);
  partial_t* p = (partial_t*)malloc(sizeof(partial_t) * (size_t)(in->n_atoms > 0 ? in->n_atoms : 1));
  evaluate_atoms(in, g, &f, p);
  v3 gs = {{0, 0, 0}}, ts = {{0, 0, 0}};
  v3 gt[64];
  memset(gt, 0, sizeof gt);
  double e = 0.0;
  for (int i = 0; i < in->n_atoms; ++i) {
    e += p[i].e;
    gs = add3(gs, p[i].grad);
    ts = add3(ts, p[i].torque);
    const int k = in->atom_torsion[i];
    if (k >= 0) gt[k] = add3(gt[k], p[i].torque);
  }
  *energy = e;
  torque[0] = ts.v[0]; torque[1] = ts.v[1]; torque[2] = ts.v[2];
  grad[0] = gs.v[0]; grad[1] = gs.v[1]; grad[2] = gs.v[2];
  grad[3] = dot3(f.ax_phi, ts);
  grad[4] = dot3(f.ax_theta, ts);
  grad[5] = dot3(f.ax_alpha, ts);
  for (int k = 0; k < in->n_rot; ++k) grad[6 + k] = dot3(tw[k], gt[k]);
  free(p);
  return MDR_OK;
}

/* ------------------------------------------------------------ ADADELTA */
/* adadelta_step docking.cpp:281-308 */
int orc_adadelta_step(int dim, double rho, double eps, double* sq_g, double* sq_u, double* geno,
                      const double* grad) {
  for (int i = 0; i < dim; ++i)
    if (!isfinite(grad[i])) return MDR_ERR_NUMERIC_DOMAIN;
  for (int i = 0; i < dim; ++i) {
    const double old_u = sq_u[i];
    sq_g[i] = rho * sq_g[i] + (1.0 - rho) * grad[i] * grad[i];
    const double delta = -sqrt(old_u + eps) / sqrt(sq_g[i] + eps) * grad[i];
    sq_u[i] = rho * old_u + (1.0 - rho) * delta * delta;
    geno[i] = geno[i] + delta;
  }
  normalize_angles(geno, dim);
  return MDR_OK;
}

static void score_stats(int method, int accum, int partition, mdr_sync_stats* st) {
  float zero7[7] = {0};
  (void)zero7;
  zero_stats(st);
  if (method == MDR_METHOD_BASELINE) {
    const uint64_t w = (uint64_t)(partition / 32);
    st->block_syncs = 21;
    st->memory_fences = 14;
    st->shared_mem_bytes = 28;
    st->atomic_adds = 7 * w;
    st->warp_shuffles = 7 * 160 * w;
  } else {
    const uint64_t ch = (uint64_t)((partition + 63) / 64);
    st->block_syncs = 4;
    st->shared_mem_bytes = 2 * ch * 512;
    st->precision_conversions = 2 * (4ull * (uint64_t)partition + (accum == MDR_ACCUM_HALF ? 4u : 256u));
    st->mma_ops = 2 * (ch + 1);
  }
}

static void scale_add_stats(mdr_sync_stats* acc, const mdr_sync_stats* one, uint64_t k) {
  acc->block_syncs += k * one->block_syncs;
  acc->warp_shuffles += k * one->warp_shuffles;
  acc->atomic_adds += k * one->atomic_adds;
  acc->memory_fences += k * one->memory_fences;
  acc->mma_ops += k * one->mma_ops;
  acc->shared_mem_bytes += k * one->shared_mem_bytes;
  acc->precision_conversions += k * one->precision_conversions;
}

/* A scorer: energy + gradient of genotype g (double views of whatever the
 * scoring path returns; the analytic path returns the reference's floats). */
typedef int (*orc_scorefn)(const void* sctx, const double* g, double* e, double* grad);

typedef struct {
  const mdr_instance* in;
  int method, accum, partition;
} analytic_sctx;

static int analytic_score(const void* sctx, const double* g, double* e, double* grad) {
  const analytic_sctx* a = (const analytic_sctx*)sctx;
  float ef, tq[3], gr[64];
  const int rc = orc_score(a->in, g, a->method, a->accum, a->partition, &ef, gr, tq, NULL);
  if (rc) return rc;
  *e = ef;
  for (int d = 0; d < 6 + a->in->n_rot; ++d) grad[d] = gr[d];
  return MDR_OK;
}

/* local_search docking.cpp:310-351 over any scorer */
static int ls_core(orc_scorefn fn, const void* sctx, int dim, const double* start, int max_iters, double tol,
                   double* out_g, double* out_e, int32_t* out_iters, int32_t* out_conv) {
  enum { WINDOW = 16 };
  double* g = (double*)malloc(sizeof(double) * (size_t)dim);
  double* sg = (double*)calloc((size_t)dim, sizeof(double));
  double* su = (double*)calloc((size_t)dim, sizeof(double));
  double* gd = (double*)malloc(sizeof(double) * (size_t)dim);
  double* hist = (double*)malloc(sizeof(double) * (size_t)(max_iters + 1));
  memcpy(g, start, sizeof(double) * (size_t)dim);
  normalize_angles(g, dim);
  double e;
  int rc = fn(sctx, g, &e, gd);
  int iters = 0, conv = 0;
  double best = e;
  memcpy(out_g, g, sizeof(double) * (size_t)dim);
  hist[0] = best;
  for (int it = 1; rc == MDR_OK && it <= max_iters; ++it) {
    rc = orc_adadelta_step(dim, 0.95, 1e-6, sg, su, g, gd);
    if (rc) break;
    rc = fn(sctx, g, &e, gd);
    if (rc) break;
    if (e < best) {
      best = e;
      memcpy(out_g, g, sizeof(double) * (size_t)dim);
    }
    hist[it] = best;
    iters = it;
    if (it >= WINDOW && hist[it - WINDOW] - best < tol) {
      conv = 1;
      break;
    }
  }
  *out_e = best;
  *out_iters = iters;
  *out_conv = conv;
  free(g); free(sg); free(su); free(gd); free(hist);
  return rc;
}

int orc_local_search(const mdr_instance* in, const double* start, int max_iters, double tol,
                     int method, int accum, int partition, double* out_g, double* out_e,
                     int32_t* out_iters, int32_t* out_conv, mdr_sync_stats* st) {
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  const analytic_sctx a = {in, method, accum, partition};
  const int rc = ls_core(analytic_score, &a, 6 + in->n_rot, start, max_iters, tol, out_g, out_e, out_iters,
                         out_conv);
  if (st) {
    mdr_sync_stats one;
    score_stats(method, accum, partition, &one);
    zero_stats(st);
    scale_add_stats(st, &one, (uint64_t)*out_iters + 1);
  }
  return rc;
}

/* random_genotype docking.cpp:360-388 */
static void random_genotype(const mdr_instance* in, orc_rng* r, double* g) {
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX}, md = 0.0;
  for (int j = 0; j < in->n_sites; ++j) {
    const double* s = in->site_xyzdd + 5 * j;
    for (int a = 0; a < 3; ++a) {
      lo[a] = s[a] < lo[a] ? s[a] : lo[a];
      hi[a] = s[a] > hi[a] ? s[a] : hi[a];
    }
    md = s[4] > md ? s[4] : md;
  }
  const double margin = md + 1.0;
  for (int a = 0; a < 3; ++a) g[a] = orc_uniform(r, lo[a] - margin, hi[a] + margin);
  for (int d = 3; d < 6 + in->n_rot; ++d) g[d] = orc_uniform(r, -ORC_PI, ORC_PI);
}

int orc_lga_max_records(const mdr_lga_settings* s) {
  const int off = s->population_size - 1;
  int ls = (int)ceil(s->ls_fraction * off);
  ls = ls < 0 ? 0 : (ls > off ? off : ls);
  return s->generations * ls + 1;
}

/* lga_run docking.cpp:392-517 */
static int lga_core(orc_scorefn fn, const void* sctx, const mdr_instance* in, const mdr_lga_settings* s,
                    uint64_t seed, double* best_e, double* best_g, int64_t* evals_out, int32_t* conv,
                    int32_t* n_records, mdr_ls_record* records, int max_records, int cr) {
  const int dim = 6 + in->n_rot, P = s->population_size;
  orc_rng r = orc_rng_make(seed, "lga");
  double* pop = (double*)malloc(sizeof(double) * (size_t)(P * dim));
  double* nxt = (double*)malloc(sizeof(double) * (size_t)(P * dim));
  double* pe = (double*)malloc(sizeof(double) * (size_t)P);
  double* ne = (double*)malloc(sizeof(double) * (size_t)P);
  int* order = (int*)malloc(sizeof(int) * (size_t)P);
  double* gr = (double*)malloc(sizeof(double) * (size_t)dim);
  double* lsg = (double*)malloc(sizeof(double) * (size_t)dim);
  double e;
  int64_t evals = 0;
  int nrec = 0, rc = MDR_OK;
  double best = DBL_MAX;
  memset(best_g, 0, sizeof(double) * (size_t)dim);
#define TRACK(G, E)                                              \
  do {                                                           \
    if ((E) < best) {                                            \
      best = (E);                                                \
      memcpy(best_g, (G), sizeof(double) * (size_t)dim);         \
    }                                                            \
  } while (0)
#define RECORD(E, IT, CV)                                        \
  do {                                                           \
    if (nrec < max_records) {                                    \
      records[nrec].best_energy = (E);                           \
      records[nrec].iterations = (IT);                           \
      records[nrec].converged = (CV);                            \
    }                                                            \
    ++nrec;                                                      \
  } while (0)
  for (int p = 0; p < P; ++p) {
    random_genotype(in, &r, pop + p * dim);
    rc = fn(sctx, pop + p * dim, &e, gr);
    if (rc) goto done;
    ++evals;
    pe[p] = e;
    TRACK(pop + p * dim, pe[p]);
  }
  {
    const int off = P - 1;
    int ls_count = (int)ceil(s->ls_fraction * off);
    ls_count = ls_count < 0 ? 0 : (ls_count > off ? off : ls_count);
    for (int gen = 0; gen < s->generations; ++gen) {
      if (evals + off + (int64_t)ls_count * (s->ls_max_iters + 1) > s->max_evaluations) break;
      int elite = 0;
      for (int i = 1; i < P; ++i)
        if (pe[i] < pe[elite]) elite = i;
      memcpy(nxt, pop + elite * dim, sizeof(double) * (size_t)dim);
      ne[0] = pe[elite];
      for (int i = 0; i < off; ++i) {
        int ia = (int)orc_index(&r, (uint64_t)P), ja = (int)orc_index(&r, (uint64_t)P);
        const int a = pe[ia] <= pe[ja] ? ia : ja;
        int ib = (int)orc_index(&r, (uint64_t)P), jb = (int)orc_index(&r, (uint64_t)P);
        const int b = pe[ib] <= pe[jb] ? ib : jb;
        double* ch = nxt + (1 + i) * dim;
        for (int d = 0; d < dim; ++d) {
          const double lam = orc_unit(&r);
          ch[d] = lam * pop[a * dim + d] + (1.0 - lam) * pop[b * dim + d];
        }
        for (int d = 0; d < dim; ++d) ch[d] = ch[d] + s->mutation_sigma * (cr ? orc_normal_cr(&r) : orc_normal(&r));
        normalize_angles(ch, dim);
        rc = fn(sctx, ch, &e, gr);
        if (rc) goto done;
        ++evals;
        ne[1 + i] = e;
        TRACK(ch, ne[1 + i]);
      }
      /* stable order of offspring 1..off by (energy, index) */
      for (int i = 0; i < off; ++i) order[i] = 1 + i;
      for (int i = 1; i < off; ++i) { /* insertion sort: ties keep index order */
        const int v = order[i];
        int j = i - 1;
        while (j >= 0 && ne[order[j]] > ne[v]) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = v;
      }
      for (int q = 0; q < ls_count; ++q) {
        const int t = order[q];
        double le;
        int32_t it, cv;
        rc = ls_core(fn, sctx, dim, nxt + t * dim, s->ls_max_iters, s->ls_convergence_tol, lsg, &le, &it,
                     &cv);
        if (rc) goto done;
        evals += it + 1;
        memcpy(nxt + t * dim, lsg, sizeof(double) * (size_t)dim);
        ne[t] = le;
        TRACK(lsg, le);
        RECORD(le, it, cv);
      }
      double* tp = pop; pop = nxt; nxt = tp;
      tp = pe; pe = ne; ne = tp;
    }
  }
  {
    const int64_t remaining = s->max_evaluations - evals;
    if (remaining > 1) {
      const int iters = (int)(s->ls_max_iters < remaining - 1 ? s->ls_max_iters : remaining - 1);
      double le;
      int32_t it, cv;
      memcpy(lsg, best_g, sizeof(double) * (size_t)dim);
      double* start = (double*)malloc(sizeof(double) * (size_t)dim);
      memcpy(start, best_g, sizeof(double) * (size_t)dim);
      rc = ls_core(fn, sctx, dim, start, iters, s->ls_convergence_tol, lsg, &le, &it, &cv);
      free(start);
      if (rc) goto done;
      evals += it + 1;
      TRACK(lsg, le);
      RECORD(le, it, cv);
      *conv = cv;
    } else {
      *conv = 0;
    }
  }
done:
  *best_e = best;
  *evals_out = evals;
  *n_records = nrec;
#undef TRACK
#undef RECORD
  free(pop); free(nxt); free(pe); free(ne); free(order); free(gr); free(lsg);
  return rc;
}

int orc_lga_run(const mdr_instance* in, int method, int accum, const mdr_lga_settings* s,
                uint64_t seed, double* best_e, double* best_g, int64_t* evals_out, int32_t* conv,
                int32_t* n_records, mdr_ls_record* records, int max_records, mdr_sync_stats* st) {
  if (s->population_size < 2) return MDR_ERR_SIZE;
  if (!partition_ok(s->partition, method)) return MDR_ERR_BLOCK_SIZE;
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  const analytic_sctx a = {in, method, accum, s->partition};
  const int rc = lga_core(analytic_score, &a, in, s, seed, best_e, best_g, evals_out, conv, n_records, records,
                          max_records, 0);
  if (st) {
    mdr_sync_stats one;
    score_stats(method, accum, s->partition, &one);
    zero_stats(st);
    scale_add_stats(st, &one, (uint64_t)*evals_out);
  }
  return rc;
}

/* ================================================================ grid mode
 * CPU restatement of the grid-map scoring mode (include/mdr.h "grid-map
 * scoring mode").  There is no reference implementation of
 * this path (SPEC.md:425 puts grid maps out of scope): the formulas are
 * AutoDock-GPU's (trilinear map interpolation, intramolecular pairs, per-
 * rotatable-bond torque) restated on the reference's genotype and torsion
 * model (build_frame docking.cpp:78-91, rotate_axis :57-60, the soft-core
 * well :113-122, the projection :217-231 with exact per-group torque as in
 * score_reference :244-268).  Everything here is double precision; the
 * device path computes in FP32 on FP32 maps (tolerance parity). */

/* receptor map builder (mdr_grid_build) */
int orc_grid_build(const mdr_instance* sites, const mdr_receptor_fields* F, const mdr_grid* shape, float* maps) {
  const int nx = shape->nx, ny = shape->ny, nz = shape->nz, nt = shape->n_types;
  const size_t stride = (size_t)nx * ny * nz;
  const double two_s2 = 2.0 * F->desolv_sigma * F->desolv_sigma;
  for (int iz = 0; iz < nz; ++iz)
    for (int iy = 0; iy < ny; ++iy)
      for (int ix = 0; ix < nx; ++ix) {
        const double P[3] = {shape->origin[0] + shape->spacing * ix, shape->origin[1] + shape->spacing * iy,
                             shape->origin[2] + shape->spacing * iz};
        const size_t o = ((size_t)iz * ny + iy) * nx + ix;
        for (int t = 0; t < nt + 2; ++t) {
          double v = 0.0;
          for (int j = 0; j < sites->n_sites; ++j) {
            const double* s = sites->site_xyzdd + 5 * j;
            const double dx = P[0] - s[0], dy = P[1] - s[1], dz = P[2] - s[2];
            const double r2 = dx * dx + dy * dy + dz * dz;
            if (t < nt) {
              const double d = s[4] * F->type_dist_scale[t];
              const double c2 = 0.5625 * d * d;
              const double u = r2 + c2;
              const double rho2 = (d * d + c2) / u;
              const double rho6 = rho2 * rho2 * rho2;
              const double rho12 = rho6 * rho6;
              v += s[3] * F->type_depth_scale[t] * (rho12 - 2.0 * rho6);
            } else if (t == nt) {
              v += F->elec_scale * F->site_charge[j] / (r2 + 0.5625 * s[4] * s[4]);
            } else {
              v += F->site_volume[j] * exp(-r2 / two_s2);
            }
          }
          maps[(size_t)t * stride + o] = (float)v;
        }
      }
  return MDR_OK;
}

typedef struct {
  const mdr_instance* in;
  const mdr_grid* G;
  const mdr_ligand_params* P;
} grid_sctx;

/* Trilinear interpolation of the atom's combined map c = w*type + q*elec +
 * |q|*desolv at world point p; returns V, dV/dp (clamped axes: 0) and the
 * outside-lattice offset d = p - clamp(p). */
static double grid_sample(const mdr_grid* G, int type, double w, double q, const double p[3], double dvdp[3],
                          double off[3]) {
  const int n[3] = {G->nx, G->ny, G->nz};
  int i0[3];
  double f[3];
  int inside[3];
  for (int a = 0; a < 3; ++a) {
    const double gc = (p[a] - G->origin[a]) / G->spacing;
    double gcc = gc < 0.0 ? 0.0 : gc;
    gcc = gcc > (double)(n[a] - 1) ? (double)(n[a] - 1) : gcc;
    int i = (int)floor(gcc);
    if (i > n[a] - 2) i = n[a] - 2;
    i0[a] = i;
    f[a] = gcc - i;
    inside[a] = gc >= 0.0 && gc <= (double)(n[a] - 1);
    off[a] = G->spacing * (gc - gcc);
  }
  const size_t stride = (size_t)G->nx * G->ny * G->nz;
  const float* mt = G->maps + (size_t)type * stride;
  const float* me = G->maps + (size_t)G->n_types * stride;
  const float* md = me + stride;
  const double aq = fabs(q);
  double c[2][2][2];
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const size_t o = ((size_t)(i0[2] + dz) * G->ny + (i0[1] + dy)) * G->nx + (i0[0] + dx);
        c[dz][dy][dx] = w * mt[o] + q * me[o] + aq * md[o];
      }
  /* x pass, y pass, z pass: value and derivatives w.r.t. the fractions */
  double vx[2][2], gx[2][2];
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy) {
      gx[dz][dy] = c[dz][dy][1] - c[dz][dy][0];
      vx[dz][dy] = c[dz][dy][0] + f[0] * gx[dz][dy];
    }
  double vy[2], gxy[2], gyy[2];
  for (int dz = 0; dz < 2; ++dz) {
    gyy[dz] = vx[dz][1] - vx[dz][0];
    vy[dz] = vx[dz][0] + f[1] * gyy[dz];
    gxy[dz] = gx[dz][0] + f[1] * (gx[dz][1] - gx[dz][0]);
  }
  const double v = vy[0] + f[2] * (vy[1] - vy[0]);
  const double dfx = gxy[0] + f[2] * (gxy[1] - gxy[0]);
  const double dfy = gyy[0] + f[2] * (gyy[1] - gyy[0]);
  const double dfz = vy[1] - vy[0];
  dvdp[0] = inside[0] ? dfx / G->spacing : 0.0;
  dvdp[1] = inside[1] ? dfy / G->spacing : 0.0;
  dvdp[2] = inside[2] ? dfz / G->spacing : 0.0;
  return v;
}

int orc_grid_score(const mdr_instance* in, const mdr_grid* G, const mdr_ligand_params* P, const double* g,
                   double* energy, double* grad, double* torque, double* e_intra_out) {
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  frame_t f;
  v3 tw[64];
  f.tors_world = tw;
  build_frame_x(in, g, &f, 1);  /* grid mode: correctly rounded trig (crmath.h) */
  const int na = in->n_atoms;
  v3* r = (v3*)malloc(sizeof(v3) * (size_t)na);
  v3* F = (v3*)calloc((size_t)na, sizeof(v3));
  v3* Fi = (v3*)calloc((size_t)na, sizeof(v3));
  const v3 t = {{g[0], g[1], g[2]}};
  double e_inter = 0.0, e_intra = 0.0;
  v3 gs = {{0, 0, 0}}, ts = {{0, 0, 0}};
  for (int i = 0; i < na; ++i) {
    const double* at = in->atom_xyzw + 4 * i;
    v3 local = {{at[0], at[1], at[2]}};
    const int k = in->atom_torsion[i];
    if (k >= 0) {
      const v3 ax = orc_torsion_axis(k);
      const double ang = g[6 + k];
      double c, s;
      cr_sincos(ang, &s, &c);
      local = add3(add3(scl3(c, local), scl3(s, cross3(ax, local))), scl3((1.0 - c) * dot3(ax, local), ax));
    }
    r[i] = mv3(&f.R, local);
    const v3 world = add3(t, r[i]);
    double dv[3], off[3];
    const double q = P->atom_charge[i];
    double e = grid_sample(G, P->atom_type[i], at[3], q, world.v, dv, off);
    for (int a = 0; a < 3; ++a) {
      e += MDR_GRID_OUTSIDE_K * off[a] * off[a];
      F[i].v[a] = dv[a] + 2.0 * MDR_GRID_OUTSIDE_K * off[a];
    }
    e_inter += e;
    gs = add3(gs, F[i]);
    ts = add3(ts, cross3(r[i], F[i]));
  }
  if (P->intra) {
    for (int i = 0; i < na; ++i)
      for (int j = i + 1; j < na; ++j) {
        if (in->atom_torsion[i] == in->atom_torsion[j]) continue;
        const v3 d = sub3(r[i], r[j]);
        const double d0 = P->atom_radius[i] + P->atom_radius[j];
        const double c2 = 0.5625 * d0 * d0;
        const double u = dot3(d, d) + c2;
        const double rho2 = (d0 * d0 + c2) / u;
        const double rho6 = rho2 * rho2 * rho2;
        const double rho12 = rho6 * rho6;
        const double eps = sqrt(P->atom_epsilon[i] * P->atom_epsilon[j]);
        const double qq = P->elec_scale * P->atom_charge[i] * P->atom_charge[j];
        e_intra += eps * (rho12 - 2.0 * rho6) + qq / u;
        const double sc = -12.0 * eps * (rho12 - rho6) / u - 2.0 * qq / (u * u);
        Fi[i] = add3(Fi[i], scl3(sc, d));
        Fi[j] = sub3(Fi[j], scl3(sc, d));
      }
  }
  *energy = e_inter + e_intra;
  if (e_intra_out) *e_intra_out = e_intra;
  torque[0] = ts.v[0]; torque[1] = ts.v[1]; torque[2] = ts.v[2];
  grad[0] = gs.v[0]; grad[1] = gs.v[1]; grad[2] = gs.v[2];
  grad[3] = dot3(f.ax_phi, ts);
  grad[4] = dot3(f.ax_theta, ts);
  grad[5] = dot3(f.ax_alpha, ts);
  for (int k = 0; k < in->n_rot; ++k) {
    v3 tk = {{0, 0, 0}};
    for (int i = 0; i < na; ++i)
      if (in->atom_torsion[i] == k) tk = add3(tk, cross3(r[i], add3(F[i], Fi[i])));
    grad[6 + k] = dot3(tw[k], tk);
  }
  free(r); free(F); free(Fi);
  return MDR_OK;
}

static int grid_score_fn(const void* sctx, const double* g, double* e, double* grad) {
  const grid_sctx* c = (const grid_sctx*)sctx;
  double tq[3];
  return orc_grid_score(c->in, c->G, c->P, g, e, grad, tq, NULL);
}

int orc_grid_local_search(const mdr_instance* in, const mdr_grid* G, const mdr_ligand_params* P,
                          const double* start, int max_iters, double tol, double* out_g, double* out_e,
                          int32_t* out_iters, int32_t* out_conv) {
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  const grid_sctx c = {in, G, P};
  return ls_core(grid_score_fn, &c, 6 + in->n_rot, start, max_iters, tol, out_g, out_e, out_iters, out_conv);
}

int orc_grid_lga_run(const mdr_instance* in, const mdr_grid* G, const mdr_ligand_params* P,
                     const mdr_lga_settings* s, uint64_t seed, double* best_e, double* best_g, int64_t* evals_out,
                     int32_t* conv, int32_t* n_records, mdr_ls_record* records, int max_records) {
  if (s->population_size < 2) return MDR_ERR_SIZE;
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  const grid_sctx c = {in, G, P};
  return lga_core(grid_score_fn, &c, in, s, seed, best_e, best_g, evals_out, conv, n_records, records,
                  max_records, 1);
}

/* ======================================================== RMSD clustering
 * SURVEY §8 f3 (north_star: "final best-pose energies and RMSD clustering
 * must match"); not in the reference.  Pose -> atom coordinates is
 * evaluate_atoms' transform (docking.cpp:101-106, FP64, reference order);
 * clustering is AutoDock's: poses in ascending (energy, index) order, each
 * joins the first existing cluster whose seed (its lowest-energy member) is
 * within rmsd < tol, else it seeds a new cluster.  RMSD is over atoms in
 * index correspondence, sqrt(sum |x_i - y_i|^2 / n_atoms). */
int orc_pose_coords(const mdr_instance* in, const double* g, double* xyz) {
  if (in->n_rot > 58) return MDR_ERR_SIZE;
  frame_t f;
  v3 tw[64];
  f.tors_world = tw;
  build_frame(in, g, &f);
  const v3 t = {{g[0], g[1], g[2]}};
  for (int i = 0; i < in->n_atoms; ++i) {
    const double* at = in->atom_xyzw + 4 * i;
    v3 local = {{at[0], at[1], at[2]}};
    const int k = in->atom_torsion[i];
    if (k >= 0) {
      const v3 ax = orc_torsion_axis(k);
      const double ang = g[6 + k], c = cos(ang), s = sin(ang);
      local = add3(add3(scl3(c, local), scl3(s, cross3(ax, local))), scl3((1.0 - c) * dot3(ax, local), ax));
    }
    const v3 w = add3(t, mv3(&f.R, local));
    xyz[3 * i] = w.v[0];
    xyz[3 * i + 1] = w.v[1];
    xyz[3 * i + 2] = w.v[2];
  }
  return MDR_OK;
}

static double rmsd_xyz(const double* a, const double* b, int na) {
  double s = 0.0;
  for (int i = 0; i < 3 * na; ++i) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  return sqrt(s / na);
}

int orc_cluster_poses(const mdr_instance* in, const double* genos, const double* energy, int n, double tol,
                      int32_t* cluster_of, double* rmsd_to_seed, int32_t* n_clusters) {
  const int dim = 6 + in->n_rot, na = in->n_atoms;
  double* xyz = (double*)malloc(sizeof(double) * 3 * (size_t)na * (size_t)(n > 0 ? n : 1));
  int* order = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int* seeds = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int rc = MDR_OK;
  for (int i = 0; i < n && rc == MDR_OK; ++i) rc = orc_pose_coords(in, genos + (size_t)i * dim, xyz + (size_t)3 * na * i);
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) { /* stable insertion sort by energy */
    const int v = order[i];
    int j = i - 1;
    while (j >= 0 && energy[order[j]] > energy[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
  int nc = 0;
  for (int q = 0; q < n && rc == MDR_OK; ++q) {
    const int p = order[q];
    int c = -1;
    double r = 0.0;
    for (int k = 0; k < nc; ++k) {
      const double d = rmsd_xyz(xyz + (size_t)3 * na * p, xyz + (size_t)3 * na * seeds[k], na);
      if (d < tol) {
        c = k;
        r = d;
        break;
      }
    }
    if (c < 0) {
      c = nc;
      seeds[nc++] = p;
      r = 0.0;
    }
    cluster_of[p] = c;
    if (rmsd_to_seed) rmsd_to_seed[p] = r;
  }
  *n_clusters = nc;
  free(xyz); free(order); free(seeds);
  return rc;
}

/* Test support: crmath.h's correctly rounded sin / cos / log on the inputs
 * of the device's crmath probe (mdr_crmath_values): input i is a = -pi + 2 pi
 * u(4i+1), u1 = ((u(4i+2) >> 11) + 1) 2^-53, z = 2 pi u(4i+3), with u(n) the
 * key-0 RngStream draw n.  out[4 i + 0..3] = sin a, cos a, log u1, cos z. */
void orc_cr_values(int64_t i0, int n, double* out) {
  for (int t = 0; t < n; ++t) {
    const uint64_t i = (uint64_t)(i0 + t);
    const double a = -ORC_PI + 2.0 * ORC_PI * ((double)(orc_mix64((4 * i + 1) * 0x9e3779b97f4a7c15ull) >> 11) * 0x1p-53);
    const double u1 = (double)((orc_mix64((4 * i + 2) * 0x9e3779b97f4a7c15ull) >> 11) + 1) * 0x1p-53;
    const double z = 2.0 * ORC_PI * ((double)(orc_mix64((4 * i + 3) * 0x9e3779b97f4a7c15ull) >> 11) * 0x1p-53);
    cr_sincos(a, &out[4 * t], &out[4 * t + 1]);
    out[4 * t + 2] = cr_log(u1);
    out[4 * t + 3] = cr_cos(z);
  }
}
