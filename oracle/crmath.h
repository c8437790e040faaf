/* oracle/crmath.h — TEST INFRASTRUCTURE (the grid-mode checker): correctly
 * rounded double sin / cos / log for the oracle's grid-mode path, the same
 * double-double algorithm and operation order as the device's
 * paper_2410_10447_b200/csrc/crmath.cuh (explicit fma, compiled with
 * -ffp-contract=off), so oracle and device agree bit for bit.
 *
 * Why the grid oracle does not call glibc: grid mode has no reference
 * implementation; the analytic paths follow the reference,
 * which calls glibc sin / cos / log, and glibc is not correctly rounded in
 * ~0.1 % of calls.  For grid mode the oracle and the device
 * share one definition instead: the correctly rounded value, so a
 * double-precision grid docking can be compared run for run.
 *
 *   sin / cos: k = rint(x 2/pi); r = x - k (C1 + C2 + C3) (three-part
 *              Cody-Waite pi/2, r a double-double); Taylor series in r^2 with
 *              the first terms in double-double; quadrant selection.
 *              Domain |x| <= 8 (otherwise glibc).
 *   log:       x = 2^e m, m in [sqrt(1/2), sqrt(2)); log m = 2 atanh(f),
 *              f = (m - 1) / (m + 1) as a double-double; + e ln2. */
#ifndef MDR_ORACLE_CRMATH_H
#define MDR_ORACLE_CRMATH_H

#include <math.h>

typedef struct {
  double hi, lo;
} cr_dd;

static inline cr_dd cr_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  cr_dd r = {s, (a - (s - bb)) + (b - bb)};
  return r;
}
static inline cr_dd cr_fast_two_sum(double a, double b) {
  const double s = a + b;
  cr_dd r = {s, b - (s - a)};
  return r;
}
static inline cr_dd cr_two_prod(double a, double b) {
  const double p = a * b;
  cr_dd r = {p, fma(a, b, -p)};
  return r;
}
static inline cr_dd cr_add(cr_dd a, cr_dd b) {
  const cr_dd s = cr_two_sum(a.hi, b.hi);
  return cr_fast_two_sum(s.hi, s.lo + (a.lo + b.lo));
}
static inline cr_dd cr_add1(cr_dd a, double b) {
  const cr_dd s = cr_two_sum(a.hi, b);
  return cr_fast_two_sum(s.hi, s.lo + a.lo);
}
static inline cr_dd cr_mul(cr_dd a, cr_dd b) {
  const cr_dd p = cr_two_prod(a.hi, b.hi);
  return cr_fast_two_sum(p.hi, p.lo + (a.hi * b.lo + a.lo * b.hi));
}
static inline cr_dd cr_mul1(cr_dd a, double b) {
  const cr_dd p = cr_two_prod(a.hi, b);
  return cr_fast_two_sum(p.hi, p.lo + a.lo * b);
}

static inline cr_dd cr_sin_c(int k) { /* (-1)^k / (2k+1)! */
  static const cr_dd c[5] = {{0x1.0000000000000p+0, 0.0},
                             {-0x1.5555555555555p-3, -0x1.5555555555555p-57},
                             {0x1.1111111111111p-7, 0x1.1111111111111p-63},
                             {-0x1.a01a01a01a01ap-13, -0x1.a01a01a01a01ap-73},
                             {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73}};
  return c[k];
}
static inline cr_dd cr_cos_c(int k) { /* (-1)^k / (2k)! */
  static const cr_dd c[5] = {{0x1.0000000000000p+0, 0.0},
                             {-0x1.0000000000000p-1, 0.0},
                             {0x1.5555555555555p-5, 0x1.5555555555555p-59},
                             {-0x1.6c16c16c16c17p-10, 0x1.f49f49f49f49fp-65},
                             {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76}};
  return c[k];
}

static inline void cr_sincos_core(cr_dd r, cr_dd* s_out, cr_dd* c_out) {
  const cr_dd s = cr_mul(r, r);
  const double z = s.hi;
  double ts = -0x1.d1ab1c2dccea3p-94;
  ts = fma(ts, z, 0x1.3f3ccdd165fa9p-84);
  ts = fma(ts, z, -0x1.761b41316381ap-75);
  ts = fma(ts, z, 0x1.71b8ef6dcf572p-66);
  ts = fma(ts, z, -0x1.2f49b46814157p-57);
  ts = fma(ts, z, 0x1.952c77030ad4ap-49);
  ts = fma(ts, z, -0x1.ae7f3e733b81fp-41);
  ts = fma(ts, z, 0x1.6124613a86d09p-33);
  ts = fma(ts, z, -0x1.ae64567f544e4p-26);
  double tc = 0x1.0a18a2635085dp-98;
  tc = fma(tc, z, -0x1.88e85fc6a4e5ap-89);
  tc = fma(tc, z, 0x1.f2cf01972f578p-80);
  tc = fma(tc, z, -0x1.0ce396db7f853p-70);
  tc = fma(tc, z, 0x1.e542ba4020225p-62);
  tc = fma(tc, z, -0x1.6827863b97d97p-53);
  tc = fma(tc, z, 0x1.ae7f3e733b81fp-45);
  tc = fma(tc, z, -0x1.93974a8c07c9dp-37);
  tc = fma(tc, z, 0x1.1eed8eff8d898p-29);
  tc = fma(tc, z, -0x1.27e4fb7789f5cp-22);
  cr_dd ps = cr_add(cr_sin_c(4), cr_mul1(s, ts));
  cr_dd pc = cr_add(cr_cos_c(4), cr_mul1(s, tc));
  for (int k = 3; k >= 0; --k) {
    ps = cr_add(cr_sin_c(k), cr_mul(s, ps));
    pc = cr_add(cr_cos_c(k), cr_mul(s, pc));
  }
  *s_out = cr_mul(r, ps);
  *c_out = pc;
}

static inline void cr_sincos(double x, double* sn, double* cs) {
  if (!(fabs(x) <= 8.0)) {
    *sn = sin(x);
    *cs = cos(x);
    return;
  }
  const double k = rint(x * 0x1.45f306dc9c883p-1);
  const double a = x - k * 0x1.921fb54400000p+0;
  cr_dd r = cr_two_sum(a, -(k * 0x1.0b4611a600000p-34));
  r = cr_add1(r, -(k * 0x1.3198a2e037073p-69));
  cr_dd s, c;
  cr_sincos_core(r, &s, &c);
  const int q = ((int)k) & 3;
  *sn = q == 0 ? s.hi : q == 1 ? c.hi : q == 2 ? -s.hi : -c.hi;
  *cs = q == 0 ? c.hi : q == 1 ? -s.hi : q == 2 ? -c.hi : s.hi;
}

static inline double cr_cos(double x) {
  double s, c;
  cr_sincos(x, &s, &c);
  return c;
}
static inline double cr_sin(double x) {
  double s, c;
  cr_sincos(x, &s, &c);
  return s;
}

static inline cr_dd cr_atanh_c(int k) { /* 1 / (2k+1) */
  static const cr_dd c[4] = {{1.0, 0.0},
                             {0x1.5555555555555p-2, 0x1.5555555555555p-56},
                             {0x1.999999999999ap-3, -0x1.999999999999ap-57},
                             {0x1.2492492492492p-3, 0x1.2492492492492p-57}};
  return c[k];
}

static inline double cr_log(double x) {
  if (!(x >= 0x1p-1022) || isinf(x)) return log(x);
  int e;
  double m = frexp(x, &e);
  if (m < 0x1.6a09e667f3bcdp-1) {
    m *= 2.0;
    e -= 1;
  }
  const double num = m - 1.0;
  const cr_dd den = cr_two_sum(m, 1.0);
  const double q1 = num / den.hi;
  const cr_dd p = cr_two_prod(q1, den.hi);
  const double rem = ((num - p.hi) - p.lo) - q1 * den.lo;
  const cr_dd f = cr_fast_two_sum(q1, rem / den.hi);
  const cr_dd f2 = cr_mul(f, f);
  const double z = f2.hi;
  double t = 0x1.8f9c18f9c18fap-6;
  t = fma(t, z, 0x1.a41a41a41a41ap-6);
  t = fma(t, z, 0x1.bacf914c1bad0p-6);
  t = fma(t, z, 0x1.d41d41d41d41dp-6);
  t = fma(t, z, 0x1.f07c1f07c1f08p-6);
  t = fma(t, z, 0x1.0842108421084p-5);
  t = fma(t, z, 0x1.1a7b9611a7b96p-5);
  t = fma(t, z, 0x1.2f684bda12f68p-5);
  t = fma(t, z, 0x1.47ae147ae147bp-5);
  t = fma(t, z, 0x1.642c8590b2164p-5);
  t = fma(t, z, 0x1.8618618618618p-5);
  t = fma(t, z, 0x1.af286bca1af28p-5);
  t = fma(t, z, 0x1.e1e1e1e1e1e1ep-5);
  t = fma(t, z, 0x1.1111111111111p-4);
  t = fma(t, z, 0x1.3b13b13b13b14p-4);
  t = fma(t, z, 0x1.745d1745d1746p-4);
  t = fma(t, z, 0x1.c71c71c71c71cp-4);
  cr_dd sr = cr_add(cr_atanh_c(3), cr_mul1(f2, t));
  for (int k = 2; k >= 0; --k) sr = cr_add(cr_atanh_c(k), cr_mul(f2, sr));
  cr_dd lm = cr_mul(f, sr);
  lm.hi *= 2.0;
  lm.lo *= 2.0;
  const double de = (double)e;
  cr_dd el = cr_two_prod(de, 0x1.62e42fefa39efp-1);
  el = cr_fast_two_sum(el.hi, el.lo + de * 0x1.abc9e3b39803fp-56);
  return cr_add(el, lm).hi;
}

#endif
