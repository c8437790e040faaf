// crmath.cuh — correctly rounded (to nearest) double sin / cos / log for the
// reference-parity paths.
//
// The reference evaluates build_frame / rotate_axis (docking.cpp:32-60,
// 78-91) and RngStream::normal (rng.cpp:47-52) with glibc, which is
// effectively correctly rounded on these domains, while CUDA's libdevice
// differs from it by an ulp in 11-17 % of sin / cos calls and 0.3 % of log
// calls (tools/libm_probe.cu).  These versions evaluate the
// function in double-double arithmetic (~2^-77 relative error before the
// final rounding, so the rounded result is the correctly rounded one except
// for inputs within 2^-77 of a rounding midpoint):
//   sin / cos: k = rint(x * 2/pi); r = x - k (C1 + C2 + C3) with a three-part
//              Cody-Waite pi/2 (k C1, k C2 exact), r kept as a double-double;
//              Taylor series in r^2: terms up to r^8 / r^9 in double-double,
//              the tail (to r^27 / r^28) in double; quadrant selection.
//              Domain |x| <= 8 (genotype angles are wrapped to [-pi, pi),
//              Box-Muller angles are in [0, 2 pi)); larger |x| falls back to
//              CUDA's sincos.
//   log:       x = 2^e m, m in [sqrt(1/2), sqrt(2)); log m = 2 atanh(f),
//              f = (m - 1) / (m + 1) as a double-double; series in f^2 with
//              terms up to f^6 in double-double and the tail to f^40 in
//              double; + e ln2 (double-double).  Domain: positive normal x.
// Coefficients are the exact rationals 1/n! and 1/(2k+1) split into
// (hi, lo) doubles (generated with Python fractions; ln2 and pi/2 from
// 80-digit decimals).  Requires --fmad=false (two_sum must not contract).
#pragma once

namespace mdr {
namespace cr {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd add(dd a, dd b) {
  const dd s = two_sum(a.hi, b.hi);
  return fast_two_sum(s.hi, s.lo + (a.lo + b.lo));
}
__device__ __forceinline__ dd add(dd a, double b) {
  const dd s = two_sum(a.hi, b);
  return fast_two_sum(s.hi, s.lo + a.lo);
}
__device__ __forceinline__ dd mul(dd a, dd b) {
  const dd p = two_prod(a.hi, b.hi);
  return fast_two_sum(p.hi, p.lo + (a.hi * b.lo + a.lo * b.hi));
}
__device__ __forceinline__ dd mul(dd a, double b) {
  const dd p = two_prod(a.hi, b);
  return fast_two_sum(p.hi, p.lo + a.lo * b);
}

// (-1)^k / (2k+1)!, k = 0..13
__device__ __forceinline__ dd sin_c(int k) {
  switch (k) {
    case 0: return {0x1.0000000000000p+0, 0.0};
    case 1: return {-0x1.5555555555555p-3, -0x1.5555555555555p-57};
    case 2: return {0x1.1111111111111p-7, 0x1.1111111111111p-63};
    case 3: return {-0x1.a01a01a01a01ap-13, -0x1.a01a01a01a01ap-73};
    default: return {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73};  // k = 4
  }
}
// (-1)^k / (2k)!, k = 0..14
__device__ __forceinline__ dd cos_c(int k) {
  switch (k) {
    case 0: return {0x1.0000000000000p+0, 0.0};
    case 1: return {-0x1.0000000000000p-1, 0.0};
    case 2: return {0x1.5555555555555p-5, 0x1.5555555555555p-59};
    case 3: return {-0x1.6c16c16c16c17p-10, 0x1.f49f49f49f49fp-65};
    default: return {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76};  // k = 4
  }
}

// sin(r), cos(r) for |r| <= ~pi/4 (r a double-double), as double-doubles.
__device__ __forceinline__ void sincos_core(dd r, dd& s_out, dd& c_out) {
  const dd s = mul(r, r);
  const double z = s.hi;
  // tails in double: sin k = 5..13, cos k = 5..14 (Horner in z)
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
  // double-double Horner for k = 4..0
  dd ps = add(sin_c(4), mul(s, ts));
  dd pc = add(cos_c(4), mul(s, tc));
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    ps = add(sin_c(k), mul(s, ps));
    pc = add(cos_c(k), mul(s, pc));
  }
  s_out = mul(r, ps);
  c_out = pc;
}

// Correctly rounded sin and cos of x.
__device__ __forceinline__ void sincos(double x, double* sn, double* cs) {
  if (!(fabs(x) <= 8.0)) {  // outside the reduced domain (or NaN): libdevice
    ::sincos(x, sn, cs);
    return;
  }
  const double k = rint(x * 0x1.45f306dc9c883p-1);  // x * 2/pi
  const double a = x - k * 0x1.921fb54400000p+0;   // exact (k C1 exact, Sterbenz)
  dd r = two_sum(a, -(k * 0x1.0b4611a600000p-34));  // k C2 exact
  r = add(r, -(k * 0x1.3198a2e037073p-69));
  dd s, c;
  sincos_core(r, s, c);
  const int q = ((int)k) & 3;
  const double sv = q == 0 ? s.hi : q == 1 ? c.hi : q == 2 ? -s.hi : -c.hi;
  const double cv = q == 0 ? c.hi : q == 1 ? -s.hi : q == 2 ? -c.hi : s.hi;
  *sn = sv;
  *cs = cv;
}

__device__ __forceinline__ double cos(double x) {
  double s, c;
  sincos(x, &s, &c);
  return c;
}

// 1 / (2k+1), k = 0..3 as double-doubles
__device__ __forceinline__ dd atanh_c(int k) {
  switch (k) {
    case 0: return {1.0, 0.0};
    case 1: return {0x1.5555555555555p-2, 0x1.5555555555555p-56};
    case 2: return {0x1.999999999999ap-3, -0x1.999999999999ap-57};
    default: return {0x1.2492492492492p-3, 0x1.2492492492492p-57};  // k = 3
  }
}

// Correctly rounded natural log of a positive normal x.
__device__ __forceinline__ double log(double x) {
  if (!(x >= 0x1p-1022) || isinf(x)) return ::log(x);
  int e;
  double m = frexp(x, &e);  // [0.5, 1)
  if (m < 0x1.6a09e667f3bcdp-1) {  // sqrt(1/2)
    m *= 2.0;
    e -= 1;
  }
  const double num = m - 1.0;  // exact (Sterbenz)
  const dd den = two_sum(m, 1.0);
  const double q1 = num / den.hi;
  const dd p = two_prod(q1, den.hi);
  const double rem = ((num - p.hi) - p.lo) - q1 * den.lo;
  const dd f = fast_two_sum(q1, rem / den.hi);
  const dd f2 = mul(f, f);
  const double z = f2.hi;
  // tail k = 4..20 of sum_k f^2k / (2k+1), in double
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
  dd sr = add(atanh_c(3), mul(f2, t));
#pragma unroll
  for (int k = 2; k >= 0; --k) sr = add(atanh_c(k), mul(f2, sr));
  dd lm = mul(f, sr);
  lm.hi *= 2.0;  // exact
  lm.lo *= 2.0;
  const double de = (double)e;
  dd el = two_prod(de, 0x1.62e42fefa39efp-1);
  el = fast_two_sum(el.hi, el.lo + de * 0x1.abc9e3b39803fp-56);
  return add(el, lm).hi;
}

}  // namespace cr
}  // namespace mdr
