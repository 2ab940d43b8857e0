// Double-double ("DD", ~106-bit significand) arithmetic for the extended-
// precision convolution path.
//
// A DD value is an unevaluated sum hi + lo with |lo| <= ulp(hi)/2.  The
// building blocks are the error-free transformations two_sum (Knuth) and
// two_prod (one FMA); sums and products renormalise with quick_two_sum.
// These are the published algorithms of Dekker (1971) and of the QD library
// (Hida, Li, Bailey), restated here; relative error of add / mul ~ 2^-104.
//
// The exponent range is that of double: DD widens the precision of the
// convolution (its FFT round-off floor drops from ~1e-16 to ~1e-32 of
// max phi), not the range, so kernel values below ~1e-300 still flush to zero.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace eik {

struct dd {
  double hi, lo;
};
// DD complex, stored as four doubles (32-byte aligned)
struct ddc {
  dd re, im;
};

__host__ __device__ __forceinline__ dd dd_make(double hi, double lo = 0.0) { return dd{hi, lo}; }

__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return dd{s, b - (s - a)};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return dd{s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return dd{p, fma(a, b, -p)};
}

// IEEE-style DD addition (accurate version: both error terms carried)
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, fma(a.lo, b.hi, p.lo));
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
// exact scaling by a power of two
__device__ __forceinline__ dd dd_ldexp(dd a, int e) { return dd{ldexp(a.hi, e), ldexp(a.lo, e)}; }

__device__ __forceinline__ dd dd_div(dd a, dd b) {
  // long division: q1 = a/b, r = a - q1 b, q2 = r/b, r -= q2 b, q3 = r/b
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}

__device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return dd{0.0, 0.0};
  const double x = sqrt(a.hi);
  // one Newton step in DD: x + (a - x^2) / (2x)
  const dd x2 = two_prod(x, x);
  const dd r = dd_sub(a, x2);
  return dd_add(dd{x, 0.0}, dd{r.hi / (2.0 * x), 0.0});
}

// exp(a) for a <= ~709; 0 below the double range.  Argument reduction
// a = k ln2 + r, r scaled by 2^-9, Taylor series to r^11/11!, then nine
// squarings of (1 + s) carried as s -> 2s + s^2.
__device__ __forceinline__ dd dd_exp(dd a) {
  if (a.hi < -745.0) return dd{0.0, 0.0};
  const dd ln2 = dd{6.931471805599452862e-01, 2.319046813846299558e-17};
  const double k = nearbyint(a.hi / ln2.hi);
  dd r = dd_sub(a, dd_mul_d(ln2, k));
  r = dd_ldexp(r, -9);
  // s = r + r^2/2! + ... + r^11/11!  (Horner)
  const double inv_fact[12] = {1.0, 1.0, 0.5, 1.6666666666666666e-01, 4.1666666666666664e-02,
                               8.3333333333333332e-03, 1.3888888888888889e-03, 1.9841269841269841e-04,
                               2.4801587301587302e-05, 2.7557319223985893e-06, 2.7557319223985888e-07,
                               2.5052108385441720e-08};
  // the low parts of 1/n! for n >= 3 matter at the 1e-32 level only through
  // terms already below 2^-104 relative to s (|r| < 7e-4), except 1/6:
  const dd c3 = dd{1.6666666666666666e-01, 9.2518585385429707e-18};
  const dd c4 = dd{4.1666666666666664e-02, 2.3129646346357427e-18};
  const dd c5 = dd{8.3333333333333332e-03, 1.1564823173178714e-19};
  dd p = dd{inv_fact[11], 0.0};
#pragma unroll
  for (int n = 10; n >= 6; --n) p = dd_add(dd_mul(p, r), dd{inv_fact[n], 0.0});
  p = dd_add(dd_mul(p, r), c5);
  p = dd_add(dd_mul(p, r), c4);
  p = dd_add(dd_mul(p, r), c3);
  p = dd_add(dd_mul(p, r), dd{0.5, 0.0});
  p = dd_add(dd_mul(p, r), dd{1.0, 0.0});
  dd s = dd_mul(p, r);  // e^r - 1
#pragma unroll
  for (int i = 0; i < 9; ++i) s = dd_add(dd_ldexp(s, 1), dd_mul(s, s));
  s = dd_add(s, dd{1.0, 0.0});
  const int ki = (int)k;
  // scale in two steps so that 2^k never overflows / flushes on its own
  const int k1 = ki / 2, k2 = ki - k1;
  return dd_ldexp(dd_ldexp(s, k1), k2);
}

// complex helpers
__device__ __forceinline__ ddc ddc_add(ddc a, ddc b) { return ddc{dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
__device__ __forceinline__ ddc ddc_sub(ddc a, ddc b) { return ddc{dd_sub(a.re, b.re), dd_sub(a.im, b.im)}; }
__device__ __forceinline__ ddc ddc_mul(ddc a, ddc b) {
  return ddc{dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im)), dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}
__device__ __forceinline__ ddc ddc_mulc(ddc a, ddc b) {  // a * conj(b)
  return ddc{dd_add(dd_mul(a.re, b.re), dd_mul(a.im, b.im)), dd_sub(dd_mul(a.im, b.re), dd_mul(a.re, b.im))};
}

__device__ __forceinline__ ddc ddc_load(const double4* p) {
  const double4 v = *p;
  return ddc{dd{v.x, v.y}, dd{v.z, v.w}};
}
__device__ __forceinline__ void ddc_store(double4* p, ddc a) { *p = make_double4(a.re.hi, a.re.lo, a.im.hi, a.im.lo); }

}  // namespace eik
