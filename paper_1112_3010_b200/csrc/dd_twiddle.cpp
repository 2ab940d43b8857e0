// Host-side double-double twiddle table for the extended-precision path:
// W_MAX^j = exp(-2 pi i j / MAX), j in [0, MAX/2), each component correctly
// rounded to a (hi, lo) double pair from binary128 (libquadmath) values.
#include <quadmath.h>

#include <cstdint>

void eik_dd_twiddles_host(int lmax, double* out) {
  const int64_t M = int64_t(1) << lmax;
  for (int64_t j = 0; j < M / 2; ++j) {
    const __float128 a = 2 * M_PIq * (__float128)j / (__float128)M;
    const __float128 c = cosq(a), s = -sinq(a);
    const double ch = (double)c, sh = (double)s;
    out[4 * j + 0] = ch;
    out[4 * j + 1] = (double)(c - (__float128)ch);
    out[4 * j + 2] = sh;
    out[4 * j + 3] = (double)(s - (__float128)sh);
  }
}

// a / b rounded to a (hi, lo) double pair (binary128 quotient)
void eik_dd_div_host(double a, double b, double* hi, double* lo) {
  const __float128 q = (__float128)a / (__float128)b;
  *hi = (double)q;
  *lo = (double)(q - (__float128)*hi);
}
