/* sx_log.h -- the one natural-log implementation shared by host and device.
 *
 * Why this exists: quadrant/octant trajectories branch on box entropies
 * (reference: /root/reference/proj/src/quadrant.cpp:18-35 -> histogram.hpp:60
 * std::log). glibc's log and CUDA's libdevice log differ by up to 1-2 ulp, so
 * bit-exact trajectories on host and device need ONE log both sides evaluate
 * identically. sx_log uses only IEEE +,-,*,/ (each correctly rounded on both
 * sides; device code uses the _rn intrinsics so nvcc cannot contract to FMA)
 * and exact bit manipulation. It agrees with glibc log to a few ulp (checked
 * in tests/test_oracle_kats.py), far inside the reference tests' 1e-12.
 *
 * Algorithm: x = m * 2^e with m in (sqrt(1/2), sqrt(2)]; s = (m-1)/(m+1);
 * log(m) = 2 atanh(s) = 2s (1 + z/3 + z^2/5 + ...), z = s^2 (|s| <= 0.1716, so
 * 12 terms reach < 2^-60); log(x) = e*ln2_hi + (e*ln2_lo + log(m)).
 */
#ifndef SALVOX_SX_LOG_H
#define SALVOX_SX_LOG_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SX_HD __host__ __device__ __forceinline__
#else
#define SX_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SX_DMUL(a, b) __dmul_rn((a), (b))
#define SX_DADD(a, b) __dadd_rn((a), (b))
#define SX_DSUB(a, b) __dsub_rn((a), (b))
#define SX_DDIV(a, b) __ddiv_rn((a), (b))
#else
#define SX_DMUL(a, b) ((a) * (b))
#define SX_DADD(a, b) ((a) + (b))
#define SX_DSUB(a, b) ((a) - (b))
#define SX_DDIV(a, b) ((a) / (b))
#endif

SX_HD uint64_t sx_dbits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, sizeof u);
  return u;
#endif
}

SX_HD double sx_dfrombits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, sizeof x);
  return x;
#endif
}

/* Natural log for finite x > 0 (the only inputs: probabilities in (0, 1]).
 * x <= 0 returns -inf / NaN like log. */
SX_HD double sx_log(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -1.0 / 0.0 : (x - x) / (x - x);
  uint64_t u = sx_dbits(x);
  int e = (int)((u >> 52) & 0x7ff);
  if (e == 0x7ff) return x; /* +inf */
  if (e == 0) {              /* subnormal: scale by 2^54 (exact) */
    x = SX_DMUL(x, 18014398509481984.0);
    u = sx_dbits(x);
    e = (int)((u >> 52) & 0x7ff) - 54;
  }
  e -= 1023;
  double m = sx_dfrombits((u & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL); /* [1,2) */
  if (m > 1.4142135623730951) {
    m = SX_DMUL(m, 0.5);
    e += 1;
  }
  const double f = SX_DSUB(m, 1.0); /* exact (Sterbenz) */
  const double s = SX_DDIV(f, SX_DADD(m, 1.0));
  const double z = SX_DMUL(s, s);
  double r = 1.0 / 25.0;
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 23.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 21.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 19.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 17.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 15.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 13.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 11.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 9.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 7.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 5.0);
  r = SX_DADD(SX_DMUL(r, z), 1.0 / 3.0);
  r = SX_DMUL(r, z);                 /* z/3 + z^2/5 + ... */
  const double two_s = SX_DADD(s, s); /* exact */
  const double logm = SX_DADD(two_s, SX_DMUL(two_s, r));
  const double ln2_hi = 6.93147180369123816490e-01; /* 0x3fe62e42fee00000 */
  const double ln2_lo = 1.90821492927058770002e-10; /* 0x3dea39ef35793c76 */
  const double de = (double)e;
  return SX_DADD(SX_DMUL(de, ln2_hi), SX_DADD(SX_DMUL(de, ln2_lo), logm));
}

/* Natural exp, same contract as sx_log (IEEE +,-,*,/, floor and exact bit
 * manipulation only, so host and device agree bit for bit). Used by the
 * Gaussian kernel profile exp(-d/2) (kernel.hpp:17-36). x = k ln2 + r with
 * k = floor(x/ln2 + 1/2) and a Cody-Waite split (k ln2_hi exact), |r| <= 0.35;
 * exp(r) by Horner over 1/n!, n <= 14 (truncation < 2^-60); then * 2^k. Agrees
 * with glibc exp to a few ulp (tests/test_oracle_kats.py). */
SX_HD double sx_ldexp_exact(double v, int k) {
  /* v * 2^k for k in [-1074, 1023]: one or two exact power-of-two scalings */
  if (k < -1022) {
    v = SX_DMUL(v, 2.2250738585072014e-308); /* 2^-1022 */
    k += 1022;
    if (k < -1022) k = -1022;
  }
  return SX_DMUL(v, sx_dfrombits((uint64_t)(k + 1023) << 52));
}

SX_HD double sx_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return 1.0 / 0.0;
  if (x < -745.1332191019412) return 0.0;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double kd = floor(SX_DADD(SX_DMUL(x, 1.4426950408889634074), 0.5));
  const double r = SX_DSUB(SX_DSUB(x, SX_DMUL(kd, ln2_hi)), SX_DMUL(kd, ln2_lo));
  double p = 1.0 / 87178291200.0; /* 1/14! */
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 6227020800.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 479001600.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 39916800.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 3628800.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 362880.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 40320.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 5040.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 720.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 120.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 24.0);
  p = SX_DADD(SX_DMUL(p, r), 1.0 / 6.0);
  p = SX_DADD(SX_DMUL(p, r), 0.5);
  p = SX_DMUL(SX_DMUL(p, r), r);        /* r^2/2 + r^3/6 + ... */
  const double er = SX_DADD(1.0, SX_DADD(r, p));
  return sx_ldexp_exact(er, (int)kd);
}

/* x^y for x >= 0 (the only use: EllipsoidWindow::scale, window.hpp:50-56,
 * det^(1/6) / det2^(1/4) of a bandwidth matrix the device updates). */
SX_HD double sx_pow(double x, double y) {
  if (x == 0.0) return y > 0.0 ? 0.0 : (y == 0.0 ? 1.0 : 1.0 / 0.0);
  if (x == 1.0 || y == 0.0) return 1.0;
  return sx_exp(SX_DMUL(y, sx_log(x)));
}

#endif
