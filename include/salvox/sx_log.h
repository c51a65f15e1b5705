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

#endif
