// host_math.h -- host-side arithmetic that must round exactly like the
// reference (compiled with -ffp-contract=off; see Makefile).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace sx {

// splitmix64 (include/salvox/rng.hpp:11-51)
struct SplitMix {
  uint64_t s;
  bool have_spare = false;
  double spare = 0.0;
  explicit SplitMix(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return double(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return next() % n; }
  double range(double lo, double hi) { return lo + (hi - lo) * unit(); }
  double gaussian() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u1 = unit();
    double u2 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(theta);
    have_spare = true;
    return r * std::cos(theta);
  }
};

// Row-major 3x3 with Eigen's 3x3 inverse / determinant formulas
// (Eigen InverseImpl.h compute_inverse<.,.,3>, Determinant.h determinant_impl<.,3>),
// as used at window.hpp:83 and window.cpp:9.
struct Mat3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
};

inline double cof3(const Mat3& a, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return a.m[i1 * 3 + j1] * a.m[i2 * 3 + j2] - a.m[i1 * 3 + j2] * a.m[i2 * 3 + j1];
}
inline Mat3 eigen_inverse(const Mat3& a) {
  const double c0 = cof3(a, 0, 0), c1 = cof3(a, 1, 0), c2 = cof3(a, 2, 0);
  const double det = (c0 * a.m[0] + c1 * a.m[3]) + c2 * a.m[6];
  const double invdet = 1.0 / det;
  Mat3 r;
  r.m[5] = cof3(a, 2, 1) * invdet;
  r.m[7] = cof3(a, 1, 2) * invdet;
  r.m[8] = cof3(a, 2, 2) * invdet;
  r.m[3] = cof3(a, 0, 1) * invdet;
  r.m[4] = cof3(a, 1, 1) * invdet;
  r.m[6] = cof3(a, 0, 2) * invdet;
  r.m[0] = c0 * invdet;
  r.m[1] = c1 * invdet;
  r.m[2] = c2 * invdet;
  return r;
}
inline double eigen_det(const Mat3& a) {
  const double x = a.m[0] * (a.m[4] * a.m[8] - a.m[5] * a.m[7]);
  const double y = a.m[1] * (a.m[3] * a.m[8] - a.m[5] * a.m[6]);
  const double z = a.m[2] * (a.m[3] * a.m[7] - a.m[4] * a.m[6]);
  return x - y + z;
}

inline Mat3 diag_from_half(double hx, double hy, double hz) {  // window.hpp:34-40
  Mat3 h;
  h.m[0] = hx * hx;
  h.m[4] = hy * hy;
  h.m[8] = hz * hz;
  return h;
}

constexpr double kPi = 3.141592653589793238462643383279502884;  // std::numbers::pi

inline double window_scale(const Mat3& H, bool two_d) {  // window.hpp:50-56
  if (two_d) {
    const double det2 = H.m[0] * H.m[4] - H.m[1] * H.m[3];
    return std::pow(std::max(det2, 0.0), 0.25);
  }
  return std::pow(std::max(eigen_det(H), 0.0), 1.0 / 6.0);
}
inline Mat3 window_scaled_to(const Mat3& H, double s_new, bool two_d) {  // window.hpp:59-66
  const double s = window_scale(H, two_d);
  Mat3 w = H;
  const double f = (s_new / s) * (s_new / s);
  for (double& v : w.m) v *= f;
  if (two_d) w.m[8] = 1.0;
  return w;
}
inline double support_volume(const Mat3& H, bool two_d) {  // window.hpp:69-75
  if (two_d) {
    const double det2 = H.m[0] * H.m[4] - H.m[1] * H.m[3];
    return kPi * std::sqrt(std::max(det2, 0.0));
  }
  return 4.0 / 3.0 * kPi * std::sqrt(std::max(eigen_det(H), 0.0));
}

struct SeedRec {
  double pos[3];
  double scale;
  double half[3] = {0.0, 0.0, 0.0};  // explicit half extents (salvox_seek); 0 -> scale
};

// plan_seeds (src/seeds.cpp:7-45)
inline void plan_seeds(int nx, int ny, int nz, int mode, double spacing, int count,
                       const double* scales, int n_scales, uint64_t rng_seed,
                       std::vector<SeedRec>& out) {
  if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
  if (mode == 0 && spacing <= 0.0) fail(SALVOX_EINVAL, "seed plan: spacing must be > 0");
  if (mode == 1 && count < 1) fail(SALVOX_EINVAL, "seed plan: count must be >= 1");
  if (n_scales < 1 || !scales) fail(SALVOX_EINVAL, "seed plan: no initial scales");
  for (int i = 0; i < n_scales; ++i)
    if (scales[i] <= 0.0) fail(SALVOX_EINVAL, "seed plan: scales must be > 0");
  std::vector<std::array<double, 3>> positions;
  if (mode == 0) {
    const int dims[3] = {nx, ny, nz};
    int counts[3];
    double start[3];
    for (int i = 0; i < 3; ++i) {
      counts[i] = std::max(1, int(std::floor(dims[i] / spacing)));
      start[i] = (dims[i] - (counts[i] - 1) * spacing) / 2.0;
      if (dims[i] == 1) {
        counts[i] = 1;
        start[i] = 0.0;
      }
    }
    auto clampd = [](double v, double hi) { return v < 0.0 ? 0.0 : (hi < v ? hi : v); };
    for (int z = 0; z < counts[2]; ++z)
      for (int y = 0; y < counts[1]; ++y)
        for (int x = 0; x < counts[0]; ++x)
          positions.push_back({clampd(start[0] + x * spacing, double(nx - 1)),
                               clampd(start[1] + y * spacing, double(ny - 1)),
                               clampd(start[2] + z * spacing, double(nz - 1))});
  } else {
    SplitMix rng(rng_seed);
    for (int i = 0; i < count; ++i) {
      const double px = rng.range(0.0, nx - 1);
      const double py = rng.range(0.0, ny - 1);
      const double pz = nz == 1 ? 0.0 : rng.range(0.0, nz - 1);
      positions.push_back({px, py, pz});
    }
  }
  out.clear();
  out.reserve(positions.size() * n_scales);
  for (const auto& p : positions)
    for (int s = 0; s < n_scales; ++s) out.push_back({{p[0], p[1], p[2]}, scales[s]});
}


// One phantom region's rasterisation geometry (phantom.cpp:198-222 region_H /
// region_extents, :252-271 the checks and bounding box), shared by the host
// generator (capi.cu) and the device one (ingest.cu).
struct PhRegion {
  int shape;            // 0 box, 1 ball, 2 ellipsoid
  double c[3], half[3];
  Mat3 Hi;              // H^-1 (Eigen 3x3 inverse); unused for boxes
  int lo[3], hi[3];     // inclusive bounding box
};

inline PhRegion phantom_region(int ri, const int dims[3], const int32_t* shape, const double* center,
                               const double* half_extents, const double* radius,
                               const double* axes) {
  PhRegion g{};
  g.shape = shape[ri];
  const double* c = center + 3 * ri;
  const double* half = half_extents + 3 * ri;
  for (int i = 0; i < 3; ++i) g.c[i] = c[i], g.half[i] = half[i];
  Mat3 H{};
  if (g.shape == 0) {  // half.cwiseProduct(half).asDiagonal()
    H.m[0] = half[0] * half[0];
    H.m[4] = half[1] * half[1];
    H.m[8] = half[2] * half[2];
  } else if (g.shape == 1) {  // Identity() * r * r
    H.m[0] = H.m[4] = H.m[8] = (1.0 * radius[ri]) * radius[ri];
  } else {  // axes * axes^T (Eigen's lazy-product redux: t0 + (t1 + t2))
    const double* a = axes + 9 * ri;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        H.m[i * 3 + j] = a[i * 3] * a[j * 3] + (a[i * 3 + 1] * a[j * 3 + 1] + a[i * 3 + 2] * a[j * 3 + 2]);
  }
  double ext[3];
  for (int i = 0; i < 3; ++i) ext[i] = g.shape == 0 ? half[i] : std::sqrt(std::max(H.m[i * 4], 0.0));
  for (int i = 0; i < 3; ++i)
    if (c[i] - ext[i] < 0.0 || c[i] + ext[i] > dims[i] - 1)
      fail(SALVOX_ERUNTIME, "make_phantom: region extends outside the volume");
  g.Hi = g.shape == 0 ? Mat3{} : eigen_inverse(H);
  for (int i = 0; i < 3; ++i) {
    g.lo[i] = std::max(0, (int)std::floor(c[i] - ext[i]));
    g.hi[i] = std::min(dims[i] - 1, (int)std::ceil(c[i] + ext[i]));
  }
  return g;
}

}  // namespace sx
