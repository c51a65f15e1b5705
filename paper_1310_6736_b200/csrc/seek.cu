// seek.cu -- the seed-grid detector on sm_100a: one warp per seed.
//
// Replaces the per-seed work of detect (/root/reference/proj/src/pipeline.cpp:311-381):
//  * saliency_shift (src/shift.cpp:36-107) with shift_step (:15-34),
//    try_candidate_histogram (src/window.cpp:5-19), pdf_difference (:30-46),
//    inbounds_support_fraction (:54-60), for_each_support_voxel (window.hpp:81-110);
//  * quadrant_seek_one / quadrant_step / box_entropy_bits (src/quadrant.cpp:18-114);
//  * NEW octant ascent: the same algorithm with 8 corner-anchored cubes.
//
// Bit-exactness: every fp64 expression that feeds a trajectory is evaluated with
// the _rn intrinsics in the reference's operation order (no FMA contraction);
// sums that the reference accumulates sequentially (per-bin histogram masses,
// the centroid num/den) are accumulated in the reference's z->y->x order: lanes
// evaluate 32 consecutive bounding-box voxels, then __match_any_sync groups the
// lanes by bin and each group's leader adds its members in lane order; four lanes
// run the num.x/num.y/num.z/den chains over the ballot of support voxels.
// Order-free integer work (support counts, box counts) uses ballots/atomics.
// Logs go through sx_log (include/salvox/sx_log.h), shared with the host oracle.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <map>

#include "../../include/salvox/sx_eig3.h"
#include "../../include/salvox/sx_log.h"
#include "common.cuh"

#ifndef ASCENT_G
#define ASCENT_G 4
#endif
#ifndef CTA_PRODUCERS
#define CTA_PRODUCERS 3
#endif
#include "host_math.h"

namespace sx {

constexpr int kMaxBins = 64;
#ifndef SEEK_KG
#define SEEK_KG 4
#endif
constexpr int kG = SEEK_KG;      // bounding-box chunks of 32 voxels per warp step (ILP)
constexpr int kStep = 32 * kG;
constexpr unsigned kFull = 0xffffffffu;
constexpr double kLn2 = 0.693147180559945309417232121458176568;  // std::numbers::ln2
constexpr double kPiD = 3.141592653589793238462643383279502884;  // std::numbers::pi

struct WinGeom {
  double Hinv[9];
  double ext[3];
  double det_fac;         // 1 / sqrt(max(det H, 1e-300))   (window.cpp:9)
  double support_volume;  // window.hpp:69-75
};

struct ScaleGeom {
  WinGeom main, lo, hi;   // window, scaled_to(s-1), scaled_to(s+1)
  double H[9];
  double pdf_fac;         // s * s / (2.0 * ds)               (window.cpp:45)
  int pdf_ok;             // s - ds >= 1                      (window.cpp:33-34)
  int pad_;
};

struct SeedIn {
  double pos[3];
  int geom;        // shift: ScaleGeom index of the seed's scale
  int seed_index;
  int slot;        // output row (launch order is longest-window-first)
  int vol;         // volume of a batch (bins at binvol + vol * vol_stride)
};

struct SeekParams {
  int nx, ny, nz, bins, method, two_d;
  int max_iters;
  int step_kernel, hist_kernel;
  double min_step, min_frac, eta;
  int n_ascent;
  int ascent_scales[64];
  int geom_of_k[129];   // ascent post-scoring: ScaleGeom index for window half-size k
  const uint8_t* binvol;  // bin + 1, x fastest, pitch nx; batches back to back
  size_t vol_stride;
  const double* q;        // target pmf (bins)
  const ScaleGeom* geoms;
  const SeedIn* seeds;
  int n_seeds;
  salvox_detection* out;
  unsigned long long* visits;
  salvox_ascent_result* ascent_out;  // raw ascent results (salvox_ascent_seek), nullable
  salvox_ascent_state* ascent_state; // the last step's state per slot (salvox_ascent_step), nullable
  int post_score;                    // ascent: score the converged window (detect)
  // ABMSOD (abmsod.hpp:19-40)
  const double* seed_H;              // 9 per output slot (row-major)
  double abm_threshold, abm_lmin, abm_lmax, abm_min_frac;
  int abm_max_iters, abm_kernel;
  salvox_abmsod_iter* abm_trace;     // max_iters records per slot, nullable
  int* abm_trace_n;
  int* err_flag;                     // device: set when a seed's call would throw
  int asc_warp_bytes;                // ascent level tables: dynamic smem per warp
};

struct WarpScratch {
  double h[kMaxBins];
  double p[kMaxBins];     // last normalized candidate histogram
  double w[kMaxBins];     // mean-shift weights / scratch pmf
  double v[kStep];        // compacted per-step values (support voxels, in order)
  double t[3][kStep];     // compacted centroid terms g*x, g*y, g*z
  int bin[kStep];         // compacted bins
  int cntb[kMaxBins];     // per-chunk support count per bin
  int startb[kMaxBins];   // per-chunk start of each bin's run in v
};

struct Box {
  int x0, x1, y0, y1, z0, z1;
};

__device__ __forceinline__ long long box_size(const Box& b) {
  if (b.x0 > b.x1 || b.y0 > b.y1 || b.z0 > b.z1) return 0;
  return (long long)(b.x1 - b.x0 + 1) * (b.y1 - b.y0 + 1) * (b.z1 - b.z0 + 1);
}

// q = floor(n / d) for 0 <= n < 2^22 - 1 and any d >= 1 through one fp32
// multiply: (n + 0.5) / d sits >= 0.5/d from an integer and the two roundings
// move it by < (n + 0.5)/d * 2^-23 < 0.5/d, so truncation is exact.
__device__ __forceinline__ int fdiv_small(int n, float inv_d) {
  return (int)(((float)n + 0.5f) * inv_d);
}

// Linear bounding-box index -> (x, y, z): two divisions by the box's row and
// plane lengths, through fdiv_small while the box holds < 2^22 - 1 voxels (every
// fixed-scale window; ABMSOD windows can grow past it and divide exactly).
struct BoxDiv {
  int Lx, Ly;
  float ix, iy;
  bool fast;
  __device__ __forceinline__ BoxDiv(int lx, int ly, int total)
      : Lx(lx), Ly(ly), ix(1.0f / (float)lx), iy(1.0f / (float)ly),
#ifdef SEEK_INT_DIV  // A/B knob: integer division only
        fast(false) {}
#else
        fast(total < (1 << 22) - 1) {}
#endif
  __device__ __forceinline__ void split(int L, const Box& b, int* x, int* y, int* z) const {
    const int t = fast ? fdiv_small(L, ix) : L / Lx;
    const int zz = fast ? fdiv_small(t, iy) : t / Ly;
    *x = b.x0 + (L - t * Lx);
    *y = b.y0 + (t - zz * Ly);
    *z = b.z0 + zz;
  }
};

// Visits a box in z->y->x order, 32 voxels per step (uniform control flow).
template <class F>
__device__ __forceinline__ void warp_box_iter(const Box& b, int lane, F&& f) {
  const int Lx = b.x1 - b.x0 + 1, Ly = b.y1 - b.y0 + 1, Lz = b.z1 - b.z0 + 1;
  if (Lx <= 0 || Ly <= 0 || Lz <= 0) return;
  const int total = Lx * Ly * Lz;
  const BoxDiv dv(Lx, Ly, total);
  for (int base = 0; base < total; base += 32) {
    const int L = base + lane;
    const bool act = L < total;
    int x = 0, y = 0, z = 0;
    if (act) dv.split(L, b, &x, &y, &z);
    f(act, x, y, z);
  }
}

// kG consecutive 32-voxel chunks per step: lane l gets voxels base + 32 j + l,
// j = 0..kG-1, so the kG independent per-voxel computations overlap (ILP), and
// the step's support list is compacted in z->y->x order.
template <class F>
__device__ __forceinline__ void warp_box_iter_g(const Box& b, int lane, F&& f) {
  const int Lx = b.x1 - b.x0 + 1, Ly = b.y1 - b.y0 + 1, Lz = b.z1 - b.z0 + 1;
  if (Lx <= 0 || Ly <= 0 || Lz <= 0) return;
  const int total = Lx * Ly * Lz;
  const BoxDiv dv(Lx, Ly, total);
  for (int base = 0; base < total; base += kStep) {
    bool act[kG];
    int x[kG], y[kG], z[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int L = base + 32 * j + lane;
      act[j] = L < total;
      dv.split(act[j] ? L : 0, b, &x[j], &y[j], &z[j]);
    }
    f(act, x, y, z);
  }
}

__device__ __forceinline__ Box window_box(const double c[3], const WinGeom& g, int nx, int ny,
                                          int nz) {  // window.hpp:84-89
  Box b;
  b.x0 = max(0, (int)ceil(__dsub_rn(c[0], g.ext[0])));
  b.x1 = min(nx - 1, (int)floor(__dadd_rn(c[0], g.ext[0])));
  b.y0 = max(0, (int)ceil(__dsub_rn(c[1], g.ext[1])));
  b.y1 = min(ny - 1, (int)floor(__dadd_rn(c[1], g.ext[1])));
  b.z0 = max(0, (int)ceil(__dsub_rn(c[2], g.ext[2])));
  b.z1 = min(nz - 1, (int)floor(__dadd_rn(c[2], g.ext[2])));
  return b;
}

// Squared Mahalanobis distance, window.hpp:95-103 operation order.
__device__ __forceinline__ double maha(const WinGeom& g, const double c[3], int x, int y, int z) {
  const double dz = __dsub_rn((double)z, c[2]);
  const double dy = __dsub_rn((double)y, c[1]);
  const double c0 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(g.Hinv[4], dy), dy),
                                        __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.Hinv[5]), dy), dz)),
                              __dmul_rn(__dmul_rn(g.Hinv[8], dz), dz));
  const double c1 = __dmul_rn(2.0, __dadd_rn(__dmul_rn(g.Hinv[1], dy), __dmul_rn(g.Hinv[2], dz)));
  const double dx = __dsub_rn((double)x, c[0]);
  return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(g.Hinv[0], dx), dx), __dmul_rn(c1, dx)), c0);
}

__device__ __forceinline__ double kernel_value(int k, double d) {  // kernel.hpp:17-24
  if (k == 0) return d;
  if (k == 1) return __dsub_rn(1.0, d);
  return sx_exp(__dmul_rn(-0.5, d));  // shared exp (sx_log.h): bit-exact vs the oracle
}
__device__ __forceinline__ double kernel_step_weight(int k, double d) {  // kernel.hpp:29-36
  if (k == 2) return __dmul_rn(0.5, sx_exp(__dmul_rn(-0.5, d)));
  return 1.0;
}

// Sequential fp64 sums in the reference's order (acc += src[0], src[1], ...):
// the terms are staged W at a time in registers so their shared-memory loads
// (and, for the moment, the products) are in flight together and only the
// dependent DADD chain remains serial. W = 16 for the CTA engine's consumer
// warp (C3 10.8 -> 10.1 ms); the warp engine keeps its unroll-4 loops (its
// 80-register occupancy variant got slower with the staging: 72 -> 74-77 ms).
template <int W>
__device__ __forceinline__ double chain_sum(double acc, const double* src, int n) {
  int k = 0;
  for (; k + W <= n; k += W) {
    double t[W];
#pragma unroll
    for (int u = 0; u < W; ++u) t[u] = src[k + u];
#pragma unroll
    for (int u = 0; u < W; ++u) acc = __dadd_rn(acc, t[u]);
  }
  for (; k < n; ++k) acc = __dadd_rn(acc, src[k]);
  return acc;
}

// acc += (v[k] * di[k]) * dj[k] in order (the bandwidth moment's outer products)
template <int W>
__device__ __forceinline__ double chain_sum_mom(double acc, const double* v, const double* di,
                                                const double* dj, int n) {
  int k = 0;
  for (; k + W <= n; k += W) {
    double t[W];
#pragma unroll
    for (int u = 0; u < W; ++u) t[u] = __dmul_rn(__dmul_rn(v[k + u], di[k + u]), dj[k + u]);
#pragma unroll
    for (int u = 0; u < W; ++u) acc = __dadd_rn(acc, t[u]);
  }
  for (; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(v[k], di[k]), dj[k]));
  return acc;
}

__device__ __forceinline__ int bin_at(const SeekParams& P, const uint8_t* vb, int x, int y, int z) {
  return (int)__ldg(vb + ((size_t)z * P.ny + y) * P.nx + x) - 1;
}

// try_candidate_histogram (window.cpp:5-19): sequential per-bin fp64 masses in
// support order, normalized into s.p. Returns ok; *support, *visited.
// Per 128-voxel chunk the support voxels are counting-sorted by bin, stably
// (__match_any_sync groups equal bins of a 32-voxel group; rank = lanes below
// in the group + the bin's count from earlier groups), so bin b's masses sit
// contiguously in z->y->x order. Lane l owns bins l and l+32 and adds only its
// own run: the dependent fp64 chain is max_b count_b long per chunk instead of
// the chunk's whole support.
// Not inlined: ONE copy of these loops serves every call site (inlined copies
// overflowed the instruction cache: "no instruction" was the top stall).
struct HistRes {
  long long visited;
  unsigned support;
  int ok;
};

__device__ __noinline__ HistRes warp_candidate_hist_impl(const uint8_t* vb, int nx, int ny, int nz,
                                                         int M, WarpScratch* sp, double c0,
                                                         double c1, double c2, const WinGeom* gp,
                                                         int kernel) {
  WarpScratch& s = *sp;
  const WinGeom& g = *gp;
  const int lane = threadIdx.x & 31;
  const double c[3] = {c0, c1, c2};
  const Box bb = window_box(c, g, nx, ny, nz);
  HistRes res{box_size(bb), 0u, 0};
  unsigned support = 0;
  double a0 = 0.0, a1 = 0.0;  // bins lane, lane + 32
  const unsigned lt = (1u << lane) - 1u;
  warp_box_iter_g(bb, lane, [&](const bool* act, const int* x, const int* y, const int* z) {
    bool in[kG];
    int bin[kG];
    double val[kG];
    uint8_t raw[kG];  // bins fetched before the Mahalanobis tests (latency overlap)
#pragma unroll
    for (int j = 0; j < kG; ++j)
      raw[j] = act[j] ? __ldg(vb + ((size_t)z[j] * ny + y[j]) * nx + x[j]) : (uint8_t)0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      in[j] = false;
      bin[j] = 0;
      val[j] = 0.0;
      if (act[j]) {
        const double d = maha(g, c, x[j], y[j], z[j]);
        in[j] = d <= 1.0;
        if (in[j]) {
          bin[j] = (int)raw[j] - 1;
          val[j] = __dmul_rn(g.det_fac, kernel_value(kernel, d));
        }
      }
    }
    s.cntb[lane] = 0;
    s.cntb[lane + 32] = 0;
    __syncwarp();
    int rank[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {  // stable per-bin ranks, group by group
      const unsigned peers = __match_any_sync(kFull, in[j] ? bin[j] : -1);
      int base = 0;
      if (in[j]) base = s.cntb[bin[j]];
      rank[j] = base + __popc(peers & lt);
      __syncwarp();
      if (in[j] && (peers & lt) == 0u) s.cntb[bin[j]] = base + __popc(peers);
      __syncwarp();
    }
    const int c0 = s.cntb[lane], c1 = s.cntb[lane + 32];
    int i0 = c0, i1 = c1;  // inclusive scans over bins 0..31 and 32..63
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(kFull, i0, o), t1 = __shfl_up_sync(kFull, i1, o);
      if (lane >= o) i0 += t0, i1 += t1;
    }
    const int tot0 = __shfl_sync(kFull, i0, 31);
    const int st0 = i0 - c0, st1 = tot0 + i1 - c1;
    s.startb[lane] = st0;
    s.startb[lane + 32] = st1;
    support += (unsigned)(tot0 + __shfl_sync(kFull, i1, 31));
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kG; ++j)
      if (in[j]) s.v[s.startb[bin[j]] + rank[j]] = val[j];
    __syncwarp();
    for (int k = 0; k < c0; ++k) a0 = __dadd_rn(a0, s.v[st0 + k]);
    if (M > 32)
      for (int k = 0; k < c1; ++k) a1 = __dadd_rn(a1, s.v[st1 + k]);
    __syncwarp();
  });
  if (lane < M) s.h[lane] = a0;
  if (lane + 32 < M) s.h[lane + 32] = a1;
  __syncwarp();
  double mass = 0.0;
  if (lane == 0)
    for (int b = 0; b < M; ++b) mass = __dadd_rn(mass, s.h[b]);  // Histogram::mass
  mass = __shfl_sync(kFull, mass, 0);
  res.support = support;
  if (support == 0 || mass <= 0.0) return res;
  for (int b = lane; b < M; b += 32) s.p[b] = __ddiv_rn(s.h[b], mass);
  __syncwarp();
  res.ok = 1;
  return res;
}

__device__ __forceinline__ bool warp_candidate_hist(const SeekParams& P, const uint8_t* vb,
                                                    WarpScratch& s, const double c[3],
                                                    const WinGeom& g, int kernel, int lane,
                                                    unsigned* support_out, long long* visited) {
  (void)lane;
  const HistRes r =
      warp_candidate_hist_impl(vb, P.nx, P.ny, P.nz, P.bins, &s, c[0], c[1], c[2], &g, kernel);
  *support_out = r.support;
  *visited = r.visited;
  return r.ok != 0;
}

// entropy_bits (histogram.hpp:56-67) of pmf p, sequential in bin order.
__device__ __noinline__ double warp_entropy_bits(const double* p, int M, int lane, double* tmp) {
  for (int b = lane; b < M; b += 32) tmp[b] = p[b] > 0.0 ? __dmul_rn(p[b], sx_log(p[b])) : 0.0;
  __syncwarp();
  double e = 0.0;
  if (lane == 0) {
    for (int b = 0; b < M; ++b)
      if (p[b] > 0.0) e = __dsub_rn(e, tmp[b]);
    e = __ddiv_rn(e < 0.0 ? 0.0 : e, kLn2);
  }
  __syncwarp();
  return __shfl_sync(kFull, e, 0);
}

__device__ __forceinline__ double dclamp(double v, double hi) {
  return v < 0.0 ? 0.0 : (hi < v ? hi : v);
}

// Final scores shared by shift and the ascent methods: entropy of p_score
// (Epanechnikov), Bhattacharyya of p_step vs q, pdf_difference (identity).
// p_step must already be in s.p. Returns false if a histogram is degenerate.
__device__ bool warp_final_scores(const SeekParams& P, const uint8_t* vb, WarpScratch& s, const double c[3],
                                  const ScaleGeom& sg, int lane, bool have_pstep,
                                  salvox_detection& d, unsigned long long& visits,
                                  bool pstep_from_shift) {
  const int M = P.bins;
  unsigned sup;
  long long vis;
  bool ok_step = have_pstep;
  // bhattacharyya(p_step, q) before s.p is overwritten
  double rho = 0.0;
  if (ok_step && lane == 0) {
    for (int b = 0; b < M; ++b) rho = __dadd_rn(rho, __dsqrt_rn(__dmul_rn(s.p[b], P.q[b])));
    rho = rho < 1.0 ? rho : 1.0;
  }
  rho = __shfl_sync(kFull, rho, 0);
  const bool ok_score = warp_candidate_hist(P, vb, s, c, sg.main, 1, lane, &sup, &vis);
  visits += (unsigned long long)vis;
  if (pstep_from_shift) visits += (unsigned long long)vis;  // reference recomputes p_step
  bool ok = true;
  if (ok_score && ok_step) {
    d.entropy_bits = warp_entropy_bits(s.p, M, lane, s.w);
    d.bhattacharyya = rho;
  } else {
    ok = false;
  }
  // pdf_difference: both flanks are evaluated before the check (window.cpp:37-39)
  double pdf = 0.0;
  if (sg.pdf_ok) {
    const bool ok_lo = warp_candidate_hist(P, vb, s, c, sg.lo, 0, lane, &sup, &vis);
    visits += (unsigned long long)vis;
    for (int b = lane; b < M; b += 32) s.w[b] = s.p[b];
    __syncwarp();
    const bool ok_hi = warp_candidate_hist(P, vb, s, c, sg.hi, 0, lane, &sup, &vis);
    visits += (unsigned long long)vis;
    if (ok_lo && ok_hi) {
      double l1 = 0.0;
      if (lane == 0) {
        for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(s.p[b], s.w[b])));
        pdf = __dmul_rn(sg.pdf_fac, l1);
      }
      pdf = __shfl_sync(kFull, pdf, 0);
    }
  }
  d.pdf_diff = pdf;
  return ok;
}

// Centroid pass (shift.cpp:25-30, abmsod.cpp:85-90): g = step_w(d) * w[bin];
// lanes 0..3 run num.x / num.y / num.z / den in support order. Not inlined (one
// copy for every caller). Returns the box visits.
struct CentRes {
  double num[3], den;
  long long visited;
};

__device__ __noinline__ CentRes warp_centroid_impl(const uint8_t* vb, int nx, int ny, int nz,
                                                   WarpScratch* sp, double c0, double c1,
                                                   double c2, const WinGeom* gp, int step_kernel) {
  WarpScratch& s = *sp;
  const WinGeom& wg = *gp;
  const int lane = threadIdx.x & 31;
  const double c[3] = {c0, c1, c2};
  double acc = 0.0;
  const Box bb = window_box(c, wg, nx, ny, nz);
  warp_box_iter_g(bb, lane, [&](const bool* act, const int* x, const int* y, const int* z) {
    bool in[kG];
    double g[kG];
    uint8_t raw[kG];  // bins fetched before the Mahalanobis tests (latency overlap)
#pragma unroll
    for (int j = 0; j < kG; ++j)
      raw[j] = act[j] ? __ldg(vb + ((size_t)z[j] * ny + y[j]) * nx + x[j]) : (uint8_t)0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      in[j] = false;
      g[j] = 0.0;
      if (act[j]) {
        const double dd = maha(wg, c, x[j], y[j], z[j]);
        in[j] = dd <= 1.0;
        if (in[j]) {
          const int b = (int)raw[j] - 1;
          g[j] = __dmul_rn(kernel_step_weight(step_kernel, dd), s.w[b]);
        }
      }
    }
    int off = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const unsigned m0 = __ballot_sync(kFull, in[j]);
      if (in[j]) {  // Eigen: num += g * Vector3d(sx, sy, sz) -> per-component products
        const int r = off + __popc(m0 & ((1u << lane) - 1u));
        s.v[r] = g[j];
        s.t[0][r] = __dmul_rn(g[j], (double)x[j]);
        s.t[1][r] = __dmul_rn(g[j], (double)y[j]);
        s.t[2][r] = __dmul_rn(g[j], (double)z[j]);
      }
      off += __popc(m0);
    }
    __syncwarp();
    if (lane < 4) {
      const double* src = lane == 3 ? s.v : s.t[lane];
#pragma unroll 4
      for (int k = 0; k < off; ++k) acc = __dadd_rn(acc, src[k]);
    }
    __syncwarp();
  });
  CentRes r;
  r.num[0] = __shfl_sync(kFull, acc, 0);
  r.num[1] = __shfl_sync(kFull, acc, 1);
  r.num[2] = __shfl_sync(kFull, acc, 2);
  r.den = __shfl_sync(kFull, acc, 3);
  r.visited = box_size(bb);
  return r;
}

__device__ __forceinline__ long long warp_centroid(const SeekParams& P, const uint8_t* vb,
                                                   WarpScratch& s, const double c[3],
                                                   const WinGeom& wg, int step_kernel, int lane,
                                                   double num[3], double* den_out) {
  (void)lane;
  const CentRes r = warp_centroid_impl(vb, P.nx, P.ny, P.nz, &s, c[0], c[1], c[2], &wg, step_kernel);
  num[0] = r.num[0], num[1] = r.num[1], num[2] = r.num[2];
  *den_out = r.den;
  return r.visited;
}

// ------------------------------------------------------------------- shift
// warps (seeds) per block; scratch is ~6.3 KB per warp. Small blocks free their
// slot as soon as their own trajectories end (lengths vary widely per seed).
// MINB > 1 caps registers for occupancy (many seeds: throughput-bound); MINB = 1
// keeps every register for the per-warp chain speed (few, long trajectories).
template <int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) shift_kernel(const SeekParams P) {
  __shared__ WarpScratch scratch[NW];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int seed = blockIdx.x * NW + wid;
  if (seed >= P.n_seeds) return;
  WarpScratch& s = scratch[wid];
  const SeedIn si = P.seeds[seed];
  const uint8_t* vb = P.binvol + (size_t)si.vol * P.vol_stride;
  const ScaleGeom& sg = P.geoms[si.geom];
  const int M = P.bins;
  const double lim[3] = {(double)(P.nx - 1), (double)(P.ny - 1), (double)(P.nz - 1)};
  salvox_detection d;
  memset(&d, 0, sizeof d);
  d.seed_index = si.seed_index;
  for (int i = 0; i < 9; ++i) d.H[i] = sg.H[i];
  unsigned long long visits = 0;
  double c[3] = {dclamp(si.pos[0], lim[0]), dclamp(si.pos[1], lim[1]), dclamp(si.pos[2], lim[2])};

  unsigned support;
  long long vis;
  bool ok = warp_candidate_hist(P, vb, s, c, sg.main, P.hist_kernel, lane, &support, &vis);
  // inbounds_support_fraction at the clamped seed (shift.cpp:53-57)
  auto frac_bad = [&](unsigned sup) {
    if (sg.main.support_volume <= 0.0) return 0.0 < P.min_frac;
    double f = __ddiv_rn((double)sup, sg.main.support_volume);
    f = f < 1.0 ? f : 1.0;
    return f < P.min_frac;
  };
  bool degenerate = frac_bad(support);
  if (!degenerate) {
    for (int it = 0; it < P.max_iters; ++it) {
      d.iterations = it + 1;
      visits += (unsigned long long)vis;  // shift_step's histogram pass
      if (!ok) {
        degenerate = true;
        break;
      }
      // weights sqrt(q_b / max(p_b, 1e-6)) (histogram.hpp:107-113)
      for (int b = lane; b < M; b += 32) {
        const double pb = s.p[b] > 1e-6 ? s.p[b] : 1e-6;
        s.w[b] = __dsqrt_rn(__ddiv_rn(P.q[b], pb));
      }
      __syncwarp();
      // centroid pass (shift.cpp:25-30): support voxels compacted per chunk; lanes
      // 0..3 run the num.x / num.y / num.z / den chains in z->y->x order
      double num[3], den;
      visits += (unsigned long long)warp_centroid(P, vb, s, c, sg.main, P.step_kernel, lane, num,
                                                  &den);
      const double nx_ = num[0], ny_ = num[1], nz_ = num[2];
      if (den <= 0.0) {
        degenerate = true;
        break;
      }
      const double moved[3] = {__ddiv_rn(nx_, den), __ddiv_rn(ny_, den), __ddiv_rn(nz_, den)};
      double cl[3], df[3];
      for (int i = 0; i < 3; ++i) cl[i] = dclamp(moved[i], lim[i]);
      for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(cl[i], moved[i]);
      if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                               __dmul_rn(df[2], df[2]))) > 0.0)
        d.flags |= SALVOX_FLAG_BOUNDARY_CLAMPED;
      for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(cl[i], c[i]);
      const double step = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                                               __dmul_rn(df[2], df[2])));
      c[0] = cl[0];
      c[1] = cl[1];
      c[2] = cl[2];
      // histogram at the new centre: its support count is the in-bounds
      // fraction check (shift.cpp:75) and its pmf the next step's p.
      ok = warp_candidate_hist(P, vb, s, c, sg.main, P.hist_kernel, lane, &support, &vis);
      if (frac_bad(support)) {
        degenerate = true;
        break;
      }
      if (step < P.min_step) {
        d.flags |= SALVOX_FLAG_CONVERGED;
        break;
      }
    }
  }
  if (degenerate) d.flags |= SALVOX_FLAG_DEGENERATE;
  d.center[0] = c[0];
  d.center[1] = c[1];
  d.center[2] = c[2];
  if (!degenerate) {
    if (!warp_final_scores(P, vb, s, c, sg, lane, ok, d, visits, true))
      d.flags |= SALVOX_FLAG_DEGENERATE;
  }
  if (lane == 0) {
    P.out[si.slot] = d;
    P.visits[si.slot] = visits;
  }
}

// --------------------------------------------- CTA engine (latency mode)
// When few seeds run (a long trajectory per SM), one seed per CTA: NP
// producer warps compute whole 128-voxel chunks (window test, bins, weights,
// the stable per-bin sort or the ordered compaction) into a double-buffered
// ring in shared memory while the consumer warp 0 runs the ordered fp64 chains
// of the previous chunks. Chunk order and every operation are those of the
// warp engine, so results are bit-identical; only the latency overlaps.
enum { PASS_HIST = 0, PASS_CENT = 1, PASS_MOM = 2 };

struct CtaSlot {
  double v[kStep];
  double t[3][kStep];
  int cnt[kMaxBins];
  int start[kMaxBins];
  int n;
};

template <int NP>
struct CtaShared {
  CtaSlot slot[2][NP];
  double h[kMaxBins], p[kMaxBins], w[kMaxBins], tmp[kMaxBins];
  double res[16];
  int ires[4];
  WinGeom g;              // ABMSOD: the current window's geometry
  double Hc[9], Hn[9];    // ABMSOD: current / updated bandwidth
};

struct PassIn {
  const uint8_t* vb;
  int nx, ny, nz, M;
  double c[3];
  const WinGeom* g;
  int kernel;
};

template <int MODE>
__device__ __forceinline__ void cta_produce(const PassIn& in, const Box& bb, int Lx, int Ly,
                                            int total, int base, CtaSlot& sl, const double* w,
                                            int lane) {
  const WinGeom& g = *in.g;
  bool inb[kG];
  int bin[kG], xs[kG], ys[kG], zs[kG];
  double val[kG];
  uint8_t raw[kG];
  // the bin of every voxel of the chunk is fetched first (the bounding box lies
  // inside the volume, so the loads are always valid): their L2 latency then
  // overlaps the Mahalanobis tests instead of following them
  // integer division here: the fp32-reciprocal form (BoxDiv) measured 2% slower in
  // this engine (C3 10.48 vs 10.24 ms) while it helps the warp engine (C1 shift)
#pragma unroll
  for (int j = 0; j < kG; ++j) {
    const int L = base + 32 * j + lane;
    const int Lc = L < total ? L : 0;
    const int t = Lc / Lx;
    xs[j] = bb.x0 + (Lc - t * Lx);
    const int zz = t / Ly;
    ys[j] = bb.y0 + (t - zz * Ly);
    zs[j] = bb.z0 + zz;
    raw[j] = __ldg(in.vb + ((size_t)zs[j] * in.ny + ys[j]) * in.nx + xs[j]);
  }
#pragma unroll
  for (int j = 0; j < kG; ++j) {
    const bool act = base + 32 * j + lane < total;
    inb[j] = false;
    bin[j] = 0;
    val[j] = 0.0;
    if (act) {
      const double d = maha(g, in.c, xs[j], ys[j], zs[j]);
      inb[j] = d <= 1.0;
      if (inb[j]) {
        bin[j] = (int)raw[j] - 1;
        if (MODE == PASS_HIST) val[j] = __dmul_rn(g.det_fac, kernel_value(in.kernel, d));
        if (MODE == PASS_CENT) val[j] = __dmul_rn(kernel_step_weight(in.kernel, d), w[bin[j]]);
        if (MODE == PASS_MOM) val[j] = w[bin[j]];
      }
    }
  }
  const unsigned lt = (1u << lane) - 1u;
  if (MODE == PASS_HIST) {  // stable counting sort by bin (as warp_candidate_hist_impl)
    sl.cnt[lane] = 0;
    sl.cnt[lane + 32] = 0;
    __syncwarp();
    int rank[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const unsigned peers = __match_any_sync(kFull, inb[j] ? bin[j] : -1);
      int b0 = 0;
      if (inb[j]) b0 = sl.cnt[bin[j]];
      rank[j] = b0 + __popc(peers & lt);
      __syncwarp();
      if (inb[j] && (peers & lt) == 0u) sl.cnt[bin[j]] = b0 + __popc(peers);
      __syncwarp();
    }
    const int c0 = sl.cnt[lane], c1 = sl.cnt[lane + 32];
    int i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(kFull, i0, o), t1 = __shfl_up_sync(kFull, i1, o);
      if (lane >= o) i0 += t0, i1 += t1;
    }
    const int tot0 = __shfl_sync(kFull, i0, 31);
    sl.start[lane] = i0 - c0;
    sl.start[lane + 32] = tot0 + i1 - c1;
    const int tot1 = __shfl_sync(kFull, i1, 31);
    if (lane == 0) sl.n = tot0 + tot1;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kG; ++j)
      if (inb[j]) sl.v[sl.start[bin[j]] + rank[j]] = val[j];
  } else {  // ordered compaction
    int off = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const unsigned m0 = __ballot_sync(kFull, inb[j]);
      if (inb[j]) {
        const int r = off + __popc(m0 & lt);
        sl.v[r] = val[j];
        if (MODE == PASS_CENT) {  // num += g * Vector3d(sx, sy, sz)
          sl.t[0][r] = __dmul_rn(val[j], (double)xs[j]);
          sl.t[1][r] = __dmul_rn(val[j], (double)ys[j]);
          sl.t[2][r] = __dmul_rn(val[j], (double)zs[j]);
        } else {  // d = x_new - s
          sl.t[0][r] = __dsub_rn(in.c[0], (double)xs[j]);
          sl.t[1][r] = __dsub_rn(in.c[1], (double)ys[j]);
          sl.t[2][r] = __dsub_rn(in.c[2], (double)zs[j]);
        }
      }
      off += __popc(m0);
    }
    if (lane == 0) sl.n = off;
  }
}

template <int MODE>
__device__ __forceinline__ void cta_consume_once(const CtaSlot& sl, int M, int lane, double& a0,
                                                 double& a1, unsigned& support);

template <int MODE>
__device__ __forceinline__ void cta_consume(const CtaSlot& sl, int M, int lane, double& a0,
                                            double& a1, unsigned& support) {
#ifdef SEEK_SKIP_CHAINS  // profiling knob: no ordered fp64 chains (results wrong)
  a0 = __dadd_rn(a0, (double)sl.n);
  if (MODE == PASS_HIST) support += (unsigned)sl.n;
  return;
#endif
#ifdef SEEK_DOUBLE_CHAINS  // profiling knob: every chain twice (same results, 2x consumer latency)
  {
    double x0 = a0, x1 = a1;
    unsigned sp = 0;
    cta_consume_once<MODE>(sl, M, lane, x0, x1, sp);
    // a fake dependence: the real chain starts only after the copy finished
    asm volatile("" : "+d"(a0), "+d"(a1), "+r"(support) : "d"(x0), "d"(x1), "r"(sp));
  }
#endif
  cta_consume_once<MODE>(sl, M, lane, a0, a1, support);
}

template <int MODE>
__device__ __forceinline__ void cta_consume_once(const CtaSlot& sl, int M, int lane, double& a0,
                                                 double& a1, unsigned& support) {
  if (MODE == PASS_HIST) {
    const int c0 = sl.cnt[lane], s0 = sl.start[lane];
    for (int k = 0; k < c0; ++k) a0 = __dadd_rn(a0, sl.v[s0 + k]);
    if (M > 32) {
      const int c1 = sl.cnt[lane + 32], s1 = sl.start[lane + 32];
      for (int k = 0; k < c1; ++k) a1 = __dadd_rn(a1, sl.v[s1 + k]);
    }
    support += (unsigned)sl.n;
  } else if (MODE == PASS_CENT) {
    if (lane < 4) a0 = chain_sum<16>(a0, lane == 3 ? sl.v : sl.t[lane], sl.n);
  } else {
    const int n = sl.n;
    if (lane < 9) a0 = chain_sum_mom<16>(a0, sl.v, sl.t[lane / 3], sl.t[lane % 3], n);
    else if (lane == 9) a0 = chain_sum<16>(a0, sl.v, n);
  }
}

// One support pass of the whole CTA. HIST: leaves the normalized pmf in S.p and
// returns ok; CENT: S.res[0..3] = num.x, num.y, num.z, den; MOM: S.res[0..9] =
// outer (row-major) and wsum. *visited = bounding-box voxels, *support.
template <int MODE, int NP>
__device__ __noinline__ int cta_pass(const PassIn in, CtaShared<NP>& S, long long* visited,
                                     unsigned* support_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Box bb = window_box(in.c, *in.g, in.nx, in.ny, in.nz);
  const long long bs = box_size(bb);
  const int Lx = bb.x1 - bb.x0 + 1, Ly = bb.y1 - bb.y0 + 1;
  const int total = (int)bs;
  const int nchunks = (total + kStep - 1) / kStep;
  const int nsteps = (nchunks + NP - 1) / NP;
  double a0 = 0.0, a1 = 0.0;
  unsigned support = 0;
  for (int step = 0; step <= nsteps; ++step) {
    if (warp > 0 && step < nsteps) {
      const int ch = step * NP + (warp - 1);
      CtaSlot& sl = S.slot[step & 1][warp - 1];
      if (ch < nchunks) {
        cta_produce<MODE>(in, bb, Lx, Ly, total, ch * kStep, sl, S.w, lane);
      } else {
        sl.cnt[lane] = 0;
        sl.cnt[lane + 32] = 0;
        if (lane == 0) sl.n = 0;
      }
    }
    if (warp == 0 && step > 0)
      for (int q = 0; q < NP; ++q)
        cta_consume<MODE>(S.slot[(step - 1) & 1][q], in.M, lane, a0, a1, support);
    __syncthreads();
  }
  int ok = 1;
  if (MODE == PASS_HIST) {
    if (warp == 0) {
      if (lane < in.M) S.h[lane] = a0;
      if (lane + 32 < in.M) S.h[lane + 32] = a1;
      __syncwarp();
      if (lane == 0) {
        double mass = 0.0;
        for (int b = 0; b < in.M; ++b) mass = __dadd_rn(mass, S.h[b]);  // Histogram::mass
        S.res[15] = mass;
        S.ires[0] = (int)support;
      }
    }
    __syncthreads();
    const double mass = S.res[15];
    const unsigned sup = (unsigned)S.ires[0];
    ok = !(sup == 0 || mass <= 0.0);
    if (ok && threadIdx.x < in.M) S.p[threadIdx.x] = __ddiv_rn(S.h[threadIdx.x], mass);
    *support_out = sup;
  } else {
    if (warp == 0 && lane < (MODE == PASS_CENT ? 4 : 10)) S.res[lane] = a0;
  }
  __syncthreads();
  *visited = bs;
  return ok;
}

__device__ __forceinline__ PassIn pass_in(const SeekParams& P, const uint8_t* vb, const double c[3],
                                          const WinGeom& g, int kernel) {
  PassIn in;
  in.vb = vb;
  in.nx = P.nx, in.ny = P.ny, in.nz = P.nz, in.M = P.bins;
  in.c[0] = c[0], in.c[1] = c[1], in.c[2] = c[2];
  in.g = &g;
  in.kernel = kernel;
  return in;
}

template <int NP>
__device__ __forceinline__ void cta_weights(const SeekParams& P, CtaShared<NP>& S) {
  if (threadIdx.x < P.bins) {  // weight_for_bin (histogram.hpp:107-113)
    const double pb = S.p[threadIdx.x] > 1e-6 ? S.p[threadIdx.x] : 1e-6;
    S.w[threadIdx.x] = __dsqrt_rn(__ddiv_rn(P.q[threadIdx.x], pb));
  }
  __syncthreads();
}

// bhattacharyya(S.p, q) (histogram.hpp:95-103), sequential, broadcast
template <int NP>
__device__ double cta_bhattacharyya(const SeekParams& P, CtaShared<NP>& S) {
  if (threadIdx.x == 0) {
    double rho = 0.0;
    for (int b = 0; b < P.bins; ++b) rho = __dadd_rn(rho, __dsqrt_rn(__dmul_rn(S.p[b], P.q[b])));
    S.res[14] = rho < 1.0 ? rho : 1.0;
  }
  __syncthreads();
  const double r = S.res[14];
  __syncthreads();
  return r;
}

template <int NP>
__device__ double cta_entropy(const SeekParams& P, CtaShared<NP>& S) {
  if ((threadIdx.x >> 5) == 0) {
    const double e = warp_entropy_bits(S.p, P.bins, threadIdx.x & 31, S.tmp);
    if (threadIdx.x == 0) S.res[13] = e;
  }
  __syncthreads();
  const double e = S.res[13];
  __syncthreads();
  return e;
}

#ifdef CTA_MINB  // A/B knob: resident CTAs per SM the register allocation must allow
#define SX_CTA_BOUNDS(NT) __launch_bounds__(NT, CTA_MINB)
#else             // default: no minimum (ptxas settles at 128 registers, 4 CTAs/SM)
#define SX_CTA_BOUNDS(NT) __launch_bounds__(NT)
#endif
template <int NP>
__global__ void SX_CTA_BOUNDS(32 * (NP + 1)) shift_cta_kernel(const SeekParams P) {
  extern __shared__ __align__(16) unsigned char cta_dyn[];
  CtaShared<NP>& S = *reinterpret_cast<CtaShared<NP>*>(cta_dyn);
  const int seed = blockIdx.x;
  if (seed >= P.n_seeds) return;
  const SeedIn si = P.seeds[seed];
  const uint8_t* vb = P.binvol + (size_t)si.vol * P.vol_stride;
  const ScaleGeom& sg = P.geoms[si.geom];
  const int M = P.bins;
  const double lim[3] = {(double)(P.nx - 1), (double)(P.ny - 1), (double)(P.nz - 1)};
  salvox_detection d;
  memset(&d, 0, sizeof d);
  d.seed_index = si.seed_index;
  for (int i = 0; i < 9; ++i) d.H[i] = sg.H[i];
  unsigned long long visits = 0;
  double c[3] = {dclamp(si.pos[0], lim[0]), dclamp(si.pos[1], lim[1]), dclamp(si.pos[2], lim[2])};
  unsigned support;
  long long vis;
  int ok = cta_pass<PASS_HIST, NP>(pass_in(P, vb, c, sg.main, P.hist_kernel), S, &vis, &support);
  auto frac_bad = [&](unsigned sup) {  // inbounds_support_fraction (shift.cpp:53-57, :75)
    if (sg.main.support_volume <= 0.0) return 0.0 < P.min_frac;
    double f = __ddiv_rn((double)sup, sg.main.support_volume);
    f = f < 1.0 ? f : 1.0;
    return f < P.min_frac;
  };
  bool degenerate = frac_bad(support);
  if (!degenerate) {
    for (int it = 0; it < P.max_iters; ++it) {
      d.iterations = it + 1;
      visits += (unsigned long long)vis;
      if (!ok) {
        degenerate = true;
        break;
      }
      cta_weights(P, S);
      long long cv;
      unsigned cs;
      cta_pass<PASS_CENT, NP>(pass_in(P, vb, c, sg.main, P.step_kernel), S, &cv, &cs);
      visits += (unsigned long long)cv;
      const double den = S.res[3];
      const double moved[3] = {__ddiv_rn(S.res[0], den), __ddiv_rn(S.res[1], den),
                               __ddiv_rn(S.res[2], den)};
      if (den <= 0.0) {
        degenerate = true;
        break;
      }
      double cl[3], df[3];
      for (int i = 0; i < 3; ++i) cl[i] = dclamp(moved[i], lim[i]);
      for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(cl[i], moved[i]);
      if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                               __dmul_rn(df[2], df[2]))) > 0.0)
        d.flags |= SALVOX_FLAG_BOUNDARY_CLAMPED;
      for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(cl[i], c[i]);
      const double step = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                                               __dmul_rn(df[2], df[2])));
      c[0] = cl[0], c[1] = cl[1], c[2] = cl[2];
      ok = cta_pass<PASS_HIST, NP>(pass_in(P, vb, c, sg.main, P.hist_kernel), S, &vis, &support);
      if (frac_bad(support)) {
        degenerate = true;
        break;
      }
      if (step < P.min_step) {
        d.flags |= SALVOX_FLAG_CONVERGED;
        break;
      }
    }
  }
  if (degenerate) d.flags |= SALVOX_FLAG_DEGENERATE;
  d.center[0] = c[0], d.center[1] = c[1], d.center[2] = c[2];
#ifdef SEEK_SKIP_FINAL  // profiling knob: no final scoring (results wrong)
  degenerate = true;
#endif
  if (!degenerate) {  // final scores (shift.cpp:89-105), as warp_final_scores
    unsigned sup;
    long long v2;
    double rho = 0.0;
    if (ok) rho = cta_bhattacharyya(P, S);
    const int ok_score = cta_pass<PASS_HIST, NP>(pass_in(P, vb, c, sg.main, 1), S, &v2, &sup);
    visits += 2ull * (unsigned long long)v2;  // the reference recomputes p_step too
    if (ok_score && ok) {
      d.entropy_bits = cta_entropy(P, S);
      d.bhattacharyya = rho;
    } else {
      d.flags |= SALVOX_FLAG_DEGENERATE;
    }
    double pdf = 0.0;
    if (sg.pdf_ok) {
      const int ok_lo = cta_pass<PASS_HIST, NP>(pass_in(P, vb, c, sg.lo, 0), S, &v2, &sup);
      visits += (unsigned long long)v2;
      if (threadIdx.x < M) S.tmp[threadIdx.x] = S.p[threadIdx.x];
      __syncthreads();
      const int ok_hi = cta_pass<PASS_HIST, NP>(pass_in(P, vb, c, sg.hi, 0), S, &v2, &sup);
      visits += (unsigned long long)v2;
      if (ok_lo && ok_hi) {
        if (threadIdx.x == 0) {
          double l1 = 0.0;
          for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(S.p[b], S.tmp[b])));
          S.res[12] = __dmul_rn(sg.pdf_fac, l1);
        }
        __syncthreads();
        pdf = S.res[12];
      }
    }
    d.pdf_diff = pdf;
  }
  if (threadIdx.x == 0) {
    P.out[si.slot] = d;
    P.visits[si.slot] = visits;
  }
}

// ------------------------------------------------------------------ ABMSOD
// abmsod_run (src/abmsod.cpp:43-169), one warp per seed: every support pass is
// the shift kernel's compacted ordered scan; the bandwidth moment runs its 9
// outer-product chains + the weight chain on lanes 0..9 in z->y->x order; the
// 3x3 symmetric eigensolver and the window geometry (Eigen inverse/determinant,
// shared exp/pow) come from include/salvox/sx_eig3.h, as in the oracle.
__device__ void dev_make_geom(const double* H, bool two_d, WinGeom& g) {  // window.hpp:69-106
  sx_inverse3(H, g.Hinv);
  for (int i = 0; i < 3; ++i) g.ext[i] = __dsqrt_rn(H[4 * i] < 0.0 ? 0.0 : H[4 * i]);
  const double det = sx_det3(H);
  g.det_fac = __ddiv_rn(1.0, __dsqrt_rn(det < 1e-300 ? 1e-300 : det));
  if (two_d) {
    const double det2 = __dsub_rn(__dmul_rn(H[0], H[4]), __dmul_rn(H[1], H[3]));
    g.support_volume = __dmul_rn(kPiD, __dsqrt_rn(det2 < 0.0 ? 0.0 : det2));
  } else {
    g.support_volume = __dmul_rn(4.0 / 3.0 * kPiD, __dsqrt_rn(det < 0.0 ? 0.0 : det));
  }
}

__device__ double dev_window_scale(const double* H, bool two_d) {  // window.hpp:50-56
  if (two_d) {
    const double det2 = __dsub_rn(__dmul_rn(H[0], H[4]), __dmul_rn(H[1], H[3]));
    return sx_pow(det2 < 0.0 ? 0.0 : det2, 0.25);
  }
  const double det = sx_det3(H);
  return sx_pow(det < 0.0 ? 0.0 : det, 1.0 / 6.0);
}

struct AbmWarp {
  WinGeom g;              // the current window's geometry
  double Hc[9], Hn[9];    // current / updated bandwidth
  double acc[10];         // moment chains (lane l writes acc[l])
};

// bandwidth_update's moment pass (abmsod.cpp:45-56): over the support of
// (xn, H), w = weight_for_bin(hp_new), d = xn - s, outer += (w d_i) d_j, wsum += w.
// Lane l < 9 owns outer element l (i = l / 3, j = l % 3), lane 9 owns wsum.
__device__ __noinline__ long long warp_moment(const SeekParams& P, const uint8_t* vb, WarpScratch& s,
                                 const double xn[3], const WinGeom& wg, int lane, double* acc_out) {
  double acc = 0.0;
  const int li = lane < 9 ? lane / 3 : 0, lj = lane < 9 ? lane % 3 : 0;
  const Box bb = window_box(xn, wg, P.nx, P.ny, P.nz);
  warp_box_iter_g(bb, lane, [&](const bool* act, const int* x, const int* y, const int* z) {
    bool in[kG];
    double w[kG];
    int braw[kG];  // bins fetched before the Mahalanobis tests (latency overlap)
#pragma unroll
    for (int j = 0; j < kG; ++j) braw[j] = act[j] ? bin_at(P, vb, x[j], y[j], z[j]) : 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      in[j] = false;
      w[j] = 0.0;
      if (act[j]) {
        const double dd = maha(wg, xn, x[j], y[j], z[j]);
        in[j] = dd <= 1.0;
        if (in[j]) w[j] = s.w[braw[j]];
      }
    }
    int off = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const unsigned m0 = __ballot_sync(kFull, in[j]);
      if (in[j]) {
        const int r = off + __popc(m0 & ((1u << lane) - 1u));
        s.v[r] = w[j];
        s.t[0][r] = __dsub_rn(xn[0], (double)x[j]);
        s.t[1][r] = __dsub_rn(xn[1], (double)y[j]);
        s.t[2][r] = __dsub_rn(xn[2], (double)z[j]);
      }
      off += __popc(m0);
    }
    __syncwarp();
    if (lane < 9) {
      const double* di = s.t[li];
      const double* dj = s.t[lj];
#pragma unroll 4
      for (int k = 0; k < off; ++k) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(s.v[k], di[k]), dj[k]));
    } else if (lane == 9) {
#pragma unroll 4
      for (int k = 0; k < off; ++k) acc = __dadd_rn(acc, s.v[k]);
    }
    __syncwarp();
  });
  *acc_out = acc;
  return box_size(bb);
}

__device__ __forceinline__ void warp_weights(const SeekParams& P, WarpScratch& s, int lane) {
  for (int b = lane; b < P.bins; b += 32) {  // weight_for_bin (histogram.hpp:107-113)
    const double pb = s.p[b] > 1e-6 ? s.p[b] : 1e-6;
    s.w[b] = __dsqrt_rn(__ddiv_rn(P.q[b], pb));
  }
  __syncwarp();
}

template <int NW>
__global__ void __launch_bounds__(32 * NW) abmsod_kernel(const SeekParams P) {
  __shared__ WarpScratch scratch[NW];
  __shared__ AbmWarp aws[NW];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int seed = blockIdx.x * NW + wid;
  if (seed >= P.n_seeds) return;
  WarpScratch& s = scratch[wid];
  AbmWarp& A = aws[wid];
  const SeedIn si = P.seeds[seed];
  const uint8_t* vb = P.binvol + (size_t)si.vol * P.vol_stride;
  const bool two_d = P.two_d != 0;
  const int M = P.bins;
  const double lim[3] = {(double)(P.nx - 1), (double)(P.ny - 1), (double)(P.nz - 1)};
  salvox_detection d;
  memset(&d, 0, sizeof d);
  d.seed_index = si.seed_index;
  double x[3] = {dclamp(si.pos[0], lim[0]), dclamp(si.pos[1], lim[1]), dclamp(si.pos[2], lim[2])};
  d.center[0] = x[0], d.center[1] = x[1], d.center[2] = x[2];  // clamp_point(seed) (abmsod.cpp:58)
  const double* H0 = P.seed_H + 9 * (size_t)si.slot;
  if (lane < 9) A.Hc[lane] = H0[lane];
  __syncwarp();
  for (int i = 0; i < 9; ++i) d.H[i] = A.Hc[i];
  double x_opt[3] = {x[0], x[1], x[2]};
  double H_opt[9];
  for (int i = 0; i < 9; ++i) H_opt[i] = A.Hc[i];
  double max_bhat = 0.0;
  int stalled = 0, n_trace = 0;
  bool any = false, failed = false;
  unsigned long long visits = 0;
  for (int it = 0; it < P.abm_max_iters; ++it) {
    if (lane == 0) dev_make_geom(A.Hc, two_d, A.g);
    __syncwarp();
    unsigned support;
    long long vis;
    // inbounds_support_fraction (window.cpp:54-60) = the histogram pass's support count
    const bool ok = warp_candidate_hist(P, vb, s, x, A.g, P.abm_kernel, lane, &support, &vis);
    double frac = 0.0;
    if (A.g.support_volume > 0.0) {
      frac = __ddiv_rn((double)support, A.g.support_volume);
      frac = frac < 1.0 ? frac : 1.0;
    }
    if (frac < P.abm_min_frac) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    visits += (unsigned long long)vis;
    if (!ok) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    warp_weights(P, s, lane);
    double num[3], den;
    visits += (unsigned long long)warp_centroid(P, vb, s, x, A.g, P.abm_kernel, lane, num, &den);
    if (den <= 0.0) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    const double moved[3] = {__ddiv_rn(num[0], den), __ddiv_rn(num[1], den), __ddiv_rn(num[2], den)};
    double xn[3], df[3];
    for (int i = 0; i < 3; ++i) xn[i] = dclamp(moved[i], lim[i]);
    for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(xn[i], moved[i]);
    if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                             __dmul_rn(df[2], df[2]))) > 0.0)
      d.flags |= SALVOX_FLAG_BOUNDARY_CLAMPED;
    // histogram at the moved centre with the old H (abmsod.cpp:100-106)
    const bool ok2 = warp_candidate_hist(P, vb, s, xn, A.g, P.abm_kernel, lane, &support, &vis);
    visits += (unsigned long long)vis;
    if (!ok2) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    warp_weights(P, s, lane);
    double acc;
    visits += (unsigned long long)warp_moment(P, vb, s, xn, A.g, lane, &acc);
    if (lane < 10) A.acc[lane] = acc;
    __syncwarp();
    int br = 0;
    if (lane == 0)
      br = sx_bandwidth_from_moment(A.acc, A.acc[9], two_d ? 2 : 3, P.abm_lmin, P.abm_lmax, A.Hn);
    br = __shfl_sync(kFull, br, 0);
    __syncwarp();
    if (br == 3) {  // std::runtime_error escapes abmsod_run
      failed = true;
      break;
    }
    if (br != 0) {  // std::invalid_argument -> degenerate (abmsod.cpp:107-112)
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    double bhat = 0.0;  // bhattacharyya(hp_new, target) (histogram.hpp:95-103)
    if (lane == 0) {
      for (int b = 0; b < M; ++b) bhat = __dadd_rn(bhat, __dsqrt_rn(__dmul_rn(s.p[b], P.q[b])));
      bhat = bhat < 1.0 ? bhat : 1.0;
    }
    bhat = __shfl_sync(kFull, bhat, 0);
    any = true;
    d.iterations = it + 1;
    const bool improved = bhat > __dadd_rn(max_bhat, P.abm_threshold);
    if (bhat > max_bhat) {
      max_bhat = bhat;
      for (int i = 0; i < 3; ++i) x_opt[i] = xn[i];
      for (int i = 0; i < 9; ++i) H_opt[i] = A.Hn[i];
    }
    if (P.abm_trace && lane == 0 && n_trace < P.abm_max_iters) {
      double ev[3], V[9];
      if (sx_sym_eigen3(A.Hn, ev, V) != 0) failed = true;
      salvox_abmsod_iter& r = P.abm_trace[(size_t)si.slot * P.abm_max_iters + n_trace];
      for (int i = 0; i < 3; ++i) r.position[i] = xn[i];
      for (int i = 0; i < 9; ++i) r.H[i] = A.Hn[i];
      r.bhattacharyya = bhat;
      r.max_bhattacharyya = max_bhat;
      r.eig_min = fmin(fmin(ev[0], ev[1]), ev[2]);
      r.eig_max = fmax(fmax(ev[0], ev[1]), ev[2]);
    }
    if (P.abm_trace) ++n_trace;
    failed = __shfl_sync(kFull, (int)failed, 0) != 0;
    if (failed) break;
    for (int i = 0; i < 3; ++i) x[i] = xn[i];
    if (lane < 9) A.Hc[lane] = A.Hn[lane];
    __syncwarp();
    stalled = improved ? 0 : stalled + 1;
    if (stalled >= 2) {
      d.flags |= SALVOX_FLAG_CONVERGED;
      break;
    }
  }
  if (!failed) {
    if (any) {  // score the best iterate (abmsod.cpp:154-165)
      d.center[0] = x_opt[0], d.center[1] = x_opt[1], d.center[2] = x_opt[2];
      for (int i = 0; i < 9; ++i) d.H[i] = H_opt[i];
      d.bhattacharyya = max_bhat;
      if (lane < 9) A.Hc[lane] = H_opt[lane];
      __syncwarp();
      if (lane == 0) dev_make_geom(A.Hc, two_d, A.g);
      __syncwarp();
      unsigned sup;
      long long vis;
      if (warp_candidate_hist(P, vb, s, x_opt, A.g, 1, lane, &sup, &vis))
        d.entropy_bits = warp_entropy_bits(s.p, M, lane, s.w);
      visits += (unsigned long long)vis;
      // pdf_difference (window.cpp:30-46), Identity kernel; throws -> 0.0
      const double sc = dev_window_scale(H_opt, two_d);
      double pdf = 0.0;
      if (!(__dsub_rn(sc, 1.0) < 1.0)) {
        double l1 = 0.0;
        bool ok_lo = false, ok_hi = false;
        for (int f = 0; f < 2; ++f) {
          const double s_new = f == 0 ? __dsub_rn(sc, 1.0) : __dadd_rn(sc, 1.0);
          const double r = __ddiv_rn(s_new, sc);
          const double fac = __dmul_rn(r, r);
          if (lane < 9) A.Hn[lane] = __dmul_rn(H_opt[lane], fac);
          __syncwarp();
          if (lane == 0) {
            if (two_d) A.Hn[8] = 1.0;
            dev_make_geom(A.Hn, two_d, A.g);
          }
          __syncwarp();
          const bool okf = warp_candidate_hist(P, vb, s, x_opt, A.g, 0, lane, &sup, &vis);
          visits += (unsigned long long)vis;
          if (f == 0) {
            ok_lo = okf;
            for (int b = lane; b < M; b += 32) s.w[b] = s.p[b];  // keep p_lo
            __syncwarp();
          } else {
            ok_hi = okf;
          }
        }
        if (ok_lo && ok_hi) {
          if (lane == 0)
            for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(s.p[b], s.w[b])));
          l1 = __shfl_sync(kFull, l1, 0);
          pdf = __dmul_rn(__ddiv_rn(__dmul_rn(sc, sc), 2.0), l1);
        }
      }
      d.pdf_diff = pdf;
    } else {
      d.flags |= SALVOX_FLAG_DEGENERATE;
    }
  } else if (lane == 0) {
    atomicOr(P.err_flag, 1);  // eigen decomposition failed: runtime_error for the call
  }
  if (lane == 0) {
    P.out[si.slot] = d;
    P.visits[si.slot] = visits;
    if (P.abm_trace_n) P.abm_trace_n[si.slot] = n_trace;
  }
}

// ABMSOD on the CTA engine (latency mode: a few hundred seeds, long passes):
// the same operations as abmsod_kernel, each support pass run by cta_pass.
template <int NP>
__global__ void __launch_bounds__(32 * (NP + 1)) abmsod_cta_kernel(const SeekParams P) {
  extern __shared__ __align__(16) unsigned char cta_dyn[];
  CtaShared<NP>& S = *reinterpret_cast<CtaShared<NP>*>(cta_dyn);
  const int seed = blockIdx.x;
  if (seed >= P.n_seeds) return;
  const SeedIn si = P.seeds[seed];
  const uint8_t* vb = P.binvol + (size_t)si.vol * P.vol_stride;
  const bool two_d = P.two_d != 0;
  const int M = P.bins;
  const double lim[3] = {(double)(P.nx - 1), (double)(P.ny - 1), (double)(P.nz - 1)};
  salvox_detection d;
  memset(&d, 0, sizeof d);
  d.seed_index = si.seed_index;
  double x[3] = {dclamp(si.pos[0], lim[0]), dclamp(si.pos[1], lim[1]), dclamp(si.pos[2], lim[2])};
  d.center[0] = x[0], d.center[1] = x[1], d.center[2] = x[2];
  const double* H0 = P.seed_H + 9 * (size_t)si.slot;
  double H_opt[9];
  for (int i = 0; i < 9; ++i) d.H[i] = H_opt[i] = H0[i];
  if (threadIdx.x < 9) S.Hc[threadIdx.x] = H0[threadIdx.x];
  __syncthreads();
  double x_opt[3] = {x[0], x[1], x[2]};
  double max_bhat = 0.0;
  int stalled = 0, n_trace = 0;
  bool any = false, failed = false;
  unsigned long long visits = 0;
  for (int it = 0; it < P.abm_max_iters; ++it) {
    if (threadIdx.x == 0) dev_make_geom(S.Hc, two_d, S.g);
    __syncthreads();
    unsigned support;
    long long vis;
    const int ok = cta_pass<PASS_HIST, NP>(pass_in(P, vb, x, S.g, P.abm_kernel), S, &vis, &support);
    double frac = 0.0;  // inbounds_support_fraction (window.cpp:54-60)
    if (S.g.support_volume > 0.0) {
      frac = __ddiv_rn((double)support, S.g.support_volume);
      frac = frac < 1.0 ? frac : 1.0;
    }
    if (frac < P.abm_min_frac) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    visits += (unsigned long long)vis;
    if (!ok) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    cta_weights(P, S);
    unsigned cs;
    cta_pass<PASS_CENT, NP>(pass_in(P, vb, x, S.g, P.abm_kernel), S, &vis, &cs);
    visits += (unsigned long long)vis;
    const double den = S.res[3];
    if (den <= 0.0) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    const double moved[3] = {__ddiv_rn(S.res[0], den), __ddiv_rn(S.res[1], den),
                             __ddiv_rn(S.res[2], den)};
    double xn[3], df[3];
    for (int i = 0; i < 3; ++i) xn[i] = dclamp(moved[i], lim[i]);
    for (int i = 0; i < 3; ++i) df[i] = __dsub_rn(xn[i], moved[i]);
    if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(df[0], df[0]), __dmul_rn(df[1], df[1])),
                             __dmul_rn(df[2], df[2]))) > 0.0)
      d.flags |= SALVOX_FLAG_BOUNDARY_CLAMPED;
    const int ok2 = cta_pass<PASS_HIST, NP>(pass_in(P, vb, xn, S.g, P.abm_kernel), S, &vis, &support);
    visits += (unsigned long long)vis;
    if (!ok2) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    cta_weights(P, S);
    cta_pass<PASS_MOM, NP>(pass_in(P, vb, xn, S.g, 0), S, &vis, &cs);
    visits += (unsigned long long)vis;
    if (threadIdx.x == 0)
      S.ires[1] = sx_bandwidth_from_moment(S.res, S.res[9], two_d ? 2 : 3, P.abm_lmin, P.abm_lmax, S.Hn);
    __syncthreads();
    const int br = S.ires[1];
    if (br == 3) {
      failed = true;
      break;
    }
    if (br != 0) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
      break;
    }
    const double bhat = cta_bhattacharyya(P, S);
    any = true;
    d.iterations = it + 1;
    const bool improved = bhat > __dadd_rn(max_bhat, P.abm_threshold);
    if (bhat > max_bhat) {
      max_bhat = bhat;
      for (int i = 0; i < 3; ++i) x_opt[i] = xn[i];
      for (int i = 0; i < 9; ++i) H_opt[i] = S.Hn[i];
    }
    if (P.abm_trace) {
      if (threadIdx.x == 0) {
        double ev[3], V[9];
        S.ires[2] = sx_sym_eigen3(S.Hn, ev, V) != 0;
        salvox_abmsod_iter& r = P.abm_trace[(size_t)si.slot * P.abm_max_iters + n_trace];
        for (int i = 0; i < 3; ++i) r.position[i] = xn[i];
        for (int i = 0; i < 9; ++i) r.H[i] = S.Hn[i];
        r.bhattacharyya = bhat;
        r.max_bhattacharyya = max_bhat;
        r.eig_min = fmin(fmin(ev[0], ev[1]), ev[2]);
        r.eig_max = fmax(fmax(ev[0], ev[1]), ev[2]);
      }
      __syncthreads();
      ++n_trace;
      if (S.ires[2]) {
        failed = true;
        break;
      }
    }
    for (int i = 0; i < 3; ++i) x[i] = xn[i];
    __syncthreads();
    if (threadIdx.x < 9) S.Hc[threadIdx.x] = S.Hn[threadIdx.x];
    __syncthreads();
    stalled = improved ? 0 : stalled + 1;
    if (stalled >= 2) {
      d.flags |= SALVOX_FLAG_CONVERGED;
      break;
    }
  }
  if (!failed) {
    if (any) {  // score the best iterate (abmsod.cpp:154-165)
      d.center[0] = x_opt[0], d.center[1] = x_opt[1], d.center[2] = x_opt[2];
      for (int i = 0; i < 9; ++i) d.H[i] = H_opt[i];
      d.bhattacharyya = max_bhat;
      __syncthreads();
      if (threadIdx.x < 9) S.Hc[threadIdx.x] = H_opt[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) dev_make_geom(S.Hc, two_d, S.g);
      __syncthreads();
      unsigned sup;
      long long vis;
      if (cta_pass<PASS_HIST, NP>(pass_in(P, vb, x_opt, S.g, 1), S, &vis, &sup))
        d.entropy_bits = cta_entropy(P, S);
      visits += (unsigned long long)vis;
      const double sc = dev_window_scale(H_opt, two_d);
      double pdf = 0.0;
      if (!(__dsub_rn(sc, 1.0) < 1.0)) {  // pdf_difference (window.cpp:30-46)
        int okf[2];
        for (int f = 0; f < 2; ++f) {
          const double s_new = f == 0 ? __dsub_rn(sc, 1.0) : __dadd_rn(sc, 1.0);
          const double r = __ddiv_rn(s_new, sc);
          const double fac = __dmul_rn(r, r);
          __syncthreads();
          if (threadIdx.x < 9) S.Hn[threadIdx.x] = __dmul_rn(H_opt[threadIdx.x], fac);
          __syncthreads();
          if (threadIdx.x == 0) {
            if (two_d) S.Hn[8] = 1.0;
            dev_make_geom(S.Hn, two_d, S.g);
          }
          __syncthreads();
          okf[f] = cta_pass<PASS_HIST, NP>(pass_in(P, vb, x_opt, S.g, 0), S, &vis, &sup);
          visits += (unsigned long long)vis;
          if (f == 0) {
            if (threadIdx.x < M) S.tmp[threadIdx.x] = S.p[threadIdx.x];
            __syncthreads();
          }
        }
        if (okf[0] && okf[1]) {
          if (threadIdx.x == 0) {
            double l1 = 0.0;
            for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(S.p[b], S.tmp[b])));
            S.res[12] = __dmul_rn(__ddiv_rn(__dmul_rn(sc, sc), 2.0), l1);
          }
          __syncthreads();
          pdf = S.res[12];
        }
      }
      d.pdf_diff = pdf;
    } else {
      d.flags |= SALVOX_FLAG_DEGENERATE;
    }
  } else if (threadIdx.x == 0) {
    atomicOr(P.err_flag, 1);
  }
  if (threadIdx.x == 0) {
    P.out[si.slot] = d;
    P.visits[si.slot] = visits;
    if (P.abm_trace_n) P.abm_trace_n[si.slot] = n_trace;
  }
}

// -------------------------------------------------------- quadrant / octant
// NE, NW, SW, SE (quadrant.cpp:14); octants: the four at z=+1, then at z=-1.
__constant__ int c_dirs[8][3] = {{+1, +1, +1}, {-1, +1, +1}, {-1, -1, +1}, {+1, -1, +1},
                                 {+1, +1, -1}, {-1, +1, -1}, {-1, -1, -1}, {+1, -1, -1}};

__device__ __forceinline__ void axis_range(double p, double dk, int n, int* lo, int* hi) {
  const double a = p, b = __dadd_rn(p, dk);  // [min, max] of (p, p + dir*k)
  *lo = max(0, (int)ceil(a < b ? a : b));
  *hi = min(n - 1, (int)floor(a < b ? b : a));
}

// Adds the voxels of box B that are not in box A (A subset of B, or A empty)
// to the per-octant counts.
__device__ void warp_count_shell(const SeekParams& P, const uint8_t* vb, unsigned* cnt, const Box& A, const Box& B,
                                 bool a_empty, int lane) {
  auto count_box = [&](const Box& bx) {
    warp_box_iter(bx, lane, [&](bool act, int x, int y, int z) {
      if (act) atomicAdd(&cnt[bin_at(P, vb, x, y, z)], 1u);
    });
  };
  if (a_empty) {
    count_box(B);
    return;
  }
  // x outside A.x
  if (B.x0 < A.x0) count_box(Box{B.x0, A.x0 - 1, B.y0, B.y1, B.z0, B.z1});
  if (B.x1 > A.x1) count_box(Box{A.x1 + 1, B.x1, B.y0, B.y1, B.z0, B.z1});
  // x inside, y outside
  if (B.y0 < A.y0) count_box(Box{A.x0, A.x1, B.y0, A.y0 - 1, B.z0, B.z1});
  if (B.y1 > A.y1) count_box(Box{A.x0, A.x1, A.y1 + 1, B.y1, B.z0, B.z1});
  // x, y inside, z outside
  if (B.z0 < A.z0) count_box(Box{A.x0, A.x1, A.y0, A.y1, B.z0, A.z0 - 1});
  if (B.z1 > A.z1) count_box(Box{A.x0, A.x1, A.y0, A.y1, A.z1 + 1, B.z1});
}


// Per-warp dynamic shared memory of the level-table ascent (AscentLevels).
struct AscentLayout {
  __host__ __device__ static size_t a16(size_t v) { return (v + 15) & ~size_t(15); }
  __host__ __device__ static size_t lvl() { return 0; }                      // 3 x 132 u8
  __host__ __device__ static size_t rng() { return 400; }                    // nS x 6 int
  __host__ __device__ static size_t boxn(int nS) { return a16(rng() + 24 * (size_t)nS); }
  __host__ __device__ static size_t es(int nS) { return a16(boxn(nS) + 4 * (size_t)nS); }
  __host__ __device__ static size_t cnt(int nS) { return a16(es(nS) + 8 * (size_t)nS); }
  __host__ __device__ static size_t term(int nS, int M) { return a16(cnt(nS) + 4 * (size_t)nS * M); }
  __host__ __device__ static size_t bytes(int nS, int M) { return a16(term(nS, M) + 8 * (size_t)nS * M); }
};

// Best (entropy, scale) of one corner-anchored direction, all scales at once.
// The boxes [p, p + k dir] are nested in k, so every voxel of the largest box
// has a level = the first scale whose box holds it (max over the three axes of
// per-axis levels, tabulated per iteration). ONE pass over the largest box
// counts (level, bin); a prefix over levels gives every scale's exact counts;
// the nS x M terms p log p are evaluated in parallel and lanes 0..nS-1 sum
// their scale's terms in bin order -- the same fp64 operations, in the same
// order, as box_entropy_bits (quadrant.cpp:18-35) per scale.
__device__ void ascent_levels(const SeekParams& P, const uint8_t* vb, unsigned char* wb,
                              const int dir[3], const double p[3], bool two_d, int min_vox,
                              int lane, double* best_e_out, int* best_k_out,
                              unsigned long long* visits) {
  const int nS = P.n_ascent, M = P.bins;
  uint8_t* lv = wb + AscentLayout::lvl();
  int* rng = reinterpret_cast<int*>(wb + AscentLayout::rng());
  int* boxn = reinterpret_cast<int*>(wb + AscentLayout::boxn(nS));
  double* es = reinterpret_cast<double*>(wb + AscentLayout::es(nS));
  unsigned* cnt = reinterpret_cast<unsigned*>(wb + AscentLayout::cnt(nS));
  double* term = reinterpret_cast<double*>(wb + AscentLayout::term(nS, M));
  const int dims[3] = {P.nx, P.ny, P.nz};
  for (int i = lane; i < nS; i += 32) {  // per-scale boxes (quadrant.cpp:20-23, 49-51)
    const double k = (double)P.ascent_scales[i];
    Box B;
    axis_range(p[0], (double)dir[0] * k, P.nx, &B.x0, &B.x1);
    axis_range(p[1], (double)dir[1] * k, P.ny, &B.y0, &B.y1);
    axis_range(p[2], two_d ? 0.0 : (double)dir[2] * k, P.nz, &B.z0, &B.z1);
    rng[6 * i + 0] = B.x0, rng[6 * i + 1] = B.x1, rng[6 * i + 2] = B.y0;
    rng[6 * i + 3] = B.y1, rng[6 * i + 4] = B.z0, rng[6 * i + 5] = B.z1;
    boxn[i] = (int)box_size(B);
  }
  for (int i = lane; i < nS * M; i += 32) cnt[i] = 0u;
  __syncwarp();
  const int* big = rng + 6 * (nS - 1);
  const int L[3] = {big[1] - big[0] + 1, big[3] - big[2] + 1, big[5] - big[4] + 1};
  const bool any = boxn[nS - 1] > 0;
  if (any) {
    for (int a = 0; a < 3; ++a)  // per-axis level of each coordinate of the largest box
      for (int t = lane; t < L[a]; t += 32) {
        const int x = big[2 * a] + t;
        int i = 0;
        while (i < nS - 1 && !(rng[6 * i + 2 * a] <= x && x <= rng[6 * i + 2 * a + 1])) ++i;
        lv[132 * a + t] = (uint8_t)i;
      }
  }
  (void)dims;
  __syncwarp();
  if (any) {
    const int total = L[0] * L[1] * L[2];
    const float ix = 1.0f / (float)L[0], iy = 1.0f / (float)L[1];
    constexpr int G = ASCENT_G;  // voxels per lane per step: bin loads in flight
    for (int base = 0; base < total; base += 32 * G) {
      int bin[G], lvl[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int n = base + 32 * j + lane;
        const int nc = n < total ? n : 0;
        const int t = fdiv_small(nc, ix);
        const int x = nc - t * L[0];
        const int zz = fdiv_small(t, iy);
        const int y = t - zz * L[1];
        bin[j] = n < total ? bin_at(P, vb, big[0] + x, big[2] + y, big[4] + zz) : -1;
        lvl[j] = max(max((int)lv[x], (int)lv[132 + y]), (int)lv[264 + zz]);
      }
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (bin[j] >= 0) atomicAdd(&cnt[lvl[j] * M + bin[j]], 1u);
    }
  }
  __syncwarp();
  for (int b = lane; b < M; b += 32) {  // counts of box i = voxels with level <= i
    unsigned run = 0;
    for (int i = 0; i < nS; ++i) {
      run += cnt[i * M + b];
      cnt[i * M + b] = run;
    }
  }
  __syncwarp();
  const float im = 1.0f / (float)M;
  for (int idx = lane; idx < nS * M; idx += 32) {
    const int i = fdiv_small(idx, im);
    const int n = boxn[i];
    const unsigned c = cnt[idx];
    double t = 0.0;
    if (n > 0 && n >= min_vox && c > 0u) {  // quadrant.cpp:24-26; p = count / mass (exact mass)
      const double pb = __ddiv_rn((double)c, (double)n);
      t = __dmul_rn(pb, sx_log(pb));
    }
    term[idx] = t;
  }
  __syncwarp();
  unsigned long long v = 0;
  for (int i = lane; i < nS; i += 32) {  // entropy_bits (histogram.hpp:56-67), bin order
    const int n = boxn[i];
    double e = 0.0;
    if (n > 0 && n >= min_vox) {
      v += (unsigned long long)n;
      for (int b = 0; b < M; ++b)
        if (cnt[i * M + b] > 0u) e = __dsub_rn(e, term[i * M + b]);
      e = __ddiv_rn(e < 0.0 ? 0.0 : e, kLn2);
    }
    es[i] = e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  *visits += v;
  __syncwarp();
  double best_e = 0.0;
  int best_k = P.ascent_scales[0];
  for (int i = 0; i < nS; ++i)  // strict: smallest scale wins ties (quadrant.cpp:52)
    if (es[i] > best_e) {
      best_e = es[i];
      best_k = P.ascent_scales[i];
    }
  *best_e_out = best_e;
  *best_k_out = best_k;
  __syncwarp();
}

// One CTA per trajectory, one warp per quadrant/octant: warp q counts its
// corner-anchored boxes for every scale (nested in k, so only the shell
// B_k \ B_{k-1} is counted) and evaluates their entropies; thread 0 combines the
// nq (entropy, scale) pairs into the move exactly as quadrant.cpp:55-81 does.
// Post-scoring runs its three window histograms on three warps in parallel.
struct AscentWarp {
  unsigned cnt[kMaxBins];
  double p[kMaxBins];
  double w[kMaxBins];
};

template <int NQ, bool LV>
__global__ void __launch_bounds__(32 * NQ, 24 / NQ) ascent_kernel(const SeekParams P) {
  extern __shared__ __align__(16) unsigned char asc_dyn[];
  __shared__ AscentWarp aw[LV ? 1 : NQ];
  __shared__ WarpScratch ps[3];
  __shared__ double ent[NQ];
  __shared__ int bk[NQ];
  __shared__ double pos[3];
  __shared__ int ctl[3];  // stop, converged, degenerate
  __shared__ unsigned long long vis[NQ];
  __shared__ double score[3];  // entropy, bhattacharyya, pdf
  __shared__ int okf[3];
  const int lane = threadIdx.x & 31;
  const int q = threadIdx.x >> 5;
  const int seed = blockIdx.x;
  if (seed >= P.n_seeds) return;  // uniform per CTA
  const SeedIn si = P.seeds[seed];
  const uint8_t* vb = P.binvol + (size_t)si.vol * P.vol_stride;
  const int M = P.bins;
  const bool two_d = NQ == 4;
  const int min_vox = two_d ? 4 : 8;
  const double lim[3] = {(double)(P.nx - 1), (double)(P.ny - 1), (double)(P.nz - 1)};
  double p[3] = {si.pos[0], si.pos[1], si.pos[2]};
  unsigned long long visits = 0;
  AscentWarp& s = aw[LV ? 0 : q];
  int iters = 0;
  for (int it = 0; it < P.max_iters; ++it) {
    double best_e = 0.0;
    int best_k = P.ascent_scales[0];
    if (LV) {
      const int dir[3] = {c_dirs[q][0], c_dirs[q][1], c_dirs[q][2]};
      ascent_levels(P, vb, asc_dyn + (size_t)q * P.asc_warp_bytes, dir, p, two_d, min_vox, lane,
                    &best_e, &best_k, &visits);
    } else {
    for (int b = lane; b < M; b += 32) s.cnt[b] = 0u;
    __syncwarp();
    Box prev{0, -1, 0, -1, 0, -1};
    bool prev_empty = true;
    for (int i = 0; i < P.n_ascent; ++i) {
      const int k = P.ascent_scales[i];
      Box B;
      axis_range(p[0], (double)c_dirs[q][0] * (double)k, P.nx, &B.x0, &B.x1);
      axis_range(p[1], (double)c_dirs[q][1] * (double)k, P.ny, &B.y0, &B.y1);
      if (two_d) {
        axis_range(p[2], 0.0, P.nz, &B.z0, &B.z1);
      } else {
        axis_range(p[2], (double)c_dirs[q][2] * (double)k, P.nz, &B.z0, &B.z1);
      }
      const long long count = box_size(B);
      if (count > 0) {
        warp_count_shell(P, vb, s.cnt, prev, B, prev_empty, lane);
        prev = B;
        prev_empty = false;
      }
      __syncwarp();
      double e = 0.0;
      if (count > 0 && count >= min_vox) {  // quadrant.cpp:24-26
        visits += (unsigned long long)count;
        const double mass = (double)count;  // exact integer mass
        for (int b = lane; b < M; b += 32) s.p[b] = __ddiv_rn((double)s.cnt[b], mass);
        __syncwarp();
        e = warp_entropy_bits(s.p, M, lane, s.w);
      }
      if (e > best_e) {  // strict: smallest scale wins ties (quadrant.cpp:52)
        best_e = e;
        best_k = k;
      }
    }
    }
    if (lane == 0) {
      ent[q] = best_e;
      bk[q] = best_k;
    }
    __syncthreads();
    iters = it + 1;
    if (threadIdx.x == 0) {
      double total = 0.0;
      for (int r = 0; r < NQ; ++r) total = __dadd_rn(total, ent[r]);
      ctl[0] = ctl[1] = ctl[2] = 0;
      salvox_ascent_state* st = P.ascent_state ? &P.ascent_state[si.slot] : nullptr;
      if (st) {  // QuadrantState (quadrant.hpp:32-38) of this step
        memset(st, 0, sizeof *st);
        for (int r = 0; r < NQ; ++r) st->entropy[r] = ent[r], st->best_scale[r] = bk[r];
      }
      if (total <= 0.0) {
        ctl[0] = ctl[2] = 1;
        pos[0] = p[0], pos[1] = p[1], pos[2] = p[2];
        if (st) st->degenerate = 1;
      } else {
        double ed[3] = {0.0, 0.0, 0.0};
        for (int r = 0; r < NQ; ++r) {
          const double ne = __ddiv_rn(ent[r], total);
          if (st) st->norm_entropy[r] = ne;
          for (int a = 0; a < (two_d ? 2 : 3); ++a)
            ed[a] = __dadd_rn(ed[a], __dmul_rn(__dmul_rn(ne, (double)c_dirs[r][a]), (double)bk[r]));
        }
        if (st) st->displacement[0] = ed[0], st->displacement[1] = ed[1], st->displacement[2] = ed[2];
        pos[0] = p[0], pos[1] = p[1], pos[2] = p[2];
        for (int a = 0; a < (two_d ? 2 : 3); ++a) pos[a] = dclamp(__dadd_rn(p[a], ed[a]), lim[a]);
        const double nrm =
            two_d ? __dsqrt_rn(__dadd_rn(__dmul_rn(ed[0], ed[0]), __dmul_rn(ed[1], ed[1])))
                  : __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ed[0], ed[0]), __dmul_rn(ed[1], ed[1])),
                                         __dmul_rn(ed[2], ed[2])));
        if (nrm < P.eta) ctl[0] = ctl[1] = 1;
      }
    }
    __syncthreads();
    p[0] = pos[0], p[1] = pos[1], p[2] = pos[2];
    if (ctl[0]) break;
  }
  const bool degenerate = ctl[2] != 0, converged = ctl[1] != 0;
  int bq = 0;
  for (int r = 1; r < NQ; ++r)
    if (ent[r] > ent[bq]) bq = r;
  const int best_scale = bk[bq];
  const double best_entropy = ent[bq];
  // post-scoring: isotropic window k = max(2, best_scale) (pipeline.cpp:343-355)
  const int kwin = max(2, best_scale);
  const ScaleGeom& sg = P.geoms[P.geom_of_k[kwin]];
  const double c[3] = {p[0], p[1], two_d ? 0.0 : p[2]};
  if (!degenerate && P.post_score && q < 3) {
    unsigned sup;
    long long v;
    WarpScratch& w = ps[q];
    if (q == 0) {  // Epanechnikov histogram: entropy + Bhattacharyya vs uniform
      const bool okp = warp_candidate_hist(P, vb, w, c, sg.main, 1, lane, &sup, &v);
      visits += (unsigned long long)v;
      double rho = 0.0, e = 0.0;
      if (okp) {
        if (lane == 0) {
          for (int b = 0; b < M; ++b) rho = __dadd_rn(rho, __dsqrt_rn(__dmul_rn(w.p[b], P.q[b])));
          rho = rho < 1.0 ? rho : 1.0;
        }
        e = warp_entropy_bits(w.p, M, lane, w.w);
      }
      if (lane == 0) {
        okf[0] = okp;
        score[0] = e;
        score[1] = rho;
      }
    } else if (sg.pdf_ok) {  // pdf_difference flanks (window.cpp:37-39), both evaluated
      const bool ok = warp_candidate_hist(P, vb, w, c, q == 1 ? sg.lo : sg.hi, 0, lane, &sup, &v);
      visits += (unsigned long long)v;
      if (lane == 0) okf[q] = ok;
    } else if (lane == 0) {
      okf[q] = 0;
    }
  }
  if (lane == 0) vis[q] = visits;
  __syncthreads();
  if (threadIdx.x == 0) {
    salvox_detection d;
    memset(&d, 0, sizeof d);
    d.seed_index = si.seed_index;
    d.H[0] = d.H[4] = d.H[8] = 1.0;
    d.iterations = iters;
    if (converged) d.flags |= SALVOX_FLAG_CONVERGED;
    d.center[0] = c[0];
    d.center[1] = c[1];
    d.center[2] = c[2];
    if (degenerate) {
      d.flags |= SALVOX_FLAG_DEGENERATE;
    } else if (P.post_score) {
      for (int i = 0; i < 9; ++i) d.H[i] = sg.H[i];
      if (okf[0]) {
        d.entropy_bits = score[0];
        d.bhattacharyya = score[1];
      }
      double pdf = 0.0;
      if (sg.pdf_ok && okf[1] && okf[2]) {
        double l1 = 0.0;
        for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(ps[2].p[b], ps[1].p[b])));
        pdf = __dmul_rn(sg.pdf_fac, l1);
      }
      d.pdf_diff = pdf;
    }
    unsigned long long tv = 0;
    for (int r = 0; r < NQ; ++r) tv += vis[r];
    P.out[si.slot] = d;
    P.visits[si.slot] = tv;
    if (P.ascent_out) {  // quadrant_seek_one's result (quadrant.cpp:276-282)
      salvox_ascent_result r;
      r.position[0] = p[0];
      r.position[1] = p[1];
      r.position[2] = p[2];
      r.iterations = iters;
      r.converged = converged;
      r.degenerate = degenerate;
      r.best_scale = degenerate ? 0 : best_scale;
      r.entropy_bits = degenerate ? 0.0 : best_entropy;
      P.ascent_out[si.slot] = r;
    }
  }
}

// ------------------------------------------------------------- window ops
// The building blocks of the seek path as callable operations (salvox_window_ops):
// the same warp routines as the seek kernels, so a pmf, a mean-shift step or a
// pdf difference computed here is the one a trajectory would compute.
struct WinOpDev {
  int op, kernel, step_kernel, min_vox;
  double c[3];
  double box[6];
  int geom;  // ScaleGeom of the op's window (HIST, SHIFT_STEP, PDF_DIFF)
  int pad_;
};

struct WinOpParams {
  int nx, ny, nz, bins, n;
  const uint8_t* binvol;
  const double* q;
  const ScaleGeom* geoms;
  const WinOpDev* ops;
  salvox_window_result* out;
  double* pmf;  // n x bins, nullable
};

// box_entropy_bits (quadrant.cpp:18-35) over an inclusive integer box: exact
// counts, p_b = count_b / count, entropy in bin order (sx_log)
__device__ double warp_box_entropy(const WinOpParams& P, const uint8_t* vb, WarpScratch& s,
                                   unsigned* cnt, const double* bx, int min_vox, int lane,
                                   unsigned long long* visits) {
  auto range = [](double a, double b, int n, int* lo, int* hi) {
    *lo = max(0, (int)ceil(a < b ? a : b));
    *hi = min(n - 1, (int)floor(a < b ? b : a));
  };
  Box B;
  range(bx[0], bx[1], P.nx, &B.x0, &B.x1);
  range(bx[2], bx[3], P.ny, &B.y0, &B.y1);
  range(bx[4], bx[5], P.nz, &B.z0, &B.z1);
  const long long count = box_size(B);
  if (count <= 0 || count < min_vox) return 0.0;
  for (int b = lane; b < P.bins; b += 32) cnt[b] = 0u;
  __syncwarp();
  warp_box_iter(B, lane, [&](bool act, int x, int y, int z) {
    if (act) atomicAdd(&cnt[(int)__ldg(vb + ((size_t)z * P.ny + y) * P.nx + x) - 1], 1u);
  });
  __syncwarp();
  *visits = (unsigned long long)count;
  for (int b = lane; b < P.bins; b += 32) s.p[b] = __ddiv_rn((double)cnt[b], (double)count);
  __syncwarp();
  return warp_entropy_bits(s.p, P.bins, lane, s.w);
}

template <int NW>
__global__ void __launch_bounds__(32 * NW) window_ops_kernel(const WinOpParams P) {
  __shared__ WarpScratch scratch[NW];
  __shared__ unsigned counts[NW][kMaxBins];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int job = blockIdx.x * NW + wid;
  if (job >= P.n) return;
  const WinOpDev op = P.ops[job];
  WarpScratch& s = scratch[wid];
  const uint8_t* vb = P.binvol;
  const int M = P.bins;
  salvox_window_result r;
  memset(&r, 0, sizeof r);
  if (op.op == SALVOX_WOP_BOX_ENTROPY) {
    unsigned long long v = 0;
    r.value[0] = warp_box_entropy(P, vb, s, counts[wid], op.box, op.min_vox, lane, &v);
    r.visits = v;
    r.ok = 1;
  } else if (op.op == SALVOX_WOP_PDF_DIFF) {
    const ScaleGeom& sg = P.geoms[op.geom];
    if (!sg.pdf_ok) {
      r.ok = -1;  // s - ds < 1: the reference throws before any pass
    } else {     // both flanks are evaluated before the check (window.cpp:37-39)
      const HistRes lo = warp_candidate_hist_impl(vb, P.nx, P.ny, P.nz, M, &s, op.c[0], op.c[1],
                                                  op.c[2], &sg.lo, op.kernel);
      for (int b = lane; b < M; b += 32) s.w[b] = s.p[b];
      __syncwarp();
      const HistRes hi = warp_candidate_hist_impl(vb, P.nx, P.ny, P.nz, M, &s, op.c[0], op.c[1],
                                                  op.c[2], &sg.hi, op.kernel);
      r.visits = (unsigned long long)(lo.visited + hi.visited);
      r.ok = lo.ok && hi.ok;
      if (r.ok && lane == 0) {
        double l1 = 0.0;
        for (int b = 0; b < M; ++b) l1 = __dadd_rn(l1, fabs(__dsub_rn(s.p[b], s.w[b])));
        r.value[0] = __dmul_rn(sg.pdf_fac, l1);
      }
    }
  } else {  // HIST, SHIFT_STEP: the candidate histogram at c first
    const ScaleGeom& sg = P.geoms[op.geom];
    const HistRes h = warp_candidate_hist_impl(vb, P.nx, P.ny, P.nz, M, &s, op.c[0], op.c[1],
                                               op.c[2], &sg.main, op.kernel);
    r.support = h.support;
    r.visits = (unsigned long long)h.visited;
    r.ok = h.ok;
    if (h.ok && P.pmf)
      for (int b = lane; b < M; b += 32) P.pmf[(size_t)job * M + b] = s.p[b];
    if (op.op == SALVOX_WOP_SHIFT_STEP && h.ok) {  // shift.cpp:21-33
      for (int b = lane; b < M; b += 32) {  // weight_for_bin (histogram.hpp:107-113)
        const double pb = s.p[b] > 1e-6 ? s.p[b] : 1e-6;
        s.w[b] = __dsqrt_rn(__ddiv_rn(P.q[b], pb));
      }
      __syncwarp();
      const CentRes cr = warp_centroid_impl(vb, P.nx, P.ny, P.nz, &s, op.c[0], op.c[1], op.c[2],
                                            &sg.main, op.step_kernel);
      r.visits += (unsigned long long)cr.visited;
      r.ok = cr.den > 0.0;
      if (r.ok)
        for (int a = 0; a < 3; ++a) r.value[a] = __ddiv_rn(cr.num[a], cr.den);
    }
  }
  if (lane == 0) P.out[job] = r;
}

// ------------------------------------------------------------------ selection
__global__ void alive_kernel(const salvox_detection* __restrict__ d, int n, double* e, double* pd,
                             unsigned char* alive) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool a = !(d[i].flags & SALVOX_FLAG_DEGENERATE) && d[i].entropy_bits > 0.0;
    alive[i] = a;
    e[i] = d[i].entropy_bits;
    pd[i] = d[i].pdf_diff;
  }
}

__global__ void passed_kernel(const salvox_detection* __restrict__ d, int n,
                              const unsigned char* alive, double et, double pt, double* key,
                              int* idx, unsigned char* pass) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool p = alive[i] && d[i].entropy_bits >= et && d[i].pdf_diff >= pt;  // pipeline.cpp:399
    pass[i] = p;
    key[i] = d[i].pdf_diff;
    idx[i] = i;
  }
}

// Greedy radius suppression over pdf-descending candidates (pipeline.cpp:168-183).
// One warp: lanes test the candidate against the kept list in parallel.
__global__ void dedupe_kernel(const salvox_detection* __restrict__ d, const int* order, int n,
                              int k, double radius, salvox_detection* out, int* n_out) {
  const int lane = threadIdx.x;
  int kept_n = 0;
  for (int i = 0; i < n && kept_n < k; ++i) {
    const salvox_detection& c = d[order[i]];
    bool clash = false;
    for (int a = lane; a < kept_n; a += 32) {
      const double dx = __dsub_rn(out[a].center[0], c.center[0]);
      const double dy = __dsub_rn(out[a].center[1], c.center[1]);
      const double dz = __dsub_rn(out[a].center[2], c.center[2]);
      const double nrm =
          __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      if (nrm <= radius) clash = true;
    }
    clash = __any_sync(kFull, clash);
    if (!clash) {
      if (lane == 0) out[kept_n] = c;
      ++kept_n;
      __syncwarp();
    }
  }
  if (lane == 0) *n_out = kept_n;
}

// ------------------------------------------------------------------ host side
namespace {

WinGeom make_geom(const Mat3& H, bool two_d) {
  WinGeom g{};
  const Mat3 Hi = eigen_inverse(H);
  std::memcpy(g.Hinv, Hi.m, sizeof g.Hinv);
  for (int i = 0; i < 3; ++i) g.ext[i] = std::sqrt(std::max(H.m[i * 4], 0.0));
  g.det_fac = 1.0 / std::sqrt(std::max(eigen_det(H), 1e-300));
  g.support_volume = support_volume(H, two_d);
  return g;
}

ScaleGeom make_scale_geom(const Mat3& H, bool two_d) {
  ScaleGeom sg{};
  sg.main = make_geom(H, two_d);
  std::memcpy(sg.H, H.m, sizeof sg.H);
  const double s = window_scale(H, two_d);
  const double ds = 1.0;
  sg.pdf_ok = !(s - ds < 1.0);
  if (sg.pdf_ok) {
    sg.lo = make_geom(window_scaled_to(H, s - ds, two_d), two_d);
    sg.hi = make_geom(window_scaled_to(H, s + ds, two_d), two_d);
    sg.pdf_fac = s * s / (2.0 * ds);
  }
  return sg;
}

struct SeekJob {
  std::vector<SeedIn> seeds;
  std::vector<ScaleGeom> geoms;
  std::vector<double> seed_H;  // ABMSOD: 9 per output slot
  SeekParams P{};
};

void check_window(const salvox_window* iw) {
  if (!iw) fail(SALVOX_EINVAL, "IntensityWindow: missing");
  if (!iw->full_range && !(iw->low < iw->high))
    fail(SALVOX_EINVAL, "IntensityWindow: low must be < high");
  if (iw->bins < 2) fail(SALVOX_EINVAL, "IntensityWindow: bins must be >= 2");
  if (iw->bins > kMaxBins) fail(SALVOX_EUNSUPPORTED, "seek (device): bins must be <= 64");
}

// Builds seeds + geometry for `method` (shift: one geometry per distinct scale;
// ascent: one per post-scoring half-size k).
void build_job(int nx, int ny, int nz, const salvox_detect_params* prm,
               const std::vector<SeedRec>& recs, const std::vector<int>& index, SeekJob& job) {
  const bool two_d = nz == 1;
  const int method = prm->method;
  SeekParams& P = job.P;
  P.nx = nx;
  P.ny = ny;
  P.nz = nz;
  P.method = method;
  P.two_d = two_d;
  if (method == SALVOX_METHOD_SHIFT) {
    if (prm->shift_min_step <= 0.0) fail(SALVOX_EINVAL, "shift: min_step must be > 0");
    if (prm->shift_max_iters < 1) fail(SALVOX_EINVAL, "shift: max_iters must be >= 1");
    P.max_iters = prm->shift_max_iters;
    P.min_step = prm->shift_min_step;
    P.step_kernel = prm->shift_step_kernel;
    P.hist_kernel = prm->shift_hist_kernel;
    P.min_frac = prm->shift_min_inbounds_fraction;
    std::map<std::array<double, 3>, int> gi;
    for (size_t i = 0; i < recs.size(); ++i) {
      const double s = recs[i].scale;
      // pipeline.cpp:365 half = (s, s, 2D ? 1 : s); shift.cpp:9 pins z to 1 in 2D
      std::array<double, 3> half = {s, s, s};
      if (recs[i].half[0] != 0.0 || recs[i].half[1] != 0.0 || recs[i].half[2] != 0.0)
        half = {recs[i].half[0], recs[i].half[1], recs[i].half[2]};
      if (!(half[0] > 0.0 && half[1] > 0.0 && half[2] > 0.0))
        fail(SALVOX_EINVAL, "shift: half extents must be > 0");  // shift.hpp:28-29
      if (two_d) half[2] = 1.0;
      auto it = gi.find(half);
      if (it == gi.end()) {
        it = gi.emplace(half, (int)job.geoms.size()).first;
        job.geoms.push_back(make_scale_geom(diag_from_half(half[0], half[1], half[2]), two_d));
      }
      SeedIn si{};
      std::memcpy(si.pos, recs[i].pos, sizeof si.pos);
      si.geom = it->second;
      si.seed_index = index[i];
      si.slot = (int)i;
      job.seeds.push_back(si);
    }
    // longest-processing-time first: seeds with the largest windows launch first
    std::stable_sort(job.seeds.begin(), job.seeds.end(), [&](const SeedIn& a, const SeedIn& b) {
      return job.geoms[a.geom].main.support_volume > job.geoms[b.geom].main.support_volume;
    });
  } else if (method == SALVOX_METHOD_ABMSOD) {
    // AbmsodParams::validate (abmsod.hpp:27-31)
    if (prm->abmsod_threshold <= 0.0) fail(SALVOX_EINVAL, "abmsod: threshold must be > 0");
    if (prm->abmsod_max_iters < 1) fail(SALVOX_EINVAL, "abmsod: max_iterations must be >= 1");
    if (prm->abmsod_lambda_min <= 0.0) fail(SALVOX_EINVAL, "abmsod: lambda_min must be > 0");
    if (prm->abmsod_kernel < 0 || prm->abmsod_kernel > 2) fail(SALVOX_EINVAL, "unknown kernel");
    P.abm_threshold = prm->abmsod_threshold;
    P.abm_max_iters = prm->abmsod_max_iters;
    P.abm_kernel = prm->abmsod_kernel;
    P.abm_lmin = prm->abmsod_lambda_min;
    double lmax = prm->abmsod_lambda_max;  // lambda_max_for (abmsod.hpp:34-38)
    if (!(lmax > 0.0)) {
      const double half = std::max({nx, ny, nz}) / 2.0;
      lmax = half * half;
    }
    P.abm_lmax = lmax;
    P.abm_min_frac = prm->abmsod_min_inbounds_fraction;
    job.seed_H.assign(recs.size() * 9, 0.0);
    for (size_t i = 0; i < recs.size(); ++i) {
      // EllipsoidWindow::isotropic(position, scale, 2D) (pipeline.cpp:373-374)
      const double r = recs[i].scale;
      double* H = &job.seed_H[9 * i];
      H[0] = r * r;
      H[4] = r * r;
      H[8] = two_d ? 1.0 : r * r;
      SeedIn si{};
      std::memcpy(si.pos, recs[i].pos, sizeof si.pos);
      si.seed_index = index[i];
      si.slot = (int)i;
      job.seeds.push_back(si);
    }
    std::stable_sort(job.seeds.begin(), job.seeds.end(), [&](const SeedIn& a, const SeedIn& b) {
      return job.seed_H[9 * a.slot] > job.seed_H[9 * b.slot];  // larger windows first
    });
  } else {
    std::vector<int> ks;
    if (prm->n_quadrant_scales > 0) {
      ks.assign(prm->quadrant_scales, prm->quadrant_scales + prm->n_quadrant_scales);
    } else {
      for (int i = 0; i < prm->n_scales; ++i) ks.push_back((int)std::lround(prm->scales[i]));
    }
    if (ks.empty()) fail(SALVOX_EINVAL, "quadrant: empty scale range");
    for (size_t i = 1; i < ks.size(); ++i)
      if (ks[i] <= ks[i - 1]) fail(SALVOX_EINVAL, "quadrant: scale range must be strictly increasing");
    if (prm->quadrant_eta <= 0.0) fail(SALVOX_EINVAL, "quadrant: eta must be > 0");
    if (prm->quadrant_max_iters < 1) fail(SALVOX_EINVAL, "quadrant: max_iters must be >= 1");
    if ((int)ks.size() > 64 || ks.back() > 128 || ks.front() < 0)
      fail(SALVOX_EUNSUPPORTED, "ascent (device): at most 64 scales in [0, 128]");
    P.max_iters = prm->quadrant_max_iters;
    P.eta = prm->quadrant_eta;
    P.post_score = 1;
    P.ascent_out = nullptr;
    P.n_ascent = (int)ks.size();
    for (size_t i = 0; i < ks.size(); ++i) P.ascent_scales[i] = ks[i];
    for (int k = 0; k <= 128; ++k) P.geom_of_k[k] = 0;
    std::vector<int> post = {2};
    for (int k : ks) post.push_back(std::max(2, k));
    for (int k : post) {
      if (P.geom_of_k[k] != 0 || (k == 2 && !job.geoms.empty())) continue;
      P.geom_of_k[k] = (int)job.geoms.size();
      const double kd = (double)k;
      job.geoms.push_back(make_scale_geom(diag_from_half(kd, kd, two_d ? 1.0 : kd), two_d));
    }
    for (size_t i = 0; i < recs.size(); ++i) {
      SeedIn si{};
      std::memcpy(si.pos, recs[i].pos, sizeof si.pos);
      si.geom = 0;
      si.seed_index = index[i];
      si.slot = (int)i;
      job.seeds.push_back(si);
    }
  }
}

// Level-table ascent when its per-warp tables fit (<= 160 KB per CTA), else the
// shell-by-shell kernel (many scales x many bins).
template <int NQ>
void launch_ascent_nq(salvox_ctx* ctx, SeekParams& P) {
  const size_t per_warp = AscentLayout::bytes(P.n_ascent, P.bins);
  static const bool force_shell = std::getenv("SALVOX_ASCENT_SHELL") != nullptr;
  if (!force_shell && per_warp * NQ <= 160 * 1024) {
    P.asc_warp_bytes = (int)per_warp;
    const int dyn = (int)(per_warp * NQ);
    SX_CUDA(cudaFuncSetAttribute(ascent_kernel<NQ, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    ascent_kernel<NQ, true><<<P.n_seeds, 32 * NQ, dyn, ctx->stream>>>(P);
  } else {
    P.asc_warp_bytes = 0;
    ascent_kernel<NQ, false><<<P.n_seeds, 32 * NQ, 0, ctx->stream>>>(P);
  }
}

void launch_ascent(salvox_ctx* ctx, SeekParams& P) {
  if (P.method == SALVOX_METHOD_QUADRANT)
    launch_ascent_nq<4>(ctx, P);
  else
    launch_ascent_nq<8>(ctx, P);
}

// Seek engine for shift: the CTA engine for few seeds (latency-bound), the
// one-warp-per-seed kernel with an 80-register cap when the seeds fill the GPU
// several times (throughput-bound). SALVOX_SEEK_ENGINE = cta | warp | warp12
// forces one (tests cover all three).
int seek_engine(int n_seeds, int sm_count) {
  static const int forced = [] {
    const char* e = std::getenv("SALVOX_SEEK_ENGINE");
    if (!e) return -1;
    const std::string v(e);
    return v == "cta" ? 0 : v == "warp" ? 1 : v == "warp12" ? 2 : -1;
  }();
  if (forced >= 0) return forced;
  return (long long)n_seeds > 64LL * sm_count ? 2 : 0;
}

constexpr int kCtaProducers = CTA_PRODUCERS;

template <int NP, class K>
void launch_cta(K kern, salvox_ctx* ctx, const SeekParams& P) {
  const int bytes = (int)sizeof(CtaShared<NP>);
  SX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  kern<<<P.n_seeds, 32 * (NP + 1), bytes, ctx->stream>>>(P);
}

// Runs the seek kernel for one volume whose bins are already on the device.
void run_seek(salvox_ctx* ctx, SeekJob& job, const uint8_t* d_bins, int bins, const double* d_q,
              salvox_detection* d_out, unsigned long long* d_visits) {
  SeekParams& P = job.P;
  P.bins = bins;
  P.binvol = d_bins;
  P.vol_stride = (size_t)P.nx * P.ny * P.nz;
  P.q = d_q;
  P.n_seeds = (int)job.seeds.size();
  P.out = d_out;
  P.visits = d_visits;
  if (P.n_seeds == 0) return;
  auto up = [](size_t b) { return ((b + 255) / 256) * 256; };
  const size_t gbytes = job.geoms.size() * sizeof(ScaleGeom);
  const size_t sbytes = job.seeds.size() * sizeof(SeedIn);
  const size_t hbytes = job.seed_H.size() * sizeof(double);
  char* d_geo = static_cast<char*>(ctx->d_geom.ensure(up(gbytes) + up(sbytes) + up(hbytes) + 256));
  char* d_sd = d_geo + up(gbytes);
  char* d_h = d_sd + up(sbytes);
  int* d_err = reinterpret_cast<int*>(d_h + up(hbytes));
  if (gbytes)
    SX_CUDA(cudaMemcpyAsync(d_geo, job.geoms.data(), gbytes, cudaMemcpyHostToDevice, ctx->stream));
  SX_CUDA(cudaMemcpyAsync(d_sd, job.seeds.data(), sbytes, cudaMemcpyHostToDevice, ctx->stream));
  if (hbytes)
    SX_CUDA(cudaMemcpyAsync(d_h, job.seed_H.data(), hbytes, cudaMemcpyHostToDevice, ctx->stream));
  SX_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), ctx->stream));
  P.geoms = reinterpret_cast<const ScaleGeom*>(d_geo);
  P.seeds = reinterpret_cast<const SeedIn*>(d_sd);
  P.seed_H = reinterpret_cast<const double*>(d_h);
  P.err_flag = d_err;
  const int engine = seek_engine(P.n_seeds, ctx->sm_count);
  if (P.method == SALVOX_METHOD_ABMSOD && engine == 0)
    launch_cta<kCtaProducers>(abmsod_cta_kernel<kCtaProducers>, ctx, P);
  else if (P.method == SALVOX_METHOD_ABMSOD)
    abmsod_kernel<2><<<(P.n_seeds + 1) / 2, 64, 0, ctx->stream>>>(P);
  else if (P.method == SALVOX_METHOD_SHIFT && engine == 0)
    launch_cta<kCtaProducers>(shift_cta_kernel<kCtaProducers>, ctx, P);
  else if (P.method == SALVOX_METHOD_SHIFT && engine == 2)
    shift_kernel<2, 12><<<(P.n_seeds + 1) / 2, 64, 0, ctx->stream>>>(P);
  else if (P.method == SALVOX_METHOD_SHIFT)
    shift_kernel<2, 1><<<(P.n_seeds + 1) / 2, 64, 0, ctx->stream>>>(P);
  else
    launch_ascent(ctx, P);
  SX_LAUNCH_CHECK(ctx);
  if (P.method == SALVOX_METHOD_ABMSOD) {
    int err = 0;
    SX_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (err) fail(SALVOX_ERUNTIME, "abmsod: eigen decomposition failed");  // abmsod.cpp:16-17
  }
}

// Bins one device volume (K1, pitch nx) into d_bins (n bytes).
void bin_into(salvox_ctx* ctx, const float* d_vol, int nx, int ny, int nz, const salvox_window* iw,
              uint8_t* d_bins) {
  double low = iw->low, high = iw->high;
  const size_t n = (size_t)nx * ny * nz;
  if (iw->full_range) device_full_range(ctx, d_vol, n, &low, &high);
  launch_bin_volume(ctx, d_vol, d_bins, nx, ny, nz, nx, low, high, iw->bins);
}

// Uploads the target pmf (uniform unless given). A given target is used as is,
// like ShiftParams/AbmsodParams::target (a Histogram) in the C++ reference; the
// Python layer normalises arrays first (histogram_from_array, py_module.cpp:46-54).
double* upload_target(salvox_ctx* ctx, const salvox_window* iw, const double* target) {
  std::vector<double> q(iw->bins);
  if (target) {
    for (int b = 0; b < iw->bins; ++b) q[b] = target[b];
  } else {
    for (int b = 0; b < iw->bins; ++b) q[b] = 1.0 / iw->bins;  // Histogram::uniform
  }
  double* d_q = static_cast<double*>(ctx->d_target.ensure(q.size() * 8));
  SX_CUDA(cudaMemcpyAsync(d_q, q.data(), q.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));  // q lives on this stack frame
  return d_q;
}

// Bins a device volume into the context's bin buffer and uploads the target pmf.
const uint8_t* prepare_volume(salvox_ctx* ctx, const float* d_vol, int nx, int ny, int nz,
                              const salvox_window* iw, const double* target, double** d_q) {
  uint8_t* d_bins = static_cast<uint8_t*>(ctx->d_seek_bins.ensure((size_t)nx * ny * nz));
  bin_into(ctx, d_vol, nx, ny, nz, iw, d_bins);
  *d_q = upload_target(ctx, iw, target);
  return d_bins;
}

// Replicates a job's seeds over `batch` volumes: one launch covers every volume,
// output rows vol * ns + slot. The longest-window-first order is kept.
void expand_batch(SeekJob& job, int batch) {
  if (batch <= 1) return;
  const int ns = (int)job.seeds.size();
  std::vector<SeedIn> all;
  all.reserve((size_t)ns * batch);
  for (const SeedIn& si : job.seeds)
    for (int v = 0; v < batch; ++v) {
      SeedIn t = si;
      t.vol = v;
      t.slot = v * ns + si.slot;
      all.push_back(t);
    }
  job.seeds.swap(all);
  if (!job.seed_H.empty()) {
    std::vector<double> h((size_t)ns * batch * 9);
    for (int v = 0; v < batch; ++v) std::copy(job.seed_H.begin(), job.seed_H.end(), h.begin() + (size_t)v * ns * 9);
    job.seed_H.swap(h);
  }
}

// Device selection: thresholds + dedupe over n detections at d_dets. Returns
// the number kept, written to d_kept (device).
int device_select(salvox_ctx* ctx, const salvox_detection* d_dets, int n, double qe, double qp,
                  int k, double radius, bool thresholds, salvox_detection* d_kept) {
  if (n <= 0 || k <= 0) return 0;
  cudaStream_t st = ctx->stream;
  const int blocks = std::min((n + 255) / 256, ctx->sm_count * 8);
  // scratch: 4 double arrays + 2 int arrays + 2 flag arrays
  char* base = static_cast<char*>(ctx->d_sel_a.ensure((size_t)n * (8 * 4 + 4 * 2 + 2) + 4096));
  double* e = reinterpret_cast<double*>(base);
  double* pd = e + n;
  double* e2 = pd + n;
  double* pd2 = e2 + n;
  int* idx = reinterpret_cast<int*>(pd2 + n);
  int* idx2 = idx + n;
  unsigned char* alive = reinterpret_cast<unsigned char*>(idx2 + n);
  unsigned char* pass = alive + n;
  int* d_cnt = static_cast<int*>(ctx->d_sel_b.ensure(64));
  double et = -INFINITY, pt = -INFINITY;
  alive_kernel<<<blocks, 256, 0, st>>>(d_dets, n, e, pd, alive);
  SX_LAUNCH_CHECK(ctx);
  if (thresholds) {
    size_t t1 = 0, t2 = 0;
    SX_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, e, alive, e2, d_cnt, n, st));
    SX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t2, e2, e, n, 0, 64, st));
    void* tmp = ctx->d_cub.ensure(std::max(t1, t2));
    SX_CUDA(cub::DeviceSelect::Flagged(tmp, t1, e, alive, e2, d_cnt, n, st));
    SX_CUDA(cub::DeviceSelect::Flagged(tmp, t1, pd, alive, pd2, d_cnt + 1, n, st));
    int na = 0;
    SX_CUDA(cudaMemcpyAsync(&na, d_cnt, 4, cudaMemcpyDeviceToHost, st));
    SX_CUDA(cudaStreamSynchronize(st));
    if (na == 0) return 0;  // pipeline.cpp:387
    SX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t2, e2, e, na, 0, 64, st));
    tmp = ctx->d_cub.ensure(t2);
    SX_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t2, e2, e, na, 0, 64, st));
    SX_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t2, pd2, pd, na, 0, 64, st));
    ctx->launches += 10;
    // quantile_threshold (pipeline.cpp:54-59)
    const size_t ie = (size_t)std::floor(qe * double(na - 1));
    const size_t ip = (size_t)std::floor(qp * double(na - 1));
    SX_CUDA(cudaMemcpyAsync(&et, e + ie, 8, cudaMemcpyDeviceToHost, st));
    SX_CUDA(cudaMemcpyAsync(&pt, pd + ip, 8, cudaMemcpyDeviceToHost, st));
    SX_CUDA(cudaStreamSynchronize(st));
  } else {
    SX_CUDA(cudaMemsetAsync(alive, 1, n, st));
  }
  passed_kernel<<<blocks, 256, 0, st>>>(d_dets, n, alive, et, pt, e, idx, pass);
  SX_LAUNCH_CHECK(ctx);
  size_t t1 = 0, t2 = 0;
  SX_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, e, pass, e2, d_cnt, n, st));
  SX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, t2, e2, pd2, idx2, idx, n, 0, 64, st));
  void* tmp = ctx->d_cub.ensure(std::max(t1, t2));
  SX_CUDA(cub::DeviceSelect::Flagged(tmp, t1, e, pass, e2, d_cnt, n, st));
  SX_CUDA(cub::DeviceSelect::Flagged(tmp, t1, idx, pass, idx2, d_cnt + 1, n, st));
  int np = 0;
  SX_CUDA(cudaMemcpyAsync(&np, d_cnt, 4, cudaMemcpyDeviceToHost, st));
  SX_CUDA(cudaStreamSynchronize(st));
  if (np == 0) return 0;
  // stable sort by pdf_diff descending (pipeline.cpp:169-170): radix sort is stable
  SX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, t2, e2, pd2, idx2, idx, np, 0, 64, st));
  tmp = ctx->d_cub.ensure(t2);
  SX_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, t2, e2, pd2, idx2, idx, np, 0, 64, st));
  ctx->launches += 8;
  dedupe_kernel<<<1, 32, 0, st>>>(d_dets, idx, np, k, radius, d_kept, d_cnt + 2);
  SX_LAUNCH_CHECK(ctx);
  int kept = 0;
  SX_CUDA(cudaMemcpyAsync(&kept, d_cnt + 2, 4, cudaMemcpyDeviceToHost, st));
  SX_CUDA(cudaStreamSynchronize(st));
  return kept;
}

void plan_and_dedupe(int nx, int ny, int nz, const salvox_detect_params* prm,
                     std::vector<SeedRec>& recs, std::vector<int>& index) {
  std::vector<SeedRec> all;
  plan_seeds(nx, ny, nz, prm->seed_mode, prm->seed_spacing, prm->seed_count, prm->scales,
             prm->n_scales, prm->rng_seed, all);
  recs.clear();
  index.clear();
  if (prm->method == SALVOX_METHOD_SHIFT || prm->method == SALVOX_METHOD_ABMSOD) {
    recs = all;  // one trajectory per seed (pipeline.cpp:360-379)
    for (size_t i = 0; i < all.size(); ++i) index.push_back((int)i);
    return;
  }
  // one trajectory per distinct consecutive position (pipeline.cpp:325-331)
  for (size_t i = 0; i < all.size(); ++i) {
    if (!recs.empty() && recs.back().pos[0] == all[i].pos[0] && recs.back().pos[1] == all[i].pos[1] &&
        (prm->method == SALVOX_METHOD_QUADRANT || recs.back().pos[2] == all[i].pos[2]))
      continue;
    recs.push_back(all[i]);
    index.push_back((int)i);
  }
}

const double* target_of(const salvox_detect_params* prm) {
  return prm->method == SALVOX_METHOD_ABMSOD ? prm->abmsod_target : prm->shift_target;
}

void check_method(const salvox_detect_params* prm, int nz) {
  if (!prm) fail(SALVOX_EINVAL, "null params");
  if (prm->method == SALVOX_METHOD_QUADRANT && nz != 1)
    fail(SALVOX_EINVAL, "detect: quadrant method requires a 2D volume (nz == 1)");
  if (prm->method != SALVOX_METHOD_QUADRANT && prm->method != SALVOX_METHOD_SHIFT &&
      prm->method != SALVOX_METHOD_OCTANT && prm->method != SALVOX_METHOD_ABMSOD)
    fail(SALVOX_EINVAL, "unknown method");
  for (int k : {prm->shift_step_kernel, prm->shift_hist_kernel})
    if (prm->method == SALVOX_METHOD_SHIFT && (k < 0 || k > 2)) fail(SALVOX_EINVAL, "unknown kernel");
}

unsigned long long sum_visits(salvox_ctx* ctx, const unsigned long long* d_v, int n) {
  if (n <= 0) return 0;
  std::vector<unsigned long long> h((size_t)n);
  SX_CUDA(cudaMemcpyAsync(h.data(), d_v, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  unsigned long long s = 0;
  for (auto v : h) s += v;
  return s;
}

}  // namespace
}  // namespace sx

using namespace sx;

extern "C" int salvox_detect(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                             int32_t nz, const salvox_window* iw, const salvox_detect_params* prm,
                             salvox_detection* out, int64_t cap, int64_t* n_out,
                             salvox_detection* per_seed, int64_t cap_seed, int64_t* n_seed,
                             uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (!volume) fail(SALVOX_EINVAL, "null volume");
    check_method(prm, nz);
    check_window(iw);
    std::vector<SeedRec> recs;
    std::vector<int> index;
    plan_and_dedupe(nx, ny, nz, prm, recs, index);
    SeekJob job;
    build_job(nx, ny, nz, prm, recs, index, job);
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t n = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(n * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, target_of(prm), &d_q);
    const int ns = (int)job.seeds.size();
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure((size_t)(ns + 1) * (sizeof(salvox_detection) + 8) * 2 + 512));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    salvox_detection* d_kept = d_all + (ns + 1);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_kept + (ns + 1));
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    const int kept = device_select(ctx, d_all, ns, prm->entropy_quantile, prm->pdf_quantile,
                                   prm->top_k, prm->dedupe_radius, true, d_kept);
    if (out && cap > 0 && kept > 0)
      SX_CUDA(cudaMemcpyAsync(out, d_kept, (size_t)std::min<int64_t>(kept, cap) * sizeof(salvox_detection),
                              cudaMemcpyDeviceToHost, ctx->stream));
    if (per_seed && cap_seed > 0 && ns > 0)
      SX_CUDA(cudaMemcpyAsync(per_seed, d_all, (size_t)std::min<int64_t>(ns, cap_seed) * sizeof(salvox_detection),
                              cudaMemcpyDeviceToHost, ctx->stream));
    const unsigned long long v = sum_visits(ctx, d_vis, ns);
    if (visits) *visits += v;
    if (n_out) *n_out = kept;
    if (n_seed) *n_seed = ns;
  });
}

extern "C" int salvox_detect_batch_device(salvox_ctx* ctx, const float* d_volumes, int32_t batch,
                                          int32_t nx, int32_t ny, int32_t nz,
                                          const salvox_window* iw,
                                          const salvox_detect_params* prm, salvox_detection* out,
                                          int64_t cap, int64_t* n_out, uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1 || batch < 0) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    check_method(prm, nz);
    check_window(iw);
    std::vector<SeedRec> recs;
    std::vector<int> index;
    plan_and_dedupe(nx, ny, nz, prm, recs, index);
    SeekJob job;
    build_job(nx, ny, nz, prm, recs, index, job);
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t n = (size_t)nx * ny * nz;
    const int ns = (int)job.seeds.size();
    const size_t nall = (size_t)ns * std::max(batch, 1) + 1;
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure(nall * (sizeof(salvox_detection) + 8) + (ns + 1) * sizeof(salvox_detection) + 512));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    salvox_detection* d_kept = d_all + nall;
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_kept + (ns + 1));
    if (batch == 0 || ns == 0) {
      for (int v = 0; v < batch; ++v)
        if (n_out) n_out[v] = 0;
      return;
    }
    // all volumes binned into one buffer, then ONE seek launch over batch x ns seeds
    uint8_t* d_bins = static_cast<uint8_t*>(ctx->d_seek_bins.ensure(n * batch));
    for (int v = 0; v < batch; ++v)
      bin_into(ctx, d_volumes + (size_t)v * n, nx, ny, nz, iw, d_bins + (size_t)v * n);
    const double* d_q = upload_target(ctx, iw, target_of(prm));
    expand_batch(job, batch);
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    for (int v = 0; v < batch; ++v) {
      const int kept = device_select(ctx, d_all + (size_t)v * ns, ns, prm->entropy_quantile,
                                     prm->pdf_quantile, prm->top_k, prm->dedupe_radius, true, d_kept);
      if (out && cap > 0 && kept > 0)
        SX_CUDA(cudaMemcpyAsync(out + (size_t)v * cap, d_kept,
                                (size_t)std::min<int64_t>(kept, cap) * sizeof(salvox_detection),
                                cudaMemcpyDeviceToHost, ctx->stream));
      if (n_out) n_out[v] = kept;
    }
    const unsigned long long vs = sum_visits(ctx, d_vis, ns * batch);
    if (visits) *visits += vs;
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

extern "C" int salvox_detect_shard(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                   int32_t nz, const salvox_window* iw,
                                   const salvox_detect_params* prm, int32_t rank, int32_t world,
                                   salvox_detection* per_seed, int64_t cap, int64_t* n_local,
                                   int64_t* n_total, uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (!volume) fail(SALVOX_EINVAL, "null volume");
    if (world < 1 || rank < 0 || rank >= world) fail(SALVOX_EINVAL, "shard: need 0 <= rank < world");
    check_method(prm, nz);
    check_window(iw);
    std::vector<SeedRec> all_recs, recs;
    std::vector<int> all_index, index;
    plan_and_dedupe(nx, ny, nz, prm, all_recs, all_index);
    // seed-order interleave: trajectory j belongs to rank j % world
    for (size_t j = (size_t)rank; j < all_recs.size(); j += (size_t)world) {
      recs.push_back(all_recs[j]);
      index.push_back(all_index[j]);
    }
    const int64_t ns = (int64_t)recs.size();
    if (n_total) *n_total = (int64_t)all_recs.size();
    if (n_local) *n_local = ns;
    if (ns > cap || (ns > 0 && !per_seed)) fail(SALVOX_EINVAL, "shard: per_seed capacity too small");
    SeekJob job;
    build_job(nx, ny, nz, prm, recs, index, job);
    if (ns == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t n = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(n * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, target_of(prm), &d_q);
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure((size_t)(ns + 1) * (sizeof(salvox_detection) + 8) + 512));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_all + (ns + 1));
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    SX_CUDA(cudaMemcpyAsync(per_seed, d_all, (size_t)ns * sizeof(salvox_detection),
                            cudaMemcpyDeviceToHost, ctx->stream));
    const unsigned long long v = sum_visits(ctx, d_vis, (int)ns);
    if (visits) *visits += v;
  });
}

extern "C" int salvox_seek(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                           int32_t nz, const salvox_window* iw, const salvox_detect_params* prm,
                           const double* seed_positions, const double* seed_scales,
                           const double* seed_half_extents, const int32_t* seed_index, int64_t n,
                           salvox_detection* out, uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    check_method(prm, nz);
    check_window(iw);
    if (n < 0 || (n > 0 && (!seed_positions || !out))) fail(SALVOX_EINVAL, "bad seed arrays");
    std::vector<SeedRec> recs((size_t)n);
    std::vector<int> index((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      std::memcpy(recs[i].pos, seed_positions + 3 * i, 3 * sizeof(double));
      recs[i].scale = seed_scales ? seed_scales[i] : 8.0;
      if (seed_half_extents) std::memcpy(recs[i].half, seed_half_extents + 3 * i, 3 * sizeof(double));
      index[i] = seed_index ? seed_index[i] : (int)i;
    }
    SeekJob job;
    build_job(nx, ny, nz, prm, recs, index, job);
    if (n == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(nv * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, target_of(prm), &d_q);
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure((size_t)(n + 1) * (sizeof(salvox_detection) + 8) * 2 + 512));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_all + 2 * (n + 1));
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    SX_CUDA(cudaMemcpyAsync(out, d_all, (size_t)n * sizeof(salvox_detection), cudaMemcpyDeviceToHost,
                            ctx->stream));
    const unsigned long long v = sum_visits(ctx, d_vis, (int)n);
    if (visits) *visits += v;
  });
}

extern "C" int salvox_ascent_seek(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                  int32_t nz, const salvox_window* iw, int32_t dims,
                                  const int32_t* scales, int32_t n_scales, double eta,
                                  int32_t max_iters, const double* seeds, int64_t n,
                                  salvox_ascent_result* out, uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (dims != 2 && dims != 3) fail(SALVOX_EINVAL, "ascent: dims must be 2 or 3");
    if (dims == 2 && nz != 1)
      fail(SALVOX_EINVAL, "quadrant_step: volume must be 2D (nz == 1)");  // quadrant.cpp:42
    check_window(iw);
    if (n < 0 || (n > 0 && (!seeds || !out))) fail(SALVOX_EINVAL, "bad seed arrays");
    salvox_detect_params prm{};
    prm.method = dims == 2 ? SALVOX_METHOD_QUADRANT : SALVOX_METHOD_OCTANT;
    prm.quadrant_scales = scales;
    prm.n_quadrant_scales = n_scales;
    prm.quadrant_eta = eta;
    prm.quadrant_max_iters = max_iters;
    if (n_scales < 1 || !scales) fail(SALVOX_EINVAL, "quadrant: empty scale range");
    std::vector<SeedRec> recs((size_t)n);
    std::vector<int> index((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      std::memcpy(recs[i].pos, seeds + 3 * i, 3 * sizeof(double));
      recs[i].scale = 0.0;
      index[i] = (int)i;
    }
    SeekJob job;
    build_job(nx, ny, nz, &prm, recs, index, job);
    if (n == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(nv * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, nullptr, &d_q);
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure(
        (size_t)(n + 1) * (sizeof(salvox_detection) + 8 + sizeof(salvox_ascent_result)) + 1024));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_all + (n + 1));
    salvox_ascent_result* d_res = reinterpret_cast<salvox_ascent_result*>(d_vis + (n + 1));
    job.P.post_score = 0;
    job.P.ascent_out = d_res;
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    SX_CUDA(cudaMemcpyAsync(out, d_res, (size_t)n * sizeof(salvox_ascent_result),
                            cudaMemcpyDeviceToHost, ctx->stream));
    const unsigned long long v = sum_visits(ctx, d_vis, (int)n);
    if (visits) *visits += v;
  });
}

extern "C" int salvox_ascent_step(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                  int32_t nz, const salvox_window* iw, int32_t dims,
                                  const int32_t* scales, int32_t n_scales, const double* points,
                                  int64_t n, double* moved, salvox_ascent_state* states,
                                  uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (dims != 2 && dims != 3) fail(SALVOX_EINVAL, "ascent: dims must be 2 or 3");
    if (dims == 2 && nz != 1)
      fail(SALVOX_EINVAL, "quadrant_step: volume must be 2D (nz == 1)");  // quadrant.cpp:42
    check_window(iw);
    if (n < 0 || (n > 0 && !points)) fail(SALVOX_EINVAL, "bad point arrays");
    salvox_detect_params prm{};
    prm.method = dims == 2 ? SALVOX_METHOD_QUADRANT : SALVOX_METHOD_OCTANT;
    prm.quadrant_scales = scales;
    prm.n_quadrant_scales = n_scales;
    prm.quadrant_eta = 1.0;
    prm.quadrant_max_iters = 1;  // one step (quadrant.cpp:37-81)
    if (n_scales < 1 || !scales) fail(SALVOX_EINVAL, "quadrant: empty scale range");
    std::vector<SeedRec> recs((size_t)n);
    std::vector<int> index((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      std::memcpy(recs[i].pos, points + 3 * i, 3 * sizeof(double));
      recs[i].scale = 0.0;
      index[i] = (int)i;
    }
    SeekJob job;
    build_job(nx, ny, nz, &prm, recs, index, job);
    if (n == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(nv * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, nullptr, &d_q);
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure(
        (size_t)(n + 1) * (sizeof(salvox_detection) + 8 + sizeof(salvox_ascent_result) +
                           sizeof(salvox_ascent_state)) + 1024));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_all + (n + 1));
    salvox_ascent_result* d_res = reinterpret_cast<salvox_ascent_result*>(d_vis + (n + 1));
    salvox_ascent_state* d_st = reinterpret_cast<salvox_ascent_state*>(d_res + (n + 1));
    job.P.post_score = 0;
    job.P.ascent_out = d_res;
    job.P.ascent_state = d_st;
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    std::vector<salvox_ascent_result> res((size_t)n);
    SX_CUDA(cudaMemcpyAsync(res.data(), d_res, (size_t)n * sizeof(salvox_ascent_result),
                            cudaMemcpyDeviceToHost, ctx->stream));
    if (states)
      SX_CUDA(cudaMemcpyAsync(states, d_st, (size_t)n * sizeof(salvox_ascent_state),
                              cudaMemcpyDeviceToHost, ctx->stream));
    const unsigned long long v = sum_visits(ctx, d_vis, (int)n);
    if (moved)
      for (int64_t i = 0; i < n; ++i) std::memcpy(moved + 3 * i, res[i].position, 3 * sizeof(double));
    if (visits) *visits += v;
  });
}

extern "C" int salvox_window_ops(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                 int32_t nz, const salvox_window* iw, const double* target,
                                 const salvox_window_op* ops, int64_t n, salvox_window_result* out,
                                 double* pmf_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    check_window(iw);
    if (n < 0 || (n > 0 && (!ops || !out))) fail(SALVOX_EINVAL, "bad op arrays");
    if (n > (int64_t)1 << 30) fail(SALVOX_EINVAL, "window ops: too many ops in one call");
    if (n == 0) return;
    const bool two_d = nz == 1;
    std::vector<WinOpDev> dev((size_t)n);
    std::vector<ScaleGeom> geoms;
    for (int64_t i = 0; i < n; ++i) {
      const salvox_window_op& o = ops[i];
      if (o.op < SALVOX_WOP_HIST || o.op > SALVOX_WOP_BOX_ENTROPY) fail(SALVOX_EINVAL, "unknown window op");
      if (o.kernel < 0 || o.kernel > 2 || o.step_kernel < 0 || o.step_kernel > 2)
        fail(SALVOX_EINVAL, "unknown kernel");
      WinOpDev& d = dev[i];
      d.op = o.op, d.kernel = o.kernel, d.step_kernel = o.step_kernel, d.min_vox = o.min_voxels;
      std::memcpy(d.c, o.center, sizeof d.c);
      std::memcpy(d.box, o.box, sizeof d.box);
      d.geom = 0;
      if (o.op != SALVOX_WOP_BOX_ENTROPY) {  // window geometry on the host (glibc pow/sqrt,
        Mat3 H;                             // Eigen's 3x3 inverse/determinant) like the seeds'
        std::memcpy(H.m, o.H, sizeof H.m);
        d.geom = (int)geoms.size();
        geoms.push_back(make_scale_geom(H, two_d));
      }
    }
    if (geoms.empty()) geoms.push_back(ScaleGeom{});
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(nv * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, target, &d_q);
    auto up = [](size_t b) { return ((b + 255) / 256) * 256; };
    const size_t ob = dev.size() * sizeof(WinOpDev), gb = geoms.size() * sizeof(ScaleGeom);
    const size_t rb = (size_t)n * sizeof(salvox_window_result);
    const size_t pb = pmf_out ? (size_t)n * iw->bins * sizeof(double) : 0;
    char* d = static_cast<char*>(ctx->d_geom.ensure(up(ob) + up(gb) + up(rb) + up(pb) + 256));
    WinOpDev* d_ops = reinterpret_cast<WinOpDev*>(d);
    ScaleGeom* d_geo = reinterpret_cast<ScaleGeom*>(d + up(ob));
    salvox_window_result* d_out = reinterpret_cast<salvox_window_result*>(d + up(ob) + up(gb));
    double* d_pmf = pmf_out ? reinterpret_cast<double*>(d + up(ob) + up(gb) + up(rb)) : nullptr;
    SX_CUDA(cudaMemcpyAsync(d_ops, dev.data(), ob, cudaMemcpyHostToDevice, ctx->stream));
    SX_CUDA(cudaMemcpyAsync(d_geo, geoms.data(), gb, cudaMemcpyHostToDevice, ctx->stream));
    WinOpParams P{};
    P.nx = nx, P.ny = ny, P.nz = nz, P.bins = iw->bins, P.n = (int)n;
    P.binvol = d_bins, P.q = d_q, P.geoms = d_geo, P.ops = d_ops, P.out = d_out, P.pmf = d_pmf;
    constexpr int NW = 2;
    window_ops_kernel<NW><<<(unsigned)((n + NW - 1) / NW), 32 * NW, 0, ctx->stream>>>(P);
    SX_LAUNCH_CHECK(ctx);
    SX_CUDA(cudaMemcpyAsync(out, d_out, rb, cudaMemcpyDeviceToHost, ctx->stream));
    if (pmf_out) SX_CUDA(cudaMemcpyAsync(pmf_out, d_pmf, pb, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

static int select_host(salvox_ctx* ctx, const salvox_detection* dets, int64_t n, double qe,
                       double qp, int32_t k, double radius, bool thresholds,
                       salvox_detection* out, int64_t* n_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (n < 0 || (n > 0 && !dets)) fail(SALVOX_EINVAL, "bad detection array");
    SX_CUDA(cudaSetDevice(ctx->device));
    char* d = static_cast<char*>(ctx->d_sel_c.ensure((size_t)(n + 1) * sizeof(salvox_detection) * 2));
    salvox_detection* d_in = reinterpret_cast<salvox_detection*>(d);
    salvox_detection* d_out = d_in + (n + 1);
    if (n > 0)
      SX_CUDA(cudaMemcpyAsync(d_in, dets, (size_t)n * sizeof(salvox_detection), cudaMemcpyHostToDevice,
                              ctx->stream));
    const int kept = device_select(ctx, d_in, (int)n, qe, qp, k, radius, thresholds, d_out);
    if (kept > 0 && out)
      SX_CUDA(cudaMemcpyAsync(out, d_out, (size_t)kept * sizeof(salvox_detection), cudaMemcpyDeviceToHost,
                              ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_out) *n_out = kept;
  });
}

extern "C" int salvox_select(salvox_ctx* ctx, const salvox_detection* dets, int64_t n,
                             double q_entropy, double q_pdf, int32_t k, double radius,
                             salvox_detection* out, int64_t* n_out) {
  return select_host(ctx, dets, n, q_entropy, q_pdf, k, radius, true, out, n_out);
}

extern "C" int salvox_dedupe_top_k(salvox_ctx* ctx, const salvox_detection* dets, int64_t n,
                                   int32_t k, double radius, salvox_detection* out,
                                   int64_t* n_out) {
  return select_host(ctx, dets, n, 0.0, 0.0, k, radius, false, out, n_out);
}

extern "C" int salvox_abmsod_run(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                 int32_t nz, const salvox_window* iw,
                                 const salvox_abmsod_params* ap, const double* seeds,
                                 const double* seed_H, const double* radii, int64_t n,
                                 salvox_detection* out, salvox_abmsod_iter* trace,
                                 int32_t* n_trace, uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (!volume || !ap) fail(SALVOX_EINVAL, "null argument");
    check_window(iw);
    if (n < 0 || (n > 0 && (!seeds || !out || (!seed_H && !radii))))
      fail(SALVOX_EINVAL, "bad seed arrays");
    salvox_detect_params prm{};
    prm.method = SALVOX_METHOD_ABMSOD;
    prm.abmsod_threshold = ap->threshold;
    prm.abmsod_max_iters = ap->max_iterations;
    prm.abmsod_kernel = ap->kernel;
    prm.abmsod_lambda_min = ap->lambda_min;
    prm.abmsod_lambda_max = ap->lambda_max;
    prm.abmsod_min_inbounds_fraction = ap->min_inbounds_fraction;
    prm.abmsod_target = ap->target;
    std::vector<SeedRec> recs((size_t)n);
    std::vector<int> index((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      std::memcpy(recs[i].pos, seeds + 3 * i, 3 * sizeof(double));
      recs[i].scale = radii ? radii[i] : 1.0;
      index[i] = -1;  // abmsod_run leaves Detection::seed_index at its default
    }
    SeekJob job;
    build_job(nx, ny, nz, &prm, recs, index, job);
    if (seed_H) std::memcpy(job.seed_H.data(), seed_H, (size_t)n * 9 * sizeof(double));
    if (n == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure(nv * 4));
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    double* d_q = nullptr;
    const uint8_t* d_bins = prepare_volume(ctx, d_vol, nx, ny, nz, iw, ap->target, &d_q);
    const size_t tr_n = trace ? (size_t)n * ap->max_iterations : 0;
    char* d_dets = static_cast<char*>(ctx->d_dets.ensure(
        (size_t)(n + 1) * (sizeof(salvox_detection) + 8 + 4) + tr_n * sizeof(salvox_abmsod_iter) + 1024));
    salvox_detection* d_all = reinterpret_cast<salvox_detection*>(d_dets);
    unsigned long long* d_vis = reinterpret_cast<unsigned long long*>(d_all + (n + 1));
    int* d_tn = reinterpret_cast<int*>(d_vis + (n + 1));
    salvox_abmsod_iter* d_tr = reinterpret_cast<salvox_abmsod_iter*>(
        d_dets + (((size_t)(n + 1) * (sizeof(salvox_detection) + 8 + 4) + 255) / 256) * 256);
    job.P.abm_trace = trace ? d_tr : nullptr;
    job.P.abm_trace_n = trace ? d_tn : nullptr;
    run_seek(ctx, job, d_bins, iw->bins, d_q, d_all, d_vis);
    SX_CUDA(cudaMemcpyAsync(out, d_all, (size_t)n * sizeof(salvox_detection), cudaMemcpyDeviceToHost,
                            ctx->stream));
    if (trace) {
      SX_CUDA(cudaMemcpyAsync(trace, d_tr, tr_n * sizeof(salvox_abmsod_iter), cudaMemcpyDeviceToHost,
                              ctx->stream));
      if (n_trace)
        SX_CUDA(cudaMemcpyAsync(n_trace, d_tn, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost,
                                ctx->stream));
    }
    const unsigned long long v = sum_visits(ctx, d_vis, (int)n);
    if (visits) *visits += v;
  });
}

extern "C" int salvox_bandwidth_from_moment(const double* outer, double weight_sum, int32_t dim,
                                            double lambda_min, double lambda_max, double* H) {
  return guarded([&] {
    if (!outer || !H) fail(SALVOX_EINVAL, "null argument");
    switch (sx_bandwidth_from_moment(outer, weight_sum, dim, lambda_min, lambda_max, H)) {
      case 1: fail(SALVOX_EINVAL, "bandwidth update: zero weight mass");
      case 2: fail(SALVOX_EINVAL, "bandwidth update: non-finite moment");
      case 3: fail(SALVOX_ERUNTIME, "abmsod: eigen decomposition failed");
      default: break;
    }
  });
}
