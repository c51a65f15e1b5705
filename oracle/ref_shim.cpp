// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// C-ABI over the REFERENCE's own C++ (compiled from /root/reference/proj/src
// where it lies, by oracle/Makefile, into oracle/_ref/libsalvox_ref.so). This
// file is glue only: every function converts plain arrays into the
// reference's types, calls the reference function named in its comment and
// copies the result back. It lets the tests check (1) the C oracle
// restatement (oracle/salvox_oracle.c) and (2) the B200 path against the
// reference itself on the same inputs, and lets bench.py's reference arm time
// the reference's own detect().
//
// The reference needs Eigen3 (absent): it is compiled against the repo's
// Eigen-API subset (oracle/ref_eigen -> cpp/third_party/eigen_subset, plus
// SelfAdjointEigenSolver from include/salvox/sx_eig3.h), so Eigen's own
// last-bit rounding stays unpinned; every salvox line is the
// reference's. Return codes: 0 ok, 1 std::invalid_argument, 2 other exception
// (message in err).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "salvox/abmsod.hpp"
#include "salvox/config.hpp"
#include "salvox/hu.hpp"
#include "salvox/meta_io.hpp"
#include "salvox/phantom.hpp"
#include "salvox/pipeline.hpp"
#include "salvox/quadrant.hpp"
#include "salvox/report.hpp"
#include "salvox/seeds.hpp"
#include "salvox/shift.hpp"

extern "C" {
#include "salvox_oracle.h"  // record layouts shared with the C oracle (sxo_detection, ...)
}

namespace {

using namespace salvox;

void put_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::strncpy(err, msg, size_t(len) - 1);
    err[len - 1] = 0;
  }
}

template <class F>
int guarded(char* err, int err_len, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(err, err_len, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 2;
  }
}

Volume make_volume(const float* vol, int nx, int ny, int nz) {
  Volume v(nx, ny, nz);
  std::memcpy(v.data().data(), vol, sizeof(float) * v.size());
  return v;
}

Kernel kernel_of(int k) {
  return k == 0 ? Kernel::Identity : k == 1 ? Kernel::Epanechnikov : Kernel::Gaussian;
}

void put_det(const Detection& d, sxo_detection* o) {
  std::memset(o, 0, sizeof(*o));
  for (int i = 0; i < 3; ++i) o->center[i] = d.center[i];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o->H[3 * r + c] = d.H(r, c);
  o->entropy_bits = d.entropy_bits;
  o->pdf_diff = d.pdf_diff;
  o->bhattacharyya = d.bhattacharyya;
  o->iterations = d.iterations;
  o->flags = d.flags;
  o->seed_index = d.seed_index;
}

Detection get_det(const sxo_detection& o) {
  Detection d;
  for (int i = 0; i < 3; ++i) d.center[i] = o.center[i];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) d.H(r, c) = o.H[3 * r + c];
  d.entropy_bits = o.entropy_bits;
  d.pdf_diff = o.pdf_diff;
  d.bhattacharyya = o.bhattacharyya;
  d.iterations = o.iterations;
  d.flags = o.flags;
  d.seed_index = o.seed_index;
  return d;
}

EllipsoidWindow window_of(const double c[3], const double H[9]) {
  EllipsoidWindow w;
  w.center = {c[0], c[1], c[2]};
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) w.H(r, k) = H[3 * r + k];
  return w;
}

Histogram target_of(const double* p, int bins) {
  if (!p) return Histogram::uniform(bins);
  Histogram h(bins);
  for (int b = 0; b < bins; ++b) h.p[b] = p[b];
  h.normalized = true;
  return h;
}

DetectParams detect_params_of(const sxo_detect_params* P) {
  DetectParams dp;
  if (P->method == 0) dp.method = Method::Quadrant;
  else if (P->method == 1) dp.method = Method::Shift;
  else if (P->method == 2) dp.method = Method::Abmsod;
  else throw std::invalid_argument("reference detect: octant ascent does not exist in the reference");
  dp.seeds.mode = P->seed_mode == 0 ? SeedPlan::Mode::Lattice : SeedPlan::Mode::Random;
  dp.seeds.spacing = P->seed_spacing;
  dp.seeds.count = P->seed_count;
  dp.seeds.rng_seed = P->rng_seed;
  dp.seeds.scales.assign(P->scales, P->scales + P->n_scales);
  dp.top_k = P->top_k;
  dp.dedupe_radius = P->dedupe_radius;
  dp.entropy_quantile = P->entropy_quantile;
  dp.pdf_quantile = P->pdf_quantile;
  dp.workers = unsigned(P->workers < 1 ? 1 : P->workers);
  dp.quadrant.eta = P->quadrant_eta;
  dp.quadrant.max_iters = P->quadrant_max_iters;
  if (P->quadrant_scales)
    dp.quadrant.scale_range.assign(P->quadrant_scales, P->quadrant_scales + P->n_quadrant_scales);
  dp.shift.min_step = P->shift_min_step;
  dp.shift.max_iters = P->shift_max_iters;
  dp.shift.step_kernel = kernel_of(P->shift_step_kernel);
  dp.shift.hist_kernel = kernel_of(P->shift_hist_kernel);
  dp.shift.min_inbounds_fraction = P->shift_min_inbounds_fraction;
  dp.abmsod.threshold = P->abmsod_threshold;
  dp.abmsod.max_iterations = P->abmsod_max_iters;
  dp.abmsod.kernel = kernel_of(P->abmsod_kernel);
  dp.abmsod.lambda_min = P->abmsod_lambda_min;
  dp.abmsod.lambda_max = P->abmsod_lambda_max;
  dp.abmsod.min_inbounds_fraction = P->abmsod_min_inbounds_fraction;
  return dp;
}

}  // namespace

extern "C" {

// phantom.cpp:99-150 PhantomSpec::from_json_text + :237-294 make_phantom.
// out: nx*ny*nz floats (cap = capacity); centroids: 3 per region (GroundTruth
// centre), up to cap_regions. dims_out receives (nx, ny, nz).
int sxr_make_phantom(const char* spec_json, float* out, int64_t cap, int* dims_out,
                     double* centers, int cap_regions, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const PhantomSpec spec = PhantomSpec::from_json_text(spec_json);
    auto [vol, truth] = make_phantom(spec);
    dims_out[0] = vol.nx(), dims_out[1] = vol.ny(), dims_out[2] = vol.nz();
    if (out) {
      if (int64_t(vol.size()) > cap) throw std::runtime_error("phantom: output too small");
      std::memcpy(out, vol.data().data(), sizeof(float) * vol.size());
    }
    for (size_t i = 0; i < truth.regions.size() && int(i) < cap_regions; ++i)
      for (int k = 0; k < 3; ++k) centers[3 * i + k] = truth.regions[i].center[k];
  });
}

// volume.hpp:102-105
int sxr_bin_of(double low, double high, int bins, double intensity) {
  return IntensityWindow(low, high, bins).bin_of(intensity);
}

// histogram.hpp:65-67 (p is normalised by the caller)
double sxr_entropy_bits(const double* p, int bins) {
  Histogram h(bins);
  for (int b = 0; b < bins; ++b) h.p[b] = p[b];
  h.normalized = true;
  return entropy_bits(h);
}

// pipeline.cpp:63-166 kadir_brady_exhaustive. Maxima as (x, y, z, score, scale).
int sxr_exhaustive(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double* scales, int n_scales, int kernel, uint64_t budget, float* score,
                   float* best_scale, double* maxima, int64_t cap, int64_t* n_maxima,
                   uint64_t* visits, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    EvalCounter counter;
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(low, high, bins),
                                            std::vector<double>(scales, scales + n_scales),
                                            kernel_of(kernel), &counter, budget);
    std::memcpy(score, res.map.score.data(), sizeof(float) * v.size());
    std::memcpy(best_scale, res.map.best_scale.data(), sizeof(float) * v.size());
    *n_maxima = int64_t(res.maxima.size());
    for (int64_t i = 0; i < cap && i < *n_maxima; ++i) {
      const auto& m = res.maxima[size_t(i)];
      double* o = maxima + 5 * i;
      o[0] = m.position.x(), o[1] = m.position.y(), o[2] = m.position.z();
      o[3] = m.score, o[4] = m.scale;
    }
    *visits = counter.count();
  });
}

// seeds.cpp:7-45 plan_seeds. pos: 3 per seed; returns the count via n_out.
int sxr_plan_seeds(int nx, int ny, int nz, int mode, double spacing, int count,
                   const double* scales, int n_scales, uint64_t rng_seed, double* pos,
                   double* seed_scale, int64_t cap, int64_t* n_out, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v(nx, ny, nz);
    SeedPlan plan;
    plan.mode = mode == 0 ? SeedPlan::Mode::Lattice : SeedPlan::Mode::Random;
    plan.spacing = spacing;
    plan.count = count;
    plan.scales.assign(scales, scales + n_scales);
    plan.rng_seed = rng_seed;
    const auto seeds = plan_seeds(v, plan);
    *n_out = int64_t(seeds.size());
    for (int64_t i = 0; i < cap && i < *n_out; ++i) {
      for (int k = 0; k < 3; ++k) pos[3 * i + k] = seeds[size_t(i)].position[k];
      seed_scale[i] = seeds[size_t(i)].scale;
    }
  });
}

// shift.cpp:15-34 shift_step (half-extent window). Returns 1 + out, 0 nullopt, <0 error.
int sxr_shift_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double x[3], const double half[3], int step_kernel, int hist_kernel,
                   const double* target, double out[3], uint64_t* visits) {
  int found = -1;
  const int rc = guarded(nullptr, 0, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    ShiftParams sp;
    sp.half_extents = {half[0], half[1], half[2]};
    sp.step_kernel = kernel_of(step_kernel);
    sp.hist_kernel = kernel_of(hist_kernel);
    if (target) sp.target = target_of(target, bins);
    EvalCounter counter;
    const auto r = shift_step(v, {x[0], x[1], x[2]}, sp, IntensityWindow(low, high, bins), &counter);
    *visits = counter.count();
    found = r ? 1 : 0;
    if (r)
      for (int k = 0; k < 3; ++k) out[k] = (*r)[k];
  });
  return rc == 0 ? found : -rc;
}

// shift.cpp:36-107 saliency_shift
int sxr_saliency_shift(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double seed[3], const double half[3], int step_kernel,
                       int hist_kernel, int max_iters, double min_step, const double* target,
                       double min_inbounds_fraction, sxo_detection* out, uint64_t* visits,
                       char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    ShiftParams sp;
    sp.half_extents = {half[0], half[1], half[2]};
    sp.step_kernel = kernel_of(step_kernel);
    sp.hist_kernel = kernel_of(hist_kernel);
    sp.max_iters = max_iters;
    sp.min_step = min_step;
    if (target) sp.target = target_of(target, bins);
    sp.min_inbounds_fraction = min_inbounds_fraction;
    EvalCounter counter;
    const auto r = saliency_shift(v, {seed[0], seed[1], seed[2]}, sp,
                                  IntensityWindow(low, high, bins), &counter);
    put_det(r.det, out);
    *visits = counter.count();
  });
}

// window.cpp:5-19 try_candidate_histogram. Returns 1 (+ p_out), 0 nullopt, <0 error.
int sxr_candidate_histogram(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, const double center[3], const double H[9], int kernel,
                            double* p_out, uint64_t* visits) {
  int found = -1;
  const int rc = guarded(nullptr, 0, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    EvalCounter counter;
    const auto p = try_candidate_histogram(v, window_of(center, H),
                                           IntensityWindow(low, high, bins), kernel_of(kernel),
                                           &counter);
    *visits = counter.count();
    found = p ? 1 : 0;
    if (p)
      for (int b = 0; b < bins; ++b) p_out[b] = p->p[b];
  });
  return rc == 0 ? found : -rc;
}

// window.cpp:30-46 pdf_difference
int sxr_pdf_difference(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double center[3], const double H[9], int kernel, double* out,
                       uint64_t* visits, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    EvalCounter counter;
    *out = pdf_difference(v, window_of(center, H), IntensityWindow(low, high, bins),
                          kernel_of(kernel), &counter);
    *visits = counter.count();
  });
}

// quadrant.cpp:18-35 box_entropy_bits (2D)
double sxr_box_entropy_bits(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, double x0, double x1, double y0, double y1, int min_pixels,
                            uint64_t* visits) {
  const Volume v = make_volume(vol, nx, ny, nz);
  EvalCounter counter;
  const double e = box_entropy_bits(v, x0, x1, y0, y1, IntensityWindow(low, high, bins),
                                    min_pixels, &counter);
  *visits = counter.count();
  return e;
}

// quadrant.cpp:37-81 quadrant_step (2D). moved: 2 doubles.
int sxr_quadrant_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                      const double p[2], const int* scales, int n_scales, double moved[2],
                      sxo_ascent_state* st, uint64_t* visits, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    QuadrantParams qp;
    qp.scale_range.assign(scales, scales + n_scales);
    EvalCounter counter;
    const auto [m, s] = quadrant_step(v, {p[0], p[1]}, qp, IntensityWindow(low, high, bins),
                                      &counter);
    moved[0] = m.x(), moved[1] = m.y();
    std::memset(st, 0, sizeof(*st));
    for (int q = 0; q < 4; ++q) {
      st->entropy[q] = s.entropy[q];
      st->best_scale[q] = s.best_scale[q];
      st->norm_entropy[q] = s.norm_entropy[q];
    }
    st->displacement[0] = s.displacement.x(), st->displacement[1] = s.displacement.y();
    st->degenerate = s.degenerate ? 1 : 0;
    *visits = counter.count();
  });
}

// quadrant.cpp:83-114 quadrant_seek_one (2D)
int sxr_quadrant_seek_one(const float* vol, int nx, int ny, int nz, double low, double high,
                          int bins, const double seed[2], const int* scales, int n_scales,
                          double eta, int max_iters, sxo_ascent_result* out, uint64_t* visits,
                          char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    QuadrantParams qp;
    qp.scale_range.assign(scales, scales + n_scales);
    qp.eta = eta;
    qp.max_iters = max_iters;
    EvalCounter counter;
    const auto r = quadrant_seek_one(v, {seed[0], seed[1]}, qp, IntensityWindow(low, high, bins),
                                     &counter);
    std::memset(out, 0, sizeof(*out));
    out->position[0] = r.position.x(), out->position[1] = r.position.y();
    out->best_scale = r.best_scale;
    out->iterations = r.iterations;
    out->entropy_bits = r.entropy_bits;
    out->converged = r.converged ? 1 : 0;
    out->degenerate = r.degenerate ? 1 : 0;
    *visits = counter.count();
  });
}

// pipeline.cpp:311-402 detect -- the reference's own end-to-end call (method
// 0 quadrant, 1 shift, 2 abmsod). Returns the selected detections.
int sxr_detect(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
               const sxo_detect_params* P, sxo_detection* out, int64_t cap, int64_t* n_out,
               uint64_t* visits, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    EvalCounter counter;
    const auto dets = detect(v, IntensityWindow(low, high, bins), detect_params_of(P), &counter);
    *n_out = int64_t(dets.size());
    for (int64_t i = 0; i < cap && i < *n_out; ++i) put_det(dets[size_t(i)], out + i);
    *visits = counter.count();
  });
}

// abmsod.cpp:43-169 abmsod_run (trace on request)
int sxr_abmsod_run(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double seed_center[3], const double seed_H[9],
                   const sxo_abmsod_params* P, sxo_detection* det, sxo_abmsod_iter* trace,
                   int trace_cap, int* n_trace, uint64_t* visits, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = make_volume(vol, nx, ny, nz);
    AbmsodParams ap;
    ap.threshold = P->threshold;
    ap.max_iterations = P->max_iterations;
    ap.kernel = kernel_of(P->kernel);
    ap.lambda_min = P->lambda_min;
    ap.lambda_max = P->lambda_max;
    ap.min_inbounds_fraction = P->min_inbounds_fraction;
    if (P->target) ap.target = target_of(P->target, bins);
    ap.record_trace = trace != nullptr;
    EvalCounter counter;
    const auto r = abmsod_run(v, window_of(seed_center, seed_H), ap,
                              IntensityWindow(low, high, bins), &counter);
    put_det(r.det, det);
    if (n_trace) *n_trace = int(r.trace.size());
    for (int i = 0; trace && i < trace_cap && i < int(r.trace.size()); ++i) {
      const auto& t = r.trace[size_t(i)];
      for (int k = 0; k < 3; ++k) trace[i].position[k] = t.position[k];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) trace[i].H[3 * a + b] = t.H(a, b);
      trace[i].bhattacharyya = t.bhattacharyya;
      trace[i].max_bhattacharyya = t.max_bhattacharyya;
      trace[i].eig_min = t.eig_min;
      trace[i].eig_max = t.eig_max;
    }
    *visits = counter.count();
  });
}

// abmsod.cpp:23-41 bandwidth_from_moment (outer row-major)
int sxr_bandwidth_from_moment(const double outer[9], double wsum, int dim, double lambda_min,
                              double lambda_max, double H[9], char* err, int err_len) {
  return guarded(err, err_len, [&] {
    Eigen::Matrix3d o;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) o(r, c) = outer[3 * r + c];
    const auto h = bandwidth_from_moment(o, wsum, dim, lambda_min, lambda_max);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) H[3 * r + c] = h(r, c);
  });
}

// pipeline.cpp:168-183 dedupe_top_k
int64_t sxr_dedupe_top_k(const sxo_detection* dets, int64_t n, int k, double radius,
                         sxo_detection* out) {
  std::vector<Detection> in;
  for (int64_t i = 0; i < n; ++i) in.push_back(get_det(dets[i]));
  const auto kept = dedupe_top_k(std::move(in), k, radius);
  for (size_t i = 0; i < kept.size(); ++i) put_det(kept[i], out + i);
  return int64_t(kept.size());
}

// pipeline.cpp:185-192 rasterize_window; returns the count (writes up to cap)
int64_t sxr_rasterize_window(int nx, int ny, int nz, const double center[3], const double H[9],
                             uint64_t* out, int64_t cap) {
  const Volume frame(nx, ny, nz);
  const auto r = rasterize_window(frame, window_of(center, H));
  for (int64_t i = 0; i < cap && i < int64_t(r.size()); ++i) out[i] = r[size_t(i)];
  return int64_t(r.size());
}

// hu.cpp:8-58 hu_moments on an nx*ny slice
int sxr_hu_moments(const float* img, int nx, int ny, double out[7], char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const auto h = hu_moments(make_volume(img, nx, ny, 1));
    for (int i = 0; i < 7; ++i) out[i] = h[size_t(i)];
  });
}

// pipeline.cpp:236-256 hu_template_distance
double sxr_hu_template_distance(const float* vol, int nx, int ny, int nz, const double center[3],
                                const double H[9], const float* tmpl, int tnx, int tny,
                                int slices) {
  Detection d;
  d.center = {center[0], center[1], center[2]};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) d.H(r, c) = H[3 * r + c];
  return hu_template_distance(d, make_volume(vol, nx, ny, nz), make_volume(tmpl, tnx, tny, 1),
                              slices);
}

// the same two calls over many windows / detections with ONE Volume built (a
// caller of the reference API holds its volume already; timing per-call copies
// of it would charge the reference for this shim)
int64_t sxr_rasterize_windows(int nx, int ny, int nz, const double* centers, const double* Hs,
                              int64_t n, int64_t* counts) {
  const Volume frame(nx, ny, nz);
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    counts[i] = int64_t(rasterize_window(frame, window_of(centers + 3 * i, Hs + 9 * i)).size());
    total += counts[i];
  }
  return total;
}

void sxr_hu_template_distances(const float* vol, int nx, int ny, int nz, const double* centers,
                               const double* Hs, int64_t n, const float* tmpl, int tnx, int tny,
                               int slices, double* out) {
  const Volume v = make_volume(vol, nx, ny, nz);
  const Volume t = make_volume(tmpl, tnx, tny, 1);
  for (int64_t i = 0; i < n; ++i) {
    Detection d;
    d.center = {centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) d.H(r, c) = Hs[9 * i + 3 * r + c];
    out[i] = hu_template_distance(d, v, t, slices);
  }
}

// meta_io.cpp:37-117 load_volume. Query dims with out == NULL.
int sxr_load_volume(const char* mhd_path, float* out, int64_t cap, int* dims_out,
                    double* spacing_out, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const Volume v = load_volume(mhd_path);
    dims_out[0] = v.nx(), dims_out[1] = v.ny(), dims_out[2] = v.nz();
    for (int k = 0; k < 3; ++k) spacing_out[k] = v.spacing()[k];
    if (out) {
      if (int64_t(v.size()) > cap) throw std::runtime_error("load_volume: output too small");
      std::memcpy(out, v.data().data(), sizeof(float) * v.size());
    }
  });
}

// meta_io.cpp:119-143 save_volume (spacing 1)
int sxr_save_volume(const float* vol, int nx, int ny, int nz, const char* mhd_path, char* err,
                    int err_len) {
  return guarded(err, err_len, [&] { save_volume(make_volume(vol, nx, ny, nz), mhd_path); });
}

// config.cpp RunConfig::from_json_text -> to_json_text (the resolved config)
int sxr_config_roundtrip(const char* config_json, char* out, int64_t cap, int64_t* len,
                         char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const std::string s = RunConfig::from_json_text(config_json).to_json_text();
    *len = int64_t(s.size());
    if (out && cap > 0) {
      std::strncpy(out, s.c_str(), size_t(cap) - 1);
      out[cap - 1] = 0;
    }
  });
}

// report.cpp:28-60 detection_report_json (config given as JSON text)
int sxr_detection_report_json(const char* config_json, const float* vol, int nx, int ny, int nz,
                              const sxo_detection* dets, int64_t n, double wall_time_ms, char* out,
                              int64_t cap, int64_t* len, char* err, int err_len) {
  return guarded(err, err_len, [&] {
    const RunConfig cfg = RunConfig::from_json_text(config_json);
    std::vector<Detection> ds;
    for (int64_t i = 0; i < n; ++i) ds.push_back(get_det(dets[i]));
    const std::string s = detection_report_json(cfg, make_volume(vol, nx, ny, nz), ds, wall_time_ms);
    *len = int64_t(s.size());
    if (out && cap > 0) {
      std::strncpy(out, s.c_str(), size_t(cap) - 1);
      out[cap - 1] = 0;
    }
  });
}

// report.cpp:12-26
uint64_t sxr_fnv1a64(const void* data, size_t len) { return fnv1a64(data, len); }

}  // extern "C"
