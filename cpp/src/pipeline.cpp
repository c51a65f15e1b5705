// The hot-path entry points of the C++ API, forwarded to the B200 C-ABI
// (reference src/pipeline.cpp:63-183, :311-402; src/seeds.cpp:7-45).
#include "salvox/pipeline.hpp"

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <limits>

#include "salvox/device.hpp"
#include "salvox/hu.hpp"
#include "salvox_capi.h"

namespace salvox {

namespace {
salvox_ctx* ctx() { return device_context(current_device()); }

salvox_detection to_c(const Detection& d) {
  salvox_detection c{};
  for (int i = 0; i < 3; ++i) c.center[i] = d.center[i];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c.H[r * 3 + k] = d.H(r, k);
  c.entropy_bits = d.entropy_bits;
  c.pdf_diff = d.pdf_diff;
  c.bhattacharyya = d.bhattacharyya;
  c.iterations = d.iterations;
  c.flags = d.flags;
  c.seed_index = d.seed_index;
  return c;
}
}  // namespace

Detection from_c(const salvox_detection& c) {
  Detection d;
  d.center = Eigen::Vector3d(c.center[0], c.center[1], c.center[2]);
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) d.H(r, k) = c.H[r * 3 + k];
  d.entropy_bits = c.entropy_bits;
  d.pdf_diff = c.pdf_diff;
  d.bhattacharyya = c.bhattacharyya;
  d.iterations = c.iterations;
  d.flags = c.flags;
  d.seed_index = c.seed_index;
  return d;
}

Method method_from_name(const std::string& name) {
  if (name == "quadrant") return Method::Quadrant;
  if (name == "shift") return Method::Shift;
  if (name == "abmsod") return Method::Abmsod;
  if (name == "octant") return Method::Octant;
  throw std::invalid_argument("unknown method '" + name + "'");
}

const char* method_name(Method m) {
  switch (m) {
    case Method::Quadrant: return "quadrant";
    case Method::Shift: return "shift";
    case Method::Abmsod: return "abmsod";
    case Method::Octant: return "octant";
  }
  return "?";
}

std::vector<Seed> plan_seeds(const Volume& v, const SeedPlan& plan) {
  plan.validate();
  const int mode = plan.mode == SeedPlan::Mode::Lattice ? 0 : 1;
  int64_t n = 0;
  check_status(salvox_plan_seeds(v.nx(), v.ny(), v.nz(), mode, plan.spacing, plan.count,
                                 plan.scales.data(), int(plan.scales.size()), plan.rng_seed,
                                 nullptr, nullptr, 0, &n));
  std::vector<double> pos(static_cast<size_t>(n) * 3), sc(static_cast<size_t>(n));
  check_status(salvox_plan_seeds(v.nx(), v.ny(), v.nz(), mode, plan.spacing, plan.count,
                                 plan.scales.data(), int(plan.scales.size()), plan.rng_seed,
                                 pos.data(), sc.data(), n, &n));
  std::vector<Seed> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    out[size_t(i)] = {Eigen::Vector3d(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]), sc[size_t(i)],
                      int(i)};
  return out;
}

ExhaustiveResult kadir_brady_exhaustive(const Volume& v, const IntensityWindow& iw,
                                        const std::vector<double>& scales, Kernel kernel,
                                        EvalCounter* counter, uint64_t budget) {
  // argument checks first, with the reference's messages (pipeline.cpp:66-72),
  // so invalid calls fail the same way with or without a device
  if (scales.empty()) throw std::invalid_argument("exhaustive scan: no scales");
  for (double s : scales)
    if (s < 2.0) throw std::invalid_argument("exhaustive scan: scales must be >= 2 voxels");
  const uint64_t evals = uint64_t(v.size()) * scales.size();
  if (evals > budget)
    throw std::invalid_argument("exhaustive scan: budget exceeded (" + std::to_string(evals) +
                                " voxel-scale evaluations)");
  ExhaustiveResult res;
  res.map.dims = Eigen::Vector3i(v.nx(), v.ny(), v.nz());
  const salvox_window w{iw.low, iw.high, iw.bins, 0};
  int64_t n = 0;
  uint64_t visits = 0;
  salvox_ctx* c = ctx();
  // The result's std::vectors value-initialise their storage (2 x 4 B per voxel
  // plus the maxima list: ~160 MB of first-touch page faults at 256^3), so they
  // are allocated on host threads WHILE the pass runs with its maps left on the
  // device, then filled by salvox_last_maps / salvox_last_maxima.
  static std::atomic<int64_t> maxima_hint{0};  // list size of the last call
  const size_t hint = size_t(maxima_hint.load() * 11 / 10);
  std::vector<salvox_maximum> mx;
  std::thread a1([&] { res.map.score.resize(v.size()); });
  std::thread a2([&] { res.map.best_scale.resize(v.size()); });
  std::thread a3([&] {
    mx.resize(hint);
    res.maxima.resize(hint);
  });
  struct Join {
    std::thread* t[3];
    ~Join() {
      for (std::thread* x : t)
        if (x->joinable()) x->join();
    }
  } join{{&a1, &a2, &a3}};
  check_status(salvox_exhaustive(c, v.data().data(), v.nx(), v.ny(), v.nz(), &w, scales.data(),
                                 int(scales.size()), int(kernel), budget, nullptr, nullptr,
                                 nullptr, 0, &n, &visits));
  a1.join();
  a2.join();
  a3.join();
  maxima_hint.store(n);
  check_status(salvox_last_maps(c, res.map.score.data(), res.map.best_scale.data()));
  mx.resize(size_t(n));
  res.maxima.resize(size_t(n));
  if (n > 0) check_status(salvox_last_maxima(c, mx.data(), n, &n));
  // records -> SaliencyMaximum (pipeline.hpp:32-36), a few threads for long lists
  const size_t nm = size_t(n);
  const size_t T = nm > 65536 ? 4 : 1;
  auto conv = [&](size_t t) {
    for (size_t i = nm * t / T; i < nm * (t + 1) / T; ++i) {
      const salvox_maximum& m = mx[i];
      res.maxima[i] = {Eigen::Vector3d(m.position[0], m.position[1], m.position[2]), m.score, m.scale};
    }
  };
  std::vector<std::thread> cv;
  for (size_t t = 1; t < T; ++t) cv.emplace_back(conv, t);
  conv(0);
  for (auto& t : cv) t.join();
  if (counter) counter->add(visits);
  return res;
}

std::vector<Detection> dedupe_top_k(std::vector<Detection> dets, int k, double radius) {
  std::vector<salvox_detection> in(dets.size()), out(dets.size() + 1);
  std::transform(dets.begin(), dets.end(), in.begin(), to_c);
  int64_t n = 0;
  check_status(salvox_dedupe_top_k(ctx(), in.data(), int64_t(in.size()), k, radius, out.data(), &n));
  std::vector<Detection> kept;
  for (int64_t i = 0; i < n; ++i) kept.push_back(from_c(out[size_t(i)]));
  return kept;
}

std::vector<Detection> detect(const Volume& v, const IntensityWindow& iw, DetectParams params,
                              EvalCounter* counter) {
  if (params.method == Method::Quadrant && !v.is_2d())
    throw std::invalid_argument("detect: quadrant method requires a 2D volume (nz == 1)");
  params.seeds.validate();
  if (params.method == Method::Shift) params.shift.validate();
  if (params.method == Method::Abmsod) params.abmsod.validate();
  salvox_detect_params p{};
  p.method = params.method == Method::Quadrant ? SALVOX_METHOD_QUADRANT
             : params.method == Method::Shift  ? SALVOX_METHOD_SHIFT
             : params.method == Method::Abmsod ? SALVOX_METHOD_ABMSOD
                                               : SALVOX_METHOD_OCTANT;
  p.seed_mode = params.seeds.mode == SeedPlan::Mode::Lattice ? 0 : 1;
  p.seed_spacing = params.seeds.spacing;
  p.seed_count = params.seeds.count;
  p.top_k = params.top_k;
  p.rng_seed = params.seeds.rng_seed;
  p.scales = params.seeds.scales.data();
  p.n_scales = int(params.seeds.scales.size());
  p.workers = int(params.workers);
  p.dedupe_radius = params.dedupe_radius;
  p.entropy_quantile = params.entropy_quantile;
  p.pdf_quantile = params.pdf_quantile;
  p.quadrant_eta = params.quadrant.eta;
  p.quadrant_max_iters = params.quadrant.max_iters;
  p.n_quadrant_scales = int(params.quadrant.scale_range.size());
  p.quadrant_scales = params.quadrant.scale_range.data();
  p.shift_min_step = params.shift.min_step;
  p.shift_max_iters = params.shift.max_iters;
  p.shift_step_kernel = int(params.shift.step_kernel);
  p.shift_hist_kernel = int(params.shift.hist_kernel);
  p.shift_min_inbounds_fraction = params.shift.min_inbounds_fraction;
  std::vector<double> target, atarget;
  if (params.shift.target) {
    target = params.shift.target->p;
    p.shift_target = target.data();
  }
  p.abmsod_threshold = params.abmsod.threshold;
  p.abmsod_max_iters = params.abmsod.max_iterations;
  p.abmsod_kernel = int(params.abmsod.kernel);
  p.abmsod_lambda_min = params.abmsod.lambda_min;
  p.abmsod_lambda_max = params.abmsod.lambda_max;
  p.abmsod_min_inbounds_fraction = params.abmsod.min_inbounds_fraction;
  if (params.abmsod.target) {
    atarget = params.abmsod.target->p;
    p.abmsod_target = atarget.data();
  }
  const salvox_window w{iw.low, iw.high, iw.bins, 0};
  std::vector<salvox_detection> out(size_t(std::max(params.top_k, 1)));
  int64_t n_out = 0, n_seed = 0;
  uint64_t visits = 0;
  check_status(salvox_detect(ctx(), v.data().data(), v.nx(), v.ny(), v.nz(), &w, &p, out.data(),
                             int64_t(out.size()), &n_out, nullptr, 0, &n_seed, &visits));
  if (counter) counter->add(visits);
  std::vector<Detection> dets;
  for (int64_t i = 0; i < n_out; ++i) dets.push_back(from_c(out[size_t(i)]));
  return dets;
}

std::vector<uint64_t> rasterize_window(const Volume& frame, const EllipsoidWindow& win) {
  double c[3], h[9];
  for (int i = 0; i < 3; ++i) c[i] = win.center[i];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) h[3 * r + k] = win.H(r, k);
  int64_t n = 0;
  check_status(salvox_rasterize_window(ctx(), frame.nx(), frame.ny(), frame.nz(), c, h, nullptr, 0, &n));
  std::vector<uint64_t> out(static_cast<size_t>(n));
  if (n > 0)
    check_status(salvox_rasterize_window(ctx(), frame.nx(), frame.ny(), frame.nz(), c, h,
                                         out.data(), n, &n));
  return out;
}

double jaccard(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
  if (a.empty() && b.empty()) throw std::invalid_argument("jaccard: both sets are empty");
  size_t i = 0, j = 0, inter = 0;  // sorted-merge intersection
  while (i < a.size() && j < b.size()) {
    if (a[i] == b[j]) {
      ++inter, ++i, ++j;
    } else if (a[i] < b[j]) {
      ++i;
    } else {
      ++j;
    }
  }
  return double(inter) / double(a.size() + b.size() - inter);
}

double jaccard(const Volume& frame, const EllipsoidWindow& win, const std::vector<uint64_t>& mask) {
  return jaccard(rasterize_window(frame, win), mask);
}

HuVector hu_moments(const Volume& slice) {  // hu.cpp:8-58 on the device
  if (!slice.is_2d()) throw std::invalid_argument("hu_moments: expected a 2D slice");
  HuVector h{};
  check_status(salvox_hu_moments(ctx(), slice.data().data(), slice.nx(), slice.ny(), h.data()));
  return h;
}

double hu_distance(const HuVector& a, const HuVector& b) {  // hu.cpp:60-64
  double d2 = 0.0;
  for (int i = 0; i < 7; ++i) d2 += (a[size_t(i)] - b[size_t(i)]) * (a[size_t(i)] - b[size_t(i)]);
  return std::sqrt(d2);
}

namespace {
std::vector<double> hu_distances(const std::vector<Detection>& dets, const Volume& v,
                                 const Volume& t, int slices) {
  if (!t.is_2d()) throw std::invalid_argument("hu_moments: expected a 2D slice");
  std::vector<salvox_detection> c(dets.size());
  std::transform(dets.begin(), dets.end(), c.begin(), to_c);
  std::vector<double> d(dets.size());
  check_status(salvox_hu_template_distance(ctx(), v.data().data(), v.nx(), v.ny(), v.nz(), c.data(),
                                           int64_t(c.size()), t.data().data(), t.nx(), t.ny(),
                                           slices, d.data()));
  return d;
}
}  // namespace

double hu_template_distance(const Detection& det, const Volume& v, const Volume& template_2d,
                            int slices) {
  return hu_distances({det}, v, template_2d, slices).front();
}

size_t hu_filter(const std::vector<Detection>& dets, const Volume& v, const Volume& template_2d,
                 int slices) {  // pipeline.cpp:258-271
  if (dets.empty()) throw std::invalid_argument("hu_filter: no detections");
  const auto d = hu_distances(dets, v, template_2d, slices);
  size_t best = 0;
  double best_d = std::numeric_limits<double>::infinity();
  for (size_t i = 0; i < d.size(); ++i)
    if (d[i] < best_d) best_d = d[i], best = i;
  return best;
}

}  // namespace salvox
