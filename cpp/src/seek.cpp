// Per-seed seek entry points of the C++ API on the B200 (reference
// src/shift.cpp:36-107, src/quadrant.cpp:83-125; octant is new).
#include <algorithm>

#include "salvox/abmsod.hpp"
#include "salvox/device.hpp"
#include "salvox/pipeline.hpp"
#include "salvox_capi.h"

namespace salvox {

Detection from_c(const salvox_detection& c);

std::vector<Detection> saliency_shift_many(const Volume& v, const std::vector<Eigen::Vector3d>& seeds,
                                           const ShiftParams& params, const IntensityWindow& iw,
                                           EvalCounter* counter) {
  params.validate();
  salvox_detect_params p{};
  p.method = SALVOX_METHOD_SHIFT;
  p.shift_min_step = params.min_step;
  p.shift_max_iters = params.max_iters;
  p.shift_step_kernel = int(params.step_kernel);
  p.shift_hist_kernel = int(params.hist_kernel);
  p.shift_min_inbounds_fraction = params.min_inbounds_fraction;
  std::vector<double> target;
  if (params.target) {
    target = params.target->p;
    p.shift_target = target.data();
  }
  const size_t n = seeds.size();
  std::vector<double> pos(3 * n), half(3 * n);
  for (size_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + size_t(k)] = seeds[i][k];
      half[3 * i + size_t(k)] = params.half_extents[k];
    }
  const salvox_window w{iw.low, iw.high, iw.bins, 0};
  std::vector<salvox_detection> out(n + 1);
  uint64_t visits = 0;
  check_status(salvox_seek(device_context(current_device()), v.data().data(), v.nx(), v.ny(),
                           v.nz(), &w, &p, pos.data(), nullptr, half.data(), nullptr, int64_t(n),
                           out.data(), &visits));
  if (counter) counter->add(visits);
  std::vector<Detection> dets;
  for (size_t i = 0; i < n; ++i) dets.push_back(from_c(out[i]));
  return dets;
}

ShiftResult saliency_shift_traced(const Volume& v, const Eigen::Vector3d& seed,
                                  const ShiftParams& params, const IntensityWindow& iw,
                                  EvalCounter* counter);  // window.cpp

ShiftResult saliency_shift(const Volume& v, const Eigen::Vector3d& seed, const ShiftParams& params,
                           const IntensityWindow& iw, EvalCounter* counter) {
  if (params.record_trace) return saliency_shift_traced(v, seed, params, iw, counter);
  ShiftResult r;
  r.det = saliency_shift_many(v, {seed}, params, iw, counter).front();
  r.det.seed_index = -1;
  return r;
}

namespace {
std::vector<salvox_ascent_result> ascent(const Volume& v, const std::vector<double>& pos,
                                         const QuadrantParams& params, const IntensityWindow& iw,
                                         int dims, EvalCounter* counter) {
  params.validate();
  const size_t n = pos.size() / 3;
  std::vector<salvox_ascent_result> out(n + 1);
  const salvox_window w{iw.low, iw.high, iw.bins, 0};
  uint64_t visits = 0;
  check_status(salvox_ascent_seek(device_context(current_device()), v.data().data(), v.nx(),
                                  v.ny(), v.nz(), &w, dims, params.scale_range.data(),
                                  int(params.scale_range.size()), params.eta, params.max_iters,
                                  pos.data(), int64_t(n), out.data(), &visits));
  if (counter) counter->add(visits);
  out.resize(n);
  return out;
}
}  // namespace

std::vector<QuadrantResult> quadrant_seek(const Volume& v, const std::vector<Eigen::Vector2d>& seeds,
                                          const QuadrantParams& params, const IntensityWindow& iw,
                                          unsigned /*workers*/, EvalCounter* counter) {
  if (seeds.empty()) throw std::invalid_argument("quadrant_seek: no seeds");
  if (!v.is_2d()) throw std::invalid_argument("quadrant_step: volume must be 2D (nz == 1)");
  std::vector<double> pos;
  for (const auto& s : seeds) pos.insert(pos.end(), {s.x(), s.y(), 0.0});
  std::vector<QuadrantResult> res;
  for (const auto& a : ascent(v, pos, params, iw, 2, counter)) {
    QuadrantResult r;
    r.position = Eigen::Vector2d(a.position[0], a.position[1]);
    r.best_scale = a.best_scale;
    r.entropy_bits = a.entropy_bits;
    r.iterations = a.iterations;
    r.converged = a.converged != 0;
    r.degenerate = a.degenerate != 0;
    res.push_back(r);
  }
  return res;
}

QuadrantResult quadrant_seek_one(const Volume& v, const Eigen::Vector2d& seed,
                                 const QuadrantParams& params, const IntensityWindow& iw,
                                 EvalCounter* counter) {
  return quadrant_seek(v, {seed}, params, iw, 1, counter).front();
}

std::vector<OctantResult> octant_seek(const Volume& v, const std::vector<Eigen::Vector3d>& seeds,
                                      const QuadrantParams& params, const IntensityWindow& iw,
                                      EvalCounter* counter) {
  if (seeds.empty()) throw std::invalid_argument("octant_seek: no seeds");
  std::vector<double> pos;
  for (const auto& s : seeds) pos.insert(pos.end(), {s.x(), s.y(), s.z()});
  std::vector<OctantResult> res;
  for (const auto& a : ascent(v, pos, params, iw, 3, counter)) {
    OctantResult r;
    r.position = Eigen::Vector3d(a.position[0], a.position[1], a.position[2]);
    r.best_scale = a.best_scale;
    r.entropy_bits = a.entropy_bits;
    r.iterations = a.iterations;
    r.converged = a.converged != 0;
    r.degenerate = a.degenerate != 0;
    res.push_back(r);
  }
  return res;
}

Eigen::Matrix3d bandwidth_from_moment(const Eigen::Matrix3d& outer, double weight_sum, int dim,
                                      double lambda_min, double lambda_max) {
  double o[9], h[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o[3 * r + c] = outer(r, c);
  check_status(salvox_bandwidth_from_moment(o, weight_sum, dim, lambda_min, lambda_max, h));
  Eigen::Matrix3d H;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) H(r, c) = h[3 * r + c];
  return H;
}

std::vector<AbmsodResult> abmsod_run_many(const Volume& v, const std::vector<EllipsoidWindow>& seeds,
                                          const AbmsodParams& params, const IntensityWindow& iw,
                                          EvalCounter* counter) {
  params.validate();
  salvox_abmsod_params p{};
  p.threshold = params.threshold;
  p.max_iterations = params.max_iterations;
  p.kernel = int(params.kernel);
  p.lambda_min = params.lambda_min;
  p.lambda_max = params.lambda_max;
  p.min_inbounds_fraction = params.min_inbounds_fraction;
  std::vector<double> target;
  if (params.target) {
    target = params.target->p;
    p.target = target.data();
  }
  const size_t n = seeds.size();
  std::vector<double> pos(3 * n), H(9 * n);
  for (size_t i = 0; i < n; ++i)
    for (int r = 0; r < 3; ++r) {
      pos[3 * i + size_t(r)] = seeds[i].center[r];
      for (int c = 0; c < 3; ++c) H[9 * i + size_t(3 * r + c)] = seeds[i].H(r, c);
    }
  const salvox_window w{iw.low, iw.high, iw.bins, 0};
  std::vector<salvox_detection> out(n + 1);
  const size_t m = size_t(std::max(params.max_iterations, 1));
  std::vector<salvox_abmsod_iter> trace(params.record_trace ? n * m : 0);
  std::vector<int32_t> n_trace(params.record_trace ? n : 0);
  uint64_t visits = 0;
  check_status(salvox_abmsod_run(device_context(current_device()), v.data().data(), v.nx(),
                                 v.ny(), v.nz(), &w, &p, pos.data(), H.data(), nullptr,
                                 int64_t(n), out.data(),
                                 params.record_trace ? trace.data() : nullptr,
                                 params.record_trace ? n_trace.data() : nullptr, &visits));
  if (counter) counter->add(visits);
  std::vector<AbmsodResult> res(n);
  for (size_t i = 0; i < n; ++i) {
    res[i].det = from_c(out[i]);
    if (!params.record_trace) continue;
    for (int32_t t = 0; t < n_trace[i]; ++t) {
      const salvox_abmsod_iter& c = trace[i * m + size_t(t)];
      AbmsodIterRecord rec;
      rec.position = Eigen::Vector3d(c.position[0], c.position[1], c.position[2]);
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) rec.H(r, k) = c.H[3 * r + k];
      rec.bhattacharyya = c.bhattacharyya;
      rec.max_bhattacharyya = c.max_bhattacharyya;
      rec.eig_min = c.eig_min;
      rec.eig_max = c.eig_max;
      res[i].trace.push_back(rec);
    }
  }
  return res;
}

AbmsodResult abmsod_run(const Volume& v, const EllipsoidWindow& seed, const AbmsodParams& params,
                        const IntensityWindow& iw, EvalCounter* counter) {
  return abmsod_run_many(v, {seed}, params, iw, counter).front();
}

}  // namespace salvox
