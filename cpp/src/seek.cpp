// Per-seed seek entry points of the C++ API on the B200 (reference
// src/shift.cpp:36-107, src/quadrant.cpp:83-125; octant is new).
#include <algorithm>

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

ShiftResult saliency_shift(const Volume& v, const Eigen::Vector3d& seed, const ShiftParams& params,
                           const IntensityWindow& iw, EvalCounter* counter) {
  if (params.record_trace)
    throw unsupported_error("saliency_shift (device): record_trace is not produced on the device");
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

}  // namespace salvox
