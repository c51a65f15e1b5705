// Window operations of the C++ API on the B200 (reference src/window.cpp:5-60,
// src/shift.cpp:15-34, src/quadrant.cpp:18-81): every histogram, centroid and
// box count runs on the device through salvox_window_ops / salvox_ascent_step,
// with the seek kernels' warp routines (the reference's fp64 summation order).
#include <algorithm>
#include <cstring>
#include <deque>

#include "salvox/device.hpp"
#include "salvox/pipeline.hpp"
#include "salvox_capi.h"

namespace salvox {

namespace {

salvox_window c_window(const IntensityWindow& iw) { return salvox_window{iw.low, iw.high, iw.bins, 0}; }

salvox_window_op window_op(int op, const EllipsoidWindow& win, Kernel kernel) {
  salvox_window_op o{};
  o.op = op;
  o.kernel = static_cast<int32_t>(kernel);
  for (int a = 0; a < 3; ++a) o.center[a] = win.center[a];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o.H[3 * r + c] = win.H(r, c);
  return o;
}

// Runs ops on the device; pmf (ops.size() x bins) when requested.
std::vector<salvox_window_result> run_ops(const Volume& v, const IntensityWindow& iw,
                                          const std::vector<salvox_window_op>& ops,
                                          const Histogram* target, std::vector<double>* pmf) {
  const salvox_window w = c_window(iw);
  std::vector<salvox_window_result> out(ops.size());
  if (pmf) pmf->assign(ops.size() * size_t(iw.bins), 0.0);
  check_status(salvox_window_ops(device_context(current_device()), v.data().data(), v.nx(), v.ny(),
                                 v.nz(), &w, target ? target->p.data() : nullptr, ops.data(),
                                 int64_t(ops.size()), out.data(), pmf ? pmf->data() : nullptr));
  return out;
}

EllipsoidWindow shift_window(const Volume& v, const Eigen::Vector3d& x, const ShiftParams& params) {
  Eigen::Vector3d half = params.half_extents;
  if (v.is_2d()) half.z() = 1.0;  // shift.cpp:9
  return EllipsoidWindow::from_half_extents(x, half);
}

}  // namespace

std::optional<Histogram> try_candidate_histogram(const Volume& v, const EllipsoidWindow& win,
                                                 const IntensityWindow& iw, Kernel kernel,
                                                 EvalCounter* counter) {
  std::vector<double> pmf;
  const auto r = run_ops(v, iw, {window_op(SALVOX_WOP_HIST, win, kernel)}, nullptr, &pmf).front();
  if (counter) counter->add(r.visits);
  if (!r.ok) return std::nullopt;
  Histogram h(iw.bins);
  std::copy(pmf.begin(), pmf.begin() + iw.bins, h.p.begin());
  h.normalized = true;
  return h;
}

Histogram candidate_histogram(const Volume& v, const EllipsoidWindow& win, const IntensityWindow& iw,
                              Kernel kernel, EvalCounter* counter) {
  auto h = try_candidate_histogram(v, win, iw, kernel, counter);
  if (!h)
    throw std::invalid_argument(
        "candidate_histogram: window support holds no usable in-bounds voxel");
  return *h;
}

double pdf_difference(const Volume& v, const EllipsoidWindow& win, const IntensityWindow& iw,
                      Kernel kernel, EvalCounter* counter) {
  if (win.scale(v.is_2d()) - 1.0 < 1.0)  // checked before any pass (window.cpp:32-34)
    throw std::invalid_argument("pdf_difference: degenerate scale (inner flank below 1 voxel)");
  const auto r = run_ops(v, iw, {window_op(SALVOX_WOP_PDF_DIFF, win, kernel)}, nullptr, nullptr)
                     .front();
  if (r.ok < 0)
    throw std::invalid_argument("pdf_difference: degenerate scale (inner flank below 1 voxel)");
  if (counter) counter->add(r.visits);
  if (r.ok == 0) throw std::invalid_argument("pdf_difference: degenerate flanking support");
  return r.value[0];
}

double pdf_difference(const Volume& v, const Eigen::Vector3d& center, const IntensityWindow& iw,
                      double scale, Kernel kernel, EvalCounter* counter) {
  return pdf_difference(v, EllipsoidWindow::isotropic(center, scale, v.is_2d()), iw, kernel,
                        counter);
}

double inbounds_support_fraction(const Volume& v, const EllipsoidWindow& win) {
  // the support count does not depend on the bins: any window labels the voxels
  const IntensityWindow iw(0.0, 1.0, 2);
  const auto r = run_ops(v, iw, {window_op(SALVOX_WOP_HIST, win, Kernel::Identity)}, nullptr,
                         nullptr).front();
  const double expected = win.support_volume(v.is_2d());
  if (expected <= 0.0) return 0.0;
  return std::min(1.0, double(r.support) / expected);
}

std::optional<Eigen::Vector3d> shift_step(const Volume& v, const Eigen::Vector3d& x,
                                          const ShiftParams& params, const IntensityWindow& iw,
                                          EvalCounter* counter) {
  salvox_window_op o = window_op(SALVOX_WOP_SHIFT_STEP, shift_window(v, x, params), params.hist_kernel);
  o.step_kernel = static_cast<int32_t>(params.step_kernel);
  const auto r = run_ops(v, iw, {o}, params.target ? &*params.target : nullptr, nullptr).front();
  if (counter) counter->add(r.visits);
  if (!r.ok) return std::nullopt;
  return Eigen::Vector3d(r.value[0], r.value[1], r.value[2]);
}

// saliency_shift with record_trace (shift.cpp:36-107): the trajectory advanced
// one device step at a time so every visited centre can be scored.
ShiftResult saliency_shift_traced(const Volume& v, const Eigen::Vector3d& seed,
                                  const ShiftParams& params, const IntensityWindow& iw,
                                  EvalCounter* counter) {
  params.validate();
  const Histogram q = params.target ? *params.target : Histogram::uniform(iw.bins);
  ShiftResult res;
  Detection& det = res.det;
  det.center = v.clamp_point(seed);
  det.H = shift_window(v, det.center, params).H;
  auto trace_point = [&](const Eigen::Vector3d& x) {
    const auto p = try_candidate_histogram(v, shift_window(v, x, params), iw, params.hist_kernel);
    res.trace.push_back({x, p ? bhattacharyya(*p, q) : 0.0});
  };
  auto too_clipped = [&](const Eigen::Vector3d& x) {
    return inbounds_support_fraction(v, shift_window(v, x, params)) < params.min_inbounds_fraction;
  };
  if (too_clipped(det.center)) {
    det.flags |= kFlagDegenerate;
    return res;
  }
  trace_point(det.center);
  for (int it = 0; it < params.max_iters; ++it) {
    const auto next = shift_step(v, det.center, params, iw, counter);
    det.iterations = it + 1;
    if (!next) {
      det.flags |= kFlagDegenerate;
      break;
    }
    const Eigen::Vector3d clamped = v.clamp_point(*next);
    if ((clamped - *next).norm() > 0.0) det.flags |= kFlagBoundaryClamped;
    const double step = (clamped - det.center).norm();
    det.center = clamped;
    trace_point(det.center);
    if (too_clipped(det.center)) {
      det.flags |= kFlagDegenerate;
      break;
    }
    if (step < params.min_step) {
      det.flags |= kFlagConverged;
      break;
    }
  }
  const EllipsoidWindow final_win = shift_window(v, det.center, params);
  det.H = final_win.H;
  if (!det.has(kFlagDegenerate)) {
    const auto p_score = try_candidate_histogram(v, final_win, iw, Kernel::Epanechnikov, counter);
    const auto p_step = try_candidate_histogram(v, final_win, iw, params.hist_kernel, counter);
    if (p_score && p_step) {
      det.entropy_bits = entropy_bits(*p_score);
      det.bhattacharyya = bhattacharyya(*p_step, q);
    } else {
      det.flags |= kFlagDegenerate;
    }
    try {
      det.pdf_diff = pdf_difference(v, final_win, iw, Kernel::Identity, counter);
    } catch (const std::invalid_argument&) {
      det.pdf_diff = 0.0;
    }
  }
  return res;
}

double box_entropy_bits(const Volume& v, double x0, double x1, double y0, double y1,
                        const IntensityWindow& iw, int min_pixels, EvalCounter* counter) {
  salvox_window_op o{};
  o.op = SALVOX_WOP_BOX_ENTROPY;
  o.min_voxels = min_pixels;
  const double box[6] = {x0, x1, y0, y1, 0.0, 0.0};  // the reference reads slice z = 0
  std::memcpy(o.box, box, sizeof box);
  const auto r = run_ops(v, iw, {o}, nullptr, nullptr).front();
  if (counter) counter->add(r.visits);
  return r.value[0];
}

std::pair<Eigen::Vector2d, QuadrantState> quadrant_step(const Volume& v, const Eigen::Vector2d& p,
                                                        const QuadrantParams& params,
                                                        const IntensityWindow& iw,
                                                        EvalCounter* counter) {
  if (!v.is_2d()) throw std::invalid_argument("quadrant_step: volume must be 2D (nz == 1)");
  params.validate();
  const salvox_window w = c_window(iw);
  const double pt[3] = {p.x(), p.y(), 0.0};
  double moved[3];
  salvox_ascent_state st{};
  uint64_t visits = 0;
  check_status(salvox_ascent_step(device_context(current_device()), v.data().data(), v.nx(), v.ny(),
                                  v.nz(), &w, 2, params.scale_range.data(),
                                  int32_t(params.scale_range.size()), pt, 1, moved, &st, &visits));
  if (counter) counter->add(visits);
  QuadrantState s;
  for (int q = 0; q < 4; ++q) {
    s.entropy[size_t(q)] = st.entropy[q];
    s.best_scale[size_t(q)] = st.best_scale[q];
    s.norm_entropy[size_t(q)] = st.norm_entropy[q];
  }
  s.displacement = Eigen::Vector2d(st.displacement[0], st.displacement[1]);
  s.degenerate = st.degenerate != 0;
  return {Eigen::Vector2d(moved[0], moved[1]), s};
}

std::vector<ThresholdComponent> threshold_baseline(const Volume& v, double threshold) {
  // breadth-first flood fill from each unvisited voxel >= threshold in scan
  // order; neighbours in the order +x, -x, +y, -y, +z, -z; centroid = the sum
  // of the member coordinates in visiting order / count
  std::vector<uint8_t> seen(v.size(), 0);
  std::vector<ThresholdComponent> comps;
  std::deque<std::array<int, 3>> frontier;
  const int step[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
  for (int z = 0; z < v.nz(); ++z)
    for (int y = 0; y < v.ny(); ++y)
      for (int x = 0; x < v.nx(); ++x) {
        const size_t start = v.index(x, y, z);
        if (seen[start] || v.at(x, y, z) < threshold) continue;
        seen[start] = 1;
        frontier.push_back({x, y, z});
        ThresholdComponent comp;
        Eigen::Vector3d sum = Eigen::Vector3d::Zero();
        while (!frontier.empty()) {
          const auto cur = frontier.front();
          frontier.pop_front();
          ++comp.voxels;
          sum += Eigen::Vector3d(cur[0], cur[1], cur[2]);
          for (const auto& d : step) {
            const int a = cur[0] + d[0], b = cur[1] + d[1], c = cur[2] + d[2];
            if (!v.contains(a, b, c)) continue;
            const size_t idx = v.index(a, b, c);
            if (seen[idx] || v.at(a, b, c) < threshold) continue;
            seen[idx] = 1;
            frontier.push_back({a, b, c});
          }
        }
        comp.centroid = sum / double(comp.voxels);
        comps.push_back(comp);
      }
  std::stable_sort(comps.begin(), comps.end(),
                   [](const ThresholdComponent& a, const ThresholdComponent& b) {
                     return a.voxels > b.voxels;
                   });
  return comps;
}

}  // namespace salvox
