// salvox C++ API (B200 drop-in) -- the hot-path entry points (reference pipeline.hpp:19-104):
// the exhaustive Kadir-Brady pass and the seed-grid detector, both on the B200.
#pragma once

#include <Eigen/Core>

#include <cstdint>
#include <string>
#include <vector>

#include "salvox/abmsod.hpp"
#include "salvox/detection.hpp"
#include "salvox/phantom.hpp"
#include "salvox/quadrant.hpp"
#include "salvox/seeds.hpp"
#include "salvox/shift.hpp"
#include "salvox/volume.hpp"
#include "salvox/window.hpp"

namespace salvox {

/// Octant is new (3D quadrant ascent).
enum class Method { Quadrant, Shift, Abmsod, Octant };

Method method_from_name(const std::string& name);
const char* method_name(Method m);

struct SaliencyMap {
  Eigen::Vector3i dims = Eigen::Vector3i::Zero();
  std::vector<float> score;
  std::vector<float> best_scale;
};

struct SaliencyMaximum {
  Eigen::Vector3d position = Eigen::Vector3d::Zero();
  double score = 0.0;
  double scale = 0.0;
};

struct ExhaustiveResult {
  SaliencyMap map;
  std::vector<SaliencyMaximum> maxima;  // strict local maxima, score-descending
};

/// Dense scan of every voxel at every scale (identity kernel on the device;
/// the same 2e6 default evaluation budget and error messages as the reference).
ExhaustiveResult kadir_brady_exhaustive(const Volume& v, const IntensityWindow& iw,
                                        const std::vector<double>& scales,
                                        Kernel kernel = Kernel::Identity,
                                        EvalCounter* counter = nullptr,
                                        uint64_t budget = 2'000'000);

std::vector<Detection> dedupe_top_k(std::vector<Detection> dets, int k, double radius);

struct DetectParams {
  Method method = Method::Shift;
  SeedPlan seeds;
  int top_k = 20;
  double dedupe_radius = 5.0;
  double entropy_quantile = 0.9;
  double pdf_quantile = 0.0;
  unsigned workers = 1;  // accepted; the device replaces the host thread pool
  QuadrantParams quadrant;
  ShiftParams shift;
  AbmsodParams abmsod;
};

std::vector<Detection> detect(const Volume& v, const IntensityWindow& iw, DetectParams params,
                              EvalCounter* counter = nullptr);

/// Hu vectors of `slices` axial crops about the window's central slice compared
/// to the template by mean Euclidean distance (pipeline.cpp:218-256). Returns the
/// argmin index; throws on an empty list.
size_t hu_filter(const std::vector<Detection>& dets, const Volume& v, const Volume& template_2d,
                 int slices = 5);
/// Per-detection mean Hu distance to the template (same slicing as hu_filter).
double hu_template_distance(const Detection& det, const Volume& v, const Volume& template_2d,
                            int slices = 5);

/// Sorted linear indices of the window's in-bounds support voxels on `frame`'s
/// grid (pipeline.cpp:185-192), rasterised on the device.
std::vector<uint64_t> rasterize_window(const Volume& frame, const EllipsoidWindow& win);
/// Jaccard index |A∩B| / |A∪B| over sorted voxel index sets (pipeline.cpp:194-211).
double jaccard(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b);
double jaccard(const Volume& frame, const EllipsoidWindow& win, const std::vector<uint64_t>& mask);

/// The evaluation-only comparison detector of the reference (pipeline.cpp:272-309):
/// 6-connected components of the voxels >= threshold, largest first (stable),
/// each with its voxel count and centroid. A host utility off the hot path
/// (DESIGN.md §7), kept so callers of the reference API find it.
struct ThresholdComponent {
  Eigen::Vector3d centroid = Eigen::Vector3d::Zero();
  uint64_t voxels = 0;
};
std::vector<ThresholdComponent> threshold_baseline(const Volume& v, double threshold);

}  // namespace salvox
