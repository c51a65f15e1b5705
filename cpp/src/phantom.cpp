// Synthetic phantoms of the C++ API: spec JSON (reference src/phantom.cpp:99-150)
// and generation through salvox_make_phantom (bit-identical volumes), plus the
// ground-truth masks (rasterised with the same membership rule).
#include "salvox/phantom.hpp"

#include <algorithm>

#include "json_min.hpp"
#include "salvox/device.hpp"
#include "salvox_capi.h"

namespace salvox {

namespace {

using json::Value;

void only_keys(const Value& j, std::initializer_list<const char*> allowed, const std::string& where) {
  if (!j.is_object()) throw std::runtime_error("expected an object in " + where);
  for (const auto& kv : j.obj) {
    bool ok = false;
    for (const char* a : allowed) ok = ok || kv.first == a;
    if (!ok) throw std::runtime_error("unknown key '" + kv.first + "' in " + where);
  }
}

Eigen::Vector3d vec3(const Value& j) {
  if (!j.is_array() || j.arr.size() != 3) throw std::runtime_error("expected a 3-vector");
  return Eigen::Vector3d(j.arr[0].as_number(), j.arr[1].as_number(), j.arr[2].as_number());
}

Value vec3_json(const Eigen::Vector3d& v) {
  Value a = Value::array();
  for (int i = 0; i < 3; ++i) a.push(Value::number(v[i]));
  return a;
}

Eigen::Matrix3d region_H(const RegionSpec& r) {
  if (r.shape == RegionSpec::Shape::Box) return r.half_extents.cwiseProduct(r.half_extents).asDiagonal();
  if (r.shape == RegionSpec::Shape::Ball) return Eigen::Matrix3d::Identity() * r.radius * r.radius;
  return r.axes * r.axes.transpose();
}

}  // namespace

PhantomSpec PhantomSpec::from_json_text(const std::string& text) {
  const Value j = json::parse(text);
  only_keys(j, {"dims", "spacing", "background", "regions", "rng_seed"}, "phantom spec");
  PhantomSpec s;
  const Value& d = j.at("dims");
  if (!d.is_array() || d.arr.size() != 3) throw std::runtime_error("dims must be a 3-array");
  s.dims = Eigen::Vector3i(int(d.arr[0].as_number()), int(d.arr[1].as_number()),
                           int(d.arr[2].as_number()));
  if (j.contains("spacing")) s.spacing = vec3(j.at("spacing"));
  if (j.contains("background")) {
    const Value& bg = j.at("background");
    only_keys(bg, {"type", "value", "mean", "sigma"}, "background");
    const std::string t = bg.at("type").as_string();
    if (t == "constant") {
      s.background.type = BackgroundSpec::Type::Constant;
      s.background.value = bg.number_or("value", 0.0);
    } else if (t == "gaussian") {
      s.background.type = BackgroundSpec::Type::Gaussian;
      s.background.mean = bg.number_or("mean", 0.0);
      s.background.sigma = bg.number_or("sigma", 1.0);
      if (s.background.sigma <= 0.0) throw std::runtime_error("background.sigma must be > 0");
    } else {
      throw std::runtime_error("unknown background type '" + t + "'");
    }
  }
  if (j.contains("regions"))
    for (const Value& rj : j.at("regions").arr) {
      only_keys(rj, {"shape", "center", "half_extents", "radius", "axes", "fill"}, "region");
      RegionSpec r;
      const std::string shape = rj.at("shape").as_string();
      r.center = vec3(rj.at("center"));
      if (shape == "box") {
        r.shape = RegionSpec::Shape::Box;
        r.half_extents = vec3(rj.at("half_extents"));
      } else if (shape == "ball") {
        r.shape = RegionSpec::Shape::Ball;
        r.radius = rj.at("radius").as_number();
      } else if (shape == "ellipsoid") {
        r.shape = RegionSpec::Shape::Ellipsoid;
        const Value& a = rj.at("axes");
        if (!a.is_array() || a.arr.size() != 3) throw std::runtime_error("expected a 3x3 matrix");
        for (int row = 0; row < 3; ++row) {
          const Eigen::Vector3d rv = vec3(a.arr[size_t(row)]);
          for (int c = 0; c < 3; ++c) r.axes(row, c) = rv[c];
        }
      } else {
        throw std::runtime_error("unknown region shape '" + shape + "'");
      }
      if (rj.contains("fill")) {
        const Value& f = rj.at("fill");
        only_keys(f, {"type", "levels", "value"}, "fill");
        const std::string t = f.at("type").as_string();
        if (t == "uniform") {
          r.fill.type = FillSpec::Type::Uniform;
          r.fill.levels = int(f.number_or("levels", 64));
          if (r.fill.levels < 2) throw std::runtime_error("fill.levels must be >= 2");
        } else if (t == "constant") {
          r.fill.type = FillSpec::Type::Constant;
          r.fill.value = f.at("value").as_number();
        } else {
          throw std::runtime_error("unknown fill type '" + t + "'");
        }
      }
      s.regions.push_back(r);
    }
  s.rng_seed = j.contains("rng_seed") ? uint64_t(j.at("rng_seed").as_number()) : 0;
  return s;
}

std::string PhantomSpec::to_json_text() const {
  Value j = Value::object();
  Value d = Value::array();
  for (int i = 0; i < 3; ++i) d.push(Value::number(dims[i]));
  j.set("dims", d);
  j.set("spacing", vec3_json(spacing));
  Value bg = Value::object();
  if (background.type == BackgroundSpec::Type::Constant) {
    bg.set("type", Value::string("constant"));
    bg.set("value", Value::number(background.value));
  } else {
    bg.set("type", Value::string("gaussian"));
    bg.set("mean", Value::number(background.mean));
    bg.set("sigma", Value::number(background.sigma));
  }
  j.set("background", bg);
  Value regs = Value::array();
  for (const RegionSpec& r : regions) {
    Value rj = Value::object();
    rj.set("center", vec3_json(r.center));
    if (r.shape == RegionSpec::Shape::Box) {
      rj.set("shape", Value::string("box"));
      rj.set("half_extents", vec3_json(r.half_extents));
    } else if (r.shape == RegionSpec::Shape::Ball) {
      rj.set("shape", Value::string("ball"));
      rj.set("radius", Value::number(r.radius));
    } else {
      rj.set("shape", Value::string("ellipsoid"));
      Value a = Value::array();
      for (int row = 0; row < 3; ++row)
        a.push(vec3_json(Eigen::Vector3d(r.axes(row, 0), r.axes(row, 1), r.axes(row, 2))));
      rj.set("axes", a);
    }
    Value f = Value::object();
    if (r.fill.type == FillSpec::Type::Uniform) {
      f.set("type", Value::string("uniform"));
      f.set("levels", Value::number(r.fill.levels));
    } else {
      f.set("type", Value::string("constant"));
      f.set("value", Value::number(r.fill.value));
    }
    rj.set("fill", f);
    regs.push(rj);
  }
  j.set("regions", regs);
  j.set("rng_seed", Value::number(double(rng_seed)));
  return json::dump(j, 2);
}

std::string GroundTruth::to_json_text() const {
  Value j = Value::object();
  Value d = Value::array();
  for (int i = 0; i < 3; ++i) d.push(Value::number(dims[i]));
  j.set("dims", d);
  Value regs = Value::array();
  for (const auto& r : regions) {
    Value rj = Value::object();
    rj.set("center", vec3_json(r.center));
    Value h = Value::array();
    for (int row = 0; row < 3; ++row)
      for (int c = 0; c < 3; ++c) h.push(Value::number(r.H(row, c)));
    rj.set("H", h);
    Value rle = Value::array();  // [start, len, start, len, ...]
    for (size_t i = 0; i < r.mask.size();) {
      size_t len = 1;
      while (i + len < r.mask.size() && r.mask[i + len] == r.mask[i] + len) ++len;
      rle.push(Value::number(double(r.mask[i])));
      rle.push(Value::number(double(len)));
      i += len;
    }
    rj.set("mask_rle", rle);
    regs.push(rj);
  }
  j.set("regions", regs);
  return json::dump(j);
}

GroundTruth GroundTruth::from_json_text(const std::string& text) {  // phantom.cpp:213-235
  const Value j = json::parse(text);
  GroundTruth gt;
  const Value& dims = j.at("dims");
  if (!dims.is_array() || dims.arr.size() < 3) throw std::invalid_argument("json: bad dims");
  for (int i = 0; i < 3; ++i) gt.dims[i] = int(dims.arr[size_t(i)].as_number());
  for (const Value& rj : j.at("regions").arr) {
    GroundTruthRegion r;
    const Value& c = rj.at("center");
    for (int i = 0; i < 3; ++i) r.center[i] = c.arr.at(size_t(i)).as_number();
    const Value& h = rj.at("H");
    if (h.arr.size() != 9) throw std::runtime_error("ground truth H must have 9 entries");
    for (int row = 0; row < 3; ++row)
      for (int col = 0; col < 3; ++col) r.H(row, col) = h.arr[size_t(row * 3 + col)].as_number();
    const Value& rle = rj.at("mask_rle");
    if (rle.arr.size() % 2 != 0) throw std::runtime_error("mask_rle must have even length");
    for (size_t i = 0; i < rle.arr.size(); i += 2) {
      const uint64_t start = uint64_t(rle.arr[i].as_number());
      const uint64_t len = uint64_t(rle.arr[i + 1].as_number());
      for (uint64_t k = 0; k < len; ++k) r.mask.push_back(start + k);
    }
    gt.regions.push_back(std::move(r));
  }
  return gt;
}

std::pair<Volume, GroundTruth> make_phantom(const PhantomSpec& spec) {
  Volume v(spec.dims[0], spec.dims[1], spec.dims[2], spec.spacing);
  const size_t nr = spec.regions.size(), m = std::max<size_t>(nr, 1);
  std::vector<int32_t> shape(m), ftype(m), flev(m, 64);
  std::vector<double> center(3 * m), half(3 * m), radius(m), axes(9 * m), fval(m), cent(3 * m);
  for (size_t i = 0; i < nr; ++i) {
    const RegionSpec& r = spec.regions[i];
    shape[i] = int32_t(r.shape);
    for (int k = 0; k < 3; ++k) {
      center[3 * i + size_t(k)] = r.center[k];
      half[3 * i + size_t(k)] = r.half_extents[k];
      for (int c = 0; c < 3; ++c) axes[9 * i + size_t(3 * k + c)] = r.axes(k, c);
    }
    radius[i] = r.radius;
    ftype[i] = r.fill.type == FillSpec::Type::Uniform ? 0 : 1;
    flev[i] = r.fill.levels;
    fval[i] = r.fill.value;
  }
  const bool gauss = spec.background.type == BackgroundSpec::Type::Gaussian;
  check_status(salvox_make_phantom(v.nx(), v.ny(), v.nz(), gauss ? 1 : 0, spec.background.value,
                                   spec.background.mean, spec.background.sigma, int32_t(nr),
                                   shape.data(), center.data(), half.data(), radius.data(),
                                   axes.data(), ftype.data(), flev.data(), fval.data(),
                                   spec.rng_seed, v.data().data(), cent.data()));
  GroundTruth gt;
  gt.dims = spec.dims;
  for (size_t i = 0; i < nr; ++i) {
    const RegionSpec& r = spec.regions[i];
    GroundTruthRegion out;
    out.H = region_H(r);
    out.center = Eigen::Vector3d(cent[3 * i], cent[3 * i + 1], cent[3 * i + 2]);
    const Eigen::Vector3d ext = r.shape == RegionSpec::Shape::Box
                                    ? r.half_extents
                                    : Eigen::Vector3d(out.H.diagonal().cwiseMax(0.0).cwiseSqrt());
    const Eigen::Matrix3d Hinv =
        r.shape == RegionSpec::Shape::Box ? Eigen::Matrix3d::Identity() : out.H.inverse();
    int lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::max(0, int(std::floor(r.center[k] - ext[k])));
      hi[k] = std::min(spec.dims[k] - 1, int(std::ceil(r.center[k] + ext[k])));
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          const Eigen::Vector3d dv(x - r.center.x(), y - r.center.y(), z - r.center.z());
          const bool in = r.shape == RegionSpec::Shape::Box
                              ? (std::abs(dv.x()) <= r.half_extents.x() &&
                                 std::abs(dv.y()) <= r.half_extents.y() &&
                                 std::abs(dv.z()) <= r.half_extents.z())
                              : dv.dot(Hinv * dv) <= 1.0;
          if (in) out.mask.push_back(v.index(x, y, z));
        }
    gt.regions.push_back(std::move(out));
  }
  return {std::move(v), std::move(gt)};
}

}  // namespace salvox
