// C++ drop-in API tests: the reference's own doctest cases (proj/tests/*.cpp),
// ported to a minimal harness and run against the B200 implementation through
// the salvox C++ API. `test_host_api cpu` runs the host-only cases (config,
// MetaImage IO, phantom, KATs); `test_host_api gpu` the device cases.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <string>
#include <vector>

#include "salvox/abmsod.hpp"
#include "salvox/config.hpp"
#include "salvox/device.hpp"
#include "salvox/histogram.hpp"
#include "salvox/hu.hpp"
#include "salvox/meta_io.hpp"
#include "salvox/phantom.hpp"
#include "salvox/pipeline.hpp"
#include "salvox/report.hpp"

using namespace salvox;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                 \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(c)) {                                                                  \
      ++g_fail;                                                                  \
      std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #c "\n";  \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, E)                                                 \
  do {                                                                           \
    ++g_checks;                                                                  \
    bool caught_ = false;                                                        \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const E&) {                                                         \
      caught_ = true;                                                            \
    } catch (...) {                                                              \
    }                                                                            \
    if (!caught_) {                                                              \
      ++g_fail;                                                                  \
      std::cerr << __FILE__ << ":" << __LINE__ << ": expected " #E " from " #expr "\n"; \
    }                                                                            \
  } while (0)

namespace {

PhantomSpec square_2d(int dim, double cx, double cy, int half, uint64_t seed) {
  PhantomSpec s;
  s.dims = Eigen::Vector3i(dim, dim, 1);
  RegionSpec r;
  r.shape = RegionSpec::Shape::Box;
  r.center = Eigen::Vector3d(cx, cy, 0.0);
  r.half_extents = Eigen::Vector3d(half, half, 0.0);
  r.fill.levels = 64;
  s.regions.push_back(r);
  s.rng_seed = seed;
  return s;
}

PhantomSpec cube_3d(int dim, int half, uint64_t seed) {
  PhantomSpec s;
  s.dims = Eigen::Vector3i(dim, dim, dim);
  RegionSpec r;
  r.shape = RegionSpec::Shape::Box;
  const double c = (dim - 1) / 2.0;
  r.center = Eigen::Vector3d(c, c, c);
  r.half_extents = Eigen::Vector3d(half, half, half);
  r.fill.levels = 64;
  s.regions.push_back(r);
  s.rng_seed = seed;
  return s;
}

// ------------------------------------------------------------------ host only
void cpu_tests() {
  {  // test_seek.cpp:427-450: bandwidth_from_moment (host 3x3 math)
    Eigen::Matrix3d outer = Eigen::Matrix3d::Zero();
    outer(0, 0) = 2.0 * 9.0;
    const Eigen::Matrix3d H = bandwidth_from_moment(outer, 2.0, 3, 4.0, 1024.0);
    CHECK(std::abs(H(0, 0) - 45.0) < 1e-9 && std::abs(H(1, 1) - 4.0) < 1e-9 &&
          std::abs(H(2, 2) - 4.0) < 1e-9);
    CHECK_THROWS_AS(bandwidth_from_moment(outer, 0.0, 3, 4.0, 4096.0), std::invalid_argument);
  }
  // test_volume.cpp:35-49
  CHECK(IntensityWindow(0, 256, 256).bin_of(0.0) == 0);
  CHECK(IntensityWindow(0, 100, 10).bin_of(55.0) == 5);
  CHECK(IntensityWindow(40, 80, 16).bin_of(1000.0) == 15);
  CHECK(IntensityWindow(40, 80, 16).bin_of(-1000.0) == 0);
  CHECK_THROWS_AS(IntensityWindow(1.0, 1.0, 8), std::invalid_argument);
  CHECK_THROWS_AS(IntensityWindow(0.0, 1.0, 1), std::invalid_argument);
  CHECK_THROWS_AS(Volume(0, 4, 4), std::invalid_argument);
  // test_entropy.cpp:13-26
  CHECK(entropy_bits(Histogram::delta(16, 3)) == 0.0);
  CHECK(std::abs(entropy_bits(Histogram::uniform(256)) - 8.0) < 1e-12);
  Histogram h(4);
  h.p = {0.5, 0.25, 0.25, 0.0};
  h.normalized = true;
  CHECK(std::abs(entropy_bits(h) - 1.5) < 1e-12);
  // MetaImage round trip + errors (test_volume.cpp:67-171)
  const auto dir = std::filesystem::temp_directory_path() / "salvox_b200_cpp_tests";
  std::filesystem::create_directories(dir);
  Volume v(9, 7, 5, Eigen::Vector3d(0.5, 0.75, 2.0));
  for (size_t i = 0; i < v.size(); ++i) v.data()[i] = float(i) * 0.37f - 3.0f;
  save_volume(v, dir / "rt.mhd");
  const Volume w = load_volume(dir / "rt.mhd");
  CHECK(w.nx() == 9 && w.ny() == 7 && w.nz() == 5);
  CHECK(w.spacing() == v.spacing());
  bool same = true;
  for (size_t i = 0; i < v.size(); ++i) same = same && v.data()[i] == w.data()[i];
  CHECK(same);
  CHECK_THROWS_AS(load_volume(dir / "missing.mhd"), std::runtime_error);
  {
    std::ofstream(dir / "u8.mhd") << "NDims = 2\nDimSize = 3 2\nElementType = MET_UCHAR\n"
                                     "ElementDataFile = u8.raw\n";
    std::ofstream raw(dir / "u8.raw", std::ios::binary);
    const unsigned char b[6] = {0, 1, 2, 250, 4, 5};
    raw.write(reinterpret_cast<const char*>(b), 6);
  }
  const Volume u = load_volume(dir / "u8.mhd");
  CHECK(u.nz() == 1 && u.at(0, 1, 0) == 250.0f);
  std::ofstream(dir / "bad.mhd") << "NDims = 3\nDimSize = 2 2 2\nElementType = MET_DOUBLE\n"
                                    "ElementDataFile = u8.raw\n";
  CHECK_THROWS_AS(load_volume(dir / "bad.mhd"), std::runtime_error);
  std::ofstream(dir / "short.mhd") << "NDims = 3\nDimSize = 2 2 2\nElementType = MET_UCHAR\n"
                                      "ElementDataFile = u8.raw\n";
  CHECK_THROWS_AS(load_volume(dir / "short.mhd"), std::runtime_error);
  std::ofstream(dir / "be.mhd") << "NDims = 2\nDimSize = 3 2\nElementType = MET_UCHAR\n"
                                   "BinaryDataByteOrderMSB = True\nElementDataFile = u8.raw\n";
  CHECK_THROWS_AS(load_volume(dir / "be.mhd"), std::runtime_error);
  // RunConfig (test_cli.cpp:137-167 semantics)
  const RunConfig c = RunConfig::from_json_text(
      R"({"method": "octant", "bins": 16, "scales": [3, 5, 7], "seeds": {"mode": "lattice",
          "spacing": 8}, "window": {"low": 0, "high": 16}, "params": {"quadrant_eta": 0.25}})");
  CHECK(c.method == "octant" && c.bins == 16 && c.scales.size() == 3 && c.seed_spacing == 8.0);
  CHECK(c.window_low && *c.window_high == 16.0 && c.quadrant_eta == 0.25);
  const RunConfig c2 = RunConfig::from_json_text(c.to_json_text());
  CHECK(c2.to_json_text() == c.to_json_text());
  CHECK(c.detect_params().method == Method::Octant);
  CHECK(c.detect_params().quadrant.scale_range == std::vector<int>({3, 5, 7}));
  CHECK_THROWS_AS(RunConfig::from_json_text(R"({"bogus": 1})"), std::invalid_argument);
  CHECK_THROWS_AS(RunConfig::from_json_text(R"({"params": {"nope": 1}})"), std::invalid_argument);
  CHECK_THROWS_AS(RunConfig::from_json_text(R"({"method": "hough"})"), std::invalid_argument);
  // phantom spec JSON round trip + deterministic generation
  PhantomSpec ps = PhantomSpec::from_json_text(
      R"({"dims": [48, 48, 48], "background": {"type": "gaussian", "mean": 8, "sigma": 2},
          "regions": [{"shape": "ball", "center": [24, 24, 24], "radius": 8,
                       "fill": {"type": "uniform", "levels": 64}}], "rng_seed": 404})");
  CHECK(PhantomSpec::from_json_text(ps.to_json_text()).to_json_text() == ps.to_json_text());
  auto [pv, gt] = make_phantom(ps);
  auto [pv2, gt2] = make_phantom(ps);
  CHECK(fnv1a64(pv.data().data(), pv.size() * 4) == fnv1a64(pv2.data().data(), pv2.size() * 4));
  CHECK(gt.regions.size() == 1 && !gt.regions[0].mask.empty());
  std::cout << "phantom404 " << fnv1a64_hex(pv.data().data(), pv.size() * 4) << "\n";
  CHECK_THROWS_AS(make_phantom(PhantomSpec::from_json_text(
                      R"({"dims": [16, 16, 16], "regions": [{"shape": "ball",
                          "center": [2, 8, 8], "radius": 5}]})")),
                  std::runtime_error);
}

// ------------------------------------------------------------------ device
void gpu_tests() {
  {  // test_pipeline.cpp:228-236
    auto [v, gt] = make_phantom(square_2d(64, 31.0, 31.0, 8, 77));
    EvalCounter counter;
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(0, 64, 64), {4.0, 6.0, 8.0, 10.0},
                                            Kernel::Identity, &counter);
    CHECK(!res.maxima.empty());
    CHECK((res.maxima.front().position - Eigen::Vector3d(31, 31, 0)).norm() <= 2.0);
    CHECK(std::abs(res.maxima.front().scale - 8.0) <= 2.0);
    CHECK(counter.count() > 0);
  }
  {  // the same fixture with the Epanechnikov kernel (exact r^2 C_b - S_b on the device)
    auto [v, gt] = make_phantom(square_2d(64, 31.0, 31.0, 8, 77));
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(0, 64, 64), {4.0, 6.0, 8.0, 10.0},
                                            Kernel::Epanechnikov);
    CHECK(!res.maxima.empty());
    CHECK((res.maxima.front().position - Eigen::Vector3d(31, 31, 0)).norm() <= 3.0);
    CHECK_THROWS_AS(kadir_brady_exhaustive(v, IntensityWindow(0, 64, 64), {4.0, 6.0},
                                           Kernel::Gaussian),
                    unsupported_error);
  }
  {  // test_pipeline.cpp:238-245
    Volume v(48, 48, 1);
    for (float& f : v.data()) f = 2.0f;
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(0, 64, 64), {4.0, 6.0});
    CHECK(res.maxima.empty());
    bool zero = true;
    for (float s : res.map.score) zero = zero && s == 0.0f;
    CHECK(zero);
  }
  {  // test_pipeline.cpp:247-270
    PhantomSpec s = square_2d(96, 24.0, 24.0, 8, 78);
    RegionSpec r2 = s.regions[0];
    r2.center = Eigen::Vector3d(68, 66, 0);
    s.regions.push_back(r2);
    auto [v, gt] = make_phantom(s);
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(0, 64, 64), {6.0, 8.0, 10.0});
    std::vector<Detection> as_dets;
    for (const auto& m : res.maxima) {
      Detection d;
      d.center = m.position;
      d.pdf_diff = m.score;
      as_dets.push_back(d);
    }
    const auto top2 = dedupe_top_k(as_dets, 2, 10.0);
    CHECK(top2.size() == 2);
    bool a = false, b = false;
    for (const auto& d : top2) {
      a = a || (d.center - Eigen::Vector3d(24, 24, 0)).norm() <= 3.0;
      b = b || (d.center - Eigen::Vector3d(68, 66, 0)).norm() <= 3.0;
    }
    CHECK(a && b);
  }
  // test_pipeline.cpp:272-276
  CHECK_THROWS_AS(kadir_brady_exhaustive(Volume(256, 256, 34), IntensityWindow(0, 64, 64), {4.0, 6.0}),
                  std::invalid_argument);
  {  // test_pipeline.cpp:296-319
    PhantomSpec s;
    s.dims = Eigen::Vector3i(64, 64, 64);
    RegionSpec r;
    r.shape = RegionSpec::Shape::Ball;
    r.center = Eigen::Vector3d(36.0, 30.0, 28.0);
    r.radius = 9.0;
    s.regions.push_back(r);
    s.rng_seed = 101;
    auto [v, gt] = make_phantom(s);
    DetectParams p;
    p.method = Method::Shift;
    p.seeds.spacing = 16.0;
    p.seeds.scales = {6.0, 9.0};
    p.top_k = 5;
    p.dedupe_radius = 6.0;
    const auto dets = detect(v, IntensityWindow(0, 64, 64), p);
    CHECK(!dets.empty());
    CHECK(!dets.empty() && (dets.front().center - gt.regions[0].center).norm() <= 2.0);
    p.method = Method::Octant;
    p.seeds.scales = {4.0, 8.0, 12.0};
    const auto od = detect(v, IntensityWindow(0, 64, 64), p);
    CHECK(!od.empty());
    p.method = Method::Abmsod;  // test_pipeline.cpp:321-354 (ABMSOD through detect)
    p.seeds.scales = {6.0, 9.0};
    const auto ad = detect(v, IntensityWindow(0, 64, 64), p);
    CHECK(!ad.empty() && (ad.front().center - gt.regions[0].center).norm() <= 3.0);
    p.abmsod.threshold = 0.0;
    CHECK_THROWS_AS(detect(v, IntensityWindow(0, 64, 64), p), std::invalid_argument);
  }
  {  // test_pipeline.cpp:381-400
    Volume v(48, 48, 48);
    for (float& f : v.data()) f = 1.0f;
    DetectParams p;
    p.seeds.spacing = 16.0;
    p.seeds.scales = {6.0};
    CHECK(detect(v, IntensityWindow(0, 64, 64), p).empty());
    DetectParams q;
    q.method = Method::Quadrant;
    CHECK_THROWS_AS(detect(Volume(16, 16, 16), IntensityWindow(0, 64, 64), q), std::invalid_argument);
  }
  {  // test_seek.cpp:148-166
    auto [v, gt] = make_phantom(square_2d(128, 63.0, 63.0, 12, 23));
    QuadrantParams qp;
    qp.scale_range = {4, 8, 12, 16};
    std::vector<Eigen::Vector2d> seeds;
    for (int y = 8; y < 128; y += 16)
      for (int x = 8; x < 128; x += 16) seeds.emplace_back(x, y);
    const auto res = quadrant_seek(v, seeds, qp, IntensityWindow(0, 64, 64));
    CHECK(res.size() == seeds.size());
    bool hit = false;
    for (const auto& r : res)
      hit = hit || (!r.degenerate && (r.position - Eigen::Vector2d(63.0, 63.0)).norm() <= 3.0);
    CHECK(hit);
  }
  {  // test_seek.cpp:333-375
    auto [v, gt] = make_phantom(cube_3d(64, 8, 71));
    ShiftParams sp;
    sp.half_extents = Eigen::Vector3d(8.0, 8.0, 8.0);
    const Eigen::Vector3d c = gt.regions[0].center;
    const auto r = saliency_shift(v, c + Eigen::Vector3d(6.0, 0.0, 0.0), sp, IntensityWindow(0, 64, 64));
    CHECK(!r.det.has(kFlagDegenerate) && r.det.iterations <= 20);
    CHECK((r.det.center - c).norm() <= 2.0);
    const auto again = saliency_shift(v, r.det.center, sp, IntensityWindow(0, 64, 64));
    CHECK(again.det.has(kFlagConverged) && again.det.iterations == 1);
    ShiftParams an;
    an.half_extents = Eigen::Vector3d(6.0, 5.0, 4.0);
    const auto d = saliency_shift(v, Eigen::Vector3d(10, 50, 20), an, IntensityWindow(0, 64, 64));
    CHECK(d.det.H == EllipsoidWindow::from_half_extents(Eigen::Vector3d::Zero(), an.half_extents).H);
    CHECK(v.contains_point(d.det.center));
    QuadrantParams qp;
    qp.scale_range = {3, 6, 9};
    const auto oc = octant_seek(v, {Eigen::Vector3d(40.0, 36.0, 26.0)}, qp, IntensityWindow(0, 64, 64));
    CHECK(!oc[0].degenerate && (oc[0].position - c).norm() <= 4.0);
  }
  {  // test_seek.cpp:495-514 + 561-571: abmsod_run on the device
    PhantomSpec s;
    s.dims = Eigen::Vector3i(64, 64, 64);
    RegionSpec r;
    r.shape = RegionSpec::Shape::Ellipsoid;
    r.center = Eigen::Vector3d(31.5, 31.5, 31.5);
    r.axes = Eigen::Matrix3d::Zero();
    r.axes(0, 0) = 9.0, r.axes(1, 1) = 6.0, r.axes(2, 2) = 4.0;
    r.fill.levels = 64;
    s.regions.push_back(r);
    s.rng_seed = 111;
    auto [v, gt] = make_phantom(s);
    EllipsoidWindow seed;
    seed.center = gt.regions[0].center;
    seed.H = gt.regions[0].H;
    AbmsodParams ap;
    ap.record_trace = true;
    const auto res = abmsod_run(v, seed, ap, IntensityWindow(0, 64, 64));
    CHECK(!res.det.has(kFlagDegenerate));
    CHECK((res.det.center - gt.regions[0].center).norm() <= 1.0);
    CHECK(!res.trace.empty() && int(res.trace.size()) == res.det.iterations);
    for (const auto& t : res.trace) CHECK(t.eig_min >= ap.lambda_min - 1e-9);
    Volume c(32, 32, 32);
    for (float& f : c.data()) f = 20.0f;
    const auto rc = abmsod_run(c, EllipsoidWindow::isotropic(Eigen::Vector3d(16, 16, 16), 6.0, false),
                               ap, IntensityWindow(0, 64, 64));
    CHECK(!rc.trace.empty() && std::abs(rc.trace.front().bhattacharyya - std::sqrt(1.0 / 64)) < 1e-12);
    CHECK(rc.det.entropy_bits == 0.0);
  }
  {  // test_pipeline.cpp:149-206: Hu invariances and the disk
    Volume img(64, 64, 1);
    uint64_t st = 31;
    for (int y = 16; y < 48; ++y)
      for (int x = 16; x < 48; ++x) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        img.at(x, y, 0) = float((st >> 40) % 64);
      }
    const HuVector base = hu_moments(img);
    Volume sh(64, 64, 1);
    for (int y = 0; y < 64; ++y)
      for (int x = 0; x < 64; ++x) sh.at((x + 5) % 64, (y + 3) % 64, 0) = img.at(x, y, 0);
    const HuVector hs = hu_moments(sh);
    for (int i = 0; i < 7; ++i) CHECK(std::abs(hs[i] - base[i]) < 1e-9);
    Volume rot(64, 64, 1);
    for (int y = 0; y < 64; ++y)
      for (int x = 0; x < 64; ++x) rot.at(63 - y, x, 0) = img.at(x, y, 0);
    const HuVector hr = hu_moments(rot);
    for (int i = 0; i < 7; ++i) CHECK(std::abs(hr[i] - base[i]) <= 1e-6 * std::max(1e-12, std::abs(base[i])));
    CHECK(hu_distance(base, base) == 0.0);
    Volume disk(64, 64, 1);
    for (int y = 0; y < 64; ++y)
      for (int x = 0; x < 64; ++x)
        disk.at(x, y, 0) = (x - 31.5) * (x - 31.5) + (y - 31.5) * (y - 31.5) <= 196.0 ? 1.0f : 0.0f;
    const HuVector hd = hu_moments(disk);
    CHECK(hd[0] > 0.15 && hd[0] < 0.17);
    for (int i = 2; i < 7; ++i) CHECK(std::abs(hd[i]) < 1e-9);
    CHECK_THROWS_AS(hu_moments(Volume(8, 8, 1)), std::invalid_argument);
    CHECK_THROWS_AS(hu_moments(Volume(8, 8, 2)), std::invalid_argument);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "all";
  try {
    if (mode == "cpu" || mode == "all") cpu_tests();
    if (mode == "gpu" || mode == "all") gpu_tests();
  } catch (const std::exception& e) {
    std::cerr << "uncaught exception: " << e.what() << "\n";
    return 2;
  }
  std::cout << g_checks << " checks, " << g_fail << " failed\n";
  return g_fail == 0 ? 0 : 1;
}
