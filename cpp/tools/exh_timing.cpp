// Timing of the C++ drop-in's kadir_brady_exhaustive (pipeline.hpp:49-53) on the
// C2 phantom (256^3, 32 bins, scales 3..15): the whole call as a reference user
// makes it (maps returned in std::vectors, maxima converted), best of N.
//   make -C cpp exh_timing && cpp/exh_timing [N]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "salvox/phantom.hpp"
#include "salvox/pipeline.hpp"

int main(int argc, char** argv) {
  using namespace salvox;
  const int reps = argc > 1 ? std::atoi(argv[1]) : 5;
  const auto spec = PhantomSpec::from_json_text(R"({"dims": [256, 256, 256],
    "background": {"type": "gaussian", "mean": 8.0, "sigma": 2.0},
    "regions": [
      {"shape": "ball", "center": [64, 64, 64], "radius": 8, "fill": {"type": "uniform", "levels": 32}},
      {"shape": "ball", "center": [180, 90, 128], "radius": 12, "fill": {"type": "uniform", "levels": 32}},
      {"shape": "ball", "center": [120, 190, 200], "radius": 15, "fill": {"type": "uniform", "levels": 32}},
      {"shape": "box", "center": [200, 200, 60], "half_extents": [10, 10, 10],
       "fill": {"type": "uniform", "levels": 32}}],
    "rng_seed": 6736})");
  auto [v, gt] = make_phantom(spec);
  std::vector<double> scales;
  for (int s = 3; s <= 15; ++s) scales.push_back(s);
  double best = 1e30;
  size_t nmax = 0;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    const auto res = kadir_brady_exhaustive(v, IntensityWindow(0.0, 32.0, 32), scales,
                                            Kernel::Identity, nullptr, 10000000000000ull);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    best = ms < best ? ms : best;
    nmax = res.maxima.size();
  }
  std::printf("kadir_brady_exhaustive C2 (C++ drop-in, std::vector maps): best %.2f ms of %d, %zu maxima\n",
              best, reps, nmax);
  return 0;
}
