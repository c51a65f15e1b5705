// capi.cu -- context management, errors, and the host-side data formats either
// side of the hot path (seed planning, synthetic phantoms).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "host_math.h"

namespace sx {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
bool debug_sync_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SALVOX_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
}  // namespace sx

using namespace sx;

salvox_ctx::~salvox_ctx() {
  for (DevBuf* b : {&d_vol, &d_bins, &d_score, &d_best, &d_keys, &d_keys_alt, &d_cub, &d_counter,
                    &d_maxima, &d_merge_idx, &d_minmax, &d_dbg, &d_seeds, &d_dets, &d_geom, &d_sel_a, &d_sel_b,
                    &d_sel_c, &d_sel_d, &d_visits, &d_target, &d_seek_vol, &d_seek_bins})
    b->release();
  h_stage.release();
  h_maps.release();
  h_vol.release();
  for (cudaEvent_t e : events) cudaEventDestroy(e);
  if (order_event) cudaEventDestroy(order_event);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (own_stream) cudaStreamDestroy(own_stream);
}

extern "C" const char* salvox_last_error(void) { return g_last_error.c_str(); }

extern "C" int salvox_version(void) { return 100; }

extern "C" int salvox_ctx_create(int device, salvox_ctx** out) {
  return guarded([&] {
    if (!out) fail(SALVOX_EINVAL, "null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      fail(SALVOX_ECUDA, std::string("no CUDA device (the B200 path has no CPU fallback): ") +
                             cudaGetErrorString(e));
    if (device < 0 || device >= n) fail(SALVOX_EINVAL, "device index out of range");
    SX_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    SX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      fail(SALVOX_ECUDA, "libsalvox_b200 is built for sm_100a (Blackwell); device is sm_" +
                             std::to_string(prop.major * 10 + prop.minor));
    auto* c = new salvox_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      fail(SALVOX_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->stream = c->own_stream;
    *out = c;
  });
}

extern "C" int salvox_ctx_destroy(salvox_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    forget_exchange_run(ctx);
    delete ctx;
  });
}

extern "C" int salvox_ctx_set_stream(salvox_ctx* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

extern "C" int salvox_ctx_wait_stream(salvox_ctx* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaStream_t other = static_cast<cudaStream_t>(stream);
    if (other == ctx->stream) return;  // same stream: already ordered
    SX_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->order_event)
      SX_CUDA(cudaEventCreateWithFlags(&ctx->order_event, cudaEventDisableTiming));
    SX_CUDA(cudaEventRecord(ctx->order_event, other));
    SX_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->order_event, 0));
  });
}

extern "C" int salvox_ctx_launch_count(salvox_ctx* ctx, uint64_t* out) {
  return guarded([&] {
    if (!ctx || !out) fail(SALVOX_EINVAL, "null argument");
    *out = ctx->launches;
  });
}

// ---------------------------------------------------------------- seeds.cpp:7-45
extern "C" int salvox_plan_seeds(int32_t nx, int32_t ny, int32_t nz, int32_t mode, double spacing,
                                 int32_t count, const double* scales, int32_t n_scales,
                                 uint64_t rng_seed, double* positions, double* seed_scales,
                                 int64_t cap, int64_t* n_out) {
  return guarded([&] {
    std::vector<SeedRec> seeds;
    plan_seeds(nx, ny, nz, mode, spacing, count, scales, n_scales, rng_seed, seeds);
    if (n_out) *n_out = (int64_t)seeds.size();
    for (int64_t i = 0; i < (int64_t)seeds.size() && i < cap; ++i) {
      if (positions) std::memcpy(positions + 3 * i, seeds[i].pos, 3 * sizeof(double));
      if (seed_scales) seed_scales[i] = seeds[i].scale;
    }
  });
}

// ------------------------------------------------------- phantom.cpp:198-222, 364-421
extern "C" int salvox_make_phantom(int32_t nx, int32_t ny, int32_t nz, int32_t bg_type,
                                   double bg_value, double bg_mean, double bg_sigma,
                                   int32_t n_regions, const int32_t* shape, const double* center,
                                   const double* half_extents, const double* radius,
                                   const double* axes, const int32_t* fill_type,
                                   const int32_t* fill_levels, const double* fill_value,
                                   uint64_t rng_seed, float* v, double* out_centroids) {
  return guarded([&] {
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (bg_type == 1 && !(bg_sigma > 0.0)) fail(SALVOX_ERUNTIME, "background.sigma must be > 0");
    const size_t n = (size_t)nx * ny * nz;
    SplitMix rng(rng_seed);
    if (bg_type == 0) {
      const float c = (float)bg_value;
      std::fill(v, v + n, c);
    } else {
      for (size_t i = 0; i < n; ++i) v[i] = (float)(bg_mean + bg_sigma * rng.gaussian());
    }
    std::vector<uint8_t> occupied(n, 0);
    const int dims[3] = {nx, ny, nz};
    for (int ri = 0; ri < n_regions; ++ri) {
      const PhRegion g = phantom_region(ri, dims, shape, center, half_extents, radius, axes);
      const double* c = g.c;
      const double* half = g.half;
      const Mat3& Hi = g.Hi;
      const int* lo = g.lo;
      const int* hi = g.hi;
      double cs[3] = {0, 0, 0};
      uint64_t cnt = 0;
      for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
          for (int x = lo[0]; x <= hi[0]; ++x) {
            const double d[3] = {x - c[0], y - c[1], z - c[2]};
            bool inside;
            if (shape[ri] == 0) {
              inside = std::abs(d[0]) <= half[0] && std::abs(d[1]) <= half[1] && std::abs(d[2]) <= half[2];
            } else {
              double hd[3];
              for (int i = 0; i < 3; ++i)
                hd[i] = Hi.m[i * 3] * d[0] + (Hi.m[i * 3 + 1] * d[1] + Hi.m[i * 3 + 2] * d[2]);
              inside = ((d[0] * hd[0] + d[1] * hd[1]) + d[2] * hd[2]) <= 1.0;
            }
            if (!inside) continue;
            const size_t idx = (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z);
            if (occupied[idx]) fail(SALVOX_ERUNTIME, "make_phantom: regions overlap");
            occupied[idx] = 1;
            v[idx] = fill_type[ri] == 0 ? (float)rng.below((uint64_t)fill_levels[ri])
                                        : (float)fill_value[ri];
            ++cnt;
            cs[0] += x;
            cs[1] += y;
            cs[2] += z;
          }
      if (cnt == 0) fail(SALVOX_ERUNTIME, "make_phantom: region rasterizes to no voxel");
      if (out_centroids)
        for (int i = 0; i < 3; ++i) out_centroids[3 * ri + i] = cs[i] / (double)cnt;
    }
  });
}
