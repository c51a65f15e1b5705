// ingest.cu -- on-device MetaImage payload widening.
//
// load_volume (reference src/meta_io.cpp:30-33, :100-105) reads a MET_UCHAR /
// MET_SHORT / MET_USHORT / MET_FLOAT payload and widens it to float on the host.
// Here the payload crosses PCIe at its native width (1-2 bytes per voxel instead
// of 4) and is widened on the device by an HBM-bound kernel; static_cast<float>
// of these integer types is exact, so the result is bit-identical.
#include "../../include/salvox_capi.h"
#include "common.cuh"
#include "host_math.h"

namespace sx {

template <class T>
__global__ void widen_kernel(const T* __restrict__ in, float* __restrict__ out, long long n) {
  // 4 elements per thread per step, grid-stride (coalesced, HBM-bound)
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k < n) out[i + k] = static_cast<float>(__ldg(in + i + k));
  }
}

size_t element_size(int type) {
  switch (type) {
    case SALVOX_MET_UCHAR: return 1;
    case SALVOX_MET_SHORT:
    case SALVOX_MET_USHORT: return 2;
    case SALVOX_MET_FLOAT: return 4;
    default: fail(SALVOX_EINVAL, "load_volume: unsupported ElementType code " + std::to_string(type));
  }
  return 0;
}

void launch_widen(salvox_ctx* ctx, int type, const void* d_raw, long long n, float* d_out) {
  if (n <= 0) return;
  const int block = 256;
  const int grid = (int)std::min<long long>((n + 4LL * block - 1) / (4LL * block), ctx->sm_count * 16LL);
  switch (type) {
    case SALVOX_MET_UCHAR:
      widen_kernel<uint8_t><<<grid, block, 0, ctx->stream>>>(static_cast<const uint8_t*>(d_raw), d_out, n);
      break;
    case SALVOX_MET_SHORT:
      widen_kernel<int16_t><<<grid, block, 0, ctx->stream>>>(static_cast<const int16_t*>(d_raw), d_out, n);
      break;
    case SALVOX_MET_USHORT:
      widen_kernel<uint16_t><<<grid, block, 0, ctx->stream>>>(static_cast<const uint16_t*>(d_raw), d_out, n);
      break;
    default:  // MET_FLOAT: already the volume's type
      if (d_raw != d_out)
        SX_CUDA(cudaMemcpyAsync(d_out, d_raw, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      return;
  }
  SX_LAUNCH_CHECK(ctx);
}

}  // namespace sx

using namespace sx;

extern "C" int salvox_widen_device(salvox_ctx* ctx, int32_t element_type, const void* d_raw,
                                   int64_t n, float* d_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    element_size(element_type);
    if (n < 0 || (n > 0 && (!d_raw || !d_out))) fail(SALVOX_EINVAL, "bad arguments");
    SX_CUDA(cudaSetDevice(ctx->device));
    launch_widen(ctx, element_type, d_raw, n, d_out);
  });
}

extern "C" int salvox_upload_widen(salvox_ctx* ctx, int32_t element_type, const void* raw,
                                   int64_t n, float* d_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t es = element_size(element_type);
    if (n < 0 || (n > 0 && (!raw || !d_out))) fail(SALVOX_EINVAL, "bad arguments");
    if (n == 0) return;
    SX_CUDA(cudaSetDevice(ctx->device));
    if (element_type == SALVOX_MET_FLOAT) {
      SX_CUDA(cudaMemcpyAsync(d_out, raw, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
    } else {  // native-width payload staged in a context buffer, then widened into d_out
      void* d_raw = ctx->d_dbg.ensure((size_t)n * es);
      SX_CUDA(cudaMemcpyAsync(d_raw, raw, (size_t)n * es, cudaMemcpyHostToDevice, ctx->stream));
      launch_widen(ctx, element_type, d_raw, n, d_out);
    }
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------------------ evaluation
// rasterize_window (reference src/pipeline.cpp:185-192): the window's support
// voxels in z->y->x order (= ascending linear index), on the device: one flag
// per bounding-box voxel (the reference's Mahalanobis expression and order,
// Eigen-identical inverse), then an ordered compaction (cub::DeviceSelect).
#include <cub/cub.cuh>

#include "../../include/salvox/sx_eig3.h"

namespace sx {

struct RasterBox {
  int x0, y0, z0, lx, ly, lz;
  double c[3];
  double Hi[9];
};

__global__ void raster_kernel(const RasterBox b, int nx, int ny, unsigned long long* idx,
                              unsigned char* flag, long long total) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / b.lx;
    const int x = b.x0 + (int)(i - t * b.lx);
    const int zz = (int)(t / b.ly);
    const int y = b.y0 + (int)(t - (long long)zz * b.ly);
    const int z = b.z0 + zz;
    // window.hpp:95-103 operation order
    const double dz = __dsub_rn((double)z, b.c[2]);
    const double dy = __dsub_rn((double)y, b.c[1]);
    const double c0 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(b.Hi[4], dy), dy),
                                          __dmul_rn(__dmul_rn(__dmul_rn(2.0, b.Hi[5]), dy), dz)),
                                __dmul_rn(__dmul_rn(b.Hi[8], dz), dz));
    const double c1 = __dmul_rn(2.0, __dadd_rn(__dmul_rn(b.Hi[1], dy), __dmul_rn(b.Hi[2], dz)));
    const double dx = __dsub_rn((double)x, b.c[0]);
    const double d = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(b.Hi[0], dx), dx), __dmul_rn(c1, dx)), c0);
    idx[i] = (unsigned long long)x + (unsigned long long)nx * ((unsigned long long)y + (unsigned long long)ny * z);
    flag[i] = d <= 1.0;
  }
}

}  // namespace sx

extern "C" int salvox_rasterize_window(salvox_ctx* ctx, int32_t nx, int32_t ny, int32_t nz,
                                       const double* center, const double* H, uint64_t* out,
                                       int64_t cap, int64_t* n_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (!center || !H) fail(SALVOX_EINVAL, "null window");
    SX_CUDA(cudaSetDevice(ctx->device));
    RasterBox b{};
    sx_inverse3(H, b.Hi);  // host: the same Eigen restatement the kernels use
    for (int i = 0; i < 3; ++i) b.c[i] = center[i];
    int lo[3], hi[3];
    const int dims[3] = {nx, ny, nz};
    for (int i = 0; i < 3; ++i) {  // window.hpp:84-92
      const double e = std::sqrt(std::max(H[4 * i], 0.0));
      lo[i] = std::max(0, (int)std::ceil(center[i] - e));
      hi[i] = std::min(dims[i] - 1, (int)std::floor(center[i] + e));
    }
    int64_t n = 0;
    if (lo[0] <= hi[0] && lo[1] <= hi[1] && lo[2] <= hi[2]) {
      b.x0 = lo[0], b.y0 = lo[1], b.z0 = lo[2];
      b.lx = hi[0] - lo[0] + 1, b.ly = hi[1] - lo[1] + 1, b.lz = hi[2] - lo[2] + 1;
      const long long total = (long long)b.lx * b.ly * b.lz;
      char* base = static_cast<char*>(ctx->d_sel_c.ensure((size_t)total * 17 + 1024));
      unsigned long long* idx = reinterpret_cast<unsigned long long*>(base);
      unsigned long long* sel = idx + total;
      unsigned char* flag = reinterpret_cast<unsigned char*>(sel + total);
      int* d_cnt = static_cast<int*>(ctx->d_sel_d.ensure(64));
      raster_kernel<<<(int)std::min<long long>((total + 255) / 256, ctx->sm_count * 16LL), 256, 0,
                      ctx->stream>>>(b, nx, ny, idx, flag, total);
      SX_LAUNCH_CHECK(ctx);
      size_t tmp = 0;
      SX_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, idx, flag, sel, d_cnt, (int)total, ctx->stream));
      void* d_tmp = ctx->d_cub.ensure(tmp);
      SX_CUDA(cub::DeviceSelect::Flagged(d_tmp, tmp, idx, flag, sel, d_cnt, (int)total, ctx->stream));
      int cnt = 0;
      SX_CUDA(cudaMemcpyAsync(&cnt, d_cnt, 4, cudaMemcpyDeviceToHost, ctx->stream));
      SX_CUDA(cudaStreamSynchronize(ctx->stream));
      n = cnt;
      if (out && cap > 0 && n > 0)
        SX_CUDA(cudaMemcpyAsync(out, sel, (size_t)std::min(n, cap) * 8, cudaMemcpyDeviceToHost,
                                ctx->stream));
      SX_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (n_out) *n_out = n;
  });
}

// ------------------------------------------------------------------ Hu moments
// hu_moments (reference src/hu.cpp:8-58) and hu_template_distance
// (src/pipeline.cpp:218-256), one warp per image: the raw and central moment
// sums run as ordered fp64 chains (lane k owns sum k, all pixels in y->x order,
// like the reference's double loop), the invariants on lane 0 in the
// reference's operation order. pow(m00, 2) = m00*m00 (exactly rounded either
// way); pow(m00, 2.5) uses the shared sx_pow (a few ulp from glibc).
#include "../../include/salvox/sx_log.h"

namespace sx {

struct HuJob {
  const float* img;  // first pixel of the crop
  int w, h;          // crop size
  int pitch;         // row pitch (floats)
};

__device__ __forceinline__ double hu_px(const HuJob& j, int i) {
  const int y = i / j.w, x = i - y * j.w;
  return (double)__ldg(j.img + (size_t)y * j.pitch + x);
}

// out[8 * k + 0..6] = Hu vector, out[8 * k + 7] = 1 if the mass is positive
__global__ void hu_kernel(const HuJob* jobs, int n, double* out) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= n) return;
  const HuJob j = jobs[k];
  const int np = j.w * j.h;
  double acc = 0.0;  // lane 0: m00, 1: m10, 2: m01
  for (int i = 0; i < np; ++i) {
    const double f = hu_px(j, i);
    const int y = i / j.w, x = i - y * j.w;
    if (lane == 0) acc = __dadd_rn(acc, f);
    else if (lane == 1) acc = __dadd_rn(acc, __dmul_rn(f, (double)x));
    else if (lane == 2) acc = __dadd_rn(acc, __dmul_rn(f, (double)y));
  }
  const double m00 = __shfl_sync(0xffffffffu, acc, 0);
  const double m10 = __shfl_sync(0xffffffffu, acc, 1);
  const double m01 = __shfl_sync(0xffffffffu, acc, 2);
  if (!(m00 > 0.0)) {  // hu_moments: zero total mass (hu.cpp:21)
    if (lane == 0) out[8 * k + 7] = 0.0;
    return;
  }
  const double cx = __ddiv_rn(m10, m00), cy = __ddiv_rn(m01, m00);
  // lane: 0 mu20, 1 mu02, 2 mu11, 3 mu30, 4 mu03, 5 mu21, 6 mu12 (hu.cpp:25-38)
  acc = 0.0;
  for (int i = 0; i < np; ++i) {
    const double f = hu_px(j, i);
    const int y = i / j.w, x = i - y * j.w;
    const double dy = __dsub_rn((double)y, cy), dx = __dsub_rn((double)x, cx);
    double t = 0.0;
    switch (lane) {
      case 0: t = __dmul_rn(__dmul_rn(f, dx), dx); break;
      case 1: t = __dmul_rn(__dmul_rn(f, dy), dy); break;
      case 2: t = __dmul_rn(__dmul_rn(f, dx), dy); break;
      case 3: t = __dmul_rn(__dmul_rn(__dmul_rn(f, dx), dx), dx); break;
      case 4: t = __dmul_rn(__dmul_rn(__dmul_rn(f, dy), dy), dy); break;
      case 5: t = __dmul_rn(__dmul_rn(__dmul_rn(f, dx), dx), dy); break;
      case 6: t = __dmul_rn(__dmul_rn(__dmul_rn(f, dx), dy), dy); break;
      default: break;
    }
    acc = __dadd_rn(acc, t);
  }
  double mu[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) mu[q] = __shfl_sync(0xffffffffu, acc, q);
  if (lane != 0) return;
  const double s2 = __dmul_rn(m00, m00);  // std::pow(m00, 2.0)
  const double s3 = sx_pow(m00, 2.5);     // std::pow(m00, 2.5)
  const double n20 = __ddiv_rn(mu[0], s2), n02 = __ddiv_rn(mu[1], s2), n11 = __ddiv_rn(mu[2], s2);
  const double n30 = __ddiv_rn(mu[3], s3), n03 = __ddiv_rn(mu[4], s3), n21 = __ddiv_rn(mu[5], s3),
               n12 = __ddiv_rn(mu[6], s3);
#define M(a, b) __dmul_rn((a), (b))
#define A(a, b) __dadd_rn((a), (b))
#define S(a, b) __dsub_rn((a), (b))
  const double a1 = S(n30, M(3.0, n12)), a2 = S(M(3.0, n21), n03);
  const double b1 = A(n30, n12), b2 = A(n21, n03);
  double h[7];
  h[0] = A(n20, n02);
  h[1] = A(M(S(n20, n02), S(n20, n02)), M(M(4.0, n11), n11));
  h[2] = A(M(a1, a1), M(a2, a2));
  h[3] = A(M(b1, b1), M(b2, b2));
  h[4] = A(M(M(a1, b1), S(M(b1, b1), M(M(3.0, b2), b2))),
           M(M(a2, b2), S(M(M(3.0, b1), b1), M(b2, b2))));
  h[5] = A(M(S(n20, n02), S(M(b1, b1), M(b2, b2))), M(M(M(4.0, n11), b1), b2));
  h[6] = S(M(M(a2, b1), S(M(b1, b1), M(M(3.0, b2), b2))),
           M(M(a1, b2), S(M(M(3.0, b1), b1), M(b2, b2))));
#undef M
#undef A
#undef S
  for (int q = 0; q < 7; ++q) out[8 * k + q] = h[q];
  out[8 * k + 7] = 1.0;
}

void run_hu(salvox_ctx* ctx, const std::vector<HuJob>& jobs, std::vector<double>& res) {
  res.assign(jobs.size() * 8, 0.0);
  if (jobs.empty()) return;
  char* base = static_cast<char*>(ctx->d_sel_c.ensure(jobs.size() * (sizeof(HuJob) + 64) + 256));
  HuJob* d_jobs = reinterpret_cast<HuJob*>(base);
  double* d_out = reinterpret_cast<double*>(base + ((jobs.size() * sizeof(HuJob) + 255) / 256) * 256);
  SX_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(HuJob), cudaMemcpyHostToDevice,
                          ctx->stream));
  hu_kernel<<<(int)(jobs.size() + 3) / 4, 128, 0, ctx->stream>>>(d_jobs, (int)jobs.size(), d_out);
  SX_LAUNCH_CHECK(ctx);
  SX_CUDA(cudaMemcpyAsync(res.data(), d_out, res.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace sx

extern "C" int salvox_hu_moments(salvox_ctx* ctx, const float* image, int32_t nx, int32_t ny,
                                 double* out7) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!image || !out7 || nx < 1 || ny < 1) fail(SALVOX_EINVAL, "hu_moments: expected a 2D slice");
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t n = (size_t)nx * ny;
    float* d_img = static_cast<float*>(ctx->d_seek_vol.ensure(n * 4));
    SX_CUDA(cudaMemcpyAsync(d_img, image, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    std::vector<double> res;
    run_hu(ctx, {HuJob{d_img, nx, ny, nx}}, res);
    if (res[7] == 0.0) fail(SALVOX_EINVAL, "hu_moments: zero total mass");
    for (int q = 0; q < 7; ++q) out7[q] = res[q];
  });
}

extern "C" int salvox_hu_template_distance(salvox_ctx* ctx, const float* volume, int32_t nx,
                                           int32_t ny, int32_t nz, const salvox_detection* dets,
                                           int64_t n, const float* tmpl, int32_t tnx, int32_t tny,
                                           int32_t slices, double* out_dist) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!volume || !tmpl || nx < 1 || ny < 1 || nz < 1 || tnx < 1 || tny < 1)
      fail(SALVOX_EINVAL, "hu_template_distance: bad arguments");
    if (n < 0 || (n > 0 && (!dets || !out_dist))) fail(SALVOX_EINVAL, "bad detection arrays");
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nv = (size_t)nx * ny * nz, nt = (size_t)tnx * tny;
    float* d_vol = static_cast<float*>(ctx->d_seek_vol.ensure((nv + nt) * 4));
    float* d_tmpl = d_vol + nv;
    SX_CUDA(cudaMemcpyAsync(d_vol, volume, nv * 4, cudaMemcpyHostToDevice, ctx->stream));
    SX_CUDA(cudaMemcpyAsync(d_tmpl, tmpl, nt * 4, cudaMemcpyHostToDevice, ctx->stream));
    // job 0: the template; then every (detection, slice) crop (pipeline.cpp:218-233)
    std::vector<HuJob> jobs{HuJob{d_tmpl, tnx, tny, tnx}};
    std::vector<std::pair<int64_t, int>> owner;
    const int half = slices / 2;
    for (int64_t i = 0; i < n; ++i) {
      const salvox_detection& d = dets[i];
      const double ex = std::sqrt(std::max(d.H[0], 1.0)), ey = std::sqrt(std::max(d.H[4], 1.0));
      const int x0 = std::max(0, (int)std::floor(d.center[0] - ex));
      const int x1 = std::min(nx - 1, (int)std::ceil(d.center[0] + ex));
      const int y0 = std::max(0, (int)std::floor(d.center[1] - ey));
      const int y1 = std::min(ny - 1, (int)std::ceil(d.center[1] + ey));
      const int zc = (int)std::lround(d.center[2]);
      for (int dz = -half; dz <= half; ++dz) {
        const int z = zc + dz;
        if (z < 0 || z >= nz) continue;  // thinner than requested: use what exists
        jobs.push_back(HuJob{d_vol + ((size_t)z * ny + y0) * nx + x0, x1 - x0 + 1, y1 - y0 + 1, nx});
        owner.emplace_back(i, dz);
      }
    }
    std::vector<double> res;
    run_hu(ctx, jobs, res);
    if (res[7] == 0.0) fail(SALVOX_EINVAL, "hu_moments: zero total mass");  // the template
    std::vector<double> sum((size_t)n, 0.0);
    std::vector<int> used((size_t)n, 0);
    for (size_t j = 1; j < jobs.size(); ++j) {  // dz ascending per detection (the reference's loop)
      if (res[8 * j + 7] == 0.0) continue;       // zero-mass crop contributes nothing
      double d2 = 0.0;                           // hu_distance (hu.cpp:60-64)
      for (int q = 0; q < 7; ++q) {
        const double e = res[8 * j + q] - res[q];
        d2 += e * e;
      }
      sum[(size_t)owner[j - 1].first] += std::sqrt(d2);
      used[(size_t)owner[j - 1].first]++;
    }
    for (int64_t i = 0; i < n; ++i)
      out_dist[i] = used[(size_t)i] == 0 ? std::numeric_limits<double>::infinity()
                                         : sum[(size_t)i] / used[(size_t)i];
  });
}

// ------------------------------------------------------------------ phantoms
// make_phantom on the device (reference src/phantom.cpp:
// 237-294, include/salvox/rng.hpp). splitmix64 is counter-based -- draw j of a
// generator seeded s is mix(s + (j + 1) * golden) -- so every voxel's draws
// are computable in parallel once the draws before it are counted:
//  * gaussian background: voxel i takes Box-Muller pair i / 2 (draws 2k, 2k+1),
//    the cosine for even i and the sine for odd i (the reference's spare);
//  * region r (bounding box in z -> y -> x order, like the reference's loops):
//    pass 1 counts the inside voxels of every box row (one warp per row), an
//    exclusive scan gives each row's first rank, pass 2 writes each inside
//    voxel with draw (background draws + earlier uniform regions + its rank).
// Every fp64 step uses the reference's operation order without contraction;
// integer fills and constant values are bit-identical to the host generator;
// the gaussian background uses libdevice log/sin/cos (<= 2 ulp in fp64), so a
// float can differ from the glibc one in the last place, rarely.
namespace sx {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t sm_draw(uint64_t seed, unsigned long long j) {
  uint64_t z = seed + (uint64_t)(j + 1ull) * kGolden;  // rng.hpp:16
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double sm_unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

struct PhDev {
  int shape;
  double c[3], half[3], Hi[9];
  int lo[3], hi[3];
};

__device__ __forceinline__ bool ph_inside(const PhDev& g, int x, int y, int z) {
  const double d0 = (double)x - g.c[0], d1 = (double)y - g.c[1], d2 = (double)z - g.c[2];
  if (g.shape == 0) return fabs(d0) <= g.half[0] && fabs(d1) <= g.half[1] && fabs(d2) <= g.half[2];
  double hd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    hd[i] = __dadd_rn(__dmul_rn(g.Hi[i * 3], d0),  // Eigen's lazy-product redux t0 + (t1 + t2)
                      __dadd_rn(__dmul_rn(g.Hi[i * 3 + 1], d1), __dmul_rn(g.Hi[i * 3 + 2], d2)));
  return __dadd_rn(__dadd_rn(__dmul_rn(d0, hd[0]), __dmul_rn(d1, hd[1])), __dmul_rn(d2, hd[2])) <= 1.0;
}

__global__ void ph_bg_kernel(float* __restrict__ v, long long n, int type, float cval, double mean,
                             double sigma, uint64_t seed, unsigned* err) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (type == 0) {
    for (long long i = t0; i < n; i += stride) v[i] = cval;
    return;
  }
  for (long long k = t0; 2 * k < n; k += stride) {
    const double u1 = sm_unit(sm_draw(seed, 2ull * k)), u2 = sm_unit(sm_draw(seed, 2ull * k + 1ull));
    if (!(u1 > 0.0)) {  // the reference redraws u1 (rng.hpp:39): a 2^-53 event per pair
      atomicOr(err, 1u);
      continue;
    }
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    const double theta = __dmul_rn(6.283185307179586476925286766559, u2);
    v[2 * k] = (float)__dadd_rn(mean, __dmul_rn(sigma, __dmul_rn(r, cos(theta))));
    if (2 * k + 1 < n) v[2 * k + 1] = (float)__dadd_rn(mean, __dmul_rn(sigma, __dmul_rn(r, sin(theta))));
  }
}

// pass 1: inside voxels per bounding-box row (one warp per row)
__global__ void ph_count_kernel(PhDev g, long long rows, unsigned long long* __restrict__ row_cnt) {
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= rows) return;
  const int ny_r = g.hi[1] - g.lo[1] + 1;
  const int y = g.lo[1] + (int)(w % ny_r), z = g.lo[2] + (int)(w / ny_r);
  unsigned long long cnt = 0;
  for (int x0 = g.lo[0]; x0 <= g.hi[0]; x0 += 32) {
    const int x = x0 + lane;
    const bool in = x <= g.hi[0] && ph_inside(g, x, y, z);
    cnt += (unsigned)__popc(__ballot_sync(0xffffffffu, in));
  }
  if (lane == 0) row_cnt[w] = cnt;
}

__global__ void ph_total_kernel(const unsigned long long* base, const unsigned long long* cnt,
                                long long rows, unsigned long long* total) {
  *total = base[rows - 1] + cnt[rows - 1];
}

// pass 2: write every inside voxel; per-region centroid sums (exact integers)
__global__ void ph_write_kernel(PhDev g, long long rows, const unsigned long long* __restrict__ row_base,
                                float* __restrict__ v, int nx, int ny, unsigned* __restrict__ occ,
                                int uniform, uint64_t levels, float cval, uint64_t seed,
                                unsigned long long draw0, unsigned long long* sums, unsigned* flag) {
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= rows) return;
  const int ny_r = g.hi[1] - g.lo[1] + 1;
  const int y = g.lo[1] + (int)(w % ny_r), z = g.lo[2] + (int)(w / ny_r);
  unsigned long long rank = row_base[w];
  unsigned long long sx = 0, sy = 0, sz = 0;
  bool overlap = false;
  for (int x0 = g.lo[0]; x0 <= g.hi[0]; x0 += 32) {
    const int x = x0 + lane;
    const bool in = x <= g.hi[0] && ph_inside(g, x, y, z);
    const unsigned m = __ballot_sync(0xffffffffu, in);
    if (in) {
      const unsigned long long idx = (unsigned long long)x + (unsigned long long)nx * ((unsigned long long)y + (unsigned long long)ny * z);
      const unsigned bit = 1u << (idx & 31);
      if (atomicOr(occ + (idx >> 5), bit) & bit) overlap = true;  // "regions overlap" (phantom.cpp:278)
      const unsigned long long r = rank + (unsigned)__popc(m & ((1u << lane) - 1u));
      v[idx] = uniform ? (float)(sm_draw(seed, draw0 + r) % levels) : cval;
      sx += (unsigned)x;
      sy += (unsigned)y;
      sz += (unsigned)z;
    }
    rank += (unsigned)__popc(m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
  }
  if (__any_sync(0xffffffffu, overlap) && lane == 0) atomicOr(flag, 1u);
  if (lane == 0 && (sx | sy | sz)) {
    atomicAdd(sums + 0, sx);
    atomicAdd(sums + 1, sy);
    atomicAdd(sums + 2, sz);
  }
}

}  // namespace sx

extern "C" int salvox_make_phantom_device(salvox_ctx* ctx, int32_t nx, int32_t ny, int32_t nz,
                                          int32_t bg_type, double bg_value, double bg_mean,
                                          double bg_sigma, int32_t n_regions, const int32_t* shape,
                                          const double* center, const double* half_extents,
                                          const double* radius, const double* axes,
                                          const int32_t* fill_type, const int32_t* fill_levels,
                                          const double* fill_value, uint64_t rng_seed, float* d_volume,
                                          double* out_centroids) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
    if (!d_volume) fail(SALVOX_EINVAL, "make_phantom (device): null output");
    if (bg_type == 1 && !(bg_sigma > 0.0)) fail(SALVOX_ERUNTIME, "background.sigma must be > 0");
    const long long n = (long long)nx * ny * nz;
    const int dims[3] = {nx, ny, nz};
    // geometry on the host; an out-of-volume region is reported in region order
    // (after the overlap / empty checks of the regions before it), like the
    // reference's single pass
    std::vector<PhDev> geo(n_regions);
    std::vector<std::string> outside(n_regions);
    std::vector<long long> rows(n_regions, 0);
    for (int r = 0; r < n_regions; ++r) {
      try {
        const PhRegion g = phantom_region(r, dims, shape, center, half_extents, radius, axes);
        PhDev& d = geo[r];
        d.shape = g.shape;
        for (int i = 0; i < 3; ++i) d.c[i] = g.c[i], d.half[i] = g.half[i], d.lo[i] = g.lo[i], d.hi[i] = g.hi[i];
        for (int i = 0; i < 9; ++i) d.Hi[i] = g.Hi.m[i];
        rows[r] = (long long)(g.hi[1] - g.lo[1] + 1) * (g.hi[2] - g.lo[2] + 1);
      } catch (const Error& e) {
        outside[r] = e.what();
      }
      if (fill_type[r] == 0 && fill_levels[r] < 1) fail(SALVOX_ERUNTIME, "fill.levels must be >= 1");
    }
    long long total_rows = 0;
    for (long long x : rows) total_rows += x;
    // scratch: occupancy bits | row counts | row bases | per-region {sums[3], total, flag}
    const size_t occ_words = (size_t)(n + 31) / 32;
    const size_t bytes = occ_words * 4 + 16 + (size_t)total_rows * 16 + (size_t)std::max(n_regions, 1) * 48 + 64;
    char* base = static_cast<char*>(ctx->d_sel_c.ensure(bytes));
    unsigned* occ = reinterpret_cast<unsigned*>(base);
    unsigned long long* row_cnt = reinterpret_cast<unsigned long long*>(base + ((occ_words * 4 + 15) & ~(size_t)15));
    unsigned long long* row_base = row_cnt + total_rows;
    unsigned long long* per = row_base + total_rows;  // 6 words per region: sx sy sz total flag pad
    unsigned* err = reinterpret_cast<unsigned*>(per + 6 * std::max(n_regions, 1));
    SX_CUDA(cudaMemsetAsync(occ, 0, occ_words * 4, ctx->stream));
    SX_CUDA(cudaMemsetAsync(per, 0, (size_t)std::max(n_regions, 1) * 48 + 8, ctx->stream));
    {
      const int block = 256;
      const long long work = bg_type == 0 ? n : (n + 1) / 2;
      const int grid = (int)std::max<long long>(1, std::min<long long>((work + block - 1) / block, ctx->sm_count * 8LL));
      ph_bg_kernel<<<grid, block, 0, ctx->stream>>>(d_volume, n, bg_type, (float)bg_value, bg_mean, bg_sigma,
                                                    rng_seed, err);
      SX_LAUNCH_CHECK(ctx);
    }
    // pass 1 + scan for every region
    long long off = 0;
    for (int r = 0; r < n_regions; ++r) {
      if (!outside[r].empty() || rows[r] == 0) continue;
      unsigned long long* cnt = row_cnt + off;
      unsigned long long* bas = row_base + off;
      const int grid = (int)((rows[r] * 32 + 255) / 256);
      ph_count_kernel<<<grid, 256, 0, ctx->stream>>>(geo[r], rows[r], cnt);
      SX_LAUNCH_CHECK(ctx);
      size_t tmp = 0;
      SX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, bas, (int)rows[r], ctx->stream));
      void* d_tmp = ctx->d_cub.ensure(tmp);
      SX_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, cnt, bas, (int)rows[r], ctx->stream));
      ph_total_kernel<<<1, 1, 0, ctx->stream>>>(bas, cnt, rows[r], per + 6 * r + 3);
      SX_LAUNCH_CHECK(ctx);
      off += rows[r];
    }
    std::vector<unsigned long long> h_per((size_t)std::max(n_regions, 1) * 6);
    SX_CUDA(cudaMemcpyAsync(h_per.data(), per, h_per.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    // pass 2: draw bases in region order
    unsigned long long draw = bg_type == 1 ? 2ull * (unsigned long long)((n + 1) / 2) : 0ull;
    off = 0;
    for (int r = 0; r < n_regions; ++r) {
      if (!outside[r].empty()) break;  // the reference stops at this region
      if (rows[r] == 0) continue;
      const int grid = (int)((rows[r] * 32 + 255) / 256);
      const bool uni = fill_type[r] == 0;
      ph_write_kernel<<<grid, 256, 0, ctx->stream>>>(
          geo[r], rows[r], row_base + off, d_volume, nx, ny, occ, uni ? 1 : 0,
          uni ? (uint64_t)fill_levels[r] : 1ull, (float)fill_value[r], rng_seed, draw, per + 6 * r,
          reinterpret_cast<unsigned*>(per + 6 * r + 4));
      SX_LAUNCH_CHECK(ctx);
      if (uni) draw += h_per[6 * r + 3];
      off += rows[r];
    }
    unsigned h_err = 0;
    SX_CUDA(cudaMemcpyAsync(h_per.data(), per, h_per.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < n_regions; ++r) {  // the reference's error order
      if (!outside[r].empty()) fail(SALVOX_ERUNTIME, outside[r]);
      if (h_per[6 * r + 4]) fail(SALVOX_ERUNTIME, "make_phantom: regions overlap");
      if (h_per[6 * r + 3] == 0) fail(SALVOX_ERUNTIME, "make_phantom: region rasterizes to no voxel");
    }
    if (h_err & 1u)
      fail(SALVOX_EUNSUPPORTED,
           "make_phantom (device): a Box-Muller pair drew u1 == 0 (the reference redraws; 2^-53 event)");
    if (out_centroids)
      for (int r = 0; r < n_regions; ++r)
        for (int i = 0; i < 3; ++i) out_centroids[3 * r + i] = (double)h_per[6 * r + i] / (double)h_per[6 * r + 3];
  });
}
