// ingest.cu -- on-device MetaImage payload widening.
//
// load_volume (reference src/meta_io.cpp:30-33, :100-105) reads a MET_UCHAR /
// MET_SHORT / MET_USHORT / MET_FLOAT payload and widens it to float on the host.
// Here the payload crosses PCIe at its native width (1-2 bytes per voxel instead
// of 4) and is widened on the device by an HBM-bound kernel; static_cast<float>
// of these integer types is exact, so the result is bit-identical.
#include "../../include/salvox_capi.h"
#include "common.cuh"

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
