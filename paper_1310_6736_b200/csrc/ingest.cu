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
