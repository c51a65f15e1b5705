// TMA 3D u8 tile-load probe (debug aid): loads a box with negative/OOB coordinates
// and checks it against a host reference. Variants: 0 = shared::cluster dst +
// fence.mbarrier_init, 1 = no fence, 2 = shared::cta barrier wait only (no TMA).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int V>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, int x0, int y0, int z0,
                      uint32_t bytes, uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* tile = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ((bytes + 15u) & ~15u));
  if (threadIdx.x == 0) {
    printf("V%d smem tile=%u bar=%u desc=%p\n", V, su32(tile), su32(bar), &tmap);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    if (V == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (V == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 2) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(tile)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(z0), "r"(su32(bar))
          : "memory");
    }
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
        : "=r"(done)
        : "r"(su32(bar))
        : "memory");
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = V == 2 ? 7 : tile[i];
}

int main(int argc, char** argv) {
  const int nx = argc > 1 ? atoi(argv[1]) : 64, ny = argc > 2 ? atoi(argv[2]) : 64,
            nz = argc > 3 ? atoi(argv[3]) : 1;
  const int BX = argc > 4 ? atoi(argv[4]) : 64, BY = argc > 5 ? atoi(argv[5]) : 38,
            BZ = argc > 6 ? atoi(argv[6]) : 1;
  const int pitch = (nx + 15) / 16 * 16;
  std::vector<uint8_t> h((size_t)pitch * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = uint8_t(1 + i % 200);
  uint8_t *d, *dout;
  cudaMalloc(&d, h.size());
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  const uint32_t bytes = BX * BY * BZ;
  cudaMalloc(&dout, bytes);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap map;
  cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  cuuint64_t gstr[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * ny};
  cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)BY, (cuuint32_t)BZ};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, gdim, gstr, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  const int x0 = argc > 7 ? atoi(argv[7]) : -11, y0 = argc > 8 ? atoi(argv[8]) : -11,
            z0 = argc > 9 ? atoi(argv[9]) : 0;
  for (int v = 2; v >= 0; --v) {
    void (*k)(const CUtensorMap, int, int, int, uint32_t, uint8_t*) =
        v == 0 ? probe<0> : (v == 1 ? probe<1> : probe<2>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 64);
    k<<<1, 128, bytes + 64>>>(map, x0, y0, z0, bytes, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", v, cudaGetErrorString(e));
    fflush(stdout);
    if (e != cudaSuccess) return 1;
    std::vector<uint8_t> o(bytes);
    cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);
    if (v < 2) {
      int bad = 0;
      for (int bz = 0; bz < BZ; ++bz)
        for (int by = 0; by < BY; ++by)
          for (int bx = 0; bx < BX; ++bx) {
            const int gx = x0 + bx, gy = y0 + by, gz = z0 + bz;
            const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny && gz >= 0 && gz < nz;
            const uint8_t want = in ? h[(size_t)gz * pitch * ny + (size_t)gy * pitch + gx] : 0;
            if (o[(size_t)bz * BX * BY + by * BX + bx] != want) ++bad;
          }
      printf("variant %d mismatches: %d\n", v, bad);
    }
  }
  return 0;
}
