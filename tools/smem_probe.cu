// Shared-memory histogram-update probe (B200, sm_100a).
//
// Measures the lane-update rate of the inner loop shape used by the exhaustive
// Kadir-Brady kernel: a u8 bin fetched from a shared-memory tile at a
// warp-uniform offset (constant-memory table), then one weighted increment of
// a lane-private shared-memory counter laid out hist[bin][thread].
//   mode 0: LDS.U8 + LDS + IADD + STS   (plain read-modify-write)
//   mode 1: LDS.U8 + ATOMS.ADD          (shared atomic, result unused)
//   mode 2: LDS.U8 only                 (bin fetch ceiling)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_probe smem_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTable = 2048;
__constant__ int32_t c_off[kTable];

template <int MODE, int NT, int NB>
__global__ void __launch_bounds__(NT, 1) probe(int iters, uint32_t* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int kTile = 65536;
  uint8_t* tile = sm;
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + kTile);
  const int tid = threadIdx.x;
  for (int i = tid; i < kTile; i += NT) {
    uint32_t h = uint32_t(i) * 2654435761u + blockIdx.x;
    h ^= h >> 15;
    tile[i] = uint8_t(h % NB);
  }
  for (int i = tid; i < NB * NT; i += NT) hist[i] = 0;
  __syncthreads();
  const int base = 32128 + (tid & 31) + 40 * ((tid >> 5) & 31);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int k0 = 0; k0 < kTable; k0 += 8) {
      uint32_t b[8], n[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int32_t e = c_off[k0 + j];
        n[j] = uint32_t(e) & 511u;
        b[j] = tile[base + (e >> 9)];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 0) {
          hist[b[j] * NT + tid] += n[j];
        } else if (MODE == 1) {
          atomicAdd(&hist[b[j] * NT + tid], n[j]);
        } else {
          acc += b[j] * n[j];
        }
      }
    }
  }
  __syncthreads();
  uint32_t s = acc;
  for (int b = 0; b < NB; ++b) s += hist[b * NT + tid];
  out[blockIdx.x * NT + tid] = s;
}

template <int MODE, int NT, int NB>
double run(int sms, int iters) {
  const size_t smem = 65536 + size_t(NB) * NT * 4;
  cudaFuncSetAttribute(probe<MODE, NT, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  uint32_t* out;
  cudaMalloc(&out, size_t(sms) * 4 * NT * 4);
  const int grid = sms * 4;
  probe<MODE, NT, NB><<<grid, NT, smem>>>(1, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<MODE, NT, NB><<<grid, NT, smem>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t err = cudaDeviceSynchronize();
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "error %s\n", cudaGetErrorString(err));
    exit(1);
  }
  cudaFree(out);
  const double updates = double(grid) * NT * iters * kTable;
  return updates / (ms * 1e-3);
}

int main() {
  int32_t h[kTable];
  uint32_t s = 12345;
  for (int k = 0; k < kTable; ++k) {
    s = s * 1664525u + 1013904223u;
    const int dz = int((s >> 8) % 33) - 16, dy = int((s >> 16) % 33) - 16, dx = int((s >> 24) % 33) - 16;
    const int off = dz * 40 * 48 + dy * 48 + dx;
    const int n = dx * dx + dy * dy + dz * dz;
    h[k] = (off << 9) | (n & 511);
  }
  cudaMemcpyToSymbol(c_off, h, sizeof(h));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 200;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  printf(", \"rmw_1024x33\": %.4e", run<0, 1024, 33>(sms, iters));
  printf(", \"atoms_1024x33\": %.4e", run<1, 1024, 33>(sms, iters));
  printf(", \"lds_only_1024\": %.4e", run<2, 1024, 33>(sms, iters));
  printf(", \"rmw_512x33\": %.4e", run<0, 512, 33>(sms, iters));
  printf(", \"atoms_512x33\": %.4e", run<1, 512, 33>(sms, iters));
  printf(", \"rmw_256x65\": %.4e", run<0, 256, 65>(sms, iters));
  printf(", \"atoms_256x65\": %.4e", run<1, 256, 65>(sms, iters));
  printf("}\n");
  fflush(stdout);
  return 0;
}
