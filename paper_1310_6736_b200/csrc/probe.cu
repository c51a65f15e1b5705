// probe.cu -- live roofline denominator for the exhaustive kernel.
//
// The exhaustive pass is bound by shared-memory traffic, not HBM or tensor
// cores, and MEASURED_PEAKS.json has no shared-memory figure,
// so bench.py measures it here on the same GPU in the same run. The probe runs
// kb_kernel's inner-loop instruction mix with nothing else: a u8 bin fetched
// from a shared-memory tile at a warp-uniform constant-table offset (+-o pair)
// and one ATOMS.ADD into a lane-private column hist[bin][thread]
// (conflict-free), one 512-thread CTA per SM, 2x33-bin columns like kb_kernel.
#include "../../include/salvox_bench.h"
#include "common.cuh"

#include <algorithm>

namespace sx {

constexpr int kProbeTable = 2048;
__constant__ int4 c_probe[kProbeTable / 4];

// MODE 0: LDS.U8 + ATOMS (kb_kernel's pair), 1: LDS.U8 only, 2: ATOMS only
// (bins from a register hash: the one-atomic-per-update floor of any design).
template <int NT, int NB, int MODE>
__global__ void __launch_bounds__(NT, 1) smem_probe_kernel(int iters, uint32_t* out) {
  static_assert(NT == 512 || NT == 1024, "probe thread mapping");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  uint8_t* tile = smem + NB * NT * 4;
  constexpr int kTile = 76800;  // 48 x 40 x 40, kb_kernel's 3D tile at R = 16
  const int tid = threadIdx.x;
  for (int i = tid; i < kTile; i += NT) {
    uint32_t h = uint32_t(i) * 2654435761u + blockIdx.x;
    h ^= h >> 15;
    tile[i] = uint8_t(h % NB);
  }
  for (int i = tid; i < NB * NT; i += NT) hist[i] = 0;
  __syncthreads();
  // 512 threads: 8x8x8 voxels; 1024 threads: 16x8x8 (kb_tmem_kernel's tile)
  const int lx = NT == 1024 ? (tid & 15) : (tid & 7);
  const int ly = NT == 1024 ? ((tid >> 4) & 7) : ((tid >> 3) & 7);
  const int lz = NT == 1024 ? (tid >> 7) : (tid >> 6);
  const uint8_t* tb = tile + (lz + 16) * 1920 + (ly + 16) * 48 + (lx + 16);
  uint32_t* hc = hist + tid;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int e4 = 0; e4 < kProbeTable / 4; ++e4) {
      const int4 w = c_probe[e4];
      const int o0 = w.x >> 9, o1 = w.y >> 9, o2 = w.z >> 9, o3 = w.w >> 9;
      uint32_t b0, b1, b2, b3, b4, b5, b6, b7;
      if (MODE == 2) {
        const uint32_t h = (uint32_t)(o0 ^ o1 ^ o2 ^ o3) * 2654435761u ^ (uint32_t)tid;
        b0 = h & 31u, b1 = (h >> 5) & 31u, b2 = (h >> 10) & 31u, b3 = (h >> 15) & 31u;
        b4 = (h >> 3) & 31u, b5 = (h >> 8) & 31u, b6 = (h >> 13) & 31u, b7 = (h >> 18) & 31u;
      } else {
        b0 = tb[o0], b1 = tb[-o0], b2 = tb[o1], b3 = tb[-o1];
        b4 = tb[o2], b5 = tb[-o2], b6 = tb[o3], b7 = tb[-o3];
      }
      const uint32_t n0 = (uint32_t)w.x & 511u, n1 = (uint32_t)w.y & 511u;
      const uint32_t n2 = (uint32_t)w.z & 511u, n3 = (uint32_t)w.w & 511u;
      if (MODE != 1) {
        atomicAdd(hc + b0 * NT, n0);
        atomicAdd(hc + b1 * NT, n0);
        atomicAdd(hc + b2 * NT, n1);
        atomicAdd(hc + b3 * NT, n1);
        atomicAdd(hc + b4 * NT, n2);
        atomicAdd(hc + b5 * NT, n2);
        atomicAdd(hc + b6 * NT, n3);
        atomicAdd(hc + b7 * NT, n3);
      } else {
        acc += (b0 + b1) * n0 + (b2 + b3) * n1 + (b4 + b5) * n2 + (b6 + b7) * n3;
      }
    }
  }
  __syncthreads();
  uint32_t s = acc;
  for (int b = 0; b < NB; ++b) s += hist[b * NT + tid];
  out[blockIdx.x * NT + tid] = s;
}

// ATOMS only, 256 threads x 4 histogram columns each (the layout of
// kb_quad_kernel): the highest atomic rate demonstrated on the SM (8 warps,
// 32 independent atomics per thread per step; tools/quad_probe.cu "QA").
__global__ void __launch_bounds__(256, 1) smem_probe_quad_kernel(int iters, uint32_t* out) {
  constexpr int NT = 256, NB = 33;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  const int tid = threadIdx.x;
  for (int i = tid; i < NB * 4 * NT; i += NT) hist[i] = 0;
  __syncthreads();
  uint32_t* hc = hist + tid;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int e4 = 0; e4 < kProbeTable / 4; ++e4) {
      const int4 w = c_probe[e4];
      const int o[4] = {w.x >> 9, w.y >> 9, w.z >> 9, w.w >> 9};
      const uint32_t n[4] = {(uint32_t)w.x & 511u, (uint32_t)w.y & 511u, (uint32_t)w.z & 511u,
                             (uint32_t)w.w & 511u};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t h = (uint32_t)(o[k]) * 2654435761u ^ (uint32_t)tid;
        const uint32_t wp = h & 0x1f1f1f1fu, wm = (h >> 3) & 0x1f1f1f1fu;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          atomicAdd(hc + (((wp >> (8 * v)) & 0xffu) * 4 + v) * NT, n[k]);
          atomicAdd(hc + (((wm >> (8 * v)) & 0xffu) * 4 + v) * NT, n[k]);
        }
      }
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int b = 0; b < NB * 4; ++b) acc += hist[b * NT + tid];
  out[blockIdx.x * NT + tid] = acc;
}

// ATOMS only in kb_quad_kernel's exact walk form: 256 threads x 4 columns,
// 16 panels of 64 columns x 33 bins, the atomic address built by ONE PRMT from
// a word of 4 bins (here from a register sequence instead of the tile), the
// panel in the RED's immediate -- the walk without its bin-word loads.
template <int G, int V>
__device__ __forceinline__ void probe_prmt_vox(uint32_t wp, uint32_t wm, uint32_t c, uint32_t n) {
  constexpr uint32_t sel = 0x7604u | (V << 4), imm = 0x400u + (V * 4 + G) * 33 * 256;
  uint32_t ap, am;
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(ap) : "r"(wp), "r"(c), "n"(sel));
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(am) : "r"(wm), "r"(c), "n"(sel));
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ap), "r"(n), "n"(imm));
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(am), "r"(n), "n"(imm));
}

template <int G>
__device__ __forceinline__ void probe_prmt_entry(uint32_t wp, uint32_t wm, uint32_t c, uint32_t n) {
  probe_prmt_vox<G, 0>(wp, wm, c, n);
  probe_prmt_vox<G, 1>(wp, wm, c, n);
  probe_prmt_vox<G, 2>(wp, wm, c, n);
  probe_prmt_vox<G, 3>(wp, wm, c, n);
}

template <int G>
__device__ __noinline__ void probe_prmt_walk(int iters, uint32_t c, uint32_t seed) {
  uint32_t h = seed;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int e4 = 0; e4 < kProbeTable / 4; ++e4) {
      const int4 w = c_probe[e4];
      const int e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        h = h * 1664525u + 1013904223u;
        probe_prmt_entry<G>(h & 0x1f1f1f1fu, (h >> 3) & 0x1f1f1f1fu, c, (uint32_t)e[k] & 511u);
      }
    }
  }
}

__global__ void __launch_bounds__(256, 1) smem_probe_prmt_kernel(int iters, uint32_t* out) {
  constexpr int NB = 33, NV = 1024;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < NB * NV; i += 256) hist[i] = 0;
  __syncthreads();
  const uint32_t hs0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if ((hs0 & 0xffffu) != 0x400u) __trap();  // the immediates assume it (as kb_quad_kernel)
  const int G = warp & 3, col = lane + 32 * (warp >> 2);
  const uint32_t c = (hs0 & 0xffff0000u) | (4u * (uint32_t)col);
  const uint32_t seed = 2654435761u * (uint32_t)(tid + 1) + blockIdx.x;
  switch (G) {
    case 0: probe_prmt_walk<0>(iters, c, seed); break;
    case 1: probe_prmt_walk<1>(iters, c, seed); break;
    case 2: probe_prmt_walk<2>(iters, c, seed); break;
    default: probe_prmt_walk<3>(iters, c, seed); break;
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = tid; i < NB * NV; i += 256) acc += hist[i];
  out[blockIdx.x * 256 + tid] = acc;
}

}  // namespace sx

using namespace sx;

constexpr int kProbeTrials = 3;
double g_prmt_probe_rate = 0.0;  // last run's PRMT-walk ATOMS rate (updates/s)

extern "C" double salvox_probe_prmt_rate() { return g_prmt_probe_rate; }

extern "C" int salvox_probe_smem_peak(salvox_ctx* ctx, int iters, double* atoms_updates_per_s,
                                      double* lds_fetches_per_s, double* atoms_only_per_s) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    SX_CUDA(cudaSetDevice(ctx->device));
    // the same +-o pair encoding as kb_kernel (48 x 40 pitch, R = 16 ball offsets)
    std::vector<int32_t> tab(kProbeTable);
    uint32_t s = 12345;
    for (int k = 0; k < kProbeTable; ++k) {
      int dx, dy, dz, n;
      do {
        s = s * 1664525u + 1013904223u;
        dx = int((s >> 8) % 33) - 16;
        dy = int((s >> 16) % 33) - 16;
        dz = int((s >> 24) % 33) - 16;
        n = dx * dx + dy * dy + dz * dz;
      } while (n > 256 || n == 0);
      const int off = dz * 1920 + dy * 48 + dx;
      tab[k] = (int32_t)((uint32_t)off << 9 | (uint32_t)n);
    }
    SX_CUDA(cudaMemcpyToSymbolAsync(c_probe, tab.data(), tab.size() * 4, 0, cudaMemcpyHostToDevice,
                                    ctx->stream));
    // both thread counts the kernels use (512: kb_kernel, 1024: kb_tmem_kernel);
    // each rate is the best of the two (the peak an SM sustains)
    constexpr int NB = 33;
    uint32_t* d_out = static_cast<uint32_t*>(ctx->d_dbg.ensure((size_t)ctx->sm_count * 2 * 1024 * 4));
    auto run = [&](auto kern, int NT, double* rate, double per_iter) {
      const size_t smem = (size_t)NB * NT * 4 + 76800;
      SX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int grid = ctx->sm_count * 2;
      kern<<<grid, NT, smem, ctx->stream>>>(1, d_out);  // warm-up
      SX_LAUNCH_CHECK(ctx);
      cudaEvent_t a, b;
      SX_CUDA(cudaEventCreate(&a));
      SX_CUDA(cudaEventCreate(&b));
      for (int trial = 0; trial < kProbeTrials; ++trial) {  // best of: clock ramp / noise
        SX_CUDA(cudaEventRecord(a, ctx->stream));
        kern<<<grid, NT, smem, ctx->stream>>>(iters, d_out);
        SX_LAUNCH_CHECK(ctx);
        SX_CUDA(cudaEventRecord(b, ctx->stream));
        SX_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SX_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double r = (double)grid * NT * iters * per_iter / (ms * 1e-3);
        if (rate && r > *rate) *rate = r;
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    };
    for (double* r : {atoms_updates_per_s, lds_fetches_per_s, atoms_only_per_s})
      if (r) *r = 0.0;
    run(smem_probe_kernel<512, NB, 0>, 512, atoms_updates_per_s, 2.0 * kProbeTable);
    run(smem_probe_kernel<512, NB, 1>, 512, lds_fetches_per_s, 2.0 * kProbeTable);
    run(smem_probe_kernel<512, NB, 2>, 512, atoms_only_per_s, 2.0 * kProbeTable);
    run(smem_probe_kernel<1024, NB, 0>, 1024, atoms_updates_per_s, 2.0 * kProbeTable);
    run(smem_probe_kernel<1024, NB, 1>, 1024, lds_fetches_per_s, 2.0 * kProbeTable);
    run(smem_probe_kernel<1024, NB, 2>, 1024, atoms_only_per_s, 2.0 * kProbeTable);
    {  // 4 columns per thread: per_iter counts the 4 voxels of each thread
      const size_t qsmem = (size_t)NB * 4 * 256 * 4;
      SX_CUDA(cudaFuncSetAttribute(smem_probe_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)qsmem));
      const int grid = ctx->sm_count * 2;
      smem_probe_quad_kernel<<<grid, 256, qsmem, ctx->stream>>>(1, d_out);
      SX_LAUNCH_CHECK(ctx);
      cudaEvent_t a, b;
      SX_CUDA(cudaEventCreate(&a));
      SX_CUDA(cudaEventCreate(&b));
      for (int trial = 0; trial < kProbeTrials; ++trial) {
        SX_CUDA(cudaEventRecord(a, ctx->stream));
        smem_probe_quad_kernel<<<grid, 256, qsmem, ctx->stream>>>(iters, d_out);
        SX_LAUNCH_CHECK(ctx);
        SX_CUDA(cudaEventRecord(b, ctx->stream));
        SX_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SX_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double r = (double)grid * 256 * 4 * iters * 2.0 * kProbeTable / (ms * 1e-3);
        if (atoms_only_per_s && r > *atoms_only_per_s) *atoms_only_per_s = r;
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    {  // kb_quad_kernel's walk without the bin-word loads (PRMT-built addresses)
      const size_t psmem = (size_t)33 * 1024 * 4;
      SX_CUDA(cudaFuncSetAttribute(smem_probe_prmt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)psmem));
      const int grid = ctx->sm_count * 2;
      smem_probe_prmt_kernel<<<grid, 256, psmem, ctx->stream>>>(1, d_out);
      SX_LAUNCH_CHECK(ctx);
      cudaEvent_t a, b;
      SX_CUDA(cudaEventCreate(&a));
      SX_CUDA(cudaEventCreate(&b));
      for (int trial = 0; trial < kProbeTrials; ++trial) {
        SX_CUDA(cudaEventRecord(a, ctx->stream));
        smem_probe_prmt_kernel<<<grid, 256, psmem, ctx->stream>>>(iters, d_out);
        SX_LAUNCH_CHECK(ctx);
        SX_CUDA(cudaEventRecord(b, ctx->stream));
        SX_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SX_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double r = (double)grid * 256 * 4 * iters * 2.0 * kProbeTable / (ms * 1e-3);
        g_prmt_probe_rate = std::max(g_prmt_probe_rate, r);
        if (atoms_only_per_s && r > *atoms_only_per_s) *atoms_only_per_s = r;
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  });
}

extern "C" int salvox_ctx_set_profiling(salvox_ctx* ctx, int on) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->profiling = on != 0;
    ctx->kb_ms_total = 0.0;
    ctx->kb_launches = 0;
    ctx->kb_updates_total = 0.0;
  });
}

extern "C" int salvox_ctx_kernel_time(salvox_ctx* ctx, double* kb_ms_total, int64_t* kb_launches,
                                      double* kb_updates_total) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (kb_ms_total) *kb_ms_total = ctx->kb_ms_total;
    if (kb_launches) *kb_launches = ctx->kb_launches;
    if (kb_updates_total) *kb_updates_total = ctx->kb_updates_total;
  });
}
