// quad_probe.cu -- would 4 voxels per thread (8 warps/SM) keep the shared-memory
// atomic pipe fed? Measures histogram updates/s for:
//   A: 1 voxel/thread, 1024 threads, LDS.U8 + ATOMS per update (kb_tmem_kernel's mix)
//   Q: 4 x-adjacent voxels/thread, 256 threads: one (aligned) or two LDS.32 +
//      funnel shift fetch 4 bins per offset, then 4 ATOMS
//   QA: as Q with bins from a register hash (ATOMS only, 8 warps)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/quad_probe tools/quad_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int kTable = 2048;
__constant__ int4 c_tab[kTable / 4];   // (byte offset << 9) | n
__constant__ int2 c_al[kTable];        // per entry: aligned word offsets for +o / -o (low 30 bits) | shift<<30 ... packed below

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(MODE == 0 ? 1024 : 256, 1) probe(int iters, uint32_t* out) {
  // MODE 3: as MODE 1, addresses built with shift + LOP3 (hist at smem 0,
  // column (v, tid) at v*1024 + 4*tid, bin stride 4096 bytes)
  constexpr int NT = MODE == 0 ? 1024 : 256;
  constexpr int NB = 33;
  constexpr int VPT = MODE == 0 ? 1 : 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  uint8_t* tile = smem + NB * NT * VPT * 4;
  constexpr int kTile = 76800;
  const int tid = threadIdx.x;
  for (int i = tid; i < kTile; i += NT) {
    uint32_t h = uint32_t(i) * 2654435761u + blockIdx.x;
    h ^= h >> 15;
    tile[i] = uint8_t(h % NB);
  }
  for (int i = tid; i < NB * NT * VPT; i += NT) hist[i] = 0;
  __syncthreads();
  int lx, ly, lz;
  if (MODE == 0) lx = tid & 15, ly = (tid >> 4) & 7, lz = tid >> 7;
  else lx = 4 * (tid & 3), ly = (tid >> 2) & 7, lz = tid >> 5;
  const int base = (lz + 16) * 1920 + (ly + 16) * 48 + (lx + 16);  // x0 multiple of 4 for MODE>0
  uint32_t* hc = hist + tid;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int e = 0; e < kTable / 4; ++e) {
      const int4 w = c_tab[e];
      const int o[4] = {w.x >> 9, w.y >> 9, w.z >> 9, w.w >> 9};
      const uint32_t n[4] = {(uint32_t)w.x & 511u, (uint32_t)w.y & 511u, (uint32_t)w.z & 511u,
                             (uint32_t)w.w & 511u};
      if (MODE == 5) {  // Q4 + 32-bit LOP3 addresses + red.shared (no memory clobber)
        const uint32_t hb = (uint32_t)__cvta_generic_to_shared(smem) + 4u * tid;
        uint32_t wv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int off = base + ((q & 1) ? -o[q >> 1] : o[q >> 1]);
          const int a = off & 3;
          const uint32_t* p = reinterpret_cast<const uint32_t*>(tile + (off - a));
          uint32_t v = p[0];
          if (a) v = __funnelshift_r(v, p[1], 8 * a);
          wv[q] = v;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t nn = n[q >> 1], w = wv[q];
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hb | ((w << 12) & 0xff000u)), "r"(nn));
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((hb + 1024u) | ((w << 4) & 0xff000u)), "r"(nn));
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((hb + 2048u) | ((w >> 4) & 0xff000u)), "r"(nn));
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((hb + 3072u) | ((w >> 12) & 0xff000u)), "r"(nn));
        }
        continue;
      }
      if (MODE == 4) {
        uint32_t wv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int off = base + ((q & 1) ? -o[q >> 1] : o[q >> 1]);
          const int a = off & 3;
          const uint32_t* p = reinterpret_cast<const uint32_t*>(tile + (off - a));
          uint32_t v = p[0];
          if (a) v = __funnelshift_r(v, p[1], 8 * a);
          wv[q] = v;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            atomicAdd(hc + (((wv[q] >> (8 * v)) & 0xffu) * 4 + v) * NT, n[q >> 1]);
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (MODE == 0) {
          const uint32_t bp = tile[base + o[k]], bm = tile[base - o[k]];
          atomicAdd(hc + bp * NT, n[k]);
          atomicAdd(hc + bm * NT, n[k]);
        } else if (MODE == 3) {
          uint8_t* hb = smem + 4u * tid;
#pragma unroll
          for (int sgn = 0; sgn < 2; ++sgn) {
            const int off = base + (sgn ? -o[k] : o[k]);
            const int a = off & 3;
            const uint32_t* p = reinterpret_cast<const uint32_t*>(tile + (off - a));
            uint32_t v = p[0];
            if (a) v = __funnelshift_r(v, p[1], 8 * a);
            atomicAdd(reinterpret_cast<uint32_t*>(hb + ((v << 12) & 0xff000u)), n[k]);
            atomicAdd(reinterpret_cast<uint32_t*>(hb + 1024u + ((v << 4) & 0xff000u)), n[k]);
            atomicAdd(reinterpret_cast<uint32_t*>(hb + 2048u + ((v >> 4) & 0xff000u)), n[k]);
            atomicAdd(reinterpret_cast<uint32_t*>(hb + 3072u + ((v >> 12) & 0xff000u)), n[k]);
          }
        } else {
          uint32_t wp, wm;
          if (MODE == 1) {
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int off = base + (s ? -o[k] : o[k]);
              const int a = off & 3;  // warp-uniform: base is 4-aligned
              const uint32_t* p = reinterpret_cast<const uint32_t*>(tile + (off - a));
              uint32_t v = p[0];
              if (a) v = __funnelshift_r(v, p[1], 8 * a);
              if (s) wm = v; else wp = v;
            }
          } else {
            const uint32_t h = (uint32_t)(o[k]) * 2654435761u ^ (uint32_t)tid;
            wp = h & 0x1f1f1f1fu;
            wm = (h >> 3) & 0x1f1f1f1fu;
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            atomicAdd(hc + (((wp >> (8 * v)) & 0xffu) * 4 + v) * NT, n[k]);
            atomicAdd(hc + (((wm >> (8 * v)) & 0xffu) * 4 + v) * NT, n[k]);
          }
        }
      }
    }
  }
  __syncthreads();
  uint32_t s = acc;
  for (int b = 0; b < NB * VPT; ++b) s += hist[b * NT + tid];
  out[blockIdx.x * NT + tid] = s;
}

template <int MODE>
int run(int sms, uint32_t* d_out, const char* name) {
  constexpr int NT = MODE == 0 ? 1024 : 256;
  constexpr int VPT = MODE == 0 ? 1 : 4;
  (void)NT;
  const size_t smem = 33 * NT * VPT * 4 + 76800;
  CK(cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  probe<MODE><<<sms * 2, NT, smem>>>(1, d_out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64;
  cudaEventRecord(a);
  probe<MODE><<<sms * 2, NT, smem>>>(iters, d_out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double updates = (double)sms * 2 * NT * VPT * iters * 2.0 * kTable;
  printf("%-40s %8.2f ms  %.3e updates/s\n", name, ms, updates / (ms * 1e-3));
  return 0;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  std::vector<int> tab(kTable);
  uint32_t s = 12345;
  for (int k = 0; k < kTable; ++k) {
    int dx, dy, dz, n;
    do {
      s = s * 1664525u + 1013904223u;
      dx = int((s >> 8) % 33) - 16;
      dy = int((s >> 16) % 33) - 16;
      dz = int((s >> 24) % 33) - 16;
      n = dx * dx + dy * dy + dz * dz;
    } while (n > 256 || n == 0);
    tab[k] = ((dz * 1920 + dy * 48 + dx) << 9) | n;
  }
  cudaMemcpyToSymbol(c_tab, tab.data(), kTable * 4);
  uint32_t* d_out;
  cudaMalloc(&d_out, sms * 2 * 1024 * 4);
  run<0>(sms, d_out, "A: 1 voxel/thread x1024, LDS.U8+ATOMS");
  run<1>(sms, d_out, "Q: 4 voxels/thread x256, LDS.32x(1|2)+ATOMS");
  run<2>(sms, d_out, "QA: 4 voxels/thread x256, ATOMS only");
  run<3>(sms, d_out, "Q3: as Q, shift+mask addresses, red.shared");
  run<4>(sms, d_out, "Q4: as Q, all 8 fetches before 32 atomics");
  run<5>(sms, d_out, "Q5: Q4 + LOP3 addresses + red.shared");
  return 0;
}
