// exhaustive.cu -- the exhaustive Kadir-Brady pass on sm_100a.
//
// Replaces kadir_brady_exhaustive (/root/reference/proj/src/pipeline.cpp:63-166).
//
// Kernels
//  K1 bin_volume_kernel   f32 -> u8 (bin_of + 1, 0 = outside), HBM-bound pre-pass
//                         (volume.hpp:102-105, same fp64 op order).
//  K2 kb_kernel           one CTA per output tile; the tile's u8 bins plus an
//                         R-voxel halo arrive in shared memory by ONE TMA 3D
//                         tensor copy (out-of-volume voxels are zero-filled by
//                         TMA, i.e. land in the "outside" bin 0). Each thread owns
//                         one voxel and a lane-private histogram column
//                         hist[bin][thread] (bank = thread, conflict-free). It
//                         walks the ball offsets sorted by |o|^2 (constant-memory
//                         table of +-o pairs) adding the integer identity-kernel
//                         weight n = |o|^2 with shared-memory atomics
//                         (ATOMS.ADD, no return). At every needed radius the
//                         column holds S_b(r) exactly (pipeline.cpp:110-117
//                         with the 1/r^2 factor cancelled by normalisation).
//                         Two register snapshots (a ring of 3 radii) give the
//                         inter-scale L1 exactly in integers; entropy in fp32.
//  K3 maxima_kernel       strict 26-neighbour maxima (pipeline.cpp:143-161) ->
//                         u64 keys (score desc, linear index asc), then a cub
//                         radix sort reproduces the stable_sort order (:163-164).
#include <cub/cub.cuh>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstring>
#include <thread>

#include <sys/mman.h>
#include <climits>
#include <cmath>
#include <map>
#include <cstdlib>

#include "common.cuh"

namespace sx {

// ----------------------------------------------------------------------------- K1
// bin + 1 of one intensity: floor((I - low) / (high - low) * bins) clamped to
// [0, bins - 1] (volume.hpp:102-105), the reference's IEEE fp64 operations in
// its order. Fast path: t' = (I - low) * (bins / range) is within a few ulp of
// the reference's t, so when t' is more than 1e-9 away from an integer (and
// |t'| < 1e6, where a few ulp are < 1e-9) floor(t') == floor(t) exactly; only
// values within 1e-9 of a bin edge take the reference's division.
__device__ __forceinline__ uint8_t bin_of(float I, double low, double range, double m,
                                          double inv, int M) {
  const double x = __dsub_rn((double)I, low);
  const double tq = __dmul_rn(x, inv);
  const double f = floor(tq);
  double t = tq;
  if (!(tq - f > 1e-9 && f + 1.0 - tq > 1e-9 && fabs(tq) < 1e6))
    t = __dmul_rn(__ddiv_rn(x, range), m);
  int b = (int)floor(t);
  b = b < 0 ? 0 : (b > M - 1 ? M - 1 : b);
  return (uint8_t)(b + 1);
}

// Rows of nx floats in, rows of `pitch` bytes out; 4 voxels per thread through
// float4 / uchar4 when the row allows it (HBM-bound: 5 B per voxel).
__global__ void bin_volume_kernel(const float* __restrict__ vol, uint8_t* __restrict__ bins,
                                  int nx, long long rows, int pitch, double low, double range,
                                  double m, int M) {
  const double inv = m / range;
  if (pitch == nx && (reinterpret_cast<uintptr_t>(vol) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(bins) & 3) == 0) {
    // rows back to back in both arrays (the exhaustive layout when nx % 16 == 0,
    // the seek layout always): one flat grid-stride pass over the whole slab, U
    // independent 16-byte loads in flight per thread, the last n % 4 voxels scalar
    constexpr int U = 4;
    const long long n = rows * nx, n4 = n >> 2;
    if (blockIdx.x == 0 && threadIdx.x < (n & 3))
      bins[n4 * 4 + threadIdx.x] = bin_of(vol[n4 * 4 + threadIdx.x], low, range, m, inv, M);
    const long long stride = (long long)gridDim.x * blockDim.x;
    const float4* v4 = reinterpret_cast<const float4*>(vol);
    uchar4* b4 = reinterpret_cast<uchar4*>(bins);
    for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < n4) v[u] = __ldg(v4 + i0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < n4) {
          uchar4 o;
          o.x = bin_of(v[u].x, low, range, m, inv, M);
          o.y = bin_of(v[u].y, low, range, m, inv, M);
          o.z = bin_of(v[u].z, low, range, m, inv, M);
          o.w = bin_of(v[u].w, low, range, m, inv, M);
          b4[i0 + u * stride] = o;
        }
    }
    return;
  }
  if ((nx & 3) == 0 && (reinterpret_cast<uintptr_t>(vol) & 15) == 0) {
    // U rows per block step: U independent 16-byte loads in flight per thread
    constexpr int U = 4;
    const int n4 = nx >> 2;
    for (long long r0 = (long long)blockIdx.x * U; r0 < rows; r0 += (long long)gridDim.x * U) {
      for (int x4 = threadIdx.x; x4 < n4; x4 += blockDim.x) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r0 + u < rows) v[u] = __ldg(reinterpret_cast<const float4*>(vol + (r0 + u) * nx) + x4);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (r0 + u < rows) {
            uchar4 o;
            o.x = bin_of(v[u].x, low, range, m, inv, M);
            o.y = bin_of(v[u].y, low, range, m, inv, M);
            o.z = bin_of(v[u].z, low, range, m, inv, M);
            o.w = bin_of(v[u].w, low, range, m, inv, M);
            reinterpret_cast<uchar4*>(bins + (r0 + u) * pitch)[x4] = o;  // pitch % 16 == 0
          }
      }
    }
    return;
  }
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* src = vol + row * nx;
    uint8_t* dst = bins + row * pitch;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) dst[x] = bin_of(src[x], low, range, m, inv, M);
  }
}

void launch_bin_volume(salvox_ctx* ctx, const float* d_vol, uint8_t* d_bins, int nx, int ny,
                       int nzs, int pitch, double low, double high, int bins,
                       cudaStream_t stream) {
  const long long rows = (long long)ny * nzs;
  const int lanes = (nx & 3) == 0 ? nx / 4 : nx;  // threads one row needs
  int block = lanes >= 128 ? 128 : ((lanes + 31) / 32) * 32;
  const long long steps = (nx & 3) == 0 ? (rows + 3) / 4 : rows;  // block steps of 4 / 1 rows
  int grid = (int)std::min<long long>(steps, (long long)ctx->sm_count * 16);
  if (pitch == nx) {  // flat form: 256 threads x U = 4 float4 each per block step
    block = 256;
    grid = (int)std::max<long long>(1, std::min<long long>((rows * nx / 4 + 1023) / 1024,
                                                           (long long)ctx->sm_count * 8));
  }
  bin_volume_kernel<<<grid, block, 0, stream ? stream : ctx->stream>>>(d_vol, d_bins, nx, rows, pitch, low,
                                                      high - low, (double)bins, bins);
  SX_LAUNCH_CHECK(ctx);
}

__device__ __forceinline__ uint32_t ordered_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float key_to_float(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

__global__ void minmax_kernel(const float* __restrict__ v, size_t n, uint32_t* out) {
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t k = ordered_key(v[i]);
    lo = min(lo, k);
    hi = max(hi, k);
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

void device_full_range(salvox_ctx* ctx, const float* d_vol, size_t n, double* low, double* high) {
  uint32_t* d = ctx->d_minmax.as<uint32_t>();
  if (!d) d = static_cast<uint32_t*>(ctx->d_minmax.ensure(64));
  SX_CUDA(cudaMemsetAsync(d, 0xff, 4, ctx->stream));
  SX_CUDA(cudaMemsetAsync(d + 1, 0x00, 4, ctx->stream));
  minmax_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(d_vol, n, d);
  SX_LAUNCH_CHECK(ctx);
  uint32_t h[2];
  SX_CUDA(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  const float lo = key_to_float(h[0]);
  float hi = key_to_float(h[1]);
  if (!(lo < hi)) hi = lo + 1.0f;  // volume.hpp:110
  *low = lo;
  *high = hi;
}

// ----------------------------------------------------------------------------- K2
struct KbBound {
  int32_t lend;   // end of this radius' run of |o|^2 levels
  int32_t flags;  // bit0: r_i is a scale (entropy); bit1: evaluate scale r_{i-1}
  int32_t rank;   // first position of scale r_{i-1} in the caller's list
  uint32_t W;     // sum of |o|^2 over B(r_i) \ {0}: T(r_i) = W - S_0 (bin 0 = outside)
  double fac;     // s * s / 2.0 (pipeline.cpp:131)
  float scale;    // (float) r_{i-1}
  // Epanechnikov (kb_kernel<EPA>): #B(r_i) incl. the centre, and q, q * r_i^2
  // with q in {1, 4} the smallest making q * r_i^2 an integer (0: none)
  uint32_t cnt;
  uint32_t r2q, q;
};

// One |o|^2 level: the +-o representatives with that squared norm are
// c_offs[start, start + count) (start is a multiple of 4), weight n. The pair
// kernel splits a level by the parity of o.x: list 0 (even) and list 1 (odd).
struct KbLevel {
  int32_t start0, start1;
  int16_t count0, count1;
  int32_t n;
};

constexpr int kMaxOffs = 10240;   // 40 KB of constant memory
constexpr int kMaxLevels = 640;
constexpr int kMaxRadii = 192;
__constant__ int4 c_offs[kMaxOffs / 4];
__constant__ KbLevel c_levels[kMaxLevels];
__constant__ KbBound c_bounds[kMaxRadii];
// kb_quad_kernel: per radius, the ends (in int4 groups of c_offs) of its three
// class runs (x, y, z); the radius' first run starts at the previous radius' z
__constant__ int4 c_qruns[kMaxRadii];
// kb_quad_kernel<DBL>: per radius, two more run ends: the x-adjacent doubles of
// class 0 and class 1 (see make_plan)
__constant__ int2 c_qruns2[kMaxRadii];

struct KbParams {
  int nx, ny, nz;   // global dims
  int zs0;          // global z of slab plane 0
  int zc0, zc1;     // computed (scored) global planes
  int R, Rz, SY, SZ;  // halo (Rz = 0 for 2D) and shared-memory strides
  int n_radii;
  int bins;
  uint32_t tile_bytes;
  int lag;          // kb_quad_kernel: warps 4-7 start the walk this many cycles late
  int lagmode;      // 0: warps 4-7 by lag; 1: warp w by w*lag/4; 3: (w%4)*lag/8 + (w/4)*lag
  float* score;     // planes [zc0, zc1)
  float* best;
  // kb_quad_kernel: also store the planes [hz0, hz1) straight into the caller's
  // pinned host maps (plane hz0 at h_score[0]); null = device maps only
  float* h_score;
  float* h_best;
  int hz0, hz1;
  const long long* dbg_vox;  // debug launch: one block per voxel
  uint32_t* dbg_out;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// EPA (Epanechnikov kernel, K(d) = 1 - d, kernel.hpp:21): a second column of
// per-bin counts C_b(r) beside the sums S_b(r), so per bin the exact integer
// q * h_b * r^2 = q r^2 C_b(r) - q S_b(r) (the centre, d = 0, weight 1, is
// counted once up front); same walk, two 32-bit shared atomics per update (a
// 64-bit count|sum word would compile to a CAS loop).
template <int NB, int TX, int TY, int TZ, bool DBG, bool EPA = false>
__global__ void __launch_bounds__(TX* TY* TZ, 1)
    kb_kernel(const __grid_constant__ CUtensorMap tmap, const KbParams p) {
  constexpr int NT = TX * TY * TZ;
  constexpr int WB = EPA ? 8 : 4;  // bytes per histogram word
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);  // EPA: sums, then counts
  uint8_t* tile = smem + NB * NT * WB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + ((p.tile_bytes + 15u) & ~15u));
  const int tid = threadIdx.x;

  int tx0, ty0, tz0;
  long long dbg_lin = -1;
  if (DBG) {
    dbg_lin = p.dbg_vox[blockIdx.x];
    const int vx = (int)(dbg_lin % p.nx);
    const int vy = (int)((dbg_lin / p.nx) % p.ny);
    const int vz = (int)(dbg_lin / ((long long)p.nx * p.ny));
    tx0 = vx / TX * TX;
    ty0 = vy / TY * TY;
    tz0 = p.zc0 + (vz - p.zc0) / TZ * TZ;
  } else {
    tx0 = blockIdx.x * TX;
    ty0 = blockIdx.y * TY;
    tz0 = p.zc0 + blockIdx.z * TZ;
  }

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // TMA needs the innermost box coordinate 16-byte aligned: start the box at
  // floor16(tx0 - R) and shift this block's voxels right by delta.
  const int xs = tx0 - p.R;
  const int xa = xs - (((xs % 16) + 16) % 16);
  const int delta = xs - xa;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(p.tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(tile)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(xa), "r"(ty0 - p.R),
        "r"(tz0 - p.Rz - p.zs0), "r"(smem_u32(bar))
        : "memory");
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int i = tid; i < NB * NT * WB / 16; i += NT) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  const int lx = tid % TX, ly = (tid / TX) % TY, lz = tid / (TX * TY);
  const int gx = tx0 + lx, gy = ty0 + ly, gz = tz0 + lz;
  const uint8_t* tb = tile + (lz + p.Rz) * p.SZ + (ly + p.R) * p.SY + (lx + p.R + delta);
  uint32_t* hc = hist + tid;
  uint32_t* hcc = hist + NB * NT + tid;  // EPA counts
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
    }
  }
  __syncthreads();
  const bool valid = gx < p.nx && gy < p.ny && gz < p.zc1;
  if (!valid) return;
  const bool dbg_me =
      DBG && ((long long)gx + (long long)p.nx * ((long long)gy + (long long)p.ny * gz)) == dbg_lin;
  if (DBG && !dbg_me) return;
  if (EPA) hcc[(uint32_t)tb[0] * NT] += 1u;  // the centre (private column)

  uint32_t A[NB], B[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) A[b] = B[b] = 0u;
  uint32_t TA = 0u, TB = 0u;
  float Hb = 0.f;
  double best = 0.0;
  float best_s = 0.f;
  int best_rank = INT_MAX;

  // Walk the |o|^2 levels in order; within a level the weight n is loop-invariant
  // (one register), each table entry is a raw tile offset o giving two updates
  // (+o and -o): per update one address add, one LDS.U8, one IMAD, one ATOMS.
  const int4* offs4 = c_offs;
  int lvl = 0;
  // A warp with no valid voxel (z-planes past zc1 in a slab's last tile layer,
  // x/y past the edge) skips the walk: its TMEM slice and histogram columns are
  // private, so the other warps run alone and finish sooner.
  const int n_radii = __any_sync(0xffffffffu, valid) ? p.n_radii : 0;
  for (int i = 0; i < n_radii; ++i) {
    const KbBound bd = c_bounds[i];
    for (; lvl < bd.lend; ++lvl) {
      const KbLevel L = c_levels[lvl];
      const uint32_t n = (uint32_t)L.n;
      auto upd = [&](uint32_t b) {
        atomicAdd(hc + b * NT, n);
        if (EPA) atomicAdd(hcc + b * NT, 1u);
      };
      const int g0 = L.start0 >> 2, g1 = (L.start0 + L.count0) >> 2;
#pragma unroll 2
      for (int g = g0; g < g1; ++g) {
        const int4 w = offs4[g];
        const uint32_t b0 = tb[w.x], b1 = tb[-w.x], b2 = tb[w.y], b3 = tb[-w.y];
        const uint32_t b4 = tb[w.z], b5 = tb[-w.z], b6 = tb[w.w], b7 = tb[-w.w];
        upd(b0);
        upd(b1);
        upd(b2);
        upd(b3);
        upd(b4);
        upd(b5);
        upd(b6);
        upd(b7);
      }
      const int rem = (L.count0 & 3);
      if (rem) {  // tail of the level (entries of the last group, in order)
        const int4 w = offs4[g1];
        const int o[3] = {w.x, w.y, w.z};
        for (int j = 0; j < rem; ++j) {
          const uint32_t bp = tb[o[j]], bm = tb[-o[j]];
          upd(bp);
          upd(bm);
        }
      }
    }
    // ---- boundary: the column now holds S_b(r_i) for b = 0..NB-1 (0 = outside)
    // (EPA: and C_b(r_i); the bin value is q r^2 C_b - q S_b)
    auto bin_value = [&](int b) -> uint32_t {
      return EPA ? bd.r2q * hcc[b * NT] - bd.q * hc[b * NT] : hc[b * NT];
    };
    const uint32_t T = EPA ? bd.r2q * (bd.cnt - hcc[0]) - bd.q * (bd.W - hc[0]) : bd.W - hc[0];
    const bool doH = (bd.flags & 1) && T > 0u;
    const bool doE = (bd.flags & 2) && T > 0u && TA > 0u && TB > 0u;
    const float invT = doH ? 1.0f / (float)T : 0.f;
    float hacc = 0.f;
    unsigned long long num = 0ull;
#pragma unroll
    for (int b = 1; b < NB; ++b) {
      const uint32_t c = bin_value(b);
      if (doH && c) {
        const float pb = (float)c * invT;
        float lg;
        if (2u * c > T) {  // the one dominant bin: log(1 - q) with q exact-ish
          lg = log1pf(-(float)(T - c) * invT) * 1.4426950408889634f;
        } else {
          lg = __log2f(pb);
        }
        hacc -= pb * lg;
      }
      if (doE) {
        const unsigned long long x = (unsigned long long)c * TA;
        const unsigned long long y = (unsigned long long)A[b] * T;
        num += x > y ? x - y : y - x;
      }
      if (DBG && b - 1 < p.bins) p.dbg_out[(size_t)i * (p.bins + 1) + (b - 1)] = c;
      A[b] = B[b];
      B[b] = c;
    }
    if (DBG) p.dbg_out[(size_t)i * (p.bins + 1) + p.bins] = T;
    if (doE) {
      const double l1 = (double)num / ((double)T * (double)TA);
      const double y = ((double)Hb * bd.fac) * l1;
      if (y > best || (y == best && y > 0.0 && bd.rank < best_rank)) {
        best = y;
        best_s = bd.scale;
        best_rank = bd.rank;
      }
    }
    TA = TB;
    TB = T;
    Hb = doH ? fmaxf(hacc, 0.f) : 0.f;
  }
  if (!DBG) {
    const size_t o = ((size_t)(gz - p.zc0) * p.ny + gy) * p.nx + gx;
    p.score[o] = (float)best;
    p.best[o] = best_s;
  }
}

__device__ __forceinline__ void pair_atom(uint32_t saddr, uint32_t n) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(n) : "memory");
}

// K2' (NB <= 33): two x-adjacent voxels per thread. One LDS.U16 fetches both
// voxels' bins for an offset: even x-offsets read the TMA tile (A), odd ones a
// one-byte-shifted copy (B[k] = A[k+1], built in shared memory after the TMA
// load), so every fetch is 2-byte aligned and bin fetches cost 0.5 wavefront
// per update instead of 1 (the ATOMS.ADD per update is the irreducible part).
// Each |o|^2 level is split by o.x parity so the copy choice is loop-invariant.
// Warp footprint 8 voxels (4 threads) x 8 rows at a 48-byte row pitch: the 8
// rows' 2-3-word spans fall in disjoint banks.
template <int NB, int TY, int TZ, bool DBG>
__global__ void __launch_bounds__(4 * TY * TZ, 1)
    kb_pair_kernel(const __grid_constant__ CUtensorMap tmap, const KbParams p) {
  constexpr int TX = 8;
  constexpr int NT = 4 * TY * TZ;  // threads
  constexpr int NC = 2 * NT;       // histogram columns (voxels)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  uint8_t* tileA = smem + NB * NC * 4;
  const uint32_t tstride = (p.tile_bytes + 127u) & ~127u;
  uint8_t* tileB = tileA + tstride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tileB + tstride);
  const int tid = threadIdx.x;

  int tx0, ty0, tz0;
  long long dbg_lin = -1;
  if (DBG) {
    dbg_lin = p.dbg_vox[blockIdx.x];
    const int vx = (int)(dbg_lin % p.nx);
    const int vy = (int)((dbg_lin / p.nx) % p.ny);
    const int vz = (int)(dbg_lin / ((long long)p.nx * p.ny));
    tx0 = vx / TX * TX;
    ty0 = vy / TY * TY;
    tz0 = p.zc0 + (vz - p.zc0) / TZ * TZ;
  } else {
    tx0 = blockIdx.x * TX;
    ty0 = blockIdx.y * TY;
    tz0 = p.zc0 + blockIdx.z * TZ;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int xs = tx0 - p.R;
  const int xa = xs - (((xs % 16) + 16) % 16);
  const int delta = xs - xa;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(p.tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(tileA)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(xa), "r"(ty0 - p.R),
        "r"(tz0 - p.Rz - p.zs0), "r"(smem_u32(bar))
        : "memory");
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int i = tid; i < NB * NC / 4; i += NT) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
    }
  }
  {  // B[k] = A[k + 1]: funnel-shift 16-byte chunks
    const uint32_t* a32 = reinterpret_cast<const uint32_t*>(tileA);
    uint4* b4 = reinterpret_cast<uint4*>(tileB);
    const int nchunk = (int)(p.tile_bytes + 15u) / 16;
    for (int i = tid; i < nchunk; i += NT) {
      const uint4 v = reinterpret_cast<const uint4*>(tileA)[i];
      const uint32_t nx4 = (4 * i + 4) * 4 < (int)tstride ? a32[4 * i + 4] : 0u;
      b4[i] = make_uint4(__funnelshift_r(v.x, v.y, 8), __funnelshift_r(v.y, v.z, 8),
                         __funnelshift_r(v.z, v.w, 8), __funnelshift_r(v.w, nx4, 8));
    }
  }
  __syncthreads();
  const int lxp = tid & 3, ly = (tid >> 2) % TY, lz = tid / (4 * TY);
  const int gx = tx0 + 2 * lxp, gy = ty0 + ly, gz = tz0 + lz;
  const bool valid0 = gx < p.nx && gy < p.ny && gz < p.zc1;
  const bool valid1 = valid0 && gx + 1 < p.nx;
  if (!valid0) return;
  const long long lin0 = (long long)gx + (long long)p.nx * ((long long)gy + (long long)p.ny * gz);
  const int dbg_which = DBG ? (lin0 == dbg_lin ? 0 : (valid1 && lin0 + 1 == dbg_lin ? 1 : -1)) : 0;
  if (DBG && dbg_which < 0) return;
  const uint8_t* tbA = tileA + (lz + p.Rz) * p.SZ + (ly + p.R) * p.SY + (2 * lxp + p.R + delta);
  const uint8_t* tbB = tbA + (tstride - 1);  // odd x-offset s: B[s - 1] = (A[s], A[s + 1])
  uint32_t* h0 = hist + tid;
  uint32_t* h1 = hist + NT + tid;
  // shared-window byte addresses: column c of bin b lives at hbase + b * NC * 4 + c * 4
  // (NC * 4 = 2^11 and the column offset < 2^11, so the bin field can be OR-ed in)
  static_assert(NC * 4 == 2048, "pair kernel assumes 512 columns");
  const uint32_t hs0 = smem_u32(h0), hs1 = smem_u32(h1);

  uint32_t A0[NB], B0[NB], A1[NB], B1[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) A0[b] = B0[b] = A1[b] = B1[b] = 0u;
  uint32_t TA0 = 0u, TB0 = 0u, TA1 = 0u, TB1 = 0u;
  float Hb0 = 0.f, Hb1 = 0.f;
  double best0 = 0.0, best1 = 0.0;
  float bs0 = 0.f, bs1 = 0.f;
  int br0 = INT_MAX, br1 = INT_MAX;

  const int4* offs4 = c_offs;
  auto run_list = [&](const uint8_t* tb, int start, int count, uint32_t n) {
    const int g0 = start >> 2, g1 = (start + count) >> 2;
#pragma unroll 2
    for (int g = g0; g < g1; ++g) {
      const int4 w = offs4[g];
      const uint32_t vs[8] = {*reinterpret_cast<const uint16_t*>(tb + w.x),
                              *reinterpret_cast<const uint16_t*>(tb - w.x),
                              *reinterpret_cast<const uint16_t*>(tb + w.y),
                              *reinterpret_cast<const uint16_t*>(tb - w.y),
                              *reinterpret_cast<const uint16_t*>(tb + w.z),
                              *reinterpret_cast<const uint16_t*>(tb - w.z),
                              *reinterpret_cast<const uint16_t*>(tb + w.w),
                              *reinterpret_cast<const uint16_t*>(tb - w.w)};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        pair_atom(hs0 + (__byte_perm(vs[j], 0u, 0x4440) << 11), n);
        pair_atom(hs1 + (__byte_perm(vs[j], 0u, 0x4441) << 11), n);
      }
    }
    const int rem = count & 3;
    if (rem) {
      const int4 w = offs4[g1];
      const int o[3] = {w.x, w.y, w.z};
      for (int j = 0; j < rem; ++j) {
        const uint32_t vp = *reinterpret_cast<const uint16_t*>(tb + o[j]);
        const uint32_t vm = *reinterpret_cast<const uint16_t*>(tb - o[j]);
        pair_atom(hs0 + (__byte_perm(vp, 0u, 0x4440) << 11), n);
        pair_atom(hs1 + (__byte_perm(vp, 0u, 0x4441) << 11), n);
        pair_atom(hs0 + (__byte_perm(vm, 0u, 0x4440) << 11), n);
        pair_atom(hs1 + (__byte_perm(vm, 0u, 0x4441) << 11), n);
      }
    }
  };

  int lvl = 0;
  for (int i = 0; i < p.n_radii; ++i) {
    const KbBound bd = c_bounds[i];
    for (; lvl < bd.lend; ++lvl) {
      const KbLevel L = c_levels[lvl];
      run_list(tbA, L.start0, L.count0, (uint32_t)L.n);
      run_list(tbB, L.start1, L.count1, (uint32_t)L.n);
    }
    // ---- boundary: both columns hold S_b(r_i)
    const uint32_t T0 = bd.W - h0[0], T1 = bd.W - h1[0];
    const bool doH0 = (bd.flags & 1) && T0 > 0u, doH1 = (bd.flags & 1) && T1 > 0u;
    const bool doE0 = (bd.flags & 2) && T0 > 0u && TA0 > 0u && TB0 > 0u;
    const bool doE1 = (bd.flags & 2) && T1 > 0u && TA1 > 0u && TB1 > 0u;
    const float invT0 = doH0 ? 1.0f / (float)T0 : 0.f;
    const float invT1 = doH1 ? 1.0f / (float)T1 : 0.f;
    float hacc0 = 0.f, hacc1 = 0.f;
    unsigned long long num0 = 0ull, num1 = 0ull;
#pragma unroll
    for (int b = 1; b < NB; ++b) {
      const uint32_t c0 = h0[b * NC], c1 = h1[b * NC];
      if (doH0 && c0) {
        const float pb = (float)c0 * invT0;
        const float lg = (2u * c0 > T0) ? log1pf(-(float)(T0 - c0) * invT0) * 1.4426950408889634f
                                        : __log2f(pb);
        hacc0 -= pb * lg;
      }
      if (doH1 && c1) {
        const float pb = (float)c1 * invT1;
        const float lg = (2u * c1 > T1) ? log1pf(-(float)(T1 - c1) * invT1) * 1.4426950408889634f
                                        : __log2f(pb);
        hacc1 -= pb * lg;
      }
      if (doE0) {
        const unsigned long long x = (unsigned long long)c0 * TA0, y = (unsigned long long)A0[b] * T0;
        num0 += x > y ? x - y : y - x;
      }
      if (doE1) {
        const unsigned long long x = (unsigned long long)c1 * TA1, y = (unsigned long long)A1[b] * T1;
        num1 += x > y ? x - y : y - x;
      }
      if (DBG && b - 1 < p.bins)
        p.dbg_out[(size_t)i * (p.bins + 1) + (b - 1)] = dbg_which == 0 ? c0 : c1;
      A0[b] = B0[b];
      B0[b] = c0;
      A1[b] = B1[b];
      B1[b] = c1;
    }
    if (DBG) p.dbg_out[(size_t)i * (p.bins + 1) + p.bins] = dbg_which == 0 ? T0 : T1;
    if (doE0) {
      const double y = ((double)Hb0 * bd.fac) * ((double)num0 / ((double)T0 * (double)TA0));
      if (y > best0 || (y == best0 && y > 0.0 && bd.rank < br0)) {
        best0 = y;
        bs0 = bd.scale;
        br0 = bd.rank;
      }
    }
    if (doE1) {
      const double y = ((double)Hb1 * bd.fac) * ((double)num1 / ((double)T1 * (double)TA1));
      if (y > best1 || (y == best1 && y > 0.0 && bd.rank < br1)) {
        best1 = y;
        bs1 = bd.scale;
        br1 = bd.rank;
      }
    }
    TA0 = TB0;
    TB0 = T0;
    TA1 = TB1;
    TB1 = T1;
    Hb0 = doH0 ? fmaxf(hacc0, 0.f) : 0.f;
    Hb1 = doH1 ? fmaxf(hacc1, 0.f) : 0.f;
  }
  if (!DBG) {
    const size_t o = ((size_t)(gz - p.zc0) * p.ny + gy) * p.nx + gx;
    p.score[o] = (float)best0;
    p.best[o] = bs0;
    if (valid1) {
      p.score[o + 1] = (float)best1;
      p.best[o + 1] = bs1;
    }
  }
}

// K2'' (3D; SALVOX_KB_VARIANT=2 at NB <= 33, SALVOX_KB65=tmem at 65 with 512 threads): 1024 threads per CTA (32 warps/SM, twice kb_kernel's
// latency hiding) with the two radius snapshots held in TENSOR MEMORY. At 1024
// threads the register file allows 64 registers per thread, too few for the
// 2 x 32 snapshot words, so each thread parks them in its TMEM lane: warp w
// owns lanes 32*(w%4).. and the 64-column slice 64*(w/4); columns [0,32) and
// [32,64) of the slice are the two ring slots (bins 1..32). At each radius the
// older slot is streamed out with tcgen05.ld (8 columns at a time), combined
// with the live shared-memory column (L1 term), and overwritten in place with
// the live column by tcgen05.st -- it becomes the newest snapshot.
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}

__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// NT = 1024 (NB <= 33: a 16x8x8 tile) or 512 (NB = 65: 16x8x4, the default
// 64-bin window of the reference). Either way each warp's lane group owns a
// 2 * NS column slice and the NT / 128 slices fill the 512 TMEM columns.
template <int NB, bool DBG, int NT = 1024>
__global__ void __launch_bounds__(NT, 1)
    kb_tmem_kernel(const __grid_constant__ CUtensorMap tmap, const KbParams p) {
  constexpr int TX = 16, TY = 8, TZ = NT / 128;
  constexpr int NS = NB - 1;  // snapshot bins (1..NB-1); multiple of 8
  static_assert(NS % 8 == 0 && 2 * NS * (NT / 128) <= 512, "TMEM: 2 * NS columns per thread");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  uint8_t* tile = smem + NB * NT * 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + ((p.tile_bytes + 15u) & ~15u));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int tx0, ty0, tz0;
  long long dbg_lin = -1;
  if (DBG) {
    dbg_lin = p.dbg_vox[blockIdx.x];
    const int vx = (int)(dbg_lin % p.nx);
    const int vy = (int)((dbg_lin / p.nx) % p.ny);
    const int vz = (int)(dbg_lin / ((long long)p.nx * p.ny));
    tx0 = vx / TX * TX;
    ty0 = vy / TY * TY;
    tz0 = p.zc0 + (vz - p.zc0) / TZ * TZ;
  } else {
    tx0 = blockIdx.x * TX;
    ty0 = blockIdx.y * TY;
    tz0 = p.zc0 + blockIdx.z * TZ;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // all 512 TMEM columns: one CTA per SM (shared memory bound)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  const int xs = tx0 - p.R;
  const int xa = xs - (((xs % 16) + 16) % 16);
  const int delta = xs - xa;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(p.tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(tile)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(xa), "r"(ty0 - p.R),
        "r"(tz0 - p.Rz - p.zs0), "r"(smem_u32(bar))
        : "memory");
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int i = tid; i < NB * NT / 4; i += NT) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
    }
  }
  __syncthreads();
  // warp footprint 8 (x) x 4 (y): lane -> (x, y); warps tile 2 (x) x 2 (y) x TZ (z)
  const int lx = (lane & 7) + 8 * (warp & 1);
  const int ly = (lane >> 3) + 4 * ((warp >> 1) & 1);
  const int lz = warp >> 2;
  const int gx = tx0 + lx, gy = ty0 + ly, gz = tz0 + lz;
  const bool valid = gx < p.nx && gy < p.ny && gz < p.zc1;
  const bool dbg_me =
      DBG && valid && ((long long)gx + (long long)p.nx * ((long long)gy + (long long)p.ny * gz)) == dbg_lin;
  // invalid threads keep walking (their tile bytes exist) so the warp-wide
  // tcgen05.ld/st stay converged; they just never store a result
  const uint8_t* tb = tile + (lz + p.Rz) * p.SZ + (ly + p.R) * p.SY + (lx + p.R + delta);
  uint32_t* hc = hist + tid;
  const uint32_t lane_base =
      tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(2 * NS * (warp >> 2));
  uint32_t slotA = lane_base, slotB = lane_base + NS;  // A: older, B: newer

  {  // zero both TMEM slots (snapshots of "radius 0")
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 2 * NS; c += 8) tm_st8(lane_base + c, z);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  uint32_t TA = 0u, TB = 0u;
  float Hb = 0.f;
  double best = 0.0;
  float best_s = 0.f;
  int best_rank = INT_MAX;

  const int4* offs4 = c_offs;
  int lvl = 0;
  // A warp with no valid voxel (z-planes past zc1 in a slab's last tile layer,
  // x/y past the edge) skips the walk: its TMEM slice and histogram columns are
  // private, so the other warps run alone and finish sooner.
  const int n_radii = __any_sync(0xffffffffu, valid) ? p.n_radii : 0;
  for (int i = 0; i < n_radii; ++i) {
    const KbBound bd = c_bounds[i];
    for (; lvl < bd.lend; ++lvl) {
      const KbLevel L = c_levels[lvl];
      const uint32_t n = (uint32_t)L.n;
      const int g0 = L.start0 >> 2, g1 = (L.start0 + L.count0) >> 2;
#pragma unroll 2
      for (int g = g0; g < g1; ++g) {
        const int4 w = offs4[g];
        const uint32_t b0 = tb[w.x], b1 = tb[-w.x], b2 = tb[w.y], b3 = tb[-w.y];
        const uint32_t b4 = tb[w.z], b5 = tb[-w.z], b6 = tb[w.w], b7 = tb[-w.w];
        atomicAdd(hc + b0 * NT, n);
        atomicAdd(hc + b1 * NT, n);
        atomicAdd(hc + b2 * NT, n);
        atomicAdd(hc + b3 * NT, n);
        atomicAdd(hc + b4 * NT, n);
        atomicAdd(hc + b5 * NT, n);
        atomicAdd(hc + b6 * NT, n);
        atomicAdd(hc + b7 * NT, n);
      }
      const int rem = (L.count0 & 3);
      if (rem) {
        const int4 w = offs4[g1];
        const int o[3] = {w.x, w.y, w.z};
        for (int j = 0; j < rem; ++j) {
          const uint32_t bp = tb[o[j]], bm = tb[-o[j]];
          atomicAdd(hc + bp * NT, n);
          atomicAdd(hc + bm * NT, n);
        }
      }
    }
    // ---- boundary
    const uint32_t T = bd.W - hc[0];
    const bool doH = (bd.flags & 1) && T > 0u;
    const bool doE = (bd.flags & 2) && T > 0u && TA > 0u && TB > 0u;
    const float invT = doH ? 1.0f / (float)T : 0.f;
    float hacc = 0.f;
    uint32_t dom = 0u;  // the bin holding more than half the mass (at most one)
    unsigned long long num = 0ull;
#pragma unroll
    for (int c = 0; c < NS; c += 8) {
      uint32_t a[8], cur[8];
      tm_ld8(slotA + c, a);
#pragma unroll
      for (int j = 0; j < 8; ++j) cur[j] = hc[(1 + c + j) * NT];
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("" : "+r"(a[j]));  // no use before the wait
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t cv = cur[j];
#ifndef KB_SKIP_MATH
        // -p log2 p with MUFU log2; a dominant bin (p > 1/2) is deferred to one
        // log1pf after the loop, so the slow path never diverges across bins
        if (2u * cv > T) {
          dom = cv;
        } else if (doH && cv) {
          const float pb = (float)cv * invT;
          hacc -= pb * __log2f(pb);
        }
#endif
        if (doE) {
          const unsigned long long x = (unsigned long long)cv * TA, y = (unsigned long long)a[j] * T;
          num += x > y ? x - y : y - x;
        }
        if (DBG && dbg_me && c + j < p.bins) p.dbg_out[(size_t)i * (p.bins + 1) + c + j] = cv;
      }
      tm_st8(slotA + c, cur);  // the older slot becomes the newest snapshot
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (doH && dom) {
      const float pb = (float)dom * invT;
      hacc -= pb * (log1pf(-(float)(T - dom) * invT) * 1.4426950408889634f);
    }
    if (DBG && dbg_me) p.dbg_out[(size_t)i * (p.bins + 1) + p.bins] = T;
    if (doE) {
      const double y = ((double)Hb * bd.fac) * ((double)num / ((double)T * (double)TA));
      if (y > best || (y == best && y > 0.0 && bd.rank < best_rank)) {
        best = y;
        best_s = bd.scale;
        best_rank = bd.rank;
      }
    }
    const uint32_t t = slotA;
    slotA = slotB;
    slotB = t;
    TA = TB;
    TB = T;
    Hb = doH ? fmaxf(hacc, 0.f) : 0.f;
  }
  if (!DBG && valid) {
    const size_t o = ((size_t)(gz - p.zc0) * p.ny + gy) * p.nx + gx;
    p.score[o] = (float)best;
    p.best[o] = best_s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

// K2-quad (3D, the default; NB = 65 runs 128 threads with paired-voxel panels,
// see QuadLayout): 256 threads, FOUR x-adjacent
// voxels per thread, built so an update costs ~2.9 instructions and ~1.44
// shared-pipe wavefronts instead of kb_tmem_kernel's ~4 and 2:
//  * bins: the tile row pitch and box start are multiples of 16 and each
//    thread's first voxel sits on a 4-byte boundary, so the 4 bins a thread
//    needs at offset o are bytes s..s+3 of two aligned words, s = o.x mod 4.
//    The table stores each +-o pair with the representative whose s is 0, 1 or
//    2 ("class"), in one run per (radius, class), so s is a template constant;
//  * address = ONE PRMT: column c of a 64-column panel is byte c*4 of the
//    address and the bin is byte 1, so PRMT(word, c*4, sel) = bin*256 + c*4 --
//    byte extract and address in one instruction -- and the panel (which of the
//    16 panels of 64 columns x NB bins: voxel v, column group G) is the atomic's
//    immediate. G = warp % 4 is the SM sub-partition, so each sub-partition runs
//    one specialisation of the loop (one copy in its instruction cache).
// Snapshots: 4 voxels x 2 slots x 32 bins = all 256 TMEM columns of the
// thread's lane (warp w: lanes 32*(w%4), columns 256*(w/4)).
__device__ __forceinline__ uint32_t lds32(const uint8_t* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}

__device__ __forceinline__ float lg2_ftz(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// p log2 p of one bin (p >= 2^-22 when the bin is not empty: no denormals; an
// empty bin gives 0 * lg2(1e-30) = 0 -- no branch, no NaN)
__device__ __forceinline__ float ent_term(float pb) {
  const float l = lg2_ftz(pb + 1e-30f);
  return __fmul_rn(pb, l);
}

// q += max(c * ta + a * nt, 0) with 32-bit signed factors and a 64-bit sum
__device__ __forceinline__ void l1_pos_acc(long long& q, int c, int ta, int a, int nt) {
  asm("{ .reg .s64 x; .reg .pred p;\n\t"
      "mul.wide.s32 x, %1, %2;\n\t"
      "mad.wide.s32 x, %3, %4, x;\n\t"
      "setp.gt.s64 p, x, 0;\n\t"
      "@p add.s64 %0, %0, x; }"
      : "+l"(q)
      : "r"(c), "r"(ta), "r"(a), "r"(nt));
}

template <class T>
__device__ __forceinline__ void rot4(T (&x)[4]) {
  const T t = x[0];
  x[0] = x[1];
  x[1] = x[2];
  x[2] = x[3];
  x[3] = t;
}

// The first byte of dynamic shared memory sits at shared::cta address
// (CTA-rank << 24) + 0x400 (1 KB reserved; the kernel checks it). The rank bits
// ride in bytes 2-3 of c, the 0x400 in the atomic's immediate.
constexpr uint32_t kDsmemBase = 0x400u;

template <int J>
__device__ __forceinline__ uint32_t quad_prmt(uint32_t w0, uint32_t w1, uint32_t c) {
  // volatile: keeps the 8 PRMTs of an entry ahead of its 8 REDs (the ALU
  // latency is then covered without relying on other warps -- 2 per SMSP)
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(J < 4 ? w0 : w1), "r"(c),
               "n"(0x7604u | ((uint32_t)(J & 3) << 4)));
  return r;
}

// Histogram panel of voxel V in column group G. NB <= 33: 16 panels [V * 4 + G]
// of 64 columns (8 warps: column = lane + 32 * (warp / 4)). NB = 65 (128
// threads, 4 warps): 8 panels [(V / 2) * 4 + G], voxels 2k and 2k + 1 in the
// two 32-column halves -- the PRMT address keeps its 256-byte bin rows and the
// 65 bins x 512 voxels fit in 133 KB.
template <int NB>
struct QuadLayout {
  static constexpr bool PP = NB > 33;            // paired-voxel panels
  static constexpr int NT = PP ? 128 : 256;      // threads
  static constexpr int TZ = PP ? 4 : 8;          // tile planes (16 x 8 x TZ voxels / 4 per thread)
  static constexpr int SL = NB - 1 < 32 ? 32 : NB - 1;  // TMEM columns per snapshot slot
  static constexpr int panel(int V, int G) { return PP ? (V >> 1) * 4 + G : V * 4 + G; }
  static constexpr int coloff(int V) { return PP ? 32 * (V & 1) : 0; }  // words
};

template <int NB, int G, int V>
__device__ __forceinline__ void quad_red1(uint32_t a, uint32_t n) {
  constexpr uint32_t IMM = kDsmemBase + (uint32_t)(QuadLayout<NB>::panel(V, G) * NB * 256);
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(a), "r"(n), "n"(IMM));
}

template <int NB, int G, int V>
__device__ __forceinline__ void quad_red2(uint32_t ap, uint32_t am, uint32_t n) {
  constexpr uint32_t IMM = kDsmemBase + (uint32_t)(QuadLayout<NB>::panel(V, G) * NB * 256);
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(ap), "r"(n), "n"(IMM));
  asm volatile("red.shared.add.u32 [%0+%2], %1;" ::"r"(am), "r"(n), "n"(IMM));
}

template <int NB, int G, int SP, int SM>
__device__ __forceinline__ void quad_entry_issue(uint32_t p0, uint32_t p1, uint32_t m0, uint32_t m1,
                                                 uint32_t c, uint32_t n) {
  // odd voxels of paired panels sit 32 columns (128 bytes) to the right
  const uint32_t co = QuadLayout<NB>::PP ? c + 128u : c;
  const uint32_t a0 = quad_prmt<0 + SP>(p0, p1, c), b0 = quad_prmt<0 + SM>(m0, m1, c);
  const uint32_t a1 = quad_prmt<1 + SP>(p0, p1, co), b1 = quad_prmt<1 + SM>(m0, m1, co);
  const uint32_t a2 = quad_prmt<2 + SP>(p0, p1, c), b2 = quad_prmt<2 + SM>(m0, m1, c);
  const uint32_t a3 = quad_prmt<3 + SP>(p0, p1, co), b3 = quad_prmt<3 + SM>(m0, m1, co);
#ifdef KB_PAIR_ORDER  // A/B knob: +o and -o atomics of a voxel back to back
  quad_red2<NB, G, 0>(a0, b0, n);
  quad_red2<NB, G, 1>(a1, b1, n);
  quad_red2<NB, G, 2>(a2, b2, n);
  quad_red2<NB, G, 3>(a3, b3, n);
#else
  // the +o atomics of the four voxels, then the -o ones: the two atomics of one
  // voxel hit the same word whenever bin(c+o) == bin(c-o) (homogeneous regions),
  // and back-to-back same-address atomics replay
  quad_red1<NB, G, 0>(a0, n);
  quad_red1<NB, G, 1>(a1, n);
  quad_red1<NB, G, 2>(a2, n);
  quad_red1<NB, G, 3>(a3, n);
  quad_red1<NB, G, 0>(b0, n);
  quad_red1<NB, G, 1>(b1, n);
  quad_red1<NB, G, 2>(b2, n);
  quad_red1<NB, G, 3>(b3, n);
#endif
}

// One int4 group = 4 table entries = 4 +-o pairs = 32 updates: all bin words
// are loaded first, then the PRMT/RED stream is issued.
template <int CLS>
struct QuadGroup {
  uint32_t p0[4], p1[4], m0[4], m1[4], n[4];
  __device__ __forceinline__ uint32_t ld(const uint8_t* p) { return lds32(p); }
  __device__ __forceinline__ void load(const uint8_t* tb, int4 w) {
    const int e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = e[k] >> 9;
      n[k] = (uint32_t)e[k] & 511u;
      const uint8_t* pp = tb + a;
      const uint8_t* pm = tb - a - (CLS ? 4 : 0);
      p0[k] = ld(pp);
      m0[k] = ld(pm);
      p1[k] = CLS ? ld(pp + 4) : 0u;
      m1[k] = CLS ? ld(pm + 4) : 0u;
    }
  }
};

template <int NB, int G, int CLS>
__device__ __forceinline__ void quad_issue(const QuadGroup<CLS>& q, uint32_t c) {
  constexpr int SP = CLS, SM = CLS == 1 ? 3 : CLS;  // byte shifts of +o and -o
#pragma unroll
  for (int k = 0; k < 4; ++k)
    quad_entry_issue<NB, G, SP, SM>(q.p0[k], q.p1[k], q.m0[k], q.m1[k], c, q.n[k]);
}

// A double = two x-adjacent offsets o1, o2 = o1 + (1,0,0) of the same radius
// run (and their mirrors -o1, -o2): the 4 voxels of a thread need bytes s..s+4
// of the +side words and bytes 3-s..7-s of the -side words, i.e. TWO words per
// side for EIGHT updates (a single needs one or two per four). Entry
// (a << 15) | ((n2 - n1 + 32) << 9) | n1, a = o1 - s; the -side words start at
// -a - 4. The representative is chosen so that s = o1.x mod 4 is 0 or 1 (the
// mirror of class 3 is class 0, of class 2 class 1).
template <int CLS>
struct QuadDbl {
  uint32_t p0[4], p1[4], m0[4], m1[4], n1[4], n2[4];
  __device__ __forceinline__ void load(const uint8_t* tb, int4 w) {
    const int e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = e[k] >> 15;
      n1[k] = (uint32_t)e[k] & 511u;
      n2[k] = n1[k] + (((uint32_t)e[k] >> 9) & 63u) - 32u;
      const uint8_t* pp = tb + a;
      const uint8_t* pm = tb - a - 4;
      p0[k] = lds32(pp);
      p1[k] = lds32(pp + 4);
      m0[k] = lds32(pm);
      m1[k] = lds32(pm + 4);
    }
  }
};

template <int NB, int G, int CLS>
__device__ __forceinline__ void quad_issue(const QuadDbl<CLS>& q, uint32_t c) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    quad_entry_issue<NB, G, CLS, 4 - CLS>(q.p0[k], q.p1[k], q.m0[k], q.m1[k], c, q.n1[k]);
    quad_entry_issue<NB, G, CLS + 1, 3 - CLS>(q.p0[k], q.p1[k], q.m0[k], q.m1[k], c, q.n2[k]);
  }
}

// One run of the doubles walk (any group type); the next group's table entries
// are fetched one iteration ahead, like quad_run (fetching two ahead and
// software-pipelining the bin-word loads were both measured slower, r01).
template <int NB, int G, class Q>
__device__ __forceinline__ void quad_run_t(const uint8_t* tb, uint32_t c, int g, int gend) {
  int4 w = c_offs[g];
#pragma unroll 1
  for (; g < gend; ++g) {
    const int4 wn = c_offs[g + 1];
    Q q;
    q.load(tb, w);
    quad_issue<NB, G>(q, c);
    w = wn;
  }
}

template <int NB, int G, int CLS>
__device__ __forceinline__ void quad_run(const uint8_t* tb, uint32_t c, int g, int gend) {
  // the next group's table entries are fetched one iteration ahead (the
  // constant-cache latency was the largest single stall); c_offs holds at
  // least one int4 past every run (make_plan), so the read never overruns
  int4 w = c_offs[g];
#pragma unroll 1
  for (; g < gend; ++g) {
    const int4 wn = c_offs[g + 1];
    QuadGroup<CLS> q;
    q.load(tb, w);
    quad_issue<NB, G, CLS>(q, c);
    w = wn;
  }
}

template <int NB, int G>
__device__ __noinline__ void quad_walk(const uint8_t* tb, uint32_t c, int g, int4 e) {
  quad_run<NB, G, 0>(tb, c, g, e.x);
  quad_run<NB, G, 1>(tb, c, e.x, e.y);
  quad_run<NB, G, 2>(tb, c, e.y, e.z);
}

template <int NB, int G>
__device__ __noinline__ void quad_walk_dbl(const uint8_t* tb, uint32_t c, int g, int4 e, int2 d) {
  quad_run_t<NB, G, QuadGroup<0>>(tb, c, g, e.x);
  quad_run_t<NB, G, QuadGroup<1>>(tb, c, e.x, e.y);
  quad_run_t<NB, G, QuadGroup<2>>(tb, c, e.y, e.z);
  quad_run_t<NB, G, QuadDbl<0>>(tb, c, e.z, d.x);
  quad_run_t<NB, G, QuadDbl<1>>(tb, c, d.x, d.y);
}

// DBL: singles + x-adjacent doubles (variant 4, the default) or singles only (3).
// VB: voxels per boundary iteration (1: one voxel's math at a time, the state
// rotating through slot 0; 2: two voxels' bins interleaved for ILP)
template <int NB, bool DBG, bool DBL, int VB = 1>
__global__ void __launch_bounds__(QuadLayout<NB>::NT, 1)
    kb_quad_kernel(const __grid_constant__ CUtensorMap tmap, const KbParams p) {
  using QL = QuadLayout<NB>;
  constexpr int TX = 16, TY = 8, TZ = QL::TZ, NT = QL::NT, NV = 4 * NT;
  constexpr int NS = NB - 1;  // snapshot bins (1..NB-1)
  constexpr int SL = QL::SL;  // TMEM columns per snapshot slot
  constexpr int PANEL = NB * 256;  // bytes: NB bins x 64 columns
  static_assert(NS % 8 == 0 && 8 * SL * (NT / 128) <= 512, "TMEM: 4 voxels x 2 slots x SL columns");
  static_assert(!QL::PP || VB == 1, "paired panels: one voxel per boundary iteration");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* hist = smem;  // 16 panels [v * 4 + G][bin][64 columns]
  uint8_t* tile = smem + NB * NV * 4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + ((p.tile_bytes + 15u) & ~15u));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int tx0, ty0, tz0;
  long long dbg_lin = -1;
  if (DBG) {
    dbg_lin = p.dbg_vox[blockIdx.x];
    const int vx = (int)(dbg_lin % p.nx);
    const int vy = (int)((dbg_lin / p.nx) % p.ny);
    const int vz = (int)(dbg_lin / ((long long)p.nx * p.ny));
    tx0 = vx / TX * TX;
    ty0 = vy / TY * TY;
    tz0 = p.zc0 + (vz - p.zc0) / TZ * TZ;
  } else {
    tx0 = blockIdx.x * TX;
    ty0 = blockIdx.y * TY;
    tz0 = p.zc0 + blockIdx.z * TZ;
    // a dependent chunk launched with programmatic serialization may take the
    // SMs this grid's tail frees (it reads nothing this grid writes)
    asm volatile("griddepcontrol.launch_dependents;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // all 512 TMEM columns: one CTA per SM (shared memory bound)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  const int xs = tx0 - p.R;
  const int xa = xs - (((xs % 16) + 16) % 16);
  const int delta = xs - xa;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(p.tile_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(tile)),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(xa), "r"(ty0 - p.R),
        "r"(tz0 - p.Rz - p.zs0), "r"(smem_u32(bar))
        : "memory");
  }
  {
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int i = tid; i < NB * NV / 4; i += NT) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0; selp.u32 %0, 1, 0, q; }"
          : "=r"(done)
          : "r"(smem_u32(bar))
          : "memory");
    }
  }
  __syncthreads();
  // thread -> 4 x-adjacent voxels; a warp covers 4 (x-quads) x 8 (y) of one z plane
  const int lx = 4 * (tid & 3), ly = (tid >> 2) & 7, lz = tid >> 5;
  const int gx = tx0 + lx, gy = ty0 + ly, gz = tz0 + lz;
  const bool rowv = gy < p.ny && gz < p.zc1;
  int dbg_v = -1;
  if (DBG && rowv)
    for (int v = 0; v < 4; ++v)
      if (gx + v < p.nx &&
          ((long long)(gx + v) + (long long)p.nx * ((long long)gy + (long long)p.ny * gz)) == dbg_lin)
        dbg_v = v;
  // (lx + R + delta) is a multiple of 4: R + delta = tx0 - xa = 0 (mod 16)
  const uint8_t* tb = tile + (lz + p.Rz) * p.SZ + (ly + p.R) * p.SY + (lx + p.R + delta);
  const int G = warp & 3, col = lane + 32 * (warp >> 2);
  const uint32_t hs0 = smem_u32(smem);
  if ((hs0 & 0xffffu) != kDsmemBase) __trap();  // the immediates below assume it
  const uint32_t cb = (hs0 & 0xffff0000u) | (4u * (uint32_t)col);  // bytes 0, 2, 3 of every address
  const uint32_t lane_base =
      tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(8 * SL * (warp >> 2));
  {  // zero all snapshot slots ("radius 0")
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 8 * SL; c += 8) tm_st8(lane_base + c, z);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  uint32_t TA[4] = {0u, 0u, 0u, 0u}, TB[4] = {0u, 0u, 0u, 0u};
  float Hb[4] = {0.f, 0.f, 0.f, 0.f};
  double best[4] = {0.0, 0.0, 0.0, 0.0};
  float best_s[4] = {0.f, 0.f, 0.f, 0.f};
  int best_rank[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
  int older = 0;  // which of the two slots (0/1) holds the older snapshot

  int g = 0;
  const bool warp_live = __any_sync(0xffffffffu, rowv && gx < p.nx);
  const int n_radii = warp_live ? p.n_radii : 0;
  {  // offset the two warps of each sub-partition so their radius boundaries
    // (little shared-pipe work) overlap the other warp's walk
    const int lag = p.lagmode == 1   ? warp * p.lag / 4
                    : p.lagmode == 3 ? (warp & 3) * p.lag / 8 + (warp >> 2) * p.lag
                                     : (warp >= 4 ? p.lag : 0);
    if (lag > 0) {
      const long long t0 = clock64();
      while (clock64() - t0 < lag) __nanosleep(256);
    }
  }
  for (int i = 0; i < n_radii; ++i) {
    const KbBound bd = c_bounds[i];
    const int4 e = c_qruns[i];
    if (DBL) {
      const int2 d = c_qruns2[i];
      switch (G) {  // warp-uniform; G = warp % 4 = the warp's SM sub-partition
        case 0: quad_walk_dbl<NB, 0>(tb, cb, g, e, d); break;
        case 1: quad_walk_dbl<NB, 1>(tb, cb, g, e, d); break;
        case 2: quad_walk_dbl<NB, 2>(tb, cb, g, e, d); break;
        default: quad_walk_dbl<NB, 3>(tb, cb, g, e, d); break;
      }
      g = d.y;
    } else {
      switch (G) {
        case 0: quad_walk<NB, 0>(tb, cb, g, e); break;
        case 1: quad_walk<NB, 1>(tb, cb, g, e); break;
        case 2: quad_walk<NB, 2>(tb, cb, g, e); break;
        default: quad_walk<NB, 3>(tb, cb, g, e); break;
      }
      g = e.z;
    }
    // ---- boundary: per voxel v, the same arithmetic as kb_tmem_kernel
    __syncwarp();
#ifdef KB_SKIP_BOUNDARY  // profiling knob: the walk alone (results are wrong)
    continue;
#endif
    // one copy of the per-voxel code (instruction cache: the unrolled 4-voxel
    // boundary was ~10k instructions, stall_no_instruction 7%): the per-voxel
    // state rotates through slot 0 and is back in place after the 4 voxels
    // The live columns of voxel v + 1 are loaded while voxel v's math runs
    // (their loads queue behind the other warps' atomics).
    if constexpr (VB == 2) {
      // two voxels per iteration: their columns, TMEM slots and per-bin terms are
      // independent, so the two chains interleave (the boundary is latency-bound)
#pragma unroll 1
      for (int vp = 0; vp < 4; vp += 2) {
        uint32_t cur[2][NS], T[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t* hc =
              reinterpret_cast<const uint32_t*>(hist + ((vp + u) * 4 + G) * PANEL) + col;
          T[u] = bd.W - hc[0];
#pragma unroll
          for (int j = 0; j < NS; ++j) cur[u][j] = hc[(1 + j) * 64];
        }
        bool doH[2], doE[2];
        float invT[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          doH[u] = (bd.flags & 1) && T[u] > 0u;
          doE[u] = (bd.flags & 2) && T[u] > 0u && TA[u] > 0u && TB[u] > 0u;
          invT[u] = doH[u] ? 1.0f / (float)T[u] : 0.f;
        }
        uint32_t a[2][NS];
        const uint32_t slot0 = lane_base + 64u * vp + (uint32_t)(32 * older);
        if constexpr (NS == 32) {
          tm_ld32(slot0, a[0]);
          tm_ld32(slot0 + 64u, a[1]);
        } else {
#pragma unroll
          for (int c = 0; c < NS; c += 8) {
            tm_ld8(slot0 + c, a[0] + c);
            tm_ld8(slot0 + 64u + c, a[1] + c);
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < NS; ++j) asm volatile("" : "+r"(a[u][j]));
        if constexpr (NS == 32) {
          tm_st32(slot0, cur[0]);
          tm_st32(slot0 + 64u, cur[1]);
        } else {
#pragma unroll
          for (int c = 0; c < NS; c += 8) {
            tm_st8(slot0 + c, cur[0] + c);
            tm_st8(slot0 + 64u + c, cur[1] + c);
          }
        }
        float hacc[2] = {0.f, 0.f};
        uint32_t dom[2] = {0u, 0u};
        unsigned long long num[2] = {0ull, 0ull};
        {
          const bool wH = bd.flags & 1, wE = bd.flags & 2;  // warp-uniform
          float h4[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          long long q[2][2] = {{0, 0}, {0, 0}};
          const int ta[2] = {(int)TA[0], (int)TA[1]}, nt[2] = {-(int)T[0], -(int)T[1]};
#pragma unroll
          for (int c = 0; c < NS; c += 8) {
            uint32_t orv = 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) orv |= cur[0][c + j] | cur[1][c + j];
            if (!__any_sync(0xffffffffu, orv != 0u)) continue;
#pragma unroll
            for (int j = c; j < c + 8; ++j) {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const uint32_t cv = cur[u][j];
#ifndef KB_SKIP_MATH
                if (wH) {
                  dom[u] = max(dom[u], cv);
                  h4[u][j & 3] -= ent_term((float)cv * invT[u]);
                }
#endif
#ifndef KB_SKIP_L1
                if (wE) l1_pos_acc(q[u][j & 1], (int)cv, ta[u], (int)a[u][j], nt[u]);
#endif
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (wH) hacc[u] = (h4[u][0] + h4[u][1]) + (h4[u][2] + h4[u][3]);
            if (doE[u]) num[u] = 2ull * (unsigned long long)(q[u][0] + q[u][1]);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (DBG && vp + u == dbg_v) {
            for (int j = 0; j < NS && j < p.bins; ++j)
              p.dbg_out[(size_t)i * (p.bins + 1) + j] = cur[u][j];
            p.dbg_out[(size_t)i * (p.bins + 1) + p.bins] = T[u];
          }
          if (doH[u] && 2u * dom[u] > T[u]) {  // dominant bin: its term again, accurately
            const float pb = (float)dom[u] * invT[u];
            hacc[u] += ent_term(pb);
            hacc[u] -= pb * (log1pf(-(float)(T[u] - dom[u]) * invT[u]) * 1.4426950408889634f);
          }
          if (doE[u]) {
            const double y = ((double)Hb[u] * bd.fac) *
                             ((double)num[u] * __drcp_rn((double)T[u] * (double)TA[u]));
            if (y > best[u] || (y == best[u] && y > 0.0 && bd.rank < best_rank[u])) {
              best[u] = y;
              best_s[u] = bd.scale;
              best_rank[u] = bd.rank;
            }
          }
          TA[u] = TB[u];
          TB[u] = T[u];
          Hb[u] = doH[u] ? fmaxf(hacc[u], 0.f) : 0.f;
        }
        rot4(TA), rot4(TB), rot4(Hb), rot4(best), rot4(best_s), rot4(best_rank);
        rot4(TA), rot4(TB), rot4(Hb), rot4(best), rot4(best_s), rot4(best_rank);
      }
    } else {
    uint32_t nxt[NS + 1];
    {
      const uint32_t* hc = reinterpret_cast<const uint32_t*>(hist + QL::panel(0, G) * PANEL) + col;
#pragma unroll
      for (int j = 0; j <= NS; ++j) nxt[j] = hc[j * 64];
    }
#pragma unroll 1
    for (int v = 0; v < 4; ++v) {
      // bin b of this voxel's column at hc[b * 64] (same panel as quad_red)
      uint32_t cur[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) cur[j] = nxt[1 + j];
      const uint32_t T = bd.W - nxt[0];
      if (v < 3) {
        const uint32_t* hn = reinterpret_cast<const uint32_t*>(hist + QL::panel(v + 1, G) * PANEL) +
                             col + QL::coloff(v + 1);
#pragma unroll
        for (int j = 0; j <= NS; ++j) nxt[j] = hn[j * 64];
      }
      const bool doH = (bd.flags & 1) && T > 0u;
      const bool doE = (bd.flags & 2) && T > 0u && TA[0] > 0u && TB[0] > 0u;
      const float invT = doH ? 1.0f / (float)T : 0.f;
      float hacc = 0.f;
      uint32_t dom = 0u;
      unsigned long long num = 0ull;
      const uint32_t slot = lane_base + (uint32_t)(2 * SL * v + SL * older);
      // one tcgen05.ld wait per voxel: the whole older slot and the live column
      // are fetched first; then the bins are reduced with independent partial
      // sums (the boundary was ~30% of the kernel's time with the serial,
      // branchy per-bin loop: KB_SKIP_BOUNDARY A/B, r01)
      uint32_t a[NS];
      if constexpr (NS == 32) {
        tm_ld32(slot, a);
      } else {
#pragma unroll
        for (int c = 0; c < NS; c += 8) tm_ld8(slot + c, a + c);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < NS; ++j) asm volatile("" : "+r"(a[j]));  // no use before the wait
      if constexpr (NS == 32) {
        tm_st32(slot, cur);  // the older slot becomes the newest
      } else {
#pragma unroll
        for (int c = 0; c < NS; c += 8) tm_st8(slot + c, cur + c);
      }
      {
        // per bin: the entropy term (radii that are scales) and the exact L1 term
        // (radii s+1), branch-free inside chunks of 8 bins; a chunk empty at r in
        // every lane of the warp is empty at r - 2 too (S_b grows with r) and
        // contributes nothing: one warp vote skips it (the high bins of a
        // mostly-background warp)
        const bool wH = bd.flags & 1, wE = bd.flags & 2;  // warp-uniform
        float h4[4] = {0.f, 0.f, 0.f, 0.f};
        long long q0 = 0, q1 = 0;  // all factors < 2^22: 32-bit signed operands, 64-bit products
        const int ta = (int)TA[0], nt = -(int)T;
#pragma unroll
        for (int c = 0; c < NS; c += 8) {
          uint32_t orv = 0u;
#pragma unroll
          for (int j = 0; j < 8; ++j) orv |= cur[c + j];
          if (!__any_sync(0xffffffffu, orv != 0u)) continue;
#pragma unroll
          for (int j = c; j < c + 8; ++j) {
            const uint32_t cv = cur[j];
#ifndef KB_SKIP_MATH
            if (wH) {
              dom = max(dom, cv);  // a bin with 2 S > T (at most one) is redone below
              h4[j & 3] -= ent_term((float)cv * invT);
            }
#endif
            // L1 numerator sum_b |S_b(hi) T_lo - S_b(lo) T_hi| exactly: the signed
            // terms sum to T_hi T_lo - T_lo T_hi = 0, so it is twice their positive part
#ifndef KB_SKIP_L1  // profiling knob (results wrong)
            if (wE) {
              if (j & 1) l1_pos_acc(q1, (int)cv, ta, (int)a[j], nt);
              else l1_pos_acc(q0, (int)cv, ta, (int)a[j], nt);
            }
#endif
          }
        }
        if (wH) hacc = (h4[0] + h4[1]) + (h4[2] + h4[3]);
        if (doE) num = 2ull * (unsigned long long)(q0 + q1);
      }
      if (DBG && v == dbg_v)
        for (int j = 0; j < NS && j < p.bins; ++j) p.dbg_out[(size_t)i * (p.bins + 1) + j] = cur[j];
      if (doH && 2u * dom > T) {  // dominant bin: its term again, accurately (log1p)
        const float pb = (float)dom * invT;
        hacc += ent_term(pb);
        hacc -= pb * (log1pf(-(float)(T - dom) * invT) * 1.4426950408889634f);
      }
      if (DBG && v == dbg_v) p.dbg_out[(size_t)i * (p.bins + 1) + p.bins] = T;
      if (doE) {
        // (reciprocal, not a correctly rounded division: y is compared within
        // the 1e-5 parity tolerance and stored as float)
        const double y = ((double)Hb[0] * bd.fac) * ((double)num * __drcp_rn((double)T * (double)TA[0]));
        if (y > best[0] || (y == best[0] && y > 0.0 && bd.rank < best_rank[0])) {
          best[0] = y;
          best_s[0] = bd.scale;
          best_rank[0] = bd.rank;
        }
      }
      TA[0] = TB[0];
      TB[0] = T;
      Hb[0] = doH ? fmaxf(hacc, 0.f) : 0.f;
      rot4(TA);
      rot4(TB);
      rot4(Hb);
      rot4(best);
      rot4(best_s);
      rot4(best_rank);
    }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // before the next radius' loads
    older ^= 1;
  }
  if (!DBG && rowv) {
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if (gx + v < p.nx) {
        const size_t o = ((size_t)(gz - p.zc0) * p.ny + gy) * p.nx + gx + v;
        p.score[o] = (float)best[v];
        p.best[o] = best_s[v];
      }
    if (gz >= p.hz0 && gz < p.hz1) {  // mapped pinned host maps (hz0 == hz1: none)
      const size_t h = ((size_t)(gz - p.hz0) * p.ny + gy) * p.nx + gx;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (gx + v < p.nx) {
          if (p.h_score) p.h_score[h + v] = (float)best[v];
          if (p.h_best) p.h_best[h + v] = best_s[v];
        }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
  // launched as a programmatic dependent: complete only after the preceding
  // grid has, so work ordered after this grid also follows that one (no-op otherwise)
  if (!DBG) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ----------------------------------------------------------------------------- K3
__global__ void maxima_kernel(const float* __restrict__ score, int nx, int ny, int nz, int zc0,
                              int z0, int z1, unsigned long long* keys, unsigned int* counter) {
  const long long rows = (long long)ny * (z1 - z0);
  const unsigned lane = threadIdx.x & 31u;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const int y = (int)(row % ny);
    const int z = z0 + (int)(row / ny);
    // every lane of a warp runs the same trips (blockDim is a multiple of 32), so
    // the maxima of a warp take ONE counter atomic (the counter was the hot spot)
    for (int xb = 0; xb < nx; xb += blockDim.x) {
      const int x = xb + (int)threadIdx.x;
      const float s0 = x < nx ? score[((size_t)(z - zc0) * ny + y) * nx + x] : 0.0f;
      bool is_max = s0 > 0.0f;
      for (int dz = -1; dz <= 1 && is_max; ++dz) {
        const int sz = z + dz;
        if (sz < 0 || sz >= nz) continue;
        for (int dy = -1; dy <= 1 && is_max; ++dy) {
          const int sy = y + dy;
          if (sy < 0 || sy >= ny) continue;
          const float* r = score + ((size_t)(sz - zc0) * ny + sy) * nx;
          for (int dx = -1; dx <= 1; ++dx) {
            const int sx = x + dx;
            if ((dx | dy | dz) == 0 || sx < 0 || sx >= nx) continue;
            if (r[sx] >= s0) {
              is_max = false;
              break;
            }
          }
        }
      }
      const unsigned found = __ballot_sync(0xffffffffu, is_max);
      if (found == 0u) continue;
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(counter, (unsigned)__popc(found));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (is_max) {
        const unsigned long long lin =
            (unsigned long long)x + (unsigned long long)nx * ((unsigned long long)y + (unsigned long long)ny * z);
        keys[base + __popc(found & ((1u << lane) - 1u))] =
            ((unsigned long long)(~__float_as_uint(s0)) << 32) | (lin & 0xffffffffull);
      }
    }
  }
}

// The same strict 26-neighbour test, tiled: a CTA owns a 32 x 8 column block
// and walks a run of planes, keeping planes z-1, z, z+1 (+ a one-voxel halo) in a
// shared-memory ring while plane z+2 is in flight in registers, so every score
// is read from L2/HBM ~1.3 times instead of up to 27 times and the load latency
// overlaps the tests. Out-of-volume neighbours are -inf (they never kill).
#ifndef MX_Z  // A/B knob: planes per CTA of the maxima pass
#define MX_Z 16
#endif
constexpr int kMxTX = 32, kMxTY = 8, kMxZ = MX_Z;
constexpr int kMxPl = (kMxTY + 2) * (kMxTX + 2);  // one plane with its halo
constexpr int kMxPer = (kMxPl + kMxTX * kMxTY - 1) / (kMxTX * kMxTY);  // elements per thread
__global__ void __launch_bounds__(kMxTX * kMxTY)
    maxima_tile_kernel(const float* __restrict__ score, int nx, int ny, int nz, int zc0, int z0,
                       int z1, unsigned long long* keys, unsigned int* counter) {
  __shared__ float pl[4][kMxTY + 2][kMxTX + 2];  // ring: z-1, z, z+1 and the plane in flight
  // the CTA's maxima are gathered here and published with ONE global atomic: a
  // single counter hit once per warp-step serialised the pass (~400k atomics).
  // At most one strict maximum per 2x2x2 cube of the block: 32*8*16/8 slots.
  __shared__ unsigned long long ckeys[kMxTX * kMxTY * kMxZ / 8];
  __shared__ unsigned int ccount, cbase;
  if (threadIdx.x == 0) ccount = 0u;
  const int tx = threadIdx.x & (kMxTX - 1), ty = threadIdx.x / kMxTX;
  const int x0 = blockIdx.x * kMxTX, y0 = blockIdx.y * kMxTY;
  const int za = z0 + blockIdx.z * kMxZ, zb = min(z1, za + kMxZ);
  const unsigned lane = threadIdx.x & 31u;
  if (za >= zb) return;
  float reg[kMxPer];
  auto fetch = [&](int z) {  // this thread's elements of plane z (+ halo) into registers
#pragma unroll
    for (int k = 0; k < kMxPer; ++k) {
      const int i = threadIdx.x + k * kMxTX * kMxTY;
      const int ly = i / (kMxTX + 2), lx = i - ly * (kMxTX + 2);
      const int x = x0 + lx - 1, y = y0 + ly - 1;
      float v = -INFINITY;
      if (i < kMxPl && z >= 0 && z < nz && x >= 0 && x < nx && y >= 0 && y < ny)
        v = score[((size_t)(z - zc0) * ny + y) * nx + x];
      reg[k] = v;
    }
  };
  auto store = [&](int slot) {
#pragma unroll
    for (int k = 0; k < kMxPer; ++k) {
      const int i = threadIdx.x + k * kMxTX * kMxTY;
      if (i < kMxPl) (&pl[slot][0][0])[i] = reg[k];
    }
  };
  fetch(za - 1);
  store((za - 1 - za + 4) & 3);
  fetch(za);
  store(0);
  fetch(za + 1);
  store(1);
  __syncthreads();
  const int x = x0 + tx, y = y0 + ty;
  for (int z = za; z < zb; ++z) {
    const int r = z - za;
    if (z + 1 < zb) fetch(z + 2);  // in flight while plane z is tested
    const int s_lo = (r + 3) & 3, s_c = r & 3, s_hi = (r + 1) & 3;
    const float s0 = pl[s_c][ty + 1][tx + 1];
    bool is_max = x < nx && y < ny && s0 > 0.0f;
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
      const int sl = dz == 0 ? s_lo : (dz == 1 ? s_c : s_hi);
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
          if (!(dz == 1 && dy == 1 && dx == 1) && pl[sl][ty + dy][tx + dx] >= s0) is_max = false;
    }
    const unsigned found = __ballot_sync(0xffffffffu, is_max);
    if (found != 0u) {
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(&ccount, (unsigned)__popc(found));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (is_max) {
        const unsigned long long lin =
            (unsigned long long)x + (unsigned long long)nx * ((unsigned long long)y + (unsigned long long)ny * z);
        ckeys[base + __popc(found & ((1u << lane) - 1u))] =
            ((unsigned long long)(~__float_as_uint(s0)) << 32) | (lin & 0xffffffffull);
      }
    }
    if (z + 1 < zb) store((r + 2) & 3);  // slot of z - 2: no longer read
    __syncthreads();
  }
  if (threadIdx.x == 0) cbase = ccount ? atomicAdd(counter, ccount) : 0u;
  __syncthreads();
  for (unsigned i = threadIdx.x; i < ccount; i += kMxTX * kMxTY) keys[cbase + i] = ckeys[i];
}

__global__ void decode_maxima_kernel(const unsigned long long* __restrict__ keys, long long n,
                                     const float* __restrict__ best, int nx, int ny, int zc0,
                                     salvox_maximum* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const unsigned long long lin = k & 0xffffffffull;
    const float s = __uint_as_float(~(uint32_t)(k >> 32));
    const int x = (int)(lin % nx);
    const int y = (int)((lin / nx) % ny);
    const int z = (int)(lin / ((unsigned long long)nx * ny));
    salvox_maximum m;
    m.position[0] = x;
    m.position[1] = y;
    m.position[2] = z;
    m.score = (double)s;
    m.scale = (double)best[((size_t)(z - zc0) * ny + y) * nx + x];
    m.linear_index = (long long)lin;
    out[i] = m;
  }
}

// ------------------------------------------------------------------------ host plan
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  if (!fn) fail(SALVOX_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

struct TileCfg {
  int nb, tx, ty, tz;
  bool pair;          // kb_pair_kernel (two voxels per thread, tx = 8)
  bool tmem = false;  // kb_tmem_kernel (1024 threads, snapshots in TMEM)
  bool quad = false;  // kb_quad_kernel (256 threads x 4 voxels -- 128 at 65 bins -- snapshots in TMEM)
  bool dbl = false;  // kb_quad_kernel<DBL>: x-adjacent offset doubles share bin words
  bool vb2 = false;  // kb_quad_kernel<.., VB = 2>: two voxels per boundary iteration
  bool epa = false;  // kb_kernel<.., EPA>: Epanechnikov, 64-bit count|sum words
};

TileCfg pick_tile(int bins, bool two_d, bool epa = false) {
  const int nb = bins <= 16 ? 17 : (bins <= 32 ? 33 : 65);
  // 3D, 65 bins (A/B knob SALVOX_KB65): "quad" (default) kb_quad_kernel<65> with
  // paired-voxel panels, 128 threads; "tmem" kb_tmem_kernel<65, 512 threads>;
  // "kb" the 8x8x4 kb_kernel
  static const int kb65 = [] {
    const char* e = std::getenv("SALVOX_KB65");
    if (e && std::string(e) == "kb") return 2;
    if (e && std::string(e) == "tmem") return 1;
    return 0;
  }();
  if (nb == 65 && !two_d && !epa && kb65 == 0)
    return TileCfg{65, 16, 8, 4, false, false, true, true, false};
  if (nb == 65 && !two_d && !epa && kb65 == 1)
    return TileCfg{65, 16, 8, 4, false, true};  // kb_tmem_kernel<65, 512 threads>
  if (epa) {  // the plain kb_kernel tiles (64-bit words: 2x the histogram bytes)
    TileCfg t = nb == 65 ? (two_d ? TileCfg{65, 32, 8, 1, false} : TileCfg{65, 8, 8, 4, false})
                         : (two_d ? TileCfg{nb, 32, 16, 1, false} : TileCfg{nb, 8, 8, 8, false});
    t.epa = true;
    return t;
  }
  if (nb == 65) return two_d ? TileCfg{65, 32, 8, 1, false} : TileCfg{65, 8, 8, 4, false};
  // Variants (A/B knob SALVOX_KB_VARIANT; measured at C2 on one B200, r01):
  //   4 (default, 3D): kb_quad_kernel<DBL> -- as 3, plus x-adjacent offset
  //      doubles of a radius run share their bin words (2 words per side for 8
  //      updates): bin-word wavefronts 4.21e9 -> 3.05e9 per launch, 64.1 ms
  //   3: kb_quad_kernel -- 256 threads x 4 voxels, 4 bins per
  //      32-bit word, one PRMT per update builds the atomic's address, snapshots
  //      in TMEM: 65.6 ms (1.53 smem wavefronts per update; latency-bound on
  //      8 warps/SM, issue active ~49%)
  //   2: kb_tmem_kernel -- 1024 threads, snapshots in TMEM, 70.7 ms (2.03
  //      wavefronts per update, shared pipe 94.5%: the LDS+ATOMS pair bound)
  //   0: kb_kernel -- 512 threads, snapshots in registers, 80.2 ms (2D default)
  //   1: kb_pair_kernel -- 2 voxels/thread, 25% fewer smem wavefronts but 247
  //      registers -> 8 warps/SM, latency-bound, 85.9 ms
  static const int mode = [] {
    const char* e = std::getenv("SALVOX_KB_VARIANT");
    return e ? std::atoi(e) : 4;
  }();
  if (mode == 1) return two_d ? TileCfg{nb, 8, 64, 1, true} : TileCfg{nb, 8, 8, 8, true};
  if (mode == 2 && !two_d) return TileCfg{nb, 16, 8, 8, false, true};
  if (mode == 3 && !two_d) return TileCfg{nb, 16, 8, 8, false, false, true};
  static const bool vb2 = [] {  // A/B knob SALVOX_KB_VB (1 or 2)
    const char* e = std::getenv("SALVOX_KB_VB");
    return e && std::atoi(e) == 2;
  }();
  if (mode == 4 && !two_d) return TileCfg{nb, 16, 8, 8, false, false, true, true, vb2};
  return two_d ? TileCfg{nb, 32, 16, 1, false} : TileCfg{nb, 8, 8, 8, false};
}

// kb_quad_kernel: warps 4-7 start their walk ~4 us late, so each sub-partition's
// two warps reach their radius boundaries (entropy/L1 math, TMEM snapshots:
// little shared-pipe work) at different times and the other warp keeps the
// atomics flowing. C2 sweeps (r01, cycles -> ms): 0 53.1, 4k 53.1, 10k 52.0,
// 20k 51.1, 40k 51.3; after the boundary rework: 0 51.7, 12k 49.5, 20k 49.8,
// 28k 50.0; final: 0 51.3, 4k 49.5, 6k 49.15, 8k 49.02, 10k 49.09, 12k 49.18.
// A/B knob SALVOX_KB_LAG.
int kb_lag() {
  static const int lag = [] {
    const char* e = std::getenv("SALVOX_KB_LAG");
    return e ? std::atoi(e) : 8000;
  }();
  return lag;
}
int kb_lagmode() {  // A/B knob SALVOX_KB_LAGMODE (see KbParams::lagmode)
  static const int m = [] {
    const char* e = std::getenv("SALVOX_KB_LAGMODE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// Dynamic shared memory of one CTA: histogram columns, tile(s), mbarrier.
size_t kb_smem(const TileCfg& tc, uint32_t tile_bytes) {
  const size_t voxels = (size_t)tc.tx * tc.ty * tc.tz;
  if (tc.pair)
    return (size_t)tc.nb * voxels * 4 + 2 * (((size_t)tile_bytes + 127) & ~(size_t)127) + 16;
  if (tc.tmem || tc.quad)
    return (size_t)tc.nb * voxels * 4 + (((size_t)tile_bytes + 15) & ~(size_t)15) + 32;
  return (size_t)tc.nb * voxels * (tc.epa ? 8 : 4) + (((size_t)tile_bytes + 15) & ~(size_t)15) + 16;
}

// Offsets of make_sphere_offsets (pipeline.cpp:37-52) for every needed radius,
// as one |o|^2-sorted table of +-o representatives with per-radius prefix ends.
struct Plan {
  std::vector<double> radii;
  std::vector<KbBound> bounds;
  std::vector<int32_t> offs;    // +-o representatives (tile offsets), grouped by level
  std::vector<KbLevel> levels;  // |o|^2 levels in increasing order
  std::vector<uint64_t> ball_size;  // |B(r_i)| incl. centre (EvalCounter, :118)
  std::vector<int32_t> qtab;  // kb_quad_kernel: (a << 9) | n per +-o pair, (radius, class) runs
  std::vector<int4> qruns;    // kb_quad_kernel: per radius, the three run ends (int4 groups)
  std::vector<int2> qruns2;   // kb_quad_kernel<DBL>: per radius, the two doubles run ends
  int R = 0;
};

bool member(int x, int y, int z, double r) {  // pipeline.cpp:39-46
  const int ri = (int)std::floor(r);
  if (std::abs(x) > ri || std::abs(y) > ri || std::abs(z) > ri) return false;
  const double d = ((double)x * x + (double)y * y + (double)z * z) / (r * r);
  return d <= 1.0;
}

Plan make_plan(const double* scales, int n_scales, bool two_d, const TileCfg& tc, int* SYo,
               int* SZo) {
  Plan pl;
  for (int i = 0; i < n_scales; ++i) {
    pl.radii.push_back(scales[i] - 1.0);
    pl.radii.push_back(scales[i]);
    pl.radii.push_back(scales[i] + 1.0);
  }
  std::sort(pl.radii.begin(), pl.radii.end());
  pl.radii.erase(std::unique(pl.radii.begin(), pl.radii.end()), pl.radii.end());
  const int NR = (int)pl.radii.size();
  if (NR > kMaxRadii) fail(SALVOX_EUNSUPPORTED, "exhaustive (device): too many radii");
  const double rmax = pl.radii.back();
  pl.R = (int)std::floor(rmax);
  if (pl.R > 16)
    fail(SALVOX_EUNSUPPORTED,
         "exhaustive (device): max scale + 1 must be <= 16 voxels (shared-memory halo)");
  const int R = pl.R;
  int dmax = 0;  // worst shift of the 16-byte-aligned box start (see kb_kernel)
  for (int k = 0; k < 16; ++k) dmax = std::max(dmax, (((tc.tx * k - R) % 16) + 16) % 16);
  int BX = ((tc.tx + 2 * R + dmax) + 15) / 16 * 16;
  if (tc.pair) BX = 48;  // 12-word pitch: conflict-free 8-row warp footprint (kb_pair_kernel)
  if (tc.tx + 2 * R + dmax > BX) fail(SALVOX_EUNSUPPORTED, "exhaustive (device): halo too wide");
  const int BY = tc.ty + 2 * R;
  const int SY = BX, SZ = BX * BY;
  *SYo = SY;
  *SZo = SZ;
  const int zr = two_d ? 0 : R;
  struct Off {
    int x, y, z, n;
  };
  std::vector<Off> cand;
  for (int z = -zr; z <= zr; ++z)
    for (int y = -R; y <= R; ++y)
      for (int x = -R; x <= R; ++x)
        if ((x | y | z) != 0 && member(x, y, z, rmax)) cand.push_back({x, y, z, x * x + y * y + z * z});
  std::stable_sort(cand.begin(), cand.end(), [](const Off& a, const Off& b) { return a.n < b.n; });
  // per radius: membership must be the |o|^2-prefix {n <= N_i}
  std::vector<int> Nmax(NR, 0);
  pl.ball_size.assign(NR, 1);
  for (int i = 0; i < NR; ++i) {
    int nm = 0;
    for (const Off& o : cand)
      if (member(o.x, o.y, o.z, pl.radii[i])) {
        nm = std::max(nm, o.n);
        pl.ball_size[i]++;
      }
    for (const Off& o : cand) {
      const bool m = member(o.x, o.y, o.z, pl.radii[i]);
      if (m != (o.n <= nm))
        fail(SALVOX_EUNSUPPORTED, "exhaustive (device): radius set is not |o|^2-nested");
    }
    Nmax[i] = nm;
  }
  // ring of 3: every scale's s-1, s, s+1 must be adjacent radii
  auto idx = [&](double r) {
    return (int)(std::lower_bound(pl.radii.begin(), pl.radii.end(), r) - pl.radii.begin());
  };
  std::vector<int> eval_rank(NR, INT_MAX);
  std::vector<bool> is_scale(NR, false);
  for (int k = 0; k < n_scales; ++k) {
    const double s = scales[k];
    const int il = idx(s - 1.0), ic = idx(s), ih = idx(s + 1.0);
    if (ic != il + 1 || ih != ic + 1)
      fail(SALVOX_EUNSUPPORTED,
           "exhaustive (device): scales need adjacent s-1, s, s+1 radii (integer scales)");
    is_scale[ic] = true;
    eval_rank[ih] = std::min(eval_rank[ih], k);
  }
  size_t c = 0;
  uint32_t W = 0;  // running sum of |o|^2 over all members (both signs)
  for (int i = 0; i < NR; ++i) {
    while (c < cand.size() && cand[c].n <= Nmax[i]) {  // one |o|^2 level
      const int n = cand[c].n;
      std::vector<int> lists[2];
      for (; c < cand.size() && cand[c].n == n; ++c) {
        const Off& o = cand[c];
        W += (uint32_t)o.n;
        const bool rep = o.z > 0 || (o.z == 0 && (o.y > 0 || (o.y == 0 && o.x > 0)));
        if (!rep) continue;
        lists[tc.pair ? (o.x & 1) : 0].push_back(o.z * SZ + o.y * SY + o.x);
      }
      KbLevel L{};
      L.n = n;
      for (int k = 0; k < 2; ++k) {
        const int st = (int)pl.offs.size();
        for (int v : lists[k]) pl.offs.push_back(v);
        while (pl.offs.size() % 4) pl.offs.push_back(0);  // next list starts 16-byte aligned
        if (k == 0) {
          L.start0 = st;
          L.count0 = (int16_t)lists[0].size();
        } else {
          L.start1 = st;
          L.count1 = (int16_t)lists[1].size();
        }
      }
      pl.levels.push_back(L);
    }
    KbBound b{};
    b.lend = (int)pl.levels.size();
    b.W = W;
    b.cnt = (uint32_t)pl.ball_size[i];
    {
      const double r2 = pl.radii[i] * pl.radii[i];
      if (r2 == std::floor(r2)) {
        b.q = 1;
        b.r2q = (uint32_t)r2;
      } else if (4.0 * r2 == std::floor(4.0 * r2)) {
        b.q = 4;
        b.r2q = (uint32_t)(4.0 * r2);
      }
    }
    b.flags = (is_scale[i] ? 1 : 0) | (eval_rank[i] != INT_MAX ? 2 : 0);
    if (eval_rank[i] != INT_MAX) {
      const double s = pl.radii[i - 1];
      b.rank = eval_rank[i];
      b.scale = (float)s;
      b.fac = s * s / 2.0;
    }
    pl.bounds.push_back(b);
  }
  if ((int)pl.offs.size() > kMaxOffs || (int)pl.levels.size() > kMaxLevels)
    fail(SALVOX_EUNSUPPORTED, "exhaustive (device): offset table too large");
  // flat form for kb_quad_kernel: per radius, three runs of (a << 9) | n, one per
  // class s = o.x mod 4 in {0, 1, 2} of the pair's representative (-o when
  // o.x = 3 mod 4), a = o - s the 4-aligned byte offset of +o's first word;
  // each run padded to whole int4 groups with zero-weight entries
  {
    int lv = 0;
    for (KbBound& b : pl.bounds) {
      std::vector<int32_t> runs[3];
      for (; lv < b.lend; ++lv) {
        const KbLevel& L = pl.levels[lv];
        for (int k = 0; k < L.count0 + L.count1; ++k) {
          int o = k < L.count0 ? pl.offs[L.start0 + k] : pl.offs[L.start1 + k - L.count0];
          if ((o & 3) == 3) o = -o;
          const int s = o & 3;
          runs[s].push_back((int32_t)((uint32_t)(o - s) << 9) | L.n);
        }
      }
      int4 e{};
      for (int s = 0; s < 3; ++s) {
        for (int32_t v : runs[s]) pl.qtab.push_back(v);
        while (pl.qtab.size() % 4) pl.qtab.push_back(0);
        (s == 0 ? e.x : s == 1 ? e.y : e.z) = (int)(pl.qtab.size() / 4);
      }
      pl.qruns.push_back(e);
    }
  }
  // kb_quad_kernel<DBL>: per radius, the representatives are grouped by row
  // (z, y); each row's contiguous x segments are cut into x-adjacent doubles
  // (an odd segment leaves one single, at an x = 0 mod 4 position when it can).
  // Singles keep the three class runs above, doubles get two more (classes 0, 1).
  if (tc.dbl) {
    pl.qtab.clear();
    pl.qruns.clear();
    size_t c2 = 0;
    for (int i = 0; i < NR; ++i) {
      std::map<std::pair<int, int>, std::vector<int>> rows;  // (z, y) -> x
      for (; c2 < cand.size() && cand[c2].n <= Nmax[i]; ++c2) {
        const Off& o = cand[c2];
        if (o.z > 0 || (o.z == 0 && (o.y > 0 || (o.y == 0 && o.x > 0))))
          rows[{o.z, o.y}].push_back(o.x);
      }
      std::vector<int32_t> runs[5];
      for (auto& kv : rows) {
        const int z = kv.first.first, y = kv.first.second;
        std::vector<int>& xs = kv.second;
        std::sort(xs.begin(), xs.end());
        auto single = [&](int x) {
          int o = z * SZ + y * SY + x;
          if ((o & 3) == 3) o = -o;
          const int s = o & 3;
          runs[s].push_back((int32_t)((uint32_t)(o - s) << 9) | (x * x + y * y + z * z));
        };
        auto dbl = [&](int x) {  // o1 = (x, y, z), o2 = (x + 1, y, z)
          int o1 = z * SZ + y * SY + x;
          int n1 = x * x + y * y + z * z, n2 = n1 + 2 * x + 1;
          if ((o1 & 3) >= 2) {  // mirror: (-o2, -o1), class 3 - s
            o1 = -(o1 + 1);
            std::swap(n1, n2);
          }
          const int s = o1 & 3;
          runs[3 + s].push_back((int32_t)((uint32_t)(o1 - s) << 15) |
                                ((n2 - n1 + 32) << 9) | n1);
        };
        size_t a = 0;
        while (a < xs.size()) {
          size_t b = a + 1;
          while (b < xs.size() && xs[b] == xs[b - 1] + 1) ++b;
          size_t one = SIZE_MAX;
          if ((b - a) % 2) {
            one = a;
            for (size_t k = a; k < b; k += 2)
              if ((xs[k] & 3) == 0) {
                one = k;
                break;
              }
          }
          for (size_t k = a; k < b;) {
            if (k == one) {
              single(xs[k]);
              ++k;
            } else {
              dbl(xs[k]);
              k += 2;
            }
          }
          a = b;
        }
      }
      int4 e{};
      int2 d{};
      for (int s = 0; s < 5; ++s) {
        for (int32_t v : runs[s]) pl.qtab.push_back(v);
        while (pl.qtab.size() % 4) pl.qtab.push_back(s < 3 ? 0 : (32 << 9));  // zero weight
        const int end = (int)(pl.qtab.size() / 4);
        if (s == 0) e.x = end; else if (s == 1) e.y = end; else if (s == 2) e.z = end;
        else if (s == 3) d.x = end; else d.y = end;
      }
      pl.qruns.push_back(e);
      pl.qruns2.push_back(d);
    }
  }
  // too large (two int4 of slack for kb_quad_kernel's look-ahead): not used
  if ((int)pl.qtab.size() + 8 > kMaxOffs) pl.qtab.clear(), pl.qruns.clear(), pl.qruns2.clear();
  return pl;
}

// The constant-memory tables are module-global: serialise their reuse across
// streams with an event recorded after each consuming launch.
std::mutex g_const_mu;
cudaEvent_t g_const_done = nullptr;

template <int NB, int TX, int TY, int TZ, bool DBG, bool EPA = false>
void launch_kb(salvox_ctx* ctx, const CUtensorMap& map, const KbParams& kp, dim3 grid,
               size_t smem) {
  auto k = kb_kernel<NB, TX, TY, TZ, DBG, EPA>;
  SX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, TX * TY * TZ, smem, ctx->stream>>>(map, kp);
  SX_LAUNCH_CHECK(ctx);
}

// pdl: launch kb_quad_kernel with programmatic stream serialization (its CTAs
// may start while the preceding KB grid's last wave drains); other variants ignore it
template <bool DBG>
void dispatch_kb(salvox_ctx* ctx, const TileCfg& tc, const CUtensorMap& map, const KbParams& kp,
                 dim3 grid, size_t smem, bool pdl = false) {
#define SX_KB(NB, TX, TY, TZ)                                             \
  if (!tc.pair && !tc.tmem && !tc.quad && tc.nb == NB && tc.tx == TX && tc.ty == TY && tc.tz == TZ) { \
    if (tc.epa) {                                                         \
      if (DBG) fail(SALVOX_EUNSUPPORTED, "exhaustive debug: identity kernel only"); \
      launch_kb<NB, TX, TY, TZ, false, true>(ctx, map, kp, grid, smem);   \
    } else {                                                              \
      launch_kb<NB, TX, TY, TZ, DBG>(ctx, map, kp, grid, smem);           \
    }                                                                     \
    return;                                                               \
  }
  SX_KB(17, 8, 8, 8)
  SX_KB(33, 8, 8, 8)
  SX_KB(65, 8, 8, 4)
  SX_KB(17, 32, 16, 1)
  SX_KB(33, 32, 16, 1)
  SX_KB(65, 32, 8, 1)
#undef SX_KB
#define SX_KP(NB, TY, TZ)                                                                    \
  if (tc.pair && tc.nb == NB && tc.ty == TY && tc.tz == TZ) {                                \
    auto k = kb_pair_kernel<NB, TY, TZ, DBG>;                                                \
    SX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<grid, 4 * TY * TZ, smem, ctx->stream>>>(map, kp);                                    \
    SX_LAUNCH_CHECK(ctx);                                                                    \
    return;                                                                                  \
  }
  if (tc.quad) {
    auto k = tc.nb == 65 ? (tc.dbl ? kb_quad_kernel<65, DBG, true, 1> : kb_quad_kernel<65, DBG, false, 1>)
           : tc.dbl ? (tc.nb == 17 ? (tc.vb2 ? kb_quad_kernel<17, DBG, true, 2> : kb_quad_kernel<17, DBG, true, 1>)
                                   : (tc.vb2 ? kb_quad_kernel<33, DBG, true, 2> : kb_quad_kernel<33, DBG, true, 1>))
                    : (tc.nb == 17 ? kb_quad_kernel<17, DBG, false> : kb_quad_kernel<33, DBG, false>);
    const int threads = tc.nb == 65 ? QuadLayout<65>::NT : 256;
    SX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (pdl && !DBG) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      SX_CUDA(cudaLaunchKernelEx(&cfg, k, map, kp));
    } else {
      k<<<grid, threads, smem, ctx->stream>>>(map, kp);
    }
    SX_LAUNCH_CHECK(ctx);
    return;
  }
  if (tc.tmem && tc.nb == 65) {
    auto k = kb_tmem_kernel<65, DBG, 512>;
    SX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 512, smem, ctx->stream>>>(map, kp);
    SX_LAUNCH_CHECK(ctx);
    return;
  }
  if (tc.tmem) {
    auto k = tc.nb == 17 ? kb_tmem_kernel<17, DBG> : kb_tmem_kernel<33, DBG>;
    SX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 1024, smem, ctx->stream>>>(map, kp);
    SX_LAUNCH_CHECK(ctx);
    return;
  }
  SX_KP(17, 8, 8)
  SX_KP(33, 8, 8)
  SX_KP(17, 64, 1)
  SX_KP(33, 64, 1)
#undef SX_KP
  fail(SALVOX_EUNSUPPORTED, "exhaustive (device): no kernel for this tile configuration");
}

struct ExhRun {
  TileCfg tc;
  Plan pl;
  CUtensorMap map;
  KbParams kp;  // kp.zc0 / zc1: the planes the KB kernel scores
  dim3 grid;
  size_t smem;
  // the score / best-scale buffers cover planes [zb0, zb1) = the owned planes
  // plus one neighbour plane each side; without the exchange (the default) the
  // kernel scores all of them, with it only the owned planes and the caller
  // supplies the neighbour planes (salvox_exhaustive_slab_maxima)
  int zb0 = 0, zb1 = 0, z0 = 0, z1 = 0;
  float* score_base = nullptr;
  float* best_base = nullptr;
  bool exch = false;
  uint64_t generation = 0;  // ctx->exh_generation when this run was set up
};

void upload_tables(salvox_ctx* ctx, const Plan& pl, bool quad = false) {
  if (!g_const_done) SX_CUDA(cudaEventCreateWithFlags(&g_const_done, cudaEventDisableTiming));
  SX_CUDA(cudaStreamWaitEvent(ctx->stream, g_const_done, 0));
  if (quad) {  // kb_quad_kernel reads the flat weighted table from the same symbol
    SX_CUDA(cudaMemcpyToSymbolAsync(c_offs, pl.qtab.data(), pl.qtab.size() * 4, 0,
                                    cudaMemcpyHostToDevice, ctx->stream));
    SX_CUDA(cudaMemcpyToSymbolAsync(c_qruns, pl.qruns.data(), pl.qruns.size() * sizeof(int4), 0,
                                    cudaMemcpyHostToDevice, ctx->stream));
    if (!pl.qruns2.empty())
      SX_CUDA(cudaMemcpyToSymbolAsync(c_qruns2, pl.qruns2.data(), pl.qruns2.size() * sizeof(int2),
                                      0, cudaMemcpyHostToDevice, ctx->stream));
  } else
    SX_CUDA(cudaMemcpyToSymbolAsync(c_offs, pl.offs.data(), pl.offs.size() * 4, 0,
                                    cudaMemcpyHostToDevice, ctx->stream));
  SX_CUDA(cudaMemcpyToSymbolAsync(c_levels, pl.levels.data(), pl.levels.size() * sizeof(KbLevel),
                                  0, cudaMemcpyHostToDevice, ctx->stream));
  SX_CUDA(cudaMemcpyToSymbolAsync(c_bounds, pl.bounds.data(), pl.bounds.size() * sizeof(KbBound),
                                  0, cudaMemcpyHostToDevice, ctx->stream));
}

void validate_exhaustive(int nx, int ny, int nz, const salvox_window* iw, const double* scales,
                         int n_scales, int kernel, uint64_t budget) {
  if (nx < 1 || ny < 1 || nz < 1) fail(SALVOX_EINVAL, "Volume: dims must be >= 1");
  if (!iw) fail(SALVOX_EINVAL, "IntensityWindow: missing");
  if (!iw->full_range && !(iw->low < iw->high))
    fail(SALVOX_EINVAL, "IntensityWindow: low must be < high");
  if (iw->bins < 2) fail(SALVOX_EINVAL, "IntensityWindow: bins must be >= 2");
  // pipeline.cpp:66-72
  if (n_scales < 1 || !scales) fail(SALVOX_EINVAL, "exhaustive scan: no scales");
  for (int i = 0; i < n_scales; ++i)
    if (scales[i] < 2.0) fail(SALVOX_EINVAL, "exhaustive scan: scales must be >= 2 voxels");
  const uint64_t evals = (uint64_t)nx * ny * nz * (uint64_t)n_scales;
  if (evals > budget)
    fail(SALVOX_EINVAL, "exhaustive scan: budget exceeded (" + std::to_string(evals) +
                            " voxel-scale evaluations)");
  if (kernel != SALVOX_KERNEL_IDENTITY && kernel != SALVOX_KERNEL_EPANECHNIKOV)
    fail(SALVOX_EUNSUPPORTED,
         "exhaustive (device): identity and Epanechnikov kernels only (the Gaussian weights have "
         "no exact integer form)");
  if (iw->bins > 64) fail(SALVOX_EUNSUPPORTED, "exhaustive (device): bins must be <= 64");
  if ((uint64_t)nx * ny * nz > 0xffffffffull)
    fail(SALVOX_EUNSUPPORTED, "exhaustive (device): volume exceeds 2^32 voxels");
}

// make_plan enumerates the (2R+1)^3 candidate offsets per radius (milliseconds
// at R = 16): plans are cached per (scales, 2D, tile config).
Plan cached_plan(const double* scales, int n_scales, bool two_d, const TileCfg& tc, int* SYo,
                 int* SZo) {
  struct Entry {
    std::vector<double> scales;
    bool two_d;
    TileCfg tc;
    Plan pl;
    int SY, SZ;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (const Entry& e : cache)
    if (e.two_d == two_d && e.tc.nb == tc.nb && e.tc.tx == tc.tx && e.tc.ty == tc.ty &&
        e.tc.tz == tc.tz && e.tc.pair == tc.pair && e.tc.tmem == tc.tmem &&
        e.scales.size() == (size_t)n_scales &&
        std::equal(e.scales.begin(), e.scales.end(), scales)) {
      *SYo = e.SY;
      *SZo = e.SZ;
      return e.pl;
    }
  Entry e;
  e.scales.assign(scales, scales + n_scales);
  e.two_d = two_d;
  e.tc = tc;
  e.pl = make_plan(scales, n_scales, two_d, tc, &e.SY, &e.SZ);
  *SYo = e.SY;
  *SZo = e.SZ;
  if (cache.size() >= 16) cache.erase(cache.begin());
  cache.push_back(e);
  return cache.back().pl;
}

// Setup of one exhaustive run over the slab planes [zs0, zs1) (device bins at
// ctx->d_bins, pitch 16-aligned): plan, tensor map, kernel parameters for the
// scored planes [zc0, zc1) = [z0-1, z1+1) clipped, score/best buffers.
ExhRun setup_exhaustive(salvox_ctx* ctx, int nx, int ny, int nz, int zs0, int zs1, int z0, int z1,
                        int bins, const double* scales, int n_scales, bool exch = false,
                        bool epa = false) {
  const bool two_d = nz == 1;
  ExhRun run;
  run.generation = ++ctx->exh_generation;  // invalidates any pending exchange-form run
  run.tc = pick_tile(bins, two_d, epa);
  int SY = 0, SZ = 0;
  run.pl = cached_plan(scales, n_scales, two_d, run.tc, &SY, &SZ);
  if (epa)
    for (const KbBound& b : run.pl.bounds)
      if (b.q == 0)
        fail(SALVOX_EUNSUPPORTED,
             "exhaustive (device): the Epanechnikov kernel needs integer or half-integer scales");
  if (run.tc.quad && run.pl.qtab.empty()) run.tc.quad = false, run.tc.tmem = true;  // table too big
  const int R = run.pl.R;
  if (zs0 > std::max(0, z0 - R - 1) || zs1 < std::min(nz, z1 + R + 1))
    fail(SALVOX_EINVAL, "exhaustive slab: the slab must cover the owned planes plus the halo");
  const int nzs = zs1 - zs0;
  const int pitch = (nx + 15) / 16 * 16;
  uint8_t* d_bins = static_cast<uint8_t*>(ctx->d_bins.ensure((size_t)pitch * ny * nzs));
  const int zb0 = std::max(0, z0 - 1), zb1 = std::min(nz, z1 + 1);
  const int zc0 = exch ? z0 : zb0, zc1 = exch ? z1 : zb1;
  const size_t nscore = (size_t)nx * ny * (zb1 - zb0);
  float* d_score = static_cast<float*>(ctx->d_score.ensure(nscore * 4));
  float* d_best = static_cast<float*>(ctx->d_best.ensure(nscore * 4));
  run.zb0 = zb0;
  run.zb1 = zb1;
  run.z0 = z0;
  run.z1 = z1;
  run.score_base = d_score;
  run.best_base = d_best;
  run.exch = exch;

  const int BX = SY, BY = SZ / SY, BZ = run.tc.tz + 2 * R;
  cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nzs};
  cuuint64_t gstride[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * ny};
  cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)BY, (cuuint32_t)(two_d ? 1 : BZ)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = encode_fn()(&run.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d_bins, gdim, gstride, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) fail(SALVOX_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));

  KbParams& kp = run.kp;
  kp.nx = nx;
  kp.ny = ny;
  kp.nz = nz;
  kp.zs0 = zs0;
  kp.zc0 = zc0;
  kp.zc1 = zc1;
  kp.R = R;
  kp.lag = kb_lag();
  kp.lagmode = kb_lagmode();
  kp.Rz = two_d ? 0 : R;
  kp.SY = SY;
  kp.SZ = SZ;
  kp.n_radii = (int)run.pl.radii.size();
  kp.bins = bins;
  kp.tile_bytes = (uint32_t)(BX * BY * (two_d ? 1 : BZ));
  kp.score = d_score + (size_t)nx * ny * (zc0 - zb0);
  kp.best = d_best + (size_t)nx * ny * (zc0 - zb0);
  kp.dbg_vox = nullptr;
  kp.dbg_out = nullptr;
  kp.h_score = nullptr;
  kp.h_best = nullptr;
  kp.hz0 = kp.hz1 = 0;
  run.smem = kb_smem(run.tc, kp.tile_bytes);
  run.grid = dim3((nx + run.tc.tx - 1) / run.tc.tx, (ny + run.tc.ty - 1) / run.tc.ty,
                  (zc1 - zc0 + run.tc.tz - 1) / run.tc.tz);
  return run;
}

// KB kernel over the scored planes [a, b) (a subrange of [zc0, zc1)); the
// constant-memory tables must already hold run.pl (caller holds g_const_mu).
// With h_score/h_best (device-accessible pinned host maps of the owned planes
// [hz0, hz1)) the epilogue also stores there; pdl as dispatch_kb.
void launch_kb_chunk(salvox_ctx* ctx, const ExhRun& run, int a, int b, float* h_score = nullptr,
                     float* h_best = nullptr, int hz0 = 0, int hz1 = 0, bool pdl = false) {
  KbParams kp = run.kp;
  kp.h_score = h_score;
  kp.h_best = h_best;
  kp.hz0 = hz0;
  kp.hz1 = hz1;
  const size_t plane = (size_t)kp.nx * kp.ny;
  kp.score = run.kp.score + (size_t)(a - run.kp.zc0) * plane;
  kp.best = run.kp.best + (size_t)(a - run.kp.zc0) * plane;
  kp.zc0 = a;
  kp.zc1 = b;
  const dim3 grid(run.grid.x, run.grid.y, (b - a + run.tc.tz - 1) / run.tc.tz);
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->profiling) {
    SX_CUDA(cudaEventCreate(&ev0));
    SX_CUDA(cudaEventCreate(&ev1));
    SX_CUDA(cudaEventRecord(ev0, ctx->stream));
  }
  dispatch_kb<false>(ctx, run.tc, run.map, kp, grid, run.smem, pdl && !ctx->profiling);
  if (ctx->profiling) {
    SX_CUDA(cudaEventRecord(ev1, ctx->stream));
    SX_CUDA(cudaEventSynchronize(ev1));
    float ms = 0.f;
    SX_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    ctx->kb_ms_total += ms;
    ctx->kb_launches += 1;
    ctx->kb_updates_total += (double)plane * (b - a) * (double)(run.pl.ball_size.back() - 1);
  }
}

// K3: strict maxima of the owned planes + sort + decode. Returns the count.
long long maxima_and_sort(salvox_ctx* ctx, const ExhRun& run, int z0, int z1) {
  const int nx = run.kp.nx, ny = run.kp.ny, nz = run.kp.nz, zc0 = run.zb0;
  const float* d_score = run.score_base;
  const float* d_best = run.best_base;
  const size_t nown = (size_t)nx * ny * (z1 - z0);
  const size_t kcap = nown / 2 + 1;
  unsigned long long* d_keys = static_cast<unsigned long long*>(ctx->d_keys.ensure(kcap * 8));
  unsigned long long* d_keys2 = static_cast<unsigned long long*>(ctx->d_keys_alt.ensure(kcap * 8));
  unsigned int* d_cnt = static_cast<unsigned int*>(ctx->d_counter.ensure(64));
  SX_CUDA(cudaMemsetAsync(d_cnt, 0, 4, ctx->stream));
  const long long rows = (long long)ny * (z1 - z0);
  static const bool row_form = [] {  // A/B knob SALVOX_MAXIMA_ROWS=1: the per-row kernel
    const char* e = std::getenv("SALVOX_MAXIMA_ROWS");
    return e && e[0] == '1';
  }();
  if (row_form) {
    maxima_kernel<<<(int)std::min<long long>(std::max<long long>(rows, 1), ctx->sm_count * 32),
                    nx >= 128 ? 128 : 32, 0, ctx->stream>>>(d_score, nx, ny, nz, zc0, z0, z1, d_keys,
                                                           d_cnt);
  } else if (z1 > z0) {
    const dim3 grid((nx + kMxTX - 1) / kMxTX, (ny + kMxTY - 1) / kMxTY, (z1 - z0 + kMxZ - 1) / kMxZ);
    maxima_tile_kernel<<<grid, kMxTX * kMxTY, 0, ctx->stream>>>(d_score, nx, ny, nz, zc0, z0, z1,
                                                                d_keys, d_cnt);
  }
  SX_LAUNCH_CHECK(ctx);
  unsigned int cnt = 0;
  SX_CUDA(cudaMemcpyAsync(&cnt, d_cnt, 4, cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  if (cnt > 1) {
    size_t tmp = 0;
    SX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, d_keys, d_keys2, (int)cnt, 0, 64,
                                           ctx->stream));
    void* d_tmp = ctx->d_cub.ensure(tmp);
    SX_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, tmp, d_keys, d_keys2, (int)cnt, 0, 64,
                                           ctx->stream));
    ctx->launches += 4;  // cub onesweep: histogram + exclusive-sum + passes (approx.)
  } else if (cnt == 1) {
    SX_CUDA(cudaMemcpyAsync(d_keys2, d_keys, 8, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  salvox_maximum* d_max =
      static_cast<salvox_maximum*>(ctx->d_maxima.ensure(std::max<size_t>(cnt, 1) * sizeof(salvox_maximum)));
  if (cnt > 0) {
    decode_maxima_kernel<<<(int)std::min<long long>((cnt + 255) / 256, ctx->sm_count * 8), 256, 0,
                           ctx->stream>>>(d_keys2, cnt, d_best, nx, ny, zc0, d_max);
    SX_LAUNCH_CHECK(ctx);
  }
  return cnt;
}

void remember_run(salvox_ctx* ctx, const ExhRun& run, int nx, int ny, int nz, int zs0, int zs1,
                  int z0, int z1, int bins, const double* scales, int n_scales) {
  ctx->exh.valid = true;  // for the debug entry point
  ctx->exh.nx = nx;
  ctx->exh.ny = ny;
  ctx->exh.nz = nz;
  ctx->exh.zs0 = zs0;
  ctx->exh.zs1 = zs1;
  ctx->exh.z0 = z0;
  ctx->exh.z1 = z1;
  ctx->exh.zb0 = run.zb0;
  ctx->exh.bins = bins;
  ctx->exh.radii = run.pl.radii;
  ctx->exh.scales.assign(scales, scales + n_scales);
}

// Core: d_slab holds planes [zs0, zs1) of the volume (device, f32). Scores planes
// [zc0, zc1) = [z0-1, z1+1) clipped, finds maxima of [z0, z1), sorts them.
// Leaves: ctx->d_score/d_best (planes zc0..zc1), sorted keys, count.
long long run_exhaustive(salvox_ctx* ctx, const float* d_slab, int nx, int ny, int nz, int zs0,
                         int zs1, int z0, int z1, double low, double high, int bins,
                         const double* scales, int n_scales, ExhRun* run_out, bool exch = false,
                         bool epa = false) {
  ExhRun run = setup_exhaustive(ctx, nx, ny, nz, zs0, zs1, z0, z1, bins, scales, n_scales, exch, epa);
  const int pitch = (nx + 15) / 16 * 16;
  launch_bin_volume(ctx, d_slab, ctx->d_bins.as<uint8_t>(), nx, ny, zs1 - zs0, pitch, low, high,
                    bins);
  {
    std::lock_guard<std::mutex> lk(g_const_mu);
    upload_tables(ctx, run.pl, run.tc.quad);
    launch_kb_chunk(ctx, run, run.kp.zc0, run.kp.zc1);
    SX_CUDA(cudaEventRecord(g_const_done, ctx->stream));
  }
  const long long cnt = exch ? 0 : maxima_and_sort(ctx, run, z0, z1);
  if (run_out) *run_out = run;
  remember_run(ctx, run, nx, ny, nz, zs0, zs1, z0, z1, bins, scales, n_scales);
  return cnt;
}

cudaEvent_t ctx_event(salvox_ctx* ctx, size_t i) {
  while (ctx->events.size() <= i) {
    cudaEvent_t e;
    SX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->events.push_back(e);
  }
  return ctx->events[i];
}

// SALVOX_E2E_TRACE=1: device timeline of the direct host-buffer form (stderr);
// the marks between the two chunks delay the second one's programmatic start.
struct E2eTrace {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, const char*>> marks;
  std::vector<std::pair<double, const char*>> hmarks;  // host-side phases
  std::chrono::steady_clock::time_point t0;
  explicit E2eTrace(cudaStream_t s) {
    static const bool env = [] {
      const char* e = std::getenv("SALVOX_E2E_TRACE");
      return e && e[0] == '1';
    }();
    on = env;
    if (on) {
      t0 = std::chrono::steady_clock::now();
      mark(s, "entry");
    }
  }
  void mark(cudaStream_t s, const char* what) {
    if (!on) return;
    cudaEvent_t e;
    SX_CUDA(cudaEventCreate(&e));
    SX_CUDA(cudaEventRecord(e, s));
    marks.emplace_back(e, what);
  }
  void host(const char* what) {
    if (on)
      hmarks.emplace_back(
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
  }
  void report() {
    if (!on) return;
    for (auto& h : hmarks) std::fprintf(stderr, "[e2e host] %8.3f ms  %s\n", h.first, h.second);
    hmarks.clear();
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (auto& m : marks) {
      float ms = 0.f;
      SX_CUDA(cudaEventSynchronize(m.first));
      SX_CUDA(cudaEventElapsedTime(&ms, marks[0].first, m.first));
      std::fprintf(stderr, "[e2e] %8.3f ms  %s\n", ms, m.second);
    }
    std::fprintf(stderr, "[e2e] %8.3f ms  host return\n", host_ms);
    for (auto& m : marks) cudaEventDestroy(m.first);
    marks.clear();
  }
};

// SALVOX_EXH_STAGED=0: pageable host maps take the plain (blocking) D2H (A/B timing).
bool staged_maps_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SALVOX_EXH_STAGED");
    return e && std::string(e) == "0";
  }();
  return off;
}

// Whether host buffer h is page-locked (any CUDA host allocation or registration).
bool pinned_host(const void* h) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy with up to 8 threads (page-sized splits): pageable buffers copy at a
// few GB/s per thread.
void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  static const int T = [] {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return (int)std::min(8u, std::max(1u, hw / 2));
  }();
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const size_t per = std::max<size_t>(((bytes + T - 1) / T + 4095) & ~(size_t)4095, 1 << 20);
  std::vector<std::thread> hs;
  for (size_t o = per; o < bytes; o += per)
    hs.emplace_back([=] { std::memcpy(d + o, s + o, std::min(per, bytes - o)); });
  std::memcpy(d, s, std::min(per, bytes));
  for (auto& h : hs) h.join();
}

// Faults the pages of host range [p, p + n) in (huge pages where THP allows),
// with up to T threads: a fresh pageable buffer written later by a memcpy
// would otherwise take its page faults inside that copy.
void prefault(char* p, size_t n, int T) {
  if (!p || n == 0) return;
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(p) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + n) & ~uintptr_t((2u << 20) - 1);
  if (a1 > a0) madvise(reinterpret_cast<void*>(a0), a1 - a0, MADV_HUGEPAGE);  // errors: harmless
  const size_t pages = (n + 4095) / 4096;
  auto touch = [=](int t) {
    for (size_t pg = pages * t / T; pg < pages * (t + 1) / T; ++pg)
      reinterpret_cast<volatile char*>(p)[pg * 4096] = 0;
  };
  std::vector<std::thread> hs;
  for (int t = 1; t < T; ++t) hs.emplace_back(touch, t);
  touch(0);
  for (auto& h : hs) h.join();
}

// Host side of the staged copy-back: one thread walks the chunks in order,
// waits for each chunk's DMA event and copies its (dst, src, bytes) parts into
// the caller's pageable buffers with up to 8 helper threads (first-touch page
// faults of a fresh buffer make one thread far slower than the DMA).
struct StagedCopier {
  std::thread th;
  std::string err;
  void start(int device, std::vector<std::pair<cudaEvent_t, std::vector<std::array<void*, 3>>>> jobs) {
    th = std::thread([this, device, jobs = std::move(jobs)] {
      cudaSetDevice(device);
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const int T = (int)std::min(8u, std::max(1u, hw / 2));
      {  // fault the destination pages in while the first chunks compute
        std::vector<std::pair<char*, size_t>> ranges;
        for (const auto& j : jobs)
          for (const auto& part : j.second) ranges.emplace_back(static_cast<char*>(part[0]), (size_t)part[2]);
        for (const auto& r : ranges) prefault(r.first, r.second, T);
      }
      for (const auto& j : jobs) {
        const cudaError_t e = cudaEventSynchronize(j.first);
        if (e != cudaSuccess) {
          err = cudaGetErrorString(e);
          return;
        }
        for (const auto& part : j.second) parallel_memcpy(part[0], part[1], (size_t)part[2]);
      }
    });
  }
  void finish() {
    if (th.joinable()) th.join();
    if (!err.empty()) fail(SALVOX_ECUDA, "staged map copy-back: " + err);
  }
  ~StagedCopier() {
    if (th.joinable()) th.join();
  }
};

// SALVOX_EXH_DIRECT=0 keeps the copy-back pipeline even for pinned host maps (A/B timing).
bool direct_maps_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SALVOX_EXH_DIRECT");
    return e && std::string(e) == "0";
  }();
  return off;
}

// The device address of host buffer [h, h + n) when it is pinned, mapped and one
// allocation (torch pin_memory, cudaHostAlloc); null otherwise.
float* mapped_host(float* h, size_t n) {
  if (!h || n == 0) return nullptr;
  cudaPointerAttributes a{}, b{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess ||
      cudaPointerGetAttributes(&b, h + n - 1) != cudaSuccess) {
    cudaGetLastError();  // clear: a pageable pointer is not an error here
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || !a.devicePointer ||
      !b.devicePointer)
    return nullptr;
  float* d = static_cast<float*>(a.devicePointer);
  if (static_cast<float*>(b.devicePointer) != d + (n - 1)) return nullptr;
  return d;
}

// Host-buffer form, pipelined: the slab goes up in pieces
// on the copy stream; the compute stream bins each piece as it lands and runs
// the KB kernel over K z-chunks of the scored planes; each chunk's owned
// score/best planes stream back on the copy stream while the next chunk
// computes. Same kernels and arithmetic as run_exhaustive.
long long run_exhaustive_pipelined(salvox_ctx* ctx, const float* h_slab, int nx, int ny, int nz,
                                   int zs0, int zs1, int z0, int z1, double low, double high,
                                   int bins, const double* scales, int n_scales,
                                   float* score_out, float* best_out, ExhRun* run_out,
                                   bool exch = false, bool epa = false) {
  if (!ctx->copy_stream) {
    // highest priority: the bin kernels queued on it behind each uploaded piece
    // get their CTAs dispatched beside a running KB chunk (which keeps the SMs
    // saturated with pending CTAs) instead of after its last CTA is placed
    int least = 0, greatest = 0;
    SX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SX_CUDA(cudaStreamCreateWithPriority(&ctx->copy_stream, cudaStreamNonBlocking, greatest));
  }
  cudaStream_t cs = ctx->stream, ps = ctx->copy_stream;
  ExhRun run = setup_exhaustive(ctx, nx, ny, nz, zs0, zs1, z0, z1, bins, scales, n_scales, exch, epa);
  const int R = run.pl.R, tz = run.tc.tz;
  const int nzs = zs1 - zs0;
  const size_t plane = (size_t)nx * ny;
  const int pitch = (nx + 15) / 16 * 16;
  float* d_vol = static_cast<float*>(ctx->d_vol.ensure(plane * nzs * 4));
  uint8_t* d_bins = ctx->d_bins.as<uint8_t>();
  // K output chunks of whole tiles; the input in pieces of the same planes
  const int zc0 = run.kp.zc0, zc1 = run.kp.zc1;
  const int ntiles = (zc1 - zc0 + tz - 1) / tz;
  const int npieces = std::max(1, std::min(8, nzs / 8));
  std::vector<int> pc(npieces + 1);
  for (int i = 0; i <= npieces; ++i) pc[i] = (int)((long long)nzs * i / npieces);
  // A pageable slab would make each piece's cudaMemcpyAsync a blocking,
  // driver-staged copy (the host could enqueue no kernel until the whole slab
  // was up): host threads copy each piece into pinned staging right before its
  // (then truly asynchronous) DMA, and pieces are enqueued only as the chunks
  // need them, so those host copies overlap the first chunk's compute.
  const bool stage_in = !staged_maps_disabled() && !pinned_host(h_slab);
  float* h_in = stage_in ? static_cast<float*>(ctx->h_vol.ensure(plane * nzs * 4)) : nullptr;
  auto upload = [&](int p0, int p1) {  // local planes [p0, p1) on the copy stream
    const size_t o = (size_t)p0 * plane, n = (size_t)(p1 - p0) * plane;
    const float* src = h_slab + o;
    if (stage_in) {
      parallel_memcpy(h_in + o, src, n * 4);
      src = h_in + o;
    }
    SX_CUDA(cudaMemcpyAsync(d_vol + o, src, n * 4, cudaMemcpyHostToDevice, ps));
  };
  float* hs = mapped_host(score_out, (size_t)(z1 - z0) * plane);
  float* hb = mapped_host(best_out, (size_t)(z1 - z0) * plane);
  static const bool no_store = [] {  // trace knob: skip the host stores (maps NOT written)
    const char* e = std::getenv("SALVOX_E2E_NOSTORE");
    return e && e[0] == '1';
  }();
  if (run.tc.quad && !direct_maps_disabled() && (score_out || best_out) && (!score_out || hs) &&
      (!best_out || hb)) {
    // Direct form: the KB epilogue stores the owned maps straight into the
    // caller's pinned host buffers (no copy-back at all), so the only reason
    // to chunk is the upload: a small first chunk starts once its own planes
    // have landed, the rest follows as a programmatic
    // dependent that fills the SMs the first chunk's tail frees. Each piece
    // is binned on the copy stream right after it lands.
    // chunk 0: 1/16 of the tile layers (1/8 when there are fewer than 16)
    const int c1 = ntiles >= 16   ? zc0 + tz * (ntiles / 16)
                   : ntiles >= 8 ? zc0 + tz * (ntiles / 8)
                                 : zc1;
    const int need0 = std::min(nzs, c1 + R + 1 - zs0);  // local planes chunk 0 reads
    // upload pieces: exactly chunk 0's planes first, then the rest in <= 7 parts
    std::vector<int> dp{0, need0};
    const int rest = nzs - need0;
    const int nrest = rest > 0 ? std::max(1, std::min(7, rest / 8)) : 0;
    for (int i = 1; i <= nrest; ++i) dp.push_back(need0 + (int)((long long)rest * i / nrest));
    const int nd = (int)dp.size() - 1;
    E2eTrace tr(cs);
    SX_CUDA(cudaEventRecord(ctx_event(ctx, 0), cs));  // order after earlier work on cs
    SX_CUDA(cudaStreamWaitEvent(ps, ctx_event(ctx, 0), 0));
    auto piece = [&](int i) {
      upload(dp[i], dp[i + 1]);
      launch_bin_volume(ctx, d_vol + (size_t)dp[i] * plane, d_bins + (size_t)dp[i] * pitch * ny, nx,
                        ny, dp[i + 1] - dp[i], pitch, low, high, bins, ps);
      SX_CUDA(cudaEventRecord(ctx_event(ctx, 1 + i), ps));
      tr.mark(ps, "piece uploaded+binned");
    };
    piece(0);
    {
      std::lock_guard<std::mutex> lk(g_const_mu);
      upload_tables(ctx, run.pl, run.tc.quad);
      SX_CUDA(cudaStreamWaitEvent(cs, ctx_event(ctx, 1), 0));  // chunk 0's planes binned
      tr.mark(cs, "chunk 0 may start");
      const int hz1 = no_store ? z0 : z1;
      launch_kb_chunk(ctx, run, zc0, c1, hs, hb, z0, hz1);
      tr.mark(cs, "chunk 0 done");
      for (int i = 1; i < nd; ++i) piece(i);
      if (c1 < zc1) {
        SX_CUDA(cudaStreamWaitEvent(cs, ctx_event(ctx, nd), 0));  // every piece binned
        launch_kb_chunk(ctx, run, c1, zc1, hs, hb, z0, hz1, /*pdl=*/true);
        tr.mark(cs, "chunk 1 done");
      }
      SX_CUDA(cudaEventRecord(g_const_done, cs));
    }
    const long long cnt = exch ? 0 : maxima_and_sort(ctx, run, z0, z1);
    tr.mark(cs, "maxima sorted");
    SX_CUDA(cudaStreamSynchronize(cs));  // the host maps are complete
    tr.report();
    if (run_out) *run_out = run;
    remember_run(ctx, run, nx, ny, nz, zs0, zs1, z0, z1, bins, scales, n_scales);
    return cnt;
  }
  const int K = std::max(1, std::min(4, ntiles / 4));
  // chunk boundaries in eighths of the tile layers: 1, 3, 3, 1 for K = 4 -- a
  // short first chunk starts after fewer uploaded planes, a short last chunk
  // leaves fewer maps to copy back after the compute ends
  static const int kEighths[5][5] = {{0}, {0, 8}, {0, 4, 8}, {0, 2, 6, 8}, {0, 1, 4, 7, 8}};
  std::vector<int> cut(K + 1);
  for (int k = 0; k <= K; ++k)
    cut[k] = std::min(zc1, zc0 + tz * (int)((long long)ntiles * kEighths[K][k] / 8));
  cut[K] = zc1;
  E2eTrace tr(cs);
  SX_CUDA(cudaEventRecord(ctx_event(ctx, 0), cs));  // order after earlier work on cs
  SX_CUDA(cudaStreamWaitEvent(ps, ctx_event(ctx, 0), 0));
  int uploaded = 0, binned = 0;  // pieces enqueued for upload / binned so far
  auto piece_up = [&] {
    upload(pc[uploaded], pc[uploaded + 1]);
    SX_CUDA(cudaEventRecord(ctx_event(ctx, 1 + uploaded), ps));
    ++uploaded;
  };
  {
    std::lock_guard<std::mutex> lk(g_const_mu);
    upload_tables(ctx, run.pl, run.tc.quad);
    for (int k = 0; k < K; ++k) {
      const int need = std::min(nzs, cut[k + 1] + R + 1 - zs0);  // local planes the chunk reads
      while (binned < npieces && pc[binned] < need) {
        while (uploaded <= binned) piece_up();
        SX_CUDA(cudaStreamWaitEvent(cs, ctx_event(ctx, 1 + binned), 0));
        const int p0 = pc[binned], p1 = pc[binned + 1];
        launch_bin_volume(ctx, d_vol + (size_t)p0 * plane, d_bins + (size_t)p0 * pitch * ny, nx, ny,
                          p1 - p0, pitch, low, high, bins);
        ++binned;
      }
      tr.host("chunk enqueue");
      tr.mark(cs, "chunk start");
      launch_kb_chunk(ctx, run, cut[k], cut[k + 1]);
      tr.mark(cs, "chunk done");
      SX_CUDA(cudaEventRecord(ctx_event(ctx, 1 + npieces + k), cs));
    }
    SX_CUDA(cudaEventRecord(g_const_done, cs));
  }
  while (uploaded < npieces) piece_up();  // planes no chunk reads (keeps d_vol whole)
  // Owned planes of each chunk back to the host while later chunks compute.
  // Pinned (mapped or not) maps take the DMA directly. Pageable maps would make
  // each cudaMemcpyAsync a blocking, driver-staged copy (C2: ~20 ms after the
  // compute), so they go through pinned staging instead: one DMA per chunk into
  // ctx->h_maps, and host threads copy each chunk into the caller's buffers as
  // soon as its DMA lands, overlapped with the later chunks' compute.
  const size_t nown = (size_t)(z1 - z0) * plane;
  const bool stage = ((score_out && !pinned_host(score_out)) || (best_out && !pinned_host(best_out))) &&
                     !staged_maps_disabled() && nown * 8 <= (size_t(1) << 31);
  float* st = stage ? static_cast<float*>(ctx->h_maps.ensure(nown * 8)) : nullptr;
  std::vector<std::array<size_t, 3>> spans;  // (dst offset, planes * plane, event index)
  for (int k = 0; k < K; ++k) {
    const int a = std::max(cut[k], z0), b = std::min(cut[k + 1], z1);
    if (a >= b) continue;
    SX_CUDA(cudaStreamWaitEvent(ps, ctx_event(ctx, 1 + npieces + k), 0));
    const size_t src = (size_t)(a - zc0) * plane, dst = (size_t)(a - z0) * plane;
    const size_t n = (size_t)(b - a) * plane;
    float* so = stage ? st + dst : score_out + dst;
    float* bo = stage ? st + nown + dst : best_out + dst;
    if (score_out)
      SX_CUDA(cudaMemcpyAsync(so, run.kp.score + src, n * 4, cudaMemcpyDeviceToHost, ps));
    if (best_out)
      SX_CUDA(cudaMemcpyAsync(bo, run.kp.best + src, n * 4, cudaMemcpyDeviceToHost, ps));
    if (stage) {
      const size_t ev = 1 + npieces + K + spans.size();
      SX_CUDA(cudaEventRecord(ctx_event(ctx, ev), ps));
      spans.push_back({dst, n, ev});
    }
    tr.mark(ps, "chunk maps D2H done");
  }
  tr.host("D2H enqueued");
  StagedCopier copier;
  if (stage) {
    std::vector<std::pair<cudaEvent_t, std::vector<std::array<void*, 3>>>> jobs;
    for (const auto& sp : spans) {
      std::vector<std::array<void*, 3>> parts;
      if (score_out) parts.push_back({score_out + sp[0], st + sp[0], (void*)(sp[1] * 4)});
      if (best_out) parts.push_back({best_out + sp[0], st + nown + sp[0], (void*)(sp[1] * 4)});
      jobs.emplace_back(ctx_event(ctx, sp[2]), std::move(parts));
    }
    copier.start(ctx->device, std::move(jobs));
  }
  const long long cnt = exch ? 0 : maxima_and_sort(ctx, run, z0, z1);
  tr.host("maxima sorted");
  copier.finish();
  tr.host("host map copies done");
  SX_CUDA(cudaStreamSynchronize(ps));
  tr.report();
  if (run_out) *run_out = run;
  remember_run(ctx, run, nx, ny, nz, zs0, zs1, z0, z1, bins, scales, n_scales);
  return cnt;
}

// SALVOX_EXH_PIPELINE=0 turns the host-buffer pipeline off (A/B timing).
bool pipeline_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SALVOX_EXH_PIPELINE");
    return e && std::string(e) == "0";
  }();
  return off;
}

uint64_t closed_form_visits(const Plan& pl, uint64_t voxels) {
  uint64_t per = 0;
  for (uint64_t b : pl.ball_size) per += b;
  return per * voxels;
}

void fetch_maxima(salvox_ctx* ctx, long long cnt, salvox_maximum* out, int64_t cap) {
  ctx->last_maxima_n = cnt;
  ctx->stage_valid = false;
  if (out && cap >= cnt) {  // straight into the caller's buffer (fast when it is pinned)
    if (cnt > 0)
      SX_CUDA(cudaMemcpyAsync(out, ctx->d_maxima.p, cnt * sizeof(salvox_maximum),
                              cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  // through pinned staging: one DMA, then the caller's share
  salvox_maximum* stage = static_cast<salvox_maximum*>(
      ctx->h_stage.ensure(std::max<size_t>((size_t)cnt, 1) * sizeof(salvox_maximum)));
  if (cnt > 0)
    SX_CUDA(cudaMemcpyAsync(stage, ctx->d_maxima.p, cnt * sizeof(salvox_maximum),
                            cudaMemcpyDeviceToHost, ctx->stream));
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stage_valid = true;
  if (out && cap > 0)
    parallel_memcpy(out, stage, (size_t)std::min<long long>(cnt, cap) * sizeof(salvox_maximum));
}

int exhaustive_host(salvox_ctx* ctx, const float* slab, int32_t nx, int32_t ny, int32_t nz,
                    int32_t zs0, int32_t zs1, int32_t z0, int32_t z1, const salvox_window* iw,
                    const double* scales, int32_t n_scales, int32_t kernel, uint64_t budget,
                    float* score_out, float* best_scale_out, salvox_maximum* maxima, int64_t cap,
                    int64_t* n_maxima, uint64_t* visits, bool slab_form) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    validate_exhaustive(nx, ny, nz, iw, scales, n_scales, kernel, budget);
    const bool epa = kernel == SALVOX_KERNEL_EPANECHNIKOV;
    if (!slab) fail(SALVOX_EINVAL, "null volume");
    if (!(0 <= zs0 && zs0 <= z0 && z0 < z1 && z1 <= zs1 && zs1 <= nz))
      fail(SALVOX_EINVAL, "exhaustive slab: need 0 <= zs0 <= z0 < z1 <= zs1 <= nz");
    if (slab_form && iw->full_range)
      fail(SALVOX_EINVAL, "exhaustive slab: pass an explicit (global) intensity window");
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nslab = (size_t)nx * ny * (zs1 - zs0);
    const size_t nown = (size_t)nx * ny * (z1 - z0);
    // a pageable maxima buffer: its pages fault in while the pass computes
    std::thread mx_fault;
    if (maxima && cap > 0 && !staged_maps_disabled() && !pinned_host(maxima))
      mx_fault = std::thread(prefault, reinterpret_cast<char*>(maxima),
                             (size_t)cap * sizeof(salvox_maximum), 2);
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } mx_join{mx_fault};
    ExhRun run;
    long long cnt;
    if (!iw->full_range && !pipeline_disabled()) {
      cnt = run_exhaustive_pipelined(ctx, slab, nx, ny, nz, zs0, zs1, z0, z1, iw->low, iw->high,
                                     iw->bins, scales, n_scales, score_out, best_scale_out, &run,
                                     false, epa);
    } else {  // full_range needs the whole slab's min/max before any binning
      float* d_vol = static_cast<float*>(ctx->d_vol.ensure(nslab * 4));
      SX_CUDA(cudaMemcpyAsync(d_vol, slab, nslab * 4, cudaMemcpyHostToDevice, ctx->stream));
      double low = iw->low, high = iw->high;
      if (iw->full_range) device_full_range(ctx, d_vol, nslab, &low, &high);
      cnt = run_exhaustive(ctx, d_vol, nx, ny, nz, zs0, zs1, z0, z1, low, high, iw->bins, scales,
                           n_scales, &run, false, epa);
      const size_t off = (size_t)nx * ny * (z0 - run.zb0);
      if (score_out)
        SX_CUDA(cudaMemcpyAsync(score_out, ctx->d_score.as<float>() + off, nown * 4,
                                cudaMemcpyDeviceToHost, ctx->stream));
      if (best_scale_out)
        SX_CUDA(cudaMemcpyAsync(best_scale_out, ctx->d_best.as<float>() + off, nown * 4,
                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (mx_fault.joinable()) mx_fault.join();
    fetch_maxima(ctx, cnt, maxima, cap);
    if (n_maxima) *n_maxima = cnt;
    if (visits) *visits += closed_form_visits(run.pl, nown);
  });
}

}  // namespace
}  // namespace sx

using namespace sx;

extern "C" int salvox_exhaustive(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                 int32_t nz, const salvox_window* iw, const double* scales,
                                 int32_t n_scales, int32_t kernel, uint64_t budget,
                                 float* score_out, float* best_scale_out, salvox_maximum* maxima,
                                 int64_t cap, int64_t* n_maxima, uint64_t* visits) {
  return exhaustive_host(ctx, volume, nx, ny, nz, 0, nz, 0, nz, iw, scales, n_scales, kernel,
                         budget, score_out, best_scale_out, maxima, cap, n_maxima, visits, false);
}

extern "C" int salvox_exhaustive_slab(salvox_ctx* ctx, const float* slab, int32_t nx, int32_t ny,
                                      int32_t nz, int32_t zs0, int32_t zs1, int32_t z0,
                                      int32_t z1, const salvox_window* iw, const double* scales,
                                      int32_t n_scales, int32_t kernel, uint64_t budget,
                                      float* score_out, float* best_scale_out,
                                      salvox_maximum* maxima, int64_t cap, int64_t* n_maxima,
                                      uint64_t* visits) {
  return exhaustive_host(ctx, slab, nx, ny, nz, zs0, zs1, z0, z1, iw, scales, n_scales, kernel,
                         budget, score_out, best_scale_out, maxima, cap, n_maxima, visits, true);
}

static int exhaustive_device_impl(salvox_ctx* ctx, const float* d_slab, int32_t nx, int32_t ny,
                                  int32_t nz, int32_t zs0, int32_t zs1, int32_t z0, int32_t z1,
                                  const salvox_window* iw, const double* scales, int32_t n_scales,
                                  int32_t kernel, uint64_t budget, float* d_score,
                                  float* d_best_scale, int64_t* n_maxima, bool slab_form) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    validate_exhaustive(nx, ny, nz, iw, scales, n_scales, kernel, budget);
    const bool epa = kernel == SALVOX_KERNEL_EPANECHNIKOV;
    if (!d_slab) fail(SALVOX_EINVAL, "null volume");
    if (!(0 <= zs0 && zs0 <= z0 && z0 < z1 && z1 <= zs1 && zs1 <= nz))
      fail(SALVOX_EINVAL, "exhaustive slab: need 0 <= zs0 <= z0 < z1 <= zs1 <= nz");
    if (slab_form && iw->full_range)
      fail(SALVOX_EINVAL, "exhaustive slab: pass an explicit (global) intensity window");
    SX_CUDA(cudaSetDevice(ctx->device));
    double low = iw->low, high = iw->high;
    if (iw->full_range) device_full_range(ctx, d_slab, (size_t)nx * ny * (zs1 - zs0), &low, &high);
    ExhRun run;
    const long long cnt = run_exhaustive(ctx, d_slab, nx, ny, nz, zs0, zs1, z0, z1, low, high,
                                         iw->bins, scales, n_scales, &run, false, epa);
    const size_t nown = (size_t)nx * ny * (z1 - z0);
    const size_t off = (size_t)nx * ny * (z0 - run.zb0);
    if (d_score)
      SX_CUDA(cudaMemcpyAsync(d_score, ctx->d_score.as<float>() + off, nown * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    if (d_best_scale)
      SX_CUDA(cudaMemcpyAsync(d_best_scale, ctx->d_best.as<float>() + off, nown * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    // device-resident form: the maxima stay in HBM (salvox_last_maxima[_device]
    // copy them on request); no host staging inside the call
    ctx->last_maxima_n = cnt;
    ctx->stage_valid = false;
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_maxima) *n_maxima = cnt;
  });
}

extern "C" int salvox_exhaustive_device(salvox_ctx* ctx, const float* d_volume, int32_t nx,
                                        int32_t ny, int32_t nz, const salvox_window* iw,
                                        const double* scales, int32_t n_scales, int32_t kernel,
                                        uint64_t budget, float* d_score, float* d_best_scale,
                                        int64_t* n_maxima) {
  return exhaustive_device_impl(ctx, d_volume, nx, ny, nz, 0, nz, 0, nz, iw, scales, n_scales,
                                kernel, budget, d_score, d_best_scale, n_maxima, false);
}

extern "C" int salvox_exhaustive_slab_device(salvox_ctx* ctx, const float* d_slab, int32_t nx,
                                             int32_t ny, int32_t nz, int32_t zs0, int32_t zs1,
                                             int32_t z0, int32_t z1, const salvox_window* iw,
                                             const double* scales, int32_t n_scales,
                                             int32_t kernel, uint64_t budget, float* d_score,
                                             float* d_best_scale, int64_t* n_maxima) {
  return exhaustive_device_impl(ctx, d_slab, nx, ny, nz, zs0, zs1, z0, z1, iw, scales, n_scales,
                                kernel, budget, d_score, d_best_scale, n_maxima, true);
}

// ---- z-slab exhaustive with a neighbour-plane exchange (multi-GPU) ----------
// The default slab call scores its owned planes plus one neighbour plane each
// side so strict maxima are decided locally; the KB kernel tiles z by 8, so the
// two extra planes are a nearly-empty extra tile layer (a 64-plane slab of the
// 512^3 C4 runs 54.3 ms instead of ~49). With the exchange the rank scores only
// its owned planes and receives the two neighbour planes from the adjacent
// ranks (one plane each way over NCCL) before the maxima pass.
namespace {
std::mutex g_exch_mu;
std::map<salvox_ctx*, ExhRun> g_exch_runs;  // the pending scores call of each context
}  // namespace

void sx::forget_exchange_run(salvox_ctx* ctx) {
  std::lock_guard<std::mutex> g(g_exch_mu);
  g_exch_runs.erase(ctx);
}

extern "C" int salvox_exhaustive_slab_scores(salvox_ctx* ctx, const float* slab, int32_t on_device,
                                             int32_t nx, int32_t ny, int32_t nz, int32_t zs0,
                                             int32_t zs1, int32_t z0, int32_t z1,
                                             const salvox_window* iw, const double* scales,
                                             int32_t n_scales, int32_t kernel, uint64_t budget,
                                             float* score_out, float* best_scale_out,
                                             uint64_t* visits) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    validate_exhaustive(nx, ny, nz, iw, scales, n_scales, kernel, budget);
    const bool epa = kernel == SALVOX_KERNEL_EPANECHNIKOV;
    if (!slab) fail(SALVOX_EINVAL, "null volume");
    if (!(0 <= zs0 && zs0 <= z0 && z0 < z1 && z1 <= zs1 && zs1 <= nz))
      fail(SALVOX_EINVAL, "exhaustive slab: need 0 <= zs0 <= z0 < z1 <= zs1 <= nz");
    if (iw->full_range)
      fail(SALVOX_EINVAL, "exhaustive slab: pass an explicit (global) intensity window");
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t nown = (size_t)nx * ny * (z1 - z0);
    ExhRun run;
    if (!on_device) {
      run_exhaustive_pipelined(ctx, slab, nx, ny, nz, zs0, zs1, z0, z1, iw->low, iw->high, iw->bins,
                               scales, n_scales, score_out, best_scale_out, &run, true, epa);
    } else {
      run_exhaustive(ctx, slab, nx, ny, nz, zs0, zs1, z0, z1, iw->low, iw->high, iw->bins, scales,
                     n_scales, &run, true, epa);
      if (score_out)
        SX_CUDA(cudaMemcpyAsync(score_out, run.kp.score, nown * 4, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      if (best_scale_out)
        SX_CUDA(cudaMemcpyAsync(best_scale_out, run.kp.best, nown * 4, cudaMemcpyDeviceToDevice,
                                ctx->stream));
      SX_CUDA(cudaStreamSynchronize(ctx->stream));  // outputs valid for any stream on return
    }
    {
      std::lock_guard<std::mutex> g(g_exch_mu);
      g_exch_runs[ctx] = run;
    }
    if (visits) *visits += closed_form_visits(run.pl, nown);
  });
}

extern "C" int salvox_exhaustive_slab_edges(salvox_ctx* ctx, float* d_first, float* d_last) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ExhRun run;
    {
      std::lock_guard<std::mutex> g(g_exch_mu);
      auto it = g_exch_runs.find(ctx);
      if (it == g_exch_runs.end()) fail(SALVOX_EINVAL, "exhaustive slab edges: no pending scores call");
      run = it->second;
      if (run.generation != ctx->exh_generation) {
        g_exch_runs.erase(it);
        fail(SALVOX_EINVAL,
             "exhaustive slab edges: another exhaustive call on this context replaced the pending "
             "scores");
      }
    }
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t plane = (size_t)run.kp.nx * run.kp.ny;
    if (d_first)
      SX_CUDA(cudaMemcpyAsync(d_first, run.kp.score, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (d_last)
      SX_CUDA(cudaMemcpyAsync(d_last, run.kp.score + plane * (run.z1 - run.z0 - 1), plane * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

extern "C" int salvox_exhaustive_slab_maxima(salvox_ctx* ctx, const float* d_below,
                                             const float* d_above, salvox_maximum* maxima,
                                             int64_t cap, int64_t* n_maxima) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    ExhRun run;
    {
      std::lock_guard<std::mutex> g(g_exch_mu);
      auto it = g_exch_runs.find(ctx);
      if (it == g_exch_runs.end()) fail(SALVOX_EINVAL, "exhaustive slab maxima: no pending scores call");
      run = it->second;
      g_exch_runs.erase(it);
      if (run.generation != ctx->exh_generation)
        fail(SALVOX_EINVAL,
             "exhaustive slab maxima: another exhaustive call on this context replaced the pending "
             "scores");
    }
    SX_CUDA(cudaSetDevice(ctx->device));
    const size_t plane = (size_t)run.kp.nx * run.kp.ny;
    if (run.z0 > 0) {  // plane z0 - 1 (the lower neighbour's last owned plane)
      if (!d_below) fail(SALVOX_EINVAL, "exhaustive slab maxima: the plane below is required");
      SX_CUDA(cudaMemcpyAsync(run.score_base, d_below, plane * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (run.z1 < run.kp.nz) {  // plane z1 (the upper neighbour's first owned plane)
      if (!d_above) fail(SALVOX_EINVAL, "exhaustive slab maxima: the plane above is required");
      SX_CUDA(cudaMemcpyAsync(run.score_base + plane * (run.zb1 - run.zb0 - 1), d_above, plane * 4,
                              cudaMemcpyDeviceToDevice, ctx->stream));
    }
    const long long cnt = maxima_and_sort(ctx, run, run.z0, run.z1);
    if (maxima) {
      fetch_maxima(ctx, cnt, maxima, cap);
    } else {  // they stay on the device (salvox_last_maxima[_device] fetch them)
      ctx->last_maxima_n = cnt;
      ctx->stage_valid = false;
    }
    if (n_maxima) *n_maxima = cnt;
  });
}

// ---- device-side maxima merge (multi-GPU) ------------------------------------
__global__ void maxima_keys_kernel(const salvox_maximum* __restrict__ in, long long n,
                                   unsigned long long* keys, unsigned int* idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float sc = (float)in[i].score;  // the map's float score, widened exactly
    keys[i] = ((unsigned long long)(~__float_as_uint(sc)) << 32) |
              ((unsigned long long)in[i].linear_index & 0xffffffffull);
    idx[i] = (unsigned int)i;
  }
}

__global__ void gather_maxima_kernel(const salvox_maximum* __restrict__ in,
                                     const unsigned int* __restrict__ idx, long long n,
                                     salvox_maximum* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}

extern "C" int salvox_last_maxima_device(salvox_ctx* ctx, salvox_maximum* d_out, int64_t cap,
                                         int64_t* n_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    const int64_t n = ctx->last_maxima_n;
    SX_CUDA(cudaSetDevice(ctx->device));
    if (d_out && cap > 0 && n > 0)
      SX_CUDA(cudaMemcpyAsync(d_out, ctx->d_maxima.p, (size_t)std::min(n, cap) * sizeof(salvox_maximum),
                              cudaMemcpyDeviceToDevice, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_out) *n_out = n;
  });
}

extern "C" int salvox_merge_maxima_device(salvox_ctx* ctx, const salvox_maximum* d_in, int64_t n,
                                          salvox_maximum* d_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    if (n < 0 || (n > 0 && (!d_in || !d_out))) fail(SALVOX_EINVAL, "merge maxima: bad arguments");
    if (n > (int64_t)UINT_MAX) fail(SALVOX_EUNSUPPORTED, "merge maxima: too many records");
    std::lock_guard<std::mutex> lk(ctx->mu);
    SX_CUDA(cudaSetDevice(ctx->device));
    if (n > 0) {
      const size_t un = (size_t)n;
      auto* keys = static_cast<unsigned long long*>(ctx->d_keys.ensure(un * 8));
      auto* keys2 = static_cast<unsigned long long*>(ctx->d_keys_alt.ensure(un * 8));
      auto* idx = static_cast<unsigned int*>(ctx->d_merge_idx.ensure(un * 8));
      unsigned int* idx2 = idx + un;
      const int grid = (int)std::min<long long>((n + 255) / 256, ctx->sm_count * 8);
      maxima_keys_kernel<<<grid, 256, 0, ctx->stream>>>(d_in, n, keys, idx);
      SX_LAUNCH_CHECK(ctx);
      size_t tmp = 0;
      SX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, idx, idx2, (int)n, 0, 64,
                                              ctx->stream));
      void* d_tmp = ctx->d_cub.ensure(tmp);
      SX_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, keys, keys2, idx, idx2, (int)n, 0, 64,
                                              ctx->stream));
      ctx->launches += 4;
      gather_maxima_kernel<<<grid, 256, 0, ctx->stream>>>(d_in, idx2, n, d_out);
      SX_LAUNCH_CHECK(ctx);
    }
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// Device map -> host buffer: pinned takes one DMA; pageable goes through two
// 16 MB pinned staging slots, the host copy of one chunk overlapping the DMA of
// the next.
void maps_to_host(salvox_ctx* ctx, const float* d, float* h, size_t n) {
  if (!h || n == 0) return;
  if (pinned_host(h)) {
    SX_CUDA(cudaMemcpyAsync(h, d, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  const size_t chunk = size_t(4) << 20;  // floats
  float* st = static_cast<float*>(ctx->h_maps.ensure(2 * chunk * 4));
  const size_t nch = (n + chunk - 1) / chunk;
  auto dma = [&](size_t i) {
    const size_t o = i * chunk, m = std::min(chunk, n - o);
    SX_CUDA(cudaMemcpyAsync(st + (i & 1) * chunk, d + o, m * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SX_CUDA(cudaEventRecord(ctx_event(ctx, i & 1), ctx->stream));
  };
  dma(0);
  for (size_t i = 0; i < nch; ++i) {
    if (i + 1 < nch) dma(i + 1);  // its slot's previous chunk (i - 1) is already copied out
    SX_CUDA(cudaEventSynchronize(ctx_event(ctx, i & 1)));
    const size_t o = i * chunk;
    parallel_memcpy(h + o, st + (i & 1) * chunk, std::min(chunk, n - o) * 4);
  }
}

extern "C" int salvox_last_maps(salvox_ctx* ctx, float* score_out, float* best_scale_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->exh.valid) fail(SALVOX_EINVAL, "salvox_last_maps: no exhaustive call on this context");
    SX_CUDA(cudaSetDevice(ctx->device));
    const sx::ExhState& e = ctx->exh;
    const size_t plane = (size_t)e.nx * e.ny;
    const size_t n = plane * (e.z1 - e.z0), off = plane * (e.z0 - e.zb0);
    maps_to_host(ctx, ctx->d_score.as<float>() + off, score_out, n);
    maps_to_host(ctx, ctx->d_best.as<float>() + off, best_scale_out, n);
  });
}

extern "C" int salvox_last_maxima(salvox_ctx* ctx, salvox_maximum* out, int64_t cap,
                                  int64_t* n_out) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    const int64_t n = ctx->last_maxima_n;
    if (out && cap > 0 && n > 0) {
      const size_t bytes = (size_t)std::min(n, cap) * sizeof(salvox_maximum);
      if (ctx->stage_valid) {
        parallel_memcpy(out, ctx->h_stage.p, bytes);
      } else {  // the device copy of the last call's maxima is still resident
        SX_CUDA(cudaSetDevice(ctx->device));
        SX_CUDA(cudaMemcpyAsync(out, ctx->d_maxima.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        SX_CUDA(cudaStreamSynchronize(ctx->stream));
      }
    }
    if (n_out) *n_out = n;
  });
}

extern "C" int salvox_exhaustive_debug_hist(salvox_ctx* ctx, const int64_t* voxels, int32_t n,
                                            uint32_t* out, double* radii_out, int32_t* n_radii) {
  return guarded([&] {
    if (!ctx) fail(SALVOX_EINVAL, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->exh.valid) fail(SALVOX_EINVAL, "no exhaustive call on this context yet");
    const ExhState& st = ctx->exh;
    SX_CUDA(cudaSetDevice(ctx->device));
    const bool two_d = st.nz == 1;
    ExhRun run;
    run.tc = pick_tile(st.bins, two_d);
    int SY = 0, SZ = 0;
    run.pl = make_plan(st.scales.data(), (int)st.scales.size(), two_d, run.tc, &SY, &SZ);
    if (run.tc.quad && run.pl.qtab.empty()) run.tc.quad = false, run.tc.tmem = true;
    const int R = run.pl.R;
    const int NR = (int)run.pl.radii.size();
    const int nzs = st.zs1 - st.zs0;
    const int pitch = (st.nx + 15) / 16 * 16;
    const int BX = SY, BY = SZ / SY, BZ = run.tc.tz + 2 * R;
    cuuint64_t gdim[3] = {(cuuint64_t)st.nx, (cuuint64_t)st.ny, (cuuint64_t)nzs};
    cuuint64_t gstride[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * st.ny};
    cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)BY, (cuuint32_t)(two_d ? 1 : BZ)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode_fn()(&run.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ctx->d_bins.p, gdim,
                              gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) fail(SALVOX_ECUDA, "cuTensorMapEncodeTiled failed");
    const long long plane = (long long)st.nx * st.ny;
    for (int i = 0; i < n; ++i)
      if (voxels[i] < plane * st.z0 || voxels[i] >= plane * st.z1)
        fail(SALVOX_EINVAL, "debug voxel outside the owned planes");
    KbParams kp{};
    kp.nx = st.nx;
    kp.ny = st.ny;
    kp.nz = st.nz;
    kp.zs0 = st.zs0;
    kp.zc0 = std::max(0, st.z0 - 1);
    kp.zc1 = std::min(st.nz, st.z1 + 1);
    kp.R = R;
  kp.lag = kb_lag();
  kp.lagmode = kb_lagmode();
    kp.Rz = two_d ? 0 : R;
    kp.SY = SY;
    kp.SZ = SZ;
    kp.n_radii = NR;
    kp.bins = st.bins;
    kp.tile_bytes = (uint32_t)(BX * BY * (two_d ? 1 : BZ));
    long long* d_vox = static_cast<long long*>(ctx->d_dbg.ensure(
        (size_t)n * 8 + (size_t)n * NR * (st.bins + 1) * 4 + 256));
    uint32_t* d_out = reinterpret_cast<uint32_t*>(d_vox + n);
    SX_CUDA(cudaMemcpyAsync(d_vox, voxels, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    SX_CUDA(cudaMemsetAsync(d_out, 0, (size_t)n * NR * (st.bins + 1) * 4, ctx->stream));
    const size_t smem = kb_smem(run.tc, kp.tile_bytes);
    std::lock_guard<std::mutex> lk2(g_const_mu);
    upload_tables(ctx, run.pl, run.tc.quad);
    for (int i = 0; i < n; ++i) {  // one block per voxel, each writes its own slice
      kp.dbg_vox = d_vox + i;
      kp.dbg_out = d_out + (size_t)i * NR * (st.bins + 1);
      dispatch_kb<true>(ctx, run.tc, run.map, kp, dim3(1), smem);
    }
    SX_CUDA(cudaEventRecord(g_const_done, ctx->stream));
    SX_CUDA(cudaMemcpyAsync(out, d_out, (size_t)n * NR * (st.bins + 1) * 4, cudaMemcpyDeviceToHost,
                            ctx->stream));
    SX_CUDA(cudaStreamSynchronize(ctx->stream));
    if (radii_out) std::memcpy(radii_out, run.pl.radii.data(), NR * sizeof(double));
    if (n_radii) *n_radii = NR;
  });
}
