// common.cuh -- shared internals of libsalvox_b200 (C-ABI implementation).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/salvox_capi.h"

namespace sx {

struct Error : std::exception {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define SX_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::sx::fail(SALVOX_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// After every launch: surface launch errors; with SALVOX_DEBUG_SYNC=1 also
// synchronise and name the kernel that faulted.
bool debug_sync_enabled();
#define SX_LAUNCH_CHECK(ctx)                                                               \
  do {                                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      ::sx::fail(SALVOX_ECUDA, std::string("kernel launch (") + __FILE__ + ":" +           \
                                   std::to_string(__LINE__) + "): " + cudaGetErrorString(e_)); \
    if (::sx::debug_sync_enabled()) {                                                      \
      e_ = cudaStreamSynchronize((ctx)->stream);                                           \
      if (e_ != cudaSuccess)                                                               \
        ::sx::fail(SALVOX_ECUDA, std::string("kernel at ") + __FILE__ + ":" +              \
                                     std::to_string(__LINE__) + ": " + cudaGetErrorString(e_)); \
    }                                                                                      \
    (ctx)->launches++;                                                                     \
  } while (0)

// Growable device buffer (never shrinks; freed with the context).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* ensure(size_t n) {
    if (n > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      SX_CUDA(cudaMalloc(&p, n < 256 ? 256 : n));
      bytes = n < 256 ? 256 : n;
    }
    return p;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Pinned host staging buffer.
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* ensure(size_t n) {
    if (n > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      SX_CUDA(cudaMallocHost(&p, n));
      bytes = n;
    }
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

// Geometry of the last exhaustive call kept for salvox_exhaustive_debug_hist.
struct ExhState {
  bool valid = false;
  int nx = 0, ny = 0, nz = 0, zs0 = 0, zs1 = 0, z0 = 0, z1 = 0;
  int zb0 = 0;  // first plane held in ctx->d_score / d_best (salvox_last_maps)
  int bins = 0;
  std::vector<double> radii;
  std::vector<double> scales;
};

}  // namespace sx

struct salvox_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host<->device copies overlapped with compute
  std::vector<cudaEvent_t> events;     // pipeline events (grown on demand)
  std::mutex mu;
  uint64_t launches = 0;
  cudaEvent_t order_event = nullptr;  // salvox_ctx_wait_stream
  // bumped by every exhaustive setup: a pending exchange-form scores call
  // (salvox_exhaustive_slab_scores) is valid only while nothing else has reused
  // d_score / d_best on this context
  uint64_t exh_generation = 0;
  // kb_kernel timing (salvox_ctx_set_profiling)
  bool profiling = false;
  double kb_ms_total = 0.0;
  int64_t kb_launches = 0;
  double kb_updates_total = 0.0;
  // exhaustive path
  sx::DevBuf d_vol, d_bins, d_score, d_best, d_keys, d_keys_alt, d_cub, d_counter, d_maxima,
      d_merge_idx, d_minmax, d_dbg;
  sx::HostBuf h_stage;       // pinned: the last call's maxima (salvox_last_maxima)
  sx::HostBuf h_maps;        // pinned staging of the maps for pageable host outputs
  sx::HostBuf h_vol;         // pinned staging of a pageable host volume
  int64_t last_maxima_n = 0;
  bool stage_valid = false;  // h_stage holds them (else read d_maxima again)
  sx::ExhState exh;
  // seek path
  sx::DevBuf d_seeds, d_dets, d_geom, d_sel_a, d_sel_b, d_sel_c, d_sel_d, d_visits, d_target,
      d_seek_vol, d_seek_bins;
  ~salvox_ctx();
};

namespace sx {

void set_last_error(const std::string& msg);

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SALVOX_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return SALVOX_ERUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SALVOX_ERUNTIME;
  }
}

// Bin volume pre-pass (volume.hpp:102-105): u8 (bin + 1), 0 = outside.
void launch_bin_volume(salvox_ctx* ctx, const float* d_vol, uint8_t* d_bins, int nx, int ny,
                       int nzs, int pitch, double low, double high, int bins,
                       cudaStream_t stream = nullptr);  // null: ctx->stream
// Observed intensity range (IntensityWindow::full_range, volume.hpp:108-112).
void device_full_range(salvox_ctx* ctx, const float* d_vol, size_t n, double* low, double* high);
// Drops a context's pending exchange-form scores call (salvox_ctx_destroy).
void forget_exchange_run(salvox_ctx* ctx);

}  // namespace sx
