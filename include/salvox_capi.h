/* salvox_capi.h -- the C-ABI boundary of the B200 salient-region hot path.
 *
 * This is the thin layer the reference's C++ API (and any FFI: ctypes, cgo,
 * JNI) binds to. Plain pointers and sizes only; no C++/torch types. Every entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj). See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - Volumes are float32, x fastest: index = x + nx*(y + ny*z)
 *    (include/salvox/volume.hpp:43-46). A 2D image has nz == 1.
 *  - Every function returns a status: SALVOX_OK, or an error whose message is
 *    available from salvox_last_error() (thread-local). The status classes
 *    mirror the reference's exception types: SALVOX_EINVAL <-> std::invalid_argument
 *    (same message text), SALVOX_ERUNTIME <-> std::runtime_error.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with SALVOX_ECUDA.
 *  - A context owns one device's streams and buffers; use one context per
 *    host thread at a time (calls on one context are serialized internally).
 */
#ifndef SALVOX_CAPI_H
#define SALVOX_CAPI_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SALVOX_API __attribute__((visibility("default")))
#else
#define SALVOX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SALVOX_OK 0
#define SALVOX_EINVAL 1      /* std::invalid_argument */
#define SALVOX_ECUDA 2       /* CUDA / device failure */
#define SALVOX_EUNSUPPORTED 3 /* valid for the reference, not implemented on device */
#define SALVOX_ERUNTIME 4    /* std::runtime_error (phantom spec, IO) */

#define SALVOX_KERNEL_IDENTITY 0     /* kernel.hpp:11-15 */
#define SALVOX_KERNEL_EPANECHNIKOV 1
#define SALVOX_KERNEL_GAUSSIAN 2

/* MetaImage ElementType codes (meta_io.cpp:85-90) for the on-device widening */
#define SALVOX_MET_UCHAR 0
#define SALVOX_MET_SHORT 1
#define SALVOX_MET_USHORT 2
#define SALVOX_MET_FLOAT 3

#define SALVOX_METHOD_QUADRANT 0 /* pipeline.hpp:19 Method */
#define SALVOX_METHOD_SHIFT 1
#define SALVOX_METHOD_ABMSOD 2 /* abmsod.cpp */
#define SALVOX_METHOD_OCTANT 3 /* NEW: 3D generalisation of quadrant.cpp */

#define SALVOX_FLAG_CONVERGED 1u /* detection.hpp:11-15 */
#define SALVOX_FLAG_DEGENERATE 2u
#define SALVOX_FLAG_BOUNDARY_CLAMPED 4u

typedef struct salvox_ctx salvox_ctx;

/* IntensityWindow (volume.hpp:91-113). full_range != 0 replaces low/high by the
 * observed range, computed on the device (IntensityWindow::full_range). */
typedef struct {
  double low;
  double high;
  int32_t bins;
  int32_t full_range;
} salvox_window;

/* SaliencyMaximum (pipeline.hpp:32-36) + its linear voxel index. */
typedef struct {
  double position[3];
  double score;
  double scale;
  int64_t linear_index;
} salvox_maximum;

/* Detection (detection.hpp:18-37); H row-major. 136 bytes. */
typedef struct {
  double center[3];
  double H[9];
  double entropy_bits;
  double pdf_diff;
  double bhattacharyya;
  int32_t iterations;
  uint32_t flags;
  int32_t seed_index;
  int32_t reserved;
} salvox_detection;

/* DetectParams (pipeline.hpp:88-99) + SeedPlan (seeds.hpp:16-32) + the method
 * parameter blocks (quadrant.hpp:14-28, shift.hpp:18-34). workers is accepted
 * and ignored (the device replaces parallel_for). */
typedef struct {
  int32_t method;
  int32_t seed_mode; /* 0 lattice, 1 random */
  double seed_spacing;
  int32_t seed_count;
  int32_t top_k;
  uint64_t rng_seed;
  const double* scales;
  int32_t n_scales;
  int32_t workers;
  double dedupe_radius;
  double entropy_quantile;
  double pdf_quantile;
  double quadrant_eta;
  int32_t quadrant_max_iters;
  int32_t n_quadrant_scales; /* 0 -> lround(scales) (pipeline.cpp:323-324) */
  const int32_t* quadrant_scales;
  double shift_min_step;
  int32_t shift_max_iters;
  int32_t shift_step_kernel;
  int32_t shift_hist_kernel;
  int32_t reserved;
  double shift_min_inbounds_fraction;
  const double* shift_target; /* NULL -> uniform over bins */
  /* AbmsodParams (abmsod.hpp:19-40); method SALVOX_METHOD_ABMSOD */
  double abmsod_threshold;   /* 1e-4 */
  int32_t abmsod_max_iters;  /* 15 */
  int32_t abmsod_kernel;     /* 2 = gaussian */
  double abmsod_lambda_min;  /* 4.0 */
  double abmsod_lambda_max;  /* 0 -> (max dim / 2)^2 */
  double abmsod_min_inbounds_fraction; /* 0.1 */
  const double* abmsod_target; /* NULL -> uniform over bins */
} salvox_detect_params;

/* AbmsodParams for salvox_abmsod_run (abmsod.hpp:19-40). */
typedef struct {
  double threshold;
  int32_t max_iterations;
  int32_t kernel; /* 0 identity, 1 epanechnikov, 2 gaussian */
  double lambda_min;
  double lambda_max;
  double min_inbounds_fraction;
  const double* target; /* NULL -> uniform over bins */
} salvox_abmsod_params;

/* AbmsodIterRecord (abmsod.hpp:42-48); H row-major. */
typedef struct {
  double position[3];
  double H[9];
  double bhattacharyya;
  double max_bhattacharyya;
  double eig_min;
  double eig_max;
} salvox_abmsod_iter;

/* ------------------------------------------------------------------ context */
SALVOX_API const char* salvox_last_error(void);
SALVOX_API int salvox_version(void);
/* Creates a context on CUDA device `device`. */
SALVOX_API int salvox_ctx_create(int device, salvox_ctx** out);
SALVOX_API int salvox_ctx_destroy(salvox_ctx* ctx);
/* Binds the context to an external CUDA stream (cudaStream_t as void*); NULL
 * restores the context's own stream. Device-pointer entry points run on it. */
SALVOX_API int salvox_ctx_set_stream(salvox_ctx* ctx, void* stream);
/* Orders the context's stream after the work already queued on `stream`
 * (cudaStream_t as void*): an event recorded on `stream`, waited on by the
 * context's stream (no host synchronisation). Callers that produce device
 * inputs on another stream call this before a device-pointer entry point. */
SALVOX_API int salvox_ctx_wait_stream(salvox_ctx* ctx, void* stream);
/* Number of this library's kernel launches issued through ctx so far. */
SALVOX_API int salvox_ctx_launch_count(salvox_ctx* ctx, uint64_t* out);

/* ------------------------------------------------------- exhaustive pass (E1)
 * Replaces kadir_brady_exhaustive (include/salvox/pipeline.hpp:49-53,
 * src/pipeline.cpp:63-166). Same validation and messages (scales >= 2,
 * budget). kernel: identity or Epanechnikov (exact integer forms); Gaussian
 * -> SALVOX_EUNSUPPORTED (its weights have no exact shell form).
 * score_out / best_scale_out (nx*ny*nz floats, nullable) receive the dense map;
 * up to `cap` maxima (score-descending, ties by linear index -- the
 * reference's stable_sort order) go to `maxima`; *n_maxima is the full count
 * (fetch all with salvox_last_maxima when it exceeds cap). *visits gets the
 * reference's EvalCounter increment (nullable). */
SALVOX_API int salvox_exhaustive(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny, int32_t nz,
                      const salvox_window* iw, const double* scales, int32_t n_scales,
                      int32_t kernel, uint64_t budget, float* score_out, float* best_scale_out,
                      salvox_maximum* maxima, int64_t cap, int64_t* n_maxima, uint64_t* visits);

/* z-slab form for multi-GPU sharding: `slab` holds planes [zs0, zs1) of a
 * volume nx*ny*nz (host pointer); the call scores and selects maxima for the
 * owned planes [z0, z1) (it needs zs0 <= max(0, z0-R-1), zs1 >= min(nz, z1+R+1),
 * R = max scale + 1). Maps cover the owned planes only; maxima positions and
 * linear indices are global. budget applies to the whole volume. */
SALVOX_API int salvox_exhaustive_slab(salvox_ctx* ctx, const float* slab, int32_t nx, int32_t ny,
                           int32_t nz, int32_t zs0, int32_t zs1, int32_t z0, int32_t z1,
                           const salvox_window* iw, const double* scales, int32_t n_scales,
                           int32_t kernel, uint64_t budget, float* score_out,
                           float* best_scale_out, salvox_maximum* maxima, int64_t cap,
                           int64_t* n_maxima, uint64_t* visits);

/* Device-resident form (inputs already in HBM; used for the kernel-only
 * timing): d_volume, d_score, d_best_scale are device pointers (d_score and
 * d_best_scale nullable). Runs on the context stream; *n_maxima is written
 * after the stream synchronises. */
SALVOX_API int salvox_exhaustive_device(salvox_ctx* ctx, const float* d_volume, int32_t nx, int32_t ny,
                             int32_t nz, const salvox_window* iw, const double* scales,
                             int32_t n_scales, int32_t kernel, uint64_t budget, float* d_score,
                             float* d_best_scale, int64_t* n_maxima);

/* Device-resident z-slab form: d_slab (device) holds planes [zs0, zs1) of the
 * volume; scores the owned planes [z0, z1) (same halo rule as
 * salvox_exhaustive_slab). d_score / d_best_scale (device, nullable) receive the
 * owned-plane maps. */
SALVOX_API int salvox_exhaustive_slab_device(salvox_ctx* ctx, const float* d_slab, int32_t nx,
                                             int32_t ny, int32_t nz, int32_t zs0, int32_t zs1,
                                             int32_t z0, int32_t z1, const salvox_window* iw,
                                             const double* scales, int32_t n_scales,
                                             int32_t kernel, uint64_t budget, float* d_score,
                                             float* d_best_scale, int64_t* n_maxima);

/* z-slab form with a neighbour-plane exchange (multi-GPU; the split of
 * salvox_exhaustive_slab a rank uses when its neighbours exchange boundary
 * planes instead of each scoring one extra plane per side -- replaces the same
 * reference call, src/pipeline.cpp:63-166, for one slab of a sharded volume).
 * 1) salvox_exhaustive_slab_scores: bins the slab and scores ONLY the owned
 *    planes [z0, z1); `slab`, `score_out`, `best_scale_out` are host pointers
 *    (on_device = 0; pipelined H2D/compute/D2H) or device pointers
 *    (on_device = 1); no maxima yet. Same validation and halo rule as
 *    salvox_exhaustive_slab; *visits gets the owned planes' EvalCounter share.
 * 2) salvox_exhaustive_slab_edges: the first and last owned score planes into
 *    device buffers (nx*ny floats each, nullable) -- what the neighbours need.
 * 3) salvox_exhaustive_slab_maxima: d_below = plane z0-1 (the lower
 *    neighbour's last owned plane; required when z0 > 0), d_above = plane z1
 *    (the upper neighbour's first; required when z1 < nz), device pointers;
 *    strict maxima of the owned planes, in the reference's order, as
 *    salvox_exhaustive_slab returns them; maxima == NULL leaves them on the
 *    device (salvox_last_maxima / salvox_last_maxima_device). */
SALVOX_API int salvox_exhaustive_slab_scores(salvox_ctx* ctx, const float* slab, int32_t on_device,
                                             int32_t nx, int32_t ny, int32_t nz, int32_t zs0,
                                             int32_t zs1, int32_t z0, int32_t z1,
                                             const salvox_window* iw, const double* scales,
                                             int32_t n_scales, int32_t kernel, uint64_t budget,
                                             float* score_out, float* best_scale_out,
                                             uint64_t* visits);
SALVOX_API int salvox_exhaustive_slab_edges(salvox_ctx* ctx, float* d_first, float* d_last);
SALVOX_API int salvox_exhaustive_slab_maxima(salvox_ctx* ctx, const float* d_below,
                                             const float* d_above, salvox_maximum* maxima,
                                             int64_t cap, int64_t* n_maxima);

/* Copies the maxima of the last exhaustive call on ctx. */
SALVOX_API int salvox_last_maxima(salvox_ctx* ctx, salvox_maximum* out, int64_t cap, int64_t* n_out);

/* The owned-plane score / best-scale maps ((z1-z0)*ny*nx floats each; either
 * nullable) of the last exhaustive call on ctx, which keeps them on the device.
 * A caller can run the pass with null maps, allocate its result arrays while
 * it runs, and fetch them here (the C++ drop-in's kadir_brady_exhaustive does).
 * Pinned buffers take one DMA; pageable ones go through pinned staging.
 * SALVOX_EINVAL when ctx has run no exhaustive call. */
SALVOX_API int salvox_last_maps(salvox_ctx* ctx, float* score_out, float* best_scale_out);
/* Device form: the last call's maxima into a device buffer (D2D). */
SALVOX_API int salvox_last_maxima_device(salvox_ctx* ctx, salvox_maximum* d_out, int64_t cap,
                                         int64_t* n_out);
/* Sorts n maxima records (device) into the reference's order -- score
 * descending, ties by linear index ascending (the stable_sort of
 * src/pipeline.cpp:163-164) -- on the device: the merge of the per-slab lists a
 * multi-GPU run all-gathers. d_in and d_out are device buffers of n records. */
SALVOX_API int salvox_merge_maxima_device(salvox_ctx* ctx, const salvox_maximum* d_in, int64_t n,
                                          salvox_maximum* d_out);

/* Exact integer identity-kernel histograms of the last exhaustive call, for
 * `n` voxels (global linear indices in the owned planes) at every needed
 * radius r (ascending, written to radii_out): out[v][r][0..bins-1] = S_b(r) and
 * out[v][r][bins] = T(r) = sum_b S_b(r) (uint32; out holds n*n_radii*(bins+1)).
 * Debug / parity entry point: recomputes those voxels with the same kernel
 * body (one CTA per voxel). radii_out must hold 3*n_scales doubles. */
SALVOX_API int salvox_exhaustive_debug_hist(salvox_ctx* ctx, const int64_t* voxels, int32_t n,
                                 uint32_t* out, double* radii_out, int32_t* n_radii);

/* ---------------------------------------------------- seed-grid detector (E2/E3)
 * Replaces detect (include/salvox/pipeline.hpp:103-104, src/pipeline.cpp:311-402):
 * seed planning, per-seed seek (shift / quadrant / octant) on the device, then
 * thresholds + dedupe on the device. out receives up to cap detections;
 * *n_out the count. per_seed (nullable, cap_seed) receives every trajectory's
 * pre-selection detection in seed order; *n_seed its count. */
SALVOX_API int salvox_detect(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny, int32_t nz,
                  const salvox_window* iw, const salvox_detect_params* params,
                  salvox_detection* out, int64_t cap, int64_t* n_out,
                  salvox_detection* per_seed, int64_t cap_seed, int64_t* n_seed,
                  uint64_t* visits);

/* Device-resident form of detect over a batch of `batch` volumes stored back
 * to back at d_volumes (device pointer). For each volume the selected
 * detections go to out[v*cap ...] and the count to n_out[v] (host arrays). */
SALVOX_API int salvox_detect_batch_device(salvox_ctx* ctx, const float* d_volumes, int32_t batch,
                               int32_t nx, int32_t ny, int32_t nz, const salvox_window* iw,
                               const salvox_detect_params* params, salvox_detection* out,
                               int64_t cap, int64_t* n_out, uint64_t* visits);

/* One rank's share of detect() on a replicated volume: the
 * seeds/trajectories of detect's plan (pipeline.cpp:311-381) with plan position
 * j % world == rank, per-seed detections in increasing j. The caller gathers
 * the shards (position j = rank + world * i), restores plan order and runs
 * salvox_select once on the whole population, because the thresholds are
 * global quantiles (pipeline.cpp:389-399). n_total = size of the whole plan. */
SALVOX_API int salvox_detect_shard(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                   int32_t nz, const salvox_window* iw,
                                   const salvox_detect_params* params, int32_t rank,
                                   int32_t world, salvox_detection* per_seed, int64_t cap,
                                   int64_t* n_local, int64_t* n_total, uint64_t* visits);

/* Per-seed seek only (saliency_shift shift.hpp:57-59 / quadrant_seek
 * quadrant.hpp:73-76 / octant), seeds given explicitly: positions (3 per seed),
 * seed_scales (shift: isotropic half extent s, window (s,s,s) or (s,s,1) in 2D;
 * ignored for quadrant/octant), seed_half_extents (nullable, 3 per seed:
 * ShiftParams::half_extents, overrides seed_scales; z is pinned to 1 in 2D as
 * shift.cpp:9 does), seed indices (nullable -> 0..n-1). Writes one detection
 * per seed in seed order. */
SALVOX_API int salvox_seek(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny, int32_t nz,
                const salvox_window* iw, const salvox_detect_params* params,
                const double* seed_positions, const double* seed_scales,
                const double* seed_half_extents, const int32_t* seed_index, int64_t n,
                salvox_detection* out, uint64_t* visits);

/* abmsod_run (abmsod.hpp:77-79, src/abmsod.cpp:43-169) for n seeds: seed window
 * = seed_H (9 doubles per seed, row-major) or, when seed_H is NULL,
 * EllipsoidWindow::isotropic(seed, radii[i]) (window.hpp:46-48). One detection
 * per seed in seed order. trace (nullable) receives max_iterations
 * AbmsodIterRecords per seed, n_trace[i] of them valid. Eigen-solver failure
 * -> SALVOX_ERUNTIME "abmsod: eigen decomposition failed" (it throws). */
SALVOX_API int salvox_abmsod_run(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                 int32_t nz, const salvox_window* iw,
                                 const salvox_abmsod_params* params, const double* seeds,
                                 const double* seed_H, const double* radii, int64_t n,
                                 salvox_detection* out, salvox_abmsod_iter* trace,
                                 int32_t* n_trace, uint64_t* visits);

/* bandwidth_from_moment (abmsod.hpp:66-70, src/abmsod.cpp:23-41): host-side 3x3
 * math shared with the kernel (include/salvox/sx_eig3.h). */
SALVOX_API int salvox_bandwidth_from_moment(const double* outer, double weight_sum, int32_t dim,
                                            double lambda_min, double lambda_max, double* H);

/* Raw ascent trajectories: quadrant_seek / quadrant_seek_one (quadrant.hpp:64-76,
 * src/quadrant.cpp:83-125; dims = 2, nz must be 1) or the NEW octant ascent
 * (dims = 3). scales = QuadrantParams::scale_range (strictly increasing);
 * seeds hold 3 doubles each. No post-scoring (unlike salvox_detect). */
typedef struct {
  double position[3];
  double entropy_bits; /* entropy of the highest-entropy quadrant/octant window */
  int32_t best_scale;  /* its argmax scale */
  int32_t iterations;
  int32_t converged;
  int32_t degenerate;
} salvox_ascent_result;

SALVOX_API int salvox_ascent_seek(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                  int32_t nz, const salvox_window* iw, int32_t dims,
                                  const int32_t* scales, int32_t n_scales, double eta,
                                  int32_t max_iters, const double* seeds, int64_t n,
                                  salvox_ascent_result* out, uint64_t* visits);

/* One ascent STEP per point: quadrant_step (quadrant.hpp:66-71,
 * src/quadrant.cpp:37-81; dims = 2, nz must be 1) or the octant step (dims = 3):
 * the moved (clamped) position in moved[3 * i] and the step's state. */
typedef struct {
  double entropy[8];      /* best entropy per quadrant (NE, NW, SW, SE) / octant (bits) */
  int32_t best_scale[8];  /* its argmax scale (smallest wins ties) */
  double norm_entropy[8]; /* entropies normalised to sum 1 (0 when degenerate) */
  double displacement[3];
  int32_t degenerate;     /* every quadrant carried zero entropy */
  int32_t pad_;
} salvox_ascent_state;

SALVOX_API int salvox_ascent_step(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                  int32_t nz, const salvox_window* iw, int32_t dims,
                                  const int32_t* scales, int32_t n_scales, const double* points,
                                  int64_t n, double* moved, salvox_ascent_state* states,
                                  uint64_t* visits);

/* Window operations of the seek path, one warp per op, all ops of a call in one
 * launch, each with the reference's fp64 operation order (bit-exact sums):
 *   SALVOX_WOP_HIST        try_candidate_histogram (window.hpp:115-117,
 *                          src/window.cpp:5-19): pmf -> pmf_out row, ok = 0 for
 *                          nullopt; support = the support voxel count (the
 *                          numerator of inbounds_support_fraction, window.cpp:54-60)
 *   SALVOX_WOP_SHIFT_STEP  shift_step (shift.hpp:49-52, src/shift.cpp:15-34):
 *                          value = the new position, ok = 0 for nullopt; pmf_out
 *                          row = the candidate pmf at the old position
 *   SALVOX_WOP_PDF_DIFF    pdf_difference (window.hpp:127-135, src/window.cpp:30-46):
 *                          value[0]; ok = -1 degenerate scale, 0 degenerate
 *                          flank (both thrown as std::invalid_argument)
 *   SALVOX_WOP_BOX_ENTROPY box_entropy_bits (quadrant.hpp:58-60,
 *                          src/quadrant.cpp:18-35) of the inclusive integer box
 *                          inside the real corners box[6] = (x0, x1, y0, y1, z0, z1),
 *                          0 below min_voxels; value[0]
 * visits = what the reference call adds to its EvalCounter. */
#define SALVOX_WOP_HIST 0
#define SALVOX_WOP_SHIFT_STEP 1
#define SALVOX_WOP_PDF_DIFF 2
#define SALVOX_WOP_BOX_ENTROPY 3
typedef struct {
  int32_t op;
  int32_t kernel;      /* histogram kernel (HIST, SHIFT_STEP, PDF_DIFF) */
  int32_t step_kernel; /* SHIFT_STEP */
  int32_t min_voxels;  /* BOX_ENTROPY */
  double center[3];
  double H[9];         /* bandwidth matrix, row-major (HIST, SHIFT_STEP, PDF_DIFF) */
  double box[6];       /* BOX_ENTROPY */
} salvox_window_op;
typedef struct {
  double value[3];
  uint64_t support;
  uint64_t visits;
  int32_t ok;
  int32_t pad_;
} salvox_window_result;

SALVOX_API int salvox_window_ops(salvox_ctx* ctx, const float* volume, int32_t nx, int32_t ny,
                                 int32_t nz, const salvox_window* iw, const double* target,
                                 const salvox_window_op* ops, int64_t n, salvox_window_result* out,
                                 double* pmf_out);

/* Thresholds + dedupe (pipeline.cpp:383-401, :54-59, :168-183) on the device. */
SALVOX_API int salvox_select(salvox_ctx* ctx, const salvox_detection* dets, int64_t n, double q_entropy,
                  double q_pdf, int32_t k, double radius, salvox_detection* out,
                  int64_t* n_out);
/* dedupe_top_k alone (pipeline.hpp:57). */
SALVOX_API int salvox_dedupe_top_k(salvox_ctx* ctx, const salvox_detection* dets, int64_t n, int32_t k,
                        double radius, salvox_detection* out, int64_t* n_out);

/* ------------------------------------------------------- host-side data formats */
/* plan_seeds (seeds.hpp:43): pass cap = 0 to query the count. */
SALVOX_API int salvox_plan_seeds(int32_t nx, int32_t ny, int32_t nz, int32_t mode, double spacing,
                      int32_t count, const double* scales, int32_t n_scales, uint64_t rng_seed,
                      double* positions, double* seed_scales, int64_t cap, int64_t* n_out);

/* load_volume's payload widening (meta_io.cpp:30-33, :100-105) on the device
 * (SURVEY 8(f) rank 2): salvox_upload_widen copies a host payload of n elements
 * at its native width and widens it to f32 into d_out (device); the _device
 * form widens a device payload. static_cast<float> of u8/i16/u16 is exact. */
SALVOX_API int salvox_upload_widen(salvox_ctx* ctx, int32_t element_type, const void* raw,
                                   int64_t n, float* d_out);
SALVOX_API int salvox_widen_device(salvox_ctx* ctx, int32_t element_type, const void* d_raw,
                                   int64_t n, float* d_out);

/* rasterize_window (pipeline.hpp:61, src/pipeline.cpp:185-192): the linear
 * indices (ascending) of the in-bounds voxels of the window (center, H
 * row-major) on an nx*ny*nz frame; up to cap go to out, *n_out = count. The
 * evaluation path of `salvox eval` (Jaccard vs ground-truth masks). */
SALVOX_API int salvox_rasterize_window(salvox_ctx* ctx, int32_t nx, int32_t ny, int32_t nz,
                                       const double* center, const double* H, uint64_t* out,
                                       int64_t cap, int64_t* n_out);

/* hu_moments (hu.hpp:16, src/hu.cpp:8-58) of an nx*ny float image on the
 * device (out7 = the 7 invariants); SALVOX_EINVAL "hu_moments: zero total
 * mass" like the reference's throw. */
SALVOX_API int salvox_hu_moments(salvox_ctx* ctx, const float* image, int32_t nx, int32_t ny,
                                 double* out7);
/* hu_template_distance (pipeline.hpp:73-74, src/pipeline.cpp:218-256) for n
 * detections: mean Hu distance of `slices` axial crops about each detection's
 * central slice to the template; +inf when no crop has mass. hu_filter is the
 * argmin of these (first minimum). */
SALVOX_API int salvox_hu_template_distance(salvox_ctx* ctx, const float* volume, int32_t nx,
                                           int32_t ny, int32_t nz, const salvox_detection* dets,
                                           int64_t n, const float* tmpl, int32_t tnx, int32_t tny,
                                           int32_t slices, double* out_dist);

/* make_phantom (phantom.hpp:125, src/phantom.cpp:364-421). shape 0 box, 1 ball,
 * 2 ellipsoid; fill_type 0 uniform(levels), 1 constant(value); bg_type 0
 * constant, 1 gaussian. Writes the volume and 3 centroid doubles per region. */
SALVOX_API int salvox_make_phantom(int32_t nx, int32_t ny, int32_t nz, int32_t bg_type, double bg_value,
                        double bg_mean, double bg_sigma, int32_t n_regions,
                        const int32_t* shape, const double* center, const double* half_extents,
                        const double* radius, const double* axes, const int32_t* fill_type,
                        const int32_t* fill_levels, const double* fill_value, uint64_t rng_seed,
                        float* out_volume, double* out_centroids);

/* make_phantom generated ON THE DEVICE: same arguments and
 * errors as salvox_make_phantom, the volume written to device memory d_volume
 * (nx*ny*nz floats). splitmix64 is counter-based, so every voxel's draw index
 * is computed from per-row inside counts (scan) instead of a serial walk.
 * Integer/constant fills are bit-identical to the host generator; the gaussian
 * background may differ in the last float place (libdevice log/sin/cos). */
SALVOX_API int salvox_make_phantom_device(salvox_ctx* ctx, int32_t nx, int32_t ny, int32_t nz,
                        int32_t bg_type, double bg_value, double bg_mean, double bg_sigma,
                        int32_t n_regions, const int32_t* shape, const double* center,
                        const double* half_extents, const double* radius, const double* axes,
                        const int32_t* fill_type, const int32_t* fill_levels,
                        const double* fill_value, uint64_t rng_seed, float* d_volume,
                        double* out_centroids);

#ifdef __cplusplus
}
#endif
#endif
