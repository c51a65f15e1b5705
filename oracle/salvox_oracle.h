/* salvox_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (salvox, /root/reference/proj) hot path,
 * used as the CHECKER by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. Nothing in the product (paper_1310_6736_b200/) links,
 * imports or calls this code.
 *
 * Parity status: the reference cannot be compiled here (Eigen3 and vendor/
 * headers are absent), so this restatement is pinned against the reference's
 * own known-answer tests and fixtures (tests/test_oracle_*.py port them), not
 * against reference binaries. Eigen 3x3 inverse/determinant rounding is
 * restated from Eigen 3.3/3.4 InverseImpl.h / Determinant.h (not verifiable
 * offline) -- see DESIGN.md "Parity".
 *
 * Arithmetic convention: compiled with -ffp-contract=off so every fp64
 * expression rounds exactly as the reference's (x86-64, no -march => no FMA).
 */
#ifndef SALVOX_ORACLE_H
#define SALVOX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:11-51 ---- */
typedef struct {
  uint64_t state;
  int have_spare;
  double spare;
} sxo_rng;

void sxo_rng_init(sxo_rng* r, uint64_t seed);
uint64_t sxo_rng_next_u64(sxo_rng* r);
double sxo_rng_next_double(sxo_rng* r);
uint64_t sxo_rng_next_below(sxo_rng* r, uint64_t n);
double sxo_rng_next_range(sxo_rng* r, double lo, double hi);
double sxo_rng_next_gaussian(sxo_rng* r);

/* ---- phantom.cpp:364-421 (make_phantom). shape: 0 box, 1 ball, 2 ellipsoid.
 * fill_type: 0 uniform(levels), 1 constant(value). bg_type: 0 constant, 1 gaussian.
 * Writes nx*ny*nz floats and 3 centroid doubles per region. Returns 0 or -1 (err). */
int sxo_make_phantom(int nx, int ny, int nz, int bg_type, double bg_value, double bg_mean,
                     double bg_sigma, int n_regions, const int* shape, const double* center,
                     const double* half_extents, const double* radius, const double* axes,
                     const int* fill_type, const int* fill_levels, const double* fill_value,
                     uint64_t rng_seed, float* out_volume, double* out_centroids, char* err,
                     int err_len);

/* ---- volume.hpp:102-105 ---- */
int sxo_bin_of(double low, double high, int bins, double intensity);

/* ---- pipeline.cpp:63-166 kadir_brady_exhaustive ----
 * mode 0 = literal (reference loop order, fp64 fl(n/r^2) sums);
 * mode 1 = exact (integer shell sums S_b(r), p_b = S_b/T in fp64).
 * kernel: 0 identity, 1 epanechnikov, 2 gaussian (literal mode only for 2).
 * z_begin/z_end and y_begin/y_end restrict the scored rows (bounded
 * CPU-baseline samples); pass 0, 0 for the whole range. threads >= 1 splits the
 * (z, y) rows over pthreads (each voxel is independent: results are identical).
 * Returns 0, or -1 with err (invalid_argument semantics). */
int sxo_exhaustive(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double* scales, int n_scales, int kernel, uint64_t budget, int mode,
                   int threads, int z_begin, int z_end, int y_begin, int y_end, float* score,
                   float* best_scale, uint64_t* visits, char* err, int err_len);

/* Exact integer histograms S_b(r) (b = 0..bins-1) and T(r) around one voxel
 * for the identity kernel: S_b(r) = sum over in-bounds offsets o with
 * make_sphere_offsets membership of |o|^2 for voxels in bin b. */
int sxo_voxel_shell_hist(const float* vol, int nx, int ny, int nz, double low, double high,
                         int bins, int x, int y, int z, double radius, uint64_t* S);

/* pipeline.cpp:143-165 strict 26-neighbour maxima, stable-sorted by score desc.
 * Writes up to cap records; returns the total count found. */
int64_t sxo_local_maxima(const float* score, const float* best_scale, int nx, int ny, int nz,
                         double* pos, double* sc, double* scale, int64_t* lin, int64_t cap);

/* ---- detection.hpp:18-37 ---- */
typedef struct {
  double center[3];
  double H[9]; /* row-major */
  double entropy_bits;
  double pdf_diff;
  double bhattacharyya;
  int32_t iterations;
  uint32_t flags;
  int32_t seed_index;
  int32_t reserved; /* oracle: 1 = abmsod eigen failure (runtime_error) */
} sxo_detection;

/* ---- seeds.cpp:7-45 ---- mode 0 lattice, 1 random. Writes positions (3 per
 * seed) and scales, index = order. Returns seed count (or -1 on invalid plan);
 * pass cap=0 to query. */
int64_t sxo_plan_seeds(int nx, int ny, int nz, int mode, double spacing, int count,
                       const double* scales, int n_scales, uint64_t rng_seed, double* pos,
                       double* seed_scale, int64_t cap);

/* math variant, a bit set: 0 = glibc log/exp/pow (reference); bit 1 = the
 * shared portable log sx_log (entropies), bit 2 = sx_exp (Gaussian kernel),
 * bit 4 = sx_pow (EllipsoidWindow::scale) -- the device's functions
 * (include/salvox/sx_log.h). */
void sxo_set_log_mode(int mode);

/* ---- shift.cpp:15-34 shift_step. kernels: 0 id, 1 epan, 2 gauss.
 * target may be NULL (uniform). Returns 1 and writes out[3], or 0 (nullopt). */
int sxo_shift_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double x[3], const double half[3], int step_kernel, int hist_kernel,
                   const double* target, double out[3], uint64_t* visits);

/* ---- shift.cpp:36-107 saliency_shift ---- */
int sxo_saliency_shift(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double seed[3], const double half[3], int step_kernel,
                       int hist_kernel, int max_iters, double min_step, const double* target,
                       double min_inbounds_fraction, sxo_detection* out, uint64_t* visits);

/* ---- window.cpp:5-19 / :30-46 / :54-60 (isotropic or diagonal windows) ---- */
int sxo_candidate_histogram(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, const double center[3], const double H[9], int kernel,
                            double* p_out, uint64_t* visits);
int sxo_pdf_difference(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double center[3], const double H[9], int kernel, double* out,
                       uint64_t* visits);
double sxo_entropy_bits(const double* p, int bins);

/* ---- quadrant.cpp:18-81 ---- */
double sxo_box_entropy_bits(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, double x0, double x1, double y0, double y1, double z0,
                            double z1, int min_voxels, uint64_t* visits);
typedef struct {
  double entropy[8];
  int32_t best_scale[8];
  double norm_entropy[8];
  double displacement[3];
  int32_t degenerate;
  int32_t pad_;
} sxo_ascent_state;
/* dims = 2 (quadrant, nz must be 1) or 3 (octant, NEW -- generalises quadrant). */
int sxo_ascent_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                    int dims, const double p[3], const int* scales, int n_scales,
                    double moved[3], sxo_ascent_state* st, uint64_t* visits);
typedef struct {
  double position[3];
  int32_t best_scale;
  int32_t iterations;
  double entropy_bits;
  int32_t converged;
  int32_t degenerate;
} sxo_ascent_result;
int sxo_ascent_seek_one(const float* vol, int nx, int ny, int nz, double low, double high,
                        int bins, int dims, const double seed[3], const int* scales, int n_scales,
                        double eta, int max_iters, sxo_ascent_result* out, uint64_t* visits);

/* ---- pipeline.cpp:311-402 detect ----
 * method: 0 quadrant, 1 shift, 3 octant (2 = abmsod is out of scope -> -1).
 * per_seed (optional, cap_seed) receives the pre-selection detections in seed
 * order; out receives the selected detections. Returns the number selected or -1. */
typedef struct {
  int method;
  int seed_mode;
  double seed_spacing;
  int seed_count;
  uint64_t rng_seed;
  const double* scales;
  int n_scales;
  int top_k;
  double dedupe_radius;
  double entropy_quantile;
  double pdf_quantile;
  int workers;
  double quadrant_eta;
  int quadrant_max_iters;
  const int* quadrant_scales; /* NULL -> lround(scales) */
  int n_quadrant_scales;
  double shift_min_step;
  int shift_max_iters;
  int shift_step_kernel;
  int shift_hist_kernel;
  double shift_min_inbounds_fraction;
  /* AbmsodParams (abmsod.hpp:19-40), method 2 */
  double abmsod_threshold;
  int abmsod_max_iters;
  int abmsod_kernel;
  double abmsod_lambda_min;
  double abmsod_lambda_max;
  double abmsod_min_inbounds_fraction;
} sxo_detect_params;
int64_t sxo_detect(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const sxo_detect_params* params, sxo_detection* per_seed, int64_t cap_seed,
                   int64_t* n_seed_out, sxo_detection* out, int64_t cap, uint64_t* visits,
                   char* err, int err_len);

/* pipeline.cpp:54-59 / :383-401 / :168-183 */
int64_t sxo_select(const sxo_detection* dets, int64_t n, double q_entropy, double q_pdf, int k,
                   double radius, sxo_detection* out);
int64_t sxo_dedupe_top_k(const sxo_detection* dets, int64_t n, int k, double radius,
                         sxo_detection* out);

/* ---- abmsod.cpp:43-169 abmsod_run. Returns 0, -1 (AbmsodParams::validate
 * throws), -2 (eigen decomposition failed: std::runtime_error). trace (nullable)
 * receives up to trace_cap AbmsodIterRecords (abmsod.hpp:42-48). */
typedef struct {
  double threshold;
  int max_iterations;
  int kernel;
  double lambda_min;
  double lambda_max;
  double min_inbounds_fraction;
  const double* target; /* NULL -> uniform */
} sxo_abmsod_params;
typedef struct {
  double position[3];
  double H[9];
  double bhattacharyya;
  double max_bhattacharyya;
  double eig_min;
  double eig_max;
} sxo_abmsod_iter;
int sxo_abmsod_run(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double seed_center[3], const double seed_H[9],
                   const sxo_abmsod_params* params, sxo_detection* det, sxo_abmsod_iter* trace,
                   int trace_cap, int* n_trace, uint64_t* visits);
/* abmsod.cpp:23-41 (0 ok, 1/2 invalid_argument, 3 runtime_error) */
int sxo_bandwidth_from_moment(const double outer[9], double wsum, int dim, double lambda_min,
                              double lambda_max, double H[9]);
/* SelfAdjointEigenSolver<Matrix3d> restatement: ascending values, vectors as columns */
int sxo_sym_eigen3(const double a[9], double values[3], double vectors[9]);
double sxo_exp_portable(double x);
double sxo_pow_portable(double x, double y);

/* pipeline.cpp:185-192 rasterize_window; returns the count (writes up to cap) */
int64_t sxo_rasterize_window(int nx, int ny, int nz, const double center[3], const double H[9],
                             uint64_t* out, int64_t cap);

/* hu.cpp:8-58 (pitch = row stride in floats); -1 on zero mass. And
 * pipeline.cpp:218-256 hu_template_distance (-1 if the template has no mass). */
int sxo_hu_moments(const float* img, int nx, int ny, int pitch, double out[7]);
double sxo_hu_template_distance(const float* vol, int nx, int ny, int nz, const double center[3],
                                const double H[9], const float* tmpl, int tnx, int tny, int slices);

/* Eigen 3x3 inverse / determinant restatement (exported for tests). */
void sxo_eigen_inverse3(const double m[9], double out[9]);
double sxo_eigen_det3(const double m[9]);
double sxo_log_portable(double x);

#ifdef __cplusplus
}
#endif
#endif
