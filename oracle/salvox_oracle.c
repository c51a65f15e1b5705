/* salvox_oracle.c -- TEST INFRASTRUCTURE ONLY (see salvox_oracle.h).
 *
 * CPU restatement of the reference hot path. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Compile with -ffp-contract=off (oracle/Makefile).
 */
#define _GNU_SOURCE
#include "salvox_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/salvox/sx_eig3.h"
#include "../include/salvox/sx_log.h"

#define LN2_STD 0.693147180559945309417232121458176568 /* std::numbers::ln2 */
#define PI_STD 3.141592653589793238462643383279502884  /* std::numbers::pi */

static int g_log_mode = 0; /* bit set: 1 sx_log, 2 sx_exp, 4 sx_pow (else glibc) */
void sxo_set_log_mode(int mode) { g_log_mode = mode; }
static double olog(double x) { return (g_log_mode & 1) ? sx_log(x) : log(x); }
static double oexp(double x) { return (g_log_mode & 2) ? sx_exp(x) : exp(x); }
static double opow(double x, double y) { return (g_log_mode & 4) ? sx_pow(x, y) : pow(x, y); }
double sxo_log_portable(double x) { return sx_log(x); }
double sxo_exp_portable(double x) { return sx_exp(x); }
double sxo_pow_portable(double x, double y) { return sx_pow(x, y); }

static void set_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    strncpy(err, msg, (size_t)len - 1);
    err[len - 1] = 0;
  }
}

static inline int imax(int a, int b) { return a > b ? a : b; }
static inline int imin(int a, int b) { return a < b ? a : b; }
static inline double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ------------------------------------------------------------------ rng.hpp:11-51 */
void sxo_rng_init(sxo_rng* r, uint64_t seed) {
  r->state = seed;
  r->have_spare = 0;
  r->spare = 0.0;
}
uint64_t sxo_rng_next_u64(sxo_rng* r) { /* rng.hpp:15-20 */
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
double sxo_rng_next_double(sxo_rng* r) { return (double)(sxo_rng_next_u64(r) >> 11) * 0x1.0p-53; }
uint64_t sxo_rng_next_below(sxo_rng* r, uint64_t n) { return sxo_rng_next_u64(r) % n; }
double sxo_rng_next_range(sxo_rng* r, double lo, double hi) {
  return lo + (hi - lo) * sxo_rng_next_double(r);
}
double sxo_rng_next_gaussian(sxo_rng* r) { /* rng.hpp:32-45 */
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = sxo_rng_next_double(r);
  double u2 = sxo_rng_next_double(r);
  while (u1 <= 0.0) u1 = sxo_rng_next_double(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(theta);
  r->have_spare = 1;
  return rr * cos(theta);
}

/* ------------------------------------------------ Eigen 3x3 (InverseImpl.h, Determinant.h)
 * Row-major m[r*3+c]. cofactor(i,j) = m(i1,j1)*m(i2,j2) - m(i1,j2)*m(i2,j1),
 * i1=(i+1)%3, i2=(i+2)%3 (same for j). det = sum(cofactor_col0 .* col0);
 * result(i,j) = cofactor(j,i) * (1/det). */
static double cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[i1 * 3 + j1] * m[i2 * 3 + j2] - m[i1 * 3 + j2] * m[i2 * 3 + j1];
}
void sxo_eigen_inverse3(const double m[9], double out[9]) {
  const double c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  const double det = (c0 * m[0] + c1 * m[3]) + c2 * m[6];
  const double invdet = 1.0 / det;
  double r[9];
  r[1 * 3 + 2] = cof3(m, 2, 1) * invdet;
  r[2 * 3 + 1] = cof3(m, 1, 2) * invdet;
  r[2 * 3 + 2] = cof3(m, 2, 2) * invdet;
  r[1 * 3 + 0] = cof3(m, 0, 1) * invdet;
  r[1 * 3 + 1] = cof3(m, 1, 1) * invdet;
  r[2 * 3 + 0] = cof3(m, 0, 2) * invdet;
  r[0] = c0 * invdet;
  r[1] = c1 * invdet;
  r[2] = c2 * invdet;
  memcpy(out, r, sizeof r);
}
double sxo_eigen_det3(const double m[9]) { /* bruteforce_det3_helper(0,1,2)-(1,0,2)+(2,0,1) */
  const double a = m[0] * (m[4] * m[8] - m[5] * m[7]);
  const double b = m[1] * (m[3] * m[8] - m[5] * m[6]);
  const double c = m[2] * (m[3] * m[7] - m[4] * m[6]);
  return a - b + c;
}

/* ------------------------------------------------------- phantom.cpp:198-222, 364-421 */
static void region_H(int shape, const double* half, double radius, const double* axes, double* H) {
  memset(H, 0, 9 * sizeof(double));
  if (shape == 0) {
    H[0] = half[0] * half[0];
    H[4] = half[1] * half[1];
    H[8] = half[2] * half[2];
  } else if (shape == 1) {
    H[0] = H[4] = H[8] = (1.0 * radius) * radius; /* Identity() * r * r */
  } else {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) /* axes * axes^T: Eigen's lazy-product redux t0 + (t1 + t2) */
        H[i * 3 + j] = axes[i * 3 + 0] * axes[j * 3 + 0] +
                       (axes[i * 3 + 1] * axes[j * 3 + 1] + axes[i * 3 + 2] * axes[j * 3 + 2]);
  }
}

int sxo_make_phantom(int nx, int ny, int nz, int bg_type, double bg_value, double bg_mean,
                     double bg_sigma, int n_regions, const int* shape, const double* center,
                     const double* half_extents, const double* radius, const double* axes,
                     const int* fill_type, const int* fill_levels, const double* fill_value,
                     uint64_t rng_seed, float* v, double* out_centroids, char* err, int err_len) {
  if (nx < 1 || ny < 1 || nz < 1) {
    set_err(err, err_len, "Volume: dims must be >= 1");
    return -1;
  }
  const size_t n = (size_t)nx * ny * nz;
  sxo_rng rng;
  sxo_rng_init(&rng, rng_seed);
  if (bg_type == 0) {
    for (size_t i = 0; i < n; ++i) v[i] = (float)bg_value;
  } else {
    for (size_t i = 0; i < n; ++i) v[i] = (float)(bg_mean + bg_sigma * sxo_rng_next_gaussian(&rng));
  }
  uint8_t* occupied = (uint8_t*)calloc(n, 1);
  const int dims[3] = {nx, ny, nz};
  for (int ri = 0; ri < n_regions; ++ri) {
    const double* c = center + 3 * ri;
    const double* half = half_extents + 3 * ri;
    double H[9], Hinv[9], ext[3];
    region_H(shape[ri], half, radius[ri], axes + 9 * ri, H);
    for (int i = 0; i < 3; ++i)
      ext[i] = shape[ri] == 0 ? half[i] : sqrt(H[i * 4] > 0.0 ? H[i * 4] : 0.0);
    for (int i = 0; i < 3; ++i) {
      if (c[i] - ext[i] < 0.0 || c[i] + ext[i] > dims[i] - 1) {
        set_err(err, err_len, "make_phantom: region extends outside the volume");
        free(occupied);
        return -1;
      }
    }
    if (shape[ri] != 0) sxo_eigen_inverse3(H, Hinv);
    int lo[3], hi[3];
    for (int i = 0; i < 3; ++i) {
      lo[i] = imax(0, (int)floor(c[i] - ext[i]));
      hi[i] = imin(dims[i] - 1, (int)ceil(c[i] + ext[i]));
    }
    double cs[3] = {0.0, 0.0, 0.0};
    uint64_t cnt = 0;
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          const double d[3] = {x - c[0], y - c[1], z - c[2]};
          int inside;
          if (shape[ri] == 0) {
            inside = fabs(d[0]) <= half[0] && fabs(d[1]) <= half[1] && fabs(d[2]) <= half[2];
          } else {
            double hd[3];
            for (int i = 0; i < 3; ++i)
              hd[i] = Hinv[i * 3 + 0] * d[0] + (Hinv[i * 3 + 1] * d[1] + Hinv[i * 3 + 2] * d[2]);
            inside = ((d[0] * hd[0] + d[1] * hd[1]) + d[2] * hd[2]) <= 1.0;
          }
          if (!inside) continue;
          const size_t idx = (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z);
          if (occupied[idx]) {
            set_err(err, err_len, "make_phantom: regions overlap");
            free(occupied);
            return -1;
          }
          occupied[idx] = 1;
          if (fill_type[ri] == 0)
            v[idx] = (float)sxo_rng_next_below(&rng, (uint64_t)fill_levels[ri]);
          else
            v[idx] = (float)fill_value[ri];
          ++cnt;
          cs[0] += x;
          cs[1] += y;
          cs[2] += z;
        }
    if (cnt == 0) {
      set_err(err, err_len, "make_phantom: region rasterizes to no voxel");
      free(occupied);
      return -1;
    }
    if (out_centroids)
      for (int i = 0; i < 3; ++i) out_centroids[3 * ri + i] = cs[i] / (double)cnt;
  }
  free(occupied);
  return 0;
}

/* ------------------------------------------------------------- volume.hpp:102-105 */
int sxo_bin_of(double low, double high, int bins, double intensity) {
  const int b = (int)floor((intensity - low) / (high - low) * bins);
  return b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
}

/* ------------------------------------------------------------ histogram.hpp:21-67 */
static int normalize_hist(double* p, int bins) { /* histogram.hpp:28-33; returns 0 if mass<=0 */
  double s = 0.0;
  for (int b = 0; b < bins; ++b) s += p[b];
  if (s <= 0.0) return 0;
  for (int b = 0; b < bins; ++b) p[b] /= s;
  return 1;
}
double sxo_entropy_bits(const double* p, int bins) { /* histogram.hpp:56-67 */
  double e = 0.0;
  for (int b = 0; b < bins; ++b)
    if (p[b] > 0.0) e -= p[b] * olog(p[b]);
  if (e < 0.0) e = 0.0;
  return e / LN2_STD;
}
static double bhattacharyya(const double* p, const double* q, int bins) { /* :95-103 */
  double rho = 0.0;
  for (int b = 0; b < bins; ++b) rho += sqrt(p[b] * q[b]);
  return rho < 1.0 ? rho : 1.0;
}
static double kernel_value(int k, double d) { /* kernel.hpp:17-24 */
  if (k == 0) return d;
  if (k == 1) return 1.0 - d;
  return oexp(-0.5 * d);
}
static double kernel_step_weight(int k, double d) { /* kernel.hpp:29-36 */
  if (k == 2) return 0.5 * oexp(-0.5 * d);
  return 1.0;
}

/* --------------------------------------------------------- pipeline.cpp:31-52 */
typedef struct {
  int n;
  int* at; /* 3 ints per offset */
  double* d;
  int* nsq;
} sphere_offsets;

static void make_sphere_offsets(double radius, int two_d, sphere_offsets* out) {
  const int r = (int)floor(radius);
  const double r2 = radius * radius;
  const int zr = two_d ? 0 : r;
  const int cap = (2 * r + 1) * (2 * r + 1) * (2 * zr + 1);
  out->at = (int*)malloc(sizeof(int) * 3 * (size_t)cap);
  out->d = (double*)malloc(sizeof(double) * (size_t)cap);
  out->nsq = (int*)malloc(sizeof(int) * (size_t)cap);
  out->n = 0;
  for (int z = -zr; z <= zr; ++z)
    for (int y = -r; y <= r; ++y)
      for (int x = -r; x <= r; ++x) {
        const double d = ((double)x * x + (double)y * y + (double)z * z) / r2;
        if (d <= 1.0) {
          out->at[3 * out->n + 0] = x;
          out->at[3 * out->n + 1] = y;
          out->at[3 * out->n + 2] = z;
          out->d[out->n] = d;
          out->nsq[out->n] = x * x + y * y + z * z;
          ++out->n;
        }
      }
}
static void free_offsets(sphere_offsets* o) {
  free(o->at);
  free(o->d);
  free(o->nsq);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* ------------------------------------------------------ pipeline.cpp:63-141 */
typedef struct {
  const float* vol;
  int nx, ny, nz, bins, kernel, mode;
  double low, high;
  const double* scales;
  int n_scales;
  const double* radii;
  int n_radii;
  sphere_offsets* offs;
  int64_t r0, r1; /* rows (z,y) of this worker, as z*ny+y in [r0, r1) */
  int ry0, ry1;    /* row window inside each plane */
  float* score;
  float* best_scale;
  uint8_t* binvol; /* exact mode: precomputed bin_of */
} exh_job;

static int radius_index(const double* radii, int n, double r) { /* lower_bound */
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (radii[mid] < r)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

static void* exh_worker(void* arg) {
  exh_job* j = (exh_job*)arg;
  const int nx = j->nx, ny = j->ny, nz = j->nz, M = j->bins, NR = j->n_radii;
  double* hists = (double*)malloc(sizeof(double) * (size_t)NR * M);
  int* normalized = (int*)malloc(sizeof(int) * (size_t)NR);
  uint64_t* S = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)NR * M);
  const int nry = j->ry1 - j->ry0;
  for (int64_t row = j->r0; row < j->r1; ++row) {
    const int z = (int)(row / nry), y = j->ry0 + (int)(row % nry);
      for (int x = 0; x < nx; ++x) {
        for (int ri = 0; ri < NR; ++ri) {
          double* h = hists + (size_t)ri * M;
          const sphere_offsets* off = &j->offs[ri];
          if (j->mode == 0) { /* literal: pipeline.cpp:105-120 */
            for (int b = 0; b < M; ++b) h[b] = 0.0;
            for (int i = 0; i < off->n; ++i) {
              const int sx = x + off->at[3 * i], sy = y + off->at[3 * i + 1],
                        sz = z + off->at[3 * i + 2];
              if (sx < 0 || sx >= nx || sy < 0 || sy >= ny || sz < 0 || sz >= nz) continue;
              const double val = j->vol[(size_t)sx + (size_t)nx * ((size_t)sy + (size_t)ny * sz)];
              h[sxo_bin_of(j->low, j->high, M, val)] += kernel_value(j->kernel, off->d[i]);
            }
            normalized[ri] = normalize_hist(h, M);
          } else { /* exact integer shell sums (identity kernel) */
            uint64_t* s = S + (size_t)ri * M;
            for (int b = 0; b < M; ++b) s[b] = 0;
            uint64_t T = 0;
            for (int i = 0; i < off->n; ++i) {
              const int sx = x + off->at[3 * i], sy = y + off->at[3 * i + 1],
                        sz = z + off->at[3 * i + 2];
              if (sx < 0 || sx >= nx || sy < 0 || sy >= ny || sz < 0 || sz >= nz) continue;
              const uint64_t w = (uint64_t)off->nsq[i];
              s[j->binvol[(size_t)sx + (size_t)nx * ((size_t)sy + (size_t)ny * sz)]] += w;
              T += w;
            }
            normalized[ri] = T > 0;
            if (T > 0)
              for (int b = 0; b < M; ++b) h[b] = (double)s[b] / (double)T;
          }
        }
        double best = 0.0, best_s = 0.0; /* pipeline.cpp:122-136 */
        for (int si = 0; si < j->n_scales; ++si) {
          const double s = j->scales[si];
          const int ic = radius_index(j->radii, NR, s), il = radius_index(j->radii, NR, s - 1.0),
                    ih = radius_index(j->radii, NR, s + 1.0);
          if (!normalized[ic] || !normalized[il] || !normalized[ih]) continue;
          const double* hc = hists + (size_t)ic * M;
          const double* hl = hists + (size_t)il * M;
          const double* hh = hists + (size_t)ih * M;
          double e = 0.0;
          for (int b = 0; b < M; ++b)
            if (hc[b] > 0.0) e -= hc[b] * log(hc[b]);
          if (e < 0.0) e = 0.0;
          e = e / LN2_STD;
          double l1 = 0.0;
          for (int b = 0; b < M; ++b) l1 += fabs(hh[b] - hl[b]);
          const double sc = e * (s * s / 2.0) * l1;
          if (sc > best) {
            best = sc;
            best_s = s;
          }
        }
        const size_t idx = (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z);
        j->score[idx] = (float)best;
        j->best_scale[idx] = (float)best_s;
      }
  }
  free(hists);
  free(normalized);
  free(S);
  return NULL;
}

int sxo_exhaustive(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double* scales, int n_scales, int kernel, uint64_t budget, int mode,
                   int threads, int z_begin, int z_end, int y_begin, int y_end, float* score,
                   float* best_scale, uint64_t* visits, char* err, int err_len) {
  if (n_scales < 1) {
    set_err(err, err_len, "exhaustive scan: no scales");
    return -1;
  }
  for (int i = 0; i < n_scales; ++i)
    if (scales[i] < 2.0) {
      set_err(err, err_len, "exhaustive scan: scales must be >= 2 voxels");
      return -1;
    }
  const uint64_t nvox = (uint64_t)nx * ny * nz;
  const uint64_t evals = nvox * (uint64_t)n_scales;
  if (evals > budget) {
    char buf[160];
    snprintf(buf, sizeof buf, "exhaustive scan: budget exceeded (%llu voxel-scale evaluations)",
             (unsigned long long)evals);
    set_err(err, err_len, buf);
    return -1;
  }
  if (mode == 1 && kernel != 0) {
    set_err(err, err_len, "oracle exact mode supports the identity kernel only");
    return -1;
  }
  const int two_d = nz == 1;
  double* radii = (double*)malloc(sizeof(double) * 3 * (size_t)n_scales);
  int nr = 0;
  for (int i = 0; i < n_scales; ++i) {
    radii[nr++] = scales[i] - 1.0;
    radii[nr++] = scales[i];
    radii[nr++] = scales[i] + 1.0;
  }
  qsort(radii, (size_t)nr, sizeof(double), cmp_double);
  int u = 0;
  for (int i = 0; i < nr; ++i)
    if (u == 0 || radii[u - 1] != radii[i]) radii[u++] = radii[i];
  nr = u;
  sphere_offsets* offs = (sphere_offsets*)calloc((size_t)nr, sizeof(sphere_offsets));
  for (int i = 0; i < nr; ++i) make_sphere_offsets(radii[i], two_d, &offs[i]);
  uint8_t* binvol = NULL;
  if (mode == 1) {
    binvol = (uint8_t*)malloc(nvox);
    for (uint64_t i = 0; i < nvox; ++i) binvol[i] = (uint8_t)sxo_bin_of(low, high, bins, vol[i]);
  }
  if (z_end <= 0 || z_end > nz) z_end = nz;
  if (z_begin < 0) z_begin = 0;
  if (y_end <= 0 || y_end > ny) y_end = ny;
  if (y_begin < 0) y_begin = 0;
  if (threads < 1) threads = 1;
  const int planes = z_end - z_begin;
  const int64_t rows = (int64_t)planes * (y_end - y_begin);
  if (threads > rows) threads = rows > 0 ? (int)rows : 1;
  exh_job* jobs = (exh_job*)calloc((size_t)threads, sizeof(exh_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    exh_job* j = &jobs[t];
    j->vol = vol;
    j->nx = nx;
    j->ny = ny;
    j->nz = nz;
    j->bins = bins;
    j->kernel = kernel;
    j->mode = mode;
    j->low = low;
    j->high = high;
    j->scales = scales;
    j->n_scales = n_scales;
    j->radii = radii;
    j->n_radii = nr;
    j->offs = offs;
    /* rows are numbered (z - z_begin) * nry + (y - y_begin); offset z by z_begin */
    j->ry0 = y_begin;
    j->ry1 = y_end;
    j->r0 = (int64_t)z_begin * (y_end - y_begin) + rows * t / threads;
    j->r1 = (int64_t)z_begin * (y_end - y_begin) + rows * (t + 1) / threads;
    j->score = score;
    j->best_scale = best_scale;
    j->binvol = binvol;
  }
  if (threads == 1) {
    exh_worker(&jobs[0]);
  } else {
    for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, exh_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  }
  if (visits) { /* pipeline.cpp:118,141: every offset of every radius, OOB included */
    uint64_t per = 0;
    for (int i = 0; i < nr; ++i) per += (uint64_t)offs[i].n;
    *visits += per * (uint64_t)nx * (uint64_t)rows;
  }
  for (int i = 0; i < nr; ++i) free_offsets(&offs[i]);
  free(offs);
  free(radii);
  free(binvol);
  free(jobs);
  free(tids);
  return 0;
}

int sxo_voxel_shell_hist(const float* vol, int nx, int ny, int nz, double low, double high,
                         int bins, int x, int y, int z, double radius, uint64_t* S) {
  sphere_offsets off;
  make_sphere_offsets(radius, nz == 1, &off);
  for (int b = 0; b < bins; ++b) S[b] = 0;
  for (int i = 0; i < off.n; ++i) {
    const int sx = x + off.at[3 * i], sy = y + off.at[3 * i + 1], sz = z + off.at[3 * i + 2];
    if (sx < 0 || sx >= nx || sy < 0 || sy >= ny || sz < 0 || sz >= nz) continue;
    const double val = vol[(size_t)sx + (size_t)nx * ((size_t)sy + (size_t)ny * sz)];
    S[sxo_bin_of(low, high, bins, val)] += (uint64_t)off.nsq[i];
  }
  free_offsets(&off);
  return 0;
}

/* ------------------------------------------------------ pipeline.cpp:143-165 */
typedef struct {
  float s;
  int64_t lin;
} max_rec;
static int cmp_max(const void* a, const void* b) { /* score desc, then scan order (stable) */
  const max_rec* x = (const max_rec*)a;
  const max_rec* y = (const max_rec*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return x->lin < y->lin ? -1 : (x->lin > y->lin ? 1 : 0);
}
int64_t sxo_local_maxima(const float* score, const float* best_scale, int nx, int ny, int nz,
                         double* pos, double* sc, double* scale, int64_t* lin, int64_t cap) {
  int64_t n = 0, capn = 1024;
  max_rec* recs = (max_rec*)malloc(sizeof(max_rec) * (size_t)capn);
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const int64_t idx = (int64_t)x + (int64_t)nx * ((int64_t)y + (int64_t)ny * z);
        const float s0 = score[idx];
        if (s0 <= 0.0f) continue;
        int is_max = 1;
        for (int dz = -1; dz <= 1 && is_max; ++dz)
          for (int dy = -1; dy <= 1 && is_max; ++dy)
            for (int dx = -1; dx <= 1 && is_max; ++dx) {
              if (dx == 0 && dy == 0 && dz == 0) continue;
              const int sx = x + dx, sy = y + dy, sz = z + dz;
              if (sx < 0 || sx >= nx || sy < 0 || sy >= ny || sz < 0 || sz >= nz) continue;
              if (score[(int64_t)sx + (int64_t)nx * ((int64_t)sy + (int64_t)ny * sz)] >= s0)
                is_max = 0;
            }
        if (!is_max) continue;
        if (n == capn) {
          capn *= 2;
          recs = (max_rec*)realloc(recs, sizeof(max_rec) * (size_t)capn);
        }
        recs[n].s = s0;
        recs[n].lin = idx;
        ++n;
      }
  qsort(recs, (size_t)n, sizeof(max_rec), cmp_max);
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const int64_t idx = recs[i].lin;
    pos[3 * i + 0] = (double)(idx % nx);
    pos[3 * i + 1] = (double)((idx / nx) % ny);
    pos[3 * i + 2] = (double)(idx / ((int64_t)nx * ny));
    sc[i] = (double)recs[i].s;
    scale[i] = (double)best_scale[idx];
    if (lin) lin[i] = idx;
  }
  free(recs);
  return n;
}

/* ------------------------------------------------------------ seeds.cpp:7-45 */
int64_t sxo_plan_seeds(int nx, int ny, int nz, int mode, double spacing, int count,
                       const double* scales, int n_scales, uint64_t rng_seed, double* pos,
                       double* seed_scale, int64_t cap) {
  if (mode == 0 && spacing <= 0.0) return -1;
  if (mode == 1 && count < 1) return -1;
  if (n_scales < 1) return -1;
  for (int i = 0; i < n_scales; ++i)
    if (scales[i] <= 0.0) return -1;
  const int dims[3] = {nx, ny, nz};
  int64_t np;
  int counts[3] = {1, 1, 1};
  double start[3] = {0, 0, 0};
  if (mode == 0) {
    for (int i = 0; i < 3; ++i) {
      counts[i] = imax(1, (int)floor(dims[i] / spacing));
      start[i] = (dims[i] - (counts[i] - 1) * spacing) / 2.0;
      if (dims[i] == 1) {
        counts[i] = 1;
        start[i] = 0.0;
      }
    }
    np = (int64_t)counts[0] * counts[1] * counts[2];
  } else {
    np = count;
  }
  const int64_t total = np * n_scales;
  if (cap <= 0 || !pos) return total;
  sxo_rng rng;
  sxo_rng_init(&rng, rng_seed);
  int64_t k = 0, pi = 0;
  for (int z = 0; z < (mode == 0 ? counts[2] : 1); ++z)
    for (int y = 0; y < (mode == 0 ? counts[1] : 1); ++y)
      for (int x = 0; x < (mode == 0 ? counts[0] : (int)np); ++x, ++pi) {
        double p[3];
        if (mode == 0) {
          p[0] = dclamp(start[0] + x * spacing, 0.0, (double)(nx - 1));
          p[1] = dclamp(start[1] + y * spacing, 0.0, (double)(ny - 1));
          p[2] = dclamp(start[2] + z * spacing, 0.0, (double)(nz - 1));
        } else {
          p[0] = sxo_rng_next_range(&rng, 0.0, nx - 1);
          p[1] = sxo_rng_next_range(&rng, 0.0, ny - 1);
          p[2] = nz == 1 ? 0.0 : sxo_rng_next_range(&rng, 0.0, nz - 1);
        }
        for (int s = 0; s < n_scales; ++s) {
          if (k < cap) {
            memcpy(pos + 3 * k, p, sizeof p);
            seed_scale[k] = scales[s];
          }
          ++k;
        }
      }
  return total;
}

/* ------------------------------------------------- window.hpp:30-110, window.cpp */
typedef struct {
  double center[3];
  double H[9];
} ewin;

static double win_scale(const ewin* w, int two_d) { /* window.hpp:50-56 */
  if (two_d) {
    const double det2 = w->H[0] * w->H[4] - w->H[1] * w->H[3];
    return opow(det2 > 0.0 ? det2 : 0.0, 0.25);
  }
  const double det = sxo_eigen_det3(w->H);
  return opow(det > 0.0 ? det : 0.0, 1.0 / 6.0);
}
static ewin win_scaled_to(const ewin* w, double s_new, int two_d) { /* window.hpp:59-66 */
  const double s = win_scale(w, two_d);
  ewin o = *w;
  const double f = (s_new / s) * (s_new / s);
  for (int i = 0; i < 9; ++i) o.H[i] *= f;
  if (two_d) o.H[8] = 1.0;
  return o;
}
static double win_support_volume(const ewin* w, int two_d) { /* window.hpp:69-75 */
  if (two_d) {
    const double det2 = w->H[0] * w->H[4] - w->H[1] * w->H[3];
    return PI_STD * sqrt(det2 > 0.0 ? det2 : 0.0);
  }
  const double det = sxo_eigen_det3(w->H);
  return 4.0 / 3.0 * PI_STD * sqrt(det > 0.0 ? det : 0.0);
}

typedef struct {
  const float* vol;
  int nx, ny, nz;
} vview;

typedef void (*support_fn)(void* ctx, int x, int y, int z, double d);

/* window.hpp:81-110 */
static uint64_t for_each_support_voxel(const vview* v, const ewin* w, support_fn fn, void* ctx) {
  double Hi[9];
  sxo_eigen_inverse3(w->H, Hi);
  double ext[3];
  for (int i = 0; i < 3; ++i) {
    const double h = w->H[i * 4];
    ext[i] = sqrt(h > 0.0 ? h : 0.0);
  }
  const int x0 = imax(0, (int)ceil(w->center[0] - ext[0]));
  const int x1 = imin(v->nx - 1, (int)floor(w->center[0] + ext[0]));
  const int y0 = imax(0, (int)ceil(w->center[1] - ext[1]));
  const int y1 = imin(v->ny - 1, (int)floor(w->center[1] + ext[1]));
  const int z0 = imax(0, (int)ceil(w->center[2] - ext[2]));
  const int z1 = imin(v->nz - 1, (int)floor(w->center[2] + ext[2]));
  uint64_t visited = 0;
  for (int z = z0; z <= z1; ++z) {
    const double dz = z - w->center[2];
    for (int y = y0; y <= y1; ++y) {
      const double dy = y - w->center[1];
      const double c0 = Hi[4] * dy * dy + 2.0 * Hi[5] * dy * dz + Hi[8] * dz * dz;
      const double c1 = 2.0 * (Hi[1] * dy + Hi[2] * dz);
      for (int x = x0; x <= x1; ++x) {
        const double dx = x - w->center[0];
        const double d = Hi[0] * dx * dx + c1 * dx + c0;
        ++visited;
        if (d <= 1.0) fn(ctx, x, y, z, d);
      }
    }
  }
  return visited;
}

typedef struct {
  const vview* v;
  double low, high;
  int bins, kernel;
  double det_fac;
  double* h;
  uint64_t support;
} hist_ctx;
static void hist_fn(void* c, int x, int y, int z, double d) {
  hist_ctx* h = (hist_ctx*)c;
  ++h->support;
  const float val = h->v->vol[(size_t)x + (size_t)h->v->nx * ((size_t)y + (size_t)h->v->ny * z)];
  h->h[sxo_bin_of(h->low, h->high, h->bins, val)] += h->det_fac * kernel_value(h->kernel, d);
}
/* window.cpp:5-19; returns 1 with normalized p, 0 for nullopt */
static int try_candidate_histogram(const vview* v, const ewin* w, double low, double high, int bins,
                                   int kernel, double* p, uint64_t* visits) {
  hist_ctx c = {v, low, high, bins, kernel, 0.0, p, 0};
  const double det = sxo_eigen_det3(w->H);
  c.det_fac = 1.0 / sqrt(det > 1e-300 ? det : 1e-300);
  for (int b = 0; b < bins; ++b) p[b] = 0.0;
  const uint64_t visited = for_each_support_voxel(v, w, hist_fn, &c);
  if (visits) *visits += visited;
  if (c.support == 0) return 0;
  return normalize_hist(p, bins);
}

int sxo_candidate_histogram(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, const double center[3], const double H[9], int kernel,
                            double* p_out, uint64_t* visits) {
  const vview v = {vol, nx, ny, nz};
  ewin w;
  memcpy(w.center, center, sizeof w.center);
  memcpy(w.H, H, sizeof w.H);
  return try_candidate_histogram(&v, &w, low, high, bins, kernel, p_out, visits);
}

/* window.cpp:30-46; returns 1 and *out, or 0 when it throws (invalid_argument) */
static int pdf_difference(const vview* v, const ewin* w, double low, double high, int bins,
                          int kernel, double* out, uint64_t* visits) {
  const int two_d = v->nz == 1;
  const double s = win_scale(w, two_d);
  const double ds = 1.0;
  if (s - ds < 1.0) return 0;
  double* lo = (double*)malloc(sizeof(double) * 2 * (size_t)bins);
  double* hi = lo + bins;
  const ewin wl = win_scaled_to(w, s - ds, two_d);
  const ewin wh = win_scaled_to(w, s + ds, two_d);
  const int okl = try_candidate_histogram(v, &wl, low, high, bins, kernel, lo, visits);
  const int okh = try_candidate_histogram(v, &wh, low, high, bins, kernel, hi, visits);
  if (!okl || !okh) {
    free(lo);
    return 0;
  }
  double l1 = 0.0;
  for (int b = 0; b < bins; ++b) l1 += fabs(hi[b] - lo[b]);
  *out = s * s / (2.0 * ds) * l1;
  free(lo);
  return 1;
}
int sxo_pdf_difference(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double center[3], const double H[9], int kernel, double* out,
                       uint64_t* visits) {
  const vview v = {vol, nx, ny, nz};
  ewin w;
  memcpy(w.center, center, sizeof w.center);
  memcpy(w.H, H, sizeof w.H);
  return pdf_difference(&v, &w, low, high, bins, kernel, out, visits);
}

typedef struct {
  uint64_t inside;
} count_ctx;
static void count_fn(void* c, int x, int y, int z, double d) {
  (void)x, (void)y, (void)z, (void)d;
  ((count_ctx*)c)->inside++;
}
static double inbounds_support_fraction(const vview* v, const ewin* w) { /* window.cpp:54-60 */
  count_ctx c = {0};
  for_each_support_voxel(v, w, count_fn, &c);
  const double expected = win_support_volume(w, v->nz == 1);
  if (expected <= 0.0) return 0.0;
  const double f = (double)c.inside / expected;
  return f < 1.0 ? f : 1.0;
}

typedef struct {
  int nx, ny;
  uint64_t* out;
  int64_t cap, n;
} raster_ctx;
static void raster_fn(void* c, int x, int y, int z, double d) {
  (void)d;
  raster_ctx* r = (raster_ctx*)c;
  if (r->n < r->cap) r->out[r->n] = (uint64_t)x + (uint64_t)r->nx * ((uint64_t)y + (uint64_t)r->ny * z);
  r->n++;
}
/* rasterize_window (pipeline.cpp:185-192): support indices in z->y->x order */
int64_t sxo_rasterize_window(int nx, int ny, int nz, const double center[3], const double H[9],
                             uint64_t* out, int64_t cap) {
  const vview v = {NULL, nx, ny, nz};
  ewin w;
  memcpy(w.center, center, sizeof w.center);
  memcpy(w.H, H, sizeof w.H);
  raster_ctx c = {nx, ny, out, cap, 0};
  for_each_support_voxel(&v, &w, raster_fn, &c);
  return c.n;
}

/* ------------------------------------------------------------ shift.cpp:7-107 */
static ewin window_at(const double x[3], const double half_in[3], int two_d) { /* shift.cpp:7-11 */
  double half[3] = {half_in[0], half_in[1], two_d ? 1.0 : half_in[2]};
  ewin w;
  memcpy(w.center, x, sizeof w.center);
  memset(w.H, 0, sizeof w.H);
  w.H[0] = half[0] * half[0];
  w.H[4] = half[1] * half[1];
  w.H[8] = half[2] * half[2];
  return w;
}

typedef struct {
  const vview* v;
  double low, high;
  int bins, step_kernel;
  const double* p;
  const double* q;
  double num[3], den;
} step_ctx;
static void step_fn(void* c, int x, int y, int z, double d) {
  step_ctx* s = (step_ctx*)c;
  const float val = s->v->vol[(size_t)x + (size_t)s->v->nx * ((size_t)y + (size_t)s->v->ny * z)];
  const int b = sxo_bin_of(s->low, s->high, s->bins, val);
  const double pb = s->p[b] > 1e-6 ? s->p[b] : 1e-6; /* histogram.hpp:107-113 */
  const double w = sqrt(s->q[b] / pb);
  const double g = kernel_step_weight(s->step_kernel, d) * w;
  s->num[0] += g * (double)x;
  s->num[1] += g * (double)y;
  s->num[2] += g * (double)z;
  s->den += g;
}

static int shift_step_impl(const vview* v, const double x[3], const double half[3], double low,
                           double high, int bins, int step_kernel, int hist_kernel, const double* q,
                           double out[3], uint64_t* visits) {
  const ewin w = window_at(x, half, v->nz == 1);
  double* p = (double*)malloc(sizeof(double) * (size_t)bins);
  if (!try_candidate_histogram(v, &w, low, high, bins, hist_kernel, p, visits)) {
    free(p);
    return 0;
  }
  step_ctx c = {v, low, high, bins, step_kernel, p, q, {0.0, 0.0, 0.0}, 0.0};
  const uint64_t visited = for_each_support_voxel(v, &w, step_fn, &c);
  if (visits) *visits += visited;
  free(p);
  if (c.den <= 0.0) return 0;
  for (int i = 0; i < 3; ++i) out[i] = c.num[i] / c.den;
  return 1;
}

static double* make_target(const double* target, int bins) {
  double* q = (double*)malloc(sizeof(double) * (size_t)bins);
  for (int b = 0; b < bins; ++b) q[b] = target ? target[b] : 1.0 / bins;
  return q;
}

int sxo_shift_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double x[3], const double half[3], int step_kernel, int hist_kernel,
                   const double* target, double out[3], uint64_t* visits) {
  const vview v = {vol, nx, ny, nz};
  double* q = make_target(target, bins);
  const int ok = shift_step_impl(&v, x, half, low, high, bins, step_kernel, hist_kernel, q, out, visits);
  free(q);
  return ok;
}

static double norm3(const double* a) { return sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]); }

int sxo_saliency_shift(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                       const double seed[3], const double half[3], int step_kernel,
                       int hist_kernel, int max_iters, double min_step, const double* target,
                       double min_inbounds_fraction, sxo_detection* det, uint64_t* visits) {
  const vview v = {vol, nx, ny, nz};
  const int two_d = nz == 1;
  if (!(half[0] > 0.0 && half[1] > 0.0 && half[2] > 0.0) || min_step <= 0.0 || max_iters < 1)
    return -1; /* ShiftParams::validate (shift.hpp:28-33) */
  double* q = make_target(target, bins);
  memset(det, 0, sizeof *det);
  det->seed_index = -1;
  const double lim[3] = {(double)(nx - 1), (double)(ny - 1), (double)(nz - 1)};
  for (int i = 0; i < 3; ++i) det->center[i] = dclamp(seed[i], 0.0, lim[i]);
  ewin w = window_at(det->center, half, two_d);
  memcpy(det->H, w.H, sizeof det->H);
  if (inbounds_support_fraction(&v, &w) < min_inbounds_fraction) {
    det->flags |= 2u;
    free(q);
    return 0;
  }
  for (int it = 0; it < max_iters; ++it) {
    double next[3];
    const int ok = shift_step_impl(&v, det->center, half, low, high, bins, step_kernel,
                                   hist_kernel, q, next, visits);
    det->iterations = it + 1;
    if (!ok) {
      det->flags |= 2u;
      break;
    }
    double clamped[3], diff[3];
    for (int i = 0; i < 3; ++i) clamped[i] = dclamp(next[i], 0.0, lim[i]);
    for (int i = 0; i < 3; ++i) diff[i] = clamped[i] - next[i];
    if (norm3(diff) > 0.0) det->flags |= 4u;
    for (int i = 0; i < 3; ++i) diff[i] = clamped[i] - det->center[i];
    const double step = norm3(diff);
    memcpy(det->center, clamped, sizeof clamped);
    w = window_at(det->center, half, two_d);
    if (inbounds_support_fraction(&v, &w) < min_inbounds_fraction) {
      det->flags |= 2u;
      break;
    }
    if (step < min_step) {
      det->flags |= 1u;
      break;
    }
  }
  w = window_at(det->center, half, two_d);
  memcpy(det->H, w.H, sizeof det->H);
  if (!(det->flags & 2u)) {
    double* ps = (double*)malloc(sizeof(double) * 2 * (size_t)bins);
    double* pt = ps + bins;
    const int oks = try_candidate_histogram(&v, &w, low, high, bins, 1, ps, visits);
    const int okt = try_candidate_histogram(&v, &w, low, high, bins, hist_kernel, pt, visits);
    if (oks && okt) {
      det->entropy_bits = sxo_entropy_bits(ps, bins);
      det->bhattacharyya = bhattacharyya(pt, q, bins);
    } else {
      det->flags |= 2u;
    }
    double pd;
    det->pdf_diff = pdf_difference(&v, &w, low, high, bins, 0, &pd, visits) ? pd : 0.0;
    free(ps);
  }
  free(q);
  return 0;
}

/* ---------------------------------------------------------- quadrant.cpp:14-114 */
/* NE, NW, SW, SE (quadrant.cpp:14); octants: the same four at z=+1, then at z=-1. */
static const int kDirs[8][3] = {{+1, +1, +1}, {-1, +1, +1}, {-1, -1, +1}, {+1, -1, +1},
                                {+1, +1, -1}, {-1, +1, -1}, {-1, -1, -1}, {+1, -1, -1}};

static double box_entropy(const vview* v, double low, double high, int bins, double x0, double x1,
                          double y0, double y1, double z0, double z1, int min_voxels,
                          uint64_t* visits, double* hbuf) { /* quadrant.cpp:18-35 (+ z axis) */
  const int ix0 = imax(0, (int)ceil(x0 < x1 ? x0 : x1));
  const int ix1 = imin(v->nx - 1, (int)floor(x0 < x1 ? x1 : x0));
  const int iy0 = imax(0, (int)ceil(y0 < y1 ? y0 : y1));
  const int iy1 = imin(v->ny - 1, (int)floor(y0 < y1 ? y1 : y0));
  const int iz0 = imax(0, (int)ceil(z0 < z1 ? z0 : z1));
  const int iz1 = imin(v->nz - 1, (int)floor(z0 < z1 ? z1 : z0));
  if (ix0 > ix1 || iy0 > iy1 || iz0 > iz1) return 0.0;
  const int count = (ix1 - ix0 + 1) * (iy1 - iy0 + 1) * (iz1 - iz0 + 1);
  if (count < min_voxels) return 0.0;
  for (int b = 0; b < bins; ++b) hbuf[b] = 0.0;
  for (int z = iz0; z <= iz1; ++z)
    for (int y = iy0; y <= iy1; ++y)
      for (int x = ix0; x <= ix1; ++x)
        hbuf[sxo_bin_of(low, high, bins,
                        v->vol[(size_t)x + (size_t)v->nx * ((size_t)y + (size_t)v->ny * z)])] += 1.0;
  if (visits) *visits += (uint64_t)count;
  normalize_hist(hbuf, bins);
  return sxo_entropy_bits(hbuf, bins);
}

double sxo_box_entropy_bits(const float* vol, int nx, int ny, int nz, double low, double high,
                            int bins, double x0, double x1, double y0, double y1, double z0,
                            double z1, int min_voxels, uint64_t* visits) {
  const vview v = {vol, nx, ny, nz};
  double* h = (double*)malloc(sizeof(double) * (size_t)bins);
  const double e = box_entropy(&v, low, high, bins, x0, x1, y0, y1, z0, z1, min_voxels, visits, h);
  free(h);
  return e;
}

static void ascent_step(const vview* v, double low, double high, int bins, int dims,
                        const double p[3], const int* scales, int n_scales, double moved[3],
                        sxo_ascent_state* st, uint64_t* visits, double* hbuf) {
  const int nq = dims == 2 ? 4 : 8;
  const int min_voxels = dims == 2 ? 4 : 8;
  memset(st, 0, sizeof *st);
  for (int q = 0; q < nq; ++q) {
    double best_e = 0.0;
    int best_k = scales[0];
    for (int i = 0; i < n_scales; ++i) {
      const int k = scales[i];
      const double dx = kDirs[q][0] * (double)k, dy = kDirs[q][1] * (double)k;
      const double dz = dims == 2 ? 0.0 : kDirs[q][2] * (double)k;
      const double e = box_entropy(v, low, high, bins, p[0], p[0] + dx, p[1], p[1] + dy, p[2],
                                   p[2] + dz, min_voxels, visits, hbuf);
      if (e > best_e) {
        best_e = e;
        best_k = k;
      }
    }
    st->entropy[q] = best_e;
    st->best_scale[q] = best_k;
  }
  double total = 0.0;
  for (int q = 0; q < nq; ++q) total += st->entropy[q];
  if (total <= 0.0) {
    st->degenerate = 1;
    memcpy(moved, p, 3 * sizeof(double));
    return;
  }
  double ed[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < nq; ++q) {
    st->norm_entropy[q] = st->entropy[q] / total;
    ed[0] += st->norm_entropy[q] * kDirs[q][0] * st->best_scale[q];
    ed[1] += st->norm_entropy[q] * kDirs[q][1] * st->best_scale[q];
    if (dims == 3) ed[2] += st->norm_entropy[q] * kDirs[q][2] * st->best_scale[q];
  }
  memcpy(st->displacement, ed, sizeof ed);
  const double lim[3] = {(double)(v->nx - 1), (double)(v->ny - 1), (double)(v->nz - 1)};
  for (int i = 0; i < 3; ++i) moved[i] = p[i] + ed[i];
  for (int i = 0; i < (dims == 2 ? 2 : 3); ++i) moved[i] = dclamp(moved[i], 0.0, lim[i]);
}

int sxo_ascent_step(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                    int dims, const double p[3], const int* scales, int n_scales,
                    double moved[3], sxo_ascent_state* st, uint64_t* visits) {
  if (dims == 2 && nz != 1) return -1; /* quadrant.cpp:42 */
  const vview v = {vol, nx, ny, nz};
  double* h = (double*)malloc(sizeof(double) * (size_t)bins);
  ascent_step(&v, low, high, bins, dims, p, scales, n_scales, moved, st, visits, h);
  free(h);
  return 0;
}

static int ascent_seek_one(const vview* v, double low, double high, int bins, int dims,
                           const double seed[3], const int* scales, int n_scales, double eta,
                           int max_iters, sxo_ascent_result* r, uint64_t* visits, double* hbuf) {
  memset(r, 0, sizeof *r);
  memcpy(r->position, seed, 3 * sizeof(double));
  sxo_ascent_state last;
  memset(&last, 0, sizeof last);
  const int nq = dims == 2 ? 4 : 8;
  for (int it = 0; it < max_iters; ++it) {
    double moved[3];
    sxo_ascent_state st;
    ascent_step(v, low, high, bins, dims, r->position, scales, n_scales, moved, &st, visits, hbuf);
    r->iterations = it + 1;
    last = st;
    if (st.degenerate) {
      r->degenerate = 1;
      break;
    }
    memcpy(r->position, moved, sizeof moved);
    const double* e = st.displacement;
    const double nrm = dims == 2 ? sqrt(e[0] * e[0] + e[1] * e[1]) : norm3(e);
    if (nrm < eta) {
      r->converged = 1;
      break;
    }
  }
  if (!r->degenerate) {
    int bq = 0;
    for (int q = 1; q < nq; ++q)
      if (last.entropy[q] > last.entropy[bq]) bq = q;
    r->best_scale = last.best_scale[bq];
    r->entropy_bits = last.entropy[bq];
  }
  return 0;
}

int sxo_ascent_seek_one(const float* vol, int nx, int ny, int nz, double low, double high,
                        int bins, int dims, const double seed[3], const int* scales, int n_scales,
                        double eta, int max_iters, sxo_ascent_result* out, uint64_t* visits) {
  if (dims == 2 && nz != 1) return -1;
  if (n_scales < 1 || eta <= 0.0 || max_iters < 1) return -1; /* quadrant.hpp:20-27 */
  for (int i = 1; i < n_scales; ++i)
    if (scales[i] <= scales[i - 1]) return -1;
  const vview v = {vol, nx, ny, nz};
  double* h = (double*)malloc(sizeof(double) * (size_t)bins);
  ascent_seek_one(&v, low, high, bins, dims, seed, scales, n_scales, eta, max_iters, out, visits, h);
  free(h);
  return 0;
}

/* --------------------------------------------------- pipeline.cpp:54-59,168-183 */
static int cmp_dbl_asc(const void* a, const void* b) { return cmp_double(a, b); }
static double quantile_threshold(double* values, int64_t n, double q) {
  if (n == 0) return 0.0;
  qsort(values, (size_t)n, sizeof(double), cmp_dbl_asc);
  const double idx = q * (double)(n - 1);
  return values[(size_t)floor(idx)];
}

int64_t sxo_dedupe_top_k(const sxo_detection* dets, int64_t n, int k, double radius,
                         sxo_detection* out) {
  /* stable sort by pdf_diff desc: insertion-order tie-break via an index sort */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t i = 1; i < n; ++i) { /* stable insertion sort (n is small) */
    const int64_t t = order[i];
    int64_t j = i - 1;
    while (j >= 0 && dets[order[j]].pdf_diff < dets[t].pdf_diff) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = t;
  }
  int64_t kept = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (kept >= k) break;
    const sxo_detection* d = &dets[order[i]];
    int clear = 1;
    for (int64_t a = 0; a < kept; ++a) {
      const double diff[3] = {out[a].center[0] - d->center[0], out[a].center[1] - d->center[1],
                              out[a].center[2] - d->center[2]};
      if (norm3(diff) <= radius) {
        clear = 0;
        break;
      }
    }
    if (clear) out[kept++] = *d;
  }
  free(order);
  return kept;
}

int64_t sxo_select(const sxo_detection* dets, int64_t n, double q_entropy, double q_pdf, int k,
                   double radius, sxo_detection* out) {
  sxo_detection* alive = (sxo_detection*)malloc(sizeof(sxo_detection) * (size_t)(n > 0 ? n : 1));
  int64_t na = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!(dets[i].flags & 2u) && dets[i].entropy_bits > 0.0) alive[na++] = dets[i];
  if (na == 0) {
    free(alive);
    return 0;
  }
  double* ev = (double*)malloc(sizeof(double) * (size_t)na);
  double* pv = (double*)malloc(sizeof(double) * (size_t)na);
  for (int64_t i = 0; i < na; ++i) {
    ev[i] = alive[i].entropy_bits;
    pv[i] = alive[i].pdf_diff;
  }
  const double et = quantile_threshold(ev, na, q_entropy);
  const double pt = quantile_threshold(pv, na, q_pdf);
  int64_t np = 0;
  for (int64_t i = 0; i < na; ++i)
    if (alive[i].entropy_bits >= et && alive[i].pdf_diff >= pt) alive[np++] = alive[i];
  const int64_t r = sxo_dedupe_top_k(alive, np, k, radius, out);
  free(alive);
  free(ev);
  free(pv);
  return r;
}

/* ------------------------------------------------------------ abmsod.cpp:23-169 */
int sxo_bandwidth_from_moment(const double outer[9], double wsum, int dim, double lambda_min,
                              double lambda_max, double H[9]) {
  return sx_bandwidth_from_moment(outer, wsum, dim, lambda_min, lambda_max, H);
}
int sxo_sym_eigen3(const double a[9], double values[3], double vectors[9]) {
  return sx_sym_eigen3(a, values, vectors);
}

typedef struct {
  const vview* v;
  double low, high;
  int bins;
  const double* p;
  const double* q;
  double xn[3];
  double outer[9], wsum;
} bw_ctx;
static void bw_fn(void* c, int x, int y, int z, double d) { /* abmsod.cpp:50-55 */
  (void)d;
  bw_ctx* b = (bw_ctx*)c;
  const float val = b->v->vol[(size_t)x + (size_t)b->v->nx * ((size_t)y + (size_t)b->v->ny * z)];
  const int bin = sxo_bin_of(b->low, b->high, b->bins, val);
  const double pb = b->p[bin] > 1e-6 ? b->p[bin] : 1e-6; /* weight_for_bin */
  const double w = sqrt(b->q[bin] / pb);
  const double dv[3] = {b->xn[0] - (double)x, b->xn[1] - (double)y, b->xn[2] - (double)z};
  for (int i = 0; i < 3; ++i) /* outer += w * d * d^T: (w d_i) d_j per element */
    for (int j = 0; j < 3; ++j) b->outer[3 * i + j] += (w * dv[i]) * dv[j];
  b->wsum += w;
}

typedef struct {
  const vview* v;
  double low, high;
  int bins, kernel;
  const double* p;
  const double* q;
  double num[3], den;
} cen_ctx;
static void cen_fn(void* c, int x, int y, int z, double d) { /* abmsod.cpp:85-90 */
  cen_ctx* s = (cen_ctx*)c;
  const float val = s->v->vol[(size_t)x + (size_t)s->v->nx * ((size_t)y + (size_t)s->v->ny * z)];
  const int b = sxo_bin_of(s->low, s->high, s->bins, val);
  const double pb = s->p[b] > 1e-6 ? s->p[b] : 1e-6;
  const double w = sqrt(s->q[b] / pb);
  const double g = kernel_step_weight(s->kernel, d) * w;
  s->num[0] += g * (double)x;
  s->num[1] += g * (double)y;
  s->num[2] += g * (double)z;
  s->den += g;
}

int sxo_abmsod_run(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const double seed_center[3], const double seed_H[9],
                   const sxo_abmsod_params* P, sxo_detection* det, sxo_abmsod_iter* trace,
                   int trace_cap, int* n_trace, uint64_t* visits) {
  if (P->threshold <= 0.0 || P->max_iterations < 1 || P->lambda_min <= 0.0) return -1;
  const vview v = {vol, nx, ny, nz};
  const int two_d = nz == 1;
  const int dim = two_d ? 2 : 3;
  double lmax = P->lambda_max; /* lambda_max_for (abmsod.hpp:34-38) */
  if (!(lmax > 0.0)) {
    const int m = imax(nx, imax(ny, nz));
    const double half = m / 2.0;
    lmax = half * half;
  }
  double* q = make_target(P->target, bins);
  double* hp = (double*)malloc(sizeof(double) * 2 * (size_t)bins);
  double* hn = hp + bins;
  memset(det, 0, sizeof *det);
  det->seed_index = -1;
  const double lim[3] = {(double)(nx - 1), (double)(ny - 1), (double)(nz - 1)};
  double x[3], H[9], x_opt[3], H_opt[9];
  for (int i = 0; i < 3; ++i) x[i] = dclamp(seed_center[i], 0.0, lim[i]);
  memcpy(det->center, x, sizeof x);
  memcpy(H, seed_H, sizeof H);
  memcpy(det->H, H, sizeof H);
  memcpy(x_opt, x, sizeof x);
  memcpy(H_opt, H, sizeof H);
  double max_bhat = 0.0;
  int stalled = 0, any = 0, nt = 0, rc = 0;
  for (int it = 0; it < P->max_iterations; ++it) {
    ewin win;
    memcpy(win.center, x, sizeof x);
    memcpy(win.H, H, sizeof H);
    if (inbounds_support_fraction(&v, &win) < P->min_inbounds_fraction) {
      det->flags |= 2u;
      break;
    }
    if (!try_candidate_histogram(&v, &win, low, high, bins, P->kernel, hp, visits)) {
      det->flags |= 2u;
      break;
    }
    cen_ctx cc = {&v, low, high, bins, P->kernel, hp, q, {0.0, 0.0, 0.0}, 0.0};
    const uint64_t vis = for_each_support_voxel(&v, &win, cen_fn, &cc);
    if (visits) *visits += vis;
    if (cc.den <= 0.0) {
      det->flags |= 2u;
      break;
    }
    double xn[3], cl[3], df[3];
    for (int i = 0; i < 3; ++i) xn[i] = cc.num[i] / cc.den;
    for (int i = 0; i < 3; ++i) cl[i] = dclamp(xn[i], 0.0, lim[i]);
    for (int i = 0; i < 3; ++i) df[i] = cl[i] - xn[i];
    if (norm3(df) > 0.0) det->flags |= 4u;
    memcpy(xn, cl, sizeof cl);
    ewin moved;
    memcpy(moved.center, xn, sizeof xn);
    memcpy(moved.H, H, sizeof H);
    if (!try_candidate_histogram(&v, &moved, low, high, bins, P->kernel, hn, visits)) {
      det->flags |= 2u;
      break;
    }
    bw_ctx bc;
    memset(&bc, 0, sizeof bc);
    bc.v = &v, bc.low = low, bc.high = high, bc.bins = bins, bc.p = hn, bc.q = q;
    memcpy(bc.xn, xn, sizeof xn);
    const uint64_t vb = for_each_support_voxel(&v, &moved, bw_fn, &bc);
    if (visits) *visits += vb;
    double Hn[9];
    const int br = sx_bandwidth_from_moment(bc.outer, bc.wsum, dim, P->lambda_min, lmax, Hn);
    if (br == 3) {
      rc = -2; /* std::runtime_error escapes abmsod_run */
      break;
    }
    if (br != 0) {
      det->flags |= 2u;
      break;
    }
    const double bhat = bhattacharyya(hn, q, bins);
    any = 1;
    det->iterations = it + 1;
    const int improved = bhat > max_bhat + P->threshold;
    if (bhat > max_bhat) {
      max_bhat = bhat;
      memcpy(x_opt, xn, sizeof xn);
      memcpy(H_opt, Hn, sizeof Hn);
    }
    if (trace && nt < trace_cap) {
      sxo_abmsod_iter* r = &trace[nt];
      double ev[3], V[9];
      if (sx_sym_eigen3(Hn, ev, V) != 0) {
        rc = -2;
        break;
      }
      memcpy(r->position, xn, sizeof xn);
      memcpy(r->H, Hn, sizeof Hn);
      r->bhattacharyya = bhat;
      r->max_bhattacharyya = max_bhat;
      r->eig_min = ev[0] < ev[1] ? (ev[0] < ev[2] ? ev[0] : ev[2]) : (ev[1] < ev[2] ? ev[1] : ev[2]);
      r->eig_max = ev[0] > ev[1] ? (ev[0] > ev[2] ? ev[0] : ev[2]) : (ev[1] > ev[2] ? ev[1] : ev[2]);
      ++nt;
    }
    memcpy(x, xn, sizeof xn);
    memcpy(H, Hn, sizeof Hn);
    stalled = improved ? 0 : stalled + 1;
    if (stalled >= 2) {
      det->flags |= 1u;
      break;
    }
  }
  if (rc == 0) {
    if (any) {
      memcpy(det->center, x_opt, sizeof x_opt);
      memcpy(det->H, H_opt, sizeof H_opt);
      det->bhattacharyya = max_bhat;
      ewin ow;
      memcpy(ow.center, x_opt, sizeof x_opt);
      memcpy(ow.H, H_opt, sizeof H_opt);
      if (try_candidate_histogram(&v, &ow, low, high, bins, 1, hp, visits))
        det->entropy_bits = sxo_entropy_bits(hp, bins);
      double pd;
      det->pdf_diff = pdf_difference(&v, &ow, low, high, bins, 0, &pd, visits) ? pd : 0.0;
    } else {
      det->flags |= 2u;
    }
  }
  if (n_trace) *n_trace = nt;
  free(hp);
  free(q);
  return rc;
}

/* ---------------------------------------------------------- pipeline.cpp:311-402 */
typedef struct {
  const vview* v;
  double low, high;
  int bins;
  const sxo_detect_params* P;
  const double* pos;
  const double* sscale;
  const int64_t* index;
  const int* qscales;
  int n_qscales;
  sxo_detection* out;
  int64_t n;
  int64_t next;
  pthread_mutex_t mu;
  uint64_t visits;
} det_job;

static void run_seed(det_job* J, int64_t i, uint64_t* visits, double* hbuf) {
  const sxo_detect_params* P = J->P;
  const vview* v = J->v;
  const int two_d = v->nz == 1;
  sxo_detection* d = &J->out[i];
  if (P->method == 2) { /* pipeline.cpp:371-379: isotropic seed window, abmsod_run */
    const double s = J->sscale[i];
    double H[9] = {s * s, 0.0, 0.0, 0.0, s * s, 0.0, 0.0, 0.0, two_d ? 1.0 : s * s};
    sxo_abmsod_params ap = {P->abmsod_threshold, P->abmsod_max_iters, P->abmsod_kernel,
                            P->abmsod_lambda_min, P->abmsod_lambda_max,
                            P->abmsod_min_inbounds_fraction, NULL};
    if (sxo_abmsod_run(v->vol, v->nx, v->ny, v->nz, J->low, J->high, J->bins, J->pos + 3 * i, H,
                       &ap, d, NULL, 0, NULL, visits) != 0)
      d->reserved = 1;
    d->seed_index = (int32_t)J->index[i];
    return;
  }
  if (P->method == 1) { /* pipeline.cpp:360-370 */
    const double s = J->sscale[i];
    const double half[3] = {s, s, two_d ? 1.0 : s};
    sxo_saliency_shift(v->vol, v->nx, v->ny, v->nz, J->low, J->high, J->bins, J->pos + 3 * i, half,
                       P->shift_step_kernel, P->shift_hist_kernel, P->shift_max_iters,
                       P->shift_min_step, NULL, P->shift_min_inbounds_fraction, d, visits);
    d->seed_index = (int32_t)J->index[i];
    return;
  }
  /* quadrant (pipeline.cpp:320-359) and octant (new, same post-scoring in 3D) */
  const int dims = P->method == 0 ? 2 : 3;
  sxo_ascent_result r;
  ascent_seek_one(v, J->low, J->high, J->bins, dims, J->pos + 3 * i, J->qscales, J->n_qscales,
                  P->quadrant_eta, P->quadrant_max_iters, &r, visits, hbuf);
  memset(d, 0, sizeof *d);
  d->center[0] = r.position[0];
  d->center[1] = r.position[1];
  d->center[2] = dims == 2 ? 0.0 : r.position[2];
  d->H[0] = d->H[4] = d->H[8] = 1.0;
  d->seed_index = (int32_t)J->index[i];
  d->iterations = r.iterations;
  if (r.converged) d->flags |= 1u;
  if (r.degenerate) {
    d->flags |= 2u;
    return;
  }
  const double k = 2.0 > (double)r.best_scale ? 2.0 : (double)r.best_scale;
  ewin w;
  memcpy(w.center, d->center, sizeof w.center);
  memset(w.H, 0, sizeof w.H);
  w.H[0] = k * k;
  w.H[4] = k * k;
  w.H[8] = two_d ? 1.0 : k * k;
  memcpy(d->H, w.H, sizeof w.H);
  double* p = (double*)malloc(sizeof(double) * (size_t)J->bins);
  if (try_candidate_histogram(v, &w, J->low, J->high, J->bins, 1, p, visits)) {
    double* q = make_target(NULL, J->bins);
    d->entropy_bits = sxo_entropy_bits(p, J->bins);
    d->bhattacharyya = bhattacharyya(p, q, J->bins);
    free(q);
  }
  free(p);
  double pd;
  d->pdf_diff = pdf_difference(v, &w, J->low, J->high, J->bins, 0, &pd, visits) ? pd : 0.0;
}

static void* det_worker(void* arg) {
  det_job* J = (det_job*)arg;
  double* hbuf = (double*)malloc(sizeof(double) * (size_t)J->bins);
  uint64_t visits = 0;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int64_t i = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (i >= J->n) break;
    run_seed(J, i, &visits, hbuf);
  }
  pthread_mutex_lock(&J->mu);
  J->visits += visits;
  pthread_mutex_unlock(&J->mu);
  free(hbuf);
  return NULL;
}

int64_t sxo_detect(const float* vol, int nx, int ny, int nz, double low, double high, int bins,
                   const sxo_detect_params* P, sxo_detection* per_seed, int64_t cap_seed,
                   int64_t* n_seed_out, sxo_detection* out, int64_t cap, uint64_t* visits,
                   char* err, int err_len) {
  if (P->method == 0 && nz != 1) {
    set_err(err, err_len, "detect: quadrant method requires a 2D volume (nz == 1)");
    return -1;
  }
  if (P->method < 0 || P->method > 3) {
    set_err(err, err_len, "oracle: unknown method");
    return -1;
  }
  if (P->method == 2 && (P->abmsod_threshold <= 0.0 || P->abmsod_max_iters < 1 ||
                         P->abmsod_lambda_min <= 0.0)) {
    set_err(err, err_len, "abmsod: invalid params");
    return -1;
  }
  const int64_t ns = sxo_plan_seeds(nx, ny, nz, P->seed_mode, P->seed_spacing, P->seed_count,
                                    P->scales, P->n_scales, P->rng_seed, NULL, NULL, 0);
  if (ns < 0) {
    set_err(err, err_len, "seed plan: invalid");
    return -1;
  }
  double* pos = (double*)malloc(sizeof(double) * 3 * (size_t)ns);
  double* sscale = (double*)malloc(sizeof(double) * (size_t)ns);
  int64_t* index = (int64_t*)malloc(sizeof(int64_t) * (size_t)ns);
  sxo_plan_seeds(nx, ny, nz, P->seed_mode, P->seed_spacing, P->seed_count, P->scales, P->n_scales,
                 P->rng_seed, pos, sscale, ns);
  int64_t n = 0;
  int* qs = NULL;
  int nqs = 0;
  if (P->method == 1 || P->method == 2) {
    for (int64_t i = 0; i < ns; ++i) index[i] = i;
    n = ns;
  } else { /* one trajectory per distinct consecutive position (pipeline.cpp:325-331) */
    for (int64_t i = 0; i < ns; ++i) {
      if (n > 0 && pos[3 * (n - 1)] == pos[3 * i] && pos[3 * (n - 1) + 1] == pos[3 * i + 1] &&
          (P->method == 0 || pos[3 * (n - 1) + 2] == pos[3 * i + 2]))
        continue;
      memmove(pos + 3 * n, pos + 3 * i, 3 * sizeof(double));
      index[n] = i;
      ++n;
    }
    if (P->quadrant_scales) {
      nqs = P->n_quadrant_scales;
      qs = (int*)malloc(sizeof(int) * (size_t)nqs);
      memcpy(qs, P->quadrant_scales, sizeof(int) * (size_t)nqs);
    } else {
      nqs = P->n_scales;
      qs = (int*)malloc(sizeof(int) * (size_t)nqs);
      for (int i = 0; i < nqs; ++i) qs[i] = (int)lround(P->scales[i]);
    }
    if (nqs < 1 || P->quadrant_eta <= 0.0 || P->quadrant_max_iters < 1) n = -1;
    for (int i = 1; i < nqs && n >= 0; ++i)
      if (qs[i] <= qs[i - 1]) n = -1;
    if (n < 0) {
      set_err(err, err_len, "quadrant: invalid params");
      free(pos), free(sscale), free(index), free(qs);
      return -1;
    }
  }
  sxo_detection* dets = (sxo_detection*)calloc((size_t)(n > 0 ? n : 1), sizeof(sxo_detection));
  const vview v = {vol, nx, ny, nz};
  det_job J;
  memset(&J, 0, sizeof J);
  J.v = &v;
  J.low = low;
  J.high = high;
  J.bins = bins;
  J.P = P;
  J.pos = pos;
  J.sscale = sscale;
  J.index = index;
  J.qscales = qs;
  J.n_qscales = nqs;
  J.out = dets;
  J.n = n;
  pthread_mutex_init(&J.mu, NULL);
  int workers = P->workers < 1 ? 1 : P->workers;
  if (workers > n) workers = (int)(n > 0 ? n : 1);
  if (workers == 1) {
    det_worker(&J);
  } else {
    pthread_t* t = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
    for (int w = 0; w < workers; ++w) pthread_create(&t[w], NULL, det_worker, &J);
    for (int w = 0; w < workers; ++w) pthread_join(t[w], NULL);
    free(t);
  }
  pthread_mutex_destroy(&J.mu);
  for (int64_t i = 0; i < n; ++i)
    if (dets[i].reserved) { /* abmsod.cpp:16-17 runtime_error escapes detect */
      set_err(err, err_len, "abmsod: eigen decomposition failed");
      free(dets), free(pos), free(sscale), free(index), free(qs);
      return -1;
    }
  if (visits) *visits += J.visits;
  if (n_seed_out) *n_seed_out = n;
  if (per_seed)
    for (int64_t i = 0; i < n && i < cap_seed; ++i) per_seed[i] = dets[i];
  sxo_detection* sel = (sxo_detection*)malloc(sizeof(sxo_detection) * (size_t)(n > 0 ? n : 1));
  const int64_t ks = sxo_select(dets, n, P->entropy_quantile, P->pdf_quantile, P->top_k,
                                P->dedupe_radius, sel);
  for (int64_t i = 0; i < ks && i < cap; ++i) out[i] = sel[i];
  free(sel);
  free(dets);
  free(pos);
  free(sscale);
  free(index);
  free(qs);
  return ks;
}

/* ------------------------------------------------------------------ hu.cpp:8-64 */
int sxo_hu_moments(const float* img, int nx, int ny, int pitch, double out[7]) {
  double m00 = 0, m10 = 0, m01 = 0;
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      const double f = img[(size_t)y * pitch + x];
      m00 += f;
      m10 += f * x;
      m01 += f * y;
    }
  if (m00 <= 0.0) return -1; /* invalid_argument: zero total mass */
  const double cx = m10 / m00, cy = m01 / m00;
  double mu20 = 0, mu02 = 0, mu11 = 0, mu30 = 0, mu03 = 0, mu21 = 0, mu12 = 0;
  for (int y = 0; y < ny; ++y) {
    const double dy = y - cy;
    for (int x = 0; x < nx; ++x) {
      const double f = img[(size_t)y * pitch + x];
      const double dx = x - cx;
      mu20 += f * dx * dx;
      mu02 += f * dy * dy;
      mu11 += f * dx * dy;
      mu30 += f * dx * dx * dx;
      mu03 += f * dy * dy * dy;
      mu21 += f * dx * dx * dy;
      mu12 += f * dx * dy * dy;
    }
  }
  const double s2 = m00 * m00 /* pow(x, 2) is exactly rounded */, s3 = opow(m00, 2.5);
  const double n20 = mu20 / s2, n02 = mu02 / s2, n11 = mu11 / s2;
  const double n30 = mu30 / s3, n03 = mu03 / s3, n21 = mu21 / s3, n12 = mu12 / s3;
  out[0] = n20 + n02;
  out[1] = (n20 - n02) * (n20 - n02) + 4.0 * n11 * n11;
  out[2] = (n30 - 3 * n12) * (n30 - 3 * n12) + (3 * n21 - n03) * (3 * n21 - n03);
  out[3] = (n30 + n12) * (n30 + n12) + (n21 + n03) * (n21 + n03);
  out[4] = (n30 - 3 * n12) * (n30 + n12) * ((n30 + n12) * (n30 + n12) - 3 * (n21 + n03) * (n21 + n03)) +
           (3 * n21 - n03) * (n21 + n03) * (3 * (n30 + n12) * (n30 + n12) - (n21 + n03) * (n21 + n03));
  out[5] = (n20 - n02) * ((n30 + n12) * (n30 + n12) - (n21 + n03) * (n21 + n03)) +
           4.0 * n11 * (n30 + n12) * (n21 + n03);
  out[6] = (3 * n21 - n03) * (n30 + n12) * ((n30 + n12) * (n30 + n12) - 3 * (n21 + n03) * (n21 + n03)) -
           (n30 - 3 * n12) * (n21 + n03) * (3 * (n30 + n12) * (n30 + n12) - (n21 + n03) * (n21 + n03));
  return 0;
}

/* pipeline.cpp:218-256 hu_template_distance (crop_slice :220-233) */
double sxo_hu_template_distance(const float* vol, int nx, int ny, int nz, const double center[3],
                                const double H[9], const float* tmpl, int tnx, int tny, int slices) {
  double target[7], h[7];
  if (sxo_hu_moments(tmpl, tnx, tny, tnx, target) != 0) return -1.0;
  const int zc = (int)lround(center[2]);
  const int half = slices / 2;
  const double ex = sqrt(H[0] > 1.0 ? H[0] : 1.0), ey = sqrt(H[4] > 1.0 ? H[4] : 1.0);
  const int x0 = imax(0, (int)floor(center[0] - ex)), x1 = imin(nx - 1, (int)ceil(center[0] + ex));
  const int y0 = imax(0, (int)floor(center[1] - ey)), y1 = imin(ny - 1, (int)ceil(center[1] + ey));
  double sum = 0.0;
  int used = 0;
  for (int dz = -half; dz <= half; ++dz) {
    const int z = zc + dz;
    if (z < 0 || z >= nz) continue;
    const float* crop = vol + ((size_t)z * ny + y0) * nx + x0;
    if (sxo_hu_moments(crop, x1 - x0 + 1, y1 - y0 + 1, nx, h) != 0) continue;
    double d2 = 0.0;
    for (int i = 0; i < 7; ++i) d2 += (h[i] - target[i]) * (h[i] - target[i]);
    sum += sqrt(d2);
    ++used;
  }
  if (used == 0) return 1.0 / 0.0;
  return sum / used;
}
