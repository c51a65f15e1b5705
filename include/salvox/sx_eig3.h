/* sx_eig3.h -- 3x3 linear algebra of the ABMSOD bandwidth update, shared by
 * the device kernel, the C++ host layer and the C oracle.
 *
 * The reference calls Eigen (abmsod.cpp:14-41): Matrix3d::inverse() /
 * determinant() for every window (window.hpp:83, window.cpp:9) and
 * SelfAdjointEigenSolver<Matrix3d> for the bandwidth matrix. Eigen is not in
 * this image and its version is unpinned, so these functions
 * restate Eigen 3.4.0's algorithms operation by operation:
 *   - inverse: InverseImpl.h compute_inverse<Matrix3>: cofactors * (1/det),
 *     det = cofactor column 0 . column 0;
 *   - determinant: Determinant.h bruteforce_det3_helper;
 *   - SelfAdjointEigenSolver::compute (SelfAdjointEigenSolver.h): scale by the
 *     largest |a_ij| of the lower triangle, Tridiagonalization.h's 3x3
 *     tridiagonalization_inplace_selector (one Householder step, explicit Q),
 *     computeFromTridiagonal_impl (deflation test (eps^-1 e)^2 <= |d_i|+|d_i+1|,
 *     at most 30 n implicit symmetric QR steps with a Wilkinson shift computed
 *     through numext::hypot, Givens rotations from JacobiRotation::makeGivens
 *     applied to Q on the right), then the selection sort by minCoeff;
 *   - V diag(l) V^T as Eigen's unvectorised coeff-based lazy product:
 *     r_ij = a_i0 v_j0 + (a_i1 v_j1 + a_i2 v_j2) (redux_novec_unroller).
 * Only IEEE +,-,*,/ and sqrt (correctly rounded on both sides; device uses the
 * _rn intrinsics) so host and device results agree bit for bit. Matrices are
 * row-major m[3 r + c]; eigenvectors are the COLUMNS of V, like Eigen.
 */
#ifndef SALVOX_SX_EIG3_H
#define SALVOX_SX_EIG3_H

#include "sx_log.h"

#if defined(__CUDA_ARCH__)
#define SX_DSQRT(a) __dsqrt_rn(a)
#else
#define SX_DSQRT(a) sqrt(a)
#endif

#define SX_M(m, r, c) (m)[3 * (r) + (c)]

SX_HD double sx_fabs(double x) { return x < 0.0 ? -x : x; }

/* Eigen cofactor(i, j) with i1 = (i+1)%3, i2 = (i+2)%3 (InverseImpl.h cofactor_3x3) */
SX_HD double sx_cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return SX_DSUB(SX_DMUL(SX_M(m, i1, j1), SX_M(m, i2, j2)), SX_DMUL(SX_M(m, i1, j2), SX_M(m, i2, j1)));
}

SX_HD void sx_inverse3(const double* m, double* out) {
  const double c0 = sx_cof3(m, 0, 0), c1 = sx_cof3(m, 1, 0), c2 = sx_cof3(m, 2, 0);
  const double det = SX_DADD(SX_DADD(SX_DMUL(c0, m[0]), SX_DMUL(c1, m[3])), SX_DMUL(c2, m[6]));
  const double invdet = SX_DDIV(1.0, det);
  double r[9];
  r[5] = SX_DMUL(sx_cof3(m, 2, 1), invdet);
  r[7] = SX_DMUL(sx_cof3(m, 1, 2), invdet);
  r[8] = SX_DMUL(sx_cof3(m, 2, 2), invdet);
  r[3] = SX_DMUL(sx_cof3(m, 0, 1), invdet);
  r[4] = SX_DMUL(sx_cof3(m, 1, 1), invdet);
  r[6] = SX_DMUL(sx_cof3(m, 0, 2), invdet);
  r[0] = SX_DMUL(c0, invdet);
  r[1] = SX_DMUL(c1, invdet);
  r[2] = SX_DMUL(c2, invdet);
  for (int i = 0; i < 9; ++i) out[i] = r[i];
}

SX_HD double sx_det3(const double* m) { /* bruteforce_det3_helper(0,1,2)-(1,0,2)+(2,0,1) */
  const double a = SX_DMUL(m[0], SX_DSUB(SX_DMUL(m[4], m[8]), SX_DMUL(m[5], m[7])));
  const double b = SX_DMUL(m[1], SX_DSUB(SX_DMUL(m[3], m[8]), SX_DMUL(m[5], m[6])));
  const double c = SX_DMUL(m[2], SX_DSUB(SX_DMUL(m[3], m[7]), SX_DMUL(m[4], m[6])));
  return SX_DADD(SX_DSUB(a, b), c);
}

/* numext::hypot -> positive_real_hypot(|x|, |y|) (MathFunctionsImpl.h) */
SX_HD double sx_hypot(double x, double y) {
  x = sx_fabs(x);
  y = sx_fabs(y);
  const double p = x < y ? y : x;
  if (p == 0.0) return 0.0;
  const double qp = SX_DDIV(x < y ? x : y, p);
  return SX_DMUL(p, SX_DSQRT(SX_DADD(1.0, SX_DMUL(qp, qp))));
}

/* JacobiRotation<double>::makeGivens(p, q) (Jacobi.h, real case) */
SX_HD void sx_givens(double p, double q, double* c, double* s) {
  if (q == 0.0) {
    *c = p < 0.0 ? -1.0 : 1.0;
    *s = 0.0;
  } else if (p == 0.0) {
    *c = 0.0;
    *s = q < 0.0 ? 1.0 : -1.0;
  } else if (sx_fabs(p) > sx_fabs(q)) {
    const double t = SX_DDIV(q, p);
    double u = SX_DSQRT(SX_DADD(1.0, SX_DMUL(t, t)));
    if (p < 0.0) u = -u;
    *c = SX_DDIV(1.0, u);
    *s = SX_DMUL(-t, *c);
  } else {
    const double t = SX_DDIV(p, q);
    double u = SX_DSQRT(SX_DADD(1.0, SX_DMUL(t, t)));
    if (q < 0.0) u = -u;
    *s = SX_DDIV(-1.0, u);
    *c = SX_DMUL(-t, *s);
  }
}

/* tridiagonal_qr_step (SelfAdjointEigenSolver.h), Q = Q * G on the right */
SX_HD void sx_tridiag_qr_step(double* diag, double* sub, int start, int end, double* Q) {
  const double td = SX_DMUL(SX_DSUB(diag[end - 1], diag[end]), 0.5);
  const double e = sub[end - 1];
  double mu = diag[end];
  if (td == 0.0) {
    mu = SX_DSUB(mu, sx_fabs(e));
  } else if (e != 0.0) {
    const double e2 = SX_DMUL(e, e);
    const double h = sx_hypot(td, e);
    const double den = SX_DADD(td, td > 0.0 ? h : -h);
    if (e2 == 0.0)
      mu = SX_DSUB(mu, SX_DDIV(e, SX_DDIV(den, e)));
    else
      mu = SX_DSUB(mu, SX_DDIV(e2, den));
  }
  double x = SX_DSUB(diag[start], mu);
  double z = sub[start];
  for (int k = start; k < end && z != 0.0; ++k) {
    double c, s;
    sx_givens(x, z, &c, &s);
    const double sdk = SX_DADD(SX_DMUL(s, diag[k]), SX_DMUL(c, sub[k]));
    const double dkp1 = SX_DADD(SX_DMUL(s, sub[k]), SX_DMUL(c, diag[k + 1]));
    diag[k] = SX_DSUB(SX_DMUL(c, SX_DSUB(SX_DMUL(c, diag[k]), SX_DMUL(s, sub[k]))),
                      SX_DMUL(s, SX_DSUB(SX_DMUL(c, sub[k]), SX_DMUL(s, diag[k + 1]))));
    diag[k + 1] = SX_DADD(SX_DMUL(s, sdk), SX_DMUL(c, dkp1));
    sub[k] = SX_DSUB(SX_DMUL(c, sdk), SX_DMUL(s, dkp1));
    if (k > start) sub[k - 1] = SX_DSUB(SX_DMUL(c, sub[k - 1]), SX_DMUL(s, z));
    x = sub[k];
    if (k < end - 1) {
      z = SX_DMUL(-s, sub[k + 1]);
      sub[k + 1] = SX_DMUL(c, sub[k + 1]);
    }
    /* applyOnTheRight(k, k+1, G) = apply_rotation_in_the_plane(col k, col k+1, G^T),
     * G^T = (c, -s): x' = c x + (-s) y, y' = s x + c y */
    for (int i = 0; i < 3; ++i) {
      const double xi = SX_M(Q, i, k), yi = SX_M(Q, i, k + 1);
      SX_M(Q, i, k) = SX_DADD(SX_DMUL(c, xi), SX_DMUL(-s, yi));
      SX_M(Q, i, k + 1) = SX_DADD(SX_DMUL(s, xi), SX_DMUL(c, yi));
    }
  }
}

/* SelfAdjointEigenSolver<Matrix3d>(a): ascending eigenvalues ev[3], eigenvectors
 * as the columns of V. Reads the lower triangle of a. Returns 0 (Success) or
 * 1 (NoConvergence after 30 n QR steps). */
SX_HD int sx_sym_eigen3(const double* a, double* ev, double* V) {
  double mat[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) SX_M(mat, r, c) = c <= r ? SX_M(a, r, c) : 0.0;
  double scale = 0.0;
  for (int i = 0; i < 9; ++i) {
    const double v = sx_fabs(mat[i]);
    if (v > scale) scale = v;
  }
  if (scale == 0.0) scale = 1.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c <= r; ++c) SX_M(mat, r, c) = SX_DDIV(SX_M(mat, r, c), scale);
  double diag[3], sub[2];
  /* tridiagonalization_inplace_selector<Matrix3, 3, false> (Tridiagonalization.h) */
  diag[0] = SX_M(mat, 0, 0);
  const double v1norm2 = SX_DMUL(SX_M(mat, 2, 0), SX_M(mat, 2, 0));
  if (v1norm2 <= 2.2250738585072014e-308) {
    diag[1] = SX_M(mat, 1, 1);
    diag[2] = SX_M(mat, 2, 2);
    sub[0] = SX_M(mat, 1, 0);
    sub[1] = SX_M(mat, 2, 1);
    for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  } else {
    const double beta = SX_DSQRT(SX_DADD(SX_DMUL(SX_M(mat, 1, 0), SX_M(mat, 1, 0)), v1norm2));
    const double inv_beta = SX_DDIV(1.0, beta);
    const double m01 = SX_DMUL(SX_M(mat, 1, 0), inv_beta);
    const double m02 = SX_DMUL(SX_M(mat, 2, 0), inv_beta);
    const double q = SX_DADD(SX_DMUL(SX_DMUL(2.0, m01), SX_M(mat, 2, 1)),
                             SX_DMUL(m02, SX_DSUB(SX_M(mat, 2, 2), SX_M(mat, 1, 1))));
    diag[1] = SX_DADD(SX_M(mat, 1, 1), SX_DMUL(m02, q));
    diag[2] = SX_DSUB(SX_M(mat, 2, 2), SX_DMUL(m02, q));
    sub[0] = beta;
    sub[1] = SX_DSUB(SX_M(mat, 2, 1), SX_DMUL(m01, q));
    V[0] = 1.0, V[1] = 0.0, V[2] = 0.0;
    V[3] = 0.0, V[4] = m01, V[5] = m02;
    V[6] = 0.0, V[7] = m02, V[8] = -m01;
  }
  /* computeFromTridiagonal_impl */
  int end = 2, start = 0, iter = 0;
  const double consider_zero = 2.2250738585072014e-308;
  const double precision_inv = 4503599627370496.0; /* 1 / DBL_EPSILON */
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (sx_fabs(sub[i]) < consider_zero) {
        sub[i] = 0.0;
      } else {
        const double scaled = SX_DMUL(precision_inv, sub[i]);
        if (SX_DMUL(scaled, scaled) <= SX_DADD(sx_fabs(diag[i]), sx_fabs(diag[i + 1]))) sub[i] = 0.0;
      }
    }
    while (end > 0 && sub[end - 1] == 0.0) end--;
    if (end <= 0) break;
    iter++;
    if (iter > 30 * 3) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;
    sx_tridiag_qr_step(diag, sub, start, end, V);
  }
  if (iter > 30 * 3) return 1;
  for (int i = 0; i < 2; ++i) { /* sort ascending: minCoeff(&k) keeps the first minimum */
    int k = 0;
    for (int j = 1; j < 3 - i; ++j)
      if (diag[i + j] < diag[i + k]) k = j;
    if (k > 0) {
      const double t = diag[i];
      diag[i] = diag[i + k];
      diag[i + k] = t;
      for (int r = 0; r < 3; ++r) {
        const double u = SX_M(V, r, i);
        SX_M(V, r, i) = SX_M(V, r, i + k);
        SX_M(V, r, i + k) = u;
      }
    }
  }
  for (int i = 0; i < 3; ++i) ev[i] = SX_DMUL(diag[i], scale);
  return 0;
}

/* V diag(l) V^T, Eigen's coefficient order r_ij = a_i0 v_j0 + (a_i1 v_j1 + a_i2 v_j2) */
SX_HD void sx_recompose3(const double* V, const double* l, double* out) {
  double A[9];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) SX_M(A, r, k) = SX_DMUL(SX_M(V, r, k), l[k]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      SX_M(out, i, j) = SX_DADD(SX_DMUL(SX_M(A, i, 0), SX_M(V, j, 0)),
                                SX_DADD(SX_DMUL(SX_M(A, i, 1), SX_M(V, j, 1)),
                                        SX_DMUL(SX_M(A, i, 2), SX_M(V, j, 2))));
}

/* bandwidth_from_moment (abmsod.cpp:23-41). Returns 0 ok, 1 zero weight mass,
 * 2 non-finite moment (both std::invalid_argument), 3 eigen decomposition
 * failed (std::runtime_error). */
SX_HD int sx_bandwidth_from_moment(const double* outer, double wsum, int dim, double lambda_min,
                                   double lambda_max, double* H) {
  if (wsum <= 0.0) return 1;
  for (int i = 0; i < 9; ++i)
    if (!(SX_DSUB(outer[i], outer[i]) == 0.0)) return 2; /* allFinite */
  double m[9], sym[9];
  for (int i = 0; i < 9; ++i) m[i] = SX_DDIV(outer[i], wsum);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) SX_M(sym, r, c) = SX_DMUL(0.5, SX_DADD(SX_M(m, r, c), SX_M(m, c, r)));
  const double f = (double)(dim + 2);
  for (int i = 0; i < 9; ++i) sym[i] = SX_DMUL(sym[i], f);
  double ev[3], V[9];
  if (sx_sym_eigen3(sym, ev, V) != 0) return 3;
  for (int i = 0; i < 3; ++i) /* std::clamp(v, lo, hi) */
    ev[i] = ev[i] < lambda_min ? lambda_min : (lambda_max < ev[i] ? lambda_max : ev[i]);
  sx_recompose3(V, ev, H);
  return 0;
}

#endif
