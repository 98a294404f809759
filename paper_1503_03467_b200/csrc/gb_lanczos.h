// Host-side half of the Lanczos-moment lambda_min estimator (level engine,
// spectral mode 1).  Pure C++, no CUDA: also exported through the C ABI
// (gb_lanczos_emulate) so the CPU test suite can check it against numpy.
//
// The reference estimates lambda_min of S B S by inverse iteration
// (sparse_core.py:258-277): x_j = A^{-1} x_{j-1} / |.|, lambda_j = x_j^T A x_j,
// stop at the first j with |lambda_j - lambda_{j-1}| <= tol/2 |lambda_j|.
// With x_0 the unit start vector, lambda_j = mu_{2j-1} / mu_{2j} where
// mu_m = x_0^T A^{-m} x_0.  m Lanczos steps from x_0 give the tridiagonal T_m
// whose Gauss quadrature mu_m ~ sum_i z_i^2 theta_i^{-m} (theta_i = Ritz
// values, z_i = first components of T_m's eigenvectors); once the quadrature
// has converged the whole inverse-iteration sequence -- and its stopping
// index -- is evaluated on the host from (alpha, beta) alone, i.e. the
// reference's iteration with exact inner solves, at the cost of one Krylov
// sequence that shares its operator passes with the subband PCG.
#pragma once
#include <math.h>
#include <stdlib.h>

namespace gb_lz {

// Eigenvalues of the symmetric tridiagonal (d[0..m), e[0..m-1)) and the first
// components z of its orthonormal eigenvectors (implicit QL with Wilkinson
// shifts; only row 0 of the eigenvector matrix is carried -- the rotations act
// on each row independently).  d, e, z are overwritten; e needs m entries.
// Returns 0, or 1 if an eigenvalue failed to converge in 60 sweeps.
inline int tridiag_eig_first(int m, double* d, double* e, double* z) {
  for (int i = 0; i < m; ++i) z[i] = (i == 0) ? 1.0 : 0.0;
  if (m > 0) e[m - 1] = 0.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 1e-17 * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) return 1;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool deflated = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            deflated = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (deflated) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  return 0;
}

// lambda_min of the reference's inverse iteration, evaluated from the Lanczos
// coefficients ab = (alpha_0, beta_0, alpha_1, beta_1, ...) of m steps.
// Writes the estimate and the outer iteration count at which the reference's
// stopping test fires (max_outer if it never does).  Returns 0, 1 on a QL
// failure, 2 on a nonpositive Ritz value (operator not SPD).
inline int emulate_inverse_iteration(const double* ab, int m, double tol, int max_outer,
                                     double* lam_out, int* outer_out, double* ritz_min,
                                     double* ritz_max) {
  if (m <= 0) return 1;
  double* d = (double*)malloc(sizeof(double) * 3 * (size_t)m);
  double* e = d + m;
  double* z = e + m;
  for (int i = 0; i < m; ++i) {
    d[i] = ab[2 * i];
    e[i] = ab[2 * i + 1];
  }
  int rc = tridiag_eig_first(m, d, e, z);
  if (rc) {
    free(d);
    return 1;
  }
  double tmin = d[0], tmax = d[0];
  for (int i = 1; i < m; ++i) {
    tmin = d[i] < tmin ? d[i] : tmin;
    tmax = d[i] > tmax ? d[i] : tmax;
  }
  if (ritz_min) *ritz_min = tmin;
  if (ritz_max) *ritz_max = tmax;
  if (!(tmin > 0.0)) {
    free(d);
    return 2;
  }
  // w_i = z_i^2, r_i = tmin / theta_i <= 1: lambda_j = tmin * S_{2j-1} / S_{2j},
  // S_p = sum_i w_i r_i^p (scaled moments, no overflow)
  for (int i = 0; i < m; ++i) {
    e[i] = z[i] * z[i];
    d[i] = tmin / d[i];
  }
  double* pw = z;  // r_i^(2j-2), starts at 1
  for (int i = 0; i < m; ++i) pw[i] = 1.0;
  double lam_prev = INFINITY, lam = 0.0;
  int j;
  for (j = 1; j <= max_outer; ++j) {
    double s_odd = 0.0, s_even = 0.0;
    for (int i = 0; i < m; ++i) {
      const double a = pw[i] * d[i];  // r^(2j-1)
      const double b = a * d[i];      // r^(2j)
      s_odd += e[i] * a;
      s_even += e[i] * b;
      pw[i] = b;
    }
    lam = tmin * s_odd / s_even;
    if (fabs(lam - lam_prev) <= 0.5 * tol * fabs(lam)) break;
    lam_prev = lam;
  }
  *lam_out = lam;
  *outer_out = j > max_outer ? max_outer : j;
  free(d);
  return 0;
}

// The same sequence without the eigen-decomposition: the reference's
// iteration run on T_m itself from e_1 (x_j = T^{-1} x_{j-1} / |.|,
// lambda_j = x_j^T T x_j = (y . x_{j-1}) / (y . y) with y = T^{-1} x_{j-1}),
// each solve two sweeps of the LDL^T factors of the tridiagonal -- O(m) per
// outer step instead of the O(m^2) QL pass, so the engine can test for
// convergence often without stalling its stream.  Same stopping test and
// return codes (2: a nonpositive pivot, T_m is not positive definite).
inline int emulate_inverse_iteration_ldl(const double* ab, int m, double tol, int max_outer,
                                         double* lam_out, int* outer_out) {
  if (m <= 0) return 1;
  double* piv = (double*)malloc(sizeof(double) * 4 * (size_t)m);
  double* l = piv + m;
  double* x = l + m;
  double* y = x + m;
  piv[0] = ab[0];
  for (int i = 0; i + 1 < m; ++i) {
    if (!(piv[i] > 0.0)) {
      free(piv);
      return 2;
    }
    l[i] = ab[2 * i + 1] / piv[i];
    piv[i + 1] = ab[2 * i + 2] - l[i] * ab[2 * i + 1];
  }
  if (!(piv[m - 1] > 0.0)) {
    free(piv);
    return 2;
  }
  for (int i = 0; i < m; ++i) x[i] = (i == 0) ? 1.0 : 0.0;
  double lam_prev = INFINITY, lam = 0.0;
  int j;
  for (j = 1; j <= max_outer; ++j) {
    y[0] = x[0];
    for (int i = 0; i + 1 < m; ++i) y[i + 1] = x[i + 1] - l[i] * y[i];
    y[m - 1] /= piv[m - 1];
    for (int i = m - 2; i >= 0; --i) y[i] = y[i] / piv[i] - l[i] * y[i + 1];
    double xy = 0.0, yy = 0.0;
    for (int i = 0; i < m; ++i) {
      xy += x[i] * y[i];
      yy += y[i] * y[i];
    }
    lam = xy / yy;
    const double inv = 1.0 / sqrt(yy);
    for (int i = 0; i < m; ++i) x[i] = y[i] * inv;
    if (fabs(lam - lam_prev) <= 0.5 * tol * fabs(lam)) break;
    lam_prev = lam;
  }
  *lam_out = lam;
  *outer_out = j > max_outer ? max_outer : j;
  free(piv);
  return 0;
}

// Stopping rule of the Lanczos sequence after m steps.  The estimate
// lam(m) converges geometrically in m (tools/lanczos_convergence.py), and
// the estimates of fewer steps come for free from the leading blocks of the
// same T: with d1 = |lam(m-16) - lam(m)|, d2 = |lam(m-32) - lam(m-16)| and
// rate = d1 / d2, the remaining error is the geometric tail
// d1 rate / (1 - rate).  Stop when the three stopping indices agree, the
// differences shrink, and the tail is below lz_tol |lam|.
constexpr int kCheckBack = 16;
inline int lanczos_check(const double* ab, int m, double tol, int max_outer, double lz_tol,
                         double* lam, int* outer, int* stop) {
  *stop = 0;
  int rc = emulate_inverse_iteration_ldl(ab, m, tol, max_outer, lam, outer);
  if (rc || m <= 2 * kCheckBack) return rc;
  double l1, l2;
  int o1, o2;
  if ((rc = emulate_inverse_iteration_ldl(ab, m - kCheckBack, tol, max_outer, &l1, &o1))) return rc;
  if ((rc = emulate_inverse_iteration_ldl(ab, m - 2 * kCheckBack, tol, max_outer, &l2, &o2)))
    return rc;
  if (o1 != *outer || o2 != *outer) return 0;
  const double d1 = fabs(l1 - *lam), d2 = fabs(l2 - l1);
  if (d1 > d2) return 0;
  double rate = d2 > 0.0 ? d1 / d2 : 0.0;
  if (rate > 0.95) rate = 0.95;
  *stop = d1 * rate / (1.0 - rate) <= lz_tol * fabs(*lam);
  return 0;
}

}  // namespace gb_lz
