/*
 * csweep.c -- TEST INFRASTRUCTURE (oracle).  Plain-C restatement of the
 * reference's per-direction upwind sweep, used by oracle/port.py's
 * sweep_many so the CPU oracle finishes the BASELINE configs at full size
 * (C2 50 steps, C3 512^2, C4 1024^2) in minutes instead of hours.  Never
 * linked into the product library.
 *
 * Per direction (transport_sn.py:142-163, 303-322):
 *   A_c   = stream + sigma_t[c] * mass        (stream = wx Gx + wy Gy +
 *           |wx| E_out,x + |wy| E_out,y, built by the caller per direction)
 *   Ainv  = inv(A_c)                          (np.linalg.inv: LU with partial
 *                                              pivoting, then solve A X = I)
 *   local = rhs_c + |wx| cx psi_xn + |wy| cy psi_yn   (neighbours upwind;
 *           absent at the inflow walls: vacuum)
 *   psi_c = Ainv local
 * Cells are visited row by row in the oriented frame (i' = sx>0 ? i : nx-1-i,
 * likewise j'), a topological order of the upwind dependencies equivalent
 * to the reference's anti-diagonal levels (each cell's arithmetic depends
 * only on its two upwind neighbours).  Directions run in parallel (OpenMP).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* 4x4 inverse the way LAPACK dgesv(A, I) forms it: dgetrf (partial
 * pivoting, row interchanges) then forward / back substitution per column. */
static void inv4(const double a_in[16], double inv[16]) {
  double a[16];
  int piv[4];
  memcpy(a, a_in, sizeof(a));
  for (int k = 0; k < 4; ++k) {
    int p = k;
    double m = a[k * 4 + k] < 0 ? -a[k * 4 + k] : a[k * 4 + k];
    for (int i = k + 1; i < 4; ++i) {
      const double v = a[i * 4 + k] < 0 ? -a[i * 4 + k] : a[i * 4 + k];
      if (v > m) { m = v; p = i; }
    }
    piv[k] = p;
    if (p != k)
      for (int j = 0; j < 4; ++j) {
        const double t = a[k * 4 + j];
        a[k * 4 + j] = a[p * 4 + j];
        a[p * 4 + j] = t;
      }
    const double r = 1.0 / a[k * 4 + k];
    for (int i = k + 1; i < 4; ++i) {
      a[i * 4 + k] *= r;
      const double l = a[i * 4 + k];
      for (int j = k + 1; j < 4; ++j) a[i * 4 + j] -= l * a[k * 4 + j];
    }
  }
  for (int c = 0; c < 4; ++c) {
    double x[4] = {0.0, 0.0, 0.0, 0.0};
    x[c] = 1.0;
    for (int k = 0; k < 4; ++k)  /* apply the row interchanges */
      if (piv[k] != k) {
        const double t = x[k];
        x[k] = x[piv[k]];
        x[piv[k]] = t;
      }
    for (int i = 1; i < 4; ++i)
      for (int j = 0; j < i; ++j) x[i] -= a[i * 4 + j] * x[j];
    for (int i = 3; i >= 0; --i) {
      for (int j = i + 1; j < 4; ++j) x[i] -= a[i * 4 + j] * x[j];
      x[i] /= a[i * 4 + i];
    }
    for (int i = 0; i < 4; ++i) inv[i * 4 + c] = x[i];
  }
}

/* D directions of one quadrant (sx, sy).  rhs / psi are (4 nx ny, ld)
 * row-major; direction d reads column rcol[d] of rhs and writes column
 * pcol[d] of psi.  stream: D x 16, mass / cx / cy: 16 (row-major). */
void csweep_quadrant(int nx, int ny, int sx, int sy, int D, const double* stream,
                     const double* mass, const double* sigma_t, const double* cx,
                     const double* cy, const double* ox, const double* oy, const double* rhs,
                     int64_t ld_rhs, const int* rcol, double* psi, int64_t ld_psi,
                     const int* pcol, int nthreads) {
  const int64_t nc = (int64_t)nx * ny;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)nc);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int d = 0; d < D; ++d) {
      const double* st = stream + 16 * (size_t)d;
      const double wx = ox[d], wy = oy[d];
      for (int jp = 0; jp < ny; ++jp) {
        const int j = sy > 0 ? jp : ny - 1 - jp;
        for (int ip = 0; ip < nx; ++ip) {
          const int i = sx > 0 ? ip : nx - 1 - ip;
          const int64_t c = (int64_t)j * nx + i;
          double a[16], ai[16], loc[4];
          const double s = sigma_t[c];
          for (int e = 0; e < 16; ++e) a[e] = st[e] + s * mass[e];
          inv4(a, ai);
          for (int l = 0; l < 4; ++l) loc[l] = rhs[(4 * c + l) * ld_rhs + rcol[d]];
          if (ip > 0) {  /* x-upwind neighbour (i - sx, j) */
            const double* u = buf + 4 * (c - sx);
            for (int l = 0; l < 4; ++l) {
              double t = 0.0;
              for (int m = 0; m < 4; ++m) t += u[m] * cx[l * 4 + m];
              loc[l] += t * wx;
            }
          }
          if (jp > 0) {  /* y-upwind neighbour (i, j - sy) */
            const double* u = buf + 4 * (c - (int64_t)sy * nx);
            for (int l = 0; l < 4; ++l) {
              double t = 0.0;
              for (int m = 0; m < 4; ++m) t += u[m] * cy[l * 4 + m];
              loc[l] += t * wy;
            }
          }
          double* out = buf + 4 * c;
          for (int l = 0; l < 4; ++l) {
            double t = 0.0;
            for (int m = 0; m < 4; ++m) t += ai[l * 4 + m] * loc[m];
            out[l] = t;
          }
        }
      }
      for (int64_t e = 0; e < 4 * nc; ++e) psi[e * ld_psi + pcol[d]] = buf[e];
    }
    free(buf);
  }
}

/* out = blockdiag(mass) u (then * coeff[c] per cell when coeff != NULL):
 * the per-cell mass application of transport_sn.py:107-116 for u (4 nc, k)
 * row-major (same per-entry arithmetic as the numpy einsum: a 4-term dot
 * product in j order, then the coefficient). */
void cmass_apply(int64_t nc, int64_t k, const double* mass, const double* coeff,
                 const double* u, double* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t c = 0; c < nc; ++c) {
    const double* uc = u + 4 * c * k;
    double* oc = out + 4 * c * k;
    const double s = coeff ? coeff[c] : 1.0;
    for (int i = 0; i < 4; ++i)
      for (int64_t col = 0; col < k; ++col) {
        double t = mass[i * 4 + 0] * uc[col];
        t += mass[i * 4 + 1] * uc[k + col];
        t += mass[i * 4 + 2] * uc[2 * k + col];
        t += mass[i * 4 + 3] * uc[3 * k + col];
        oc[i * k + col] = coeff ? t * s : t;
      }
  }
}
