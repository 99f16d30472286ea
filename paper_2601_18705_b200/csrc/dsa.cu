// K6: diffusion synthetic acceleration (DSA) of the source iteration on the
// device (transport_sn.py:166-198 dsa_system, :325-350 pcg, :353-367
// dsa_correct, applied at :439-441).
//
// The reference assembles the SPD even-parity operator
//
//   A = (Px^T Mt^-1 Px + Py^T Mt^-1 Py) / 3 + 2 kx Jx + 2 ky Jy + M_(sigma_t - sigma_s)
//
// as a scipy CSR matrix and solves A delta = M (sigma_s (phi_half - phi)) by
// Jacobi-preconditioned CG.  Here A is never stored: on the structured grid
// every term is a cell stencil of the 4x4 reference blocks (the same ones
// the sweep uses), so A p at a cell is evaluated from p on the cell and its
// x/y neighbours up to distance 2, with Mt^-1 = Mhat^-1 / (sigma_t dx dy) per
// cell.  The whole CG runs in ONE cooperative launch: per iteration three
// grid barriers (p.Ap, then r.r and r.z, then the new direction), fixed-order
// block partials (deterministic), the reference's exact CG recurrences and
// stopping rule (||r|| <= tol ||b||).
//
// Block structure of Px (transport_sn.py:228-258): the diagonal block of
// every cell is Gx + 1/2 E_R - 1/2 E_L (interior and boundary faces give the
// same diagonal), the off-diagonal blocks couple a cell's right-edge dofs to
// the right neighbour's left-edge dofs with +1/2 e2 and its left-edge dofs
// to the left neighbour's right-edge dofs with -1/2 e2.  Jx has 1/2 E_R +
// 1/2 E_L on the diagonal and -1/2 e2 to both neighbours.  y alike with the
// bottom (0,1) / top (2,3) edges.

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace dlrsn {
namespace {

constexpr int kDsaT = 256;

struct DsaArgs {
  int nx, ny;
  double mass[16], gx[16], gy[16], minv[16];
  double e2x[4], e2y[4];
  double kx2, ky2;  // 2 kx, 2 ky (penalty weights)
  const double* sigma_t;
  const double* sigma_s;
  const double* phi_half;
  const double* phi_old;
  double* phi_out;  // phi_half + delta
  double *x, *r, *z, *p, *dinv, *part;
  double tol;
  int max_iters;
  int* info;  // [0] iterations, [1] status (0 ok, 1 CG cap reached)
  double* history;
  int hist_cap;
  // one-call step (dsa_correct_launch): penalty weights (kx, ky) read from
  // the device, the launch returns at once when *skip is set (a converged
  // source iteration), and info accumulates over the step's launches:
  // [1] sticky failure, [2] total CG iterations, [3] launches that solved
  const double* k_dev;
  const int* skip;
  int accumulate;
};

__device__ __forceinline__ void ld4(const double* v, int64_t c, double o[4]) {
  const double2 a = reinterpret_cast<const double2*>(v)[2 * c];
  const double2 b = reinterpret_cast<const double2*>(v)[2 * c + 1];
  o[0] = a.x;
  o[1] = a.y;
  o[2] = b.x;
  o[3] = b.y;
}
__device__ __forceinline__ void st4(double* v, int64_t c, const double o[4]) {
  reinterpret_cast<double2*>(v)[2 * c] = make_double2(o[0], o[1]);
  reinterpret_cast<double2*>(v)[2 * c + 1] = make_double2(o[2], o[3]);
}

// e2 (2x2) applied to an edge pair / its transpose
__device__ __forceinline__ void e2mul(const double* e, double u0, double u1, double& o0,
                                      double& o1) {
  o0 = e[0] * u0 + e[1] * u1;
  o1 = e[2] * u0 + e[3] * u1;
}
__device__ __forceinline__ void e2tmul(const double* e, double u0, double u1, double& o0,
                                       double& o1) {
  o0 = e[0] * u0 + e[2] * u1;
  o1 = e[1] * u0 + e[3] * u1;
}

// w = Mt_c^-1 (Px v)_c  (axis 0) or Mt_c^-1 (Py v)_c (axis 1)
// edges: axis 0: lo = left (0,2), hi = right (1,3); axis 1: lo = bottom (0,1), hi = top (2,3)
template <int AX>
__device__ void mtinv_p(const DsaArgs& a, const double* v, int i, int j, double w[4]) {
  const int64_t c = (int64_t)j * a.nx + i;
  const double* G = AX == 0 ? a.gx : a.gy;
  const double* e = AX == 0 ? a.e2x : a.e2y;
  constexpr int lo0 = 0, lo1 = AX == 0 ? 2 : 1, hi0 = AX == 0 ? 1 : 2, hi1 = 3;
  double vc[4], o[4];
  ld4(v, c, vc);
#pragma unroll
  for (int l = 0; l < 4; ++l)
    o[l] = G[4 * l] * vc[0] + G[4 * l + 1] * vc[1] + G[4 * l + 2] * vc[2] + G[4 * l + 3] * vc[3];
  double t0, t1;
  e2mul(e, vc[hi0], vc[hi1], t0, t1);
  o[hi0] += 0.5 * t0;
  o[hi1] += 0.5 * t1;
  e2mul(e, vc[lo0], vc[lo1], t0, t1);
  o[lo0] -= 0.5 * t0;
  o[lo1] -= 0.5 * t1;
  const bool has_hi = AX == 0 ? i < a.nx - 1 : j < a.ny - 1;
  const bool has_lo = AX == 0 ? i > 0 : j > 0;
  const int64_t step = AX == 0 ? 1 : a.nx;
  if (has_hi) {  // neighbour's lo edge -> my hi edge, +1/2 e2
    double vn[4];
    ld4(v, c + step, vn);
    e2mul(e, vn[lo0], vn[lo1], t0, t1);
    o[hi0] += 0.5 * t0;
    o[hi1] += 0.5 * t1;
  }
  if (has_lo) {  // neighbour's hi edge -> my lo edge, -1/2 e2
    double vn[4];
    ld4(v, c - step, vn);
    e2mul(e, vn[hi0], vn[hi1], t0, t1);
    o[lo0] -= 0.5 * t0;
    o[lo1] -= 0.5 * t1;
  }
  const double s = 1.0 / a.sigma_t[c];
#pragma unroll
  for (int l = 0; l < 4; ++l)
    w[l] = s * (a.minv[4 * l] * o[0] + a.minv[4 * l + 1] * o[1] + a.minv[4 * l + 2] * o[2] +
                a.minv[4 * l + 3] * o[3]);
}

// (P^T w)_c for w = Mt^-1 P v, accumulated into acc; plus pen * (J v)_c
template <int AX>
__device__ void pt_mtinv_p_plus_j(const DsaArgs& a, const double* v, int i, int j, double pen,
                                  double acc[4]) {
  const double* G = AX == 0 ? a.gx : a.gy;
  const double* e = AX == 0 ? a.e2x : a.e2y;
  constexpr int lo0 = 0, lo1 = AX == 0 ? 2 : 1, hi0 = AX == 0 ? 1 : 2, hi1 = 3;
  const bool has_hi = AX == 0 ? i < a.nx - 1 : j < a.ny - 1;
  const bool has_lo = AX == 0 ? i > 0 : j > 0;
  const int di = AX == 0 ? 1 : 0, dj = AX == 0 ? 0 : 1;
  double w[4], o[4], t0, t1;
  mtinv_p<AX>(a, v, i, j, w);
  // D^T w: G^T w + 1/2 E_hi^T w - 1/2 E_lo^T w
#pragma unroll
  for (int l = 0; l < 4; ++l) o[l] = G[l] * w[0] + G[4 + l] * w[1] + G[8 + l] * w[2] + G[12 + l] * w[3];
  e2tmul(e, w[hi0], w[hi1], t0, t1);
  o[hi0] += 0.5 * t0;
  o[hi1] += 0.5 * t1;
  e2tmul(e, w[lo0], w[lo1], t0, t1);
  o[lo0] -= 0.5 * t0;
  o[lo1] -= 0.5 * t1;
  if (has_hi) {  // block (row c+1, col c) = -1/2 e2 (c+1's lo <- my hi)
    double wn[4];
    mtinv_p<AX>(a, v, i + di, j + dj, wn);
    e2tmul(e, wn[lo0], wn[lo1], t0, t1);
    o[hi0] -= 0.5 * t0;
    o[hi1] -= 0.5 * t1;
  }
  if (has_lo) {  // block (row c-1, col c) = +1/2 e2 (c-1's hi <- my lo)
    double wn[4];
    mtinv_p<AX>(a, v, i - di, j - dj, wn);
    e2tmul(e, wn[hi0], wn[hi1], t0, t1);
    o[lo0] += 0.5 * t0;
    o[lo1] += 0.5 * t1;
  }
#pragma unroll
  for (int l = 0; l < 4; ++l) acc[l] += o[l] * (1.0 / 3.0);
  // penalty: J v = 1/2 E_hi v_c + 1/2 E_lo v_c - 1/2 e2 (neighbours)
  const int64_t c = (int64_t)j * a.nx + i;
  const int64_t step = AX == 0 ? 1 : a.nx;
  double vc[4];
  ld4(v, c, vc);
  double jv[4] = {0.0, 0.0, 0.0, 0.0};
  e2mul(e, vc[hi0], vc[hi1], t0, t1);
  jv[hi0] += 0.5 * t0;
  jv[hi1] += 0.5 * t1;
  e2mul(e, vc[lo0], vc[lo1], t0, t1);
  jv[lo0] += 0.5 * t0;
  jv[lo1] += 0.5 * t1;
  if (has_hi) {
    double vn[4];
    ld4(v, c + step, vn);
    e2mul(e, vn[lo0], vn[lo1], t0, t1);
    jv[hi0] -= 0.5 * t0;
    jv[hi1] -= 0.5 * t1;
  }
  if (has_lo) {
    double vn[4];
    ld4(v, c - step, vn);
    e2mul(e, vn[hi0], vn[hi1], t0, t1);
    jv[lo0] -= 0.5 * t0;
    jv[lo1] -= 0.5 * t1;
  }
#pragma unroll
  for (int l = 0; l < 4; ++l) acc[l] += pen * jv[l];
}

__device__ void apply_a(const DsaArgs& a, double kx2, double ky2, const double* v, int i, int j,
                        double out[4]) {
  const int64_t c = (int64_t)j * a.nx + i;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  pt_mtinv_p_plus_j<0>(a, v, i, j, kx2, acc);
  pt_mtinv_p_plus_j<1>(a, v, i, j, ky2, acc);
  double vc[4];
  ld4(v, c, vc);
  const double sa = a.sigma_t[c] - a.sigma_s[c];
#pragma unroll
  for (int l = 0; l < 4; ++l)
    out[l] = acc[l] + sa * (a.mass[4 * l] * vc[0] + a.mass[4 * l + 1] * vc[1] +
                            a.mass[4 * l + 2] * vc[2] + a.mass[4 * l + 3] * vc[3]);
}

// quadratic form u^T (minv / s) u over the dof pair (d0, d1) with u = (u0, u1)
__device__ __forceinline__ double qf2(const DsaArgs& a, int d0, int d1, double u0, double u1,
                                      double s) {
  return (u0 * (a.minv[4 * d0 + d0] * u0 + a.minv[4 * d0 + d1] * u1) +
          u1 * (a.minv[4 * d1 + d0] * u0 + a.minv[4 * d1 + d1] * u1)) / s;
}

// diag(A) at (cell, local l) -- the Jacobi preconditioner (transport_sn.py:196)
template <int AX>
__device__ double diag_axis(const DsaArgs& a, int i, int j, int l, double pen) {
  const double* G = AX == 0 ? a.gx : a.gy;
  const double* e = AX == 0 ? a.e2x : a.e2y;
  constexpr int lo0 = 0, lo1 = AX == 0 ? 2 : 1, hi0 = AX == 0 ? 1 : 2, hi1 = 3;
  const int64_t c = (int64_t)j * a.nx + i;
  const int64_t step = AX == 0 ? 1 : a.nx;
  // column l of the diagonal block D
  double col[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) col[k] = G[4 * k + l];
  const int phi = l == hi0 ? 0 : (l == hi1 ? 1 : -1);
  const int plo = l == lo0 ? 0 : (l == lo1 ? 1 : -1);
  if (phi >= 0) {
    col[hi0] += 0.5 * e[phi];
    col[hi1] += 0.5 * e[2 + phi];
  }
  if (plo >= 0) {
    col[lo0] -= 0.5 * e[plo];
    col[lo1] -= 0.5 * e[2 + plo];
  }
  double q = 0.0;
  const double s = a.sigma_t[c];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) t += a.minv[4 * k + m] * col[m];
    q += col[k] * t;
  }
  q /= s;
  const bool has_hi = AX == 0 ? i < a.nx - 1 : j < a.ny - 1;
  const bool has_lo = AX == 0 ? i > 0 : j > 0;
  if (plo >= 0 && has_lo)  // block (row c-1, col c): +1/2 e2 into c-1's hi edge
    q += qf2(a, hi0, hi1, 0.5 * e[plo], 0.5 * e[2 + plo], a.sigma_t[c - step]);
  if (phi >= 0 && has_hi)  // block (row c+1, col c): -1/2 e2 into c+1's lo edge
    q += qf2(a, lo0, lo1, -0.5 * e[phi], -0.5 * e[2 + phi], a.sigma_t[c + step]);
  double jd = 0.0;
  if (phi >= 0) jd += 0.5 * e[3 * phi];
  if (plo >= 0) jd += 0.5 * e[3 * plo];
  return q / 3.0 + pen * jd;
}

// block sum of two values; result valid in thread 0
__device__ __forceinline__ void block_sum2(double& v0, double& v1, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_down_sync(kFull, v0, o);
    v1 += __shfl_down_sync(kFull, v1, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[2 * w] = v0;
    red[2 * w + 1] = v1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      s0 += red[2 * k];
      s1 += red[2 * k + 1];
    }
    v0 = s0;
    v1 = s1;
  }
}

// grid total of the per-block partial pairs (fixed order, identical in
// every block); result broadcast to all threads
__device__ __forceinline__ void grid_total2(const double* part, double& t0, double& t1,
                                            double* bc) {
  if (threadIdx.x < 32) {
    double s0 = 0.0, s1 = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
      s0 += __ldcg(part + 2 * b);
      s1 += __ldcg(part + 2 * b + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_down_sync(kFull, s0, o);
      s1 += __shfl_down_sync(kFull, s1, o);
    }
    if (threadIdx.x == 0) {
      bc[0] = s0;
      bc[1] = s1;
    }
  }
  __syncthreads();
  t0 = bc[0];
  t1 = bc[1];
  __syncthreads();
}

__global__ void __launch_bounds__(kDsaT) dsa_pcg_kernel(const DsaArgs a) {
  if (a.skip && *a.skip) return;  // uniform over the grid: no barrier is reached
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[2 * (kDsaT / 32)];
  __shared__ double bc[2];
  const double kx2 = a.k_dev ? 2.0 * a.k_dev[0] : a.kx2;
  const double ky2 = a.k_dev ? 2.0 * a.k_dev[1] : a.ky2;
  const int nc = a.nx * a.ny;
  const int nth = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  double* part0 = a.part;
  double* part1 = a.part + 2 * gridDim.x;
  // setup: b = M (sigma_s (phi_half - phi_old)); x = 0; r = b; z = D^-1 r; p = z
  double s0 = 0.0, s1 = 0.0;
  for (int c = t0; c < nc; c += nth) {
    const int i = c % a.nx, j = c / a.nx;
    double ph[4], po[4], u[4], b[4], x0[4] = {0.0, 0.0, 0.0, 0.0}, z[4], dv[4];
    ld4(a.phi_half, c, ph);
    ld4(a.phi_old, c, po);
    const double ss = a.sigma_s[c];
#pragma unroll
    for (int l = 0; l < 4; ++l) u[l] = ss * (ph[l] - po[l]);
#pragma unroll
    for (int l = 0; l < 4; ++l)
      b[l] = a.mass[4 * l] * u[0] + a.mass[4 * l + 1] * u[1] + a.mass[4 * l + 2] * u[2] +
             a.mass[4 * l + 3] * u[3];
    const double sa = a.sigma_t[c] - a.sigma_s[c];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const double d = diag_axis<0>(a, i, j, l, kx2) + diag_axis<1>(a, i, j, l, ky2) +
                       sa * a.mass[5 * l];
      dv[l] = 1.0 / d;
      z[l] = dv[l] * b[l];
      s0 += b[l] * b[l];
      s1 += b[l] * z[l];
    }
    st4(a.dinv, c, dv);
    st4(a.x, c, x0);
    st4(a.r, c, b);
    st4(a.z, c, z);
    st4(a.p, c, z);
  }
  block_sum2(s0, s1, red);
  if (threadIdx.x == 0) {
    part0[2 * blockIdx.x] = s0;
    part0[2 * blockIdx.x + 1] = s1;
  }
  grid.sync();
  double bb, rz;
  grid_total2(part0, bb, rz, bc);
  const double bnorm = sqrt(bb);
  if (bnorm == 0.0) {  // dsa_correct: no residual, no correction (:364-365)
    for (int c = t0; c < nc; c += nth) {
      double ph[4];
      ld4(a.phi_half, c, ph);
      st4(a.phi_out, c, ph);
    }
    if (t0 == 0) {
      a.info[0] = 0;
      if (!a.accumulate) a.info[1] = 0;
    }
    return;
  }
  // the history of a step's first failed solve is kept (accumulate mode)
  const bool hist_on = a.history && !(a.accumulate && a.info[1]);
  if (t0 == 0 && hist_on && a.hist_cap > 0) a.history[0] = bnorm;
  int it = 1;
  bool done = false;
  for (; it <= a.max_iters; ++it) {
    // ap = A p (kept in z), partial p.ap
    s0 = 0.0;
    s1 = 0.0;
    for (int c = t0; c < nc; c += nth) {
      const int i = c % a.nx, j = c / a.nx;
      double ap[4], pc[4];
      apply_a(a, kx2, ky2, a.p, i, j, ap);
      ld4(a.p, c, pc);
#pragma unroll
      for (int l = 0; l < 4; ++l) s0 += pc[l] * ap[l];
      st4(a.z, c, ap);
    }
    block_sum2(s0, s1, red);
    if (threadIdx.x == 0) {
      part0[2 * blockIdx.x] = s0;
      part0[2 * blockIdx.x + 1] = 0.0;
    }
    grid.sync();
    double pap, dummy;
    grid_total2(part0, pap, dummy, bc);
    const double alpha = rz / pap;
    // x += alpha p; r -= alpha ap; z = D^-1 r; partial r.r, r.z
    s0 = 0.0;
    s1 = 0.0;
    for (int c = t0; c < nc; c += nth) {
      double x[4], r[4], p[4], ap[4], dv[4], z[4];
      ld4(a.x, c, x);
      ld4(a.r, c, r);
      ld4(a.p, c, p);
      ld4(a.z, c, ap);
      ld4(a.dinv, c, dv);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        x[l] += alpha * p[l];
        r[l] -= alpha * ap[l];
        z[l] = dv[l] * r[l];
        s0 += r[l] * r[l];
        s1 += r[l] * z[l];
      }
      st4(a.x, c, x);
      st4(a.r, c, r);
      st4(a.z, c, z);
    }
    block_sum2(s0, s1, red);
    if (threadIdx.x == 0) {
      part1[2 * blockIdx.x] = s0;
      part1[2 * blockIdx.x + 1] = s1;
    }
    grid.sync();
    double rr, rz_new;
    grid_total2(part1, rr, rz_new, bc);
    const double rnorm = sqrt(rr);
    if (t0 == 0 && hist_on && it < a.hist_cap) a.history[it] = rnorm;
    if (rnorm <= a.tol * bnorm) {
      done = true;
      break;
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int c = t0; c < nc; c += nth) {
      double p[4], z[4];
      ld4(a.p, c, p);
      ld4(a.z, c, z);
#pragma unroll
      for (int l = 0; l < 4; ++l) p[l] = z[l] + beta * p[l];
      st4(a.p, c, p);
    }
    grid.sync();
  }
  // phi_out = phi_half + delta (transport_sn.py:440-441)
  for (int c = t0; c < nc; c += nth) {
    double ph[4], x[4];
    ld4(a.phi_half, c, ph);
    ld4(a.x, c, x);
#pragma unroll
    for (int l = 0; l < 4; ++l) ph[l] += x[l];
    st4(a.phi_out, c, ph);
  }
  if (t0 == 0) {
    a.info[0] = done ? it : a.max_iters;
    if (!a.accumulate) {
      a.info[1] = done ? 0 : 1;
    } else {
      if (!done) a.info[1] = 1;
      a.info[2] += done ? it : a.max_iters;
      a.info[3] += 1;
    }
  }
}

void inv4(const double* m, double* out) {
  // Gauss-Jordan with partial pivoting on the (symmetric positive definite) mass block
  double a[4][8];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 8; ++j) a[i][j] = j < 4 ? m[4 * i + j] : (j - 4 == i ? 1.0 : 0.0);
  for (int k = 0; k < 4; ++k) {
    int piv = k;
    for (int i = k + 1; i < 4; ++i)
      if (fabs(a[i][k]) > fabs(a[piv][k])) piv = i;
    if (piv != k)
      for (int j = 0; j < 8; ++j) {
        const double t = a[k][j];
        a[k][j] = a[piv][j];
        a[piv][j] = t;
      }
    const double d = a[k][k];
    for (int j = 0; j < 8; ++j) a[k][j] /= d;
    for (int i = 0; i < 4; ++i)
      if (i != k) {
        const double f = a[i][k];
        for (int j = 0; j < 8; ++j) a[i][j] -= f * a[k][j];
      }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = a[i][j + 4];
}

}  // namespace

int dsa_correct_launch(const dlrsn_cellops* ops, const double* sigma_t, const double* sigma_s,
                       double kx, double ky, const double* k_dev, const double* phi_half,
                       const double* phi_old, double* phi_out, double tol, int max_iters,
                       double* workspace, int* info, double* history, int hist_cap,
                       const int* skip, int accumulate, cudaStream_t st) {
  const int64_t nd = 4 * (int64_t)ops->nx * ops->ny;
  DsaArgs a;
  a.nx = ops->nx;
  a.ny = ops->ny;
  memcpy(a.mass, ops->mass, sizeof(a.mass));
  memcpy(a.gx, ops->gx, sizeof(a.gx));
  memcpy(a.gy, ops->gy, sizeof(a.gy));
  memcpy(a.e2x, ops->e2x, sizeof(a.e2x));
  memcpy(a.e2y, ops->e2y, sizeof(a.e2y));
  inv4(ops->mass, a.minv);
  a.kx2 = 2.0 * kx;
  a.ky2 = 2.0 * ky;
  a.sigma_t = sigma_t;
  a.sigma_s = sigma_s;
  a.phi_half = phi_half;
  a.phi_old = phi_old;
  a.phi_out = phi_out;
  a.x = workspace;
  a.r = workspace + nd;
  a.z = workspace + 2 * nd;
  a.p = workspace + 3 * nd;
  a.dinv = workspace + 4 * nd;
  a.part = workspace + 5 * nd;
  a.tol = tol;
  a.max_iters = max_iters;
  a.info = info;
  a.history = history;
  a.hist_cap = history ? hist_cap : 0;
  a.k_dev = k_dev;
  a.skip = skip;
  a.accumulate = accumulate;
  static thread_local int cached_dev = -1, cached_cap = 0;
  int dev = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  if (dev != cached_dev) {  // the occupancy query is not capturable: once per device
    int sms = 0, occ = 0;
    DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dsa_pcg_kernel, kDsaT, 0));
    cached_cap = sms * (occ < 1 ? 1 : (occ > 8 ? 8 : occ));
    cached_dev = dev;
  }
  const int nc = ops->nx * ops->ny;
  int blocks = (nc + kDsaT - 1) / kDsaT;
  if (blocks > cached_cap) blocks = cached_cap;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  void* params[] = {&a};
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  DLRSN_TRY_CUDA(cudaLaunchCooperativeKernel((const void*)dsa_pcg_kernel, dim3(blocks),
                                             dim3(kDsaT), params, 0, st));
  return DLRSN_OK;
}

}  // namespace dlrsn

using namespace dlrsn;

extern "C" {

int64_t dlrsn_dsa_workspace_len(int nx, int ny) {
  const int64_t nd = 4 * (int64_t)nx * ny;
  return 5 * nd + 4 * 148 * 8 + 64;
}

int dlrsn_dsa_correct(const dlrsn_cellops* ops, const double* sigma_t, const double* sigma_s,
                      double kx, double ky, const double* phi_half, const double* phi_old,
                      double* phi_out, double tol, int max_iters, double* workspace,
                      int64_t workspace_len, int* info, double* history, int hist_cap,
                      dlrsn_stream_t stream) {
  DLRSN_REQUIRE(ops && sigma_t && sigma_s && phi_half && phi_old && phi_out && workspace && info,
                "bad arguments to dlrsn_dsa_correct");
  DLRSN_REQUIRE(max_iters >= 1, "max_iters must be positive");
  DLRSN_REQUIRE(workspace_len >= dlrsn_dsa_workspace_len(ops->nx, ops->ny),
                "dsa workspace too small");
  return dsa_correct_launch(ops, sigma_t, sigma_s, kx, ky, nullptr, phi_half, phi_old, phi_out, tol,
                            max_iters, workspace, info, history, hist_cap, nullptr, 0,
                            as_stream(stream));
}

}  // extern "C"
