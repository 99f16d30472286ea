// K2/K3/K5: the Galerkin side of one DLR-SN step on the device.
//
//  * rowmix       Y = X K (+ beta Y): tall-skinny times small (evaluate_rows,
//                 phi = X l, l_full = W gamma, X R^-1)      lowrank.py:220-227
//  * mgram        G = sum_c coeff_c X_c^T M_c Y_c            lowrank.py:23-25,68-81
//  * project      the six reduced operators + q-hat in one pass over the
//                 cells, face terms included                 dlr_sn.py:61-71
//  * reduce       fixed-order sum of per-chunk partials (deterministic)
//  * small dense  Cholesky / triangular inverse (CholQR2), batched
//                 Gauss-Jordan with partial pivoting (row system), the row
//                 system combine, DEIM by left-to-right GEPP, closure/gamma
//                 solves, and an exact twice-projected CGS2 with the
//                 reference's deficiency + completion rules
//                 (angular.py:104-160,217-238; lowrank.py:158-205,235-259)
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace dlrsn {

constexpr int kRB = 256;  // threads per block for the row kernels

// ---------------------------------------------------------------------------
// rowmix: Y[i, :] = X[i, :] K  (+ beta * Y[i, :]);  X (n, kx) ld_x, K (kx, ky)
// ld_k, Y (n, ky) ld_y.  K is staged in shared memory.
__global__ void rowmix_kernel(int n, int kx, int ky, const double* __restrict__ X, int ldx,
                              const double* __restrict__ K, int ldk, double beta,
                              double* __restrict__ Y, int ldy) {
  extern __shared__ double sK[];
  for (int e = threadIdx.x; e < kx * ky; e += blockDim.x) sK[e] = K[(e / ky) * ldk + e % ky];
  __syncthreads();
  const int64_t total = (int64_t)n * ky;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / ky;
    const int j = (int)(idx - i * ky);
    const double* x = X + i * ldx;
    double acc = 0.0;
    for (int p = 0; p < kx; ++p) acc = fma(__ldg(x + p), sK[p * ky + j], acc);
    double* y = Y + i * ldy + j;
    *y = beta == 0.0 ? acc : fma(beta, *y, acc);
  }
}

// ---------------------------------------------------------------------------
// Partial-sum plumbing: kernels that reduce over cells write one partial per
// (chunk, output) and reduce_partials sums them in chunk order.
// block = 32 consecutive outputs x 8 warps; warp w sums chunks w, w+8, ...
// (coalesced), then the 8 warp sums are added in fixed order.
__global__ void reduce_partials_kernel(int nchunks, int64_t len, const double* __restrict__ part,
                                       double* __restrict__ out, double alpha) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < len)
    for (int c = w; c < nchunks; c += 8) s += part[(int64_t)c * len + e];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < len) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += red[q][lane];
    out[e] = alpha * t;
  }
}

// ---------------------------------------------------------------------------
// mgram: G (ra x rb) = sum_c coeff_c * A_c^T M B_c; A_c = rows 4c..4c+3.
// Block = one chunk of cells x one (TI x TJ) output tile; thread (i, j) of
// the tile accumulates serially over the chunk (deterministic order).
constexpr int kTile = 16;
constexpr int kChunk = 32;   // cells per smem pass (mgram)
constexpr int kChunkP = 8;  // cells per smem pass (project)

__global__ void mgram_kernel(int ncell, int ra, int rb, const double* __restrict__ A, int lda,
                             const double* __restrict__ B, int ldb,
                             const double* __restrict__ coeff, dlrsn_cellops ops, int cells_per_block,
                             double* __restrict__ part) {
  __shared__ double sA[kChunk * 4][kTile + 1];
  __shared__ double sB[kChunk * 4][kTile + 1];
  const int ti = threadIdx.x / kTile, tj = threadIdx.x % kTile;
  const int tiles_j = (rb + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * cells_per_block;
  const int c_end = min(ncell, c_begin + cells_per_block);
  double acc = 0.0;
  for (int c0 = c_begin; c0 < c_end; c0 += kChunk) {
    const int nc = min(kChunk, c_end - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * 4 * kTile; e += blockDim.x) {
      const int row = e / kTile, col = e % kTile;
      const int64_t grow = (int64_t)c0 * 4 + row;
      sA[row][col] = (i0 + col < ra) ? A[grow * lda + i0 + col] : 0.0;
    }
    // B rows pre-multiplied by coeff_c * M
    for (int e = threadIdx.x; e < nc * kTile; e += blockDim.x) {
      const int cl = e / kTile, col = e % kTile;
      const int c = c0 + cl;
      double b[4];
#pragma unroll
      for (int l = 0; l < 4; ++l)
        b[l] = (j0 + col < rb) ? B[((int64_t)c * 4 + l) * ldb + j0 + col] : 0.0;
      const double w = coeff ? coeff[c] : 1.0;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const double mb = ops.mass[4 * l] * b[0] + ops.mass[4 * l + 1] * b[1] +
                          ops.mass[4 * l + 2] * b[2] + ops.mass[4 * l + 3] * b[3];
        sB[cl * 4 + l][col] = coeff ? mb * w : mb;
      }
    }
    __syncthreads();
    for (int row = 0; row < nc * 4; ++row) acc = fma(sA[row][ti], sB[row][tj], acc);
  }
  const int i = i0 + ti, j = j0 + tj;
  if (i < ra && j < rb) part[(int64_t)blockIdx.x * ra * rb + (int64_t)i * rb + j] = acc;
}

// ---------------------------------------------------------------------------
// project: per output tile (i0.., j0..) and chunk of cells, accumulate
//   out[0] px = sum X^T Gx X + vertical faces 1/2 u^T e2x v
//   out[1] py = sum X^T Gy X + horizontal faces 1/2 u^T e2y v
//   out[2] jx = vertical faces 1/2 u^T e2x u
//   out[3] jy = horizontal faces 1/2 u^T e2y u
//   out[4] mt = sum sigma_t X^T M X
//   out[5] ms = sum sigma_s X^T M X
//   out[6] mo = sum Xold^T M X            (project_initial, dlr_sn.py:50-58)
// with u = a - b, v = a + b, a = minus-side edge trace (0 outside the
// domain), b = plus-side trace: this is exactly the reference's interior +
// boundary face assembly (transport_sn.py:230-258) applied to X.
// q-hat (out vector) = sum_c q_c src_row . X_c, written by tile row 0.
struct ProjArgs {
  int nx, ny, r;
  const double* X;
  const double* Xold;
  const double* sigma_t;
  const double* sigma_s;
  const double* q;
  double* part;  // [chunk][7*r*r + r]
  int cells_per_block;
};

__device__ inline void edge_pair(const double* X, int r, int cell, int l0, int l1, int col,
                                 double& v0, double& v1) {
  if (cell < 0) {
    v0 = v1 = 0.0;
    return;
  }
  v0 = __ldg(X + ((int64_t)cell * 4 + l0) * r + col);
  v1 = __ldg(X + ((int64_t)cell * 4 + l1) * r + col);
}

__global__ void project_kernel(ProjArgs pa, dlrsn_cellops ops) {
  // staged per chunk: X_c (4 rows), transformed rows for j
  __shared__ double sX[kChunkP][4][kTile + 1];    // X rows, tile-i columns
  __shared__ double sXo[kChunkP][4][kTile + 1];   // Xold rows, tile-i columns
  __shared__ double sMX[kChunkP][4][kTile + 1];   // M X, tile-j columns
  __shared__ double sGX[kChunkP][4][kTile + 1];   // Gx X
  __shared__ double sGY[kChunkP][4][kTile + 1];   // Gy X
  __shared__ double sUi[kChunkP][4][kTile + 1];   // x-face u (2), y-face u (2), tile-i
  __shared__ double sFj[kChunkP][8][kTile + 1];   // 1/2 e2 v (x,y) and 1/2 e2 u (x,y), tile-j
  __shared__ double sC[kChunkP][3];               // sigma_t, sigma_s, q
  const int r = pa.r, nx = pa.nx;
  const int ncell = pa.nx * pa.ny;
  const int ti = threadIdx.x / kTile, tj = threadIdx.x % kTile;
  const int tiles_j = (r + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  double qacc = 0.0;
  for (int c0 = c_begin; c0 < c_end; c0 += kChunkP) {
    const int nc = min(kChunkP, c_end - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * kTile * 2; e += blockDim.x) {
      const int side = e / (nc * kTile);  // 0: tile-i columns, 1: tile-j columns
      const int rem = e % (nc * kTile);
      const int cl = rem / kTile, col = rem % kTile;
      const int c = c0 + cl;
      const int gcol = (side == 0 ? i0 : j0) + col;
      const bool ok = gcol < r;
      const int ci = c % nx, cj = c / nx;
      double x[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) x[l] = ok ? __ldg(pa.X + ((int64_t)c * 4 + l) * r + gcol) : 0.0;
      // face traces: left face (minus = left neighbour right edge (1,3), plus
      // = this cell's left edge (0,2)); bottom face (minus = lower neighbour
      // top edge (2,3), plus = this cell's bottom edge (0,1))
      double ax0 = 0, ax1 = 0, ay0 = 0, ay1 = 0;
      if (ok) {
        edge_pair(pa.X, r, ci > 0 ? c - 1 : -1, 1, 3, gcol, ax0, ax1);
        edge_pair(pa.X, r, cj > 0 ? c - nx : -1, 2, 3, gcol, ay0, ay1);
      }
      const double ux0 = ax0 - x[0], ux1 = ax1 - x[2], vx0 = ax0 + x[0], vx1 = ax1 + x[2];
      const double uy0 = ay0 - x[0], uy1 = ay1 - x[1], vy0 = ay0 + x[0], vy1 = ay1 + x[1];
      if (side == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sX[cl][l][col] = x[l];
          sXo[cl][l][col] = (ok && pa.Xold) ? __ldg(pa.Xold + ((int64_t)c * 4 + l) * r + gcol) : 0.0;
        }
        sUi[cl][0][col] = ux0; sUi[cl][1][col] = ux1;
        sUi[cl][2][col] = uy0; sUi[cl][3][col] = uy1;
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double m = 0, gx = 0, gy = 0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            m += ops.mass[4 * l + p] * x[p];
            gx += ops.gx[4 * l + p] * x[p];
            gy += ops.gy[4 * l + p] * x[p];
          }
          sMX[cl][l][col] = m;
          sGX[cl][l][col] = gx;
          sGY[cl][l][col] = gy;
        }
        // 1/2 e2 v and 1/2 e2 u for both faces
        sFj[cl][0][col] = 0.5 * (ops.e2x[0] * vx0 + ops.e2x[1] * vx1);
        sFj[cl][1][col] = 0.5 * (ops.e2x[2] * vx0 + ops.e2x[3] * vx1);
        sFj[cl][2][col] = 0.5 * (ops.e2y[0] * vy0 + ops.e2y[1] * vy1);
        sFj[cl][3][col] = 0.5 * (ops.e2y[2] * vy0 + ops.e2y[3] * vy1);
        sFj[cl][4][col] = 0.5 * (ops.e2x[0] * ux0 + ops.e2x[1] * ux1);
        sFj[cl][5][col] = 0.5 * (ops.e2x[2] * ux0 + ops.e2x[3] * ux1);
        sFj[cl][6][col] = 0.5 * (ops.e2y[0] * uy0 + ops.e2y[1] * uy1);
        sFj[cl][7][col] = 0.5 * (ops.e2y[2] * uy0 + ops.e2y[3] * uy1);
      }
    }
    for (int e = threadIdx.x; e < nc; e += blockDim.x) {
      sC[e][0] = pa.sigma_t[c0 + e];
      sC[e][1] = pa.sigma_s[c0 + e];
      sC[e][2] = pa.q[c0 + e];
    }
    __syncthreads();
    for (int cl = 0; cl < nc; ++cl) {
      double xm = 0, gx = 0, gy = 0, om = 0;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const double xi = sX[cl][l][ti];
        xm = fma(xi, sMX[cl][l][tj], xm);
        gx = fma(xi, sGX[cl][l][tj], gx);
        gy = fma(xi, sGY[cl][l][tj], gy);
        om = fma(sXo[cl][l][ti], sMX[cl][l][tj], om);
      }
      const double uxi0 = sUi[cl][0][ti], uxi1 = sUi[cl][1][ti];
      const double uyi0 = sUi[cl][2][ti], uyi1 = sUi[cl][3][ti];
      acc[0] += gx + (uxi0 * sFj[cl][0][tj] + uxi1 * sFj[cl][1][tj]);
      acc[1] += gy + (uyi0 * sFj[cl][2][tj] + uyi1 * sFj[cl][3][tj]);
      acc[2] += uxi0 * sFj[cl][4][tj] + uxi1 * sFj[cl][5][tj];
      acc[3] += uyi0 * sFj[cl][6][tj] + uyi1 * sFj[cl][7][tj];
      acc[4] = fma(sC[cl][0], xm, acc[4]);
      acc[5] = fma(sC[cl][1], xm, acc[5]);
      acc[6] += om;
    }
    // q-hat (dlr_sn.py:70): the (i0 == 0) tiles own columns j0..j0+15
    if (i0 == 0 && ti == 0) {
      for (int cl = 0; cl < nc; ++cl) {
        const int c = c0 + cl;
        const int col = j0 + tj;
        if (col < r) {
          double s = 0;
#pragma unroll
          for (int l = 0; l < 4; ++l) s = fma(ops.src_row[l], __ldg(pa.X + ((int64_t)c * 4 + l) * r + col), s);
          qacc = fma(sC[cl][2], s, qacc);
        }
      }
    }
  }
  // right / top boundary faces of the cells in this block's range
  // (a = this cell's right/top edge trace, b = 0); enumerate only those cells
  {
    const int i = i0 + ti, j = j0 + tj;
    if (i < r && j < r) {
      const int first_right = c_begin + ((nx - 1 - c_begin % nx) % nx + nx) % nx;
      for (int c = first_right; c < c_end; c += nx) {
        double ai0, ai1, aj0, aj1;
        edge_pair(pa.X, r, c, 1, 3, i, ai0, ai1);
        edge_pair(pa.X, r, c, 1, 3, j, aj0, aj1);
        const double f0 = 0.5 * (ops.e2x[0] * aj0 + ops.e2x[1] * aj1);
        const double f1 = 0.5 * (ops.e2x[2] * aj0 + ops.e2x[3] * aj1);
        const double val = ai0 * f0 + ai1 * f1;
        acc[0] += val;
        acc[2] += val;
      }
      for (int c = max(c_begin, (pa.ny - 1) * nx); c < c_end; ++c) {
        double ai0, ai1, aj0, aj1;
        edge_pair(pa.X, r, c, 2, 3, i, ai0, ai1);
        edge_pair(pa.X, r, c, 2, 3, j, aj0, aj1);
        const double f0 = 0.5 * (ops.e2y[0] * aj0 + ops.e2y[1] * aj1);
        const double f1 = 0.5 * (ops.e2y[2] * aj0 + ops.e2y[3] * aj1);
        const double val = ai0 * f0 + ai1 * f1;
        acc[1] += val;
        acc[3] += val;
      }
    }
  }
  const int i = i0 + ti, j = j0 + tj;
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)blockIdx.x * stride;
  if (i < r && j < r) {
#pragma unroll
    for (int o = 0; o < 7; ++o) out[(int64_t)o * r * r + (int64_t)i * r + j] = acc[o];
  }
  if (i0 == 0 && ti == 0 && j < r) out[7 * (int64_t)r * r + j] = qacc;
}

// ---------------------------------------------------------------------------
// Small dense kernels: one CTA, matrices in global memory (L2 resident).

// Cholesky G = R^T R (R upper) and Rinv = R^-1 (upper).  flag[0] = 1 if a
// pivot is not positive; diag_ratio[k] = R_kk / max(sqrt(G_kk), 1) (the
// reference's deficiency test quantity, angular.py:137).
__global__ void chol_upper_kernel(int r, const double* __restrict__ G, double* __restrict__ R,
                                  double* __restrict__ Rinv, double* __restrict__ diag_ratio,
                                  int* flag) {
  extern __shared__ double sm[];
  double* a = sm;          // r*r working copy (becomes R)
  double* inv = sm + r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    a[e] = G[e];
    inv[e] = 0.0;
  }
  __syncthreads();
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      const double d = a[k * r + k];
      const double g = G[k * r + k];
      if (!(d > 0.0)) {
        bad = 1;
        a[k * r + k] = 0.0;
        diag_ratio[k] = 0.0;
        diag_ratio[r + k] = 0.0;
      } else {
        a[k * r + k] = sqrt(d);
        const double on = sqrt(fmax(g, 0.0));
        diag_ratio[k] = on > 0.0 ? a[k * r + k] / on : 0.0;
        diag_ratio[r + k] = a[k * r + k] / fmax(on, 1.0);
      }
    }
    __syncthreads();
    const double rkk = a[k * r + k];
    for (int j = k + 1 + threadIdx.x; j < r; j += blockDim.x) a[k * r + j] = rkk > 0 ? a[k * r + j] / rkk : 0.0;
    __syncthreads();
    // trailing update a[i][j] -= a[k][i] a[k][j], i,j > k (upper part only)
    const int m = r - k - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = k + 1 + e / m, j = k + 1 + e % m;
      if (j >= i) a[i * r + j] -= a[k * r + i] * a[k * r + j];
    }
    __syncthreads();
  }
  // R: zero the strict lower part
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    R[e] = j >= i ? a[e] : 0.0;
  }
  __syncthreads();
  // Rinv by columns: solve R x = e_j (back substitution), one thread/column
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    for (int i = j; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int p = i + 1; p <= j; ++p) s -= a[i * r + p] * inv[p * r + j];
      const double d = a[i * r + i];
      inv[i * r + j] = d > 0 ? s / d : 0.0;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Rinv[e] = inv[e];
  if (threadIdx.x == 0 && flag) *flag = bad;
}

// C = A B for small square r x r (one CTA); used for R = R2 R1 etc.
__global__ void small_matmul_kernel(int m, int k, int n, const double* __restrict__ A,
                                    const double* __restrict__ B, double* __restrict__ C,
                                    int transA) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    double s = 0.0;
    for (int p = 0; p < k; ++p) s = fma(transA ? A[p * m + i] : A[i * k + p], B[p * n + j], s);
    C[e] = s;
  }
}

// Batched inverse by Gauss-Jordan with partial pivoting, one CTA per matrix
// (solve_row_system: np.linalg.inv, lowrank.py:245-252).  B_d is built
// in place from the projections: B_d = wx px + wy py + |wx| jx + |wy| jy + mt
// (row_matrices, dlr_sn.py:74-83).  status[d] = 1 if singular/non-finite.
__global__ void row_inverse_kernel(int r, const double* __restrict__ proj,
                                   const double* __restrict__ om_sel, double* __restrict__ Binv,
                                   double* __restrict__ Bout, int* status) {
  // om_sel == nullptr: proj holds the node matrices B_d directly (n x r x r)
  extern __shared__ double sm[];
  const int d = blockIdx.x;
  const int w = 2 * r;
  double* a = sm;  // r x 2r augmented [B | I]
  __shared__ int piv;
  __shared__ int sing;
  const double wx = om_sel ? om_sel[3 * d] : 0.0, wy = om_sel ? om_sel[3 * d + 1] : 0.0;
  const int64_t rr = (int64_t)r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const double b = om_sel ? wx * proj[e] + wy * proj[rr + e] + fabs(wx) * proj[2 * rr + e] +
                                  fabs(wy) * proj[3 * rr + e] + proj[4 * rr + e]
                            : proj[d * rr + e];
    const int i = e / r, j = e % r;
    a[i * w + j] = b;
    a[i * w + r + j] = (i == j) ? 1.0 : 0.0;
    if (Bout) Bout[(int64_t)d * rr + e] = b;
  }
  if (threadIdx.x == 0) sing = 0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double best = fabs(a[k * w + k]);
      for (int i = k + 1; i < r; ++i) {
        const double v = fabs(a[i * w + k]);
        if (v > best) { best = v; p = i; }
      }
      piv = p;
      if (!(best > 0.0) || !isfinite(best)) sing = 1;
    }
    __syncthreads();
    if (sing) break;
    const int p = piv;
    if (p != k)
      for (int j = threadIdx.x; j < w; j += blockDim.x) {
        const double t = a[k * w + j];
        a[k * w + j] = a[p * w + j];
        a[p * w + j] = t;
      }
    __syncthreads();
    const double inv = 1.0 / a[k * w + k];
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += blockDim.x) a[k * w + j] *= inv;
    __syncthreads();
    for (int e = threadIdx.x; e < r * w; e += blockDim.x) {
      const int i = e / w, j = e % w;
      if (i != k) {
        const double f = a[i * w + k];
        if (j != k) a[i * w + j] -= f * a[k * w + j];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += blockDim.x)
      if (i != k) a[i * w + k] = 0.0;
    __syncthreads();
  }
  if (sing) {
    if (threadIdx.x == 0) status[d] = 1;
    return;
  }
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const double v = a[(e / r) * w + r + e % r];
    if (!isfinite(v)) status[d] = 1;
    Binv[(int64_t)d * rr + e] = v;
  }
}

// LU with partial pivoting of an n x n matrix in shared memory (one CTA)
// and solve with nrhs right-hand sides stored column-major after it.
__device__ void cta_lu_solve(int n, double* a, int lda, double* b, int ldb, int nrhs, int* perm,
                             int* sing) {
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int p = k;
      double best = fabs(a[k * lda + k]);
      for (int i = k + 1; i < n; ++i) {
        const double v = fabs(a[i * lda + k]);
        if (v > best) { best = v; p = i; }
      }
      perm[k] = p;
      if (!(best > 0.0)) *sing = 1;
    }
    __syncthreads();
    const int p = perm[k];
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double t = a[k * lda + j]; a[k * lda + j] = a[p * lda + j]; a[p * lda + j] = t;
      }
      for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {
        const double t = b[k * ldb + j]; b[k * ldb + j] = b[p * ldb + j]; b[p * ldb + j] = t;
      }
    }
    __syncthreads();
    const double piv = a[k * lda + k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) a[i * lda + k] = piv != 0.0 ? a[i * lda + k] / piv : 0.0;
    __syncthreads();
    const int m = n - k - 1;
    for (int e = threadIdx.x; e < m * (m + nrhs); e += blockDim.x) {
      const int i = k + 1 + e / (m + nrhs), jj = e % (m + nrhs);
      const double l = a[i * lda + k];
      if (jj < m) a[i * lda + k + 1 + jj] -= l * a[k * lda + k + 1 + jj];
      else b[i * ldb + (jj - m)] -= l * b[k * ldb + (jj - m)];
    }
  }
  __syncthreads();
  // back substitution, one thread per rhs
  for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {
    for (int i = n - 1; i >= 0; --i) {
      double s = b[i * ldb + j];
      for (int p = i + 1; p < n; ++p) s -= a[i * lda + p] * b[p * ldb + j];
      b[i * ldb + j] = a[i * lda + i] != 0.0 ? s / a[i * lda + i] : 0.0;
    }
  }
  __syncthreads();
}

// Row system combine (lowrank.py:253-259):
//   cbar = sum_d w_d Binv_d ; zeta = sum_d w_d Binv_d Q_d
//   lbar = solve(I - cbar ms / 4pi, zeta); L_d = Binv_d (Q_d + ms lbar / 4pi)
__global__ void row_combine_kernel(int n, int r, const double* __restrict__ Binv,
                                   const double* __restrict__ ms, const double* __restrict__ Q,
                                   const double* __restrict__ wts, double* __restrict__ L,
                                   double* __restrict__ lbar, int* status) {
  extern __shared__ double sm[];
  double* cbar = sm;              // r*r
  double* lhs = cbar + r * r;     // r*r
  double* zeta = lhs + r * r;     // r
  double* msl = zeta + r;         // r
  int* perm = reinterpret_cast<int*>(msl + r);
  __shared__ int sing;
  const int64_t rr = (int64_t)r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += wts[d] * Binv[d * rr + e];
    cbar[e] = s;
  }
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < n; ++d) {
      double bq = 0.0;
      for (int j = 0; j < r; ++j) bq += Binv[d * rr + i * r + j] * Q[d * r + j];
      s += wts[d] * bq;
    }
    zeta[i] = s;
  }
  if (threadIdx.x == 0) sing = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double s = 0.0;
    for (int p = 0; p < r; ++p) s += cbar[i * r + p] * ms[p * r + j];
    lhs[e] = (i == j ? 1.0 : 0.0) - s / kFourPi;
  }
  __syncthreads();
  cta_lu_solve(r, lhs, r, zeta, 1, 1, perm, &sing);
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    lbar[i] = zeta[i];
    double s = 0.0;
    for (int p = 0; p < r; ++p) s += ms[i * r + p] * zeta[p];
    msl[i] = s / kFourPi;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) {
    const int d = e / r, i = e % r;
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += Binv[d * rr + i * r + j] * (Q[d * r + j] + msl[j]);
    L[e] = s;
  }
  if (threadIdx.x == 0 && sing) *status = 1;
}

// DEIM (lowrank.py:168-205) as Gaussian elimination with row pivoting on a
// working copy of W (n x r): column j's Schur-complement column is exactly
// the interpolation residual W[:,j] - W[:,:j] W[p,:j]^-1 W[p,j]; the pivot is
// its first maximal |entry| (np.argmax).  Produces the picks, the unit lower
// factor rows L[p,:] and U (so W[p,:] = Lhat U), all in pick order.
__global__ void deim_kernel(int n, int r, double* __restrict__ Wk_global /* n x r work copy */,
                            const double* __restrict__ W, int* __restrict__ idx,
                            double* __restrict__ Lhat, double* __restrict__ U, int* err_col,
                            int in_smem) {
  extern __shared__ double dsm[];
  double* Wk = in_smem ? dsm : Wk_global;  // work copy resident in smem when it fits
  __shared__ double bv[33];
  __shared__ int bi[32];
  __shared__ int pick;
  __shared__ double pval;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = -1;
  // working copy and floor = 1e-14 * max(1, max|W|) (lowrank.py:185)
  double mx = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)n * r; e += blockDim.x) {
    const double v = W[e];
    Wk[(e % r) * n + e / r] = v;  // column-major work copy (coalesced column access)
    mx = fmax(mx, fabs(v));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0) bv[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) m = fmax(m, bv[q]);
    bv[32] = 1e-14 * fmax(1.0, m);
  }
  __syncthreads();
  const double floor_ = bv[32];
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    // argmax |Wk[:, j]|, lowest index on ties
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double v = fabs(Wk[(int64_t)j * n + i]);
      if (v > best || (v == best && i < bidx)) { best = v; bidx = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(kFull, best, o);
      const int oi = __shfl_down_sync(kFull, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { bv[w] = best; bi[w] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int ii = 0x7fffffff;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
        if (bv[q] > b || (bv[q] == b && bi[q] < ii)) { b = bv[q]; ii = bi[q]; }
      pick = ii;
      pval = Wk[(int64_t)j * n + ii];
      if (!(fabs(pval) > floor_)) fail = j;
      for (int q = 0; q < j; ++q)
        if (idx[q] == ii) fail = j;
      idx[j] = ii;
    }
    __syncthreads();
    if (fail >= 0) break;
    const int p = pick;
    const double pv = pval;
    // U row j = pivot row of the current (updated) matrix, columns j..r-1
    for (int k = threadIdx.x; k < r; k += blockDim.x) U[j * r + k] = k >= j ? Wk[(int64_t)k * n + p] : 0.0;
    __syncthreads();
    // l = col / pivot; trailing update W[:, k] -= l * W[p, k] for k > j
    for (int64_t e = threadIdx.x; e < (int64_t)n; e += blockDim.x) {
      const double l = Wk[(int64_t)j * n + e] / pv;
      Wk[(int64_t)j * n + e] = l;  // keep the multiplier column
      for (int k = j + 1; k < r; ++k) Wk[(int64_t)k * n + e] -= l * U[j * r + k];
    }
    __syncthreads();
  }
  if (fail >= 0) {
    if (threadIdx.x == 0) *err_col = fail;
    return;
  }
  // Lhat[q, j] = multiplier of column j at the q-th picked row (unit lower)
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int q = e / r, j = e % r;
    Lhat[e] = j < q ? Wk[(int64_t)j * n + idx[q]] : (j == q ? 1.0 : 0.0);
  }
  if (threadIdx.x == 0) *err_col = -1;
}

// Solves with W_hat = Lhat U (pick order):
//   mode 0 (interpolation_coefficients): X = W_hat^-1 V   (V r x m)
//   mode 1 (closure_weights):            x = W_hat^-T v   (v r)
__global__ void what_solve_kernel(int r, int m, const double* __restrict__ Lhat,
                                  const double* __restrict__ U, const double* __restrict__ V,
                                  double* __restrict__ X, int mode) {
  extern __shared__ double sw[];
  double* sL = sw;               // r x r
  double* sU = sL + r * r;       // r x r
  double* sX = sU + r * r;       // r x m
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    sL[e] = Lhat[e];
    sU[e] = U[e];
  }
  for (int e = threadIdx.x; e < r * m; e += blockDim.x) sX[e] = V[e];
  __syncthreads();
  // one warp per right-hand side: the row recurrences are sequential, the
  // inner products over the solved entries are split across the lanes
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < m; c += nw) {
    if (mode == 0) {
      for (int i = 0; i < r; ++i) {  // L y = v
        double s = 0.0;
        for (int p = lane; p < i; p += 32) s += sL[i * r + p] * sX[p * m + c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
        if (lane == 0) sX[i * m + c] -= s;
        __syncwarp();
      }
      for (int i = r - 1; i >= 0; --i) {  // U x = y
        double s = 0.0;
        for (int p = i + 1 + lane; p < r; p += 32) s += sU[i * r + p] * sX[p * m + c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
        if (lane == 0) sX[i * m + c] = (sX[i * m + c] - s) / sU[i * r + i];
        __syncwarp();
      }
    } else {
      for (int i = 0; i < r; ++i) {  // U^T y = v
        double s = 0.0;
        for (int p = lane; p < i; p += 32) s += sU[p * r + i] * sX[p * m + c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
        if (lane == 0) sX[i * m + c] = (sX[i * m + c] - s) / sU[i * r + i];
        __syncwarp();
      }
      for (int i = r - 1; i >= 0; --i) {  // L^T x = y
        double s = 0.0;
        for (int p = i + 1 + lane; p < r; p += 32) s += sL[p * r + i] * sX[p * m + c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(kFull, s, o);
        if (lane == 0) sX[i * m + c] -= s;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * m; e += blockDim.x) X[e] = sX[e];
}

}  // namespace dlrsn

using namespace dlrsn;

static int grid_for(int64_t n, int block = kRB) {
  int64_t b = (n + block - 1) / block;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}

extern "C" {

int dlrsn_rowmix(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
                 double beta, double* Y, int ldy, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(kx >= 0 && ky >= 0 && kx * ky <= 48 * 1024 / 8 * 4, "rowmix operand too large");
  if (n == 0 || ky == 0) return DLRSN_OK;
  const size_t smem = (size_t)kx * ky * sizeof(double);
  if (smem > 48 * 1024)
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rowmix_kernel<<<grid_for(n * ky), kRB, smem, as_stream(stream)>>>((int)n, kx, ky, X, ldx, K, ldk,
                                                                   beta, Y, ldy);
  DLRSN_CHECK_LAUNCH("rowmix_kernel");
  return DLRSN_OK;
}

// cells per block of the cell-reduction kernels: about 4 CTAs per SM in
// total over all output tiles, in whole smem chunks
static int cells_per_block(int ncell, int tiles) {
  const int target = (4 * 148 + tiles - 1) / tiles;
  int cpb = (ncell + target - 1) / target;
  cpb = (cpb + kChunk - 1) / kChunk * kChunk;
  return cpb < kChunk ? kChunk : cpb;
}

int64_t dlrsn_partials_len(int ncell, int ra, int rb, int kind) {
  // partial buffer (doubles) for mgram (kind 0) / project (kind 1)
  const int tiles = ((ra + kTile - 1) / kTile) * ((rb + kTile - 1) / kTile);
  const int cpb = cells_per_block(ncell, tiles);
  const int64_t nblk = (ncell + cpb - 1) / cpb;
  return kind == 0 ? nblk * ra * rb : nblk * (7 * (int64_t)ra * ra + ra);
}

int dlrsn_mgram(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda,
                const double* B, int ldb, const double* coeff, double* G, double* partial,
                dlrsn_stream_t stream) {
  const int ncell = ops->nx * ops->ny;
  const int tiles = ((ra + kTile - 1) / kTile) * ((rb + kTile - 1) / kTile);
  const int cpb = cells_per_block(ncell, tiles);
  const int nblk = (ncell + cpb - 1) / cpb;
  cudaStream_t st = as_stream(stream);
  mgram_kernel<<<dim3(nblk, tiles), kTile * kTile, 0, st>>>(ncell, ra, rb, A, lda, B, ldb, coeff,
                                                            *ops, cpb, partial);
  DLRSN_CHECK_LAUNCH("mgram_kernel");
  const int64_t len = (int64_t)ra * rb;
  reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 256, 0, st>>>(nblk, len, partial, G, 1.0);
  DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
  return DLRSN_OK;
}

int dlrsn_project(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
                  const double* sigma_t, const double* sigma_s, const double* q, double* out,
                  double* partial, dlrsn_stream_t stream) {
  const int ncell = ops->nx * ops->ny;
  const int tiles = ((r + kTile - 1) / kTile) * ((r + kTile - 1) / kTile);
  const int cpb = cells_per_block(ncell, tiles);
  const int nblk = (ncell + cpb - 1) / cpb;
  ProjArgs pa;
  pa.nx = ops->nx; pa.ny = ops->ny; pa.r = r;
  pa.X = X; pa.Xold = Xold; pa.sigma_t = sigma_t; pa.sigma_s = sigma_s; pa.q = q;
  pa.part = partial; pa.cells_per_block = cpb;
  cudaStream_t st = as_stream(stream);
  // partial slots not written by some tiles must be zero
  DLRSN_TRY_CUDA(cudaMemsetAsync(partial, 0, sizeof(double) * (size_t)nblk * (7 * (size_t)r * r + r), st));
  project_kernel<<<dim3(nblk, tiles), kTile * kTile, 0, st>>>(pa, *ops);
  DLRSN_CHECK_LAUNCH("project_kernel");
  const int64_t len = 7 * (int64_t)r * r + r;
  reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 256, 0, st>>>(nblk, len, partial, out, 1.0);
  DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
  return DLRSN_OK;
}

int dlrsn_chol_upper(int r, const double* G, double* R, double* Rinv, double* diag_ratio,
                     int* flag, dlrsn_stream_t stream) {
  const size_t smem = 2 * (size_t)r * r * sizeof(double);
  DLRSN_REQUIRE(smem <= 200 * 1024, "rank %d too large for chol_upper", r);
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(chol_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_upper_kernel<<<1, 256, smem, as_stream(stream)>>>(r, G, R, Rinv, diag_ratio, flag);
  DLRSN_CHECK_LAUNCH("chol_upper_kernel");
  return DLRSN_OK;
}

int dlrsn_small_matmul(int m, int k, int n, const double* A, const double* B, double* C,
                       int transA, dlrsn_stream_t stream) {
  small_matmul_kernel<<<1, 256, 0, as_stream(stream)>>>(m, k, n, A, B, C, transA);
  DLRSN_CHECK_LAUNCH("small_matmul_kernel");
  return DLRSN_OK;
}

int dlrsn_row_inverse(int n, int r, const double* proj, const double* om_sel, double* Binv,
                      double* Bout, int* status, dlrsn_stream_t stream) {
  const size_t smem = 2 * (size_t)r * r * sizeof(double);
  DLRSN_REQUIRE(smem <= 200 * 1024, "rank %d too large for row_inverse", r);
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (n == 0) return DLRSN_OK;
  row_inverse_kernel<<<n, 256, smem, as_stream(stream)>>>(r, proj, om_sel, Binv, Bout, status);
  DLRSN_CHECK_LAUNCH("row_inverse_kernel");
  return DLRSN_OK;
}

int dlrsn_row_combine(int n, int r, const double* Binv, const double* ms, const double* Q,
                      const double* wts, double* L, double* lbar, int* status,
                      dlrsn_stream_t stream) {
  const size_t smem = (2 * (size_t)r * r + 2 * r) * sizeof(double) + r * sizeof(int);
  DLRSN_REQUIRE(smem <= 200 * 1024, "rank %d too large for row_combine", r);
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  row_combine_kernel<<<1, 256, smem, as_stream(stream)>>>(n, r, Binv, ms, Q, wts, L, lbar, status);
  DLRSN_CHECK_LAUNCH("row_combine_kernel");
  return DLRSN_OK;
}

int dlrsn_deim(int n, int r, double* Wwork, const double* W, int* idx, double* Lhat, double* U,
               int* err_col, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(r <= n, "rank %d exceeds the %d available nodes", r, n);
  const size_t smem = (size_t)n * r * sizeof(double);
  const int in_smem = smem <= 200 * 1024;
  if (in_smem)
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(deim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  deim_kernel<<<1, 1024, in_smem ? smem : 0, as_stream(stream)>>>(n, r, Wwork, W, idx, Lhat, U,
                                                                  err_col, in_smem);
  DLRSN_CHECK_LAUNCH("deim_kernel");
  return DLRSN_OK;
}

int dlrsn_what_solve(int r, int m, const double* Lhat, const double* U, const double* V,
                     double* X, int mode, dlrsn_stream_t stream) {
  const size_t smem = (2 * (size_t)r * r + (size_t)r * m) * sizeof(double);
  DLRSN_REQUIRE(smem <= 200 * 1024, "W_hat solve too large for shared memory");
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(what_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  what_solve_kernel<<<1, 512, smem, as_stream(stream)>>>(r, m, Lhat, U, V, X, mode);
  DLRSN_CHECK_LAUNCH("what_solve_kernel");
  return DLRSN_OK;
}

}  // extern "C"
