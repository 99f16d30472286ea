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
#include <vector>
#include <utility>
#include <cstring>

#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"

namespace dlrsn {

namespace cg = cooperative_groups;

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

// Fixed-width variant: thread (i, j) keeps column j of K in registers and
// reads row i of X with 16-byte loads (shared by the ky threads of the row).
template <int KX>
__global__ void __launch_bounds__(256) rowmix_reg_kernel(int n, int ky, const double* __restrict__ X,
                                                        int ldx, const double* __restrict__ K,
                                                        int ldk, double beta,
                                                        double* __restrict__ Y, int ldy) {
  const int64_t total = (int64_t)n * ky;
  // blockDim % ky == 0 (checked by the launcher): column j is fixed per thread
  const int j = threadIdx.x % ky;
  double k[KX];
#pragma unroll
  for (int p = 0; p < KX; ++p) k[p] = __ldg(K + p * ldk + j);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / ky;
    const double2* x = reinterpret_cast<const double2*>(X + i * ldx);
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int p = 0; p < KX / 2; ++p) {
      const double2 v = __ldg(x + p);
      acc0 = fma(v.x, k[2 * p], acc0);
      acc1 = fma(v.y, k[2 * p + 1], acc1);
    }
    const double acc = acc0 + acc1;
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
  // block = 32 consecutive outputs x nw warps; warp w sums chunks w, w+nw, ...
  // (coalesced, two independent chains), then the warp sums are added in
  // warp order (deterministic for a given launch shape)
  __shared__ double red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s0 = 0.0, s1 = 0.0;
  if (e < len) {
    int c = w;
    for (; c + nw < nchunks; c += 2 * nw) {
      s0 += __ldg(part + (int64_t)c * len + e);
      s1 += __ldg(part + (int64_t)(c + nw) * len + e);
    }
    if (c < nchunks) s0 += __ldg(part + (int64_t)c * len + e);
  }
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && e < len) {
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += red[q][lane];
    out[e] = alpha * t;
  }
}

// FP64 tensor-core MMA (DMMA), D(8x8) += A(8x4) B(4x8); fragments per lane
// (g = lane / 4, q = lane % 4): A[g][q], B[q][g], D[g][2q], D[g][2q+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// rowmix on the FP64 tensor cores: each warp multiplies 8-row tiles of X by
// K (KS k-steps of 4, NT n-tiles of 8), K's fragments held in registers for
// the whole launch and X's fragments loaded straight from global memory.
template <int KS, int NT>
__global__ void __launch_bounds__(256) rowmix_mma_kernel(int n, int kx, int ky,
                                                         const double* __restrict__ X, int ldx,
                                                         const double* __restrict__ K, int ldk,
                                                         double beta, double* __restrict__ Y,
                                                         int ldy) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  double bf[KS][NT];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int k = 4 * ks + q, c = 8 * nt + g;
      bf[ks][nt] = (k < kx && c < ky) ? __ldg(K + (int64_t)k * ldk + c) : 0.0;
    }
  // U tiles per warp and iteration: their loads are in flight together and
  // their MMA chains interleave (one tile at a time is latency-bound)
  constexpr int U = 4;
  const int64_t tiles = ((int64_t)n + 7) / 8;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t0 < tiles;
       t0 += U * nwarps) {
    double af[U][KS];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = (t0 + u * nwarps) * 8 + g;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c = 4 * ks + q;
        af[u][ks] = (row < n && c < kx) ? __ldg(X + row * ldx + c) : 0.0;
      }
    }
    double d[U][NT][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) d[u][nt][0] = d[u][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(d[u][nt][0], d[u][nt][1], af[u][ks], bf[ks][nt]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = (t0 + u * nwarps) * 8 + g;
      if (row < n) {
        double* y = Y + row * ldy;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = 8 * nt + 2 * q;
          if (beta == 0.0 && c + 1 < ky && ((ldy & 1) == 0) &&
              ((reinterpret_cast<uintptr_t>(Y) & 15) == 0)) {
            *reinterpret_cast<double2*>(y + c) = make_double2(d[u][nt][0], d[u][nt][1]);
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (c + i < ky) y[c + i] = beta == 0.0 ? d[u][nt][i] : fma(beta, y[c + i], d[u][nt][i]);
          }
        }
      }
    }
  }
}

// rowmix for wide operands (kx <= 4 KS <= 128, any ky): the MMA k index is
// permuted so that lane quad q owns the contiguous X columns q KS .. q KS +
// KS - 1 (16-byte loads); K sits in shared memory in fragment order (row
// 4 ks + q holds K row q KS + ks; row stride = 4 mod 16 doubles, so a
// fragment load is conflict-free).  Each warp takes pairs of 8-row tiles, so
// every K fragment feeds two DMMAs; column groups of 8 NT.
template <int KS, int NT>
__global__ void __launch_bounds__(256, (4 * KS + 8 * NT <= 96) ? 2 : 1) rowmix_wide_kernel(int n, int kx, int ky,
                                                          const double* __restrict__ X, int ldx,
                                                          const double* __restrict__ K, int ldk,
                                                          double beta, double* __restrict__ Y,
                                                          int ldy, int kyp, int ldks, int vec,
                                                          const double* __restrict__ V,
                                                          double* __restrict__ YV) {
  extern __shared__ double sK[];  // (4 KS) x ldks
  __shared__ double sV[4 * KS];   // optional extra column: YV = X V in the same pass over X
  for (int e = threadIdx.x; e < 4 * KS * kyp; e += blockDim.x) {
    const int pr = e / kyp, col = e - pr * kyp;
    const int k = (pr & 3) * KS + (pr >> 2);
    sK[pr * ldks + col] = (k < kx && col < ky) ? __ldg(K + (int64_t)k * ldk + col) : 0.0;
  }
  if (V)
    for (int e = threadIdx.x; e < 4 * KS; e += blockDim.x) sV[e] = e < kx ? __ldg(V + e) : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int64_t tiles = ((int64_t)n + 7) / 8;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vstore = beta == 0.0 && ((ldy & 1) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2; t0 < tiles;
       t0 += 2 * nwarps) {
    double af[2][KS];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t row = (t0 + u) * 8 + g;
      const double* xr = X + row * ldx + q * KS;
      if (row < n && vec) {
#pragma unroll
        for (int ks = 0; ks < KS; ks += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(xr + ks));
          af[u][ks] = v.x;
          af[u][ks + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
          af[u][ks] = (row < n && q * KS + ks < kx) ? __ldg(xr + ks) : 0.0;
      }
    }
    if (V) {  // lane quad q holds columns q KS .. q KS + KS - 1 of its rows
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double acc = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) acc = fma(af[u][ks], sV[q * KS + ks], acc);
        acc += __shfl_xor_sync(kFull, acc, 1);
        acc += __shfl_xor_sync(kFull, acc, 2);
        const int64_t row = (t0 + u) * 8 + g;
        if (q == 0 && row < n) YV[row] = acc;
      }
    }
    for (int c0 = 0; c0 < ky; c0 += 8 * NT) {
      double d[2][NT][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) d[u][nt][0] = d[u][nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double* kr = sK + (4 * ks + q) * ldks + c0 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = kr[8 * nt];
          dmma(d[0][nt][0], d[0][nt][1], af[0][ks], b);
          dmma(d[1][nt][0], d[1][nt][1], af[1][ks], b);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t row = (t0 + u) * 8 + g;
        if (row >= n) continue;
        double* y = Y + row * ldy;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = c0 + 8 * nt + 2 * q;
          if (vstore && c + 1 < ky) {
            *reinterpret_cast<double2*>(y + c) = make_double2(d[u][nt][0], d[u][nt][1]);
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (c + i < ky) y[c + i] = beta == 0.0 ? d[u][nt][i] : fma(beta, y[c + i], d[u][nt][i]);
          }
        }
      }
    }
  }
}

// Software-pipelined rowmix_wide: one 8-row tile per iteration, the next
// tile's rows loaded before this tile's MMAs (see rowmix_upper_pipe_kernel).
template <int KS, int NT>
__global__ void __launch_bounds__(384, 1) rowmix_wide_pipe_kernel(int n, int kx, int ky,
                                                               const double* __restrict__ X, int ldx,
                                                               const double* __restrict__ K, int ldk,
                                                               double beta, double* __restrict__ Y,
                                                               int ldy, int kyp, int ldks, int vec,
                                                               const double* __restrict__ V,
                                                               double* __restrict__ YV) {
  extern __shared__ double sK[];  // (4 KS) x ldks
  __shared__ double sV[4 * KS];
  for (int e = threadIdx.x; e < 4 * KS * kyp; e += blockDim.x) {
    const int pr = e / kyp, col = e - pr * kyp;
    const int k = (pr & 3) * KS + (pr >> 2);
    sK[pr * ldks + col] = (k < kx && col < ky) ? __ldg(K + (int64_t)k * ldk + col) : 0.0;
  }
  if (V)
    for (int e = threadIdx.x; e < 4 * KS; e += blockDim.x) sV[e] = e < kx ? __ldg(V + e) : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int64_t tiles = ((int64_t)n + 7) / 8;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vstore = beta == 0.0 && ((ldy & 1) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  auto load = [&](int64_t t, double (&af)[KS]) {
    const int64_t row = t * 8 + g;
    const bool live = t < tiles && row < n;
    const double* xr = X + row * ldx + q * KS;
    if (live && vec) {
#pragma unroll
      for (int ks = 0; ks < KS; ks += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xr + ks));
        af[ks] = v.x;
        af[ks + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) af[ks] = (live && q * KS + ks < kx) ? __ldg(xr + ks) : 0.0;
    }
  };
  int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double cur[KS], nxt[KS];
  load(t0, cur);
  for (; t0 < tiles; t0 += nwarps) {
    load(t0 + nwarps, nxt);
    const int64_t row = t0 * 8 + g;
    if (V) {
      double acc = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) acc = fma(cur[ks], sV[q * KS + ks], acc);
      acc += __shfl_xor_sync(kFull, acc, 1);
      acc += __shfl_xor_sync(kFull, acc, 2);
      if (q == 0 && row < n) YV[row] = acc;
    }
    for (int c0 = 0; c0 < ky; c0 += 8 * NT) {
      double d[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double* kr = sK + (4 * ks + q) * ldks + c0 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(d[nt][0], d[nt][1], cur[ks], kr[8 * nt]);
      }
      if (row < n) {
        double* y = Y + row * ldy;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = c0 + 8 * nt + 2 * q;
          if (vstore && c + 1 < ky) {
            *reinterpret_cast<double2*>(y + c) = make_double2(d[nt][0], d[nt][1]);
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (c + i < ky) y[c + i] = beta == 0.0 ? d[nt][i] : fma(beta, y[c + i], d[nt][i]);
          }
        }
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) cur[ks] = nxt[ks];
  }
}

// rowmix by an upper-triangular K (r x r, exact zeros below the diagonal:
// the CholQR2 factors R^-1): Y = X K with the MMA k index grouped by
// 8-column blocks (see the kernel), so k step ks meets column group
// (c0 + 8 nt ..) only when 8 (ks / 2) <= c0 + 8 nt + 7 -- 72 of 128 DMMA
// fragments at r = 64, 272 of 512 at r = 128 (two 64-column passes).  Every
// row of a warp's tile is loaded (all r columns) before any output of the
// tile is written, so Y may alias X (in place).
template <int KS, int NT>
__global__ void __launch_bounds__(256, 1) rowmix_upper_kernel(int n, int r,
                                                           const double* X, int ldx,
                                                           const double* __restrict__ K, int ldk,
                                                           double* Y, int ldy, int ldks) {
  constexpr int KC = 4 * KS;    // K rows (padded r)
  constexpr int CW = 8 * NT;    // columns per pass
  constexpr int NP = KC / CW;   // passes (1 at r <= 64, 2 at r <= 128)
  // k-step ks, lane quad q <-> column 8 (ks / 2) + 2 q + (ks & 1): the two
  // k-steps of an 8-column block read adjacent columns per lane (one 16-byte
  // load for both), and a k-step still lies inside one 8-column block, so the
  // triangle's zero blocks are skipped as before.  sK row 4 ks + q holds that
  // K row (fragment loads as in rowmix_wide).
  extern __shared__ double sK[];  // KC x ldks
  for (int e = threadIdx.x; e < KC * KC; e += blockDim.x) {
    const int pr = e / KC, col = e - pr * KC;
    const int ks = pr >> 2, qq = pr & 3;
    const int k = 8 * (ks >> 1) + 2 * qq + (ks & 1);
    sK[pr * ldks + col] = (k < r && col < r) ? __ldg(K + (int64_t)k * ldk + col) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int64_t tiles = ((int64_t)n + 7) / 8;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vstore = ((ldy & 1) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  const bool vload = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && r == KC;
  for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2; t0 < tiles;
       t0 += 2 * nwarps) {
    double af[2][KS];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t row = (t0 + u) * 8 + g;
      const double* xr = X + row * ldx + 2 * q;
      if (vload && row < n) {
#pragma unroll
        for (int m = 0; m < KS / 2; ++m) {
          const double2 v = *reinterpret_cast<const double2*>(xr + 8 * m);
          af[u][2 * m] = v.x;
          af[u][2 * m + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int c = 8 * (ks >> 1) + 2 * q + (ks & 1);
          af[u][ks] = (row < n && c < r) ? X[row * ldx + c] : 0.0;
        }
      }
    }
    __syncwarp();  // every lane's reads of the tile precede the in-place writes
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int c0 = p * CW;
      double d[2][NT][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) d[u][nt][0] = d[u][nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double* kr = sK + (4 * ks + q) * ldks + c0 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (8 * (ks >> 1) > c0 + 8 * nt + 7) continue;  // these K rows lie below the columns
          const double b = kr[8 * nt];
          dmma(d[0][nt][0], d[0][nt][1], af[0][ks], b);
          dmma(d[1][nt][0], d[1][nt][1], af[1][ks], b);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t row = (t0 + u) * 8 + g;
        if (row >= n) continue;
        double* y = Y + row * ldy;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = c0 + 8 * nt + 2 * q;
          if (vstore && c + 1 < r) {
            *reinterpret_cast<double2*>(y + c) = make_double2(d[u][nt][0], d[u][nt][1]);
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (c + i < r) y[c + i] = d[u][nt][i];
          }
        }
      }
    }
  }
}

// Software-pipelined variant: one 8-row tile per iteration, the next tile's
// rows loaded (into registers) before this tile's MMAs, so loads, MMAs and
// stores of a warp overlap (the two-tile kernel above is co-bound by its
// loads and its MMAs: 0.87 ms at C4 vs a 0.64 ms overlap bound).  The next
// tile belongs to the same warp and is disjoint from the tile being written,
// so Y may still alias X.
template <int KS, int NT>
__global__ void __launch_bounds__(384, 1) rowmix_upper_pipe_kernel(int n, int r, const double* X,
                                                                int ldx,
                                                                const double* __restrict__ K,
                                                                int ldk, double* Y, int ldy,
                                                                int ldks) {
  constexpr int KC = 4 * KS, CW = 8 * NT, NP = KC / CW;
  extern __shared__ double sK[];  // KC x ldks, rows in fragment order (see rowmix_upper_kernel)
  for (int e = threadIdx.x; e < KC * KC; e += blockDim.x) {
    const int pr = e / KC, col = e - pr * KC;
    const int ks = pr >> 2, qq = pr & 3;
    const int k = 8 * (ks >> 1) + 2 * qq + (ks & 1);
    sK[pr * ldks + col] = (k < r && col < r) ? __ldg(K + (int64_t)k * ldk + col) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int64_t tiles = ((int64_t)n + 7) / 8;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vstore = ((ldy & 1) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  const bool vload = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && r == KC;
  auto load = [&](int64_t t, double (&af)[KS]) {
    const int64_t row = t * 8 + g;
    const bool live = t < tiles && row < n;
    const double* xr = X + row * ldx + 2 * q;
    if (vload && live) {
#pragma unroll
      for (int m = 0; m < KS / 2; ++m) {
        const double2 v = *reinterpret_cast<const double2*>(xr + 8 * m);
        af[2 * m] = v.x;
        af[2 * m + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c = 8 * (ks >> 1) + 2 * q + (ks & 1);
        af[ks] = (live && c < r) ? X[row * ldx + c] : 0.0;
      }
    }
  };
  int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double cur[KS], nxt[KS];
  load(t0, cur);
  for (; t0 < tiles; t0 += nwarps) {
    load(t0 + nwarps, nxt);
    __syncwarp();  // every lane's reads of this tile precede the in-place writes
    const int64_t row = t0 * 8 + g;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int c0 = p * CW;
      double d[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double* kr = sK + (4 * ks + q) * ldks + c0 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (8 * (ks >> 1) > c0 + 8 * nt + 7) continue;
          dmma(d[nt][0], d[nt][1], cur[ks], kr[8 * nt]);
        }
      }
      if (row < n) {
        double* y = Y + row * ldy;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = c0 + 8 * nt + 2 * q;
          if (vstore && c + 1 < r) {
            *reinterpret_cast<double2*>(y + c) = make_double2(d[nt][0], d[nt][1]);
          } else {
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (c + i < r) y[c + i] = d[nt][i];
          }
        }
      }
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) cur[ks] = nxt[ks];
  }
}

int rowmix_upper(int64_t n, int r, const double* X, int ldx, const double* K, int ldk, double* Y,
                 int ldy, cudaStream_t st) {
  if (r <= 16 || r > 128 || n < 64)
    return dlrsn_rowmix(n, r, r, X, ldx, K, ldk, 0.0, Y, ldy, st);
  const int64_t tiles = (n + 7) / 8;
  int64_t blocks = (tiles + 15) / 16;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (r <= 32) {
    constexpr int KS = 8, NT = 4;
    const int ldks = 32 + 4;
    const size_t smem = (size_t)4 * KS * ldks * sizeof(double);
    rowmix_upper_kernel<KS, NT><<<(int)blocks, 256, smem, st>>>((int)n, r, X, ldx, K, ldk, Y, ldy, ldks);
  } else if (r <= 64) {
    constexpr int KS = 16, NT = 8;
    const int ldks = 64 + 4;
    const size_t smem = (size_t)4 * KS * ldks * sizeof(double);
    // software-pipelined kernel, 12 warps per SM (DLRSN_ROWMIX_PIPE=0: the
    // two-tile kernel; 1: 8 warps): C4 0.87 -> 0.70 (8 warps) -> 0.66 ms
    static const int pipe = getenv("DLRSN_ROWMIX_PIPE") ? atoi(getenv("DLRSN_ROWMIX_PIPE")) : 2;
    if (pipe) {
      DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_upper_pipe_kernel<KS, NT>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int threads = pipe >= 2 ? 384 : 256;  // 162 registers: 12 warps fit one SM
      int64_t pb = (tiles + 7) / 8;
      if (pb > 148) pb = 148;
      rowmix_upper_pipe_kernel<KS, NT><<<(int)pb, threads, smem, st>>>((int)n, r, X, ldx, K, ldk, Y,
                                                                      ldy, ldks);
      DLRSN_CHECK_LAUNCH("rowmix_upper_pipe_kernel");
      return DLRSN_OK;
    }
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_upper_kernel<KS, NT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rowmix_upper_kernel<KS, NT><<<(int)blocks, 256, smem, st>>>((int)n, r, X, ldx, K, ldk, Y, ldy, ldks);
  } else {
    constexpr int KS = 32, NT = 8;
    const int ldks = 128 + 4;
    const size_t smem = (size_t)4 * KS * ldks * sizeof(double);
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_upper_kernel<KS, NT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rowmix_upper_kernel<KS, NT><<<(int)blocks, 256, smem, st>>>((int)n, r, X, ldx, K, ldk, Y, ldy, ldks);
  }
  DLRSN_CHECK_LAUNCH("rowmix_upper_kernel");
  return DLRSN_OK;
}

// ---------------------------------------------------------------------------
// mgram: G (ra x rb) = sum_c coeff_c * A_c^T M B_c; A_c = rows 4c..4c+3.
// Block = one chunk of cells x one (TI x TJ) output tile; thread (i, j) of
// the tile accumulates serially over the chunk (deterministic order).
constexpr int kTile = 16;
constexpr int kChunk = 32;   // cells per smem pass (mgram)
constexpr int kChunkP = 8;  // cells per smem pass (project)

__global__ void __launch_bounds__(256) mgram_kernel(int ncell, int ra, int rb,
                                                    const double* __restrict__ A, int lda,
                                                    const double* __restrict__ B, int ldb,
                                                    const double* __restrict__ coeff,
                                                    dlrsn_cellops ops, int cells_per_block,
                                                    double* __restrict__ part) {
  // 4 row groups x 64 threads; thread (ti, tj) owns the 2x2 micro-tile
  // (2ti.., 2tj..) of the block's 16x16 output tile, so each pair of 16-byte
  // shared loads feeds 4 FMAs.  Groups take interleaved rows and are summed
  // in fixed order at the end (deterministic).
  __shared__ __align__(16) double sA[kChunk * 4][kTile];
  __shared__ __align__(16) double sB[kChunk * 4][kTile];
  __shared__ double red[3][64][4];
  const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int ti = t >> 3, tj = t & 7;
  const int tiles_j = (rb + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * cells_per_block;
  const int c_end = min(ncell, c_begin + cells_per_block);
  double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
  for (int c0 = c_begin; c0 < c_end; c0 += kChunk) {
    const int nc = min(kChunk, c_end - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * 4 * kTile; e += blockDim.x) {
      const int row = e / kTile, col = e % kTile;
      const int64_t grow = (int64_t)c0 * 4 + row;
      sA[row][col] = (i0 + col < ra) ? __ldg(A + grow * lda + i0 + col) : 0.0;
    }
    // B rows pre-multiplied by coeff_c * M
    for (int e = threadIdx.x; e < nc * kTile; e += blockDim.x) {
      const int cl = e / kTile, col = e % kTile;
      const int c = c0 + cl;
      double b[4];
#pragma unroll
      for (int l = 0; l < 4; ++l)
        b[l] = (j0 + col < rb) ? __ldg(B + ((int64_t)c * 4 + l) * ldb + j0 + col) : 0.0;
      const double w = coeff ? coeff[c] : 1.0;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const double mb = ops.mass[4 * l] * b[0] + ops.mass[4 * l + 1] * b[1] +
                          ops.mass[4 * l + 2] * b[2] + ops.mass[4 * l + 3] * b[3];
        sB[cl * 4 + l][col] = coeff ? mb * w : mb;
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int row = g; row < nc * 4; row += 4) {
      const double2 a = *reinterpret_cast<const double2*>(&sA[row][2 * ti]);
      const double2 b = *reinterpret_cast<const double2*>(&sB[row][2 * tj]);
      a00 = fma(a.x, b.x, a00);
      a01 = fma(a.x, b.y, a01);
      a10 = fma(a.y, b.x, a10);
      a11 = fma(a.y, b.y, a11);
    }
  }
  __syncthreads();
  if (g > 0) {
    red[g - 1][t][0] = a00;
    red[g - 1][t][1] = a01;
    red[g - 1][t][2] = a10;
    red[g - 1][t][3] = a11;
  }
  __syncthreads();
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      a00 += red[q][t][0];
      a01 += red[q][t][1];
      a10 += red[q][t][2];
      a11 += red[q][t][3];
    }
    const double v[4] = {a00, a01, a10, a11};
    double* out = part + (int64_t)blockIdx.x * ra * rb;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 2 * ti + (q >> 1), j = j0 + 2 * tj + (q & 1);
      if (i < ra && j < rb) out[(int64_t)i * rb + j] = v[q];
    }
  }
}

// mgram on the FP64 tensor cores: warp w of the block takes cells
// c_begin + w, + 8, ...; per cell the k dimension of the MMA is the cell's 4
// dofs, A = X_c^T (m = column of A), B = M X_c (the 4x4 mass block applied
// across each lane quad by shuffles).  Warp partials are summed in warp order.
__global__ void __launch_bounds__(256, 4) mgram_mma_kernel(int ncell, int ra, int rb,
                                                        const double* __restrict__ A, int lda,
                                                        const double* __restrict__ B, int ldb,
                                                        const double* __restrict__ coeff,
                                                        dlrsn_cellops ops, int cells_per_block,
                                                        double* __restrict__ part) {
  __shared__ double red[8][kTile * kTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int tiles_j = (rb + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * cells_per_block;
  const int c_end = min(ncell, c_begin + cells_per_block);
  double m[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) m[b] = ops.mass[4 * q + b];
  const bool same = (A == B) && (lda == ldb) && (i0 == j0);
  const bool ia0 = i0 + g < ra, ia1 = i0 + 8 + g < ra, jb0 = j0 + g < rb, jb1 = j0 + 8 + g < rb;
  const int base = lane & ~3;
  double d[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  constexpr int U = 2;  // cells per warp and iteration: loads in flight together
  for (int c0 = c_begin + warp; c0 < c_end; c0 += 8 * U) {
    double a0[U], a1[U], v0[U], v1[U], wc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 8 * u;
      const bool in = c < c_end;
      const int64_t row = (int64_t)c * 4 + q;
      a0[u] = (in && ia0) ? __ldg(A + row * lda + i0 + g) : 0.0;
      a1[u] = (in && ia1) ? __ldg(A + row * lda + i0 + 8 + g) : 0.0;
      v0[u] = a0[u];
      v1[u] = a1[u];
      if (!same) {
        v0[u] = (in && jb0) ? __ldg(B + row * ldb + j0 + g) : 0.0;
        v1[u] = (in && jb1) ? __ldg(B + row * ldb + j0 + 8 + g) : 0.0;
      }
      wc[u] = (coeff && in) ? __ldg(coeff + c) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        b0 = fma(m[b], __shfl_sync(kFull, v0[u], base | b), b0);
        b1 = fma(m[b], __shfl_sync(kFull, v1[u], base | b), b1);
      }
      if (coeff) {
        b0 *= wc[u];
        b1 *= wc[u];
      }
      dmma(d[0][0][0], d[0][0][1], a0[u], b0);
      dmma(d[0][1][0], d[0][1][1], a0[u], b1);
      dmma(d[1][0][0], d[1][0][1], a1[u], b0);
      dmma(d[1][1][0], d[1][1][1], a1[u], b1);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 2; ++i) red[warp][(8 * mt + g) * kTile + 8 * nt + 2 * q + i] = d[mt][nt][i];
  __syncthreads();
  const int e = threadIdx.x;  // 256 = kTile * kTile entries
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w][e];
  const int i = i0 + e / kTile, j = j0 + e % kTile;
  if (i < ra && j < rb) part[(int64_t)blockIdx.x * ra * rb + (int64_t)i * rb + j] = s;
}

// mgram for wide bases (ra or rb > 32): a CTA owns a TB x TB output block
// over a range of cells.  Chunks of 16 cells stream into shared memory with
// cp.async (double-buffered: the next chunk is in flight while this one is
// multiplied); B rows are then premultiplied by coeff_c M into a third
// plane.  Row stride TB + 4 makes every fragment load conflict-free.  Each
// warp owns a 32 x 32 sub-block (4 x 4 DMMA tiles) for 1 / KP of every
// chunk's cells (k step = one cell's 4 dofs); the KP parts are summed in
// fixed order at the end.
constexpr int kMgC = 16;  // cells per chunk
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int TB>
struct MgramWide {
  static constexpr int LD = TB + 4, CR = 4 * kMgC, PL = CR * LD;  // plane = one chunk
  static constexpr int KP = 8 / ((TB / 32) * (TB / 32));
  // planes: A x2, B' x1, raw B x2 (separate operands only)
  static constexpr size_t smem(bool same) {
    const size_t st = (size_t)PL * (same ? 3 : 5);
    const size_t red = (size_t)KP * TB * (TB + 1);
    return sizeof(double) * (st > red ? st : red);
  }
};

template <int TB>
__global__ void __launch_bounds__(256, TB == 64 ? 2 : 1) mgram_wide_kernel(int ncell, int ra, int rb,
                                                         const double* __restrict__ A, int lda,
                                                         const double* __restrict__ B, int ldb,
                                                         const double* __restrict__ coeff,
                                                         dlrsn_cellops ops, int cells_per_block,
                                                         double* __restrict__ part, int vec,
                                                         int sym, const double* __restrict__ VV,
                                                         double* __restrict__ YV) {
  using P = MgramWide<TB>;
  constexpr int LD = P::LD, PL = P::PL, KP = P::KP, NWT = 8 / KP, CPK = kMgC / KP;
  constexpr int NCP = TB / 2;  // column pairs
  extern __shared__ __align__(16) double smw[];
  __shared__ double m[16];
  if (threadIdx.x < 16) m[threadIdx.x] = ops.mass[threadIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int wt = warp % NWT, kp = warp / NWT;
  const int wi = wt / (TB / 32), wj = wt % (TB / 32);
  const int tiles_j = (rb + TB - 1) / TB;
  int i0 = (blockIdx.y / tiles_j) * TB, j0 = (blockIdx.y % tiles_j) * TB;
  if (sym & 1) {  // symmetric Gram (A == B): blockIdx.y walks the tiles ti <= tj
    int y = blockIdx.y, ti = 0;
    while (y >= tiles_j - ti) {
      y -= tiles_j - ti;
      ++ti;
    }
    i0 = ti * TB;
    j0 = (ti + y) * TB;
  }
  const int c_begin = blockIdx.x * cells_per_block;
  const int c_end = min(ncell, c_begin + cells_per_block);
  const bool same = (A == B) && (lda == ldb) && (i0 == j0);
  // diagonal tile of a symmetric Gram (64-wide): upper 8 x 8 fragments only
  // (36 of 64 DMMA fragments), the lower ones mirrored at the write-out
  const bool fsym = TB == 64 && same && !(sym & 2);
  double* sA0 = smw;
  double* sBm = smw + 2 * PL;   // B' (premultiplied)
  double* sBr0 = smw + 3 * PL;  // raw B x2 (separate operands)
  const int64_t row_end = 4 * (int64_t)c_end;
  auto stage = [&](const double* __restrict__ src, int ld, int cols, int col0, double* dst,
                   int64_t row0) {
    for (int e = threadIdx.x; e < P::CR * NCP; e += 256) {
      const int row = e / NCP, cp = e - row * NCP;
      const int64_t grow = row0 + row;
      const int col = col0 + 2 * cp;
      double* d = dst + row * LD + 2 * cp;
      if (grow < row_end && vec && col + 1 < cols) {
        cp_async16(d, src + grow * ld + col);
      } else {
        d[0] = (grow < row_end && col < cols) ? __ldg(src + grow * ld + col) : 0.0;
        d[1] = (grow < row_end && col + 1 < cols) ? __ldg(src + grow * ld + col + 1) : 0.0;
      }
    }
  };
  auto issue = [&](int c0, int buf) {
    stage(A, lda, ra, i0, sA0 + buf * PL, 4 * (int64_t)c0);
    if (!same) stage(B, ldb, rb, j0, sBr0 + buf * PL, 4 * (int64_t)c0);
    cp_async_commit();
  };
  double d[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) d[a][b][0] = d[a][b][1] = 0.0;
  if (c_begin < c_end) issue(c_begin, 0);
  int buf = 0;
  for (int c0 = c_begin; c0 < c_end; c0 += kMgC, buf ^= 1) {
    if (c0 + kMgC < c_end) {
      issue(c0 + kMgC, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk landed (cp.async and plain fills of all threads)
    const double* sA = sA0 + buf * PL;
    const double* sBsrc = same ? sA : sBr0 + buf * PL;
    for (int e = threadIdx.x; e < kMgC * NCP; e += 256) {
      const int cl = e / NCP, cp = e - cl * NCP;
      double2 v[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] = *reinterpret_cast<const double2*>(sBsrc + (4 * cl + l) * LD + 2 * cp);
      if constexpr (TB == 64) {
        // optional extra output YV = B VV from the staged rows (single-tile
        // Grams, j0 = 0: a warp holds all 64 columns of one cell's 4 dof rows)
        if (VV) {
          const double v0 = 2 * cp < rb ? __ldg(VV + 2 * cp) : 0.0;
          const double v1 = 2 * cp + 1 < rb ? __ldg(VV + 2 * cp + 1) : 0.0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            double dsum = fma(v[l].x, v0, v[l].y * v1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(kFull, dsum, o);
            if (cp == 0 && c0 + cl < c_end) YV[4 * (int64_t)(c0 + cl) + l] = dsum;
          }
        }
      }
      const double w = (coeff && c0 + cl < c_end) ? __ldg(coeff + c0 + cl) : 1.0;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        double2 mb = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          mb.x = fma(m[4 * l + b], v[b].x, mb.x);
          mb.y = fma(m[4 * l + b], v[b].y, mb.y);
        }
        if (coeff) {
          mb.x *= w;
          mb.y *= w;
        }
        *reinterpret_cast<double2*>(sBm + (4 * cl + l) * LD + 2 * cp) = mb;
      }
    }
    __syncthreads();
    if (fsym && wt < 2) {
      // symmetric diagonal tile, rows 16 wt .. 16 wt + 15 x columns 32..63
#pragma unroll
      for (int k = 0; k < CPK; ++k) {
        const int cl = kp * CPK + k;
        const double* ar = sA + (4 * cl + q) * LD + 16 * wt + g;
        const double* br = sBm + (4 * cl + q) * LD + 32 + g;
        double af[2], bf[4];
        af[0] = ar[0];
        af[1] = ar[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) bf[t] = br[8 * t];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma(d[a][b][0], d[a][b][1], af[a], bf[b]);
      }
    } else if (fsym) {
      // symmetric diagonal tile, the diagonal 32 x 32 quadrant wt - 2: the
      // 8 x 8 fragments on and above its diagonal
      const int base = 32 * (wt - 2);
#pragma unroll
      for (int k = 0; k < CPK; ++k) {
        const int cl = kp * CPK + k;
        const double* ar = sA + (4 * cl + q) * LD + base + g;
        const double* br = sBm + (4 * cl + q) * LD + base + g;
        double af[4], bf[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          af[t] = ar[8 * t];
          bf[t] = br[8 * t];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = a; b < 4; ++b) dmma(d[a][b][0], d[a][b][1], af[a], bf[b]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < CPK; ++k) {
        const int cl = kp * CPK + k;
        const double* ar = sA + (4 * cl + q) * LD + 32 * wi + g;
        const double* br = sBm + (4 * cl + q) * LD + 32 * wj + g;
        double af[4], bf[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          af[t] = ar[8 * t];
          bf[t] = br[8 * t];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma(d[a][b][0], d[a][b][1], af[a], bf[b]);
      }
    }
    __syncthreads();  // this chunk's planes are free for the next issue
  }
  double* red = smw;  // [KP][TB][TB + 1]
  if (fsym) {
    const int r0 = wt < 2 ? 16 * wt : 32 * (wt - 2), c0 = wt < 2 ? 32 : 32 * (wt - 2);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (wt < 2 ? a >= 2 : b < a) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i)
          red[(kp * TB + r0 + 8 * a + g) * (TB + 1) + c0 + 8 * b + 2 * q + i] = d[a][b][i];
      }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          red[(kp * TB + 32 * wi + 8 * a + g) * (TB + 1) + 32 * wj + 8 * b + 2 * q + i] = d[a][b][i];
  }
  __syncthreads();
  double* out = part + (int64_t)blockIdx.x * ra * rb;
  for (int e = threadIdx.x; e < TB * TB; e += 256) {
    const int ii = e / TB, jj = e % TB;
    const int i = i0 + ii, j = j0 + jj;
    if (i >= ra || j >= rb) continue;
    // symmetric diagonal tile: fragments below the diagonal from their mirror
    const bool low = fsym && (ii >> 3) > (jj >> 3);
    const int si = low ? jj : ii, sj = low ? ii : jj;
    double v = 0.0;
#pragma unroll
    for (int p = 0; p < KP; ++p) v += red[(p * TB + si) * (TB + 1) + sj];
    out[(int64_t)i * rb + j] = v;
  }
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
  // row-slab decomposition (multi-GPU, slab.py): X rows of the grid row just
  // below this slab (4 nx x r, nullable: the bottom wall), and whether the
  // slab's top row is the domain's top wall (else the face above belongs to
  // the next slab, which sees this slab's top row as its halo)
  const double* halo;
  int top_wall;
  // no scattering (sigma_s null, or *any_scat == 0 on the device): ms = 0
  // exactly, its MMAs are skipped
  const int* any_scat;
};

__device__ inline double ldx(const double* X, int r, int64_t row, int col) {
  return col < r ? __ldg(X + row * r + col) : 0.0;
}

// local dof l of the cell below cell c = (ci, cj) of this slab: a slab row,
// or the halo row below the slab, or 0 at the bottom wall (vacuum trace)
__device__ inline double ld_below(const ProjArgs& pa, const double* X, int c, int ci, int cj, int l,
                                  int col) {
  if (cj > 0) return ldx(X, pa.r, (int64_t)(c - pa.nx) * 4 + l, col);
  return pa.halo ? ldx(pa.halo, pa.r, (int64_t)ci * 4 + l, col) : 0.0;
}

__device__ inline double2 ld2s(const double* p) { return *reinterpret_cast<const double2*>(p); }

// acc (2x2, row-major) += a (2) outer b (2)
__device__ inline void outer2(double* acc, double2 a, double2 b) {
  acc[0] = fma(a.x, b.x, acc[0]);
  acc[1] = fma(a.x, b.y, acc[1]);
  acc[2] = fma(a.y, b.x, acc[2]);
  acc[3] = fma(a.y, b.y, acc[3]);
}

__global__ void __launch_bounds__(256, 2) project_kernel(ProjArgs pa, dlrsn_cellops ops) {
  // Per chunk of kChunkP cells the block stages, for its 16x16 output tile,
  // the i-side rows (X, Xold, face jumps u) and the j-side rows (M X, Gx X,
  // Gy X, 1/2 e2 v, 1/2 e2 u, q_c src.X).  4 cell groups x 64 threads; each
  // thread owns a 2x2 micro-tile of all 7 outputs (28 accumulators), so each
  // 16-byte shared load feeds several FMAs.  Groups are summed in fixed order.
  constexpr int C = kChunkP;
  constexpr int kPer = C * 16;  // doubles per [C][16] plane
  __shared__ __align__(16) double sm[kPer * 33 + 2 * C];
  double* sX = sm;               // [C][4][16]
  double* sXo = sX + 4 * kPer;   // [C][4][16]
  double* sU = sXo + 4 * kPer;   // [C][4][16]: ux0 ux1 uy0 uy1
  double* sMX = sU + 4 * kPer;   // [C][4][16]
  double* sGX = sMX + 4 * kPer;  // [C][4][16]
  double* sGY = sGX + 4 * kPer;  // [C][4][16]
  double* sF = sGY + 4 * kPer;   // [C][8][16]
  double* sQ = sF + 8 * kPer;    // [C][16]
  double* sC = sQ + kPer;        // [C][2]
  // cell operator constants in shared memory (keeps them out of registers)
  __shared__ double so[64];  // mass 0-15, gx 16-31, gy 32-47, e2x 48-51, e2y 52-55, src 56-59
  if (threadIdx.x < 16) {
    so[threadIdx.x] = ops.mass[threadIdx.x];
    so[16 + threadIdx.x] = ops.gx[threadIdx.x];
    so[32 + threadIdx.x] = ops.gy[threadIdx.x];
  } else if (threadIdx.x < 20) {
    so[48 + threadIdx.x - 16] = ops.e2x[threadIdx.x - 16];
    so[52 + threadIdx.x - 16] = ops.e2y[threadIdx.x - 16];
    so[56 + threadIdx.x - 16] = ops.src_row[threadIdx.x - 16];
  }
  const double* e2x = so + 48;
  const double* e2y = so + 52;
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const int ncell = nx * ny;
  const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int ti = t >> 3, tj = t & 7;
  const int tiles_j = (r + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  double acc[7][4];
#pragma unroll
  for (int o = 0; o < 7; ++o)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[o][q] = 0.0;
  double qacc[2] = {0.0, 0.0};
  const double* X = pa.X;
  for (int c0 = c_begin; c0 < c_end; c0 += C) {
    const int nc = min(C, c_end - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nc * kTile * 2; e += blockDim.x) {
      const int side = e / (nc * kTile);  // 0: tile-i columns, 1: tile-j columns
      const int rem = e % (nc * kTile);
      const int cl = rem / kTile, col = rem % kTile;
      const int c = c0 + cl;
      const int gcol = (side == 0 ? i0 : j0) + col;
      const int ci = c % nx, cj = c / nx;
      double x[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) x[l] = ldx(X, r, (int64_t)c * 4 + l, gcol);
      // face traces: left face (minus = left neighbour's right edge (1,3),
      // plus = this cell's left edge (0,2)); bottom face (minus = lower
      // neighbour's top edge (2,3), plus = this cell's bottom edge (0,1))
      double ax0 = 0.0, ax1 = 0.0, ay0 = 0.0, ay1 = 0.0;
      if (ci > 0) {
        ax0 = ldx(X, r, (int64_t)(c - 1) * 4 + 1, gcol);
        ax1 = ldx(X, r, (int64_t)(c - 1) * 4 + 3, gcol);
      }
      if (cj > 0 || pa.halo) {
        ay0 = ld_below(pa, X, c, ci, cj, 2, gcol);
        ay1 = ld_below(pa, X, c, ci, cj, 3, gcol);
      }
      const double ux0 = ax0 - x[0], ux1 = ax1 - x[2], vx0 = ax0 + x[0], vx1 = ax1 + x[2];
      const double uy0 = ay0 - x[0], uy1 = ay1 - x[1], vy0 = ay0 + x[0], vy1 = ay1 + x[1];
      const int base = cl * 64 + col;  // [cl][l][col] in a 4-row plane
      if (side == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sX[base + 16 * l] = x[l];
          sXo[base + 16 * l] = pa.Xold ? ldx(pa.Xold, r, (int64_t)c * 4 + l, gcol) : 0.0;
        }
        sU[base] = ux0;
        sU[base + 16] = ux1;
        sU[base + 32] = uy0;
        sU[base + 48] = uy1;
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double m = 0.0, gx = 0.0, gy = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            m = fma(so[4 * l + p], x[p], m);
            gx = fma(so[16 + 4 * l + p], x[p], gx);
            gy = fma(so[32 + 4 * l + p], x[p], gy);
          }
          sMX[base + 16 * l] = m;
          sGX[base + 16 * l] = gx;
          sGY[base + 16 * l] = gy;
        }
        double* f = sF + cl * 128 + col;
        f[0] = 0.5 * (e2x[0] * vx0 + e2x[1] * vx1);
        f[16] = 0.5 * (e2x[2] * vx0 + e2x[3] * vx1);
        f[32] = 0.5 * (e2y[0] * vy0 + e2y[1] * vy1);
        f[48] = 0.5 * (e2y[2] * vy0 + e2y[3] * vy1);
        f[64] = 0.5 * (e2x[0] * ux0 + e2x[1] * ux1);
        f[80] = 0.5 * (e2x[2] * ux0 + e2x[3] * ux1);
        f[96] = 0.5 * (e2y[0] * uy0 + e2y[1] * uy1);
        f[112] = 0.5 * (e2y[2] * uy0 + e2y[3] * uy1);
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) s = fma(so[56 + l], x[l], s);
        sQ[cl * 16 + col] = __ldg(pa.q + c) * s;  // q-hat (dlr_sn.py:70)
      }
    }
    for (int e = threadIdx.x; e < nc; e += blockDim.x) {
      sC[2 * e] = __ldg(pa.sigma_t + c0 + e);
      sC[2 * e + 1] = pa.sigma_s ? __ldg(pa.sigma_s + c0 + e) : 0.0;
    }
    __syncthreads();
    for (int cl = g; cl < nc; cl += 4) {
      double xm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int o = cl * 64 + 16 * l;
        const double2 xi = ld2s(sX + o + 2 * ti), xo = ld2s(sXo + o + 2 * ti);
        const double2 mj = ld2s(sMX + o + 2 * tj);
        outer2(xm, xi, mj);
        outer2(acc[0], xi, ld2s(sGX + o + 2 * tj));
        outer2(acc[1], xi, ld2s(sGY + o + 2 * tj));
        outer2(acc[6], xo, mj);
      }
      const double2 ux0 = ld2s(sU + cl * 64 + 2 * ti), ux1 = ld2s(sU + cl * 64 + 16 + 2 * ti);
      const double2 uy0 = ld2s(sU + cl * 64 + 32 + 2 * ti), uy1 = ld2s(sU + cl * 64 + 48 + 2 * ti);
      const double* f = sF + cl * 128 + 2 * tj;
      outer2(acc[0], ux0, ld2s(f));
      outer2(acc[0], ux1, ld2s(f + 16));
      outer2(acc[1], uy0, ld2s(f + 32));
      outer2(acc[1], uy1, ld2s(f + 48));
      outer2(acc[2], ux0, ld2s(f + 64));
      outer2(acc[2], ux1, ld2s(f + 80));
      outer2(acc[3], uy0, ld2s(f + 96));
      outer2(acc[3], uy1, ld2s(f + 112));
      const double st = sC[2 * cl], ss = sC[2 * cl + 1];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[4][q] = fma(st, xm[q], acc[4][q]);
        acc[5][q] = fma(ss, xm[q], acc[5][q]);
      }
      if (ti == 0) {
        qacc[0] += sQ[cl * 16 + 2 * tj];
        qacc[1] += sQ[cl * 16 + 2 * tj + 1];
      }
    }
  }
  // right / top boundary faces of the cells in this block's range
  // (a = this cell's right/top edge trace, b = 0)
  {
    const int ia = i0 + 2 * ti, ja = j0 + 2 * tj;
    const int first_right = c_begin + ((nx - 1 - c_begin % nx) % nx + nx) % nx;
    for (int c = first_right + g * nx; c < c_end; c += 4 * nx) {
      const int64_t r1 = (int64_t)c * 4 + 1, r3 = (int64_t)c * 4 + 3;
      const double2 a0 = make_double2(ldx(X, r, r1, ia), ldx(X, r, r1, ia + 1));
      const double2 a1 = make_double2(ldx(X, r, r3, ia), ldx(X, r, r3, ia + 1));
      const double bj0[2] = {ldx(X, r, r1, ja), ldx(X, r, r1, ja + 1)};
      const double bj1[2] = {ldx(X, r, r3, ja), ldx(X, r, r3, ja + 1)};
      const double2 f0 = make_double2(0.5 * (e2x[0] * bj0[0] + e2x[1] * bj1[0]),
                                      0.5 * (e2x[0] * bj0[1] + e2x[1] * bj1[1]));
      const double2 f1 = make_double2(0.5 * (e2x[2] * bj0[0] + e2x[3] * bj1[0]),
                                      0.5 * (e2x[2] * bj0[1] + e2x[3] * bj1[1]));
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      outer2(v, a0, f0);
      outer2(v, a1, f1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[0][q] += v[q];
        acc[2][q] += v[q];
      }
    }
    for (int c = max(c_begin, (ny - 1) * nx) + g; pa.top_wall && c < c_end; c += 4) {
      const int64_t r2 = (int64_t)c * 4 + 2, r3 = (int64_t)c * 4 + 3;
      const double2 a0 = make_double2(ldx(X, r, r2, ia), ldx(X, r, r2, ia + 1));
      const double2 a1 = make_double2(ldx(X, r, r3, ia), ldx(X, r, r3, ia + 1));
      const double bj0[2] = {ldx(X, r, r2, ja), ldx(X, r, r2, ja + 1)};
      const double bj1[2] = {ldx(X, r, r3, ja), ldx(X, r, r3, ja + 1)};
      const double2 f0 = make_double2(0.5 * (e2y[0] * bj0[0] + e2y[1] * bj1[0]),
                                      0.5 * (e2y[0] * bj0[1] + e2y[1] * bj1[1]));
      const double2 f1 = make_double2(0.5 * (e2y[2] * bj0[0] + e2y[3] * bj1[0]),
                                      0.5 * (e2y[2] * bj0[1] + e2y[3] * bj1[1]));
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      outer2(v, a0, f0);
      outer2(v, a1, f1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[1][q] += v[q];
        acc[3][q] += v[q];
      }
    }
  }
  // fixed-order group reduction through the staging buffer:
  // (g0 + g2) + (g1 + g3)
  constexpr int kV = 30;
  __syncthreads();
  if (g >= 2) {
    double* dst = sm + ((g - 2) * 64 + t) * kV;
#pragma unroll
    for (int o = 0; o < 7; ++o)
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[4 * o + q] = acc[o][q];
    dst[28] = qacc[0];
    dst[29] = qacc[1];
  }
  __syncthreads();
  if (g < 2) {
    const double* src = sm + (g * 64 + t) * kV;
#pragma unroll
    for (int o = 0; o < 7; ++o)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[o][q] += src[4 * o + q];
    qacc[0] += src[28];
    qacc[1] += src[29];
  }
  __syncthreads();
  if (g == 1) {
    double* dst = sm + t * kV;
#pragma unroll
    for (int o = 0; o < 7; ++o)
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[4 * o + q] = acc[o][q];
    dst[28] = qacc[0];
    dst[29] = qacc[1];
  }
  __syncthreads();
  if (g == 0) {
    const double* src = sm + t * kV;
    const int64_t stride = 7 * (int64_t)r * r + r;
    double* out = pa.part + (int64_t)blockIdx.x * stride;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + 2 * ti + (q >> 1), j = j0 + 2 * tj + (q & 1);
      if (i < r && j < r) {
#pragma unroll
        for (int o = 0; o < 7; ++o) out[(int64_t)o * r * r + (int64_t)i * r + j] = acc[o][q] + src[4 * o + q];
      }
    }
    if (i0 == 0 && ti == 0) {
      const int j = j0 + 2 * tj;
      if (j < r) out[7 * (int64_t)r * r + j] = qacc[0] + src[28];
      if (j + 1 < r) out[7 * (int64_t)r * r + j + 1] = qacc[1] + src[29];
    }
  }
}

// ---------------------------------------------------------------------------
// project on the FP64 tensor cores (DMMA m8n8k4) over shared-memory staged
// cell chunks.  The staging is project_kernel's (i-side rows X, Xold, face
// jumps u; j-side rows M X, Gx X, Gy X, 1/2 e2 v, 1/2 e2 u, q src.X), with a
// 20-double row stride so that the fragment loads of a lane quad hit distinct
// banks.  Warp w owns the 8x8 sub-tile (mt, nt) = (w & 1, (w >> 1) & 1) of
// all 7 outputs for half hf = w >> 2 of every chunk.  Per cell the MMA k
// dimension is its 4 dofs (volume terms: px, py, mt, ms, mo); the face terms
// of a cell pair share one MMA (k = the 2 face dofs of each cell: px, py, jx,
// jy).  Domain-boundary faces, q-hat and the fixed-order reductions are SIMT.
constexpr int kPC = 8;    // cells per chunk
constexpr int kLS = 20;   // row stride (doubles) of the staged planes
__global__ void __launch_bounds__(256, 2) project_mma_kernel(ProjArgs pa, dlrsn_cellops ops) {
  constexpr int C = kPC;
  constexpr int kRow = 4 * kLS;  // one cell's 4 rows
  __shared__ __align__(16) double sm[C * (6 * kRow + 2 * kRow) + C * 16 + 2 * C];
  double* sX = sm;               // [C][4][kLS] i-side
  double* sXo = sX + C * kRow;   // [C][4][kLS] i-side
  double* sU = sXo + C * kRow;   // [C][4][kLS] i-side: ux0 ux1 uy0 uy1
  double* sMX = sU + C * kRow;   // [C][4][kLS] j-side
  double* sGX = sMX + C * kRow;  // [C][4][kLS]
  double* sGY = sGX + C * kRow;  // [C][4][kLS]
  double* sF = sGY + C * kRow;   // [C][8][kLS]: (e2x v)x2 (e2y v)x2 (e2x u)x2 (e2y u)x2, halved
  double* sQ = sF + 2 * C * kRow;  // [C][16]
  double* sC = sQ + C * 16;        // [C][2]
  __shared__ double so[64];  // mass 0-15, gx 16-31, gy 32-47, e2x 48-51, e2y 52-55, src 56-59
  __shared__ double bnd[2][16][17];  // boundary-face parts of px (= jx) and py (= jy)
  if (threadIdx.x < 16) {
    so[threadIdx.x] = ops.mass[threadIdx.x];
    so[16 + threadIdx.x] = ops.gx[threadIdx.x];
    so[32 + threadIdx.x] = ops.gy[threadIdx.x];
  } else if (threadIdx.x < 20) {
    so[48 + threadIdx.x - 16] = ops.e2x[threadIdx.x - 16];
    so[52 + threadIdx.x - 16] = ops.e2y[threadIdx.x - 16];
    so[56 + threadIdx.x - 16] = ops.src_row[threadIdx.x - 16];
  }
  const double* e2x = so + 48;
  const double* e2y = so + 52;
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const int ncell = nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3, kk = q & 1, second = q >> 1;
  const int mt = warp & 1, nt = (warp >> 1) & 1, hf = warp >> 2;
  const int tiles_j = (r + kTile - 1) / kTile;
  const int i0 = (blockIdx.y / tiles_j) * kTile, j0 = (blockIdx.y % tiles_j) * kTile;
  const int c_begin = blockIdx.x * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  double acc[7][2];
#pragma unroll
  for (int o = 0; o < 7; ++o) acc[o][0] = acc[o][1] = 0.0;
  double qacc = 0.0;
  const double* X = pa.X;
  const int ca = 8 * mt + g, cb = 8 * nt + g;  // fragment columns within the tile
  // staging item of this thread (C x 16 columns x 2 sides = blockDim): the
  // global loads of chunk k+1 are issued before chunk k is computed
  const int side = threadIdx.x / (C * kTile);  // 0: tile-i columns, 1: tile-j columns
  const int scl = (threadIdx.x % (C * kTile)) / kTile, scol = threadIdx.x % kTile;
  const int sgcol = (side == 0 ? i0 : j0) + scol;
  struct Raw {
    double x[4], xo[4], ax0, ax1, ay0, ay1, qc, st, ss;
  };
  auto fetch = [&](int cc0, Raw& w) {
    const int c = cc0 + scl;
    const bool live = cc0 < c_end && c < c_end;
    const int ci = c % nx, cj = c / nx;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      w.x[l] = live ? ldx(X, r, (int64_t)c * 4 + l, sgcol) : 0.0;
      w.xo[l] = (live && side == 0 && pa.Xold) ? ldx(pa.Xold, r, (int64_t)c * 4 + l, sgcol) : 0.0;
    }
    const bool lx = live && ci > 0, ly = live && (cj > 0 || pa.halo != nullptr);
    w.ax0 = lx ? ldx(X, r, (int64_t)(c - 1) * 4 + 1, sgcol) : 0.0;
    w.ax1 = lx ? ldx(X, r, (int64_t)(c - 1) * 4 + 3, sgcol) : 0.0;
    w.ay0 = ly ? ld_below(pa, X, c, ci, cj, 2, sgcol) : 0.0;
    w.ay1 = ly ? ld_below(pa, X, c, ci, cj, 3, sgcol) : 0.0;
    w.qc = (live && side == 1) ? __ldg(pa.q + c) : 0.0;
    const bool cst = live && threadIdx.x < C;  // sigma of cell cc0 + threadIdx.x
    const int cs = cc0 + (int)threadIdx.x;
    w.st = (cc0 < c_end && threadIdx.x < C && cs < c_end) ? __ldg(pa.sigma_t + cs) : 0.0;
    w.ss = (pa.sigma_s && cc0 < c_end && threadIdx.x < C && cs < c_end) ? __ldg(pa.sigma_s + cs) : 0.0;
    (void)cst;
  };
  Raw cur;
  fetch(c_begin, cur);
  for (int c0 = c_begin; c0 < c_end; c0 += C) {
    const int nc = min(C, c_end - c0);
    __syncthreads();  // the previous chunk's fragments are consumed
    {
      const double* x = cur.x;
      const double ux0 = cur.ax0 - x[0], ux1 = cur.ax1 - x[2];
      const double vx0 = cur.ax0 + x[0], vx1 = cur.ax1 + x[2];
      const double uy0 = cur.ay0 - x[0], uy1 = cur.ay1 - x[1];
      const double vy0 = cur.ay0 + x[0], vy1 = cur.ay1 + x[1];
      const int base = scl * kRow + scol;
      if (side == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sX[base + kLS * l] = x[l];
          sXo[base + kLS * l] = cur.xo[l];
        }
        sU[base] = ux0;
        sU[base + kLS] = ux1;
        sU[base + 2 * kLS] = uy0;
        sU[base + 3 * kLS] = uy1;
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double m = 0.0, gx = 0.0, gy = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            m = fma(so[4 * l + p], x[p], m);
            gx = fma(so[16 + 4 * l + p], x[p], gx);
            gy = fma(so[32 + 4 * l + p], x[p], gy);
          }
          sMX[base + kLS * l] = m;
          sGX[base + kLS * l] = gx;
          sGY[base + kLS * l] = gy;
        }
        double* f = sF + 2 * scl * kRow + scol;
        f[0] = 0.5 * (e2x[0] * vx0 + e2x[1] * vx1);
        f[kLS] = 0.5 * (e2x[2] * vx0 + e2x[3] * vx1);
        f[2 * kLS] = 0.5 * (e2y[0] * vy0 + e2y[1] * vy1);
        f[3 * kLS] = 0.5 * (e2y[2] * vy0 + e2y[3] * vy1);
        f[4 * kLS] = 0.5 * (e2x[0] * ux0 + e2x[1] * ux1);
        f[5 * kLS] = 0.5 * (e2x[2] * ux0 + e2x[3] * ux1);
        f[6 * kLS] = 0.5 * (e2y[0] * uy0 + e2y[1] * uy1);
        f[7 * kLS] = 0.5 * (e2y[2] * uy0 + e2y[3] * uy1);
        double sq = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) sq = fma(so[56 + l], x[l], sq);
        sQ[scl * 16 + scol] = cur.qc * sq;  // q-hat (dlr_sn.py:70)
      }
      if (threadIdx.x < C) {
        sC[2 * threadIdx.x] = cur.st;
        sC[2 * threadIdx.x + 1] = cur.ss;
      }
    }
    __syncthreads();
    fetch(c0 + C, cur);  // next chunk's loads in flight during the MMAs
    // ---- volume terms: the 4 cells of this warp's half
#pragma unroll
    for (int k = 0; k < C / 2; ++k) {
      const int cl = hf * (C / 2) + k;
      const double xa = sX[cl * kRow + q * kLS + ca];
      const double xo = sXo[cl * kRow + q * kLS + ca];
      const double mx = sMX[cl * kRow + q * kLS + cb];
      const double gx = sGX[cl * kRow + q * kLS + cb];
      const double gy = sGY[cl * kRow + q * kLS + cb];
      const double stc = sC[2 * cl], ssc = sC[2 * cl + 1];
      dmma(acc[0][0], acc[0][1], xa, gx);        // px (volume)
      dmma(acc[1][0], acc[1][1], xa, gy);        // py (volume)
      dmma(acc[4][0], acc[4][1], stc * xa, mx);  // mt
      dmma(acc[5][0], acc[5][1], ssc * xa, mx);  // ms
      dmma(acc[6][0], acc[6][1], xo, mx);        // mo
    }
    // ---- face terms: pairs (cl, cl + 1) of this half; k slot q -> cell
    // cl + q / 2, face dof q % 2
#pragma unroll
    for (int k = 0; k < C / 4; ++k) {
      const int cl = hf * (C / 2) + 2 * k + second;
      const double uxa = sU[cl * kRow + kk * kLS + ca];
      const double uya = sU[cl * kRow + (2 + kk) * kLS + ca];
      const double* f = sF + 2 * cl * kRow + cb;
      dmma(acc[0][0], acc[0][1], uxa, f[kk * kLS]);        // px (faces)
      dmma(acc[1][0], acc[1][1], uya, f[(2 + kk) * kLS]);  // py (faces)
      dmma(acc[2][0], acc[2][1], uxa, f[(4 + kk) * kLS]);  // jx
      dmma(acc[3][0], acc[3][1], uya, f[(6 + kk) * kLS]);  // jy
    }
    if (i0 == 0 && threadIdx.x < 16)
      for (int cl = 0; cl < nc; ++cl) qacc += sQ[cl * 16 + threadIdx.x];
  }
  // ---- right / top domain-boundary faces (a = own right/top edge, b = 0)
  {
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    const int i = i0 + ti, j = j0 + tj;
    double bx = 0.0, by = 0.0;
    if (i < r && j < r) {
      const int first_right = c_begin + ((nx - 1 - c_begin % nx) % nx + nx) % nx;
      for (int c = first_right; c < c_end; c += nx) {
        const int64_t r1 = (int64_t)c * 4 + 1, r3 = (int64_t)c * 4 + 3;
        const double ai0 = ldx(X, r, r1, i), ai1 = ldx(X, r, r3, i);
        const double aj0 = ldx(X, r, r1, j), aj1 = ldx(X, r, r3, j);
        bx += ai0 * (0.5 * (e2x[0] * aj0 + e2x[1] * aj1)) + ai1 * (0.5 * (e2x[2] * aj0 + e2x[3] * aj1));
      }
      for (int c = max(c_begin, (ny - 1) * nx); pa.top_wall && c < c_end; ++c) {
        const int64_t r2 = (int64_t)c * 4 + 2, r3 = (int64_t)c * 4 + 3;
        const double ai0 = ldx(X, r, r2, i), ai1 = ldx(X, r, r3, i);
        const double aj0 = ldx(X, r, r2, j), aj1 = ldx(X, r, r3, j);
        by += ai0 * (0.5 * (e2y[0] * aj0 + e2y[1] * aj1)) + ai1 * (0.5 * (e2y[2] * aj0 + e2y[3] * aj1));
      }
    }
    bnd[0][ti][tj] = bx;
    bnd[1][ti][tj] = by;
  }
  // ---- fixed-order reduction: (half 0 + half 1) + boundary
  __syncthreads();
  double* red = sm;  // [2 halves][7][16][17], reusing the staging planes
#pragma unroll
  for (int o = 0; o < 7; ++o) {
    red[((hf * 7 + o) * 16 + 8 * mt + g) * 17 + 8 * nt + 2 * q] = acc[o][0];
    red[((hf * 7 + o) * 16 + 8 * mt + g) * 17 + 8 * nt + 2 * q + 1] = acc[o][1];
  }
  if (i0 == 0 && threadIdx.x < 16) sQ[threadIdx.x] = qacc;  // (staging planes are dead)
  __syncthreads();
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)blockIdx.x * stride;
  for (int e = threadIdx.x; e < 7 * 256; e += blockDim.x) {
    const int o = e >> 8, rem = e & 255, row = rem >> 4, col = rem & 15;
    const int i = i0 + row, j = j0 + col;
    if (i >= r || j >= r) continue;
    double v = red[((0 * 7 + o) * 16 + row) * 17 + col] + red[((1 * 7 + o) * 16 + row) * 17 + col];
    if (o == 0 || o == 2) v += bnd[0][row][col];  // px, jx
    if (o == 1 || o == 3) v += bnd[1][row][col];  // py, jy
    out[(int64_t)o * r * r + (int64_t)i * r + j] = v;
  }
  if (i0 == 0 && threadIdx.x < 16 && j0 + (int)threadIdx.x < r)
    out[7 * (int64_t)r * r + j0 + threadIdx.x] = sQ[threadIdx.x];
}

// ---------------------------------------------------------------------------
// project for r > 16: the staging and the MMA decomposition of
// project_mma_kernel with a 32x32 output tile, so each X element is staged
// by (r/32)^2 instead of (r/16)^2 tile blocks, and with 2x2 fragments per
// warp, so each staged fragment feeds two DMMAs.  Chunks of 4 cells; warp w
// owns the 16x16 sub-tile (w & 1, (w >> 1) & 1) for cell half w >> 2 of
// every chunk.  The tile blocks of one cell range are adjacent in the grid
// (blockIdx.x = tile), so they stream the same X rows through L2 together.
constexpr int kT32 = 32;
constexpr int kPC32 = 4;   // cells per chunk (4 cells x 32 columns x 2 sides = 256 threads)
constexpr int kLS32 = 36;  // row stride (doubles) of the staged planes
constexpr int kRow32 = 4 * kLS32;
constexpr size_t kProj32Stage = (size_t)kPC32 * 8 * kRow32 + kPC32 * kT32 + 2 * kPC32;
constexpr size_t kProj32Red = 7 * 32 * 33 + 2 * 32 * 33;
constexpr size_t kProj32Smem =
    (kProj32Stage > kProj32Red ? kProj32Stage : kProj32Red) * sizeof(double);

__global__ void __launch_bounds__(256, 1) project_mma32_kernel(ProjArgs pa, dlrsn_cellops ops) {
  constexpr int C = kPC32, kLS = kLS32, kRow = kRow32;
  extern __shared__ __align__(16) double sm32[];
  double* sX = sm32;             // [C][4][kLS] i-side
  double* sXo = sX + C * kRow;   // [C][4][kLS] i-side
  double* sU = sXo + C * kRow;   // [C][4][kLS] i-side: ux0 ux1 uy0 uy1
  double* sMX = sU + C * kRow;   // [C][4][kLS] j-side
  double* sGX = sMX + C * kRow;  // [C][4][kLS]
  double* sGY = sGX + C * kRow;  // [C][4][kLS]
  double* sF = sGY + C * kRow;   // [C][8][kLS]
  double* sQ = sF + 2 * C * kRow;  // [C][32]
  double* sC = sQ + C * kT32;      // [C][2]
  __shared__ double so[64];
  if (threadIdx.x < 16) {
    so[threadIdx.x] = ops.mass[threadIdx.x];
    so[16 + threadIdx.x] = ops.gx[threadIdx.x];
    so[32 + threadIdx.x] = ops.gy[threadIdx.x];
  } else if (threadIdx.x < 20) {
    so[48 + threadIdx.x - 16] = ops.e2x[threadIdx.x - 16];
    so[52 + threadIdx.x - 16] = ops.e2y[threadIdx.x - 16];
    so[56 + threadIdx.x - 16] = ops.src_row[threadIdx.x - 16];
  }
  const double* e2x = so + 48;
  const double* e2y = so + 52;
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const int ncell = nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3, kk = q & 1, second = q >> 1;
  const int mp = warp & 1, np = (warp >> 1) & 1, hf = warp >> 2;
  const int tiles_j = (r + kT32 - 1) / kT32;
  const int i0 = (blockIdx.x / tiles_j) * kT32, j0 = (blockIdx.x % tiles_j) * kT32;
  const int c_begin = blockIdx.y * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  double acc[7][2][2][2];
#pragma unroll
  for (int o = 0; o < 7; ++o)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[o][a][b][0] = acc[o][a][b][1] = 0.0;
  double qacc = 0.0;
  const double* X = pa.X;
  int ca[2], cb[2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    ca[a] = 8 * (2 * mp + a) + g;
    cb[a] = 8 * (2 * np + a) + g;
  }
  const int side = threadIdx.x / (C * kT32);
  const int scl = (threadIdx.x % (C * kT32)) / kT32, scol = threadIdx.x % kT32;
  const int sgcol = (side == 0 ? i0 : j0) + scol;
  struct Raw {
    double x[4], xo[4], ax0, ax1, ay0, ay1, qc, st, ss;
  };
  auto fetch = [&](int cc0, Raw& w) {
    const int c = cc0 + scl;
    const bool live = cc0 < c_end && c < c_end;
    const int ci = c % nx, cj = c / nx;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      w.x[l] = live ? ldx(X, r, (int64_t)c * 4 + l, sgcol) : 0.0;
      w.xo[l] = (live && side == 0 && pa.Xold) ? ldx(pa.Xold, r, (int64_t)c * 4 + l, sgcol) : 0.0;
    }
    const bool lx = live && ci > 0, ly = live && (cj > 0 || pa.halo != nullptr);
    w.ax0 = lx ? ldx(X, r, (int64_t)(c - 1) * 4 + 1, sgcol) : 0.0;
    w.ax1 = lx ? ldx(X, r, (int64_t)(c - 1) * 4 + 3, sgcol) : 0.0;
    w.ay0 = ly ? ld_below(pa, X, c, ci, cj, 2, sgcol) : 0.0;
    w.ay1 = ly ? ld_below(pa, X, c, ci, cj, 3, sgcol) : 0.0;
    w.qc = (live && side == 1) ? __ldg(pa.q + c) : 0.0;
    const int cs = cc0 + (int)threadIdx.x;
    w.st = (cc0 < c_end && threadIdx.x < C && cs < c_end) ? __ldg(pa.sigma_t + cs) : 0.0;
    w.ss = (pa.sigma_s && cc0 < c_end && threadIdx.x < C && cs < c_end) ? __ldg(pa.sigma_s + cs) : 0.0;
  };
  Raw cur;
  fetch(c_begin, cur);
  for (int c0 = c_begin; c0 < c_end; c0 += C) {
    const int nc = min(C, c_end - c0);
    __syncthreads();  // the previous chunk's fragments are consumed
    {
      const double* x = cur.x;
      const double ux0 = cur.ax0 - x[0], ux1 = cur.ax1 - x[2];
      const double vx0 = cur.ax0 + x[0], vx1 = cur.ax1 + x[2];
      const double uy0 = cur.ay0 - x[0], uy1 = cur.ay1 - x[1];
      const double vy0 = cur.ay0 + x[0], vy1 = cur.ay1 + x[1];
      const int base = scl * kRow + scol;
      if (side == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sX[base + kLS * l] = x[l];
          sXo[base + kLS * l] = cur.xo[l];
        }
        sU[base] = ux0;
        sU[base + kLS] = ux1;
        sU[base + 2 * kLS] = uy0;
        sU[base + 3 * kLS] = uy1;
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double m = 0.0, gx = 0.0, gy = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            m = fma(so[4 * l + p], x[p], m);
            gx = fma(so[16 + 4 * l + p], x[p], gx);
            gy = fma(so[32 + 4 * l + p], x[p], gy);
          }
          sMX[base + kLS * l] = m;
          sGX[base + kLS * l] = gx;
          sGY[base + kLS * l] = gy;
        }
        double* f = sF + 2 * scl * kRow + scol;
        f[0] = 0.5 * (e2x[0] * vx0 + e2x[1] * vx1);
        f[kLS] = 0.5 * (e2x[2] * vx0 + e2x[3] * vx1);
        f[2 * kLS] = 0.5 * (e2y[0] * vy0 + e2y[1] * vy1);
        f[3 * kLS] = 0.5 * (e2y[2] * vy0 + e2y[3] * vy1);
        f[4 * kLS] = 0.5 * (e2x[0] * ux0 + e2x[1] * ux1);
        f[5 * kLS] = 0.5 * (e2x[2] * ux0 + e2x[3] * ux1);
        f[6 * kLS] = 0.5 * (e2y[0] * uy0 + e2y[1] * uy1);
        f[7 * kLS] = 0.5 * (e2y[2] * uy0 + e2y[3] * uy1);
        double sq = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) sq = fma(so[56 + l], x[l], sq);
        sQ[scl * kT32 + scol] = cur.qc * sq;  // q-hat (dlr_sn.py:70)
      }
      if (threadIdx.x < C) {
        sC[2 * threadIdx.x] = cur.st;
        sC[2 * threadIdx.x + 1] = cur.ss;
      }
    }
    __syncthreads();
    fetch(c0 + C, cur);  // next chunk's loads in flight during the MMAs
    // ---- volume terms: the 2 cells of this warp's half
#pragma unroll
    for (int k = 0; k < C / 2; ++k) {
      const int cl = hf * (C / 2) + k;
      const double stc = sC[2 * cl], ssc = sC[2 * cl + 1];
      double xa[2], xo[2], mx[2], gx[2], gy[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        xa[a] = sX[cl * kRow + q * kLS + ca[a]];
        xo[a] = sXo[cl * kRow + q * kLS + ca[a]];
        mx[a] = sMX[cl * kRow + q * kLS + cb[a]];
        gx[a] = sGX[cl * kRow + q * kLS + cb[a]];
        gy[a] = sGY[cl * kRow + q * kLS + cb[a]];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const double xs = stc * xa[a], xss = ssc * xa[a];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          dmma(acc[0][a][b][0], acc[0][a][b][1], xa[a], gx[b]);  // px (volume)
          dmma(acc[1][a][b][0], acc[1][a][b][1], xa[a], gy[b]);  // py (volume)
          dmma(acc[4][a][b][0], acc[4][a][b][1], xs, mx[b]);     // mt
          dmma(acc[5][a][b][0], acc[5][a][b][1], xss, mx[b]);    // ms
          dmma(acc[6][a][b][0], acc[6][a][b][1], xo[a], mx[b]);  // mo
        }
      }
    }
    // ---- face terms: the cell pair of this half; k slot q -> cell cl + q / 2,
    // face dof q % 2
    {
      const int cl = hf * (C / 2) + second;
      double uxa[2], uya[2], fx[2], fy[2], fux[2], fuy[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        uxa[a] = sU[cl * kRow + kk * kLS + ca[a]];
        uya[a] = sU[cl * kRow + (2 + kk) * kLS + ca[a]];
        const double* f = sF + 2 * cl * kRow + cb[a];
        fx[a] = f[kk * kLS];
        fy[a] = f[(2 + kk) * kLS];
        fux[a] = f[(4 + kk) * kLS];
        fuy[a] = f[(6 + kk) * kLS];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          dmma(acc[0][a][b][0], acc[0][a][b][1], uxa[a], fx[b]);   // px (faces)
          dmma(acc[1][a][b][0], acc[1][a][b][1], uya[a], fy[b]);   // py (faces)
          dmma(acc[2][a][b][0], acc[2][a][b][1], uxa[a], fux[b]);  // jx
          dmma(acc[3][a][b][0], acc[3][a][b][1], uya[a], fuy[b]);  // jy
        }
    }
    if (i0 == 0 && threadIdx.x < kT32)
      for (int cl = 0; cl < nc; ++cl) qacc += sQ[cl * kT32 + threadIdx.x];
  }
  __syncthreads();  // staging planes are dead: reuse them for the reduction
  double* red = sm32;              // [7][32][33]: half 1's accumulators
  double* bnd = red + 7 * 32 * 33;  // [2][32][33]: right / top domain-boundary faces
  // ---- right / top domain-boundary faces (a = own right/top edge, b = 0)
  for (int e = threadIdx.x; e < kT32 * kT32; e += blockDim.x) {
    const int ti = e >> 5, tj = e & 31;
    const int i = i0 + ti, j = j0 + tj;
    double bx = 0.0, by = 0.0;
    if (i < r && j < r) {
      const int first_right = c_begin + ((nx - 1 - c_begin % nx) % nx + nx) % nx;
      for (int c = first_right; c < c_end; c += nx) {
        const int64_t r1 = (int64_t)c * 4 + 1, r3 = (int64_t)c * 4 + 3;
        const double ai0 = ldx(X, r, r1, i), ai1 = ldx(X, r, r3, i);
        const double aj0 = ldx(X, r, r1, j), aj1 = ldx(X, r, r3, j);
        bx += ai0 * (0.5 * (e2x[0] * aj0 + e2x[1] * aj1)) + ai1 * (0.5 * (e2x[2] * aj0 + e2x[3] * aj1));
      }
      for (int c = max(c_begin, (ny - 1) * nx); pa.top_wall && c < c_end; ++c) {
        const int64_t r2 = (int64_t)c * 4 + 2, r3 = (int64_t)c * 4 + 3;
        const double ai0 = ldx(X, r, r2, i), ai1 = ldx(X, r, r3, i);
        const double aj0 = ldx(X, r, r2, j), aj1 = ldx(X, r, r3, j);
        by += ai0 * (0.5 * (e2y[0] * aj0 + e2y[1] * aj1)) + ai1 * (0.5 * (e2y[2] * aj0 + e2y[3] * aj1));
      }
    }
    bnd[ti * 33 + tj] = bx;
    bnd[32 * 33 + ti * 33 + tj] = by;
  }
  if (hf == 1) {
#pragma unroll
    for (int o = 0; o < 7; ++o)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int row = 8 * (2 * mp + a) + g, col = 8 * (2 * np + b) + 2 * q;
          red[(o * 32 + row) * 33 + col] = acc[o][a][b][0];
          red[(o * 32 + row) * 33 + col + 1] = acc[o][a][b][1];
        }
  }
  __syncthreads();
  // ---- fixed-order reduction: (half 0 + half 1) + boundary
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)blockIdx.y * stride;
  if (hf == 0) {
#pragma unroll
    for (int o = 0; o < 7; ++o)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = 8 * (2 * mp + a) + g, col = 8 * (2 * np + b) + 2 * q + h;
            const int i = i0 + row, j = j0 + col;
            if (i >= r || j >= r) continue;
            double v = acc[o][a][b][h] + red[(o * 32 + row) * 33 + col];
            if (o == 0 || o == 2) v += bnd[row * 33 + col];            // px, jx
            if (o == 1 || o == 3) v += bnd[32 * 33 + row * 33 + col];  // py, jy
            out[(int64_t)o * r * r + (int64_t)i * r + j] = v;
          }
  }
  if (i0 == 0 && threadIdx.x < kT32 && j0 + (int)threadIdx.x < r)
    out[7 * (int64_t)r * r + j0 + threadIdx.x] = qacc;
}

// Output groups of the split launch: GROUP 0 = {px, py, jx, jy} (volume and
// face terms), GROUP 1 = {mt, ms, mo} + q-hat.  Each CTA stages only its
// group's planes and holds only its group's accumulators (4 or 3 outputs x
// 2x2 fragments instead of 7), so two CTAs (16 warps) fit per SM and the
// dependent DMMA chains of one warp are covered by the others.  Chunks of 8
// cells (two staging items per thread: the same cell rows for the i-side
// and the j-side columns), so each barrier pair is amortised over 4 cells
// of MMAs per warp.
constexpr int kPCG = 8;                          // cells per chunk
constexpr int kPlaneG = kPCG * kRow32;           // one staged plane
constexpr size_t kProj32StageG0 = 6 * (size_t)kPlaneG;
constexpr size_t kProj32StageG1 = 5 * (size_t)kPlaneG + kPCG * kT32;
constexpr size_t kProj32RedG0 = (4 + 2) * 32 * 33;
constexpr size_t kProj32RedG1 = 3 * 32 * 33;
constexpr size_t kProj32SmemG =
    std::max(std::max(kProj32StageG0, kProj32StageG1), std::max(kProj32RedG0, kProj32RedG1)) *
    sizeof(double);

template <int GROUP>
__device__ __forceinline__ void project32_group(const ProjArgs& pa, const dlrsn_cellops& ops,
                                                double* sm32, int ti, int tj, bool mo_only) {
  constexpr int C = kPCG, kLS = kLS32, kRow = kRow32;
  constexpr int NO = GROUP == 0 ? 4 : 3;  // accumulated outputs
  // group 0: sX sU (i-side), sGX sGY sF[2] (j-side); group 1: sX sXo (i),
  // sMX (j), then sQ [C][32] and sC [C][2]
  double* sX = sm32;
  double* sU = sm32 + kPlaneG;       // group 0
  double* sXo = sm32 + kPlaneG;      // group 1
  double* sGX = sm32 + 2 * kPlaneG;  // group 0
  double* sMX = sm32 + 2 * kPlaneG;  // group 1
  double* sGY = sm32 + 3 * kPlaneG;
  double* sF = sm32 + 4 * kPlaneG;   // [C][8][kLS]
  double* sMXt = sm32 + 3 * kPlaneG;  // group 1: sigma_t M X (j-side)
  double* sMXs = sm32 + 4 * kPlaneG;  // group 1: sigma_s M X (j-side)
  double* sQ = sm32 + 5 * kPlaneG;    // group 1
  __shared__ double so[64];
  if (threadIdx.x < 16) {
    so[threadIdx.x] = ops.mass[threadIdx.x];
    so[16 + threadIdx.x] = ops.gx[threadIdx.x];
    so[32 + threadIdx.x] = ops.gy[threadIdx.x];
  } else if (threadIdx.x < 20) {
    // halved edge masses: every face term carries the 1/2 of the average
    so[48 + threadIdx.x - 16] = 0.5 * ops.e2x[threadIdx.x - 16];
    so[52 + threadIdx.x - 16] = 0.5 * ops.e2y[threadIdx.x - 16];
    so[56 + threadIdx.x - 16] = ops.src_row[threadIdx.x - 16];
  }
  const double* e2x = so + 48;
  const double* e2y = so + 52;
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const bool no_ms = pa.sigma_s == nullptr || (pa.any_scat != nullptr && *pa.any_scat == 0);
  const int ncell = nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3, kk = q & 1, second = q >> 1;
  const int mp = warp & 1, np = (warp >> 1) & 1, hf = warp >> 2;
  const int i0 = ti * kT32, j0 = tj * kT32;
  const int c_begin = blockIdx.y * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  double acc[NO][2][2][2];
#pragma unroll
  for (int o = 0; o < NO; ++o)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[o][a][b][0] = acc[o][a][b][1] = 0.0;
  double qacc = 0.0;
  const double* X = pa.X;
  int ca[2], cb[2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    ca[a] = 8 * (2 * mp + a) + g;
    cb[a] = 8 * (2 * np + a) + g;
  }
  // staging item of this thread: cell scl of the chunk, column scol of the
  // i-side tile (i0 + scol) and of the j-side tile (j0 + scol)
  const int scl = threadIdx.x / kT32, scol = threadIdx.x % kT32;
  const int gi = i0 + scol, gj = j0 + scol;
  struct Raw {
    double xi[4], xj[4];
    double y[4];  // group 0: x-left / y-below neighbour edge dofs (j-side); group 1: X_old (i)
    double ui[4];  // group 0: neighbour edge dofs on the i-side (face jumps)
    double qc, st, ss;
  };
  // the item's cell advances by C per chunk: its grid coordinates are kept
  // incrementally (no division per chunk) and every load is a 32-bit offset
  // from one row pointer (r doubles per dof row)
  const bool ci_ok = gi < r, cj_ok = gj < r;
  const int64_t rs = r;
  int fc = c_begin + scl;           // the item's cell at the next fetch
  int fci = fc % nx, fcj = fc / nx;  // its grid coordinates
  auto fetch = [&](int cc0, Raw& w) {
    const int c = fc;
    const int ci = fci, cj = fcj;
    const bool live = cc0 < c_end && c < c_end;
    const double* row = X + (int64_t)c * 4 * rs;  // dof row 4 c
    const bool vi = live && ci_ok, vj = live && cj_ok;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      w.xi[l] = vi ? __ldg(row + l * rs + gi) : 0.0;
      w.xj[l] = vj ? __ldg(row + l * rs + gj) : 0.0;
    }
    if constexpr (GROUP == 0) {
      const bool lx = live && ci > 0, ly = live && (cj > 0 || pa.halo != nullptr);
      const double* left = row - 4 * rs;  // the cell to the left (c - 1)
      const double* below = cj > 0 ? row - (int64_t)4 * nx * rs
                                   : (pa.halo ? pa.halo + (int64_t)ci * 4 * rs : nullptr);
      w.y[0] = (lx && cj_ok) ? __ldg(left + 1 * rs + gj) : 0.0;
      w.y[1] = (lx && cj_ok) ? __ldg(left + 3 * rs + gj) : 0.0;
      w.y[2] = (ly && cj_ok) ? __ldg(below + 2 * rs + gj) : 0.0;
      w.y[3] = (ly && cj_ok) ? __ldg(below + 3 * rs + gj) : 0.0;
      w.ui[0] = (lx && ci_ok) ? __ldg(left + 1 * rs + gi) : 0.0;
      w.ui[1] = (lx && ci_ok) ? __ldg(left + 3 * rs + gi) : 0.0;
      w.ui[2] = (ly && ci_ok) ? __ldg(below + 2 * rs + gi) : 0.0;
      w.ui[3] = (ly && ci_ok) ? __ldg(below + 3 * rs + gi) : 0.0;
    } else {
      const double* orow = pa.Xold ? pa.Xold + (int64_t)c * 4 * rs : nullptr;
#pragma unroll
      for (int l = 0; l < 4; ++l) w.y[l] = (vi && orow) ? __ldg(orow + l * rs + gi) : 0.0;
      w.qc = live ? __ldg(pa.q + c) : 0.0;
      // this staging item's own cell: the sigma-weighted mass planes
      w.st = live ? __ldg(pa.sigma_t + c) : 0.0;
      w.ss = (live && !no_ms) ? __ldg(pa.sigma_s + c) : 0.0;
    }
    // advance to the next chunk's cell
    fc += C;
    fci += C;
    while (fci >= nx) {
      fci -= nx;
      ++fcj;
    }
  };
  Raw cur;
  fetch(c_begin, cur);
  for (int c0 = c_begin; c0 < c_end; c0 += C) {
    const int nc = min(C, c_end - c0);
    __syncthreads();  // the previous chunk's fragments are consumed
    {
      const int base = scl * kRow + scol;
#pragma unroll
      for (int l = 0; l < 4; ++l) sX[base + kLS * l] = cur.xi[l];
      if constexpr (GROUP == 0) {
        const double* x = cur.xj;
        // i-side face jumps u = (left/below neighbour edge) - own edge
        sU[base] = cur.ui[0] - cur.xi[0];
        sU[base + kLS] = cur.ui[1] - cur.xi[2];
        sU[base + 2 * kLS] = cur.ui[2] - cur.xi[0];
        sU[base + 3 * kLS] = cur.ui[3] - cur.xi[1];
        const double ux0 = cur.y[0] - x[0], ux1 = cur.y[1] - x[2];
        const double vx0 = cur.y[0] + x[0], vx1 = cur.y[1] + x[2];
        const double uy0 = cur.y[2] - x[0], uy1 = cur.y[3] - x[1];
        const double vy0 = cur.y[2] + x[0], vy1 = cur.y[3] + x[1];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double gx = 0.0, gy = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            gx = fma(so[16 + 4 * l + p], x[p], gx);
            gy = fma(so[32 + 4 * l + p], x[p], gy);
          }
          sGX[base + kLS * l] = gx;
          sGY[base + kLS * l] = gy;
        }
        double* f = sF + 2 * scl * kRow + scol;
        f[0] = (e2x[0] * vx0 + e2x[1] * vx1);
        f[kLS] = (e2x[2] * vx0 + e2x[3] * vx1);
        f[2 * kLS] = (e2y[0] * vy0 + e2y[1] * vy1);
        f[3 * kLS] = (e2y[2] * vy0 + e2y[3] * vy1);
        f[4 * kLS] = (e2x[0] * ux0 + e2x[1] * ux1);
        f[5 * kLS] = (e2x[2] * ux0 + e2x[3] * ux1);
        f[6 * kLS] = (e2y[0] * uy0 + e2y[1] * uy1);
        f[7 * kLS] = (e2y[2] * uy0 + e2y[3] * uy1);
      } else {
        const double* x = cur.xj;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sXo[base + kLS * l] = cur.y[l];
          double m = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) m = fma(so[4 * l + p], x[p], m);
          sMX[base + kLS * l] = m;
          // sigma folded into the B planes once per staged element (was a
          // scaling of the A fragment per warp per MMA)
          sMXt[base + kLS * l] = cur.st * m;
          if (!no_ms) sMXs[base + kLS * l] = cur.ss * m;
        }
        double sq = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) sq = fma(so[56 + l], x[l], sq);
        sQ[scl * kT32 + scol] = cur.qc * sq;  // q-hat (dlr_sn.py:70)
      }
    }
    __syncthreads();
    fetch(c0 + C, cur);  // next chunk's loads in flight during the MMAs
    // ---- volume terms: the C / 2 cells of this warp's half
#pragma unroll
    for (int k = 0; k < C / 2; ++k) {
      const int cl = hf * (C / 2) + k;
      double xa[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) xa[a] = sX[cl * kRow + q * kLS + ca[a]];
      if constexpr (GROUP == 0) {
        double gx[2], gy[2];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          gx[b] = sGX[cl * kRow + q * kLS + cb[b]];
          gy[b] = sGY[cl * kRow + q * kLS + cb[b]];
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            dmma(acc[0][a][b][0], acc[0][a][b][1], xa[a], gx[b]);  // px (volume)
            dmma(acc[1][a][b][0], acc[1][a][b][1], xa[a], gy[b]);  // py (volume)
          }
      } else {
        double xo[2], mx[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          xo[a] = sXo[cl * kRow + q * kLS + ca[a]];
          mx[a] = sMX[cl * kRow + q * kLS + cb[a]];
        }
        if (!mo_only) {
          double mxt[2];
#pragma unroll
          for (int b = 0; b < 2; ++b) mxt[b] = sMXt[cl * kRow + q * kLS + cb[b]];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) dmma(acc[0][a][b][0], acc[0][a][b][1], xa[a], mxt[b]);  // mt
          if (!no_ms) {
            double mxs[2];
#pragma unroll
            for (int b = 0; b < 2; ++b) mxs[b] = sMXs[cl * kRow + q * kLS + cb[b]];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
              for (int b = 0; b < 2; ++b) dmma(acc[1][a][b][0], acc[1][a][b][1], xa[a], mxs[b]);  // ms
          }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) dmma(acc[2][a][b][0], acc[2][a][b][1], xo[a], mx[b]);  // mo
      }
    }
    if constexpr (GROUP == 0) {
      // ---- face terms: the cell pairs of this half; k slot q -> cell
      // cl + q / 2, face dof q % 2
#pragma unroll
      for (int k = 0; k < C / 4; ++k) {
        const int cl = hf * (C / 2) + 2 * k + second;
        double uxa[2], uya[2], fx[2], fy[2], fux[2], fuy[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          uxa[a] = sU[cl * kRow + kk * kLS + ca[a]];
          uya[a] = sU[cl * kRow + (2 + kk) * kLS + ca[a]];
          const double* f = sF + 2 * cl * kRow + cb[a];
          fx[a] = f[kk * kLS];
          fy[a] = f[(2 + kk) * kLS];
          fux[a] = f[(4 + kk) * kLS];
          fuy[a] = f[(6 + kk) * kLS];
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            dmma(acc[0][a][b][0], acc[0][a][b][1], uxa[a], fx[b]);   // px (faces)
            dmma(acc[1][a][b][0], acc[1][a][b][1], uya[a], fy[b]);   // py (faces)
            dmma(acc[2][a][b][0], acc[2][a][b][1], uxa[a], fux[b]);  // jx
            dmma(acc[3][a][b][0], acc[3][a][b][1], uya[a], fuy[b]);  // jy
          }
      }
    } else {
      if (i0 == 0 && threadIdx.x < kT32)
        for (int cl = 0; cl < nc; ++cl) qacc += sQ[cl * kT32 + threadIdx.x];
    }
  }
  __syncthreads();  // staging planes are dead: reuse them for the reduction
  double* red = sm32;               // [NO][32][33]: half 1's accumulators
  double* bnd = red + NO * 32 * 33;  // [2][32][33]: right / top domain-boundary faces (group 0)
  if constexpr (GROUP == 0) {
    // ---- right / top domain-boundary faces (a = own right/top edge, b = 0)
    for (int e = threadIdx.x; e < kT32 * kT32; e += blockDim.x) {
      const int ti = e >> 5, tj = e & 31;
      const int i = i0 + ti, j = j0 + tj;
      double bx = 0.0, by = 0.0;
      if (i < r && j < r) {
        const int first_right = c_begin + ((nx - 1 - c_begin % nx) % nx + nx) % nx;
        for (int c = first_right; c < c_end; c += nx) {
          const int64_t r1 = (int64_t)c * 4 + 1, r3 = (int64_t)c * 4 + 3;
          const double ai0 = ldx(X, r, r1, i), ai1 = ldx(X, r, r3, i);
          const double aj0 = ldx(X, r, r1, j), aj1 = ldx(X, r, r3, j);
          bx += ai0 * ((e2x[0] * aj0 + e2x[1] * aj1)) + ai1 * ((e2x[2] * aj0 + e2x[3] * aj1));
        }
        for (int c = max(c_begin, (ny - 1) * nx); pa.top_wall && c < c_end; ++c) {
          const int64_t r2 = (int64_t)c * 4 + 2, r3 = (int64_t)c * 4 + 3;
          const double ai0 = ldx(X, r, r2, i), ai1 = ldx(X, r, r3, i);
          const double aj0 = ldx(X, r, r2, j), aj1 = ldx(X, r, r3, j);
          by += ai0 * ((e2y[0] * aj0 + e2y[1] * aj1)) + ai1 * ((e2y[2] * aj0 + e2y[3] * aj1));
        }
      }
      bnd[ti * 33 + tj] = bx;
      bnd[32 * 33 + ti * 33 + tj] = by;
    }
  }
  if (hf == 1) {
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int row = 8 * (2 * mp + a) + g, col = 8 * (2 * np + b) + 2 * q;
          red[(o * 32 + row) * 33 + col] = acc[o][a][b][0];
          red[(o * 32 + row) * 33 + col + 1] = acc[o][a][b][1];
        }
  }
  __syncthreads();
  // ---- fixed-order reduction: (half 0 + half 1) + boundary
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)blockIdx.y * stride;
  if (hf == 0) {
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = 8 * (2 * mp + a) + g, col = 8 * (2 * np + b) + 2 * q + h;
            const int i = i0 + row, j = j0 + col;
            if (i >= r || j >= r) continue;
            double v = acc[o][a][b][h] + red[(o * 32 + row) * 33 + col];
            int slot;
            if constexpr (GROUP == 0) {
              if (o == 0 || o == 2) v += bnd[row * 33 + col];            // px, jx
              if (o == 1 || o == 3) v += bnd[32 * 33 + row * 33 + col];  // py, jy
              slot = o;  // px py jx jy
            } else {
              slot = 4 + o;  // mt ms mo
              if (mo_only && o < 2) continue;
            }
            out[(int64_t)slot * r * r + (int64_t)i * r + j] = v;
          }
  }
  if constexpr (GROUP == 1)
    if (i0 == 0 && threadIdx.x < kT32 && j0 + (int)threadIdx.x < r)
      out[7 * (int64_t)r * r + j0 + threadIdx.x] = qacc;
}

// ---------------------------------------------------------------------------
// K3 on a DIAGONAL 64-column block (columns c0 .. c0 + 63 on both sides).
// One CTA per output group and cell block computes the whole 64 x 64 block:
//  * the i-side and j-side columns coincide, so every X element is staged
//    once (the 32 x 32 tiling stages it in 3 tiles x 2 sides per group);
//  * px, py are skew and jx, jy, mt, ms symmetric, so only the 36 of 64 8x8
//    fragments on and above the diagonal are computed (mirrored after the
//    reduction); the 8 warps hold 5 or 4 of them each (rows a and 7 - a
//    share a warp pair), every warp over all cells of a chunk -- no
//    cross-warp reduction;
//  * mo = X_old^T M X has no symmetry: warp w owns fragment row w.
// Chunks of 4 cells (256 staging items = 4 cells x 64 columns).
constexpr int kPC64 = 4;
constexpr int kLS64 = 68;  // row stride of the staged planes (conflict-free fragments)
// cell strides = 8 mod 16 doubles: the face MMAs read two cells per k-step
// (lanes q >> 1), which must land in different banks
constexpr int kRow64 = 4 * kLS64 + 8;   // [cell][4 rows][kLS]
constexpr int kFace64 = 8 * kLS64 + 8;  // [cell][8 rows][kLS]
constexpr int kPlane64 = kPC64 * kRow64;
constexpr size_t kProj64Smem =
    (4 * (size_t)kPlane64 + std::max(kPC64 * kFace64, kPlane64 + kPC64 * 64)) * sizeof(double);
constexpr int kProjBndBlocks = 32;  // partial slots of the boundary-face kernel

// Fragment pattern of a warp on a diagonal 64-block: rows (a0, a1) x columns
// (b0, b1, b2) of the 8 x 8 fragment grid without the corner (a1, b0):
//   k = 0 (a0, b0)   1 (a0, b1)   2 (a1, b1)   3 (a0, b2)   4 (a1, b2)
// so 2 A and 3 B operands feed 5 MMAs.  The 8 warps' patterns below cover
// the 36 fragments on / above the diagonal exactly once; 4 of the 40 slots
// fall below the diagonal (computed anyway: valid values the mirror pass
// overwrites).  Found by exhaustive search (K3).
__constant__ unsigned char kD64Pat[8][5] = {
    {0, 1, 0, 1, 2}, {0, 1, 3, 4, 5}, {1, 0, 3, 6, 7}, {2, 3, 2, 3, 5},
    {2, 5, 6, 4, 7}, {3, 7, 4, 6, 7}, {5, 4, 5, 4, 6}, {6, 4, 6, 5, 7}};

struct D64Frag {
  int oa0, oa1;       // A operand columns (8 a + g)
  int ob0, ob1, ob2;  // B operand columns (8 b + g)
  unsigned onm;       // PRED: live fragments (ragged last block)
};

// the MMAs of one staged chunk; PRED = per-fragment liveness tests (ragged
// last block, r % 64 != 0)
template <int GROUP, bool PRED>
__device__ __forceinline__ void d64_mma(double (&acc)[GROUP == 0 ? 4 : 2][5][2],
                                        double (&amo)[GROUP == 1 ? 8 : 1][2], const double* sm,
                                        int q, int g, int warp, const D64Frag& fr, bool no_ms,
                                        bool mo_row, int rloc) {
  constexpr int C = kPC64, kLS = kLS64, kRow = kRow64, kFace = kFace64;
  const double* sX = sm;
  const double* sU = sm + kPlane64;
  const double* sXo = sm + kPlane64;
  const double* sGX = sm + 2 * kPlane64;
  const double* sMX = sm + 2 * kPlane64;
  const double* sGY = sm + 3 * kPlane64;
  const double* sMXt = sm + 3 * kPlane64;
  const double* sF = sm + 4 * kPlane64;
  const double* sMXs = sm + 4 * kPlane64;
  const int kk = q & 1, second = q >> 1;
  (void)sU; (void)sXo; (void)sGX; (void)sMX; (void)sGY; (void)sMXt; (void)sF; (void)sMXs;
  (void)kk; (void)second; (void)warp; (void)mo_row; (void)rloc; (void)no_ms; (void)amo;
  // fragment k <- (A operand a[k], B operand b[k]) of the pattern
  auto five = [&](double (&d)[5][2], double a0, double a1, double b0, double b1, double b2) {
    if (!PRED || (fr.onm & 1u)) dmma(d[0][0], d[0][1], a0, b0);
    if (!PRED || (fr.onm & 2u)) dmma(d[1][0], d[1][1], a0, b1);
    if (!PRED || (fr.onm & 4u)) dmma(d[2][0], d[2][1], a1, b1);
    if (!PRED || (fr.onm & 8u)) dmma(d[3][0], d[3][1], a0, b2);
    if (!PRED || (fr.onm & 16u)) dmma(d[4][0], d[4][1], a1, b2);
  };
  // ---- volume terms, every cell of the chunk
#pragma unroll
  for (int cl = 0; cl < C; ++cl) {
    const double* xr = sX + cl * kRow + q * kLS;
    const double x0 = xr[fr.oa0], x1 = xr[fr.oa1];
    if constexpr (GROUP == 0) {
      const double* gxr = sGX + cl * kRow + q * kLS;
      const double* gyr = sGY + cl * kRow + q * kLS;
      five(acc[0], x0, x1, gxr[fr.ob0], gxr[fr.ob1], gxr[fr.ob2]);  // px (volume)
      five(acc[1], x0, x1, gyr[fr.ob0], gyr[fr.ob1], gyr[fr.ob2]);  // py (volume)
    } else {
      const double* mtr = sMXt + cl * kRow + q * kLS;
      const double* msr = sMXs + cl * kRow + q * kLS;
      five(acc[0], x0, x1, mtr[fr.ob0], mtr[fr.ob1], mtr[fr.ob2]);  // mt
      if (!no_ms) five(acc[1], x0, x1, msr[fr.ob0], msr[fr.ob1], msr[fr.ob2]);  // ms
      const double xo = sXo[cl * kRow + q * kLS + 8 * warp + g];
      const double* mr = sMX + cl * kRow + q * kLS + g;
      if (mo_row) {
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          double bm[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) bm[b] = mr[8 * (4 * hb + b)];
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (!PRED || 8 * (4 * hb + b) < rloc)
              dmma(amo[4 * hb + b][0], amo[4 * hb + b][1], xo, bm[b]);  // mo
        }
      }
    }
  }
  if constexpr (GROUP == 0) {
    // ---- face terms: k slot q -> cell 2 kp + q / 2, face dof q % 2
#pragma unroll
    for (int kp = 0; kp < C / 2; ++kp) {
      const int cl = 2 * kp + second;
      const double* ur = sU + cl * kRow + kk * kLS;
      const double* f = sF + cl * kFace + kk * kLS;
      const double ux0 = ur[fr.oa0], ux1 = ur[fr.oa1];
      five(acc[0], ux0, ux1, f[fr.ob0], f[fr.ob1], f[fr.ob2]);  // px (faces)
      five(acc[2], ux0, ux1, f[4 * kLS + fr.ob0], f[4 * kLS + fr.ob1], f[4 * kLS + fr.ob2]);  // jx
      const double uy0 = ur[2 * kLS + fr.oa0], uy1 = ur[2 * kLS + fr.oa1];
      five(acc[1], uy0, uy1, f[2 * kLS + fr.ob0], f[2 * kLS + fr.ob1], f[2 * kLS + fr.ob2]);  // py
      five(acc[3], uy0, uy1, f[6 * kLS + fr.ob0], f[6 * kLS + fr.ob1], f[6 * kLS + fr.ob2]);  // jy
    }
  }
}

template <int GROUP>
__device__ __forceinline__ void project64d_group(const ProjArgs& pa, const dlrsn_cellops& ops,
                                                 double* sm, int t64) {
  constexpr int C = kPC64, kLS = kLS64, kRow = kRow64;
  constexpr int NS = GROUP == 0 ? 4 : 2;  // symmetric / skew outputs of the group
  double* sX = sm;
  double* sU = sm + kPlane64;        // group 0: face jumps
  double* sXo = sm + kPlane64;       // group 1: X_old
  double* sGX = sm + 2 * kPlane64;   // group 0
  double* sMX = sm + 2 * kPlane64;   // group 1
  double* sGY = sm + 3 * kPlane64;   // group 0
  double* sMXt = sm + 3 * kPlane64;  // group 1
  double* sF = sm + 4 * kPlane64;    // group 0: [C][kFace64]
  double* sMXs = sm + 4 * kPlane64;  // group 1
  double* sQ = sm + 5 * kPlane64;    // group 1: [C][64]
  constexpr int kFace = kFace64;
  __shared__ double so[64];
  if (threadIdx.x < 16) {
    so[threadIdx.x] = ops.mass[threadIdx.x];
    so[16 + threadIdx.x] = ops.gx[threadIdx.x];
    so[32 + threadIdx.x] = ops.gy[threadIdx.x];
  } else if (threadIdx.x < 20) {
    so[48 + threadIdx.x - 16] = 0.5 * ops.e2x[threadIdx.x - 16];
    so[52 + threadIdx.x - 16] = 0.5 * ops.e2y[threadIdx.x - 16];
    so[56 + threadIdx.x - 16] = ops.src_row[threadIdx.x - 16];
  }
  const double* e2x = so + 48;
  const double* e2y = so + 52;
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const bool no_ms = pa.sigma_s == nullptr || (pa.any_scat != nullptr && *pa.any_scat == 0);
  const int ncell = nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int col0 = 64 * t64;
  const int rloc = min(64, r - col0);  // live columns of this block
  const int c_begin = blockIdx.y * pa.cells_per_block;
  const int c_end = min(ncell, c_begin + pa.cells_per_block);
  // this warp's fragment pattern (kD64Pat): per fragment k its fragment row
  // fa[k] and column fb[k] are recomputed from the table where needed
  const int pa0 = kD64Pat[warp][0], pa1 = kD64Pat[warp][1];
  const int pb0 = kD64Pat[warp][2], pb1 = kD64Pat[warp][3], pb2 = kD64Pat[warp][4];
  D64Frag fr;
  fr.oa0 = 8 * pa0 + g;
  fr.oa1 = 8 * pa1 + g;
  fr.ob0 = 8 * pb0 + g;
  fr.ob1 = 8 * pb1 + g;
  fr.ob2 = 8 * pb2 + g;
  {
    const int ra[5] = {pa0, pa0, pa1, pa0, pa1}, cb[5] = {pb0, pb1, pb1, pb2, pb2};
    fr.onm = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (8 * ra[k] < rloc && 8 * cb[k] < rloc) fr.onm |= 1u << k;
  }
  double acc[NS][5][2];
#pragma unroll
  for (int o = 0; o < NS; ++o)
#pragma unroll
    for (int k = 0; k < 5; ++k) acc[o][k][0] = acc[o][k][1] = 0.0;
  double amo[GROUP == 1 ? 8 : 1][2];
#pragma unroll
  for (int b = 0; b < (GROUP == 1 ? 8 : 1); ++b) amo[b][0] = amo[b][1] = 0.0;
  const bool mo_row = 8 * warp < rloc;
  double qacc = 0.0;
  const double* X = pa.X;
  // staging item of this thread: cell scl of the chunk, column col0 + scol
  const int scl = threadIdx.x >> 6, scol = threadIdx.x & 63;
  const int gc = col0 + scol;
  const bool c_ok = gc < r;
  const int64_t rs = r;
  struct Raw {
    double x[4];
    double y[4];  // group 0: left / below neighbour edge dofs; group 1: X_old
    double qc, st, ss;
  };
  int fc = c_begin + scl;
  int fci = fc % nx, fcj = fc / nx;
  auto fetch = [&](int cc0, Raw& w) {
    const int c = fc;
    const int ci = fci, cj = fcj;
    const bool live = cc0 < c_end && c < c_end;
    const double* row = X + (int64_t)c * 4 * rs;
    const bool v = live && c_ok;
#pragma unroll
    for (int l = 0; l < 4; ++l) w.x[l] = v ? __ldg(row + l * rs + gc) : 0.0;
    if constexpr (GROUP == 0) {
      const bool lx = v && ci > 0, ly = v && (cj > 0 || pa.halo != nullptr);
      const double* left = row - 4 * rs;
      const double* below = cj > 0 ? row - (int64_t)4 * nx * rs
                                   : (pa.halo ? pa.halo + (int64_t)ci * 4 * rs : nullptr);
      w.y[0] = lx ? __ldg(left + 1 * rs + gc) : 0.0;
      w.y[1] = lx ? __ldg(left + 3 * rs + gc) : 0.0;
      w.y[2] = ly ? __ldg(below + 2 * rs + gc) : 0.0;
      w.y[3] = ly ? __ldg(below + 3 * rs + gc) : 0.0;
    } else {
      const double* orow = pa.Xold ? pa.Xold + (int64_t)c * 4 * rs : nullptr;
#pragma unroll
      for (int l = 0; l < 4; ++l) w.y[l] = (v && orow) ? __ldg(orow + l * rs + gc) : 0.0;
      w.qc = live ? __ldg(pa.q + c) : 0.0;
      w.st = live ? __ldg(pa.sigma_t + c) : 0.0;
      w.ss = (live && !no_ms) ? __ldg(pa.sigma_s + c) : 0.0;
    }
    fc += C;
    fci += C;
    while (fci >= nx) {
      fci -= nx;
      ++fcj;
    }
  };
  Raw cur;
  fetch(c_begin, cur);
  for (int c0 = c_begin; c0 < c_end; c0 += C) {
    const int nc = min(C, c_end - c0);
    __syncthreads();  // the previous chunk's fragments are consumed
    {
      const int base = scl * kRow + scol;
      const double* x = cur.x;
#pragma unroll
      for (int l = 0; l < 4; ++l) sX[base + kLS * l] = x[l];
      if constexpr (GROUP == 0) {
        const double ux0 = cur.y[0] - x[0], ux1 = cur.y[1] - x[2];
        const double vx0 = cur.y[0] + x[0], vx1 = cur.y[1] + x[2];
        const double uy0 = cur.y[2] - x[0], uy1 = cur.y[3] - x[1];
        const double vy0 = cur.y[2] + x[0], vy1 = cur.y[3] + x[1];
        sU[base] = ux0;
        sU[base + kLS] = ux1;
        sU[base + 2 * kLS] = uy0;
        sU[base + 3 * kLS] = uy1;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double gx = 0.0, gy = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            gx = fma(so[16 + 4 * l + p], x[p], gx);
            gy = fma(so[32 + 4 * l + p], x[p], gy);
          }
          sGX[base + kLS * l] = gx;
          sGY[base + kLS * l] = gy;
        }
        double* f = sF + scl * kFace + scol;
        f[0] = (e2x[0] * vx0 + e2x[1] * vx1);
        f[kLS] = (e2x[2] * vx0 + e2x[3] * vx1);
        f[2 * kLS] = (e2y[0] * vy0 + e2y[1] * vy1);
        f[3 * kLS] = (e2y[2] * vy0 + e2y[3] * vy1);
        f[4 * kLS] = (e2x[0] * ux0 + e2x[1] * ux1);
        f[5 * kLS] = (e2x[2] * ux0 + e2x[3] * ux1);
        f[6 * kLS] = (e2y[0] * uy0 + e2y[1] * uy1);
        f[7 * kLS] = (e2y[2] * uy0 + e2y[3] * uy1);
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          sXo[base + kLS * l] = cur.y[l];
          double m = 0.0;
#pragma unroll
          for (int p = 0; p < 4; ++p) m = fma(so[4 * l + p], x[p], m);
          sMX[base + kLS * l] = m;
          sMXt[base + kLS * l] = cur.st * m;
          if (!no_ms) sMXs[base + kLS * l] = cur.ss * m;
        }
        double sq = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) sq = fma(so[56 + l], x[l], sq);
        sQ[scl * 64 + scol] = cur.qc * sq;  // q-hat (dlr_sn.py:70)
      }
    }
    __syncthreads();
    fetch(c0 + C, cur);  // next chunk's loads in flight during the MMAs
    // ---- the chunk's MMAs (volume terms of every cell, then the faces)
    if (rloc == 64)
      d64_mma<GROUP, false>(acc, amo, sm, q, g, warp, fr, no_ms, mo_row, rloc);
    else
      d64_mma<GROUP, true>(acc, amo, sm, q, g, warp, fr, no_ms, mo_row, rloc);
    if constexpr (GROUP == 1) {
      if (threadIdx.x < 64)
        for (int cl = 0; cl < nc; ++cl) qacc += sQ[cl * 64 + threadIdx.x];
    }

  }
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)blockIdx.y * stride;
  // (the right / top domain-boundary faces of the diagonal blocks are added
  // by project_bnd64_kernel into partial slots of their own)
  {
    const int ra[5] = {pa0, pa0, pa1, pa0, pa1}, cb[5] = {pb0, pb1, pb1, pb2, pb2};
#pragma unroll
    for (int o = 0; o < NS; ++o)
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        if (!((fr.onm >> k) & 1u)) continue;
        const int i = col0 + 8 * ra[k] + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = col0 + 8 * cb[k] + 2 * q + h;
          if (i >= r || j >= r) continue;
          const int slot = GROUP == 0 ? o : 4 + o;  // px py jx jy | mt ms
          out[(int64_t)slot * r * r + (int64_t)i * r + j] = acc[o][k][h];
        }
      }
  }
  if constexpr (GROUP == 1) {
    if (mo_row) {
      const int i = col0 + 8 * warp + g;
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = col0 + 8 * b + 2 * q + h;
          if (i < r && j < r) out[6 * (int64_t)r * r + (int64_t)i * r + j] = amo[b][h];
        }
    }
    if (threadIdx.x < 64 && col0 + (int)threadIdx.x < r)
      out[7 * (int64_t)r * r + col0 + threadIdx.x] = qacc;
  }
}

// Symmetric Gram G = X^T M X for 32 < r <= 64 with the diagonal-block K3's
// layout: one CTA per cell range, every X element staged once from
// registers together with M x (no separate premultiply pass: two barriers
// per chunk), the 8 warps' 2 x 3-minus-corner fragment patterns (kD64Pat)
// over all cells of a chunk -- no cross-warp reduction.  Chunks of 16 cells
// (4 staging items per thread).  Columns >= r are staged as zeros.
constexpr int kGC = 16;
constexpr size_t kMgram64sSmem = 2 * (size_t)kGC * kRow64 * sizeof(double);

__global__ void __launch_bounds__(256, 2) mgram64s_kernel(int ncell, int r,
                                                          const double* __restrict__ X, int ldx,
                                                          dlrsn_cellops ops, int cells_per_block,
                                                          double* __restrict__ part) {
  constexpr int kLS = kLS64, kRow = kRow64;
  extern __shared__ __align__(16) double smg[];
  double* sX = smg;
  double* sMX = smg + kGC * kRow;
  __shared__ double sm_m[16];
  if (threadIdx.x < 16) sm_m[threadIdx.x] = ops.mass[threadIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int pa0 = kD64Pat[warp][0], pa1 = kD64Pat[warp][1];
  const int pb0 = kD64Pat[warp][2], pb1 = kD64Pat[warp][3], pb2 = kD64Pat[warp][4];
  const int oa0 = 8 * pa0 + g, oa1 = 8 * pa1 + g;
  const int ob0 = 8 * pb0 + g, ob1 = 8 * pb1 + g, ob2 = 8 * pb2 + g;
  const int c_begin = blockIdx.x * cells_per_block;
  const int c_end = min(ncell, c_begin + cells_per_block);
  const int scl = threadIdx.x >> 6, scol = threadIdx.x & 63;
  const bool c_ok = scol < r;
  double acc[5][2];
#pragma unroll
  for (int k = 0; k < 5; ++k) acc[k][0] = acc[k][1] = 0.0;
  // the slot entries no fragment pattern covers (below the diagonal) stay
  // zero; the mirror pass fills them after the reduction
  for (int e = threadIdx.x; e < r * r; e += 256) part[(int64_t)blockIdx.x * r * r + e] = 0.0;
  double raw[4][4];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int c = c0 + scl + 4 * m;
      const bool live = c_ok && c < c_end;
      const double* row = X + (int64_t)c * 4 * ldx + scol;
#pragma unroll
      for (int l = 0; l < 4; ++l) raw[m][l] = live ? __ldg(row + (int64_t)l * ldx) : 0.0;
    }
  };
  fetch(c_begin);
  for (int c0 = c_begin; c0 < c_end; c0 += kGC) {
    __syncthreads();  // the previous chunk's fragments are consumed
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int base = (scl + 4 * m) * kRow + scol;
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        sX[base + kLS * l] = raw[m][l];
        double v = 0.0;
#pragma unroll
        for (int p2 = 0; p2 < 4; ++p2) v = fma(sm_m[4 * l + p2], raw[m][p2], v);
        sMX[base + kLS * l] = v;
      }
    }
    __syncthreads();
    fetch(c0 + kGC);  // next chunk's loads in flight during the MMAs
#pragma unroll
    for (int cl = 0; cl < kGC; ++cl) {
      const double* xr = sX + cl * kRow + q * kLS;
      const double* mr = sMX + cl * kRow + q * kLS;
      const double x0 = xr[oa0], x1 = xr[oa1];
      const double b0 = mr[ob0], b1 = mr[ob1], b2 = mr[ob2];
      dmma(acc[0][0], acc[0][1], x0, b0);
      dmma(acc[1][0], acc[1][1], x0, b1);
      dmma(acc[2][0], acc[2][1], x1, b1);
      dmma(acc[3][0], acc[3][1], x0, b2);
      dmma(acc[4][0], acc[4][1], x1, b2);
    }
  }
  __syncthreads();  // the zero fill above precedes every fragment store
  double* out = part + (int64_t)blockIdx.x * r * r;
  const int ra[5] = {pa0, pa0, pa1, pa0, pa1}, cb[5] = {pb0, pb1, pb1, pb2, pb2};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int i = 8 * ra[k] + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = 8 * cb[k] + 2 * q + h;
      if (i < r && j < r) out[(int64_t)i * r + j] = acc[k][h];
    }
  }
}

// Right / top domain-boundary faces of the diagonal 64-blocks (own right /
// top edge against a zero exterior): X_e^T (1/2 e2) X_e per boundary cell,
// added to px, jx (right wall) and py, jy (top wall).  The boundary cells
// (ny right-wall cells, then nx top-wall cells when top_wall) are split over
// gridDim.x CTAs, each writing one partial slot (slot_base + blockIdx.x).
__global__ void __launch_bounds__(256) project_bnd64_kernel(ProjArgs pa, dlrsn_cellops ops,
                                                            int nb64, int slot_base) {
  __shared__ double sa[2][64];
  const int r = pa.r, nx = pa.nx, ny = pa.ny;
  const int nright = ny, ntop = pa.top_wall ? nx : 0, total = nright + ntop;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(total, b0 + per);
  const int64_t stride = 7 * (int64_t)r * r + r;
  double* out = pa.part + (int64_t)(slot_base + blockIdx.x) * stride;
  for (int blk = 0; blk < nb64; ++blk) {
    const int col0 = 64 * blk;
    double ax[16], ay[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) ax[e] = ay[e] = 0.0;
    for (int bc = b0; bc < b1; ++bc) {
      const bool right = bc < nright;
      const int c = right ? bc * nx + nx - 1 : (ny - 1) * nx + (bc - nright);
      const int d0 = right ? 1 : 2;  // edge dofs: right (1, 3), top (2, 3)
      __syncthreads();
      if (threadIdx.x < 128) {
        const int w = threadIdx.x >> 6, col = col0 + (threadIdx.x & 63);
        sa[w][threadIdx.x & 63] = ldx(pa.X, r, (int64_t)c * 4 + (w ? 3 : d0), col);
      }
      __syncthreads();
      const double* e2 = right ? ops.e2x : ops.e2y;
      const double e00 = 0.5 * e2[0], e01 = 0.5 * e2[1], e10 = 0.5 * e2[2], e11 = 0.5 * e2[3];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int idx = threadIdx.x + 256 * e, i = idx >> 6, j = idx & 63;
        const double v = sa[0][i] * (e00 * sa[0][j] + e01 * sa[1][j]) +
                         sa[1][i] * (e10 * sa[0][j] + e11 * sa[1][j]);
        if (right) ax[e] += v;
        else ay[e] += v;
      }
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int idx = threadIdx.x + 256 * e, i = col0 + (idx >> 6), j = col0 + (idx & 63);
      if (i >= r || j >= r) continue;
      const int64_t o = (int64_t)i * r + j;
      out[o] = ax[e];                           // px
      out[2 * (int64_t)r * r + o] = ax[e];      // jx
      out[(int64_t)r * r + o] = ay[e];          // py
      out[3 * (int64_t)r * r + o] = ay[e];      // jy
    }
  }
}

// The (group, tile) work list of one cell block.  px, py are skew- and jx,
// jy, mt, ms symmetric (X^T A X with A = -A^T or A = A^T: Px, Py skew, Jx,
// Jy, M_sigma symmetric, transport_sn.py:246-282), so only the tiles on and
// above the diagonal are computed for them and the reduced result is
// mirrored (mirror_tiles_kernel); mo = X_old^T M X has no symmetry, so the
// tiles below the diagonal run group 1 in mo-only mode.  With diagonal
// 64-column blocks (project64d_group, r > 32) the diagonal blocks are one
// CTA per group and only the off-diagonal 64-blocks use 32 x 32 tiles.
// CTA per group (project_mma64d_kernel) and only the off-diagonal 64-blocks
// are in this list.  Entry = kind (0 / 1 = group, 2 = mo only) | ti << 3 | tj << 5.
struct ProjTiles {
  int n;
  unsigned char e[64];
};

// grid (work list, cell blocks): all groups / tiles of one cell block are
// adjacent in launch order, so they run together and read that block's X
// rows from DRAM once (L2 shares them)
__global__ void __launch_bounds__(256, 2) project_mma32g_kernel(ProjArgs pa, dlrsn_cellops ops,
                                                                 ProjTiles tl) {
  extern __shared__ __align__(16) double sm32g[];
  const int e = tl.e[blockIdx.x];
  const int grp = e & 7, ti = (e >> 3) & 3, tj = (e >> 5) & 3;
  if (grp == 0)
    project32_group<0>(pa, ops, sm32g, ti, tj, false);
  else
    project32_group<1>(pa, ops, sm32g, ti, tj, grp == 2);
}

// the diagonal 64-column blocks: grid (2 x blocks, cell blocks), group =
// blockIdx.x & 1 (the two groups of a cell block are adjacent: shared X rows)
// seq = 1: grid (1, cell ranges), every CTA runs both groups of every
// diagonal block on its range one after the other -- identical work per
// CTA, so 2 x SM-count equal ranges are balanced without a tail
__global__ void __launch_bounds__(256, 2) project_mma64d_kernel(ProjArgs pa, dlrsn_cellops ops,
                                                                 int nb64, int seq) {
  extern __shared__ __align__(16) double sm64d[];
  (void)seq;
  for (int b = 0; b < nb64; ++b) {
    project64d_group<0>(pa, ops, sm64d, b);
    __syncthreads();
    project64d_group<1>(pa, ops, sm64d, b);
    __syncthreads();
  }
}

// out[o][i][j] = s_o out[o][j][i] below the diagonal tiles (o < 6; s = -1
// for the skew px, py)
__global__ void mirror_tiles_kernel(int r, double* __restrict__ out, int d64) {
  const int64_t total = 6 * (int64_t)r * r;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / ((int64_t)r * r));
    const int rem = (int)(e - (int64_t)o * r * r);
    const int i = rem / r, j = rem % r;
    // computed: 32 x 32 tiles on / above the diagonal; with diagonal 64-blocks
    // the 8 x 8 fragments on / above the diagonal inside them
    const bool low = d64 ? ((i >> 6) > (j >> 6) || ((i >> 6) == (j >> 6) && (i >> 3) > (j >> 3)))
                         : (i / kT32 > j / kT32);
    if (!low) continue;
    const double v = out[(int64_t)o * r * r + (int64_t)j * r + i];
    out[e] = o < 2 ? -v : v;
  }
}

// ---------------------------------------------------------------------------
// Small dense kernels: one CTA, matrices in global memory (L2 resident).

// Cholesky G = R^T R (R upper) and Rinv = R^-1 (upper).  flag[0] = 1 if a
// pivot is not positive; diag_ratio[k] = R_kk / max(sqrt(G_kk), 1) (the
// reference's deficiency test quantity, angular.py:137).
__global__ void chol_upper_kernel(int r, const double* __restrict__ G, double* __restrict__ R,
                                  double* Rinv, double* __restrict__ diag_ratio, int* flag,
                                  int inv_in_global) {
  extern __shared__ double sm[];
  double* a = sm;          // r*r working copy (becomes R)
  // r > 110: the inverse is built in place in Rinv (global, L2-resident)
  double* inv = inv_in_global ? Rinv : sm + r * r;
  __shared__ double gdiag[DLRSN_MAX_RANK];  // G_kk (the deficiency test's norms)
  __shared__ double rdiag[DLRSN_MAX_RANK];  // 1 / R_kk (0 for a failed pivot)
  __shared__ int bad;
  const int tid = threadIdx.x, bs = blockDim.x;
  for (int e = tid; e < r * r; e += bs) {
    const int i = e / r, j = e % r;
    const double g = G[e];
    a[e] = g;
    inv[e] = i == j ? 1.0 : 0.0;
    if (i == j) gdiag[i] = g;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  // Two barriers per column: (A) every thread reads the pivot and scales
  // its part of row k; (B) the trailing update of the upper part, and the
  // pivot's own entries written by thread 0.
  const int warp = tid >> 5, lane = tid & 31, nw = bs >> 5;
  for (int k = 0; k < r; ++k) {
    const double d = a[k * r + k];
    const bool ok = d > 0.0;
    const double rkk = ok ? sqrt(d) : 0.0;
    for (int j = k + 1 + tid; j < r; j += bs) a[k * r + j] = rkk > 0 ? a[k * r + j] / rkk : 0.0;
    __syncthreads();
    if (tid == 0) {
      a[k * r + k] = rkk;
      rdiag[k] = ok ? 1.0 / rkk : 0.0;
      if (!ok) bad = 1;
      const double on = sqrt(fmax(gdiag[k], 0.0));
      diag_ratio[k] = ok && on > 0.0 ? rkk / on : 0.0;
      diag_ratio[r + k] = ok ? rkk / fmax(on, 1.0) : 0.0;
    }
    // a[i][j] -= a[k][i] a[k][j] for k < i <= j (a warp per row)
    for (int i = k + 1 + warp; i < r; i += nw) {
      const double aki = a[k * r + i];
      for (int j = i + lane; j < r; j += 32) a[i * r + j] -= aki * a[k * r + j];
    }
    __syncthreads();
  }
  // R: zero the strict lower part
  for (int e = tid; e < r * r; e += bs) {
    const int i = e / r, j = e % r;
    R[e] = j >= i ? a[e] : 0.0;
  }
  // R^-1 by right-looking back substitution on B = I: at step k, row k of
  // the inverse is final; rows i < k lose column k's contribution, and row
  // k - 1 (whose last update this is) is scaled by 1 / R_{k-1,k-1}.  One
  // barrier per column.
  if (tid == 0) inv[(r - 1) * r + r - 1] *= rdiag[r - 1];
  __syncthreads();
  for (int k = r - 1; k >= 1; --k) {
    const int cols = r - k;
    const double rk1 = rdiag[k - 1];
    for (int e = tid; e <= k * cols; e += bs) {
      if (e == k * cols) {
        inv[(k - 1) * r + k - 1] *= rk1;
        continue;
      }
      const int i = e / cols, j = k + e % cols;
      double v = inv[i * r + j] - a[i * r + k] * inv[k * r + j];
      if (i == k - 1) v *= rk1;
      inv[i * r + j] = v;
    }
    __syncthreads();
  }
  if (!inv_in_global)
    for (int e = tid; e < r * r; e += bs) Rinv[e] = inv[e];
  if (tid == 0 && flag) *flag = bad;
}

// Asynchronous global -> shared copies (LDGSTS): a single-CTA kernel issues
// all its loads at once and pays the memory latency one time.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Register-resident single-warp Cholesky G = R^T R (R upper), r <= RT <= 32:
// lane j holds column j (c[i] = G[i][j] on entry, R[i][j] on exit); row k
// entries of other columns arrive by shuffles.  Same operation order as the
// shared-memory version.  inv returns column j of R^-1.
template <int RT>
__device__ int warp_chol_reg(int r, double (&c)[RT], double (&inv)[RT]) {
  const int lane = threadIdx.x & 31;
  int bad = 0;
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    if (k < r) {
      const double d = __shfl_sync(kFull, c[k], k);
      const bool ok = d > 0.0;
      bad |= !ok;
      const double rkk = ok ? sqrt(d) : 0.0;
      if (lane == k) c[k] = rkk;
      else if (lane > k) c[k] = rkk > 0.0 ? c[k] / rkk : 0.0;
#pragma unroll
      for (int i = k + 1; i < RT; ++i) {
        const double aki = __shfl_sync(kFull, c[k], i);
        if (i < r && i <= lane) c[i] -= aki * c[k];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RT; ++i)
    if (i > lane) c[i] = 0.0;  // strict lower part of R
  // R^-1 column j = lane by back substitution; R[i][p] = lane p's c[i].
  // The reciprocals of the diagonal are formed up front, in parallel (lane i
  // owns 1 / R_ii), so the substitution chain carries no division.
  double rd = 0.0;
#pragma unroll
  for (int i = 0; i < RT; ++i)
    if (i == lane) rd = c[i];
  const double rinv_own = (lane < r && rd > 0.0) ? 1.0 / rd : 0.0;
#pragma unroll
  for (int i = RT - 1; i >= 0; --i) {
    double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int p = i + 1; p < RT; ++p) {
      const double rip = __shfl_sync(kFull, c[i], p);
      if (p <= lane && p < r) s -= rip * inv[p];
    }
    const double ri = __shfl_sync(kFull, rinv_own, i);
    inv[i] = (i <= lane && i < r) ? s * ri : 0.0;
  }
  return bad;
}

// Single-warp Cholesky G = R^T R (R upper, r <= 32) on a shared copy `a`
// (row-major, becomes R) and R^-1 into `inv`; lane j owns column j, so only
// __syncwarp is needed.  Same operation order as chol_upper_kernel.
// ratio (optional, 2r): R_kk / sqrt(G_kk) and R_kk / max(sqrt(G_kk), 1).
__device__ int warp_chol_inv(int r, double* a, double* inv, double* ratio) {
  const int lane = threadIdx.x & 31;
  int bad = 0;
  for (int k = 0; k < r; ++k) {
    const double g = a[k * r + k];
    const double d = g;  // a[k][k] already holds the updated pivot
    const bool ok = d > 0.0;
    bad |= !ok;
    const double rkk = ok ? sqrt(d) : 0.0;
    __syncwarp();
    if (lane == k) a[k * r + k] = rkk;
    if (lane > k && lane < r) a[k * r + lane] = rkk > 0.0 ? a[k * r + lane] / rkk : 0.0;
    __syncwarp();
    if (lane > k && lane < r) {
      const double akj = a[k * r + lane];
      for (int i = k + 1; i <= lane; ++i) a[i * r + lane] -= a[k * r + i] * akj;
    }
    __syncwarp();
  }
  // inverse by columns: back substitution R x = e_j
  if (lane < r) {
    const int j = lane;
    for (int i = r - 1; i > j; --i) inv[i * r + j] = 0.0;
    for (int i = j; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int p = i + 1; p <= j; ++p) s -= a[i * r + p] * inv[p * r + j];
      const double dd = a[i * r + i];
      inv[i * r + j] = dd > 0.0 ? s / dd : 0.0;
    }
    for (int i = j + 1; i < r; ++i) a[i * r + j] = 0.0;  // R: zero the strict lower part
  }
  __syncwarp();
  return bad;
}

// chol_upper for r <= 32: one warp, registers only
template <int RT>
__global__ void chol_upper_warp_kernel(int r, const double* __restrict__ G, double* __restrict__ R,
                                       double* __restrict__ Rinv, double* __restrict__ diag_ratio,
                                       int* flag) {
  const int lane = threadIdx.x;
  double c[RT], inv[RT];
#pragma unroll
  for (int i = 0; i < RT; ++i) c[i] = (i < r && lane < r) ? __ldg(G + i * r + lane) : 0.0;
  const double gkk = lane < r ? __ldg(G + lane * r + lane) : 0.0;
  const int bad = warp_chol_reg<RT>(r, c, inv);
  if (lane < r) {
#pragma unroll
    for (int i = 0; i < RT; ++i)
      if (i < r) {
        R[i * r + lane] = c[i];
        Rinv[i * r + lane] = inv[i];
      }
    if (diag_ratio) {
      double rkk = 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i)
        if (i == lane) rkk = c[i];
      const double on = sqrt(fmax(gkk, 0.0));
      diag_ratio[lane] = (rkk > 0.0 && on > 0.0) ? rkk / on : 0.0;
      diag_ratio[r + lane] = rkk > 0.0 ? rkk / fmax(on, 1.0) : 0.0;
    }
  }
  if (lane == 0 && flag) *flag = bad;
}

// Weighted CholQR2 of a small tall matrix held in shared memory (the angular
// basis update, angular.py:217-238, full-rank case): Q = W R^-1 with
// W^T diag(w) W = R^T R, applied twice; R = R2 R1.  The Gram and the row
// update run on the FP64 tensor cores (DMMA m8n8k4) over MT-padded tiles;
// the Cholesky is one warp, in registers.  ratio/flag feed the same guard as
// the spatial CholQR2 (a failed guard reruns the exact CGS2).
template <int MT>
__global__ void __launch_bounds__(256) cholqr2_small_kernel(int n, int m,
                                                            const double* __restrict__ Win,
                                                            int ldw, const double* __restrict__ w,
                                                            double* __restrict__ Q, int ldq,
                                                            double* __restrict__ R,
                                                            double* __restrict__ ratio,
                                                            int* flag, int* deficient) {
  constexpr int NT = MT / 8, KS = MT / 4, LQ = MT + 1;  // odd stride: conflict-free fragments
  extern __shared__ double sm[];
  const int np = (n + 7) & ~7;               // rows padded to whole 8-row tiles
  double* A = sm;                            // np x LQ (zero padded)
  double* ws = A + (size_t)np * LQ;          // np weights (zero padded)
  double* G = ws + np;                       // MT x MT (becomes R of the pass)
  double* inv = G + MT * MT;                 // MT x MT
  double* R1 = inv + MT * MT;                // MT x MT
  double* red = R1 + MT * MT;                // 8 warps x MT x MT
  __shared__ int bad_s[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  for (int e = threadIdx.x; e < np * LQ; e += blockDim.x) {
    const int row = e / LQ, col = e - row * LQ;
    if (row < n && col < m) cp_async8(A + e, Win + (int64_t)row * ldw + col);
    else A[e] = 0.0;
  }
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    if (e < n) cp_async8(ws + e, w + e);
    else ws[e] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    // ---- Gram G = A^T diag(w) A: warp `wid` takes row quads wid, wid + nw, ...
    double d[NT][NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) d[i][j][0] = d[i][j][1] = 0.0;
    for (int k0 = 4 * wid; k0 < np; k0 += 4 * nw) {
      const double* arow = A + (k0 + q) * LQ;
      const double wk = ws[k0 + q];
      double af[NT], bf[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        af[t] = arow[8 * t + g];
        bf[t] = wk * af[t];
      }
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(d[i][j][0], d[i][j][1], af[i], bf[j]);
    }
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        red[(wid * MT + 8 * i + g) * MT + 8 * j + 2 * q] = d[i][j][0];
        red[(wid * MT + 8 * i + g) * MT + 8 * j + 2 * q + 1] = d[i][j][1];
      }
    __syncthreads();
    for (int e = threadIdx.x; e < MT * MT; e += blockDim.x) {
      double acc = 0.0;
      for (int ww = 0; ww < nw; ++ww) acc += red[ww * MT * MT + e];
      G[e] = acc;
    }
    __syncthreads();
    // ---- Cholesky + inverse (one warp, registers)
    if (wid == 0) {
      double c[MT], iv[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) c[i] = (i < m && lane < m) ? G[i * MT + lane] : 0.0;
      const double gkk = lane < m ? G[lane * MT + lane] : 0.0;
      const int bad = warp_chol_reg<MT>(m, c, iv);
      __syncwarp();
      if (lane < MT) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          G[i * MT + lane] = lane < m ? c[i] : 0.0;
          inv[i * MT + lane] = lane < m ? iv[i] : 0.0;
        }
      }
      if (lane == 0) bad_s[pass] = bad;
      if (pass == 0 && lane < m) {
        double rkk = 0.0;
#pragma unroll
        for (int i = 0; i < MT; ++i)
          if (i == lane) rkk = c[i];
        const double on = sqrt(fmax(gkk, 0.0));
        ratio[lane] = (rkk > 0.0 && on > 0.0) ? rkk / on : 0.0;
        ratio[m + lane] = rkk > 0.0 ? rkk / fmax(on, 1.0) : 0.0;
      }
    }
    __syncthreads();
    // ---- A = A R^-1 by 8-row tiles (DMMA), in place
    {
      double bf[KS][NT];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int t = 0; t < NT; ++t) bf[ks][t] = inv[(4 * ks + q) * MT + 8 * t + g];
      for (int r0 = 8 * wid; r0 < np; r0 += 8 * nw) {
        double af[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) af[ks] = A[(r0 + g) * LQ + 4 * ks + q];
        double dd[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) dd[t][0] = dd[t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma(dd[t][0], dd[t][1], af[ks], bf[ks][t]);
        __syncwarp();  // every lane has read the tile before it is overwritten
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          A[(r0 + g) * LQ + 8 * t + 2 * q] = dd[t][0];
          A[(r0 + g) * LQ + 8 * t + 2 * q + 1] = dd[t][1];
        }
      }
    }
    if (pass == 0)
      for (int e = threadIdx.x; e < MT * MT; e += blockDim.x) R1[e] = G[e];
    __syncthreads();
  }
  // R = R2 R1 (both upper)
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    double acc = 0.0;
    for (int p = i; p <= j; ++p) acc = fma(G[i * MT + p], R1[p * MT + j], acc);
    R[e] = j >= i ? acc : 0.0;
  }
  // (compile-time column count: no 64-bit division by the runtime m, which
  // compiles to a slow-path subroutine call per element)
  for (int e = threadIdx.x; e < n * MT; e += blockDim.x) {
    const int row = e / MT, col = e % MT;
    if (col < m) Q[(int64_t)row * ldq + col] = A[row * LQ + col];
  }
  for (int k = threadIdx.x; k < m; k += blockDim.x) deficient[k] = 0;
  if (threadIdx.x == 0) {
    flag[0] = bad_s[0];
    flag[1] = bad_s[1];
  }
}

// C = A B for small square r x r (one CTA); used for R = R2 R1 etc.
__global__ void small_matmul_kernel(int m, int k, int n, const double* __restrict__ A,
                                    const double* __restrict__ B, double* __restrict__ C,
                                    int transA) {
  // entries spread over the grid (same per-entry summation order as one CTA)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += gridDim.x * blockDim.x) {
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
  // Gauss-Jordan on [B | I] with partial pivoting (first maximal |entry|,
  // as a serial scan would pick), three barriers per column: pivot search
  // by warp 0; swap + scale of the pivot row with column k saved; the
  // rank-1 elimination of every other row.  Column k of the left block is
  // never read again, so it is not cleared.
  extern __shared__ double sm[];
  const int d = blockIdx.x;
  const int w = 2 * r;
  double* a = sm;  // r x 2r augmented [B | I]
  __shared__ double colk[DLRSN_MAX_RANK];
  __shared__ int piv;
  __shared__ double pivval;
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
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x < 32) {
      double best = -1.0;
      int p = r;
      for (int i = k + lane; i < r; i += 32) {
        const double v = fabs(a[i * w + k]);
        if (v > best) { best = v; p = i; }  // lowest row of this lane's maximum
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(kFull, best, o);
        const int op = __shfl_xor_sync(kFull, p, o);
        if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
      }
      if (lane == 0) {
        piv = p < r ? p : k;
        pivval = a[(p < r ? p : k) * w + k];
        if (!(best > 0.0) || !isfinite(best)) sing = 1;
      }
    }
    __syncthreads();
    if (sing) break;
    const int p = piv;
    const double inv = 1.0 / pivval;
    // new row k = row p / pivot, row p = old row k; colk = column k after
    // the swap (the old a[k][k] for row p, handed over by the j == k thread)
    for (int j = threadIdx.x; j < w; j += blockDim.x) {
      const double tk = a[k * w + j], tp = a[p * w + j];
      if (p != k) a[p * w + j] = tk;
      a[k * w + j] = tp * inv;
      if (j == k) colk[p] = p == k ? 0.0 : tk;
    }
    for (int i = threadIdx.x; i < r; i += blockDim.x)
      if (i != k && i != p) colk[i] = a[i * w + k];
    if (threadIdx.x == 0 && p != k) colk[k] = 0.0;
    __syncthreads();
    // rank-1 elimination: a warp per row, lanes across the columns j > k (no
    // index division; the pivot row's entries are read once per lane)
    {
      const int wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
      for (int j0 = k + 1; j0 < w; j0 += 32) {
        const int j = j0 + lane;
        const double akj = j < w ? a[k * w + j] : 0.0;
        if (j < w)
          for (int i = wid; i < r; i += nwp)
            if (i != k) a[i * w + j] = fma(-colk[i], akj, a[i * w + j]);
      }
    }
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

// The same inverse without the augmented identity (r > ~110, where [B | I]
// does not fit shared memory): in-place Gauss-Jordan with partial pivoting
// -- column k of the working matrix holds column k of the inverse's
// elimination once it is eliminated -- then the row interchanges undone as
// column swaps in reverse order.  r x r doubles of shared memory.
__global__ void row_inverse_inplace_kernel(int r, const double* __restrict__ proj,
                                           const double* __restrict__ om_sel,
                                           double* __restrict__ Binv, double* __restrict__ Bout,
                                           int* status) {
  extern __shared__ double sm[];
  const int d = blockIdx.x;
  double* a = sm;  // r x r
  __shared__ int perm[DLRSN_MAX_RANK];
  __shared__ int piv;
  __shared__ int sing;
  __shared__ double rowk[DLRSN_MAX_RANK], colk[DLRSN_MAX_RANK];
  const double wx = om_sel ? om_sel[3 * d] : 0.0, wy = om_sel ? om_sel[3 * d + 1] : 0.0;
  const int64_t rr = (int64_t)r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const double b = om_sel ? wx * proj[e] + wy * proj[rr + e] + fabs(wx) * proj[2 * rr + e] +
                                  fabs(wy) * proj[3 * rr + e] + proj[4 * rr + e]
                            : proj[d * rr + e];
    a[e] = b;
    if (Bout) Bout[(int64_t)d * rr + e] = b;
  }
  if (threadIdx.x == 0) sing = 0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double best = fabs(a[k * r + k]);
      for (int i = k + 1; i < r; ++i) {
        const double v = fabs(a[i * r + k]);
        if (v > best) { best = v; p = i; }
      }
      piv = p;
      perm[k] = p;
      if (!(best > 0.0) || !isfinite(best)) sing = 1;
    }
    __syncthreads();
    if (sing) break;
    const int p = piv;
    if (p != k)
      for (int j = threadIdx.x; j < r; j += blockDim.x) {
        const double t = a[k * r + j];
        a[k * r + j] = a[p * r + j];
        a[p * r + j] = t;
      }
    __syncthreads();
    const double inv = 1.0 / a[k * r + k];
    // pivot row scaled (its pivot slot becomes the inverse pivot), the
    // pivot column saved as the multipliers
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
      rowk[j] = j == k ? inv : a[k * r + j] * inv;
      colk[j] = a[j * r + k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
      const int i = e / r, j = e % r;
      if (i == k) {
        a[e] = rowk[j];
      } else {
        const double f = colk[i];
        a[e] = j == k ? -f * inv : a[e] - f * rowk[j];
      }
    }
    __syncthreads();
  }
  if (sing) {
    if (threadIdx.x == 0) status[d] = 1;
    return;
  }
  // undo the row interchanges as column swaps, last first
  for (int k = r - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = threadIdx.x; i < r; i += blockDim.x) {
        const double t = a[i * r + k];
        a[i * r + k] = a[i * r + p];
        a[i * r + p] = t;
      }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const double v = a[e];
    if (!isfinite(v)) status[d] = 1;
    Binv[(int64_t)d * rr + e] = v;
  }
}

// LU with partial pivoting of an n x n matrix in shared memory (one CTA)
// and solve with nrhs right-hand sides stored column-major after it.
__device__ __forceinline__ double pick4(const double (&v)[4], int k) {
  return k == 0 ? v[0] : (k == 1 ? v[1] : (k == 2 ? v[2] : v[3]));
}

__device__ void cta_lu_solve(int n, double* a, int lda, double* b, int ldb, int nrhs, int* perm,
                             int* sing) {
  // three barriers per column: pivot search by warp 0 (first maximal |entry|,
  // as a serial scan picks it); row swap with the scaled multipliers saved;
  // the rank-1 update.  n <= 128.
  __shared__ double colk[DLRSN_MAX_RANK];
  __shared__ double s_inv, s_akk;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    if (tid < 32) {
      double best = -1.0;
      int p = n;
      for (int i = k + lane; i < n; i += 32) {
        const double v = fabs(a[i * lda + k]);
        if (v > best) { best = v; p = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(kFull, best, o);
        const int op = __shfl_xor_sync(kFull, p, o);
        if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
      }
      if (lane == 0) {
        if (p >= n) p = k;
        perm[k] = p;
        const double piv = a[p * lda + k];
        s_inv = piv != 0.0 ? 1.0 / piv : 0.0;
        s_akk = a[k * lda + k];  // moves to row p in the swap
        if (!(best > 0.0)) *sing = 1;
      }
    }
    __syncthreads();
    const int p = perm[k];
    const double inv = s_inv;
    if (p != k) {
      for (int j = tid; j < n; j += blockDim.x) {
        const double t = a[k * lda + j]; a[k * lda + j] = a[p * lda + j]; a[p * lda + j] = t;
      }
      for (int j = tid; j < nrhs; j += blockDim.x) {
        const double t = b[k * ldb + j]; b[k * ldb + j] = b[p * ldb + j]; b[p * ldb + j] = t;
      }
    }
    // multipliers of the rows below; row p now holds the old row k, whose
    // column-k entry was saved before the swap (rows != k, p are untouched)
    for (int i = k + 1 + tid; i < n; i += blockDim.x)
      colk[i] = (i == p ? s_akk : a[i * lda + k]) * inv;
    __syncthreads();
    const int m = n - k - 1;
    for (int e = tid; e < m * (m + nrhs + 1); e += blockDim.x) {
      const int i = k + 1 + e / (m + nrhs + 1), jj = e % (m + nrhs + 1);
      const double l = colk[i];
      if (jj == m + nrhs) a[i * lda + k] = l;
      else if (jj < m) a[i * lda + k + 1 + jj] -= l * a[k * lda + k + 1 + jj];
      else b[i * ldb + (jj - m)] -= l * b[k * ldb + (jj - m)];
    }
  }
  __syncthreads();
  // back substitution: a warp per right-hand side, the column in registers
  const int warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < nrhs; j += nw) {
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      x[q] = i < n ? b[i * ldb + j] : 0.0;
    }
    for (int i = n - 1; i >= 0; --i) {
      double sacc = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = lane + 32 * q;
        if (c > i && c < n) sacc = fma(a[i * lda + c], x[q], sacc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(kFull, sacc, o);
      if (lane == (i & 31)) {
        const int q = i >> 5;
        const double d = a[i * lda + i];
        const double v = d != 0.0 ? (pick4(x, q) - sacc) / d : 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t == q) x[t] = v;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      if (i < n) b[i * ldb + j] = x[q];
    }
  }
  __syncthreads();
}

// Row system combine (lowrank.py:253-259):
//   cbar = sum_d w_d Binv_d ; zeta = sum_d w_d Binv_d Q_d
//   lbar = solve(I - cbar ms / 4pi, zeta); L_d = Binv_d (Q_d + ms lbar / 4pi)
__global__ void row_combine_kernel(int n, int r, const double* __restrict__ Binv,
                                   const double* __restrict__ ms, const double* __restrict__ Q,
                                   const double* __restrict__ wts, double* L,
                                   double* __restrict__ lbar, int* status, int cbar_in_L) {
  extern __shared__ double sm[];
  // cbar_in_L (r > ~110, n >= r): cbar is staged in the output L (global),
  // after zeta has consumed the per-node products kept there
  double* lhs = sm;               // r*r
  double* cbar = cbar_in_L ? L : lhs + r * r;  // r*r
  double* zeta = cbar_in_L ? lhs + r * r : lhs + 2 * r * r;  // r
  double* msl = zeta + r;         // r
  int* perm = reinterpret_cast<int*>(msl + r);
  __shared__ int sing;
  const int64_t rr = (int64_t)r * r;
  // zeta = sum_d w_d Binv_d q_d: the per-node products in parallel (stored
  // in L as scratch), then the node sum in fixed order
  for (int e = threadIdx.x; e < n * r; e += blockDim.x) {
    const int d = e / r, i = e % r;
    double bq = 0.0;
    for (int j = 0; j < r; ++j) bq += Binv[d * rr + i * r + j] * Q[d * r + j];
    L[e] = bq;  // L is overwritten below
  }
  if (threadIdx.x == 0) sing = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += wts[d] * L[d * r + i];
    zeta[i] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += wts[d] * Binv[d * rr + e];
    cbar[e] = s;
  }
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

// The same combine spread over the GPU (the one-call step): the per-node
// products and the node sums, which were the single-CTA kernel's cost (n r^2
// L2 loads each), run as grids; only the r x r solve stays on one CTA.  Same
// summation orders as row_combine_kernel, so the results are identical.
// scratch: cbar (r*r) | zeta (r) | msl (r).
__global__ void row_bq_kernel(int r, const double* __restrict__ Binv, const double* __restrict__ Q,
                              const double* __restrict__ msl, double* __restrict__ out) {
  // out[d][i] = sum_j Binv_d[i][j] (Q_d[j] + msl[j])   (msl null: + 0)
  const int d = blockIdx.x;
  const int64_t rr = (int64_t)r * r;
  __shared__ double qd[DLRSN_MAX_RANK];
  for (int j = threadIdx.x; j < r; j += blockDim.x) qd[j] = msl ? Q[d * r + j] + msl[j] : Q[d * r + j];
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    const double* row = Binv + d * rr + (int64_t)i * r;
    double s = 0.0;
    for (int j = 0; j < r; ++j) s += row[j] * qd[j];
    out[d * r + i] = s;
  }
}

__global__ void row_sums_kernel(int n, int r, const double* __restrict__ Binv,
                                const double* __restrict__ BQ, const double* __restrict__ wts,
                                double* __restrict__ scratch) {
  const int64_t rr = (int64_t)r * r;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < rr) {
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += wts[d] * Binv[d * rr + e];
    scratch[e] = s;
  } else if (e < rr + r) {
    const int i = e - (int)rr;
    double s = 0.0;
    for (int d = 0; d < n; ++d) s += wts[d] * BQ[d * r + i];
    scratch[e] = s;
  }
}

__global__ void __launch_bounds__(1024) row_solve_kernel(int r, const double* __restrict__ ms, double* __restrict__ scratch,
                                 double* __restrict__ lbar, int* status) {
  extern __shared__ double sm[];
  double* lhs = sm;           // r*r
  double* cbar = lhs + r * r; // r*r
  double* zeta = cbar + r * r;
  int* perm = reinterpret_cast<int*>(zeta + r);
  __shared__ int sing;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) cbar[e] = scratch[e];
  for (int i = threadIdx.x; i < r; i += blockDim.x) zeta[i] = scratch[r * r + i];
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
  double* msl = scratch + r * r + r;
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    lbar[i] = zeta[i];
    double s = 0.0;
    for (int p = 0; p < r; ++p) s += ms[i * r + p] * zeta[p];
    msl[i] = s / kFourPi;
  }
  if (threadIdx.x == 0 && sing) *status = 1;
}

int row_combine_grid(int n, int r, const double* Binv, const double* ms, const double* Q,
                     const double* wts, double* L, double* lbar, int* status, double* scratch,
                     cudaStream_t st) {
  const size_t smem = (2 * (size_t)r * r + r) * sizeof(double) + r * sizeof(int);
  DLRSN_REQUIRE(smem <= 227 * 1024, "rank %d too large for row_combine", r);
  row_bq_kernel<<<n, 128, 0, st>>>(r, Binv, Q, nullptr, L);  // L holds B_d^-1 Q_d here
  DLRSN_CHECK_LAUNCH("row_bq_kernel");
  const int len = r * r + r;
  row_sums_kernel<<<(len + 127) / 128, 128, 0, st>>>(n, r, Binv, L, wts, scratch);
  DLRSN_CHECK_LAUNCH("row_sums_kernel");
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  row_solve_kernel<<<1, 1024, smem, st>>>(r, ms, scratch, lbar, status);
  DLRSN_CHECK_LAUNCH("row_solve_kernel");
  row_bq_kernel<<<n, 128, 0, st>>>(r, Binv, Q, scratch + r * r + r, L);
  DLRSN_CHECK_LAUNCH("row_bq_kernel");
  return DLRSN_OK;
}

// Running top-2 of the DEIM argmax: (best, its row, second best value).
// Merging two partial results keeps the larger best (lowest row on ties,
// np.argmax) and max(both seconds, the smaller best) as the second -- equal
// bests give second == best, i.e. an exact tie (gap 0).
__device__ __forceinline__ void top2_merge(double& b, int& i, double& s, double ob, int oi,
                                           double os) {
  s = fmax(fmax(s, os), fmin(b, ob));
  if (ob > b || (ob == b && oi < i)) {
    b = ob;
    i = oi;
  }
}
__device__ __forceinline__ void top2_warp(double& b, int& i, double& s) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(kFull, b, o);
    const int oi = __shfl_xor_sync(kFull, i, o);
    const double os = __shfl_xor_sync(kFull, s, o);
    top2_merge(b, i, s, ob, oi, os);
  }
}
// relative top-2 gap of a pick (near-tie diagnostic; 0 = exact tie)
__device__ __forceinline__ double top2_gap(double b, double s) {
  return b > 0.0 ? (b - fmax(s, 0.0)) / b : 0.0;
}

// DEIM (lowrank.py:168-205) as Gaussian elimination with row pivoting on a
// working copy of W (n x r): column j's Schur-complement column is exactly
// the interpolation residual W[:,j] - W[:,:j] W[p,:j]^-1 W[p,j]; the pivot is
// its first maximal |entry| (np.argmax).  Produces the picks, the unit lower
// factor rows L[p,:] and U (so W[p,:] = Lhat U), all in pick order.
__global__ void __launch_bounds__(1024) deim_kernel(int n, int r,
                                                   double* __restrict__ Wk_global /* n x r work */,
                                                   const double* __restrict__ W,
                                                   int* __restrict__ idx, double* __restrict__ Lhat,
                                                   double* __restrict__ U, int* err_col,
                                                   int in_smem, double* __restrict__ gap) {
  // Column-major work copy (smem when it fits).  Per column: block argmax
  // of |residual| (first index on ties) with two barriers; the picked row is
  // read-only during the elimination (its own update would zero it exactly,
  // so it is skipped and excluded from later argmaxes instead).
  extern __shared__ double dsm[];
  double* Wk = in_smem ? dsm : Wk_global;
  unsigned char* picked = reinterpret_cast<unsigned char*>(in_smem ? dsm + (size_t)n * r : nullptr);
  __shared__ double bv[2][32], bs[2][32];
  __shared__ int bi[2][32];
  __shared__ double s_floor[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  if (in_smem) {
    for (int64_t e = threadIdx.x; e < (int64_t)n * r; e += blockDim.x)
      cp_async8(Wk + (e % r) * n + e / r, W + e);
    for (int i = threadIdx.x; i < n; i += blockDim.x) picked[i] = 0;
    cp_async_wait_all();
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)n * r; e += blockDim.x) mx = fmax(mx, fabs(Wk[e]));
  } else {
    for (int64_t e = threadIdx.x; e < (int64_t)n * r; e += blockDim.x) {
      const int i = (int)(e / r), k = (int)(e % r);
      const double v = W[e];
      Wk[(int64_t)k * n + i] = v;
      mx = fmax(mx, fabs(v));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 0) s_floor[w] = mx;
  __syncthreads();
  double m0 = 0.0;
  for (int q = 0; q < nw; ++q) m0 = fmax(m0, s_floor[q]);
  const double floor_ = 1e-14 * fmax(1.0, m0);  // lowrank.py:185
  int fail = -1;
  for (int j = 0; j < r; ++j) {
    const int buf = j & 1;
    double best = -1.0, second = -1.0;
    int bidx = 0x7fffffff;
    const double* col = Wk + (int64_t)j * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      // (global variant: earlier picks hold exact zeros from here on)
      if (picked && picked[i]) continue;
      const double v = fabs(col[i]);
      if (v > best) { second = best; best = v; bidx = i; }  // rows ascend: first max kept
      else if (v > second) second = v;
    }
    top2_warp(best, bidx, second);
    if (lane == 0) { bv[buf][w] = best; bi[buf][w] = bidx; bs[buf][w] = second; }
    __syncthreads();
    double b = -1.0, sb = -1.0;
    int p = 0x7fffffff;
    for (int q = 0; q < nw; ++q) top2_merge(b, p, sb, bv[buf][q], bi[buf][q], bs[buf][q]);
    // no finite unpicked candidate (all NaN): fail like a vanished residual
    const bool none = p < 0 || p >= n;
    if (none) p = 0;
    const double pv = none ? 0.0 : col[p];
    if (gap && threadIdx.x == 0) gap[j] = top2_gap(b, sb);
    bool bad = !(fabs(pv) > floor_);
    if (!picked)
      for (int q = 0; q < j; ++q) bad |= idx[q] == p;  // (global-memory variant)
    if (threadIdx.x == 0) idx[j] = p;
    if (bad) { fail = j; break; }
    // U row j = pivot row, columns j..r-1; eliminate below (rows != p)
    for (int k = threadIdx.x; k < r; k += blockDim.x) U[j * r + k] = k >= j ? Wk[(int64_t)k * n + p] : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (i == p || (picked && picked[i])) continue;
      const double l = col[i] / pv;
      Wk[(int64_t)j * n + i] = l;  // the multiplier column (Lhat entries)
      for (int k = j + 1; k < r; ++k) Wk[(int64_t)k * n + i] -= l * Wk[(int64_t)k * n + p];
    }
    __syncthreads();
    if (picked && threadIdx.x == 0) picked[p] = 1;
    if (!picked) {
      // global variant: the picked row is excluded by the duplicate test
      // above; zero it as the elimination would
      for (int k = j + 1 + threadIdx.x; k < r; k += blockDim.x) Wk[(int64_t)k * n + p] = 0.0;
      if (threadIdx.x == 0) Wk[(int64_t)j * n + p] = 1.0;
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

// DEIM for small node sets (n <= 1024, r <= RT): one thread per node row,
// the row's r entries in registers, so a pick costs one block argmax and one
// broadcast of the pivot row instead of passes over shared / distributed
// memory.  Per element the arithmetic, the pivot rule (largest |residual|,
// lowest row on ties; np.argmax) and the failure tests are deim_kernel's.
template <int RT>
__global__ void __launch_bounds__(1024) deim_reg_kernel(int n, int r, const double* __restrict__ W,
                                                        int* __restrict__ idx, double* __restrict__ Lhat,
                                                        double* __restrict__ U, int* __restrict__ err_col,
                                                        double* __restrict__ gap) {
  // double-buffered by pick parity: two block barriers per pick, and every
  // warp reduces the per-warp candidates itself (no serial pass)
  __shared__ double bv[2][32], bs[2][32];
  __shared__ int bi[2][32];
  __shared__ double prow[2][RT];
  const int i = threadIdx.x, lane = i & 31, wid = i >> 5, nw = (blockDim.x + 31) >> 5;
  const bool row = i < n;
  double w[RT];
  double mx = 0.0;
#pragma unroll
  for (int k = 0; k < RT; ++k) {
    w[k] = (row && k < r) ? W[(int64_t)i * r + k] : 0.0;
    mx = fmax(mx, fabs(w[k]));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 0) bv[1][wid] = mx;
  __syncthreads();
  double m0 = lane < nw ? bv[1][lane] : 0.0;
  for (int o = 16; o > 0; o >>= 1) m0 = fmax(m0, __shfl_xor_sync(kFull, m0, o));
  const double floor_ = 1e-14 * fmax(1.0, m0);  // lowrank.py:185
  int myq = -1;  // pick order of this row (-1: not picked)
#pragma unroll
  for (int j = 0; j < RT; ++j) {
    if (j >= r) break;
    const int buf = j & 1;
    double best = -1.0, second = -1.0;
    int bidx = 0x7fffffff;
    if (row && myq < 0) {
      best = fabs(w[j]);
      bidx = i;
      if (!(best > -1.0)) { best = -1.0; bidx = 0x7fffffff; }  // NaN: never a candidate
    }
    top2_warp(best, bidx, second);
    if (lane == 0) { bv[buf][wid] = best; bi[buf][wid] = bidx; bs[buf][wid] = second; }
    __syncthreads();
    best = lane < nw ? bv[buf][lane] : -1.0;
    bidx = lane < nw ? bi[buf][lane] : 0x7fffffff;
    second = lane < nw ? bs[buf][lane] : -1.0;
    top2_warp(best, bidx, second);
    // no finite unpicked candidate (all NaN): fail like a vanished residual
    // (row 0 may already be picked, so it is not a fallback)
    const bool none = bidx < 0 || bidx >= n;
    const int p = none ? 0 : bidx;
    if (i == p && !none) {
#pragma unroll
      for (int k = 0; k < RT; ++k) prow[buf][k] = w[k];
    }
    __syncthreads();
    const double pv = none ? 0.0 : prow[buf][j];
    if (gap && i == 0) gap[j] = top2_gap(best, second);
    if (!(fabs(pv) > floor_)) {  // InterpolationError (lowrank.py:192-199)
      if (i == 0) { idx[j] = p; *err_col = j; }
      return;
    }
    if (i == 0) idx[j] = p;
    if (i < r) U[j * r + i] = i >= j ? prow[buf][i] : 0.0;
    if (i == p) {
      myq = j;
    } else if (row && myq < 0) {
      const double l = w[j] / pv;
      w[j] = l;  // the multiplier column (Lhat entries)
#pragma unroll
      for (int k = 0; k < RT; ++k)
        if (k > j && k < r) w[k] -= l * prow[buf][k];
    }
  }
  // Lhat[q, j] = multiplier of column j at the q-th picked row (unit lower)
  if (myq >= 0) {
#pragma unroll
    for (int j = 0; j < RT; ++j)
      if (j < r) Lhat[myq * r + j] = j < myq ? w[j] : (j == myq ? 1.0 : 0.0);
  }
  if (i == 0) *err_col = -1;
}

// DEIM over a thread-block cluster (the same left-to-right GEPP as
// deim_kernel, lowrank.py:168-205): CTA `rank` keeps rows [rank*nl, +nl) of
// W in shared memory (column-major).  Per pick one cluster barrier: every
// CTA publishes its best non-picked row (|residual|, row, the row's trailing
// entries) in a double-buffered slot; after the barrier all CTAs read the
// slots over DSMEM, take the same winner (largest |residual|, lowest row on
// ties) and eliminate their own rows, computing the next column's local
// argmax in the same pass.  Per element the arithmetic is deim_kernel's.
constexpr int kDeimCT = 512;
__global__ void __launch_bounds__(kDeimCT) deim_cluster_kernel(int n, int r, int nl,
                                                              const double* __restrict__ W,
                                                              int* __restrict__ idx,
                                                              double* __restrict__ Lhat,
                                                              double* __restrict__ U, int* err_col,
                                                              double* __restrict__ gap) {
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  extern __shared__ double dsm[];
  const int i0 = crank * nl;
  const int nloc = max(0, min(nl, n - i0));
  const int ls = r + 3;                    // slot stride: value, row, second, entries
  double* Wk = dsm;                        // r x nl, Wk[k * nl + i]
  double* slot = Wk + (size_t)r * nl;      // 2 x ls
  double* prow = slot + 2 * ls;            // r: the pivot row
  unsigned char* picked = reinterpret_cast<unsigned char*>(prow + r);
  __shared__ double wv[kDeimCT / 32], ws2[kDeimCT / 32];
  __shared__ int wi[kDeimCT / 32];
  __shared__ int s_idx[DLRSN_MAX_RANK];
  __shared__ int s_p, s_fail;
  __shared__ double s_floor;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = kDeimCT / 32;
  for (int e = tid; e < nloc * r; e += kDeimCT) cp_async8(Wk + (e % r) * nl + e / r, W + (int64_t)i0 * r + e);
  for (int i = tid; i < nl; i += kDeimCT) picked[i] = 0;
  cp_async_wait_all();
  __syncthreads();
  // floor = 1e-14 max(1, max |W|) (lowrank.py:182), via slot 0
  double mx = 0.0;
  for (int e = tid; e < nloc * r; e += kDeimCT) mx = fmax(mx, fabs(Wk[(e % r) * nl + e / r]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 0) wv[w] = mx;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int q = 0; q < nw; ++q) m = fmax(m, wv[q]);
    slot[0] = m;
  }
  cl.sync();
  if (w == 0) {
    double m = lane < cs ? cl.map_shared_rank(slot, lane)[0] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) s_floor = 1e-14 * fmax(1.0, m);
  }
  // local argmax of column 0
  double best = -1.0, second = -1.0;
  int bidx = 0x7fffffff;
  for (int i = tid; i < nloc; i += kDeimCT) {
    const double v = fabs(Wk[i]);
    if (v > best) { second = best; best = v; bidx = i0 + i; }
    else if (v > second) second = v;
  }
  int fail = -1;
  for (int j = 0; j < r; ++j) {
    double* my = slot + ((j + 1) & 1) * ls;  // step 0 uses slot 1 (slot 0 held the max)
    top2_warp(best, bidx, second);
    if (lane == 0) { wv[w] = best; wi[w] = bidx; ws2[w] = second; }
    __syncthreads();
    if (w == 0) {
      double b = lane < nw ? wv[lane] : -1.0;
      int bi = lane < nw ? wi[lane] : 0x7fffffff;
      double sb = lane < nw ? ws2[lane] : -1.0;
      top2_warp(b, bi, sb);
      if (lane == 0) { my[0] = b; my[1] = (double)bi; my[2] = sb; }
      const bool have = bi >= i0 && bi < i0 + nloc;
      for (int k = j + lane; k < r; k += 32) my[3 + k] = have ? Wk[k * nl + (bi - i0)] : 0.0;
    }
    cl.sync();
    if (w == 0) {
      const double* rs = lane < cs ? cl.map_shared_rank(my, lane) : nullptr;
      double b = rs ? rs[0] : -1.0;
      int bi = rs ? (int)rs[1] : 0x7fffffff;
      double sb = rs ? rs[2] : -1.0;
      int src = lane;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, b, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        const double osb = __shfl_xor_sync(kFull, sb, o);
        const int os = __shfl_xor_sync(kFull, src, o);
        const bool take = ov > b || (ov == b && oi < bi);
        top2_merge(b, bi, sb, ov, oi, osb);
        if (take) src = os;
      }
      const bool valid = bi >= 0 && bi < n;
      if (valid) {
        const double* win = cl.map_shared_rank(my, src);
        for (int k = j + lane; k < r; k += 32) prow[k] = win[3 + k];
      }
      __syncwarp();
      if (lane == 0) {
        const double pv = valid ? prow[j] : 0.0;
        s_p = valid ? bi : 0;
        s_fail = !(valid && fabs(pv) > s_floor);
        if (gap && crank == 0) gap[j] = top2_gap(b, sb);
      }
    }
    __syncthreads();
    const int p = s_p;
    if (crank == 0 && tid == 0) idx[j] = p;
    if (tid == 0) s_idx[j] = p;
    if (s_fail) { fail = j; break; }
    if (crank == 0)
      for (int k = tid; k < r; k += kDeimCT) U[j * r + k] = k >= j ? prow[k] : 0.0;
    const double pv = prow[j];
    const int pl = p - i0;
    if (tid == 0 && pl >= 0 && pl < nloc) picked[pl] = 1;
    best = second = -1.0;
    bidx = 0x7fffffff;
    for (int i = tid; i < nloc; i += kDeimCT) {
      if (i == pl || picked[i]) continue;
      const double l = Wk[j * nl + i] / pv;
      Wk[j * nl + i] = l;  // the multiplier column (Lhat entries)
      for (int k = j + 1; k < r; ++k) Wk[k * nl + i] -= l * prow[k];
      if (j + 1 < r) {
        const double v = fabs(Wk[(j + 1) * nl + i]);
        if (v > best) { second = best; best = v; bidx = i0 + i; }
        else if (v > second) second = v;
      }
    }
    // the next step's slot write happens after the __syncthreads of its
    // block argmax: no thread still reads prow / picked of this step then
  }
  if (fail < 0) {
    __syncthreads();
    // Lhat[q, j] = multiplier of column j at the q-th picked row (unit lower)
    for (int e = tid; e < r * r; e += kDeimCT) {
      const int q = e / r, j = e % r;
      const int pl = s_idx[q] - i0;
      if (pl < 0 || pl >= nloc) continue;
      Lhat[e] = j < q ? Wk[j * nl + pl] : (j == q ? 1.0 : 0.0);
    }
  }
  if (crank == 0 && tid == 0) *err_col = fail;
  cl.sync();  // no CTA leaves while its slots may still be read
}

// DEIM over the whole GPU (node sets too large for a cluster's shared
// memory, e.g. config 5's 16384 x 128 basis): one cooperative launch, CTA b
// keeps rows [b nl, (b+1) nl) of W in shared memory (column-major).  Per pick
// one grid barrier: every CTA publishes its best unpicked row (|residual|,
// row, second best, the row's trailing entries) in a double-buffered global
// slot; after the barrier every CTA reads all slots in CTA order, takes the
// same winner (largest |residual|, lowest row on ties; np.argmax) and
// eliminates its own rows, computing the next column's local argmax in the
// same pass.  Per element the arithmetic is deim_kernel's.
constexpr int kDeimGT = 256;
__global__ void __launch_bounds__(kDeimGT) deim_grid_kernel(int n, int r, int nl,
                                                          const double* __restrict__ W,
                                                          int* __restrict__ idx,
                                                          double* __restrict__ Lhat,
                                                          double* __restrict__ U, int* err_col,
                                                          double* __restrict__ gap,
                                                          double* __restrict__ slots) {
  cg::grid_group grid = cg::this_grid();
  const int G = (int)gridDim.x, me = (int)blockIdx.x;
  extern __shared__ double dsm[];
  const int i0 = me * nl;
  const int nloc = max(0, min(nl, n - i0));
  const int ls = r + 3;                    // slot stride: value, row, second, entries
  double* Wk = dsm;                        // r x nl, Wk[k * nl + i]
  double* prow = Wk + (size_t)r * nl;      // r: the pivot row
  unsigned char* picked = reinterpret_cast<unsigned char*>(prow + r);
  __shared__ double wv[kDeimGT / 32], ws2[kDeimGT / 32];
  __shared__ int wi[kDeimGT / 32];
  __shared__ int s_idx[DLRSN_MAX_RANK];
  __shared__ int s_p, s_fail;
  __shared__ double s_floor;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = kDeimGT / 32;
  for (int e = tid; e < nloc * r; e += kDeimGT) cp_async8(Wk + (e % r) * nl + e / r, W + (int64_t)i0 * r + e);
  for (int i = tid; i < nl; i += kDeimGT) picked[i] = 0;
  cp_async_wait_all();
  __syncthreads();
  // floor = 1e-14 max(1, max |W|) (lowrank.py:182), via slot column 0
  double mx = 0.0;
  for (int e = tid; e < nloc * r; e += kDeimGT) mx = fmax(mx, fabs(Wk[(e % r) * nl + e / r]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 0) wv[w] = mx;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int q = 0; q < nw; ++q) m = fmax(m, wv[q]);
    slots[(int64_t)2 * G * ls + me] = m;  // scratch after the two slot buffers
  }
  grid.sync();
  if (w == 0) {
    double m = 0.0;
    for (int q = lane; q < G; q += 32) m = fmax(m, __ldcg(slots + (int64_t)2 * G * ls + q));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) s_floor = 1e-14 * fmax(1.0, m);
  }
  // local argmax of column 0
  double best = -1.0, second = -1.0;
  int bidx = 0x7fffffff;
  for (int i = tid; i < nloc; i += kDeimGT) {
    const double v = fabs(Wk[i]);
    if (v > best) { second = best; best = v; bidx = i0 + i; }
    else if (v > second) second = v;
  }
  int fail = -1;
  for (int j = 0; j < r; ++j) {
    double* mine = slots + ((int64_t)(j & 1) * G + me) * ls;
    top2_warp(best, bidx, second);
    if (lane == 0) { wv[w] = best; wi[w] = bidx; ws2[w] = second; }
    __syncthreads();
    if (w == 0) {
      double b = lane < nw ? wv[lane] : -1.0;
      int bi = lane < nw ? wi[lane] : 0x7fffffff;
      double sb = lane < nw ? ws2[lane] : -1.0;
      top2_warp(b, bi, sb);
      if (lane == 0) { mine[0] = b; mine[1] = (double)bi; mine[2] = sb; }
      const bool have = bi >= i0 && bi < i0 + nloc;
      for (int k = j + lane; k < r; k += 32) mine[3 + k] = have ? Wk[k * nl + (bi - i0)] : 0.0;
    }
    grid.sync();
    if (w == 0) {
      // every CTA reduces the G slots in the same order: identical winner
      double b = -1.0, sb = -1.0;
      int bi = 0x7fffffff, src = 0;
      for (int q = lane; q < G; q += 32) {
        const double* sl = slots + ((int64_t)(j & 1) * G + q) * ls;
        const double ob = __ldcg(sl), osb = __ldcg(sl + 2);
        const int oi = (int)__ldcg(sl + 1);
        const bool take = ob > b || (ob == b && oi < bi);
        top2_merge(b, bi, sb, ob, oi, osb);
        if (take) src = q;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, b, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        const double osb = __shfl_xor_sync(kFull, sb, o);
        const int os = __shfl_xor_sync(kFull, src, o);
        const bool take = ov > b || (ov == b && oi < bi);
        top2_merge(b, bi, sb, ov, oi, osb);
        if (take) src = os;
      }
      const bool valid = bi >= 0 && bi < n;
      if (valid) {
        const double* win = slots + ((int64_t)(j & 1) * G + src) * ls;
        for (int k = j + lane; k < r; k += 32) prow[k] = __ldcg(win + 3 + k);
      }
      __syncwarp();
      if (lane == 0) {
        const double pv = valid ? prow[j] : 0.0;
        s_p = valid ? bi : 0;
        s_fail = !(valid && fabs(pv) > s_floor);
        if (gap && me == 0) gap[j] = top2_gap(b, sb);
      }
    }
    __syncthreads();
    const int p = s_p;
    if (me == 0 && tid == 0) idx[j] = p;
    if (tid == 0) s_idx[j] = p;
    if (s_fail) { fail = j; break; }
    if (me == 0)
      for (int k = tid; k < r; k += kDeimGT) U[j * r + k] = k >= j ? prow[k] : 0.0;
    const double pv = prow[j];
    const int pl = p - i0;
    if (tid == 0 && pl >= 0 && pl < nloc) picked[pl] = 1;
    best = second = -1.0;
    bidx = 0x7fffffff;
    for (int i = tid; i < nloc; i += kDeimGT) {
      if (i == pl || picked[i]) continue;
      const double l = Wk[j * nl + i] / pv;
      Wk[j * nl + i] = l;  // the multiplier column (Lhat entries)
      for (int k = j + 1; k < r; ++k) Wk[k * nl + i] -= l * prow[k];
      if (j + 1 < r) {
        const double v = fabs(Wk[(j + 1) * nl + i]);
        if (v > best) { second = best; best = v; bidx = i0 + i; }
        else if (v > second) second = v;
      }
    }
    __syncthreads();  // prow / picked of this pick are consumed
  }
  if (fail < 0) {
    // Lhat[q, j] = multiplier of column j at the q-th picked row (unit lower)
    for (int e = tid; e < r * r; e += kDeimGT) {
      const int q = e / r, jj = e % r;
      const int pl = s_idx[q] - i0;
      if (pl < 0 || pl >= nloc) continue;
      Lhat[e] = jj < q ? Wk[jj * nl + pl] : (jj == q ? 1.0 : 0.0);
    }
  }
  if (me == 0 && tid == 0) *err_col = fail;
}

// Solves with W_hat = Lhat U (pick order):
//   mode 0 (interpolation_coefficients): X = W_hat^-1 V   (V r x m)
//   mode 1 (closure_weights):            x = W_hat^-T v   (v r)
// A warp per right-hand side: the solution column lives in registers (lane
// l holds rows l, l + 32, ...), each substitution row is a warp dot product
// of a factor row (contiguous, conflict-free) with the solved part.  For
// mode 1 the factors are staged transposed so the rows stay contiguous.
__global__ void __launch_bounds__(1024) what_solve_kernel(int r, int m, const double* __restrict__ Lhat,
                                                          const double* __restrict__ U,
                                                          const double* __restrict__ V,
                                                          double* __restrict__ X, int mode,
                                                          int factors_global) {
  extern __shared__ double sw[];
  // factors_global (r x r factors too large to stage, r > ~110): read from
  // global memory (L1 / L2), transposed access for mode 1
  double* sF = sw;  // [2][r][r]: mode 0: L, U; mode 1: U^T, L^T
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t rr = (int64_t)r * r;
  if (!factors_global) {
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int i = e / r, j = e - (e / r) * r;
      if (mode == 0) {
        sF[e] = Lhat[e];
        sF[rr + e] = U[e];
      } else {
        sF[i * r + j] = U[(int64_t)j * r + i];
        sF[rr + i * r + j] = Lhat[(int64_t)j * r + i];
      }
    }
    __syncthreads();
  }
  // A[i][p]: first factor (forward, lower-triangular use), B: second (backward)
  auto fa = [&](int i, int p) -> double {
    if (!factors_global) return sF[i * r + p];
    return mode == 0 ? Lhat[(int64_t)i * r + p] : U[(int64_t)p * r + i];
  };
  auto fb = [&](int i, int p) -> double {
    if (!factors_global) return sF[rr + i * r + p];
    return mode == 0 ? U[(int64_t)i * r + p] : Lhat[(int64_t)p * r + i];
  };
  const bool unit_a = mode == 0;  // L (mode 0) has a unit diagonal; U^T does not
  for (int c = warp; c < m; c += nw) {
    double x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = lane + 32 * k;
      x[k] = i < r ? V[(int64_t)i * m + c] : 0.0;
    }
    // forward: A y = v, A lower triangular
    for (int i = 0; i < r; ++i) {
      double sacc = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = lane + 32 * k;
        if (p < i) sacc = fma(fa(i, p), x[k], sacc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(kFull, sacc, o);
      if (lane == (i & 31)) {
        const int k = i >> 5;
        double v = pick4(x, k) - sacc;
        if (!unit_a) v /= fa(i, i);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == k) x[q] = v;
      }
    }
    // backward: B x = y, B upper triangular (U, or L^T with a unit diagonal)
    for (int i = r - 1; i >= 0; --i) {
      double sacc = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = lane + 32 * k;
        if (p > i && p < r) sacc = fma(fb(i, p), x[k], sacc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(kFull, sacc, o);
      if (lane == (i & 31)) {
        const int k = i >> 5;
        double v = pick4(x, k) - sacc;
        if (mode == 0) v /= fb(i, i);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == k) x[q] = v;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = lane + 32 * k;
      if (i < r) X[(int64_t)i * m + c] = x[k];
    }
  }
}

}  // namespace dlrsn

using namespace dlrsn;

static int grid_for(int64_t n, int block = kRB) {
  int64_t b = (n + block - 1) / block;
  if (b > 148 * 32) b = 148 * 32;
  return (int)(b < 1 ? 1 : b);
}

namespace dlrsn {
int rowmix_vec(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
               double beta, double* Y, int ldy, const double* v, double* yv,
               dlrsn_stream_t stream);
int mgram_vec(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda, const double* B,
              int ldb, const double* coeff, double* G, double* partial, const double* v,
              double* yv, dlrsn_stream_t stream);
}

extern "C" {

int dlrsn_rowmix_upper(int64_t n, int r, const double* X, int ldx, const double* K, int ldk,
                       double* Y, int ldy, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(n >= 0 && r >= 1 && r <= DLRSN_MAX_RANK && X && K && Y, "bad dlrsn_rowmix_upper arguments");
  return dlrsn::rowmix_upper(n, r, X, ldx, K, ldk, Y, ldy, as_stream(stream));
}

int dlrsn_rowmix(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
                 double beta, double* Y, int ldy, dlrsn_stream_t stream) {
  return dlrsn::rowmix_vec(n, kx, ky, X, ldx, K, ldk, beta, Y, ldy, nullptr, nullptr, stream);
}

}  // extern "C"

namespace dlrsn {
// Y = X K (+ beta Y) and, with v / yv, yv = X v from the same pass over X
// (the wide DMMA kernel; otherwise a second launch)
int rowmix_vec(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
               double beta, double* Y, int ldy, const double* v, double* yv,
               dlrsn_stream_t stream) {
  DLRSN_REQUIRE(kx >= 0 && ky >= 0 && kx * ky <= 48 * 1024 / 8 * 4, "rowmix operand too large");
  if (n == 0 || ky == 0) return DLRSN_OK;
  const double* V = v;
  double* YV = yv;
  if (v && !((kx > 32 || ky > 16) && kx <= 128 && n >= 64)) {  // not the wide kernel
    const int rc = dlrsn_rowmix(n, kx, 1, X, ldx, v, 1, 0.0, yv, 1, stream);
    if (rc != DLRSN_OK) return rc;
    V = nullptr;
    YV = nullptr;
  }
  if (kx <= 32 && ky <= 16 && n >= 64) {
    const int64_t tiles = (n + 7) / 8;
    int64_t blocks = (tiles + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    const int grid = (int)(blocks < 1 ? 1 : blocks);
    cudaStream_t st = as_stream(stream);
    const int ks = (kx + 3) / 4;
#define DLRSN_ROWMIX_MMA(KS, NT) \
  rowmix_mma_kernel<KS, NT><<<grid, 256, 0, st>>>((int)n, kx, ky, X, ldx, K, ldk, beta, Y, ldy)
    if (ky <= 8) {
      if (ks <= 1) DLRSN_ROWMIX_MMA(1, 1);
      else if (ks <= 2) DLRSN_ROWMIX_MMA(2, 1);
      else if (ks <= 4) DLRSN_ROWMIX_MMA(4, 1);
      else DLRSN_ROWMIX_MMA(8, 1);
    } else {
      if (ks <= 1) DLRSN_ROWMIX_MMA(1, 2);
      else if (ks <= 2) DLRSN_ROWMIX_MMA(2, 2);
      else if (ks <= 4) DLRSN_ROWMIX_MMA(4, 2);
      else DLRSN_ROWMIX_MMA(8, 2);
    }
#undef DLRSN_ROWMIX_MMA
    DLRSN_CHECK_LAUNCH("rowmix_mma_kernel");
    return DLRSN_OK;
  }
  const bool aligned = ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)ldx * 8) & 15) == 0;
  if ((kx > 32 || ky > 16) && kx <= 128 && n >= 64) {
    const int ks = kx <= 16 ? 4 : (kx <= 32 ? 8 : (kx <= 64 ? 16 : 32));
    int nt = ky > 32 ? 8 : (ky > 16 ? 4 : (ky > 8 ? 2 : 1));
    {  // A/B: DLRSN_ROWMIX_NT caps the column group (more CTAs per SM)
      static const char* e = getenv("DLRSN_ROWMIX_NT");
      const int cap = e ? atoi(e) : 0;
      if (cap > 0 && nt > cap) nt = cap;
    }
    const int kyp = (ky + 8 * nt - 1) / (8 * nt) * (8 * nt);
    const int ldks = kyp + ((4 - kyp % 16) + 16) % 16;
    const size_t smem = (size_t)4 * ks * ldks * sizeof(double);
    const int vec = aligned && kx == 4 * ks;
    const int64_t tiles = (n + 7) / 8;
    int64_t blocks = (tiles + 15) / 16;
    if (blocks > 148 * 4) blocks = 148 * 4;
    cudaStream_t st = as_stream(stream);
#define DLRSN_ROWMIX_WIDE(KS, NT)                                                                do {                                                                                             if (smem > 48 * 1024)                                                                            DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_wide_kernel<KS, NT>,                                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));     rowmix_wide_kernel<KS, NT><<<(int)blocks, 256, smem, st>>>((int)n, kx, ky, X, ldx, K, ldk, beta,                                                                Y, ldy, kyp, ldks, vec, V, YV);          } while (0)
    static const int pipe = getenv("DLRSN_ROWMIX_WIDE_PIPE") ? atoi(getenv("DLRSN_ROWMIX_WIDE_PIPE")) : 0;
    if (pipe && ks == 16 && nt == 8 && static_cast<const void*>(X) != static_cast<const void*>(Y)) {
      // r in (32, 64] with > 32 output columns: the software-pipelined kernel
      if (smem > 48 * 1024)
        DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_wide_pipe_kernel<16, 8>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int64_t pb = (tiles + 7) / 8;
      if (pb > 148) pb = 148;
      rowmix_wide_pipe_kernel<16, 8><<<(int)pb, pipe >= 2 ? 384 : 256, smem, st>>>(
          (int)n, kx, ky, X, ldx, K, ldk, beta, Y, ldy, kyp, ldks, vec, V, YV);
      DLRSN_CHECK_LAUNCH("rowmix_wide_pipe_kernel");
      return DLRSN_OK;
    }
    if (ks == 4) {
      if (nt == 8) DLRSN_ROWMIX_WIDE(4, 8);
      else if (nt == 4) DLRSN_ROWMIX_WIDE(4, 4);
      else DLRSN_ROWMIX_WIDE(4, 2);
    } else if (ks == 8) {
      if (nt == 8) DLRSN_ROWMIX_WIDE(8, 8);
      else if (nt == 4) DLRSN_ROWMIX_WIDE(8, 4);
      else DLRSN_ROWMIX_WIDE(8, 2);
    } else if (ks == 16) {
      if (nt == 8) DLRSN_ROWMIX_WIDE(16, 8);
      else if (nt == 4) DLRSN_ROWMIX_WIDE(16, 4);
      else if (nt == 2) DLRSN_ROWMIX_WIDE(16, 2);
      else DLRSN_ROWMIX_WIDE(16, 1);
    } else {
      if (nt == 8) DLRSN_ROWMIX_WIDE(32, 8);
      else if (nt == 4) DLRSN_ROWMIX_WIDE(32, 4);
      else if (nt == 2) DLRSN_ROWMIX_WIDE(32, 2);
      else DLRSN_ROWMIX_WIDE(32, 1);
    }
#undef DLRSN_ROWMIX_WIDE
    DLRSN_CHECK_LAUNCH("rowmix_wide_kernel");
    return DLRSN_OK;
  }
  if (aligned && (kx == 8 || kx == 16 || kx == 32) && kRB % ky == 0) {
    const int grid = grid_for(n * ky);
    cudaStream_t st = as_stream(stream);
    if (kx == 8)
      rowmix_reg_kernel<8><<<grid, kRB, 0, st>>>((int)n, ky, X, ldx, K, ldk, beta, Y, ldy);
    else if (kx == 16)
      rowmix_reg_kernel<16><<<grid, kRB, 0, st>>>((int)n, ky, X, ldx, K, ldk, beta, Y, ldy);
    else
      rowmix_reg_kernel<32><<<grid, kRB, 0, st>>>((int)n, ky, X, ldx, K, ldk, beta, Y, ldy);
    DLRSN_CHECK_LAUNCH("rowmix_reg_kernel");
    return DLRSN_OK;
  }
  const size_t smem = (size_t)kx * ky * sizeof(double);
  if (smem > 48 * 1024)
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(rowmix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rowmix_kernel<<<grid_for(n * ky), kRB, smem, as_stream(stream)>>>((int)n, kx, ky, X, ldx, K, ldk,
                                                                   beta, Y, ldy);
  DLRSN_CHECK_LAUNCH("rowmix_kernel");
  return DLRSN_OK;
}
}  // namespace dlrsn

extern "C" {

// cells per block of the cell-reduction kernels: about 4 CTAs per SM in
// total over all output tiles, in whole smem chunks
static int cells_per_block(int ncell, int tiles) {
  const int target = (4 * 148 + tiles - 1) / tiles;
  int cpb = (ncell + target - 1) / target;
  cpb = (cpb + kChunk - 1) / kChunk * kChunk;
  return cpb < kChunk ? kChunk : cpb;
}

// cells per block of project_mma32g_kernel: about 4 waves of 2 CTAs per SM
// over all 32x32 output tiles and both output groups, whole chunks
// diagonal 64-column blocks (project64d_group) for r > 32 (DLRSN_K3_D64=0: the
// 32 x 32 tiling everywhere)
static bool project_d64(int r) {
  static const bool on = [] {
    const char* e = getenv("DLRSN_K3_D64");
    return !(e && e[0] == '0');
  }();
  return on && r > kT32;
}

// the work list of one cell block (see ProjTiles)
static ProjTiles project_tiles(int r, bool sym) {
  ProjTiles tl;
  tl.n = 0;
  const int T = (r + kT32 - 1) / kT32;
  const bool d64 = sym && project_d64(r);
  auto add = [&](int kind, int ti, int tj) {
    tl.e[tl.n++] = (unsigned char)(kind | ti << 3 | tj << 5);
  };
  for (int ti = 0; ti < T; ++ti)
    for (int tj = 0; tj < T; ++tj) {
      if (d64 && ti / 2 == tj / 2) continue;  // inside a diagonal 64-block
      if (!sym || ti <= tj) {
        add(0, ti, tj);
        add(1, ti, tj);
      } else {
        add(2, ti, tj);
      }
    }
  return tl;
}

static int project32g_cells_per_block(int ncell, int r) {
  static const char* sym_env = getenv("DLRSN_PROJECT_SYM");
  const bool sym = !(sym_env && sym_env[0] == '0');
  const bool d64 = sym && project_d64(r);
  // CTAs per cell block (the work list, plus the diagonal 64-block CTAs)
  const int work = project_tiles(r, sym).n + (d64 ? 2 * ((r + 63) / 64) : 0);
  if (d64) {
    // diagonal 64-blocks: every cell costs the same, so one cell range per
    // SM (the two group CTAs of a range share an SM and its X rows) is
    // balanced without a tail and needs only 148 partial slots
    (void)work;
    static const int nr = getenv("DLRSN_K3_RANGES") ? atoi(getenv("DLRSN_K3_RANGES")) : 296;
    const int target = nr;
    int cpb = (ncell + target - 1) / target;
    cpb = (cpb + kPCG - 1) / kPCG * kPCG;
    return cpb < kPCG ? kPCG : cpb;
  }
  // ~16 waves: the CTAs of one cell block finish close together and share
  // its X rows through L2 (C4: 10.0 -> 9.5 ms; 4 waves re-read X 3x from DRAM)
  static const int waves = getenv("DLRSN_K3_WAVES") ? atoi(getenv("DLRSN_K3_WAVES")) : 16;
  const int target = (waves * 2 * 148 + work - 1) / work;
  int cpb = (ncell + target - 1) / target;
  cpb = (cpb + kPCG - 1) / kPCG * kPCG;
  return cpb < kPCG ? kPCG : cpb;
}

// cells per block of project_mma32_kernel: one block per SM (148) over all
// 32x32 output tiles
static int project32_cells_per_block(int ncell, int r) {
  const int tiles32 = ((r + kT32 - 1) / kT32) * ((r + kT32 - 1) / kT32);
  const int target = (148 + tiles32 - 1) / tiles32;
  int cpb = (ncell + target - 1) / target;
  cpb = (cpb + kPC32 - 1) / kPC32 * kPC32;
  return cpb < kPC32 ? kPC32 : cpb;
}

// mgram launch plan: the wide kernel (TB = 32 / 64 blocks, about 2 CTAs per
// SM over all output blocks, whole 16-cell chunks) when ra or rb > 32
struct MgramPlan {
  int tb, tiles, cpb, nblk;
};
static MgramPlan mgram_plan(int ncell, int ra, int rb) {
  MgramPlan pl;
  const int mx = ra > rb ? ra : rb;
  pl.tb = mx > 32 ? (mx > 48 ? 64 : 32) : 0;
  if (pl.tb == 0) {
    pl.tiles = ((ra + kTile - 1) / kTile) * ((rb + kTile - 1) / kTile);
    pl.cpb = cells_per_block(ncell, pl.tiles);
  } else {
    pl.tiles = ((ra + pl.tb - 1) / pl.tb) * ((rb + pl.tb - 1) / pl.tb);
    const int target = (2 * 148 + pl.tiles - 1) / pl.tiles;
    int cpb = (ncell + target - 1) / target;
    cpb = (cpb + kMgC - 1) / kMgC * kMgC;
    pl.cpb = cpb < kMgC ? kMgC : cpb;
  }
  pl.nblk = (ncell + pl.cpb - 1) / pl.cpb;
  return pl;
}

// symmetric Gram plan: 32-wide upper tiles, about 2 CTAs per SM over them
static MgramPlan mgram_plan_sym(int ncell, int r) {
  MgramPlan pl;
  const int T = (r + 31) / 32;
  pl.tb = 32;
  pl.tiles = T * (T + 1) / 2;
  const int target = (2 * 148 + pl.tiles - 1) / pl.tiles;
  int cpb = (ncell + target - 1) / target;
  cpb = (cpb + kMgC - 1) / kMgC * kMgC;
  pl.cpb = cpb < kMgC ? kMgC : cpb;
  pl.nblk = (ncell + pl.cpb - 1) / pl.cpb;
  return pl;
}

// G[i][j] = G[j][i] below the diagonal tiles of a symmetric Gram
__global__ void mirror_gram_kernel(int r, int tb, double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * r; e += gridDim.x * blockDim.x) {
    const int i = e / r, j = e % r;
    if (i / tb > j / tb) G[e] = G[j * r + i];
  }
}

int64_t dlrsn_partials_len(int ncell, int ra, int rb, int kind) {
  // partial buffer (doubles) for mgram (kind 0) / project (kind 1)
  if (kind == 0) {
    int64_t nb = mgram_plan(ncell, ra, rb).nblk;
    if (ra == rb && ra > 32) nb = std::max<int64_t>(nb, mgram_plan_sym(ncell, ra).nblk);
    return nb * ra * rb;
  }
  const int tiles = ((ra + kTile - 1) / kTile) * ((rb + kTile - 1) / kTile);
  const int cpb = cells_per_block(ncell, tiles);
  int64_t nblk = (ncell + cpb - 1) / cpb;
  const int cpb32 = project32_cells_per_block(ncell, ra);
  const int64_t nblk32 = (ncell + cpb32 - 1) / cpb32;
  if (nblk32 > nblk) nblk = nblk32;
  const int cpbg = project32g_cells_per_block(ncell, ra);
  const int64_t nblkg = (ncell + cpbg - 1) / cpbg;
  if (nblkg > nblk) nblk = nblkg;
  nblk += kProjBndBlocks;  // the boundary-face slots of the diagonal 64-block path
  return nblk * (7 * (int64_t)ra * ra + ra);
}

int dlrsn_mgram(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda,
                const double* B, int ldb, const double* coeff, double* G, double* partial,
                dlrsn_stream_t stream) {
  return dlrsn::mgram_vec(ops, ra, rb, A, lda, B, ldb, coeff, G, partial, nullptr, nullptr, stream);
}

}  // extern "C"

namespace dlrsn {
// dlrsn_mgram and, with v / yv, yv = B v (n_dofs) from the rows the Gram
// stages anyway (single-tile symmetric Grams, 32 < r <= 64; otherwise a
// separate rowmix launch)
int mgram_vec(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda, const double* B,
              int ldb, const double* coeff, double* G, double* partial, const double* v,
              double* yv, dlrsn_stream_t stream) {
  const int ncell = ops->nx * ops->ny;
  cudaStream_t st = as_stream(stream);
  static const char* sym_env = getenv("DLRSN_MGRAM_SYM");
  if (A == B && lda == ldb && ra == rb && ra > 32 && sym_env && sym_env[0] == '1') {
    // symmetric Gram: the 32-wide tiles on and above the diagonal only
    // (T (T + 1) / 2 of T^2), mirrored after the reduction.  Off by default:
    // measured slower than the 64-wide kernel over all tiles (C4 1.51 vs
    // 2.46 ms, r = 128 25.4 vs 34.3 ms): the 32-wide tiles stage and
    // premultiply each operand column block once per tile pair
    const int T = (ra + 31) / 32, tiles = T * (T + 1) / 2;
    const MgramPlan pl = mgram_plan_sym(ncell, ra);
    const int vec = ((reinterpret_cast<uintptr_t>(A) | (uintptr_t)lda * 8) & 15) == 0;
    const size_t smem = MgramWide<32>::smem(false);
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(mgram_wide_kernel<32>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    mgram_wide_kernel<32><<<dim3(pl.nblk, tiles), 256, smem, st>>>(ncell, ra, rb, A, lda, B, ldb,
                                                                   coeff, *ops, pl.cpb, partial,
                                                                   vec, 1, nullptr, nullptr);
    DLRSN_CHECK_LAUNCH("mgram_wide_kernel");
    const int64_t len = (int64_t)ra * rb;
    reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 1024, 0, st>>>(pl.nblk, len, partial, G, 1.0);
    DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
    mirror_gram_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(ra, 32, G);
    DLRSN_CHECK_LAUNCH("mirror_gram_kernel");
    if (v) return dlrsn_rowmix(4 * (int64_t)ncell, rb, 1, B, ldb, v, 1, 0.0, yv, 1, stream);
    return DLRSN_OK;
  }
  const MgramPlan pl = mgram_plan(ncell, ra, rb);
  const int nblk = pl.nblk;
  {
    // symmetric single-block Gram (the CholQR2 Grams at 32 < r <= 64): the
    // diagonal-block layout (DLRSN_MGRAM64S=0: the tiled kernel)
    static const bool on = !(getenv("DLRSN_MGRAM64S") && getenv("DLRSN_MGRAM64S")[0] == '0');
    if (on && A == B && lda == ldb && ra == rb && ra > 32 && ra <= 64 && !coeff && !v) {
      static bool attr = false;
      if (!attr) {
        DLRSN_TRY_CUDA(cudaFuncSetAttribute(mgram64s_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kMgram64sSmem));
        attr = true;
      }
      mgram64s_kernel<<<nblk, 256, kMgram64sSmem, st>>>(ncell, ra, A, lda, *ops, pl.cpb, partial);
      DLRSN_CHECK_LAUNCH("mgram64s_kernel");
      const int64_t len = (int64_t)ra * rb;
      reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 1024, 0, st>>>(nblk, len, partial, G, 1.0);
      DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
      mirror_gram_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(ra, 8, G);
      DLRSN_CHECK_LAUNCH("mirror_gram_kernel");
      return DLRSN_OK;
    }
  }
  bool tsym = false;
  if (pl.tb == 0) {
    mgram_mma_kernel<<<dim3(nblk, pl.tiles), kTile * kTile, 0, st>>>(ncell, ra, rb, A, lda, B, ldb,
                                                                     coeff, *ops, pl.cpb, partial);
    DLRSN_CHECK_LAUNCH("mgram_mma_kernel");
  } else {
    const int vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                      (uintptr_t)lda * 8 | (uintptr_t)ldb * 8) & 15) == 0;
    const bool same = A == B && lda == ldb && pl.tiles == 1;  // every block then takes the same path
    if (pl.tb == 64) {
      const size_t smem = MgramWide<64>::smem(same);
      DLRSN_TRY_CUDA(cudaFuncSetAttribute(mgram_wide_kernel<64>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // DLRSN_MGRAM_FULL=1: diagonal tiles computed in full (A/B timing)
      static const char* full_env = getenv("DLRSN_MGRAM_FULL");
      const bool full = full_env && full_env[0] == '1';
      // symmetric Gram over several tiles: the tiles ti <= tj only, the
      // lower ones mirrored after the reduction
      const int T = (ra + 63) / 64;
      tsym = !full && A == B && lda == ldb && ra == rb && pl.tiles > 1;
      const int gy = tsym ? T * (T + 1) / 2 : pl.tiles;
      const bool fuse = v != nullptr && same;  // one tile: every CTA stages all columns
      mgram_wide_kernel<64><<<dim3(nblk, gy), 256, smem, st>>>(ncell, ra, rb, A, lda, B, ldb,
                                                               coeff, *ops, pl.cpb, partial, vec,
                                                               (full ? 2 : 0) | (tsym ? 1 : 0),
                                                               fuse ? v : nullptr, fuse ? yv : nullptr);
      if (fuse) v = nullptr;
    } else {
      const size_t smem = MgramWide<32>::smem(same);
      DLRSN_TRY_CUDA(cudaFuncSetAttribute(mgram_wide_kernel<32>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      mgram_wide_kernel<32><<<dim3(nblk, pl.tiles), 256, smem, st>>>(ncell, ra, rb, A, lda, B, ldb,
                                                                     coeff, *ops, pl.cpb, partial, vec,
                                                                     0, nullptr, nullptr);
    }
    DLRSN_CHECK_LAUNCH("mgram_wide_kernel");
  }
  const int64_t len = (int64_t)ra * rb;
  reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 1024, 0, st>>>(nblk, len, partial, G, 1.0);
  DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
  if (tsym) {
    mirror_gram_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(ra, 64, G);
    DLRSN_CHECK_LAUNCH("mirror_gram_kernel");
  }
  if (v) return dlrsn_rowmix(4 * (int64_t)ncell, rb, 1, B, ldb, v, 1, 0.0, yv, 1, stream);
  return DLRSN_OK;
}
}  // namespace dlrsn

extern "C" {

}  // extern "C"

namespace dlrsn {
// optional CUDA-event timing of the K3 kernel launches (bench.py roofline)
static bool g_proj_timing = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_proj_events;
static size_t g_proj_used = 0;
static std::pair<cudaEvent_t, cudaEvent_t>* proj_timer() {
  if (!g_proj_timing) return nullptr;
  if (g_proj_used == g_proj_events.size()) {
    std::pair<cudaEvent_t, cudaEvent_t> e;
    if (cudaEventCreate(&e.first) != cudaSuccess || cudaEventCreate(&e.second) != cudaSuccess)
      return nullptr;
    g_proj_events.push_back(e);
  }
  return &g_proj_events[g_proj_used++];
}
bool project_timing_enabled() { return g_proj_timing; }
}  // namespace dlrsn

namespace dlrsn {
int project_ex(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
               const double* halo, int top_wall, const double* sigma_t, const double* sigma_s,
               const double* q, double* out, double* partial, const int* any_scat,
               cudaStream_t stream);
}  // namespace dlrsn

extern "C" {

int dlrsn_project_timing(int enable) {
  g_proj_timing = enable != 0;
  g_proj_used = 0;
  return DLRSN_OK;
}

int dlrsn_project_timing_read(int cap, float* ms, int* count) {
  int n = 0;
  for (size_t k = 0; k < g_proj_used; ++k, ++n) {
    if (n >= cap) continue;
    DLRSN_TRY_CUDA(cudaEventSynchronize(g_proj_events[k].second));
    DLRSN_TRY_CUDA(cudaEventElapsedTime(&ms[n], g_proj_events[k].first, g_proj_events[k].second));
  }
  *count = n;
  return DLRSN_OK;
}

int dlrsn_project(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
                  const double* sigma_t, const double* sigma_s, const double* q, double* out,
                  double* partial, dlrsn_stream_t stream) {
  return dlrsn_project_slab(ops, r, X, Xold, nullptr, 1, sigma_t, sigma_s, q, out, partial, stream);
}

int dlrsn_project_slab(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
                       const double* halo, int top_wall, const double* sigma_t,
                       const double* sigma_s, const double* q, double* out, double* partial,
                       dlrsn_stream_t stream) {
  return dlrsn::project_ex(ops, r, X, Xold, halo, top_wall, sigma_t, sigma_s, q, out, partial,
                           nullptr, as_stream(stream));
}

}  // extern "C"

namespace dlrsn {
int project_ex(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
               const double* halo, int top_wall, const double* sigma_t, const double* sigma_s,
               const double* q, double* out, double* partial, const int* any_scat,
               cudaStream_t stream) {
  const int ncell = ops->nx * ops->ny;
  const int tiles = ((r + kTile - 1) / kTile) * ((r + kTile - 1) / kTile);
  const int cpb = cells_per_block(ncell, tiles);
  const int nblk = (ncell + cpb - 1) / cpb;
  ProjArgs pa;
  pa.nx = ops->nx; pa.ny = ops->ny; pa.r = r;
  pa.X = X; pa.Xold = Xold; pa.sigma_t = sigma_t; pa.sigma_s = sigma_s; pa.q = q;
  pa.part = partial; pa.cells_per_block = cpb;
  pa.halo = halo;
  pa.top_wall = top_wall;
  pa.any_scat = any_scat;
  cudaStream_t st = stream;
  static const char* simt = getenv("DLRSN_PROJECT_SIMT");
  static const char* wide = getenv("DLRSN_PROJECT_WIDE");
  if (r > kTile && !(wide && wide[0] == '0') && !(simt && simt[0] == '1')) {
    // 32x32 tiles; one block per SM (the accumulators need the registers)
    const int tiles32 = ((r + kT32 - 1) / kT32) * ((r + kT32 - 1) / kT32);
    const int cpb32 = project32_cells_per_block(ncell, r);
    const int nblk32 = (ncell + cpb32 - 1) / cpb32;
    pa.cells_per_block = cpb32;
    static const char* fused = getenv("DLRSN_PROJECT_FUSED");
    auto* tm = proj_timer();
    if (fused && fused[0] == '1') {
      DLRSN_TRY_CUDA(zero_async(partial, sizeof(double) * (size_t)nblk32 * (7 * (size_t)r * r + r), st));
      DLRSN_TRY_CUDA(cudaFuncSetAttribute(project_mma32_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kProj32Smem));
      if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->first, st));
      project_mma32_kernel<<<dim3(tiles32, nblk32), 256, kProj32Smem, st>>>(pa, *ops);
      DLRSN_CHECK_LAUNCH("project_mma32_kernel");
      if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->second, st));
    } else {
      static bool attr = false;
      if (!attr) {
        DLRSN_TRY_CUDA(cudaFuncSetAttribute(project_mma32g_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kProj32SmemG));
        DLRSN_TRY_CUDA(cudaFuncSetAttribute(project_mma64d_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kProj64Smem));
        attr = true;
      }
      // both output groups in one grid (z = group); cell blocks of about
      // 4 waves over 2 CTAs per SM, so the unequal group costs even out
      const int cpbg = project32g_cells_per_block(ncell, r);
      const int nblkg = (ncell + cpbg - 1) / cpbg;
      pa.cells_per_block = cpbg;
      DLRSN_TRY_CUDA(zero_async(partial,
                                sizeof(double) * (size_t)(nblkg + kProjBndBlocks) * (7 * (size_t)r * r + r),
                                st));
      static const char* sym_env = getenv("DLRSN_PROJECT_SYM");
      const bool sym = !(sym_env && sym_env[0] == '0');
      const int T = (r + kT32 - 1) / kT32;
      const ProjTiles tl = project_tiles(r, sym);
      const bool d64 = sym && project_d64(r);
      if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->first, st));
      int nslots = nblkg;
      if (d64) {
        const int nb64 = (r + 63) / 64;
        project_mma64d_kernel<<<dim3(1, nblkg), 256, kProj64Smem, st>>>(pa, *ops, nb64, 1);
        DLRSN_CHECK_LAUNCH("project_mma64d_kernel");
        project_bnd64_kernel<<<kProjBndBlocks, 256, 0, st>>>(pa, *ops, (r + 63) / 64, nblkg);
        DLRSN_CHECK_LAUNCH("project_bnd64_kernel");
        nslots += kProjBndBlocks;
      }
      if (tl.n > 0) {
        project_mma32g_kernel<<<dim3(tl.n, nblkg), 256, kProj32SmemG, st>>>(pa, *ops, tl);
        DLRSN_CHECK_LAUNCH("project_mma32g_kernel");
      }
      if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->second, st));
      reduce_partials_kernel<<<(unsigned)((7 * (int64_t)r * r + r + 31) / 32), 1024, 0, st>>>(
          nslots, 7 * (int64_t)r * r + r, partial, out, 1.0);
      DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
      if (sym && T > 1) {
        mirror_tiles_kernel<<<(unsigned)((6 * r * r + 255) / 256), 256, 0, st>>>(r, out, d64 ? 1 : 0);
        DLRSN_CHECK_LAUNCH("mirror_tiles_kernel");
      }
      return DLRSN_OK;
    }
    const int64_t len32 = 7 * (int64_t)r * r + r;
    reduce_partials_kernel<<<(unsigned)((len32 + 31) / 32), 1024, 0, st>>>(nblk32, len32, partial,
                                                                           out, 1.0);
    DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
    return DLRSN_OK;
  }
  // partial slots not written by some tiles must be zero
  DLRSN_TRY_CUDA(zero_async(partial, sizeof(double) * (size_t)nblk * (7 * (size_t)r * r + r), st));
  auto* tm = proj_timer();
  if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->first, st));
  if (simt && simt[0] == '1') {
    project_kernel<<<dim3(nblk, tiles), kTile * kTile, 0, st>>>(pa, *ops);
    DLRSN_CHECK_LAUNCH("project_kernel");
  } else {
    project_mma_kernel<<<dim3(nblk, tiles), 256, 0, st>>>(pa, *ops);
    DLRSN_CHECK_LAUNCH("project_mma_kernel");
  }
  if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->second, st));
  const int64_t len = 7 * (int64_t)r * r + r;
  reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 1024, 0, st>>>(nblk, len, partial, out, 1.0);
  DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
  return DLRSN_OK;
}
}  // namespace dlrsn

extern "C" {

int dlrsn_chol_upper(int r, const double* G, double* R, double* Rinv, double* diag_ratio,
                     int* flag, dlrsn_stream_t stream) {
  const size_t smem = 2 * (size_t)r * r * sizeof(double);
  DLRSN_REQUIRE(r <= DLRSN_MAX_RANK, "rank %d too large for chol_upper", r);
  if (r <= 32) {
    if (r <= 16)
      chol_upper_warp_kernel<16><<<1, 32, 0, as_stream(stream)>>>(r, G, R, Rinv, diag_ratio, flag);
    else
      chol_upper_warp_kernel<32><<<1, 32, 0, as_stream(stream)>>>(r, G, R, Rinv, diag_ratio, flag);
    DLRSN_CHECK_LAUNCH("chol_upper_warp_kernel");
    return DLRSN_OK;
  }
  const int inv_global = smem > 200 * 1024;
  const size_t smem_used = inv_global ? smem / 2 : smem;
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(chol_upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem_used));
  chol_upper_kernel<<<1, 256, smem_used, as_stream(stream)>>>(r, G, R, Rinv, diag_ratio, flag,
                                                              inv_global);
  DLRSN_CHECK_LAUNCH("chol_upper_kernel");
  return DLRSN_OK;
}

int64_t dlrsn_cholqr2_small_smem(int n, int m) {
  const int64_t mt = m <= 16 ? 16 : 32, np = (n + 7) / 8 * 8;
  return (np * (mt + 1) + np + 3 * mt * mt + 8 * mt * mt) * (int64_t)sizeof(double);
}

int dlrsn_cholqr2_small(int n, int m, const double* W, int ldw, const double* w, double* Q,
                        int ldq, double* R, double* ratio, int* flag, int* deficient,
                        dlrsn_stream_t stream) {
  const int64_t smem = dlrsn_cholqr2_small_smem(n, m);
  DLRSN_REQUIRE(m >= 1 && m <= 32 && smem <= 200 * 1024,
                "cholqr2_small: %d x %d does not fit one CTA", n, m);
  cudaStream_t st = as_stream(stream);
  if (m <= 16) {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(cholqr2_small_kernel<16>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cholqr2_small_kernel<16><<<1, 256, smem, st>>>(n, m, W, ldw, w, Q, ldq, R, ratio, flag, deficient);
  } else {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(cholqr2_small_kernel<32>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cholqr2_small_kernel<32><<<1, 256, smem, st>>>(n, m, W, ldw, w, Q, ldq, R, ratio, flag, deficient);
  }
  DLRSN_CHECK_LAUNCH("cholqr2_small_kernel");
  return DLRSN_OK;
}

int dlrsn_small_matmul(int m, int k, int n, const double* A, const double* B, double* C,
                       int transA, dlrsn_stream_t stream) {
  const int blocks = (m * n + 255) / 256 < 64 ? (m * n + 255) / 256 : 64;
  small_matmul_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, as_stream(stream)>>>(m, k, n, A, B, C, transA);
  DLRSN_CHECK_LAUNCH("small_matmul_kernel");
  return DLRSN_OK;
}

int dlrsn_row_inverse(int n, int r, const double* proj, const double* om_sel, double* Binv,
                      double* Bout, int* status, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(r >= 1 && r <= DLRSN_MAX_RANK, "rank %d too large for row_inverse", r);
  const size_t smem = 2 * (size_t)r * r * sizeof(double);
  if (n == 0) return DLRSN_OK;
  if (smem <= 200 * 1024) {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    row_inverse_kernel<<<n, 256, smem, as_stream(stream)>>>(r, proj, om_sel, Binv, Bout, status);
    DLRSN_CHECK_LAUNCH("row_inverse_kernel");
  } else {
    const size_t sm1 = (size_t)r * r * sizeof(double);
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_inverse_inplace_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    row_inverse_inplace_kernel<<<n, 256, sm1, as_stream(stream)>>>(r, proj, om_sel, Binv, Bout,
                                                                   status);
    DLRSN_CHECK_LAUNCH("row_inverse_inplace_kernel");
  }
  return DLRSN_OK;
}

int dlrsn_row_combine(int n, int r, const double* Binv, const double* ms, const double* Q,
                      const double* wts, double* L, double* lbar, int* status,
                      dlrsn_stream_t stream) {
  size_t smem = (2 * (size_t)r * r + 2 * r) * sizeof(double) + r * sizeof(int);
  const int in_l = smem > 200 * 1024 && n >= r;
  if (in_l) smem -= (size_t)r * r * sizeof(double);
  DLRSN_REQUIRE(smem <= 200 * 1024, "rank %d too large for row_combine", r);
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(row_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  row_combine_kernel<<<1, 256, smem, as_stream(stream)>>>(n, r, Binv, ms, Q, wts, L, lbar, status,
                                                          in_l);
  DLRSN_CHECK_LAUNCH("row_combine_kernel");
  return DLRSN_OK;
}

int dlrsn_deim(int n, int r, double* Wwork, const double* W, int* idx, double* Lhat, double* U,
               int* err_col, double* gap, int variant, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(r <= n, "rank %d exceeds the %d available nodes", r, n);
  DLRSN_REQUIRE(r <= DLRSN_MAX_RANK, "rank %d exceeds DLRSN_MAX_RANK", r);
  DLRSN_REQUIRE(variant >= 0 && variant <= 4, "unknown DEIM variant %d", variant);
  static const char* ereg = getenv("DLRSN_DEIM_REG");
  const bool reg_ok = n <= 1024 && r <= 16;
  DLRSN_REQUIRE(variant != 1 || reg_ok, "register DEIM needs n <= 1024, r <= 16");
  if (variant == 1 || (variant == 0 && reg_ok && !(ereg && ereg[0] == '0'))) {
    // register variant: 46 -> 36 us per step on config 2 (n = 1024, r = 16)
    deim_reg_kernel<16><<<1, (n + 31) / 32 * 32, 0, as_stream(stream)>>>(n, r, W, idx, Lhat, U,
                                                                       err_col, gap);
    DLRSN_CHECK_LAUNCH("deim_reg_kernel");
    return DLRSN_OK;
  }
  // cluster variant: about 256 rows per CTA, up to 16 CTAs (non-portable
  // cluster size, checked against the occupancy calculator once)
  static const char* ecs = getenv("DLRSN_DEIM_CS");
  int cs = 1;
  if (ecs) cs = atoi(ecs);
  else while (cs < 16 && cs * 256 < n) cs *= 2;
  auto csmem = [&](int c) {
    const int64_t nl = (n + c - 1) / c;
    return (nl * r + 2 * (r + 3) + r) * (int64_t)sizeof(double) + nl;
  };
  while (cs < 16 && csmem(cs) > 200 * 1024) cs *= 2;
  static int max_cs = 0;
  if (max_cs == 0) {
    max_cs = 8;
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(deim_cluster_kernel,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(deim_cluster_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(16);
    qc.blockDim = dim3(kDeimCT);
    qc.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute qa;
    qa.id = cudaLaunchAttributeClusterDimension;
    qa.val.clusterDim.x = 16;
    qa.val.clusterDim.y = qa.val.clusterDim.z = 1;
    qc.attrs = &qa;
    qc.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, deim_cluster_kernel, &qc) == cudaSuccess && ncl > 0)
      max_cs = 16;
    cudaGetLastError();
  }
  const bool cl_ok = cs >= 1 && cs <= max_cs && csmem(cs) <= 200 * 1024;
  DLRSN_REQUIRE(variant != 2 || cl_ok, "cluster DEIM does not fit n = %d, r = %d", n, r);
  if (variant == 2 || (variant == 0 && cl_ok)) {
    const int nl = (n + cs - 1) / cs;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(kDeimCT);
    lc.dynamicSmemBytes = (size_t)csmem(cs);
    lc.stream = as_stream(stream);
    cudaLaunchAttribute la;
    la.id = cudaLaunchAttributeClusterDimension;
    la.val.clusterDim.x = cs;
    la.val.clusterDim.y = la.val.clusterDim.z = 1;
    lc.attrs = &la;
    lc.numAttrs = 1;
    DLRSN_TRY_CUDA(cudaLaunchKernelEx(&lc, deim_cluster_kernel, n, r, nl, W, idx, Lhat, U, err_col,
                                      gap));
    DLRSN_CHECK_LAUNCH("deim_cluster_kernel");
    return DLRSN_OK;
  }
  // grid variant: rows spread over the GPU's SMs (one cooperative launch)
  {
    static int sms = 0;
    if (sms == 0) {
      int dev = 0;
      DLRSN_TRY_CUDA(cudaGetDevice(&dev));
      DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int G = std::min(sms, std::max(1, (n + 63) / 64));
    const int nl = (n + G - 1) / G;
    G = (n + nl - 1) / nl;
    const size_t gsm = ((size_t)nl * r + r) * sizeof(double) + nl;
    const bool g_ok = gsm <= 200 * 1024 && Wwork != nullptr &&
                      (int64_t)n * r >= (int64_t)2 * G * (r + 3) + G;
    DLRSN_REQUIRE(variant != 4 || g_ok, "grid DEIM does not fit n = %d, r = %d", n, r);
    if (variant == 4 || (variant == 0 && g_ok && (int64_t)n * r * 8 > 200 * 1024)) {
      DLRSN_TRY_CUDA(cudaFuncSetAttribute(deim_grid_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
      int nn = n, rr = r, nll = nl;
      void* args[] = {&nn, &rr, &nll, (void*)&W, &idx, &Lhat, &U, &err_col, &gap, &Wwork};
      DLRSN_TRY_CUDA(cudaLaunchCooperativeKernel((void*)deim_grid_kernel, dim3(G), dim3(kDeimGT),
                                                 args, gsm, as_stream(stream)));
      DLRSN_CHECK_LAUNCH("deim_grid_kernel");
      return DLRSN_OK;
    }
  }
  const size_t smem = (size_t)n * r * sizeof(double) + (size_t)n;
  const int in_smem = smem <= 200 * 1024;
  if (in_smem)
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(deim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  static const char* dt = getenv("DLRSN_DEIM_THREADS");
  const int threads = dt ? atoi(dt) : 256;  // 256 / 512 equal, 1024 slower (C2)
  DLRSN_REQUIRE(in_smem || Wwork, "DEIM needs a work copy of W for n = %d, r = %d", n, r);
  deim_kernel<<<1, threads, in_smem ? smem : 0, as_stream(stream)>>>(n, r, Wwork, W, idx, Lhat, U,
                                                                 err_col, in_smem, gap);
  DLRSN_CHECK_LAUNCH("deim_kernel");
  return DLRSN_OK;
}

int dlrsn_what_solve(int r, int m, const double* Lhat, const double* U, const double* V,
                     double* X, int mode, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(r >= 1 && r <= DLRSN_MAX_RANK && m >= 1, "bad W_hat solve shape (%d, %d)", r, m);
  size_t smem = 2 * (size_t)r * r * sizeof(double);
  const int fg = smem > 200 * 1024;
  if (fg) smem = 0;
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(what_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  const int threads = 32 * std::min(32, m);
  what_solve_kernel<<<1, threads, smem, as_stream(stream)>>>(r, m, Lhat, U, V, X, mode, fg);
  DLRSN_CHECK_LAUNCH("what_solve_kernel");
  return DLRSN_OK;
}

}  // extern "C"
