// Exact twice-projected classical Gram-Schmidt (angular.py:104-160) as one
// cooperative grid launch.
//
// Same contract as the reference: columns = Q R, R upper triangular with
// R_kk = the M-norm left after two projection passes; a column whose norm
// drops to <= 1e-12 * max(orig, 1) is deficient (R_kk = 0) and its Q column
// is the first completion candidate that keeps > 1e-6 * max(|cand|, 1) after
// two passes (deterministic candidate stream shared across columns).
//
// Parallel layout: block b owns a contiguous range of "units" (rows for the
// weighted angular metric, cells = 4 rows for the block-mass metric); every
// inner product is a block partial sum + one grid.sync + a fixed-order sum of
// the per-block partials that every block performs redundantly, so all blocks
// take identical (deterministic) decisions without further communication.
#include <cooperative_groups.h>

#include <cmath>
#include <cstring>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace dlrsn {

constexpr int kCgT = 256;  // threads per block
constexpr int kCgCh = 16;  // coefficients reduced per grid sync

struct Cgs2Args {
  int n, m;
  const double* cols;
  int ldc;
  double* Q;
  int ldq;
  double* R;         // m x m
  int* deficient;    // m flags
  int metric;        // 0: weighted rows, 1: per-cell mass blocks
  const double* w;   // metric 0 weights (n)
  dlrsn_cellops ops; // metric 1 mass
  int comp_kind;     // 0: angular monomials + unit vectors, 1: spatial monomials
  int ncomp;
  const int* comp_exp;
  const double* coords;  // kind 0: omegas (n x 3); kind 1: extent (x0,y0,lx,ly)
  double* work;          // n doubles
  double* part;          // 2 x gridDim x kCgCh doubles
  int* status;
  int strict;
};

__device__ double cand_value(const Cgs2Args& g, int k, int i) {
  if (g.comp_kind == 0) {
    if (k < g.ncomp) {
      const double* o = g.coords + 3 * (int64_t)i;
      const int* e = g.comp_exp + 3 * k;
      double vx = 1.0, vy = 1.0, vz = 1.0;
      for (int p = 0; p < e[0]; ++p) vx *= o[0];
      for (int p = 0; p < e[1]; ++p) vy *= o[1];
      for (int p = 0; p < e[2]; ++p) vz *= o[2];
      return vx * vy * vz;
    }
    return (k - g.ncomp) == i ? 1.0 : 0.0;
  }
  // spatial monomials at dof i: corner coordinates of cell i/4 (mesh.py:251-265)
  const int c = i >> 2, l = i & 3;
  const int nx = g.ops.nx;
  const double x = (g.ops.x0 + (c % nx) * g.ops.dx) + (l & 1) * g.ops.dx;
  const double y = (g.ops.y0 + (c / nx) * g.ops.dy) + (l >> 1) * g.ops.dy;
  const double xh = 2.0 * (x - g.coords[0]) / g.coords[2] - 1.0;
  const double yh = 2.0 * (y - g.coords[1]) / g.coords[3] - 1.0;
  const int* e = g.comp_exp + 2 * k;
  double vx = 1.0, vy = 1.0;
  for (int p = 0; p < e[0]; ++p) vx *= xh;
  for (int p = 0; p < e[1]; ++p) vy *= yh;
  return vx * vy;
}

// grid barrier; a single-block launch only needs the block barrier
__device__ inline void gsync(cg::grid_group& grid) {
  if (gridDim.x == 1)
    __syncthreads();
  else
    grid.sync();
}

struct Cgs2State {
  int u0, u1;  // unit range of this block
  int rpu;     // rows per unit (1 or 4)
  int buf;     // partial double-buffer index
};

// grid-wide sum of nv (<= kCgCh) per-thread values; result in out[0..nv)
__device__ void grid_sum(cg::grid_group& grid, const Cgs2Args& g, Cgs2State& s, double* v, int nv,
                         double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < kCgCh; ++j) {
    if (j < nv) {
      double x = v[j];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(kFull, x, o);
      if (lane == 0) red[wid * kCgCh + j] = x;
    }
  }
  __syncthreads();
  if (gridDim.x == 1) {  // single block: no global round trip
    if (threadIdx.x < nv) {
      double x = 0.0;
      for (int q = 0; q < nw; ++q) x += red[q * kCgCh + threadIdx.x];
      out[threadIdx.x] = x;
    }
    __syncthreads();
    return;
  }
  double* mine = g.part + ((int64_t)s.buf * gridDim.x + blockIdx.x) * kCgCh;
  if (threadIdx.x < nv) {
    double x = 0.0;
    for (int q = 0; q < nw; ++q) x += red[q * kCgCh + threadIdx.x];
    mine[threadIdx.x] = x;
  }
  gsync(grid);
  if (threadIdx.x < nv) {
    const double* all = g.part + (int64_t)s.buf * gridDim.x * kCgCh;
    double x = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) x += __ldcg(all + (int64_t)b * kCgCh + threadIdx.x);
    out[threadIdx.x] = x;
  }
  s.buf ^= 1;
  __syncthreads();
}

// metric-applied work vector for one unit: mw[l] (rpu values)
__device__ inline void metric_apply(const Cgs2Args& g, int u, double* x, double* mw) {
  if (g.metric == 0) {
    mw[0] = g.w[u] * x[0];
  } else {
#pragma unroll
    for (int l = 0; l < 4; ++l)
      mw[l] = g.ops.mass[4 * l] * x[0] + g.ops.mass[4 * l + 1] * x[1] +
              g.ops.mass[4 * l + 2] * x[2] + g.ops.mass[4 * l + 3] * x[3];
  }
}

__device__ inline void load_unit(const Cgs2Args& g, const Cgs2State& s, int u, double* x) {
  for (int l = 0; l < s.rpu; ++l) x[l] = g.work[(int64_t)u * s.rpu + l];
}

// <work, work> in the metric
__device__ double norm2(cg::grid_group& grid, const Cgs2Args& g, Cgs2State& s, double* red,
                        double* out) {
  double acc = 0.0;
  for (int u = s.u0 + threadIdx.x; u < s.u1; u += blockDim.x) {
    double x[4], mw[4];
    load_unit(g, s, u, x);
    metric_apply(g, u, x, mw);
    for (int l = 0; l < s.rpu; ++l) acc += x[l] * mw[l];
  }
  double v[1] = {acc};
  grid_sum(grid, g, s, v, 1, red, out);
  return out[0];
}

// two classical projection passes of work against Q[:, :k]; total (if
// non-null) accumulates the coefficients of both passes
__device__ void project_twice(cg::grid_group& grid, const Cgs2Args& g, Cgs2State& s, int k,
                              double* red, double* coef, double* total) {
  for (int pass = 0; pass < 2; ++pass) {
    for (int i0 = 0; i0 < k; i0 += kCgCh) {
      const int nv = min(kCgCh, k - i0);
      double v[kCgCh];
#pragma unroll
      for (int j = 0; j < kCgCh; ++j) v[j] = 0.0;
      for (int u = s.u0 + threadIdx.x; u < s.u1; u += blockDim.x) {
        double x[4], mw[4];
        load_unit(g, s, u, x);
        metric_apply(g, u, x, mw);
        for (int l = 0; l < s.rpu; ++l) {
          const double* qrow = g.Q + ((int64_t)u * s.rpu + l) * g.ldq + i0;
#pragma unroll
          for (int j = 0; j < kCgCh; ++j)
            if (j < nv) v[j] += qrow[j] * mw[l];
        }
      }
      grid_sum(grid, g, s, v, nv, red, coef + i0);
    }
    if (total)
      for (int i = threadIdx.x; i < k; i += blockDim.x) total[i] = pass == 0 ? coef[i] : total[i] + coef[i];
    // work -= Q[:, :k] coef  (own rows only)
    for (int64_t r = (int64_t)s.u0 * s.rpu + threadIdx.x; r < (int64_t)s.u1 * s.rpu; r += blockDim.x) {
      double x = g.work[r];
      const double* qrow = g.Q + r * g.ldq;
      for (int i = 0; i < k; ++i) x -= qrow[i] * coef[i];
      g.work[r] = x;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCgT) cgs2_grid_kernel(Cgs2Args g) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* red = sm;                       // 8 warps x kCgCh
  double* coef = red + 8 * kCgCh;         // m
  double* total = coef + g.m;             // m
  __shared__ double out[kCgCh];
  const double tol = 1e-12;  // DEFICIENCY_TOL (angular.py:24)
  Cgs2State s;
  s.rpu = g.metric == 0 ? 1 : 4;
  const int units = g.n / s.rpu;
  const int per = (units + gridDim.x - 1) / gridDim.x;
  s.u0 = min(units, (int)blockIdx.x * per);
  s.u1 = min(units, s.u0 + per);
  s.buf = 0;
  const int64_t r0 = (int64_t)s.u0 * s.rpu, r1 = (int64_t)s.u1 * s.rpu;
  int next_cand = 0;
  const int max_cand = g.comp_kind == 0 ? g.ncomp + g.n : g.ncomp;

  for (int k = 0; k < g.m; ++k) {
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) g.work[r] = g.cols[r * g.ldc + k];
    __syncthreads();
    const double orig = sqrt(fmax(norm2(grid, g, s, red, out), 0.0));
    project_twice(grid, g, s, k, red, coef, total);
    const double nrm = sqrt(fmax(norm2(grid, g, s, red, out), 0.0));
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < g.m; i += blockDim.x) g.R[(int64_t)i * g.m + k] = i < k ? total[i] : 0.0;
    if (nrm <= tol * fmax(orig, 1.0)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) g.deficient[k] = 1;
      bool placed = false;
      while (next_cand < max_cand) {
        const int cand = next_cand++;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) g.work[r] = cand_value(g, cand, (int)r);
        __syncthreads();
        const double c0 = sqrt(fmax(norm2(grid, g, s, red, out), 0.0));
        project_twice(grid, g, s, k, red, coef, nullptr);
        const double c1 = sqrt(fmax(norm2(grid, g, s, red, out), 0.0));
        if (c1 > sqrt(tol) * fmax(c0, 1.0)) {
          for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) g.Q[r * g.ldq + k] = g.work[r] / c1;
          placed = true;
          break;
        }
      }
      if (!placed) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && g.strict) *g.status = 1;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) g.Q[r * g.ldq + k] = 0.0;
      }
    } else {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        g.deficient[k] = 0;
        g.R[(int64_t)k * g.m + k] = nrm;
      }
      for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) g.Q[r * g.ldq + k] = g.work[r] / nrm;
    }
    // Q[:, k] must be visible grid-wide before the next column's projections
    gsync(grid);
  }
}

// Single-CTA variant with Q, the work vector and the weights resident in
// shared memory (used when n (m + 2) doubles fit): every inner product is a
// block reduction, no global round trips.  Same operation order and
// decisions as cgs2_grid_kernel.
constexpr int kSmT = 1024;

__device__ double block_dot(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < nw; ++q) s += red[q];
  return s;
}

__global__ void __launch_bounds__(kSmT) cgs2_smem_kernel(Cgs2Args g) {
  extern __shared__ double sm[];
  const int n = g.n, m = g.m;
  const int lq = m | 1;                  // odd row stride: conflict-free column walks
  double* Qs = sm;                       // n x lq
  double* work = Qs + (size_t)n * lq;    // n
  double* wts = work + n;                // n (metric 0 weights)
  double* coef = wts + n;                // m
  double* total = coef + m;              // m
  __shared__ double red[32];
  const double tol = 1e-12;
  const int rpu = g.metric == 0 ? 1 : 4;
  const int units = n / rpu;
  for (int i = threadIdx.x; i < n; i += blockDim.x) wts[i] = g.metric == 0 ? g.w[i] : 0.0;
  __syncthreads();

  auto mw_of = [&](int u, int l) -> double {  // (metric applied to work)[u*rpu + l]
    if (rpu == 1) return wts[u] * work[u];
    const double* x = work + 4 * u;
    return g.ops.mass[4 * l] * x[0] + g.ops.mass[4 * l + 1] * x[1] + g.ops.mass[4 * l + 2] * x[2] +
           g.ops.mass[4 * l + 3] * x[3];
  };
  auto norm2 = [&]() -> double {
    double acc = 0.0;
    for (int u = threadIdx.x; u < units; u += blockDim.x)
      for (int l = 0; l < rpu; ++l) acc += work[u * rpu + l] * mw_of(u, l);
    return block_dot(acc, red);
  };
  // mw = metric applied to work, materialised once per pass; then warp w
  // computes the coefficients i = w, w + 32, ... over all rows (lane-strided,
  // shuffle-reduced: fixed order), one block barrier per pass
  double* mw = total + m;                // n
  auto project_twice = [&](int k, bool keep) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int pass = 0; pass < 2; ++pass) {
      for (int u = threadIdx.x; u < units; u += blockDim.x)
        for (int l = 0; l < rpu; ++l) mw[u * rpu + l] = mw_of(u, l);
      __syncthreads();
      for (int i = wid; i < k; i += nw) {
        double acc = 0.0;
        for (int r = lane; r < n; r += 32) acc += Qs[(size_t)r * lq + i] * mw[r];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
        if (lane == 0) {
          coef[i] = acc;
          if (keep) total[i] = pass == 0 ? acc : total[i] + acc;
        }
      }
      __syncthreads();
      for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double x = work[r];
        for (int i = 0; i < k; ++i) x -= Qs[(size_t)r * lq + i] * coef[i];
        work[r] = x;
      }
      __syncthreads();
    }
  };

  int next_cand = 0;
  const int max_cand = g.comp_kind == 0 ? g.ncomp + n : g.ncomp;
  for (int k = 0; k < m; ++k) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) work[r] = g.cols[(int64_t)r * g.ldc + k];
    __syncthreads();
    const double orig = sqrt(fmax(norm2(), 0.0));
    project_twice(k, true);
    const double nrm = sqrt(fmax(norm2(), 0.0));
    for (int i = threadIdx.x; i < m; i += blockDim.x) g.R[(int64_t)i * m + k] = i < k ? total[i] : 0.0;
    if (nrm <= tol * fmax(orig, 1.0)) {
      if (threadIdx.x == 0) g.deficient[k] = 1;
      bool placed = false;
      while (next_cand < max_cand) {
        const int cand = next_cand++;
        for (int r = threadIdx.x; r < n; r += blockDim.x) work[r] = cand_value(g, cand, r);
        __syncthreads();
        const double c0 = sqrt(fmax(norm2(), 0.0));
        project_twice(k, false);
        const double c1 = sqrt(fmax(norm2(), 0.0));
        if (c1 > sqrt(tol) * fmax(c0, 1.0)) {
          for (int r = threadIdx.x; r < n; r += blockDim.x) Qs[(size_t)r * lq + k] = work[r] / c1;
          placed = true;
          break;
        }
      }
      if (!placed) {
        if (threadIdx.x == 0 && g.strict) *g.status = 1;
        for (int r = threadIdx.x; r < n; r += blockDim.x) Qs[(size_t)r * lq + k] = 0.0;
      }
    } else {
      if (threadIdx.x == 0) {
        g.deficient[k] = 0;
        g.R[(int64_t)k * m + k] = nrm;
      }
      for (int r = threadIdx.x; r < n; r += blockDim.x) Qs[(size_t)r * lq + k] = work[r] / nrm;
    }
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < (int64_t)n * m; e += blockDim.x)
    g.Q[(e / m) * g.ldq + e % m] = Qs[(size_t)(e / m) * lq + e % m];
}

}  // namespace dlrsn

using namespace dlrsn;

extern "C" {

int64_t dlrsn_cgs2_workspace_len(int n) { return (int64_t)n + 2 * 148 * 8 * kCgCh + 64; }

int dlrsn_cgs2(int n, int m, const double* cols, int ldc, double* Q, int ldq, double* R,
               int* deficient, int metric, const double* w, const dlrsn_cellops* ops,
               int comp_kind, int ncomp, const int* comp_exp, const double* coords,
               double* workspace, int* status, int strict, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(metric == 0 || metric == 1, "bad metric");
  DLRSN_REQUIRE(metric == 0 || (ops && n % 4 == 0), "block-mass metric needs 4 rows per cell");
  if (m == 0) return DLRSN_OK;
  Cgs2Args g;
  g.n = n; g.m = m; g.cols = cols; g.ldc = ldc; g.Q = Q; g.ldq = ldq; g.R = R;
  g.deficient = deficient; g.metric = metric; g.w = w;
  if (ops) g.ops = *ops; else memset(&g.ops, 0, sizeof(g.ops));
  g.comp_kind = comp_kind; g.ncomp = ncomp; g.comp_exp = comp_exp; g.coords = coords;
  g.work = workspace;
  g.status = status; g.strict = strict;
  const size_t lq = (size_t)(m | 1);
  const size_t smem_res = ((size_t)n * lq + 3 * (size_t)n + 2 * (size_t)m) * sizeof(double);
  if (smem_res <= 200 * 1024 && (metric == 0 || n <= 16384)) {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(cgs2_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem_res));
    cgs2_smem_kernel<<<1, kSmT, smem_res, as_stream(stream)>>>(g);
    DLRSN_CHECK_LAUNCH("cgs2_smem_kernel");
    return DLRSN_OK;
  }
  int dev = 0, sms = 0, occ = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = (8 * kCgCh + 2 * (size_t)m) * sizeof(double);
  DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cgs2_grid_kernel, kCgT, smem));
  const int units = metric == 0 ? n : n / 4;
  int blocks = (units + 4 * kCgT - 1) / (4 * kCgT);  // >= 4 units per thread
  const int cap = sms * (occ < 1 ? 1 : (occ > 8 ? 8 : occ));
  if (blocks > cap) blocks = cap;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  g.part = workspace + ((n + 7) / 8) * 8;
  void* params[] = {&g};
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  DLRSN_TRY_CUDA(cudaLaunchCooperativeKernel((const void*)cgs2_grid_kernel, dim3(blocks), dim3(kCgT),
                                             params, smem, as_stream(stream)));
  return DLRSN_OK;
}

}  // extern "C"
