// Native orchestration of one DLR-SN step (dlr_sn.py:86-151) in a single
// C-ABI call: the ~45 kernel launches of the step are issued from C++ with
// few host synchronisations (DEIM picks + closure + input checks, one per
// source iteration, the final status readback), so the Python host stays off
// the critical path.  Memory comes from a caller-owned workspace carved by a
// bump arena (dlrsn_step_workspace_bytes); small host transfers go through a
// pinned staging block owned by the library.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sweep_common.cuh"

namespace dlrsn {

// ---- small glue kernels (r <= 128, one CTA) -------------------------------

// K[i][d] = sum_j S[i][j] W[idx[d]][j] (evaluate_rows, lowrank.py:220-227);
// Sb = S beta (scalar_flux, :60-62); om_sel = omegas[idx]
__global__ void ks_kernel(int r, const double* __restrict__ S, const double* __restrict__ W,
                          const int* __restrict__ idx, const double* __restrict__ beta,
                          double* __restrict__ K, double* __restrict__ Sb,
                          const double* __restrict__ omegas, double* __restrict__ om_sel) {
  // a warp per output, lanes along the contraction index (coalesced row
  // reads of S and of the gathered W rows; a thread per output made every
  // warp load touch 32 different rows of W); rows spread over the CTAs
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (K)
    for (int i = blockIdx.x; i < r; i += gridDim.x)
      for (int d = warp; d < r; d += nw) {
        const double* w = W + (int64_t)idx[d] * r;
        double s = 0.0;
        for (int j = lane; j < r; j += 32) s = fma(S[i * r + j], w[j], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (lane == 0) K[i * r + d] = s;
      }
  if (Sb)
    for (int i = blockIdx.x * nw + warp; i < r; i += gridDim.x * nw) {
      double s = 0.0;
      for (int j = lane; j < r; j += 32) s = fma(S[i * r + j], beta[j], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
      if (lane == 0) Sb[i] = s;
    }
  if (om_sel && blockIdx.x == 0)
    for (int e = threadIdx.x; e < 3 * r; e += blockDim.x)
      om_sel[e] = omegas[(int64_t)idx[e / 3] * 3 + e % 3];
}

// *out |= any(sigma_t - sigma_s <= 0)  (transport_sn.py:208-209)
__global__ void sigma_check_kernel(int n, const double* __restrict__ st,
                                   const double* __restrict__ ss, int* out) {
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (!(st[i] - ss[i] > 0.0)) bad = 1;
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(out, 1);
}

// Gw = W^T diag(w) W and W^T w over row blocks (DlrState.check,
// lowrank.py:68-81; beta = W^T w, angular.py:181-183): per-block partials,
// summed in block order by reduce_partials_kernel (dense.cu).
static int wgram_rows(int r) { return std::max(1, std::min(64, 4096 / r)); }

__global__ void wgram_part_kernel(int n, int r, int rows, const double* __restrict__ W,
                                  const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double sW[4096];
  __shared__ double sw[64];
  const int k0 = blockIdx.x * rows;
  const int nr = min(rows, n - k0);
  for (int e = threadIdx.x; e < nr * r; e += blockDim.x) sW[e] = W[(int64_t)k0 * r + e];
  for (int e = threadIdx.x; e < nr; e += blockDim.x) sw[e] = w[k0 + e];
  __syncthreads();
  const int len = r * r + r;
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    double s = 0.0;
    if (e < r * r) {
      const int i = e / r, j = e % r;
      for (int k = 0; k < nr; ++k) s = fma(sw[k] * sW[k * r + i], sW[k * r + j], s);
    } else {
      const int j = e - r * r;
      for (int k = 0; k < nr; ++k) s = fma(sw[k], sW[k * r + j], s);
    }
    part[(int64_t)blockIdx.x * len + e] = s;
  }
}

__global__ void reduce_partials_kernel(int nchunks, int64_t len, const double* __restrict__ part,
                                       double* __restrict__ out, double alpha);

static int wgram(int n, int r, const double* W, const double* w, double* part, double* out,
                 cudaStream_t st) {
  const int rows = wgram_rows(r);
  const int nb = (n + rows - 1) / rows;
  const int64_t len = (int64_t)r * r + r;
  wgram_part_kernel<<<nb, 256, 0, st>>>(n, r, rows, W, w, part);
  DLRSN_CHECK_LAUNCH("wgram_part_kernel");
  reduce_partials_kernel<<<(unsigned)((len + 31) / 32), 256, 0, st>>>(nb, len, part, out, 1.0);
  DLRSN_CHECK_LAUNCH("reduce_partials_kernel");
  return DLRSN_OK;
}

// out[0] = max |Gx - I|, out[1] = max |Gw - I| (DlrState.check, lowrank.py:68-81)
// Gx == nullptr: the spatial residual is already known (*x_known, written
// by the step that produced X); x_copy (optional) receives out[0].
__global__ void ortho_residual_kernel(int r, const double* __restrict__ Gx,
                                      const double* __restrict__ Gw, double* out,
                                      const double* x_known = nullptr, double* x_copy = nullptr) {
  __shared__ double red[2][32];
  double m[2] = {0.0, 0.0};
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const double d = (e / r == e % r) ? 1.0 : 0.0;
    if (Gx) m[0] = fmax(m[0], fabs(Gx[e] - d));
    m[1] = fmax(m[1], fabs(Gw[e] - d));
  }
  if (!Gx && threadIdx.x == 0) m[0] = *x_known;
  for (int q = 0; q < 2; ++q) {
    double v = m[q];
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(kFull, v, o));
    if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double v = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) v = fmax(v, red[threadIdx.x][k]);
    out[threadIdx.x] = v;
    if (threadIdx.x == 0 && x_copy) *x_copy = v;
  }
}

// q_all[d][j] = qhat[j] + inv_cdt * (W_sel (S^T mo))[d][j]  (dlr_sn.py:130-131)
// + sum_w max(-omega_d.n_w, 0) psi_b,w h[w][j]: the projected inflow load of
// the selected direction d (isotropic inflow walls, h = X_new^T g_w; hin null
// for vacuum walls, the reference's case)
__global__ void __launch_bounds__(1024) qall_kernel(int r, const double* __restrict__ S, const double* __restrict__ mo,
                            const double* __restrict__ qhat, const double* __restrict__ W,
                            const int* __restrict__ idx, double inv_cdt, double* __restrict__ T,
                            double* __restrict__ qall, const double* __restrict__ hin,
                            Inflow4 inflow, const double* __restrict__ om_sel, int staged) {
  // staged (3 r^2 doubles of shared memory): S, mo and T in shared memory
  extern __shared__ double sq[];
  const double* sS = staged ? sq : S;
  const double* sM = staged ? sq + r * r : mo;
  double* sT = staged ? sq + 2 * r * r : T;
  if (staged) {
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
      sq[e] = S[e];
      sq[r * r + e] = mo[e];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int i = e / r, j = e % r;
    double s = 0.0;
    for (int k = 0; k < r; ++k) s = fma(sS[k * r + i], sM[k * r + j], s);
    sT[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int d = e / r, j = e % r;
    const double* w = W + (int64_t)idx[d] * r;
    double s = 0.0;
    for (int i = 0; i < r; ++i) s = fma(w[i], sT[i * r + j], s);
    double v = qhat[j] + inv_cdt * s;
    if (hin) {
      const double ox = om_sel[3 * d], oy = om_sel[3 * d + 1];
      const double c[4] = {inflow.v[0] * fmax(ox, 0.0), inflow.v[1] * fmax(-ox, 0.0),
                           inflow.v[2] * fmax(oy, 0.0), inflow.v[3] * fmax(-oy, 0.0)};
      double a = 0.0;
#pragma unroll
      for (int w = 0; w < 4; ++w) a = fma(c[w], hin[w * r + j], a);
      v += a;
    }
    qall[e] = v;
  }
}

// S_new = R^T (dlr_sn.py:139); beta_new from the wgram output
__global__ void finish_kernel(int r, const double* __restrict__ R, const double* __restrict__ wg,
                              double* __restrict__ S_new, double* __restrict__ beta_new) {
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) S_new[e] = R[(e % r) * r + e / r];
  for (int j = threadIdx.x; j < r; j += blockDim.x) beta_new[j] = wg[r * r + j];
}

// Step start in one launch: zero the control words (flags, statuses, the
// combine's block counter, the iteration control) and write the completion
// exponents (spatial_monomials / angular_monomials, angular.py:198-214) and
// the domain extent used by the CGS2 completion candidates.
struct InitArgs {
  int* flags;
  int* statw;
  int* statx;
  void* red_ws;
  SiCtl* ctl;
  int* sexp;
  int* aexp;
  double* extent;
  int count;  // r + 8 candidates
  double x0, y0, lx, ly;
};

__global__ void init_kernel(InitArgs a) {
  const int t = threadIdx.x;
  if (t < 8) a.flags[t] = 0;
  if (t < 64) reinterpret_cast<unsigned*>(a.red_ws)[t] = 0u;
  if (t == 0) {
    *a.statw = 0;
    *a.statx = 0;
    memset(a.ctl, 0, sizeof(SiCtl));
    a.extent[0] = a.x0;
    a.extent[1] = a.y0;
    a.extent[2] = a.lx;
    a.extent[3] = a.ly;
  } else if (t == 32) {
    int cnt = 0;
    for (int deg = 0; cnt < a.count; ++deg)
      for (int x = deg; x >= 0 && cnt < a.count; --x, ++cnt) {
        a.sexp[2 * cnt] = x;
        a.sexp[2 * cnt + 1] = deg - x;
      }
  } else if (t == 64) {
    int cnt = 1;
    a.aexp[0] = a.aexp[1] = a.aexp[2] = 0;
    for (int deg = 1; cnt < a.count; ++deg)
      for (int kx = deg; kx >= 0 && cnt < a.count; --kx)
        for (int ky = deg - kx; ky >= 0 && cnt < a.count; --ky, ++cnt) {
          a.aexp[3 * cnt] = kx;
          a.aexp[3 * cnt + 1] = ky;
          a.aexp[3 * cnt + 2] = deg - kx - ky;
        }
  }
}

// Readback packing: copy scattered device words into one staging block so
// that a single device-to-host copy carries every status of the step.
struct PackList {
  const unsigned* src[24];
  int words[24];
  int off[24];
  int n;
};

__global__ void pack_kernel(PackList l, unsigned* __restrict__ dst) {
  for (int k = 0; k < l.n; ++k)
    for (int w = threadIdx.x; w < l.words[k]; w += blockDim.x) dst[l.off[k] + w] = l.src[k][w];
}

// Forced DEIM selection (the angle_indices override of a step): the picks
// come from the caller, W_hat = W[idx, :] is factored as Lhat U without
// further pivoting (the factorisation DEIM's elimination produces when it
// picks these rows in this order); err_col = j if pivot j vanishes below the
// DEIM floor (lowrank.py:185,192-199) or an index repeats / is out of range.
struct ForcedPicks {
  int idx[DLRSN_MAX_RANK];
};
__global__ void deim_forced_kernel(int n, int r, const double* __restrict__ W, ForcedPicks fp,
                                   int* __restrict__ idx_out, double* __restrict__ Lhat,
                                   double* __restrict__ U, int* __restrict__ err_col,
                                   double* __restrict__ gap) {
  extern __shared__ double a[];  // r x r, row q = W[idx[q], :]
  __shared__ double s_mx;
  __shared__ int s_bad;
  const int t = threadIdx.x;
  if (t == 0) {
    s_bad = -1;
    for (int q = 0; q < r && s_bad < 0; ++q) {
      bool bad = fp.idx[q] < 0 || fp.idx[q] >= n;
      for (int e = 0; e < q; ++e) bad |= fp.idx[e] == fp.idx[q];
      if (bad) s_bad = q;
    }
  }
  double mx = 0.0;
  for (int64_t e = t; e < (int64_t)n * r; e += blockDim.x) mx = fmax(mx, fabs(W[e]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (t == 0) s_mx = 0.0;
  __syncthreads();
  if ((t & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_mx),
                               (unsigned long long)__double_as_longlong(mx));
  __syncthreads();
  const double floor_ = 1e-14 * fmax(1.0, s_mx);  // lowrank.py:185
  int fail = s_bad;
  if (fail < 0) {
    for (int e = t; e < r * r; e += blockDim.x) a[e] = W[(int64_t)fp.idx[e / r] * r + e % r];
    __syncthreads();
    for (int j = 0; j < r; ++j) {  // Doolittle, rows in pick order
      const double pv = a[j * r + j];
      if (!(fabs(pv) > floor_)) { fail = j; break; }
      for (int e = t; e < (r - j - 1) * (r - j); e += blockDim.x) {
        const int q = j + 1 + e / (r - j), k = j + e % (r - j);
        const double l = a[q * r + j] / pv;
        if (k == j) continue;
        a[q * r + k] -= l * a[j * r + k];
      }
      __syncthreads();
      for (int q = j + 1 + t; q < r; q += blockDim.x) a[q * r + j] /= pv;
      __syncthreads();
    }
  }
  if (fail >= 0) {
    if (t == 0) {
      *err_col = fail;
      for (int q = 0; q < r; ++q) idx_out[q] = fp.idx[q] >= 0 && fp.idx[q] < n ? fp.idx[q] : 0;
    }
    return;
  }
  for (int e = t; e < r * r; e += blockDim.x) {
    const int q = e / r, k = e % r;
    Lhat[e] = k < q ? a[e] : (k == q ? 1.0 : 0.0);
    U[e] = k >= q ? a[e] : 0.0;
  }
  for (int q = t; q < r; q += blockDim.x) {
    idx_out[q] = fp.idx[q];
    if (gap) gap[q] = 1.0;  // forced: no argmax, no tie
  }
  if (t == 0) *err_col = -1;
}

// ---- workspace arena ---------------------------------------------------------
struct Arena {
  char* base;
  size_t off = 0;
  explicit Arena(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

// upload block: group table, quadrant codes, completion exponents, extent
struct Upload {
  dlrsn_group groups[DLRSN_MAX_RANK];
  int quads[DLRSN_MAX_RANK];
  int sexp[2 * (DLRSN_MAX_RANK + 8)];
  int aexp[3 * (DLRSN_MAX_RANK + 8)];
  double extent[4];
};

struct StepBufs {
  int *err_idx, *flags, *rowstat, *defw, *statw, *defx, *statx, *cholflag;
  double *Wk, *Lhat, *U, *closure, *chk_in, *chk_out, *deimgap;
  double *sig4, *rhs_sk, *psi_sk, *phi_part, *scat, *psi_time, *phi0, *phi1, *norms, *red_ws;
  double *om_sel, *K, *Sb, *psi, *G, *R1, *R1inv, *ratio, *ratio2, *X1, *R2, *R2inv, *Rtot;
  double *part, *proj, *Binv, *L, *lbar, *T, *qall, *gamma, *lfull, *Rang, *cgsws;
  double *wpart, *wg;
  double* rcs;  // row-combine scratch: cbar | zeta | msl
  CgTable* cgtab;  // grouped sweep: direction groups
  int* cg_quad;
  double* cg_w;
  int *idx, *quads, *mine;
  int64_t* place;
  double* cw_local;
  double* phiq;
  dlrsn_group* groups;
  SiCtl* ctl;
  unsigned* rbdev;
  double* ratiow;
  int* cholw;
  double *Rw1, *Rw1inv, *Rw2, *Rw2inv, *ratiow2, *lq1;  // angular CholQR2, r > 32
  double* hin;  // X_new^T of the unit inflow load per wall (4 x r)
  // DSA inside the step: phi_half, the PCG workspace, {kx, ky}, the info words
  double *dsa_half, *dsa_ws, *dsa_k;
  int* dsa_info;
  Upload* up;
};

static size_t carve(Arena& ar, StepBufs& b, int nx, int ny, int r, int no, int world) {
  const int64_t nc = (int64_t)nx * ny, N = 4 * nc;
  const int64_t V = sk_vec_len(nx, ny), S4 = sk_scalar_len(nx, ny);
  const int64_t nb = (nc + 255) / 256;
  const int64_t part = std::max(dlrsn_partials_len((int)nc, r, r, 0), dlrsn_partials_len((int)nc, r, r, 1));
  const int64_t rl = (r + world - 1) / world + 1;  // local directions (upper bound)
  b.err_idx = ar.take<int>(r + 1);
  b.flags = ar.take<int>(8);
  b.rowstat = ar.take<int>(r + 1);
  b.defw = ar.take<int>(r);
  b.statw = ar.take<int>(1);
  b.defx = ar.take<int>(r);
  b.statx = ar.take<int>(1);
  b.cholflag = ar.take<int>(2);
  b.Wk = ar.take<double>((size_t)no * r);
  b.deimgap = ar.take<double>(r);
  b.Lhat = ar.take<double>((size_t)r * r);
  b.U = ar.take<double>((size_t)r * r);
  b.closure = ar.take<double>(r);
  b.chk_in = ar.take<double>(2);
  b.chk_out = ar.take<double>(2);
  b.sig4 = ar.take<double>(4 * S4);
  b.rhs_sk = ar.take<double>(rl * V);
  b.psi_sk = ar.take<double>(rl * V);
  b.phi_part = ar.take<double>(rl * V);
  b.scat = ar.take<double>(4 * V);
  b.psi_time = ar.take<double>(N * r);
  b.phi0 = ar.take<double>(N);
  b.phi1 = ar.take<double>(N);
  b.norms = ar.take<double>(2);
  b.red_ws = ar.take<double>(32 + 2 * nb + 8);
  b.om_sel = ar.take<double>(3 * r);
  b.K = ar.take<double>((size_t)r * r);
  b.Sb = ar.take<double>(r);
  b.psi = ar.take<double>(N * r);
  b.G = ar.take<double>((size_t)r * r);
  b.R1 = ar.take<double>((size_t)r * r);
  b.R1inv = ar.take<double>((size_t)r * r);
  b.ratio = ar.take<double>(2 * r);
  b.ratio2 = ar.take<double>(2 * r);
  b.X1 = ar.take<double>(N * r);
  b.R2 = ar.take<double>((size_t)r * r);
  b.R2inv = ar.take<double>((size_t)r * r);
  b.Rtot = ar.take<double>((size_t)r * r);
  b.part = ar.take<double>(part);
  b.proj = ar.take<double>(7 * (size_t)r * r + r);
  b.Binv = ar.take<double>((size_t)r * r * r);
  b.L = ar.take<double>((size_t)r * r);
  b.lbar = ar.take<double>(r);
  b.T = ar.take<double>((size_t)r * r);
  b.qall = ar.take<double>((size_t)r * r);
  b.gamma = ar.take<double>((size_t)r * r);
  b.lfull = ar.take<double>((size_t)no * r);
  b.Rang = ar.take<double>((size_t)r * r);
  b.cgsws = ar.take<double>(std::max(dlrsn_cgs2_workspace_len((int)N), dlrsn_cgs2_workspace_len(no)));
  b.wpart = ar.take<double>((size_t)((no + wgram_rows(r) - 1) / wgram_rows(r)) * (r * r + r));
  b.wg = ar.take<double>((size_t)r * r + r);
  b.idx = ar.take<int>(r);
  b.quads = ar.take<int>(r);
  b.mine = ar.take<int>(r);
  b.place = ar.take<int64_t>(r);
  b.cw_local = ar.take<double>(r);
  b.phiq = ar.take<double>(4 * N);
  b.groups = ar.take<dlrsn_group>(r);
  b.ctl = ar.take<SiCtl>(1);
  b.rbdev = ar.take<unsigned>(8192);
  b.ratiow = ar.take<double>(2 * r);
  b.cholw = ar.take<int>(2);
  b.Rw1 = ar.take<double>((size_t)r * r);
  b.Rw1inv = ar.take<double>((size_t)r * r);
  b.Rw2 = ar.take<double>((size_t)r * r);
  b.Rw2inv = ar.take<double>((size_t)r * r);
  b.ratiow2 = ar.take<double>(2 * r);
  b.lq1 = ar.take<double>((size_t)no * r);
  b.hin = ar.take<double>(4 * (size_t)r);
  b.rcs = ar.take<double>((size_t)r * r + 2 * r);
  b.cgtab = ar.take<CgTable>(1);
  b.cg_quad = ar.take<int>(r);
  b.cg_w = ar.take<double>(r);
  b.dsa_half = ar.take<double>(N);
  b.dsa_ws = ar.take<double>(dlrsn_dsa_workspace_len(nx, ny));
  b.dsa_k = ar.take<double>(2);
  b.dsa_info = ar.take<int>(4);
  b.up = ar.take<Upload>(1);
  return ar.off;
}

// CholQR2 guard threshold (min R_kk / |a_k| over the columns) and a debug
// print of the observed minimum (DLRSN_GUARD_RATIO / DLRSN_GUARD_DEBUG)
static double guard_ratio() {
  static const double v = [] {
    const char* e = getenv("DLRSN_GUARD_RATIO");
    return e ? atof(e) : 1e-6;
  }();
  return v;
}
static bool guard_debug() {
  static const bool v = getenv("DLRSN_GUARD_DEBUG") != nullptr;
  return v;
}

#define DLRSN_RET(expr)              \
  do {                               \
    int rc_ = (expr);                \
    if (rc_ != DLRSN_OK) return rc_; \
  } while (0)

// ---- the status block: every word the host needs after a segment, packed
// on the device into a fixed layout and read back with one copy -----------
struct StepStatus {
  int err_idx[DLRSN_MAX_RANK + 1];  // [0] DEIM failure column (-1 ok), then the picks
  int flags[8];                     // [0] sigma check, [1] any scattering
  double chk_in[2], chk_out[2];     // orthonormality residuals (in / out)
  SiCtl ctl;
  double closure[DLRSN_MAX_RANK];
  int rowstat[DLRSN_MAX_RANK + 1];
  int defw[DLRSN_MAX_RANK], defx[DLRSN_MAX_RANK];
  int statw, statx;
  double ratio[2 * DLRSN_MAX_RANK], ratiow[2 * DLRSN_MAX_RANK];
  int cholflag[2], cholw[2];
  int sweep_status;                 // sweep workspace word 1 (2: handoff timeout)
  double deim_gap[DLRSN_MAX_RANK];
  int dsa[4];  // last CG iterations, failure, total CG iterations, solves
};

// pinned, device-mapped host copy of the status block (one per host thread;
// its address is baked into captured graphs, so it is never reallocated).
// The pack kernel stores into it directly: no copy-engine transfer, so the
// step's readback never queues behind bulk copies of other streams.
static thread_local StepStatus* g_status_dev = nullptr;
static int status_block(StepStatus** out) {
  static thread_local StepStatus* hs = nullptr;
  if (!hs) {
    void* ptr = nullptr;
    DLRSN_TRY_CUDA(cudaHostAlloc(&ptr, sizeof(StepStatus), cudaHostAllocMapped));
    void* dptr = nullptr;
    DLRSN_TRY_CUDA(cudaHostGetDevicePointer(&dptr, ptr, 0));
    hs = static_cast<StepStatus*>(ptr);
    g_status_dev = static_cast<StepStatus*>(dptr);
  }
  *out = hs;
  return DLRSN_OK;
}

// pack kernel + one device-to-host copy of the status block
static int enqueue_status(cudaStream_t st, const StepBufs& b, int r, StepStatus* hs,
                          const void* sweep_ws) {
  PackList l;
  l.n = 0;
  StepStatus* dev = reinterpret_cast<StepStatus*>(b.rbdev);
  auto add = [&](const void* src, size_t bytes, const void* dst_field) {
    l.src[l.n] = static_cast<const unsigned*>(src);
    l.words[l.n] = (int)((bytes + 3) / 4);
    l.off[l.n] = (int)((reinterpret_cast<const char*>(dst_field) - reinterpret_cast<const char*>(dev)) / 4);
    ++l.n;
  };
  add(b.err_idx, (r + 1) * sizeof(int), dev->err_idx);
  add(b.flags, 8 * sizeof(int), dev->flags);
  add(b.chk_in, 2 * sizeof(double), dev->chk_in);
  add(b.chk_out, 2 * sizeof(double), dev->chk_out);
  add(b.ctl, sizeof(SiCtl), &dev->ctl);
  add(b.closure, r * sizeof(double), dev->closure);
  add(b.rowstat, (r + 1) * sizeof(int), dev->rowstat);
  add(b.defw, r * sizeof(int), dev->defw);
  add(b.defx, r * sizeof(int), dev->defx);
  add(b.statw, sizeof(int), &dev->statw);
  add(b.statx, sizeof(int), &dev->statx);
  add(b.ratio, 2 * r * sizeof(double), dev->ratio);
  add(b.ratiow, 2 * r * sizeof(double), dev->ratiow);
  add(b.cholflag, 2 * sizeof(int), dev->cholflag);
  add(b.cholw, 2 * sizeof(int), dev->cholw);
  add(reinterpret_cast<const int*>(sweep_ws) + 1, sizeof(int), &dev->sweep_status);
  add(b.deimgap, r * sizeof(double), dev->deim_gap);
  add(b.dsa_info, 4 * sizeof(int), dev->dsa);
  (void)hs;
  pack_kernel<<<1, 256, 0, st>>>(l, reinterpret_cast<unsigned*>(g_status_dev));
  DLRSN_CHECK_LAUNCH("pack_kernel");
  return DLRSN_OK;
}

// ---- a second stream for the step's parallel branches (fork / join by
// events; captured into a graph they become parallel branches) -------------
struct Fork {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
// Off by default: measured on C2 the forked graph was slower (1.49 vs 1.35 ms
// per step; the side branch's grid-wide kernels stretch the critical path
// more than the overlap with the single-CTA kernels gains).  DLRSN_STEP_FORK=1
// enables it.
static bool fork_enabled() {
  static const char* e = getenv("DLRSN_STEP_FORK");
  return e && e[0] == '1';
}
static int fork_streams(Fork** out) {
  static thread_local Fork f;
  if (!fork_enabled()) {  // serial variant: the "side" work stays on the caller's stream
    static thread_local Fork none;
    *out = &none;
    return DLRSN_OK;
  }
  if (!f.side) {
    DLRSN_TRY_CUDA(cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking));
    DLRSN_TRY_CUDA(cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming));
    DLRSN_TRY_CUDA(cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming));
  }
  *out = &f;
  return DLRSN_OK;
}
// side stream starts after everything enqueued on `st` so far
static int fork_to(Fork* f, cudaStream_t st) {
  if (!f->fork) {
    f->side = st;
    return DLRSN_OK;
  }
  DLRSN_TRY_CUDA(cudaEventRecord(f->fork, st));
  DLRSN_TRY_CUDA(cudaStreamWaitEvent(f->side, f->fork, 0));
  return DLRSN_OK;
}
// `st` continues after everything enqueued on the side stream
static int join_from(const Fork* f, cudaStream_t st) {
  if (!f->join) return DLRSN_OK;
  DLRSN_TRY_CUDA(cudaEventRecord(f->join, f->side));
  DLRSN_TRY_CUDA(cudaStreamWaitEvent(st, f->join, 0));
  return DLRSN_OK;
}

// ---- X_new device-to-host copy overlapped with the rest of the step --------
struct OutCopy {
  cudaStream_t cs = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
};
static int out_copy_stream(OutCopy** out) {
  static thread_local OutCopy oc;
  if (!oc.cs) {
    DLRSN_TRY_CUDA(cudaStreamCreateWithFlags(&oc.cs, cudaStreamNonBlocking));
    DLRSN_TRY_CUDA(cudaEventCreateWithFlags(&oc.ready, cudaEventDisableTiming));
    DLRSN_TRY_CUDA(cudaEventCreateWithFlags(&oc.done, cudaEventDisableTiming));
  }
  *out = &oc;
  return DLRSN_OK;
}

// ---- CUDA-graph replay of the step's first segment --------------------------
// The segment's ~50 launches depend only on the buffers, the parameters and
// the iteration batch; a driver loop hands the same buffers back every other
// step (the caching allocator), so the segment is captured once per buffer
// set and replayed with one graph launch (no per-kernel host cost, no launch
// gaps).  Everything baked into the graph is part of the key.
struct GraphKey {
  unsigned char bytes[sizeof(dlrsn_cellops) + sizeof(dlrsn_step_params) + sizeof(dlrsn_advance) +
                      24 * sizeof(void*)];
  void set(const dlrsn_cellops* ops, const dlrsn_step_params* p, const void* X, const void* S,
           const void* W, const void* beta, const void* st, const void* ss, const void* q,
           const void* Xn, const void* Sn, const void* Wn, const void* bn, const void* phi,
           const void* siphi, const void* ws, const void* sws, int64_t sws_bytes, int batch,
           int exact, int exact_w) {
    memset(bytes, 0, sizeof(bytes));
    size_t o = 0;
    memcpy(bytes + o, ops, sizeof(*ops));
    o += sizeof(*ops);
    dlrsn_step_params pp = *p;
    pp.omegas_host = nullptr;  // read on the host only
    pp.advance = nullptr;      // compared by content below
    memcpy(bytes + o, &pp, sizeof(pp));
    o += sizeof(pp);
    if (p->advance) memcpy(bytes + o, p->advance, sizeof(dlrsn_advance));
    o += sizeof(dlrsn_advance);
    const void* ptrs[] = {X, S, W, beta, st, ss, q, Xn, Sn, Wn, bn, phi, siphi, ws, sws};
    memcpy(bytes + o, ptrs, sizeof(ptrs));
    o += sizeof(ptrs);
    const int64_t extra[4] = {sws_bytes, batch, exact, exact_w};
    memcpy(bytes + o, extra, sizeof(extra));
  }
  bool operator==(const GraphKey& k) const { return memcmp(bytes, k.bytes, sizeof(bytes)) == 0; }
};

struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec;
  int device;
  uint64_t used;
  int64_t kernels;  // launches captured (added to the launch counter per replay)
};

static bool graphs_enabled() {
  static const char* e = getenv("DLRSN_STEP_GRAPH");
  return !(e && e[0] == '0');
}

template <class F>
static int graph_run(const GraphKey& key, F&& enqueue, cudaStream_t st, bool chained) {
  static thread_local std::vector<GraphEntry> cache;
  static thread_local uint64_t tick = 0;
  static thread_local cudaStream_t cs = nullptr;
  int dev = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  ++tick;
  GraphEntry* seen = nullptr;
  for (auto& e : cache)
    if (e.device == dev && e.key == key) {
      e.used = tick;
      if (e.exec) {
        DLRSN_TRY_CUDA(cudaGraphLaunch(e.exec, st));
        launch_counter().fetch_add(e.kernels, std::memory_order_relaxed);
        return DLRSN_OK;
      }
      seen = &e;
      break;
    }
  auto evict = [&]() {
    if (cache.size() < 64) return;
    size_t lru = 0;
    for (size_t i = 1; i < cache.size(); ++i)
      if (cache[i].used < cache[lru].used) lru = i;
    if (cache[lru].exec) cudaGraphExecDestroy(cache[lru].exec);
    cache.erase(cache.begin() + lru);
  };
  if (!seen && !chained) {
    // first sighting: launch directly and remember the key; buffers that
    // come back (a driver loop) are captured on their second use, one-off
    // buffers (fresh allocations every step) never pay for a capture
    evict();
    GraphEntry e;
    e.key = key;
    e.exec = nullptr;
    e.device = dev;
    e.used = tick;
    e.kernels = 0;
    cache.push_back(e);
    return enqueue(st);
  }
  if (!seen) {  // a chained step (its input is a previous step's output): capture now
    evict();
    GraphEntry e;
    e.key = key;
    e.exec = nullptr;
    e.device = dev;
    e.used = tick;
    e.kernels = 0;
    cache.push_back(e);
    seen = &cache.back();
  }
  if (!cs) DLRSN_TRY_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  {
    static const bool dbg = getenv("DLRSN_GRAPH_DEBUG") != nullptr;
    if (dbg) {
      uint64_t h = 1469598103934665603ull;
      for (size_t i = 0; i < sizeof(key.bytes); ++i) h = (h ^ key.bytes[i]) * 1099511628211ull;
      fprintf(stderr, "dlrsn graph: capture #%zu key %016llx (chained %d)\n", cache.size(),
              (unsigned long long)h, (int)chained);
    }
  }
  // capture on a private stream (the caller's may be the legacy default stream)
  DLRSN_TRY_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const int64_t k0 = launch_counter().load();
  const int rc = enqueue(cs);
  const int64_t kernels = launch_counter().load() - k0;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  if (rc != DLRSN_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  DLRSN_TRY_CUDA(ec);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  DLRSN_TRY_CUDA(ei);
  seen->exec = exec;
  seen->kernels = kernels;
  DLRSN_TRY_CUDA(cudaGraphLaunch(exec, st));
  return DLRSN_OK;
}

// ---- device-side planning (no host round trip for the DEIM picks) ---------
__device__ __host__ inline int quad_code(const double* om) {
  return (om[0] >= 0.0 ? 0 : 1) | (om[1] >= 0.0 ? 0 : 2);
}

// From the DEIM picks: a valid index set (identity when DEIM failed, so the
// speculative work stays in bounds; the error is reported at the readback),
// the direction partition of sharding.partition_directions (quadrant-major
// round robin), this rank's single-direction sweep groups in quadrant order
// (transport.plan_groups), and the gather / placement tables of the sharded
// step.  One thread: r <= 128.
__global__ void plan_kernel(int r, int no, int world, int rank, const int* __restrict__ err,
                            const int* __restrict__ idx_raw, const double* __restrict__ omegas,
                            const double* __restrict__ closure, int* __restrict__ idx,
                            dlrsn_group* __restrict__ groups, int* __restrict__ quads,
                            int* __restrict__ mine, int64_t* __restrict__ place, int64_t n_dofs,
                            int width, double* __restrict__ cw_local) {
  // thread d = selected direction d (r <= 128); every rank / position is a
  // count over the r directions (O(r) per thread)
  __shared__ int sq[DLRSN_MAX_RANK], sown[DLRSN_MAX_RANK];
  const int d = threadIdx.x;
  const bool bad = err[0] >= 0;
  int v = d;
  if (d < r) {
    v = bad ? d : idx_raw[d];
    if (v < 0 || v >= no) v = d;
    idx[d] = v;
    sq[d] = quad_code(omegas + 3 * (int64_t)v);
  }
  __syncthreads();
  int owner = 0;
  if (d < r) {
    int before = 0;  // position in quadrant-major order (partition_directions)
    for (int e = 0; e < r; ++e) before += (sq[e] < sq[d]) || (sq[e] == sq[d] && e < d);
    owner = before % world;
    sown[d] = owner;
  }
  __syncthreads();
  if (d < r) {
    int pos = 0;
    for (int e = 0; e < d; ++e) pos += sown[e] == owner;
    place[d] = (int64_t)owner * n_dofs * width + pos;
    if (owner == rank) {
      mine[pos] = d;
      quads[pos] = sq[d];
      cw_local[pos] = closure[d];
      int gi = 0;  // this rank's groups in quadrant order (transport.plan_groups)
      for (int e = 0; e < r; ++e)
        gi += sown[e] == rank && ((sq[e] < sq[d]) || (sq[e] == sq[d] && e < d));
      const double* om = omegas + 3 * (int64_t)v;
      dlrsn_group g;
      memset(&g, 0, sizeof(g));
      g.quad = sq[d];
      g.ndir = 1;
      g.slot[0] = pos;
      g.ox[0] = fabs(om[0]);
      g.oy[0] = fabs(om[1]);
      g.cw[0] = closure[d];
      groups[gi] = g;
    }
  }
}

// dst (n x nl) = src[:, mine] (src n x r): this rank's psi_time columns
__global__ void gather_cols_kernel(int64_t n, int r, int nl, const int* __restrict__ mine,
                                   const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t total = n * nl;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nl;
    const int k = (int)(e - i * nl);
    dst[e] = src[i * r + mine[k]];
  }
}

// psi (n x r)[:, d] = recv[place[d] + i * width] (allgathered swept columns)
__global__ void place_cols_kernel(int64_t n, int r, int width, const int64_t* __restrict__ place,
                                  const double* __restrict__ recv, double* __restrict__ psi) {
  const int64_t total = n * r;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r;
    const int d = (int)(e - i * r);
    psi[e] = recv[place[d] + i * width];
  }
}

// si_phi = the flux of the converged iteration (ping-pong buffer iters % 2)
__global__ void si_select_kernel(int64_t n, const SiCtl* __restrict__ ctl,
                                 const double* __restrict__ p0, const double* __restrict__ p1,
                                 double* __restrict__ out) {
  const double* src = (ctl->iters & 1) ? p1 : p0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = src[e];
}

// DSA "collocation" penalty weights of the step's own selection
// (transport_sn.py:186-188): k = 1/2 closure.|omega_{x,y}| / (4 pi)
__global__ void dsa_penalty_kernel(int r, const double* __restrict__ closure,
                                   const double* __restrict__ om_sel, double* __restrict__ k) {
  if (threadIdx.x < 2) {
    double acc = 0.0;
    for (int d = 0; d < r; ++d) acc += closure[d] * fabs(om_sel[3 * d + threadIdx.x]);
    k[threadIdx.x] = 0.5 * acc / (4.0 * 3.14159265358979323846);
  }
}

static int grid_n(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

// X_new of the previous successful step: a step whose X is it is part of a
// driver loop, whose buffers come back, so its graph is captured at once
static thread_local const void* g_last_xnew = nullptr;

}  // namespace dlrsn

using namespace dlrsn;

extern "C" {

int dlrsn_deim_forced(int n, int r, const double* W, const int64_t* indices, int* idx,
                      double* Lhat, double* U, int* err_col, double* gap, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(r >= 1 && r <= n && r <= DLRSN_MAX_RANK, "rank %d outside [1, min(%d, %d)]", r, n,
                DLRSN_MAX_RANK);
  DLRSN_REQUIRE((size_t)r * r * sizeof(double) <= 48 * 1024, "forced selection needs r <= 78");
  DLRSN_REQUIRE(indices, "null angle indices");
  ForcedPicks fp;
  for (int d = 0; d < r; ++d) fp.idx[d] = (indices[d] >= 0 && indices[d] < n) ? (int)indices[d] : -1;
  deim_forced_kernel<<<1, 256, (size_t)r * r * sizeof(double), as_stream(stream)>>>(
      n, r, W, fp, idx, Lhat, U, err_col, gap);
  DLRSN_CHECK_LAUNCH("deim_forced_kernel");
  return DLRSN_OK;
}

int64_t dlrsn_step_workspace_bytes(int nx, int ny, int r, int n_omega, int world_size) {
  StepBufs b;
  Arena ar(nullptr);
  return (int64_t)carve(ar, b, nx, ny, r, n_omega, world_size < 1 ? 1 : world_size) + 256;
}

int dlrsn_step_collocation(const dlrsn_cellops* ops, const dlrsn_step_params* p, const double* X,
                           const double* S, const double* W, const double* beta,
                           const double* sigma_t, const double* sigma_s, const double* q,
                           double* X_new, double* S_new, double* W_new, double* beta_new,
                           double* phi_out, double* si_phi, void* workspace,
                           int64_t workspace_bytes, void* sweep_ws, int64_t sweep_ws_bytes,
                           const dlrsn_comm* comm, dlrsn_step_info* info, dlrsn_stream_t stream) {
  const cudaStream_t st0 = as_stream(stream);
  const int r = p->rank, no = p->n_omega, nx = ops->nx, ny = ops->ny;
  DLRSN_REQUIRE(r >= 1 && r <= DLRSN_MAX_RANK, "rank %d outside [1, %d]", r, DLRSN_MAX_RANK);
  DLRSN_REQUIRE(r <= no, "rank %d exceeds the %d available nodes", r, no);
  DLRSN_REQUIRE(p->sweep_dw <= 1, "the one-call step sweeps single-direction groups (sweep_dw 1)");
  DLRSN_REQUIRE(!p->use_dsa || p->dsa_penalty == 0 || p->dsa_penalty == 1,
                "unknown dsa penalty variant %d", p->dsa_penalty);
  const int world = comm ? comm->world_size : 1;
  const int rank_id = comm ? comm->rank : 0;
  DLRSN_REQUIRE(world >= 1 && world <= 8 && rank_id >= 0 && rank_id < world,
                "rank %d of %d outside the supported 1..8 ranks", rank_id, world);
  DLRSN_REQUIRE(world == 1 || (comm->allreduce_sum && comm->allgather && comm->reduce_buf &&
                               comm->gather_send && comm->gather_recv &&
                               comm->gather_width >= (r + world - 1) / world),
                "incomplete dlrsn_comm");
  StepBufs b;
  Arena ar(workspace);
  const size_t need = carve(ar, b, nx, ny, r, no, world);
  DLRSN_REQUIRE((int64_t)need <= workspace_bytes, "step workspace too small (%lld < %lld)",
                (long long)workspace_bytes, (long long)need);
  const int nc = nx * ny;
  const int64_t N = 4 * (int64_t)nc;
  memset(info, 0, sizeof(*info));
  info->error_index = -1;
  const int nl = (r - rank_id + world - 1) / world;  // this rank's directions
  const int G = nl;                                  // single-direction groups
  // grouped sweep with the fused closure: one GPU, enough direction-strips
  // for the throughput kernel (the warp-specialised kernel below that)
  int sms_count = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms_count, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool grouped = world == 1 && nl > 0 && !p->use_dsa && sweep_group_width() > 0 &&
                       sk_strips(ny) * G > 4 * sms_count;
  // full-rank fast path of the angular update: one-CTA weighted CholQR2
  const bool ang_fast = r <= 32 && dlrsn_cholqr2_small_smem(no, r) <= 200 * 1024;
  StepStatus* hs = nullptr;
  DLRSN_RET(status_block(&hs));
  ForcedPicks forced;
  memset(&forced, 0, sizeof(forced));
  if (p->angle_override) {
    DLRSN_REQUIRE(p->angle_indices_in, "angle_override without angle_indices_in");
    DLRSN_REQUIRE((size_t)r * r * sizeof(double) <= 48 * 1024, "forced selection needs r <= 78");
    for (int d = 0; d < r; ++d) {
      const int64_t v = p->angle_indices_in[d];
      forced.idx[d] = (v >= 0 && v < no) ? (int)v : -1;
    }
  }
  double* P[2] = {b.phi0, b.phi1};
  Inflow4 infl;
  bool has_inflow = false;
  for (int w = 0; w < 4; ++w) {
    infl.v[w] = p->inflow[w];
    has_inflow |= p->inflow[w] != 0.0;
  }

  // ---- the step as segments of device work, each closed by the packed
  // status readback (so a segment is one host synchronisation) ------------
  // head: constants, DEIM, closure weights, input checks, plan, rhs
  auto enqueue_head = [&](cudaStream_t st) -> int {
    void* s = st;
    InitArgs ia;
    ia.flags = b.flags;
    ia.statw = b.statw;
    ia.statx = b.statx;
    ia.red_ws = b.red_ws;
    ia.ctl = b.ctl;
    ia.sexp = b.up->sexp;
    ia.aexp = b.up->aexp;
    ia.extent = b.up->extent;
    ia.count = r + 8;
    ia.x0 = ops->x0;
    ia.y0 = ops->y0;
    ia.lx = ops->nx * ops->dx;
    ia.ly = ops->ny * ops->dy;
    init_kernel<<<1, 96, 0, st>>>(ia);
    DLRSN_CHECK_LAUNCH("init_kernel");
    // Two branches: the DEIM chain (one CTA for most of it) on `st`, the
    // checks / scalar flux / scattering source / sigma layout on the side
    // stream, so the single-CTA kernels overlap GPU-wide work.
    Fork* fk = nullptr;
    DLRSN_RET(fork_streams(&fk));
    DLRSN_RET(fork_to(fk, st));
    {
      cudaStream_t sd = fk->side;
      void* ss2 = sd;
      sigma_check_kernel<<<std::min(1024, (nc + 255) / 256), 256, 0, sd>>>(nc, sigma_t, sigma_s,
                                                                           b.flags);
      DLRSN_CHECK_LAUNCH("sigma_check_kernel");
      if (p->check_state) {
        // the input Gram is skipped when the producing step already checked X
        if (!p->x_check_in) DLRSN_RET(dlrsn_mgram(ops, r, r, X, r, X, r, nullptr, b.G, b.part, ss2));
        DLRSN_RET(wgram(no, r, W, p->weights_dev, b.wpart, b.wg, sd));
        ortho_residual_kernel<<<1, 256, 0, sd>>>(r, p->x_check_in ? nullptr : b.G, b.wg,
                                                 b.chk_in, p->x_check_in);
        DLRSN_CHECK_LAUNCH("ortho_residual_kernel");
      }
      DLRSN_RET(dlrsn_cells_to_sk4(ops, sigma_t, b.sig4, ss2));
    }
    // 1. DEIM, closure weights (errors reported at the readback)
    if (p->angle_override) {
      deim_forced_kernel<<<1, 256, (size_t)r * r * sizeof(double), st>>>(
          no, r, W, forced, b.err_idx + 1, b.Lhat, b.U, b.err_idx, b.deimgap);
      DLRSN_CHECK_LAUNCH("deim_forced_kernel");
    } else {
      DLRSN_RET(dlrsn_deim(no, r, b.Wk, W, b.err_idx + 1, b.Lhat, b.U, b.err_idx, b.deimgap, 0, s));
    }
    DLRSN_RET(dlrsn_what_solve(r, 1, b.Lhat, b.U, beta, b.closure, 1, s));
    const int width = world > 1 ? comm->gather_width : 1;
    plan_kernel<<<1, DLRSN_MAX_RANK, 0, st>>>(r, no, world, rank_id, b.err_idx, b.err_idx + 1,
                                              p->omegas_dev, b.closure, b.idx, b.groups, b.quads,
                                              b.mine, b.place, N, width, b.cw_local);
    DLRSN_CHECK_LAUNCH("plan_kernel");
    if (grouped)
      DLRSN_RET(cgroup_plan_launch(G, b.groups, sweep_group_width(), r, b.cgtab, b.cg_quad, b.cg_w,
                                   st));
    // 2. evaluate_rows (dlr_sn.py:110-121) and the sweep rhs
    ks_kernel<<<r, 256, 0, st>>>(r, S, W, b.idx, beta, b.K, nullptr, p->omegas_dev, b.om_sel);
    DLRSN_CHECK_LAUNCH("ks_kernel");
    if (p->use_dsa) {
      DLRSN_TRY_CUDA(zero_async(b.dsa_info, 4 * sizeof(int), st));
      if (p->dsa_penalty == 1) {
        dsa_penalty_kernel<<<1, 32, 0, st>>>(r, b.closure, b.om_sel, b.dsa_k);
        DLRSN_CHECK_LAUNCH("dsa_penalty_kernel");
      }
    }
    // scalar_flux (lowrank.py:60-62) -> the first scattering source; phi0 = X
    // (S beta) comes out of the same pass over X as psi_time = X K
    ks_kernel<<<(r + 7) / 8, 256, 0, st>>>(r, S, W, nullptr, beta, nullptr, b.Sb, p->omegas_dev, nullptr);
    DLRSN_CHECK_LAUNCH("ks_kernel");
    DLRSN_RET(rowmix_vec(N, r, r, X, r, b.K, r, 0.0, b.psi_time, r, b.Sb, b.phi0, s));
    DLRSN_RET(dlrsn_scatter_source(ops, b.phi0, sigma_s, b.scat, b.flags + 1, s));
    const double* pt_local = b.psi_time;
    int ld_pt = r;
    if (world > 1 && nl > 0) {
      gather_cols_kernel<<<grid_n(N * nl), 256, 0, st>>>(N, r, nl, b.mine, b.psi_time, b.psi);
      DLRSN_CHECK_LAUNCH("gather_cols_kernel");
      pt_local = b.psi;
      ld_pt = nl;
    }
    if (nl > 0) {
      DLRSN_RET(dlrsn_rhs_build(ops, nl, b.quads, q, p->inv_cdt, pt_local, ld_pt, nullptr, 1,
                                b.rhs_sk, s));
      if (has_inflow)
        DLRSN_RET(dlrsn_inflow_add(ops, nl, b.quads, b.om_sel, b.mine, p->inflow, b.rhs_sk, s));
    }
    DLRSN_RET(join_from(fk, st));
    return DLRSN_OK;
  };
  // 3. source iterations it_from..it_to (transport_sn.py:408-447): the
  // convergence test runs on the device (si_decide) and iterations past it
  // return at once; then the converged flux / swept columns are selected
  const double dsa_tol = p->dsa_tol > 0.0 ? p->dsa_tol : 1e-10;  // pcg defaults, :325-328
  const int dsa_cap = p->dsa_max_iters > 0
                          ? p->dsa_max_iters
                          : (int)std::min<int64_t>(10 * N, (int64_t)INT32_MAX);
  auto dsa_launch = [&](double* phi_half, const double* phi_old, cudaStream_t st) -> int {
    return dsa_correct_launch(ops, sigma_t, sigma_s, 0.25, 0.25,
                              p->dsa_penalty == 1 ? b.dsa_k : nullptr, phi_half, phi_old, phi_half,
                              dsa_tol, dsa_cap, b.dsa_ws, b.dsa_info, p->dsa_history,
                              p->dsa_hist_cap, &b.ctl->done, 1, st);
  };
  auto enqueue_si = [&](cudaStream_t st, int it_from, int it_to) -> int {
    void* s = st;
    for (int it = it_from; it <= it_to; ++it) {
      const double* phi = P[(it - 1) & 1];
      double* phin = P[it & 1];
      if (grouped) {
        // psi and the per-group closure partials in one pass, then the
        // partial slabs summed per quadrant (fixed order) like swept columns
        DLRSN_RET(sweep_grouped_launch(ops, G, b.groups, b.cgtab, b.sig4, b.scat, b.rhs_sk,
                                       b.psi_sk, b.phi_part, sweep_ws, sweep_ws_bytes,
                                       &b.ctl->done, st));
        DLRSN_RET(phi_closure_launch(ops, r, b.cg_quad, b.cg_w, b.phi_part, b.phiq, phi, sigma_s,
                                     phin, b.scat, b.norms, b.red_ws, b.ctl, it, p->si_tol,
                                     b.flags + 1, nullptr, st));
        continue;
      }
      if (nl > 0)
        DLRSN_RET(sweep_launch(ops, G, b.groups, 1, b.sig4, b.scat, b.rhs_sk, b.psi_sk, nullptr,
                               sweep_ws, sweep_ws_bytes, 0, &b.ctl->done, st));
      if (world == 1 && p->use_dsa) {
        // phi_half = psi closure, phi_half += delta (K6, one cooperative
        // launch, skipped on the device once converged), then the norms and
        // the next scattering source from the corrected flux (:439-446)
        DLRSN_RET(phi_closure_launch(ops, nl, b.quads, b.cw_local, b.psi_sk, b.phiq, phi, sigma_s,
                                     nullptr, nullptr, b.norms, b.red_ws, b.ctl, -1, p->si_tol,
                                     nullptr, b.dsa_half, st));
        DLRSN_RET(dsa_launch(b.dsa_half, phi, st));
        DLRSN_RET(phi_finish_launch(ops, b.dsa_half, phin, phi, sigma_s, b.scat, b.norms, b.red_ws,
                                    b.ctl, it, p->si_tol, b.flags + 1, st));
      } else if (world == 1) {
        DLRSN_RET(phi_closure_launch(ops, nl, b.quads, b.cw_local, b.psi_sk, b.phiq, phi, sigma_s,
                                     phin, b.scat, b.norms, b.red_ws, b.ctl, it, p->si_tol,
                                     b.flags + 1, nullptr, st));
      } else {
        if (nl > 0)
          DLRSN_RET(phi_closure_launch(ops, nl, b.quads, b.cw_local, b.psi_sk, b.phiq, phi,
                                       sigma_s, nullptr, nullptr, b.norms, b.red_ws, b.ctl, -1,
                                       p->si_tol, nullptr, comm->reduce_buf, st));
        else
          DLRSN_TRY_CUDA(zero_async(comm->reduce_buf, N * sizeof(double), st));
        if (comm->allreduce_sum(comm->user) != 0) {
          set_error("allreduce of the closure flux failed");
          return DLRSN_ECUDA;
        }
        // DSA replicated on every rank from the summed flux
        if (p->use_dsa) DLRSN_RET(dsa_launch(comm->reduce_buf, phi, st));
        DLRSN_RET(phi_finish_launch(ops, comm->reduce_buf, phin, phi, sigma_s, b.scat, b.norms,
                                    b.red_ws, b.ctl, it, p->si_tol, b.flags + 1, st));
      }
    }
    si_select_kernel<<<grid_n(N), 256, 0, st>>>(N, b.ctl, b.phi0, b.phi1, si_phi);
    DLRSN_CHECK_LAUNCH("si_select_kernel");
    if (world > 1) {  // swept columns of all ranks (allgather), canonical layout
      if (nl > 0)
        DLRSN_RET(dlrsn_sk_to_canonical(ops, nl, b.quads, b.psi_sk, comm->gather_send,
                                        comm->gather_width, s));
      if (comm->allgather(comm->user) != 0) {
        set_error("allgather of the swept columns failed");
        return DLRSN_ECUDA;
      }
      place_cols_kernel<<<grid_n(N * r), 256, 0, st>>>(N, r, comm->gather_width, b.place,
                                                       comm->gather_recv, b.psi);
      DLRSN_CHECK_LAUNCH("place_cols_kernel");
    } else {
      DLRSN_RET(dlrsn_sk_to_canonical(ops, r, b.quads, b.psi_sk, b.psi, r, s));
    }
    return DLRSN_OK;
  };
  // 4. Galerkin side (dlr_sn.py:123-150) with the chosen Gram-Schmidt paths
  auto enqueue_tail = [&](cudaStream_t st, int exact, int exact_w, bool reset) -> int {
    void* s = st;
    if (reset) {
      DLRSN_TRY_CUDA(zero_async(b.statw, sizeof(int), st));
      DLRSN_TRY_CUDA(zero_async(b.statx, sizeof(int), st));
    }
    if (!exact) {
      DLRSN_RET(dlrsn_mgram(ops, r, r, b.psi, r, b.psi, r, nullptr, b.G, b.part, s));
      DLRSN_RET(dlrsn_chol_upper(r, b.G, b.R1, b.R1inv, b.ratio, b.cholflag, s));
      DLRSN_RET(rowmix_upper(N, r, b.psi, r, b.R1inv, r, b.X1, r, st));
      DLRSN_RET(dlrsn_mgram(ops, r, r, b.X1, r, b.X1, r, nullptr, b.G, b.part, s));
      DLRSN_RET(dlrsn_chol_upper(r, b.G, b.R2, b.R2inv, b.ratio2, b.cholflag + 1, s));
      DLRSN_RET(rowmix_upper(N, r, b.X1, r, b.R2inv, r, X_new, r, st));
    } else {
      DLRSN_RET(dlrsn_cgs2((int)N, r, b.psi, r, X_new, r, b.Rtot, b.defx, 1, nullptr, ops, 1,
                           r + 8, b.up->sexp, b.up->extent, b.cgsws, b.statx, 1, s));
    }
    OutCopy* oc = nullptr;
    if (p->x_new_host) {  // X_new is final: its host copy runs under the rest of the step
      DLRSN_RET(out_copy_stream(&oc));
      DLRSN_TRY_CUDA(cudaEventRecord(oc->ready, st));
      DLRSN_TRY_CUDA(cudaStreamWaitEvent(oc->cs, oc->ready, 0));
      DLRSN_TRY_CUDA(cudaMemcpyAsync(p->x_new_host, X_new, (size_t)N * r * sizeof(double),
                                     cudaMemcpyDeviceToHost, oc->cs));
      DLRSN_TRY_CUDA(cudaEventRecord(oc->done, oc->cs));
    }
    DLRSN_RET(project_ex(ops, r, X_new, X, nullptr, 1, sigma_t, sigma_s, q, b.proj, b.part,
                         b.flags + 1, st));
    if (has_inflow) DLRSN_RET(dlrsn_inflow_project(ops, r, X_new, r, p->inflow, b.hin, s));
    {
      const size_t qsm = 3 * (size_t)r * r * sizeof(double);
      const int staged = qsm <= 160 * 1024;
      if (staged)
        DLRSN_TRY_CUDA(cudaFuncSetAttribute(qall_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)qsm));
      qall_kernel<<<1, 1024, staged ? qsm : 0, st>>>(r, S, b.proj + 6 * r * r, b.proj + 7 * r * r,
                                                     W, b.idx, p->inv_cdt, b.T, b.qall,
                                                     has_inflow ? b.hin : nullptr, infl, b.om_sel,
                                                     staged);
    }
    DLRSN_CHECK_LAUNCH("qall_kernel");
    DLRSN_TRY_CUDA(zero_async(b.rowstat, (r + 1) * sizeof(int), st));
    DLRSN_RET(dlrsn_row_inverse(r, r, b.proj, b.om_sel, b.Binv, nullptr, b.rowstat, s));
    DLRSN_RET(row_combine_grid(r, r, b.Binv, b.proj + 5 * r * r, b.qall, b.closure, b.L,
                               b.lbar, b.rowstat + r, b.rcs, st));
    DLRSN_RET(dlrsn_what_solve(r, r, b.Lhat, b.U, b.L, b.gamma, 0, s));
    // two branches: the angular update (one CTA) on `st`; the flux of the
    // new state, the step boundary and the spatial check on the side stream
    Fork* fk = nullptr;
    DLRSN_RET(fork_streams(&fk));
    DLRSN_RET(fork_to(fk, st));
    {
      cudaStream_t sd = fk->side;
      void* ss2 = sd;
      // the flux of the new state phi = X_new lbar comes out of the spatial
      // check's pass over X_new (single-tile Gram, r <= 64; else its own launch)
      if (p->check_state)
        DLRSN_RET(mgram_vec(ops, r, r, X_new, r, X_new, r, nullptr, b.G, b.part, b.lbar, phi_out, ss2));
      else
        DLRSN_RET(dlrsn_rowmix(N, r, 1, X_new, r, b.lbar, 1, 0.0, phi_out, 1, ss2));
      if (p->advance) DLRSN_RET(advance_launch(p->advance, phi_out, sd));
    }
    DLRSN_RET(dlrsn_rowmix(no, r, r, W, r, b.gamma, r, 0.0, b.lfull, r, s));
    if (!exact_w && ang_fast) {
      DLRSN_RET(dlrsn_cholqr2_small(no, r, b.lfull, r, p->weights_dev, W_new, r, b.Rang,
                                    b.ratiow, b.cholw, b.defw, s));
    } else if (!exact_w) {
      // the same weighted CholQR2 over row blocks (r > 32): Gram, Cholesky,
      // Q = W R^-1, twice; R = R2 R1
      DLRSN_RET(wgram(no, r, b.lfull, p->weights_dev, b.wpart, b.wg, st));
      DLRSN_RET(dlrsn_chol_upper(r, b.wg, b.Rw1, b.Rw1inv, b.ratiow, b.cholw, s));
      DLRSN_RET(dlrsn_rowmix(no, r, r, b.lfull, r, b.Rw1inv, r, 0.0, b.lq1, r, s));
      DLRSN_RET(wgram(no, r, b.lq1, p->weights_dev, b.wpart, b.wg, st));
      DLRSN_RET(dlrsn_chol_upper(r, b.wg, b.Rw2, b.Rw2inv, b.ratiow2, b.cholw + 1, s));
      DLRSN_RET(dlrsn_rowmix(no, r, r, b.lq1, r, b.Rw2inv, r, 0.0, W_new, r, s));
      DLRSN_RET(dlrsn_small_matmul(r, r, r, b.Rw2, b.Rw1, b.Rang, 0, s));
      DLRSN_TRY_CUDA(zero_async(b.defw, r * sizeof(int), st));
    } else
      DLRSN_RET(dlrsn_cgs2(no, r, b.lfull, r, W_new, r, b.Rang, b.defw, 0, p->weights_dev,
                           nullptr, 0, r + 8, b.up->aexp, p->omegas_dev, b.cgsws, b.statw, 1, s));
    DLRSN_RET(wgram(no, r, W_new, p->weights_dev, b.wpart, b.wg, st));
    finish_kernel<<<1, 256, 0, st>>>(r, b.Rang, b.wg, S_new, beta_new);
    DLRSN_CHECK_LAUNCH("finish_kernel");
    DLRSN_RET(join_from(fk, st));
    if (p->check_state) {
      ortho_residual_kernel<<<1, 256, 0, st>>>(r, b.G, b.wg, b.chk_out, nullptr, p->x_check_out);
      DLRSN_CHECK_LAUNCH("ortho_residual_kernel");
    }
    if (oc) DLRSN_TRY_CUDA(cudaStreamWaitEvent(st, oc->done, 0));  // join the host copy
    return enqueue_status(st, b, r, hs, sweep_ws);
  };

  // angular-only fallback: the exact CGS2 of W gamma (still in lfull) and
  // what depends on it; X_new, the projections, phi and T stay as they are
  auto enqueue_angular = [&](cudaStream_t st) -> int {
    DLRSN_TRY_CUDA(zero_async(b.statw, sizeof(int), st));
    DLRSN_RET(dlrsn_cgs2(no, r, b.lfull, r, W_new, r, b.Rang, b.defw, 0, p->weights_dev, nullptr,
                         0, r + 8, b.up->aexp, p->omegas_dev, b.cgsws, b.statw, 1, st));
    DLRSN_RET(wgram(no, r, W_new, p->weights_dev, b.wpart, b.wg, st));
    finish_kernel<<<1, 256, 0, st>>>(r, b.Rang, b.wg, S_new, beta_new);
    DLRSN_CHECK_LAUNCH("finish_kernel");
    if (p->check_state) {
      ortho_residual_kernel<<<1, 256, 0, st>>>(r, b.G, b.wg, b.chk_out, nullptr, p->x_check_out);
      DLRSN_CHECK_LAUNCH("ortho_residual_kernel");
    }
    return enqueue_status(st, b, r, hs, sweep_ws);
  };

  int exact = p->gs_method == 1 ? 1 : 0;
  int exact_w = 0;
  // iteration batch: the caller's per-problem hint (the largest iteration
  // count of its earlier steps + 1, so it only grows and the graph keys stay
  // stable); every rank of a sharded step passes the same value
  const int batch0 = std::min(std::max(p->si_batch_hint, 6), 24);
  info->si_batch_hint = batch0;
  int it_next = std::min(p->si_max_iters, batch0) + 1;
  // ---- segment 1 (the whole step in the common case): replayed as a CUDA
  // graph when the same buffers come back (world 1; see graph_cache)
  {
    auto seg1 = [&](cudaStream_t st) -> int {
      DLRSN_RET(enqueue_head(st));
      DLRSN_RET(enqueue_si(st, 1, it_next - 1));
      return enqueue_tail(st, exact, exact_w, false);
    };
    GraphKey key;
    const bool graphed = world == 1 && graphs_enabled() && !sweep_timing_enabled() &&
                         !project_timing_enabled() &&
                         !p->angle_override;
    if (graphed) {
      key.set(ops, p, X, S, W, beta, sigma_t, sigma_s, q, X_new, S_new, W_new, beta_new, phi_out,
              si_phi, workspace, sweep_ws, sweep_ws_bytes, batch0, exact, exact_w);
      DLRSN_RET(graph_run(key, seg1, st0, X == g_last_xnew));
    } else {
      DLRSN_RET(seg1(st0));
    }
  }
  DLRSN_TRY_CUDA(cudaStreamSynchronize(st0));
  for (int d = 0; d < r; ++d) info->deim_gap[d] = hs->deim_gap[d];
  // errors of the reference's order (dlr_sn.py:99-109)
  if (hs->err_idx[0] >= 0) {  // InterpolationError (lowrank.py:192-199)
    info->error_index = hs->err_idx[0];
    set_error("interpolation residual vanished; basis is rank deficient");
    return DLRSN_EINTERP;
  }
  for (int d = 0; d < r; ++d) info->angle_indices[d] = hs->err_idx[d + 1];
  if (hs->flags[0]) {
    set_error("pseudo absorption sigma_t - sigma_s must stay positive");
    return DLRSN_EINVAL;
  }
  info->check_in[0] = hs->chk_in[0];
  info->check_in[1] = hs->chk_in[1];
  if (p->check_state && (hs->chk_in[0] > 1e-10 || hs->chk_in[1] > 1e-10)) {
    set_error("factor orthonormality violated: spatial %.2e, angular %.2e", hs->chk_in[0],
              hs->chk_in[1]);
    return DLRSN_EINVAL;
  }
  // ---- further segments: more iterations (the batch fell short) or an
  // exact Gram-Schmidt pass (a CholQR2 guard failed) -- rare, not graphed
  int batch = batch0;
  for (int guard = 0; guard < 1 << 20; ++guard) {
    info->sweep_status = hs->sweep_status;
    if (hs->sweep_status) {  // a strip handoff timed out: psi is not trustworthy
      DLRSN_RET(dlrsn_sweep_workspace_init(sweep_ws, sweep_ws_bytes, st0));
      DLRSN_TRY_CUDA(cudaStreamSynchronize(st0));
      set_error("sweep strip handoff timed out (status %d); workspace re-armed",
                hs->sweep_status);
      return DLRSN_ECUDA;
    }
    for (int d = 0; d < r; ++d) info->closure[d] = hs->closure[d];
    info->residual = hs->ctl.change;
    info->dsa_iterations = p->use_dsa ? hs->dsa[2] : 0;
    info->dsa_solves = p->use_dsa ? hs->dsa[3] : 0;
    if (p->use_dsa && hs->dsa[1]) {  // CgError (transport_sn.py:350)
      info->iterations = dsa_cap;
      set_error("dsa failed to reach tol %g", dsa_tol);
      return DLRSN_ECG;
    }
    if (!hs->ctl.done) {
      if (it_next > p->si_max_iters) {
        info->iterations = p->si_max_iters;
        set_error("source iteration did not converge (iterations=%d, residual=%.3e)",
                  p->si_max_iters, hs->ctl.change);
        return DLRSN_EITER;
      }
      batch = std::max(2, batch / 2);
      const int it_end = std::min(p->si_max_iters, it_next + batch - 1);
      DLRSN_RET(enqueue_si(st0, it_next, it_end));
      it_next = it_end + 1;
      DLRSN_RET(enqueue_tail(st0, exact, exact_w, true));
      DLRSN_TRY_CUDA(cudaStreamSynchronize(st0));
      continue;
    }
    info->iterations = hs->ctl.iters;
    // next step's batch hint: grows to cover this step's count (stable
    // batches keep the graph keys stable; a shortfall costs one more segment)
    // (above 8, rounded up to a multiple of 8: a slowly growing count -- the
    // Marshak wave's 15, 16, 19, 20 -- re-captures the step graphs once, not
    // at every change; iterations past convergence return at once)
    {
      const int want = hs->ctl.iters + 1;
      info->si_batch_hint = std::max(batch0, want <= 8 ? want : (want + 7) / 8 * 8);
    }
    if (!exact) {
      // CholQR's R_kk is accurate to ~eps/rel^2: keep it only when every
      // column retains >= 1e-6 of its M-norm and sits 100x above the
      // reference's deficiency threshold 1e-12 max(|v|, 1) (angular.py:137)
      bool ok = hs->cholflag[0] == 0;
      if (guard_debug()) {
        double mn = 1e300;
        for (int k = 0; k < r; ++k) mn = std::min(mn, hs->ratio[k]);
        fprintf(stderr, "dlrsn guard: spatial min ratio %.3e\n", mn);
      }
      for (int k = 0; k < r && ok; ++k) ok = hs->ratio[k] >= guard_ratio() && hs->ratio[r + k] >= 1e-10;
      if (!ok) {
        info->gs_fallback |= 1;
        exact = 1;
        DLRSN_RET(enqueue_tail(st0, exact, exact_w, true));
        DLRSN_TRY_CUDA(cudaStreamSynchronize(st0));
        continue;
      }
      info->spatial_deficiency = 0;
    } else {
      if (hs->statx) {
        set_error("ran out of completion vectors during orthonormalization");
        return DLRSN_ECOMPLETION;
      }
      int nd = 0;
      for (int k = 0; k < r; ++k) nd += hs->defx[k] != 0;
      info->spatial_deficiency = nd;
    }
    if (!exact_w) {  // same guard for the angular CholQR2 (angular.py:137 threshold)
      bool ok = hs->cholw[0] == 0 && hs->cholw[1] == 0;
      if (guard_debug()) {
        double mn = 1e300;
        for (int k = 0; k < r; ++k) mn = std::min(mn, hs->ratiow[k]);
        fprintf(stderr, "dlrsn guard: angular min ratio %.3e\n", mn);
      }
      for (int k = 0; k < r && ok; ++k) ok = hs->ratiow[k] >= guard_ratio() && hs->ratiow[r + k] >= 1e-10;
      if (!ok) {
        info->gs_fallback |= 2;
        exact_w = 1;
        DLRSN_RET(enqueue_angular(st0));
        DLRSN_TRY_CUDA(cudaStreamSynchronize(st0));
        continue;
      }
    }
    for (int d = 0; d < r; ++d)
      if (hs->rowstat[d]) {
        info->error_index = d;
        set_error("singular reduced transport operator at node %d", d);
        return DLRSN_ESINGULAR;
      }
    if (hs->rowstat[r]) {
      set_error("singular closure-coupled reduced system");
      return DLRSN_ESINGULAR;
    }
    if (hs->statw) {
      set_error("ran out of completion vectors during orthonormalization");
      return DLRSN_ECOMPLETION;
    }
    int na = 0;
    for (int k = 0; k < r; ++k) na += hs->defw[k] != 0;
    info->angular_deficiency = na;
    info->check_out[0] = hs->chk_out[0];
    info->check_out[1] = hs->chk_out[1];
    if (p->check_state && (hs->chk_out[0] > 1e-10 || hs->chk_out[1] > 1e-10)) {
      set_error("factor orthonormality violated: spatial %.2e, angular %.2e", hs->chk_out[0],
                hs->chk_out[1]);
      return DLRSN_EINVAL;
    }
    g_last_xnew = X_new;
    return DLRSN_OK;
  }
  set_error("internal: step did not settle");
  return DLRSN_ECUDA;
}

}  // extern "C"
