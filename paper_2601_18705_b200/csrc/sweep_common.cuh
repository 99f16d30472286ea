// Shared pieces of the two sweep kernels (sweep.cu: general group width;
// sweep_ws.cu: warp-specialised single-direction groups).
#pragma once

#include "common.cuh"

namespace dlrsn {

struct SweepArgs {
  int nx, ny, G;
  const dlrsn_group* groups;
  const double* sigma_sk4;
  const double* scat_sk4;
  const double* rhs_sk;
  double* psi_sk;
  double* phi_sk;
  int* ticket;
  double* handoff;
  int* status;
  double mass[16];
  double gxp[16];  // Gx + e2x embedded at the right edge (oriented +x outflow)
  double gyp[16];  // Gy + e2y embedded at the top edge
  double ex[4];    // e2x (left inflow coupling)
  double ey[4];    // e2y (bottom inflow coupling)
  int64_t vlen, slen;
  unsigned long long* trace;  // debug timeline (dlrsn_debug_trace), null in production
  int trace_chunks;
  const int* skip;  // device flag: return at once when set (speculative iterations)
  int debug;        // bit 0: ignore the strip inflow (timing experiments only)
  // closure-only sweeps (full-SN stress, no psi storage): rhs_sk holds 4
  // quadrant slabs of one rhs shared by every direction, psi_sk is null and
  // the group's closure sum is added into the canonical phi_atomic
  int rhs_shared;
  double* phi_atomic;
};

// Direction groups of the grouped single-direction sweep (sweep1g_kernel):
// up to kCgWarps directions of one quadrant swept by one CTA in lock step,
// their closure summed in shared memory (one partial slab per group).
// first/count index the quadrant-ordered single-direction group list.
constexpr int kMaxCg = DLRSN_MAX_RANK + 4;
struct CgTable {
  int ncg;
  int pad[3];
  int first[kMaxCg];
  int count[kMaxCg];
  int quad[kMaxCg];
};

// isotropic inflow psi_b on the left, right, bottom, top walls (0: vacuum)
struct Inflow4 {
  double v[4];
};

// Device-side control of a batched source iteration (step.cu): iterations
// enqueued past convergence see done = 1 and return immediately.
struct SiCtl {
  int done;    // converged (or pure absorber after one sweep)
  int iters;   // iteration that converged
  int last;    // last iteration that ran
  int pad;
  double change;  // last relative change
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Empty handoff slot: a signalling NaN with a fixed payload.  Arithmetic only
// produces quiet NaNs, so a swept value can never alias it.
constexpr unsigned long long kEmpty = 0x7FF4DEADBEEFCAFEull;
__device__ __forceinline__ bool is_empty(double v) {
  return (unsigned long long)__double_as_longlong(v) == kEmpty;
}

// 1/x without the IEEE slow path: hardware approximation + two Newton steps
// (relative error ~1 ulp; A's pivots are positive and normal).
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ void solve4(double* a, double* b, double* x) {
  // Gaussian elimination without pivoting: A has a positive-definite
  // symmetric part (sigma_t M + upwind outflow terms), so the pivots are
  // positive.  The reference inverts with LAPACK (transport_sn.py:158); the
  // two differ only at round-off.
  const double p0 = rcp64(a[0]);
  double l = a[4] * p0;
  a[5] -= l * a[1]; a[6] -= l * a[2]; a[7] -= l * a[3]; b[1] -= l * b[0];
  l = a[8] * p0;
  a[9] -= l * a[1]; a[10] -= l * a[2]; a[11] -= l * a[3]; b[2] -= l * b[0];
  l = a[12] * p0;
  a[13] -= l * a[1]; a[14] -= l * a[2]; a[15] -= l * a[3]; b[3] -= l * b[0];
  const double p1 = rcp64(a[5]);
  l = a[9] * p1;
  a[10] -= l * a[6]; a[11] -= l * a[7]; b[2] -= l * b[1];
  l = a[13] * p1;
  a[14] -= l * a[6]; a[15] -= l * a[7]; b[3] -= l * b[1];
  const double p2 = rcp64(a[10]);
  l = a[14] * p2;
  a[15] -= l * a[11]; b[3] -= l * b[2];
  x[3] = b[3] * rcp64(a[15]);
  x[2] = (b[2] - a[11] * x[3]) * p2;
  x[1] = (b[1] - a[6] * x[2] - a[7] * x[3]) * p1;
  x[0] = (b[0] - a[1] * x[1] - a[2] * x[2] - a[3] * x[3]) * p0;
}


int launch_sweep_ws(const SweepArgs& a, int max_ctas, cudaStream_t st);

bool sweep_timing_enabled();
bool project_timing_enabled();
int advance_launch(const dlrsn_advance* av, const double* phi, cudaStream_t st);
// sweep.cu: the grouped single-direction sweep (psi + per-group closure
// partials, one partial slab of sk_vec_len doubles per group)
int sweep_grouped_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                         const CgTable* tab, const double* sigma_t_sk4, const double* scat_sk4,
                         const double* rhs_sk, double* psi_sk, double* part, void* workspace,
                         int64_t workspace_bytes, const int* skip, cudaStream_t st);
int cgroup_plan_launch(int G, const dlrsn_group* groups, int wpc, int dmax, CgTable* tab,
                       int* cg_quad, double* cg_w, cudaStream_t st);
int sweep_group_width();
// dense.cu: dlrsn_project_slab with the device scattering flag (ms = 0 and
// its MMAs skipped when *any_scat == 0)
int project_ex(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
               const double* halo, int top_wall, const double* sigma_t, const double* sigma_s,
               const double* q, double* out, double* partial, const int* any_scat,
               cudaStream_t stream);
// dense.cu: Y = X K for an upper-triangular r x r K (skips the zero blocks)
// dense.cu: Y = X K (+ beta Y) and, with v / yv, yv = X v from the same pass over X
int rowmix_vec(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
               double beta, double* Y, int ldy, const double* v, double* yv,
               dlrsn_stream_t stream);
// dense.cu: dlrsn_mgram and, with v / yv, yv = B v from the rows the Gram stages
int mgram_vec(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda, const double* B,
              int ldb, const double* coeff, double* G, double* partial, const double* v,
              double* yv, dlrsn_stream_t stream);
int rowmix_upper(int64_t n, int r, const double* X, int ldx, const double* K, int ldk, double* Y,
                 int ldy, cudaStream_t st);
// dense.cu: the row-system combine as grids (scratch r*r + 2r doubles)
int row_combine_grid(int n, int r, const double* Binv, const double* ms, const double* Q,
                     const double* wts, double* L, double* lbar, int* status, double* scratch,
                     cudaStream_t st);  // physics.cu  // dlrsn_sweep_timing on (the step then skips graphs)

// internal entry points of the step (step.cu); the public C-ABI calls pass
// skip / ctl = nullptr
int sweep_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                 const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk,
                 double* psi_sk, double* phi_part_sk, void* workspace, int64_t workspace_bytes,
                 int max_ctas, const int* skip, cudaStream_t st);
int phi_combine_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                       const double* phi_part_sk, const double* psi_sk, const double* phi_old,
                       const double* sigma_s, double* phi_new, double* scat_sk4, double* norms,
                       void* partial_ws, SiCtl* ctl, int it, double tol, const int* any_scat,
                       cudaStream_t st);
// closure flux in two coalesced passes over the SK slabs of D swept slots:
// per-quadrant partials into phiq (4 x n_dofs), then the sum + norms +
// scattering source (partial_out != nullptr: rank partial only, sharded)
int phi_closure_launch(const dlrsn_cellops* ops, int D, const int* quads, const double* cw,
                       const double* psi_sk, double* phiq, const double* phi_old,
                       const double* sigma_s, double* phi_new, double* scat_sk4, double* norms,
                       void* partial_ws, SiCtl* ctl, int it, double tol, const int* any_scat,
                       double* partial_out, cudaStream_t st);
// K6 inside the one-call step (dsa.cu): phi_out = phi_half + delta; k_dev
// (device, nullable) overrides (kx, ky); *skip != 0 returns at once; with
// accumulate, info = {last iterations, sticky failure, total iterations, solves}
int dsa_correct_launch(const dlrsn_cellops* ops, const double* sigma_t, const double* sigma_s,
                       double kx, double ky, const double* k_dev, const double* phi_half,
                       const double* phi_old, double* phi_out, double tol, int max_iters,
                       double* workspace, int* info, double* history, int hist_cap,
                       const int* skip, int accumulate, cudaStream_t st);
int phi_finish_launch(const dlrsn_cellops* ops, const double* phi_src, double* phi_dst,
                      const double* phi_old, const double* sigma_s, double* scat_sk4,
                      double* norms, void* partial_ws, SiCtl* ctl, int it, double tol,
                      const int* any_scat, cudaStream_t st);

}  // namespace dlrsn
