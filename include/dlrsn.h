/*
 * dlrsn.h -- C ABI of the B200 (sm_100a) SN-like DLR hot path.
 *
 * The reference (greytrt, Python/numpy) has no FFI: its boundary is the
 * Python function API.  These entry points are what a maintainer would bind
 * (ctypes / cffi) to replace the numpy kernels under
 * that API.  Each declaration cites the reference function it replaces
 * (paths relative to /root/reference/pkg/src/greytrt).
 *
 * Conventions
 *  - All pointers are caller-owned DEVICE pointers, except `ops`
 *    (const dlrsn_cellops*), which points to HOST memory.  fp64 throughout ("f64"); ints are int32 unless noted.
 *  - `stream` is a cudaStream_t passed as void*.  No entry point allocates
 *    device memory or synchronises the host; workspaces are caller-owned.
 *  - Return: 0 = DLRSN_OK, negative = error (see codes).  The Python shim
 *    maps them onto the reference's exceptions (errors.py:4-41);
 *    dlrsn_last_error() gives the message of the last failing call.
 *  - Canonical layout = the reference's: dof = 4*cell + local,
 *    cell = j*nx + i, local 0..3 = corners (0,0),(1,0),(0,1),(1,1)
 *    (mesh.py:28-33,117-118); psi/X are (n_dofs, ld) row-major.
 *  - "SK" layout (sweep-native, per direction or per quadrant): for the
 *    quadrant (sx,sy) a cell (i,j) is addressed by oriented coordinates
 *    i' = sx>0 ? i : nx-1-i, j' = sy>0 ? j : ny-1-j, strip s = j'/32,
 *    lane = j'%32, step t = i' + lane; a 4-dof slab is
 *    [n_strips][nx+31][2 dof-pairs][32 lanes][2] f64 with local dofs stored
 *    in the oriented frame (local' = local ^ (sx<0) ^ 2*(sy<0)); a scalar
 *    slab is [n_strips][nx+31][32].  dlrsn_sk_vec_len / dlrsn_sk_scalar_len
 *    give the per-slab element counts.
 */
#ifndef DLRSN_H
#define DLRSN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* dlrsn_stream_t;

enum {
  DLRSN_OK = 0,
  DLRSN_EINVAL = -1,      /* ContractViolation */
  DLRSN_ESINGULAR = -2,   /* SolverError (singular reduced operator) */
  DLRSN_ENONFINITE = -3,  /* SolverError (non-finite values) */
  DLRSN_ECUDA = -4,       /* CUDA runtime failure */
  DLRSN_EINTERP = -5,     /* InterpolationError */
  DLRSN_ECOMPLETION = -6, /* ContractViolation: ran out of completion vectors */
  DLRSN_EITER = -7,       /* IterationLimitError (info->iterations, info->residual) */
  DLRSN_ECG = -8          /* CgError: the DSA conjugate gradient hit its iteration cap */
};

#define DLRSN_MAX_RANK 128 /* largest rank r of the step-level entry point */

#define DLRSN_MAX_DW 8 /* directions per sweep group (one warp) */

/* Per-cell reference blocks, computed on the host exactly as the reference
 * does (mesh.py:285-313 scaled as in transport_sn.py:213-227). */
typedef struct dlrsn_cellops {
  int nx, ny;
  double x0, y0, dx, dy;
  double mass[16];   /* dx*dy*Mhat, row-major */
  double gx[16];     /* -dy*Ghat_xi   (grad_cell[0]) */
  double gy[16];     /* -dx*Ghat_eta  (grad_cell[1]) */
  double e2x[4];     /* dy*Ehat (vertical faces) */
  double e2y[4];     /* dx*Ehat (horizontal faces) */
  double src_row[4]; /* mass.sum(axis=1) (transport_sn.py:124-127) */
} dlrsn_cellops;

/* One sweep group: up to DLRSN_MAX_DW directions of one quadrant swept by
 * one warp per 32-row strip.  quad = (sx<0) | 2*(sy<0). */
typedef struct dlrsn_group {
  int32_t quad;
  int32_t ndir;
  int32_t slot[DLRSN_MAX_DW]; /* direction slot (column of rhs/psi) */
  double ox[DLRSN_MAX_DW];    /* |omega_x| */
  double oy[DLRSN_MAX_DW];    /* |omega_y| */
  double cw[DLRSN_MAX_DW];    /* closure weight (phi = sum_d cw_d psi_d) */
} dlrsn_group;

int dlrsn_version(void);
const char* dlrsn_last_error(void);
/* number of kernels this library has launched since it was loaded */
int64_t dlrsn_launch_count(void);
int dlrsn_device_sm_count(int* out);

int64_t dlrsn_sk_vec_len(int nx, int ny);
int64_t dlrsn_sk_scalar_len(int nx, int ny);
/* bytes of workspace dlrsn_sweep needs for G groups of width dw; a new
 * workspace must be initialised once with dlrsn_sweep_workspace_init (the
 * sweep leaves it re-armed, so it can be reused across launches and plans).
 * Word 1 of the workspace is a sticky status (2 = a handoff wait timed out). */
/* Measurement hook: while enabled, every dlrsn_sweep records a CUDA event
 * pair around its launch on the caller's stream; _read synchronises on them
 * and returns per-launch ms, group count and width (cap entries at most;
 * *count = launches recorded).  Enabling resets the list. */
int dlrsn_sweep_timing(int enable);
int dlrsn_sweep_timing_read(int cap, float* ms, int* groups, int* dw, int* count);
int64_t dlrsn_sweep_workspace_bytes(int nx, int ny, int n_groups, int dw);
int dlrsn_sweep_workspace_init(void* workspace, int64_t workspace_bytes, dlrsn_stream_t stream);
/* debug: record globaltimer per (work item, chunk) before/after the strip
 * handoff wait into buf[(item*chunks + m)*2 + {0,1}]; buf NULL disables. */
int dlrsn_debug_trace(unsigned long long* buf, int chunks);
int dlrsn_debug_flags(int flags); /* debug: bit0 = no speculative handoff prefetch */

/* FP64 tensor-core peak probe: blocks x warps_per_block warps, each issuing
 * 8 independent chains of `iters` mma.sync m8n8k4 f64 (DMMA) on registers;
 * FLOPs = 4096 * iters * blocks * warps_per_block.  sink: device double. */
int dlrsn_dmma_probe(int blocks, int warps_per_block, int iters, double* sink,
                     dlrsn_stream_t stream);

/* ---- K4: per-cell physics (physics.py:63-132, driver.py:344-346,532-534) */

/* linearize (physics.py:94-120) + BASELINE adapters: sigma_t += ss_phys,
 * sigma_s += ss_phys, q += q_ext (nullable).  status (device int, OR-ed)
 * gets 1 if a contract fails (T<0, sigma_a<0, rho_cv<=0). */
int dlrsn_linearize(int n, const double* T0, const double* sigma_a, const double* rho_cv,
                    double dt, double c, double a_r, const double* ss_phys,
                    const double* q_ext, double* sigma_t, double* sigma_s, double* q,
                    double* denom, int* status, dlrsn_stream_t stream);

/* update_temperature (physics.py:123-132); phi is per cell, or per dof
 * (phi_per_dof=1: cell mean of the 4 dofs first, driver.py:344-346).
 * T = max(T0 + dt*sigma_a*(phi - 4 pi B(T0))/denom, t_floor). */
int dlrsn_update_temperature(int n, const double* phi, int phi_per_dof, const double* T0,
                             const double* sigma_a, const double* denom, double dt, double c,
                             double a_r, double t_floor, double* T, dlrsn_stream_t stream);

/* Fused driver step boundary: T update of the finished step followed by the
 * linearisation of the next one (driver.py:486-487,532-534 +
 * physics.py:94-120).  sigma_a(T) = sigma_a0 * T^opacity_power when
 * opacity_power != 0 (Marshak), else sigma_a0. */
/* sigma_a_in / denom_in are the finished step's coefficients (they may alias
 * the outputs sigma_a / denom); T0_out (optional) receives a copy of the new
 * T (the next step's linearisation point). */
int dlrsn_advance_relinearize(int n, const double* phi_dofs, double* T,
                              const double* sigma_a_in, const double* denom_in, double* sigma_a,
                              const double* sigma_a0, double opacity_power,
                              const double* rho_cv, double dt, double c, double a_r,
                              double t_floor, const double* ss_phys, const double* q_ext,
                              double* sigma_t, double* sigma_s, double* q, double* denom,
                              double* T0_out, int* status, dlrsn_stream_t stream);

/* ---- K1: sweep data movement (transport_sn.py:377-450) */

/* rhs_sk[d] = source_vector(q) + inv_cdt * M psi_time[:, d] + extra[:, d]
 * (transport_sn.py:403-407) for D direction slots of quadrant quad[d]
 * (host-built int array on device).  psi_time / extra are canonical
 * (n_dofs, ld_*) and nullable. */
int dlrsn_rhs_build(const dlrsn_cellops* ops, int D, const int* quad, const double* q,
                    double inv_cdt, const double* psi_time, int ld_psi_time,
                    const double* extra, int ld_extra, double* rhs_sk, dlrsn_stream_t stream);

/* Isotropic inflow boundary (BASELINE config 3; the reference is vacuum-only,
 * transport_sn.py:11-13).  inflow = HOST double[4]: psi_b on the left,
 * right, bottom, top walls (0 = vacuum).  Adds |omega.n| psi_b (e2 row sums)
 * to the wall edge dofs of each direction's SK rhs -- the reference's
 * `extra_source` slot of source_iteration (transport_sn.py:387,406-407).
 * omegas: device (rows, 3); slot d uses row map[d] (map NULL: row d). */
int dlrsn_inflow_add(const dlrsn_cellops* ops, int D, const int* quad, const double* omegas,
                     const int* map, const double* inflow, double* rhs_sk,
                     dlrsn_stream_t stream);
/* h (4 x r, device) = X^T g_w for the unit inflow load g_w of each wall w
 * with inflow[w] != 0 (0 elsewhere): the inflow part of the projected row
 * source, q_all[d] += sum_w max(-omega_d.n_w, 0) psi_b,w h[w]. */
int dlrsn_inflow_project(const dlrsn_cellops* ops, int r, const double* X, int ldx,
                         const double* inflow, double* h, dlrsn_stream_t stream);

/* Closure-only sweep (full-SN stress sweeps whose psi cannot be stored, e.g.
 * config 5's 16384 directions on 4096^2 = 8.8 TB): every direction sees the
 * same rhs (rhs_sk4 = 4 quadrant SK slabs of one rhs, e.g. an isotropic
 * source), psi is not written, and each group adds its closure sum
 * sum_d cw_d psi_d into the canonical phi (n_dofs, caller-initialised) with
 * fp64 atomics -- the summation order over groups is not fixed, so phi is
 * reproducible to round-off only.  transport_sn.py:303-322 + the closure
 * psi @ closure of :438. */
int dlrsn_sweep_closure(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                        const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk4,
                        double* phi, void* workspace, int64_t workspace_bytes, int max_ctas,
                        dlrsn_stream_t stream);

/* ---- K6: diffusion synthetic acceleration (transport_sn.py:166-198,
 * 325-367, applied at :439-441) */

/* doubles of workspace dlrsn_dsa_correct needs */
int64_t dlrsn_dsa_workspace_len(int nx, int ny);
/* phi_out = phi_half + delta, delta the Jacobi-PCG solution (x0 = 0, stop at
 * ||r|| <= tol ||b||, at most max_iters) of the consistent diffusion system
 * ((Px^T Mt^-1 Px + Py^T Mt^-1 Py)/3 + 2 kx Jx + 2 ky Jy + M_(sigma_t-sigma_s))
 * delta = M (sigma_s (phi_half - phi_old)), matrix-free on the structured
 * grid, in one cooperative launch.  kx = ky = 1/4 is the reference's
 * "simplified" penalty, the "collocation" one is 1/2 cw.|omega_x| / (4 pi).
 * info (device int[2]) = {CG iterations, 1 if max_iters was reached};
 * history (device, nullable) gets ||r_k|| for k < hist_cap. */
int dlrsn_dsa_correct(const dlrsn_cellops* ops, const double* sigma_t, const double* sigma_s,
                      double kx, double ky, const double* phi_half, const double* phi_old,
                      double* phi_out, double tol, int max_iters, double* workspace,
                      int64_t workspace_len, int* info, double* history, int hist_cap,
                      dlrsn_stream_t stream);

/* scalar per cell -> 4 quadrant SK slabs (out + k*sk_scalar_len) */
int dlrsn_cells_to_sk4(const dlrsn_cellops* ops, const double* cell_values, double* out_sk4,
                       dlrsn_stream_t stream);

/* scatter = M (sigma_s * phi) / 4 pi (transport_sn.py:436) written to the 4
 * quadrant SK slabs; also OR-s 1 into *any_scatter if some sigma_s != 0
 * (transport_sn.py:410). */
int dlrsn_scatter_source(const dlrsn_cellops* ops, const double* phi, const double* sigma_s,
                         double* scat_sk4, int* any_scatter, dlrsn_stream_t stream);

/* phi_new = sum_g phi_part[g] (fixed order) -- or, with phi_part_sk NULL,
 * sum_g sum_k cw[g][k] psi[slot[g][k]] read from the swept psi_sk -- plus
 * the scattering source for the next iteration and norms[0] =
 * ||phi_new - phi_old||^2, norms[1] = ||phi_new||^2 (deterministic
 * reduction; transport_sn.py:438,442-446).  scat_sk4 nullable.  partial_ws
 * >= 256 bytes + 2*ceil(n_cells/256) doubles (its first word must start 0). */
int dlrsn_phi_combine(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                      const double* phi_part_sk, const double* psi_sk, const double* phi_old,
                      const double* sigma_s,
                      double* phi_new, double* scat_sk4, double* norms, void* partial_ws,
                      dlrsn_stream_t stream);

/* Direction-sharded iteration (multi-GPU): phi_new is the rank-summed
 * closure flux (canonical); norms against phi_old and the next scattering
 * source, as dlrsn_phi_combine does for the unsharded case. */
int dlrsn_phi_finish(const dlrsn_cellops* ops, const double* phi_new, const double* phi_old,
                     const double* sigma_s, double* scat_sk4, double* norms, void* partial_ws,
                     dlrsn_stream_t stream);

/* psi (n_dofs, ld) canonical <- psi_sk[d] for d < D */
int dlrsn_sk_to_canonical(const dlrsn_cellops* ops, int D, const int* quad,
                          const double* psi_sk, double* psi, int ld, dlrsn_stream_t stream);

/* ---- K1: the sweep (transport_sn.py:142-163,303-322 batched over
 * directions, sweep_all :419-427, phi_half :438).
 * One persistent launch sweeps every direction of every group: warp =
 * (group, 32-row strip), lanes = rows, marching the oriented x axis; inputs
 * are staged to shared memory by TMA bulk copies; the strip above is fed
 * through an L2 handoff of self-flagging slots.  rhs_sk / psi_sk: D slabs; sigma_t_sk4 / scat_sk4: quadrant
 * slabs (scat nullable => no scattering term); phi_part_sk: G slabs
 * (nullable).  dw = template width >= max group ndir (1,2,4,8). */
int dlrsn_sweep(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk,
                double* psi_sk, double* phi_part_sk, void* workspace, int64_t workspace_bytes,
                int max_ctas, dlrsn_stream_t stream);

/* ---- K2/K3/K5: the Galerkin side of step_collocation (dlr_sn.py:86-151) */

/* Y = X K (+ beta Y): (n, kx) times small (kx, ky).  evaluate_rows
 * (lowrank.py:220-227: X (S W_sel^T)), scalar_flux (:60-62), info.phi =
 * X lbar (dlr_sn.py:147), l_full = W gamma (:136), X R^-1 (CholQR). */
int dlrsn_rowmix(int64_t n, int kx, int ky, const double* X, int ldx, const double* K, int ldk,
                 double beta, double* Y, int ldy, dlrsn_stream_t stream);

/* Y = X K for an upper-triangular r x r K (exact zeros below the diagonal:
 * the CholQR2 factors R^-1, angular.py:104-160 restated as CholQR2), r <=
 * 128: the zero blocks are skipped (72/128 of the MMAs at r = 64).  Y may
 * alias X (in place, X's row stride = Y's). */
int dlrsn_rowmix_upper(int64_t n, int r, const double* X, int ldx, const double* K, int ldk,
                       double* Y, int ldy, dlrsn_stream_t stream);

/* doubles of `partial` scratch needed by dlrsn_mgram (kind 0: ra x rb) or
 * dlrsn_project (kind 1: rank ra) */
int64_t dlrsn_partials_len(int ncell, int ra, int rb, int kind);

/* G (ra x rb) = sum_c coeff_c A_c^T M B_c (coeff nullable): mass_inner
 * Grams for Gram-Schmidt and DlrState.check (lowrank.py:23-25,68-81).
 * Deterministic fixed-order reduction. */
int dlrsn_mgram(const dlrsn_cellops* ops, int ra, int rb, const double* A, int lda,
                const double* B, int ldb, const double* coeff, double* G, double* partial,
                dlrsn_stream_t stream);

/* Measurement hook: while enabled, every dlrsn_project records a CUDA event
 * pair around its main kernel (not the partial-sum reduction); _read
 * synchronises and returns the per-launch ms (cap entries at most). */
int dlrsn_project_timing(int enable);
int dlrsn_project_timing_read(int cap, float* ms, int* count);

/* Fused reduced operators (project_row_operators, dlr_sn.py:61-71, plus
 * X_old^T M X of project_initial, :50-58) in one pass over the cells:
 * out = [px, py, jx, jy, mt, ms, mo] (7 r x r, row-major) then q-hat (r).
 * Xold nullable (mo = 0). */
int dlrsn_project(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
                  const double* sigma_t, const double* sigma_s, const double* q, double* out,
                  double* partial, dlrsn_stream_t stream);

/* dlrsn_project on one row slab of a larger grid (multi-GPU row slabs,
 * slab.py): ops describes the slab (nx x ny_slab cells), halo (nullable) the
 * X rows of the grid row just below the slab (4 nx x r) for the horizontal
 * faces on the slab's bottom edge (NULL: the domain's bottom wall), and
 * top_wall = 1 when the slab's top row is the domain's top wall (0: the face
 * above is counted by the next slab).  Summing the outputs over the slabs of
 * a grid gives dlrsn_project on the whole grid. */
int dlrsn_project_slab(const dlrsn_cellops* ops, int r, const double* X, const double* Xold,
                       const double* halo, int top_wall, const double* sigma_t,
                       const double* sigma_s, const double* q, double* out, double* partial,
                       dlrsn_stream_t stream);

/* G = R^T R (R upper) and R^-1; diag_ratio (2r): [k] = R_kk / sqrt(G_kk)
 * (relative norm left after projection), [r+k] = R_kk / max(sqrt(G_kk), 1)
 * (the CGS2 deficiency quantity of angular.py:137); *flag = 1 on a
 * non-positive pivot.  r <= 128. */
int dlrsn_chol_upper(int r, const double* G, double* R, double* Rinv, double* diag_ratio,
                     int* flag, dlrsn_stream_t stream);

/* C (m x n) = op(A) B, op = transpose if transA; small, one CTA. */
int dlrsn_small_matmul(int m, int k, int n, const double* A, const double* B, double* C,
                       int transA, dlrsn_stream_t stream);

/* Node matrices and their inverses (row_matrices dlr_sn.py:74-83 +
 * np.linalg.inv lowrank.py:245-252): B_d = wx px + wy py + |wx| jx + |wy| jy
 * + mt from the dlrsn_project output and om_sel (n x 3); om_sel NULL: proj
 * holds B (n x r x r).  status[d] = 1 if node d is singular. */
int dlrsn_row_inverse(int n, int r, const double* proj, const double* om_sel, double* Binv,
                      double* Bout, int* status, dlrsn_stream_t stream);

/* solve_row_system tail (lowrank.py:253-259): cbar, zeta, lbar, L (n x r). */
int dlrsn_row_combine(int n, int r, const double* Binv, const double* ms, const double* Q,
                      const double* wts, double* L, double* lbar, int* status,
                      dlrsn_stream_t stream);

/* deim_select (lowrank.py:168-205) by Gaussian elimination with row
 * pivoting on a work copy of W (n x r): idx (r picks), W[idx,:] = Lhat U.
 * *err_col = -1 on success, else the column whose residual vanished (or
 * that has no finite candidate left).  gap (r doubles, nullable): per pick
 * (|best| - |second best|) / |best| of the residual over the unpicked rows
 * -- 0 is an exact tie, which np.argmax (lowrank.py:191) breaks by the
 * lowest row, as this kernel does; near-ties are where round-off can flip a
 * pick.  variant: 0 auto, 1 one-thread-per-row registers (n <= 1024,
 * r <= 16), 2 thread-block cluster (DSMEM), 3 one CTA over shared / global
 * memory (Wwork used when n r doubles exceed shared memory), 4 one
 * cooperative grid over all SMs (Wwork holds the per-CTA candidate slots). */
int dlrsn_deim(int n, int r, double* Wwork, const double* W, int* idx, double* Lhat, double* U,
               int* err_col, double* gap, int variant, dlrsn_stream_t stream);

/* Forced selection (the angle_indices override of a step): idx = indices
 * (HOST int64, r entries, pick order), W[idx,:] = Lhat U without further
 * pivoting; *err_col = j when pivot j vanishes below the DEIM floor or
 * index j repeats / is out of range, else -1; gap[j] = 1.  r <= 78. */
int dlrsn_deim_forced(int n, int r, const double* W, const int64_t* indices, int* idx,
                      double* Lhat, double* U, int* err_col, double* gap, dlrsn_stream_t stream);

/* W_hat solves: mode 0 X = W_hat^-1 V (interpolation_coefficients,
 * lowrank.py:158-160), mode 1 x = W_hat^-T v (closure_weights, :162-165). */
int dlrsn_what_solve(int r, int m, const double* Lhat, const double* U, const double* V,
                     double* X, int mode, dlrsn_stream_t stream);

/* Exact twice-projected classical Gram-Schmidt with the reference's
 * deficiency test and deterministic completion (angular.py:104-160), one
 * cooperative grid launch.  metric 0: weighted rows (w, angular); 1: block
 * mass (ops, spatial, n = 4*cells).  comp_kind 0: ncomp angular monomials
 * (exponent triples, coords = omegas n x 3) then unit vectors; 1: spatial
 * monomials (exponent pairs, coords = extent x0,y0,lx,ly).  workspace:
 * dlrsn_cgs2_workspace_len(n) doubles; *status = 1 if the candidates ran
 * out (strict). */
/* Weighted CholQR2 of a small tall n x m matrix (m <= 32, fits one CTA):
 * Q R = W with Q^T diag(w) Q = I; ratio (2m) and flag (2) feed the
 * speculative-CholQR guard (see dlrsn_chol_upper); deficient[k] = 0.  The
 * full-rank fast path of the angular re-orthonormalisation. */
int64_t dlrsn_cholqr2_small_smem(int n, int m);
int dlrsn_cholqr2_small(int n, int m, const double* W, int ldw, const double* w, double* Q,
                        int ldq, double* R, double* ratio, int* flag, int* deficient,
                        dlrsn_stream_t stream);
int64_t dlrsn_cgs2_workspace_len(int n);
int dlrsn_cgs2(int n, int m, const double* cols, int ldc, double* Q, int ldq, double* R,
               int* deficient, int metric, const double* w, const dlrsn_cellops* ops,
               int comp_kind, int ncomp, const int* comp_exp, const double* coords,
               double* workspace, int* status, int strict, dlrsn_stream_t stream);

/* ---- One whole step (dlr_sn.py:86-151) ----------------------------------- */

/* Optional fused step boundary of a driver loop (driver.py:486-487,532-534):
 * after the step, T_out = the updated temperature of the finished step and
 * (sigma_a .. denom) = the next step's linearisation (dlrsn_advance_relinearize
 * out of place: T_in and the *_in fields are not written, so a failing step
 * leaves the caller's state untouched). */
typedef struct dlrsn_advance {
  int n;                     /* cells */
  const double* T_in;
  const double* sigma_a_in;
  const double* denom_in;
  const double* sigma_a0;
  double opacity_power;
  const double* rho_cv;
  double dt, c, a_r, t_floor;
  const double* ss_phys;     /* optional */
  const double* q_ext;       /* optional */
  double* T_out;
  double* sigma_a;
  double* sigma_t;
  double* sigma_s;
  double* q;
  double* denom;
} dlrsn_advance;

typedef struct dlrsn_step_params {
  int rank;                  /* r <= DLRSN_MAX_RANK */
  int n_omega;               /* quadrature size */
  const double* omegas_host; /* (n_omega, 3), HOST */
  const double* omegas_dev;  /* (n_omega, 3), device */
  const double* weights_dev; /* (n_omega), device */
  double inv_cdt;            /* LinearizedStep.inv_cdt */
  double si_tol;             /* source iteration tolerance */
  int si_max_iters;
  int check_state;           /* DlrState.check on input and output */
  int gs_method;             /* 0: CholQR2 guarded by exact CGS2, 1: exact CGS2 */
  int sweep_dw;              /* sweep group width (0 = 1) */
  const dlrsn_advance* advance; /* optional fused T update + re-linearisation (NULL: none) */
  double inflow[4];          /* isotropic inflow psi_b: left, right, bottom, top (0: vacuum) */
  const double* x_check_in;  /* device, optional: max|X^T M X - I| of the input X, already
                                computed by the step that produced it (the input Gram is then
                                skipped; M depends on the grid only, so the value is the one
                                the Gram would give).  NULL: compute it */
  double* x_check_out;       /* device, optional: receives max|X_new^T M X_new - I| */
  int si_batch_hint;         /* source iterations enqueued before the first convergence
                                readback (0: library default 6).  The caller keeps it per
                                problem (step_info.si_batch_hint of the previous step); with
                                world_size > 1 every rank must pass the same value, since the
                                batch fixes the number of allreduce callbacks per segment */
  int angle_override;        /* 1: use angle_indices_in instead of the DEIM picks
                                (forced-selection parity, lowrank.py:168-205 hazard (i)) */
  const int64_t* angle_indices_in; /* HOST, r entries, read when angle_override */
  double* x_new_host;        /* HOST pinned (n_dofs x r), optional: X_new is copied here on a
                                copy stream as soon as it is final (after K2), overlapping the
                                projections and the angular update; the call returns after the
                                copy (a caller holding its state in host memory) */
  int use_dsa;               /* 1: diffusion synthetic acceleration of every source iteration
                                inside the call (transport_sn.py:439-441; K6 on the device, no
                                host synchronisation per iteration) */
  int dsa_penalty;           /* 0: "simplified" (kx = ky = 1/4), 1: "collocation" (1/2
                                closure.|omega_x|/(4 pi) of the step's own DEIM selection,
                                dlr_sn.py:104, transport_sn.py:183-188; formed on the device) */
  double dsa_tol;            /* PCG relative tolerance (0: the reference's 1e-10) */
  int dsa_max_iters;         /* PCG cap (0: the reference's 10 n_dofs) */
  double* dsa_history;       /* device, optional: ||r_k|| of the (first failed, else last) PCG */
  int dsa_hist_cap;
} dlrsn_step_params;

typedef struct dlrsn_step_info { /* HOST, filled by the call */
  int iterations;
  int spatial_deficiency;
  int angular_deficiency;
  int error_index;           /* InterpolationError column / singular node, else -1 */
  int gs_fallback;           /* bit 0: exact CGS2 replaced the spatial CholQR2,
                                bit 1: ... the angular one */
  double residual;           /* last source-iteration change */
  double check_in[2];        /* input orthonormality residuals (spatial, angular) */
  double check_out[2];
  int64_t angle_indices[DLRSN_MAX_RANK];
  double closure[DLRSN_MAX_RANK];
  int si_batch_hint;         /* suggested si_batch_hint for the next step of this problem */
  int sweep_status;          /* sweep workspace status word (2: a strip handoff timed out;
                                the call then fails with DLRSN_ECUDA and re-arms the workspace) */
  double deim_gap[DLRSN_MAX_RANK]; /* per pick: (|top| - |second|) / |top| of the DEIM
                                residual (near-tie diagnostic, lowrank.py:191 argmax) */
  int dsa_iterations;        /* use_dsa: PCG iterations summed over the step's source iterations */
  int dsa_solves;            /* use_dsa: diffusion solves that ran (zero-residual ones excluded) */
} dlrsn_step_info;

/* Multi-GPU hooks (NULL = one GPU): the step calls allreduce_sum(user) to
 * sum reduce_buf (n_dofs doubles, device) over ranks once per source
 * iteration, and allgather(user) to gather gather_send (n_dofs x
 * gather_width) of every rank into gather_recv (world_size blocks). */
typedef struct dlrsn_comm {
  int rank, world_size;
  void* user;
  int (*allreduce_sum)(void* user);
  int (*allgather)(void* user);
  double* reduce_buf;
  double* gather_send;
  double* gather_recv;
  int gather_width;
} dlrsn_comm;

int64_t dlrsn_step_workspace_bytes(int nx, int ny, int r, int n_omega, int world_size);

/* step_collocation (dlr_sn.py:86-151) in one call: DEIM, closure, collocated
 * source iteration, M-orthonormal spatial basis (CholQR2 / CGS2), fused
 * projections, row solve, angular re-orthonormalisation, checks.  Inputs
 * X (n_dofs, r), S (r, r), W (n_omega, r), beta (r), per-cell sigma_t,
 * sigma_s, q; outputs X_new, S_new, W_new, beta_new, phi = X_new lbar (the
 * flux of the temperature update) and si_phi (source-iteration flux).
 * Returns DLRSN_EINTERP / DLRSN_EINVAL / DLRSN_EITER / DLRSN_ESINGULAR /
 * DLRSN_ECOMPLETION like the reference raises (errors in its order). */
int dlrsn_step_collocation(const dlrsn_cellops* ops, const dlrsn_step_params* p, const double* X,
                           const double* S, const double* W, const double* beta,
                           const double* sigma_t, const double* sigma_s, const double* q,
                           double* X_new, double* S_new, double* W_new, double* beta_new,
                           double* phi, double* si_phi, void* workspace, int64_t workspace_bytes,
                           void* sweep_ws, int64_t sweep_ws_bytes, const dlrsn_comm* comm,
                           dlrsn_step_info* info, dlrsn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DLRSN_H */
