"""Memory-lean DLR-SN step for pure absorbers (BASELINE config 5 on one GPU).

``step_collocation(..., engine="lean")`` runs the same algorithm as the
reference (dlr_sn.py:86-151) for sigma_s = 0, where the source iteration is
a single sweep whose flux is never used by the step (transport_sn.py:410,
430-432; dlr_sn.py:111-150 reads only psi and the iteration count), with a
working set of about 2 x N_x r doubles instead of the ~6 x N_x r of the
one-call native step:

* the selected directions are swept in chunks of ``chunk`` directions: the
  chunk's psi_time = X (S W_sel^T)[:, chunk] (evaluate_rows,
  lowrank.py:220-227) is formed in a chunk buffer, laid out as the sweep rhs
  (transport_sn.py:403-407), swept IN PLACE (the rhs of a step is staged
  before that step's psi is written), and its psi columns are written
  straight into the N_x x r buffer Psi;
* CholQR2 in the M inner product (K2) runs on Psi in place (row blocks
  through a chunk buffer), so Psi becomes X_new;
* the projections (K3) read X_new and the caller's X; everything else is
  r x r or N_Omega x r.

At config 5 (N_x = 67.1 M, r = 128) the step holds X (68.7 GB), Psi / X_new
(68.7 GB) and ~18 GB of chunk buffers on one 180 GB B200.  The exact CGS2
fallback of a failed CholQR2 guard needs a separate copy of Psi, which this
mode does not have: it raises instead (the guard never fires on the
BASELINE configs).
"""

from __future__ import annotations

import ctypes
import os
import sys

import numpy as np
import torch

from . import _lib
from ._device import empty, stream
from .angular import AngularBasis, orthonormalize_async
from .errors import ContractViolation, SolverError
from .lowrank import (
    DlrState,
    _chol,
    _row_solve_async,
    _cgs2_flags,
    cgs2_spatial_async,
    check_ties,
    cholqr_guard_ok,
    deim_finish,
    deim_forced_launch,
    deim_launch,
    mass_gram,
    raise_row_status,
    rowmix,
    rowmix_upper,
)
from .transport import _SweepPlan, _sweep, assemble_operators, raise_sweep_status, sweep_status_word


def rowmix_inplace(A, K, block_rows=None):
    """A <- A K (K square) in place: the rowmix kernels load every row of a
    warp's row tile (all kx columns, into registers) before writing that
    tile's outputs, and no other warp touches those rows, so Y = X is safe
    (each element is read once, then written once, by the same warp).  The
    one-thread-per-element fallback (n < 64) is not: it goes through a copy."""
    if A.shape[0] < 64 or A.shape[1] > 128:
        A.copy_(rowmix(A, K))
        return A
    return rowmix(A, K, out=A)


class _Phases:
    """Optional per-phase device timing of the lean step (DLRSN_LEAN_PROFILE=1,
    printed to stderr): synchronises between phases, so off by default."""

    def __init__(self):
        self.on = bool(os.environ.get("DLRSN_LEAN_PROFILE"))
        self.marks = []

    def mark(self, name):
        if self.on:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append((name, ev))

    def report(self):
        if self.on and len(self.marks) > 1:
            torch.cuda.synchronize()
            parts = [f"{b[0]} {a[1].elapsed_time(b[1]):.1f}" for a, b in zip(self.marks, self.marks[1:])]
            print("dlrsn lean ms: " + ", ".join(parts), file=sys.stderr)


def _chunk_width(n, r, vl, limit=24):
    """Directions per sweep chunk: as many as fit next to the chunk's two
    buffers (psi_time n x D, SK rhs / psi D x vl) in the free device memory,
    up to ``limit`` (each chunk re-reads X once; 32 at config 5 leaves too
    little headroom for the projections' workspace)."""
    free, _ = torch.cuda.mem_get_info()
    per = 8 * (n + vl)
    fit = int(0.9 * free) // per
    return max(1, min(limit, r, fit))


def step_lean(grid, step, quad, state, *, si_tol, si_max_iters, check_state, chunk=None,
              angle_indices=None, deim_tie_tol=0.0, block_rows=None):
    from .dlr_sn import CollocationStepInfo, _NativeSelection, project_operators

    ph = _Phases()
    ph.mark("start")
    r = state.rank
    n = grid.n_dofs
    X, S, W = state.X, state.S, state.W.values
    beta = state.W.beta if state.W.beta is not None else state.W.bind(quad).beta
    # ---- DEIM, closure weights, input checks (one readback) ---------------
    if angle_indices is not None:
        sel, err_idx = deim_forced_launch(W, angle_indices)
    else:
        sel, err_idx = deim_launch(W)
    closure = sel.closure_weights(beta)
    ops = assemble_operators(grid, step, validate=False)
    st = ops.step
    flags = torch.stack([(st.sigma_t - st.sigma_s <= 0).any(), (st.sigma_s != 0).any()])
    parts = [err_idx.to(torch.float64), closure, flags.to(torch.float64), sel.gap_dev]
    if check_state:
        # DlrState.check (lowrank.py:68-81); the spatial residual of an X this
        # engine produced and checked (same tensor, unmodified) is reused
        xc = getattr(state, "_xcheck", None)
        if xc is not None and xc[1] is X and xc[2] == X._version and not state.W.pinned:
            eye = torch.eye(r, dtype=torch.float64, device=X.device)
            wq = quad.weights_device()
            parts.append(torch.stack([xc[0], ((W * wq[:, None]).T @ W - eye).abs().max()]))
        else:
            parts.append(state.check_values(ops, quad))
    host = torch.cat(parts).cpu().numpy()
    deim_finish(sel, host[:r + 1], host[2 * r + 3:3 * r + 3])
    cw = host[r + 1:2 * r + 1].copy()
    if host[2 * r + 1]:
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    if host[2 * r + 2]:
        raise ContractViolation("the lean step is for pure absorbers (sigma_s = 0): one sweep "
                                "per step (transport_sn.py:410,430-432)")
    if check_state:
        state.raise_check(host[3 * r + 3:])
    if angle_indices is None:
        check_ties(sel.gaps, deim_tie_tol)
    om_sel = quad.omegas[sel.indices]
    ph.mark("deim+checks")
    # ---- the sweep, chunk by chunk (dlr_sn.py:110-121) --------------------
    K = S @ W[sel.indices_dev].T  # (r, r): psi_time = X K (evaluate_rows)
    psi = empty(n, r)
    vl = ops.vec_len
    if chunk is None:
        env = os.environ.get("DLRSN_LEAN_CHUNK")
        chunk = int(env) if env else _chunk_width(n, r, vl)
    cbuf = empty(n * chunk)  # psi_time of a chunk, then the row-block buffer
    skbuf = empty(chunk * vl)  # rhs -> psi (in place), SK layout
    for c0 in range(0, r, chunk):
        c1 = min(r, c0 + chunk)
        D = c1 - c0
        pt = cbuf[:n * D].view(n, D)
        rowmix(X, K[:, c0:c1].contiguous(), out=pt)
        ph.mark(f"rowmix{c0}")
        plan = _SweepPlan(ops, om_sel[c0:c1], cw[c0:c1], dw=1)
        sk = skbuf[:D * vl]
        _lib.call("dlrsn_rhs_build", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev), _lib.ptr(st.q),
                  float(st.inv_cdt), _lib.ptr(pt), D, None, 1, _lib.ptr(sk), stream())
        ph.mark(f"rhs{c0}")
        _sweep(ops, plan, sk, sk)
        ph.mark(f"sweep{c0}")
        _lib.call("dlrsn_sk_to_canonical", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev),
                  _lib.ptr(sk), ctypes.c_void_p(psi.data_ptr() + 8 * c0), r, stream())
        ph.mark(f"tocanon{c0}")
        raise_sweep_status(sweep_status_word(plan.workspace).item(), plan.workspace)
    del cbuf, skbuf
    # ---- K2 in place (Psi -> X_new): CholQR2 when its guard holds (every
    # column keeps >= 1e-6 of its M-norm, read back before Psi is touched),
    # else the reference's exact CGS2 with deficiency / completion, in place
    R1, R1inv, ratio, flag = _chol(mass_gram(ops, psi))
    guard = torch.cat([ratio, flag.to(torch.float64)]).cpu().numpy()
    ph.mark("gram1")
    sdef = 0
    if cholqr_guard_ok(guard, r):
        # R^-1 is upper triangular: the in-place product skips its zero blocks
        rowmix_upper(psi, R1inv, out=psi) if r <= 128 else rowmix_inplace(psi, R1inv, block_rows)
        ph.mark("rowmix1")
        R2, R2inv, _, flag2 = _chol(mass_gram(ops, psi))
        ph.mark("gram2")
        rowmix_upper(psi, R2inv, out=psi) if r <= 128 else rowmix_inplace(psi, R2inv, block_rows)
        ph.mark("rowmix2")
        if int(flag2.item()):
            raise SolverError("lean step: second CholQR pass lost positive definiteness")
        gs_fallback = 0
    else:
        _, _, defi_x, status_x = cgs2_spatial_async(ops.cellops, psi, r + 8, True, out=psi)
        hx = torch.cat([defi_x[:r].to(torch.float64), status_x.to(torch.float64)]).cpu().numpy()
        sdef = len(_cgs2_flags(hx[:r], hx[r:], r))
        gs_fallback = 1
    if os.environ.get("DLRSN_GUARD_DEBUG"):
        print(f"dlrsn lean guard: min ratio {guard[:r].min():.3e}, fallback {gs_fallback}",
              file=sys.stderr)
    x_new = psi
    # ---- K3 + the reduced row system + the angular update (dlr_sn.py:126-141)
    ph.mark("k2")
    proj, packed = project_operators(ops, x_new, x_old=X, no_scatter=True)  # checked above
    ph.mark("k3")
    w_sel = W[sel.indices_dev]
    q_all = (proj["q"][None, :] + st.inv_cdt * (w_sel @ (S.T @ proj["mo"]))).contiguous()
    om_dev = quad.omegas_device()[sel.indices_dev].contiguous()
    l_nodes, l_bar, row_status = _row_solve_async(r, r, packed, om_dev, proj["ms"].contiguous(),
                                                  q_all, closure)
    gamma = sel.interpolation_coefficients(l_nodes)
    l_full = rowmix(W, gamma)
    basis_new, r_ang, defi_w, status_w = orthonormalize_async(l_full, quad)
    new_state = DlrState(X=x_new, S=r_ang.T.contiguous(), W=basis_new)
    parts = [row_status.to(torch.float64), defi_w[:r].to(torch.float64),
             status_w.to(torch.float64)]
    if check_state:
        out_check = new_state.check_values(ops, quad)
        parts.append(out_check)
        new_state._xcheck = (out_check[0].clone(), x_new, x_new._version)
    host = torch.cat(parts).cpu().numpy()
    ph.mark("rows+angular+check")
    ph.report()
    raise_row_status(host[:r + 1], r)
    adef = host[r + 1:2 * r + 1]
    _cgs2_flags(adef, [host[2 * r + 1]], r)
    if check_state:
        new_state.raise_check(host[2 * r + 2:])
    info = CollocationStepInfo(
        iterations=1, selection=_NativeSelection(sel.indices, W), angle_indices=sel.indices.copy(),
        phi=rowmix(x_new, l_bar.reshape(-1, 1))[:, 0], spatial_deficiency=sdef,
        angular_deficiency=int(np.count_nonzero(adef)))
    info.deim_gaps = sel.gaps
    info.gs_fallback = gs_fallback
    return new_state, info
