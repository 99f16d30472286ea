"""One implicit SN-like DLR step on the B200 (mirror of dlr_sn.py:40-151).

Algorithm 1 of the paper, same call signature and
results as the reference ``step_collocation``:

1. DEIM angles of the current angular basis, closure weights;
2. collocated source iteration over the selected directions (K1 sweeps);
3. new spatial basis from the swept columns (M-orthonormal, K2);
4. reduced row system from the fused projections (K3) solved at the nodes;
5. nodal rows -> angular functions through the old basis, orthonormalised.

All arrays stay on the device; the host only sees the r selected indices
and closure weights (to lay out the sweep groups) and the convergence
scalars of the source iteration.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from ._device import as_device, empty, stream
from .angular import orthonormalize_async
from .errors import ContractViolation
from .lowrank import (
    DlrState,
    _addr,
    _cellops_of,
    _cgs2_flags,
    _row_solve_async,
    cgs2_spatial_async,
    cholqr2_speculative,
    cholqr_guard_ok,
    deim_finish,
    deim_launch,
    evaluate_rows,
    raise_row_status,
    rowmix,
)
from .transport import assemble_operators, source_iteration

FOUR_PI = 4.0 * np.pi


@dataclass(eq=False)
class CollocationStepInfo:
    """dlr_sn.py:40-47; ``phi`` is a device tensor, the condition number of
    W_hat is evaluated on first access."""

    iterations: int
    selection: object
    angle_indices: np.ndarray
    phi: torch.Tensor
    spatial_deficiency: int
    angular_deficiency: int
    si_phi: torch.Tensor | None = None

    @cached_property
    def interpolation_condition(self):
        return self.selection.cond


def project_operators(ops, x, x_old=None):
    """Fused reduced operators: dict px, py, jx, jy, mt, ms, mo (r x r) and q
    (project_row_operators dlr_sn.py:61-71; mo = X_old^T M x for
    project_initial :50-58).  Returns (dict, packed device buffer)."""
    co = _cellops_of(ops)
    x = as_device(x).contiguous()
    r = x.shape[1]
    nc = co.nx * co.ny
    part = empty(max(int(_lib.load().dlrsn_partials_len(nc, r, r, 1)), 1))
    out = empty(7 * r * r + r)
    xo = None if x_old is None else as_device(x_old).contiguous()
    st = ops.step
    _lib.call("dlrsn_project", _addr(co), r, _lib.ptr(x), _lib.ptr(xo), _lib.ptr(st.sigma_t),
              _lib.ptr(st.sigma_s), _lib.ptr(st.q), _lib.ptr(out), _lib.ptr(part), stream())
    mats = out[:7 * r * r].reshape(7, r, r)
    names = ("px", "py", "jx", "jy", "mt", "ms", "mo")
    proj = {k: mats[i] for i, k in enumerate(names)}
    proj["q"] = out[7 * r * r:]
    return proj, out


def project_row_operators(ops, x):
    """dlr_sn.py:61-71."""
    proj, _ = project_operators(ops, x)
    proj.pop("mo")
    return proj


def row_matrices(proj, omegas):
    """dlr_sn.py:74-83."""
    om = as_device(np.asarray(omegas, dtype=float))
    return (om[:, 0, None, None] * proj["px"] + om[:, 1, None, None] * proj["py"]
            + om[:, 0].abs()[:, None, None] * proj["jx"] + om[:, 1].abs()[:, None, None] * proj["jy"]
            + proj["mt"][None])


def project_initial(state, x_new, ops):
    """Old factors against a new spatial basis (dlr_sn.py:50-58)."""
    from .lowrank import mass_gram

    mo = mass_gram(ops, state.X, x_new)
    return state.W.values @ (state.S.T @ mo)


def step_collocation(grid, step, quad, state, *, si_tol=1e-8, si_max_iters=200, use_dsa=True,
                     dsa_penalty="simplified", threads=0, check_state=True, gs_method="cholqr2",
                     sweep_dw=None, comm=None):
    """Advance one linearised step; returns (new DlrState, CollocationStepInfo).

    Host synchronisations: one before the source iteration (DEIM picks,
    closure weights and the input checks come back together), one per source
    iteration (convergence test) and one at the end (Gram-Schmidt guard,
    row-system status, angular deficiencies, output check).  Errors are raised
    in the reference's order (dlr_sn.py:99-141).
    """
    r = state.rank
    # ---- DEIM + closure + input checks: one readback ------------------------
    selection, err_idx = deim_launch(state.W.values)
    closure = selection.closure_weights(state.W.beta)
    ops = assemble_operators(grid, step, dsa_penalty=dsa_penalty, validate=False)
    bad_sigma = (step.sigma_t - step.sigma_s <= 0).any().to(torch.float64).reshape(1)
    parts = [err_idx.to(torch.float64), closure, bad_sigma]
    if check_state:
        parts.append(state.check_values(ops, quad))
    host = torch.cat(parts).cpu().numpy()
    deim_finish(selection, host[:r + 1])                       # InterpolationError
    closure_host = host[r + 1:2 * r + 1].copy()
    if host[2 * r + 1]:                                        # transport_sn.py:208-209
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    if check_state:
        state.raise_check(host[2 * r + 2:])                    # lowrank.py:68-81
    omegas_sel = quad.omegas[selection.indices]
    if dsa_penalty == "collocation":
        ops.penalty_closure = (omegas_sel, closure_host)

    # ---- collocated source iteration (dlr_sn.py:110-121) ---------------------
    flux0 = evaluate_rows(state, selection)
    result = source_iteration(
        ops, omegas_sel, closure_host, psi_time=flux0.values, use_dsa=use_dsa, tol=si_tol,
        max_iters=si_max_iters, phi_start=state.scalar_flux(), threads=threads, dw=sweep_dw,
        comm=comm)

    # ---- Galerkin side, speculative CholQR2 (dlr_sn.py:123-141) --------------
    tail = _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result,
                          gs_method, check_state)
    if gs_method == "cholqr2" and not tail["gs_ok"]:
        tail = _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result,
                              "cgs2", check_state)
    new_state = tail["state"]
    info = CollocationStepInfo(
        iterations=result.iterations,
        selection=selection,
        angle_indices=selection.indices.copy(),
        phi=tail["phi"],
        spatial_deficiency=tail["sdef"],
        angular_deficiency=tail["adef"],
        si_phi=result.phi,
    )
    return new_state, info


def _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result, gs_method,
                   check_state):
    r = state.rank
    co = _cellops_of(ops)
    if gs_method == "cholqr2":
        x_new, _, guard = cholqr2_speculative(co, result.psi)
        defi_x = status_x = None
    else:
        x_new, _, defi_x, status_x = cgs2_spatial_async(co, result.psi, r + 8, True)
        guard = None

    proj, packed = project_operators(ops, x_new, x_old=state.X)
    w_sel = state.W.values[selection.indices_dev]
    l_time = w_sel @ (state.S.T @ proj["mo"])
    q_all = (proj["q"][None, :] + step.inv_cdt * l_time).contiguous()
    om_sel = quad.omegas_device()[selection.indices_dev].contiguous()
    l_nodes, l_bar, row_status = _row_solve_async(r, r, packed, om_sel, proj["ms"].contiguous(),
                                                  q_all, closure)
    gamma = selection.interpolation_coefficients(l_nodes)
    l_full = rowmix(state.W.values, gamma)
    basis_new, r_ang, defi_w, status_w = orthonormalize_async(l_full, quad)
    new_state = DlrState(X=x_new, S=r_ang.T.contiguous(), W=basis_new)

    parts = [row_status.to(torch.float64), defi_w[:r].to(torch.float64),
             status_w.to(torch.float64)]
    if guard is not None:
        parts.append(guard)
    else:
        parts += [defi_x[:r].to(torch.float64), status_x.to(torch.float64)]
    if check_state:
        parts.append(new_state.check_values(ops, quad))
    host = torch.cat(parts).cpu().numpy()
    o = r + 1
    row_flags = host[:o]
    adef = host[o:o + r]
    st_w = host[o + r]
    o += r + 1
    if guard is not None:
        gs_ok = cholqr_guard_ok(host[o:o + 2 * r + 1], r)
        o += 2 * r + 1
        if not gs_ok:
            return {"gs_ok": False}
        sdef = 0
    else:
        sdef = len(_cgs2_flags(host[o:o + r], host[o + r:o + r + 1], r))
        o += r + 1
    raise_row_status(row_flags, r)                             # SolverError
    _cgs2_flags(adef, [st_w], r)                               # ContractViolation
    if check_state:
        new_state.raise_check(host[o:])
    return {"gs_ok": True, "state": new_state, "sdef": sdef,
            "adef": int(np.count_nonzero(adef)),
            "phi": rowmix(x_new, l_bar.reshape(-1, 1))[:, 0]}
