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
from .angular import orthonormalize
from .lowrank import (
    DlrState,
    _addr,
    _cellops_of,
    _row_solve,
    deim_select,
    evaluate_rows,
    gram_schmidt_mass,
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
    """Advance one linearised step; returns (new DlrState, CollocationStepInfo)."""
    selection = deim_select(state.W.values)
    closure = selection.closure_weights(state.W.beta)
    closure_host = closure.cpu().numpy()
    omegas_sel = quad.omegas[selection.indices]

    penalty_closure = (omegas_sel, closure_host) if dsa_penalty == "collocation" else None
    ops = assemble_operators(grid, step, dsa_penalty=dsa_penalty, penalty_closure=penalty_closure)
    if check_state:
        state.check(ops, quad)

    flux0 = evaluate_rows(state, selection)
    result = source_iteration(
        ops, omegas_sel, closure_host, psi_time=flux0.values, use_dsa=use_dsa, tol=si_tol,
        max_iters=si_max_iters, phi_start=state.scalar_flux(), threads=threads, dw=sweep_dw,
        comm=comm)

    # new spatial basis from the converged swept columns (dlr_sn.py:123-125)
    x_new, _, deficient_x = gram_schmidt_mass(ops, result.psi, state.rank + 8, method=gs_method)

    # reduced row solve against the new basis (dlr_sn.py:127-132)
    r = state.rank
    proj, packed = project_operators(ops, x_new, x_old=state.X)
    w_sel = state.W.values[selection.indices_dev]
    l_time = w_sel @ (state.S.T @ proj["mo"])
    q_all = (proj["q"][None, :] + step.inv_cdt * l_time).contiguous()
    om_sel = as_device(omegas_sel).contiguous()
    l_nodes, l_bar = _row_solve(r, r, packed, om_sel, proj["ms"].contiguous(), q_all, closure)

    # nodal rows -> angular functions through the old basis (dlr_sn.py:134-137)
    gamma = selection.interpolation_coefficients(l_nodes)
    l_full = rowmix(state.W.values, gamma)
    basis_new, r_ang, deficient_w = orthonormalize(l_full, quad)

    new_state = DlrState(X=x_new, S=r_ang.T.contiguous(), W=basis_new)
    if check_state:
        new_state.check(ops, quad)
    info = CollocationStepInfo(
        iterations=result.iterations,
        selection=selection,
        angle_indices=selection.indices.copy(),
        phi=rowmix(x_new, l_bar.reshape(-1, 1))[:, 0],
        spatial_deficiency=len(deficient_x),
        angular_deficiency=len(deficient_w),
        si_phi=result.phi,
    )
    return new_state, info
