"""Oracle time loop for the BASELINE configs -- TEST INFRASTRUCTURE ONLY.

Restates the dlr-sn branch of the reference driver (``driver.py:485-539``:
linearize -> step_collocation -> dofs_to_cells -> update_temperature ->
floor) on top of ``oracle.port``, with the SURVEY Appendix B adapters
(physical scattering / external source added to the linearised step the way
``tests/test_transport_sn.py:22-36`` does).
"""

from __future__ import annotations

import numpy as np

from . import port as P


def grid_of(spec):
    x0, y0, lx, ly = spec.extent
    return P.Grid(spec.nx, spec.ny, x0, y0, lx, ly)


def quad_of(spec):
    return P.build_quadrature(spec.n_polar, spec.n_azimuthal)


def constants_of(spec):
    return P.Constants(c=spec.c, a_r=spec.a_r)


def orthonormal_factors(spec, Xraw, Wraw):
    """Random-orthonormal X (M inner product, spatial-monomial completion) and
    W (quadrature-weighted), SURVEY Appendix B."""
    grid, quad = grid_of(spec), quad_of(spec)
    ops = P.assemble_operators(grid, _dummy_step(spec), with_matrices=False)
    comp = P.spatial_monomials(P.dof_coordinates(grid), grid.extent, spec.rank + 8)
    X, _, dx = P.gram_schmidt(Xraw, P.mass_dot(ops), comp)
    W, _, dw = P.orthonormalize(Wraw, quad)
    assert not dx and not dw
    return X, W


def initial_state(spec, X, W, T=None):
    """S = (X^T M b0) beta^T: projection of the isotropic B(T0) state."""
    grid, quad = grid_of(spec), quad_of(spec)
    ops = P.assemble_operators(grid, _dummy_step(spec), with_matrices=False)
    T = spec.T0 if T is None else T
    b0, _ = P.planck(P.cells_to_dofs(T), constants_of(spec))
    beta = W.T @ quad.weights
    S = np.outer(X.T @ ops.mass_apply(b0), beta)
    return P.State(X, S, W, beta)


def linearized(spec, T):
    """Per-step coefficients (physics.py:94-120 plus the BASELINE adapters)."""
    k = constants_of(spec)
    if spec.frozen:
        icdt = 1.0 / (spec.c * spec.dt)
        n = spec.n_cells
        st = P.linearize(T, np.asarray(spec.frozen_sigma_t) - icdt, spec.rho_cv, spec.dt, k)
        st.sigma_t = np.asarray(spec.frozen_sigma_t, float).copy()
        st.sigma_s = np.zeros(n)
        st.q = np.asarray(spec.frozen_q, float).copy()
        return st
    st = P.linearize(T, spec.opacity_at(T), spec.rho_cv, spec.dt, k)
    st.sigma_t = st.sigma_t + spec.sigma_s_phys
    st.sigma_s = st.sigma_s + spec.sigma_s_phys
    st.q = st.q + spec.q_ext
    return st


def advance_temperature(spec, lin, phi_dofs):
    """driver.py:532-534: cell means, Newton update, then the floor."""
    raw = P.update_temperature(P.dofs_to_cells(phi_dofs), lin, -np.inf)
    return np.maximum(raw, spec.t_floor)


def run(spec, state, n_steps, *, si_tol=1e-12, si_max_iters=400, use_dsa=False,
        check_state=True, T=None, record=None):
    grid, quad = grid_of(spec), quad_of(spec)
    T = np.asarray(spec.T0 if T is None else T, dtype=float).copy()
    infos = []
    for _ in range(n_steps):
        lin = linearized(spec, T)
        state, info = P.step_collocation(grid, lin, quad, state, si_tol=si_tol,
                                         si_max_iters=si_max_iters, use_dsa=use_dsa,
                                         check_state=check_state,
                                         inflow=getattr(spec, "inflow", None))
        T = advance_temperature(spec, lin, info.phi)
        infos.append(info)
        if record is not None:
            record(state, info, T)
    return state, T, infos


def _dummy_step(spec):
    n = spec.n_cells
    one = np.ones(n)
    return P.Step(one * 2.0, one, one, one, one, one, one, 1.0, 1.0)


def run_sn(spec, n_steps, *, si_tol=1e-12, si_max_iters=400, use_dsa=False):
    """The reference driver's full-SN method (driver.py:463-466, 492-504)
    with its energy rows (driver.py:521-553): returns (psi, records) with
    records[k] = (T, phi, iterations, (e_mat, e_rad, outflow, residual,
    floor_source))."""
    grid, quad = grid_of(spec), quad_of(spec)
    k = constants_of(spec)
    T = np.asarray(spec.T0, dtype=float).copy()
    b0, _ = P.planck(P.cells_to_dofs(T), k)
    psi = np.tile(b0[:, None], (1, quad.n_angles))
    phi = psi @ quad.weights
    area = grid.cell_area
    e_mat = float(np.sum(spec.rho_cv * T) * area)
    e_rad = float(P.dofs_to_cells(phi).sum() * area) / k.c
    recs = []
    for _ in range(n_steps):
        lin = linearized(spec, T)
        ops = P.assemble_operators(grid, lin)
        res = P.source_iteration(ops, quad.omegas, quad.weights, psi_time=psi, use_dsa=use_dsa,
                                 tol=si_tol, max_iters=si_max_iters, phi_start=phi)
        psi, phi = res.psi, res.phi
        raw = P.update_temperature(P.dofs_to_cells(phi), lin, -np.inf)
        Tn = np.maximum(raw, spec.t_floor)
        floor_source = float(np.sum(spec.rho_cv * (Tn - raw)) * area)
        outflow = P.boundary_outflow(grid, psi, quad.omegas, quad.weights)
        e_mat_n = float(np.sum(spec.rho_cv * Tn) * area)
        e_rad_n = float(P.dofs_to_cells(psi @ quad.weights).sum() * area) / k.c
        total = e_mat_n + e_rad_n
        resid = (total - e_mat - e_rad + spec.dt * outflow - floor_source) / max(abs(total), 1e-300)
        e_mat, e_rad = e_mat_n, e_rad_n
        T = Tn
        recs.append((T, phi, res.iterations, np.array([e_mat, e_rad, outflow, resid, floor_source])))
    return psi, recs
