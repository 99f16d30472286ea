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
