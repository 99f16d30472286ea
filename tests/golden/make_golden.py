"""Generate the golden vectors that pin the oracle (and, through it, the GPU
path) to the REAL reference implementation.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``greytrt`` read-only, runs it on small seeded inputs covering the
hot path (physics, quadrature, sweeps incl. every quadrant and a grazing
angle, source iteration with/without scattering and with DSA, CGS2 with
deficiency + completion, DEIM, projections, row solve, full DLR-SN steps on
checkerboard problems incl. config 1 itself, cold-empty and full-rank edge
cases) and writes ``tests/golden/*.npz``.  Nothing under /root/reference is
copied; only its outputs are stored.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from greytrt import angular, dlr_sn, driver, lowrank, mesh, physics, transport_sn  # noqa: E402

from paper_2601_18705_b200 import problems  # noqa: E402

FOUR_PI = 4.0 * np.pi


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(np.asarray(v).nbytes for v in arrays.values()), "bytes raw")


def manual_step(n, sigma_t, sigma_s, q, inv_cdt):
    """tests/test_transport_sn.py:22-36 pattern with per-cell arrays."""
    sigma_t = np.asarray(sigma_t, float)
    return physics.LinearizedStep(
        sigma_t=sigma_t, sigma_s=np.asarray(sigma_s, float), sigma_a=sigma_t - inv_cdt,
        q=np.asarray(q, float), T0=np.zeros(n), denom=np.ones(n), rho_cv=np.ones(n),
        dt=1.0, inv_cdt=float(inv_cdt))


def gen_physics():
    rng = np.random.default_rng(101)
    T = np.concatenate([[0.0, 1.0, 1e-4, 0.3], rng.uniform(0, 2, 12)])
    sa = np.concatenate([[0.0, 5.0, 1e4, 0.2], rng.uniform(0, 50, 12)])
    rc = rng.uniform(0.1, 3.0, T.size)
    out = {"T": T, "sigma_a": sa, "rho_cv": rc}
    for tag, k in (("default", physics.PhysicsConstants()), ("unit", physics.PhysicsConstants(1.0, 1.0))):
        B, dB = physics.planck(T, k)
        st = physics.linearize(T, sa, rc, 0.37, k)
        phi = rng.uniform(0, 3, T.size)
        Tn = physics.update_temperature(phi, st)
        out.update({f"{tag}_B": B, f"{tag}_dB": dB, f"{tag}_sigma_t": st.sigma_t,
                    f"{tag}_sigma_s": st.sigma_s, f"{tag}_q": st.q, f"{tag}_denom": st.denom,
                    f"{tag}_inv_cdt": st.inv_cdt, f"{tag}_phi": phi, f"{tag}_Tnew": Tn,
                    f"{tag}_c": k.c, f"{tag}_a_r": k.a_r})
    save("physics", dt=0.37, **out)


def gen_quadrature():
    out = {}
    for npol, naz in ((2, 4), (4, 8), (16, 16), (3, 6)):
        q = angular.build_quadrature(npol, naz)
        out[f"om_{npol}_{naz}"] = q.omegas
        out[f"w_{npol}_{naz}"] = q.weights
        out[f"anti_{npol}_{naz}"] = q.antipode
    save("quadrature", **out)


def gen_sweep():
    out = {}
    for tag, (nx, ny, ext, seed) in {"a": (5, 4, (0.0, 0.0, 1.0, 2.0), 33),
                                      "b": (7, 9, (1.0, -2.0, 3.5, 2.0), 34)}.items():
        rng = np.random.default_rng(seed)
        g = mesh.build_grid(nx, ny, extent=ext)
        n = g.n_cells
        sig = np.exp(rng.uniform(np.log(1e-2), np.log(1e4), n))
        st = manual_step(n, sig, 0.0 * sig, np.zeros(n), 0.5)
        ops = transport_sn.assemble_operators(g, st)
        quad = angular.build_quadrature(2, 4)
        om = np.vstack([quad.omegas, [[0.0, 0.9, 0.1], [-0.7, 0.0, 0.3], [0.0, -0.4, 0.2]]])
        rhs = rng.standard_normal((g.n_dofs, om.shape[0]))
        psi = np.stack([transport_sn.sweep_solve(ops, om[d], rhs[:, d]) for d in range(om.shape[0])], 1)
        out.update({f"{tag}_grid": np.array([nx, ny, *ext]), f"{tag}_sigma_t": sig,
                    f"{tag}_omegas": om, f"{tag}_rhs": rhs, f"{tag}_psi": psi})
    save("sweep", **out)


def gen_source_iteration():
    out = {}
    rng = np.random.default_rng(44)
    g = mesh.build_grid(6, 5, extent=(0.0, 0.0, 1.2, 1.0))
    n = g.n_cells
    sig = np.exp(rng.uniform(np.log(0.5), np.log(50.0), n))
    ss = sig * rng.uniform(0.2, 0.9, n)
    q = rng.uniform(0, 1, n)
    quad = angular.build_quadrature(2, 6)
    om = quad.omegas[[0, 3, 5, 7, 8, 10, 11]]
    clo = rng.uniform(0.5, 2.5, om.shape[0])
    pt = rng.standard_normal((g.n_dofs, om.shape[0]))
    ps = rng.standard_normal(g.n_dofs)
    ext = 0.1 * rng.standard_normal((g.n_dofs, om.shape[0]))
    out.update(grid=np.array([6, 5, 0.0, 0.0, 1.2, 1.0]), sigma_t=sig, sigma_s=ss, q=q,
               omegas=om, closure=clo, psi_time=pt, phi_start=ps, extra=ext, inv_cdt=0.4)
    for tag, dsa in (("plain", False), ("dsa", True)):
        ops = transport_sn.assemble_operators(g, manual_step(n, sig, ss, q, 0.4))
        res = transport_sn.source_iteration(ops, om, clo, psi_time=pt, use_dsa=dsa, tol=1e-12,
                                            max_iters=400, phi_start=ps, extra_source=ext)
        out.update({f"{tag}_psi": res.psi, f"{tag}_phi": res.phi, f"{tag}_iters": res.iterations})
    ops = transport_sn.assemble_operators(g, manual_step(n, sig, 0 * ss, q, 0.4))
    res = transport_sn.source_iteration(ops, om, clo, psi_time=pt, use_dsa=False, tol=1e-12)
    out.update(absorber_psi=res.psi, absorber_phi=res.phi, absorber_iters=res.iterations)
    # iteration-limit behaviour (tests/test_transport_sn.py:229-240 pattern)
    g8 = mesh.build_grid(8, 8)
    ops = transport_sn.assemble_operators(
        g8, manual_step(64, np.full(64, 100.0), np.full(64, 99.99), np.ones(64), 0.0))
    q24 = angular.build_quadrature(2, 4)
    try:
        transport_sn.source_iteration(ops, q24.omegas, q24.weights, use_dsa=False, tol=1e-8, max_iters=10)
    except Exception as err:  # IterationLimitError
        out.update(limit_iters=err.iterations, limit_residual=err.residual)
    save("source_iteration", **out)


def gen_gram_schmidt():
    out = {}
    rng = np.random.default_rng(55)
    g = mesh.build_grid(5, 4, extent=(0.0, 0.0, 2.0, 1.0))
    mass = driver.assemble_mass(g)
    cols = rng.standard_normal((g.n_dofs, 6))
    cols[:, 3] = 0.5 * cols[:, 0] - 2.0 * cols[:, 1]  # exactly dependent -> completion
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, 6 + 8)
    q, r, defi = angular.gram_schmidt(cols, lowrank.mass_inner(mass), comp)
    out.update(x_cols=cols, x_q=q, x_r=r, x_def=np.array(defi))
    quad = angular.build_quadrature(3, 6)
    wc = rng.standard_normal((quad.n_angles, 5))
    wc[:, 2] = wc[:, 0] * 1e-3
    wc[:, 4] = 0.0
    basis, rr, dw = angular.orthonormalize(wc, quad)
    out.update(w_cols=wc, w_q=basis.values, w_r=rr, w_def=np.array(dw), w_beta=basis.beta)
    save("gram_schmidt", **out)


def gen_deim():
    out = {}
    rng = np.random.default_rng(66)
    quad = angular.build_quadrature(4, 8)
    for r in (1, 3, 6, 12):
        W, _, _ = angular.orthonormalize(rng.standard_normal((quad.n_angles, r)), quad)
        sel = lowrank.deim_select(W.values)
        out.update({f"W{r}": W.values, f"idx{r}": sel.indices, f"cond{r}": sel.cond,
                    f"closure{r}": sel.closure_weights(W.beta),
                    f"gamma{r}": sel.interpolation_coefficients(rng.standard_normal((r, r)))})
        out[f"vals{r}"] = rng.standard_normal((r, r))
        out[f"gamma{r}"] = sel.interpolation_coefficients(out[f"vals{r}"])
    save("deim", **out)


def gen_projections():
    rng = np.random.default_rng(77)
    g = mesh.build_grid(6, 5, extent=(0.0, 0.0, 1.5, 1.0))
    n = g.n_cells
    mass = driver.assemble_mass(g)
    sig = rng.uniform(1, 20, n)
    ss = sig * rng.uniform(0.1, 0.8, n)
    q = rng.uniform(0, 1, n)
    st = manual_step(n, sig, ss, q, 0.3)
    ops = transport_sn.assemble_operators(g, st)
    x = angular.gram_schmidt(rng.standard_normal((g.n_dofs, 5)), lowrank.mass_inner(mass))[0]
    proj = dlr_sn.project_row_operators(ops, x)
    quad = angular.build_quadrature(2, 6)
    state = lowrank.DlrState(
        X=angular.gram_schmidt(rng.standard_normal((g.n_dofs, 5)), lowrank.mass_inner(mass))[0],
        S=rng.standard_normal((5, 5)),
        W=angular.orthonormalize(rng.standard_normal((quad.n_angles, 5)), quad)[0])
    pinit = dlr_sn.project_initial(state, x, mass)
    bm = dlr_sn.row_matrices(proj, quad.omegas[:5])
    Q = rng.standard_normal((5, 5))
    clo = rng.uniform(0.5, 2.0, 5)
    L, lbar = lowrank.solve_row_system(bm, proj["ms"], Q, clo)
    save("projections", sigma_t=sig, sigma_s=ss, q=q, x=x, inv_cdt=0.3,
         old_X=state.X, old_S=state.S, old_W=state.W.values, pinit=pinit,
         omegas=quad.omegas[:5], B=bm, Q=Q, closure=clo, L=L, lbar=lbar,
         **{f"p_{k}": v for k, v in proj.items()})


def sketch(X, S, W, seed=9):
    rng = np.random.default_rng(seed)
    phi = rng.standard_normal((X.shape[0], 12))
    om = rng.standard_normal((W.shape[0], 12))
    return (phi.T @ X) @ S @ (W.T @ om)


def diag_row(g, quad, spec, T_prev, T, raw_T, psi_full, e_prev):
    """driver.run_problem's per-step energy diagnostics (driver.py:532-553):
    (e_mat, e_rad, outflow, residual, floor_source) via the reference's own
    boundary_outflow / integrate_dofs on the dense intensity."""
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    floor_source = float(np.sum(spec.rho_cv * (T - raw_T)) * g.cell_area)
    outflow = transport_sn.boundary_outflow(g, psi_full, quad.omegas, quad.weights)
    e_mat = float(np.sum(spec.rho_cv * T) * g.cell_area)
    e_rad = driver.integrate_dofs(g, psi_full @ quad.weights) / k.c
    total = e_mat + e_rad
    residual = (total - e_prev[0] - e_prev[1] + spec.dt * outflow - floor_source) / max(abs(total), 1e-300)
    return np.array([e_mat, e_rad, outflow, residual, floor_source])


def initial_energies(g, quad, spec, phi_dofs):
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    return (float(np.sum(spec.rho_cv * spec.T0) * g.cell_area),
            driver.integrate_dofs(g, phi_dofs) / k.c)


def gen_sn():
    """The reference driver's full-SN method (driver.py:463-466, 492-504:
    psi0 = B(T0) on every direction, source_iteration over all quadrature
    nodes with psi_time = psi) plus its energy diagnostics, on a small
    checkerboard (SURVEY App. B adapters), with and without DSA."""
    spec = problems.checkerboard(2, rank=4, n_polar=4, n_azimuthal=4, seed=21, n_steps=3)
    g = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    quad = angular.build_quadrature(spec.n_polar, spec.n_azimuthal)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    out = {}
    for tag, dsa in (("plain", False), ("dsa", True)):
        T = spec.T0.copy()
        b0, _ = physics.planck(driver.cells_to_dofs(g, T), k)
        psi = np.tile(b0[:, None], (1, quad.n_angles))
        phi = psi @ quad.weights
        e_prev = initial_energies(g, quad, spec, phi)
        for s in range(spec.n_steps):
            lin = physics.linearize(T, spec.sigma_a, spec.rho_cv, spec.dt, k)
            lin.sigma_t = lin.sigma_t + spec.sigma_s_phys
            lin.sigma_s = lin.sigma_s + spec.sigma_s_phys
            lin.q = lin.q + spec.q_ext
            ops = transport_sn.assemble_operators(g, lin)
            res = transport_sn.source_iteration(ops, quad.omegas, quad.weights, psi_time=psi,
                                                use_dsa=dsa, tol=1e-12, max_iters=400,
                                                phi_start=phi)
            psi, phi = res.psi, res.phi
            raw = physics.update_temperature(driver.dofs_to_cells(g, phi), lin, -np.inf)
            Tn = np.maximum(raw, spec.t_floor)
            row = diag_row(g, quad, spec, T, Tn, raw, psi, e_prev)
            e_prev = (row[0], row[1])
            T = Tn
            out.update({f"{tag}{s}_T": T, f"{tag}{s}_phi": phi, f"{tag}{s}_iters": res.iterations,
                        f"{tag}{s}_diag": row})
            print("sn", tag, s, res.iterations, row)
        out[f"{tag}_psi"] = psi
    save("sn", **out)


def run_checker(tag, per, r, nq, nsteps, seed, compact=False):
    """Reference dlr-sn loop on a checkerboard (SURVEY App. B adapters).
    ``compact``: BASELINE-size runs (config 2) keep phi, T and the sketches
    but not the quadrature flux, and skip the dense energy rows."""
    spec = problems.checkerboard(per, rank=r, n_polar=nq, n_azimuthal=nq, seed=seed)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    # reference-side orthonormalisation of the seeded draws
    g = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    quad = angular.build_quadrature(nq, nq)
    mass = driver.assemble_mass(g)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, r + 8)
    X, _, _ = angular.gram_schmidt(Xr, lowrank.mass_inner(mass), comp)
    Wb, _, _ = angular.orthonormalize(Wr, quad)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    b0, _ = physics.planck(driver.cells_to_dofs(g, spec.T0), k)
    S = np.outer(X.T @ (mass @ b0), Wb.beta)
    state = lowrank.DlrState(X=X, S=S, W=Wb)
    out = {"X0_mb0": X.T @ (mass @ b0), "X0_colsum": X.sum(axis=0), "W0": Wb.values, "S0": S}
    T = spec.T0.copy()
    e_prev = initial_energies(g, quad, spec, state.scalar_flux())
    for s in range(nsteps):
        lin = physics.linearize(T, spec.sigma_a, spec.rho_cv, spec.dt, k)
        lin.sigma_t = lin.sigma_t + spec.sigma_s_phys
        lin.sigma_s = lin.sigma_s + spec.sigma_s_phys
        lin.q = lin.q + spec.q_ext
        state, info = dlr_sn.step_collocation(g, lin, quad, state, si_tol=1e-12, si_max_iters=400,
                                              use_dsa=False)
        raw = physics.update_temperature(driver.dofs_to_cells(g, info.phi), lin, -np.inf)
        Tn = np.maximum(raw, 1e-6)
        if not compact:
            row = diag_row(g, quad, spec, T, Tn, raw, state.reconstruct(), e_prev)
            e_prev = (row[0], row[1])
            out[f"s{s}_diag"] = row
            out[f"s{s}_phiq"] = state.scalar_flux()
        T = Tn
        out.update({f"s{s}_idx": info.angle_indices, f"s{s}_iters": info.iterations,
                    f"s{s}_cond": info.interpolation_condition, f"s{s}_phi": info.phi,
                    f"s{s}_T": T, f"s{s}_S": state.S, f"s{s}_W": state.W.values,
                    f"s{s}_sketch": sketch(state.X, state.S, state.W.values),
                    f"s{s}_xsketch": np.random.default_rng(19).standard_normal(
                        (12, state.X.shape[0])) @ state.X,
                    f"s{s}_sdef": info.spatial_deficiency, f"s{s}_adef": info.angular_deficiency})
        print(tag, "step", s, info.iterations, info.angle_indices)
    if per <= 3:
        out.update(final_X=state.X, final_S=state.S, final_W=state.W.values)
    save(tag, nsteps=nsteps, per=per, rank=r, nq=nq, seed=seed, **out)


def run_c1_twenty():
    """BASELINE config 1 in full: all 20 steps of the real reference's dlr-sn
    loop (driver.py:485-539 restated as in run_checker), kept small: per step
    the picks, SI count, T, S, W and random sketches of phi and X S W^T."""
    tag, per, r, nq, nsteps, seed = "dlr_c1_20", 10, 8, 16, 20, 1
    spec = problems.checkerboard(per, rank=r, n_polar=nq, n_azimuthal=nq, seed=seed)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    g = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    quad = angular.build_quadrature(nq, nq)
    mass = driver.assemble_mass(g)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, r + 8)
    X, _, _ = angular.gram_schmidt(Xr, lowrank.mass_inner(mass), comp)
    Wb, _, _ = angular.orthonormalize(Wr, quad)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    b0, _ = physics.planck(driver.cells_to_dofs(g, spec.T0), k)
    S = np.outer(X.T @ (mass @ b0), Wb.beta)
    state = lowrank.DlrState(X=X, S=S, W=Wb)
    proj = np.random.default_rng(23).standard_normal((12, g.n_dofs))
    out = {}
    T = spec.T0.copy()
    for s in range(nsteps):
        lin = physics.linearize(T, spec.sigma_a, spec.rho_cv, spec.dt, k)
        lin.sigma_t = lin.sigma_t + spec.sigma_s_phys
        lin.sigma_s = lin.sigma_s + spec.sigma_s_phys
        lin.q = lin.q + spec.q_ext
        state, info = dlr_sn.step_collocation(g, lin, quad, state, si_tol=1e-12, si_max_iters=400,
                                              use_dsa=False)
        raw = physics.update_temperature(driver.dofs_to_cells(g, info.phi), lin, -np.inf)
        T = np.maximum(raw, 1e-6)
        out.update({f"s{s}_idx": info.angle_indices, f"s{s}_iters": info.iterations,
                    f"s{s}_phisk": proj @ info.phi, f"s{s}_T": T, f"s{s}_S": state.S,
                    f"s{s}_W": state.W.values,
                    f"s{s}_sketch": sketch(state.X, state.S, state.W.values),
                    f"s{s}_sdef": info.spatial_deficiency, f"s{s}_adef": info.angular_deficiency})
        print(tag, "step", s, info.iterations, info.angle_indices, flush=True)
    save(tag, nsteps=nsteps, per=per, rank=r, nq=nq, seed=seed, proj_seed=23, **out)


def run_c2_fifty():
    """BASELINE config 2 in full: all 50 steps of the real reference (~40 s a
    step here), stored as projections only (the fixture stays small): per
    step the picks, SI and deficiency counts, S, and 12-row random
    projections of T, info.phi, W and X S W^T."""
    tag, per, r, nq, nsteps, seed = "dlr_c2_50", 40, 16, 32, 50, 2
    spec = problems.checkerboard(per, rank=r, n_polar=nq, n_azimuthal=nq, seed=seed)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    g = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    quad = angular.build_quadrature(nq, nq)
    mass = driver.assemble_mass(g)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, r + 8)
    X, _, _ = angular.gram_schmidt(Xr, lowrank.mass_inner(mass), comp)
    Wb, _, _ = angular.orthonormalize(Wr, quad)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    b0, _ = physics.planck(driver.cells_to_dofs(g, spec.T0), k)
    S = np.outer(X.T @ (mass @ b0), Wb.beta)
    state = lowrank.DlrState(X=X, S=S, W=Wb)
    pr = np.random.default_rng(29)
    pT = pr.standard_normal((12, g.n_cells))
    pphi = pr.standard_normal((12, g.n_dofs))
    pW = pr.standard_normal((12, quad.n_angles))
    out = {}
    T = spec.T0.copy()
    for s in range(nsteps):
        lin = physics.linearize(T, spec.sigma_a, spec.rho_cv, spec.dt, k)
        lin.sigma_t = lin.sigma_t + spec.sigma_s_phys
        lin.sigma_s = lin.sigma_s + spec.sigma_s_phys
        lin.q = lin.q + spec.q_ext
        state, info = dlr_sn.step_collocation(g, lin, quad, state, si_tol=1e-12, si_max_iters=400,
                                              use_dsa=False)
        raw = physics.update_temperature(driver.dofs_to_cells(g, info.phi), lin, -np.inf)
        T = np.maximum(raw, 1e-6)
        out.update({f"s{s}_idx": info.angle_indices, f"s{s}_iters": info.iterations,
                    f"s{s}_Tp": pT @ T, f"s{s}_phip": pphi @ info.phi, f"s{s}_S": state.S,
                    f"s{s}_Wp": pW @ state.W.values,
                    f"s{s}_sketch": sketch(state.X, state.S, state.W.values),
                    f"s{s}_sdef": info.spatial_deficiency, f"s{s}_adef": info.angular_deficiency})
        print(tag, "step", s, info.iterations, info.angle_indices, flush=True)
        if s % 10 == 9:  # checkpoint: a long run survives an interruption
            save(tag, nsteps=s + 1, per=per, rank=r, nq=nq, seed=seed, proj_seed=29, **out)
    save(tag, nsteps=nsteps, per=per, rank=r, nq=nq, seed=seed, proj_seed=29, **out)


def ref_step_inflow(g, og, step, quad, state, inflow, si_tol):
    """step_collocation (dlr_sn.py:99-151) composed from the reference's own
    functions, plus the two inflow terms of the restatement (the reference
    is vacuum-only and does not forward extra_source): the load joins the
    sweep rhs via source_iteration(extra_source=...) and the rows via
    X_new^T load."""
    from oracle import port as OP

    sel = lowrank.deim_select(state.W.values)
    closure = sel.closure_weights(state.W.beta)
    om = quad.omegas[sel.indices]
    ops = transport_sn.assemble_operators(g, step)
    mass = ops.mass_matrix()
    state.check(mass, quad)
    flux0 = lowrank.evaluate_rows(state, sel)
    extra = OP.inflow_load(og, om, inflow)
    res = transport_sn.source_iteration(ops, om, closure, psi_time=flux0.values, use_dsa=False,
                                        tol=si_tol, max_iters=800, phi_start=state.scalar_flux(),
                                        extra_source=extra)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, state.rank + 8)
    x_new, _, dx = angular.gram_schmidt(res.psi, lowrank.mass_inner(mass), comp)
    proj = dlr_sn.project_row_operators(ops, x_new)
    B = dlr_sn.row_matrices(proj, om)
    l_time = dlr_sn.project_initial(state, x_new, mass)[sel.indices]
    q_all = proj["q"][None, :] + step.inv_cdt * l_time + (x_new.T @ extra).T
    l_nodes, l_bar = lowrank.solve_row_system(B, proj["ms"], q_all, closure)
    gamma = sel.interpolation_coefficients(l_nodes)
    basis, r_ang, dw = angular.orthonormalize(state.W.values @ gamma, quad)
    new = lowrank.DlrState(X=x_new, S=r_ang.T.copy(), W=basis)
    new.check(mass, quad)
    return new, res.iterations, sel.indices.copy(), x_new @ l_bar


def gen_inflow():
    """Inflow boundary restatement pinned on the reference's operators:
    (1) known answer -- isotropic inflow psi_b on every wall with
    q = (sigma_t - sigma_s) psi_b reproduces psi = psi_b exactly (the DG
    upwind scheme is exact for constants); (2) a left-wall inflow source
    iteration with scattering; (3) 3 DLR steps of a small Marshak problem
    (sigma_a = 300 T^-3, left inflow at T_b = 1) composed from the
    reference's step functions."""
    from oracle import port as OP

    out = {}
    rng = np.random.default_rng(71)
    g = mesh.build_grid(6, 5, extent=(0.0, 0.0, 1.2, 1.0))
    og = OP.Grid(6, 5, 0.0, 0.0, 1.2, 1.0)
    n = g.n_cells
    sig = np.exp(rng.uniform(np.log(0.5), np.log(50.0), n))
    ss = sig * rng.uniform(0.2, 0.9, n)
    quad = angular.build_quadrature(2, 6)
    psib = 0.37
    ops = transport_sn.assemble_operators(g, manual_step(n, sig, ss, (sig - ss) * psib, 0.0))
    ext = OP.inflow_load(og, quad.omegas, (psib,) * 4)
    res = transport_sn.source_iteration(ops, quad.omegas, quad.weights, use_dsa=False, tol=1e-14,
                                        max_iters=800, extra_source=ext)
    out.update(const_psi=res.psi, const_phi=res.phi, const_iters=res.iterations,
               const_sigma_t=sig, const_sigma_s=ss, const_psib=psib)
    q = rng.uniform(0, 1, n)
    om = quad.omegas
    pt = rng.standard_normal((g.n_dofs, om.shape[0]))
    ops = transport_sn.assemble_operators(g, manual_step(n, sig, ss, q, 0.4))
    ext = OP.inflow_load(og, om, {"left": 0.8, "top": 0.3})
    res = transport_sn.source_iteration(ops, om, quad.weights, psi_time=pt, use_dsa=False,
                                        tol=1e-13, max_iters=800, extra_source=ext)
    out.update(si_q=q, si_psi_time=pt, si_load=ext, si_psi=res.psi, si_phi=res.phi,
               si_iters=res.iterations)
    # 3 Marshak steps (8x8, r=4, 4x4 quadrature), reference-orthonormalised draws
    spec = problems.marshak(n=8, rank=4, n_polar=4, n_azimuthal=4, dt=1e-3, n_steps=3, seed=3,
                            T_init=0.05)
    r = spec.rank
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    gm = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    ogm = OP.Grid(spec.nx, spec.ny, *spec.extent)
    qm = angular.build_quadrature(spec.n_polar, spec.n_azimuthal)
    mass = driver.assemble_mass(gm)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(gm), gm.extent, r + 8)
    X, _, _ = angular.gram_schmidt(Xr, lowrank.mass_inner(mass), comp)
    Wb, _, _ = angular.orthonormalize(Wr, qm)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    b0, _ = physics.planck(driver.cells_to_dofs(gm, spec.T0), k)
    S = np.outer(X.T @ (mass @ b0), Wb.beta)
    state = lowrank.DlrState(X=X, S=S, W=Wb)
    out.update(m_X0=X, m_S0=S, m_W0=Wb.values, m_inflow=np.array(spec.inflow))
    T = spec.T0.copy()
    for s in range(spec.n_steps):
        lin = physics.linearize(T, spec.opacity_at(T), spec.rho_cv, spec.dt, k)
        state, it, idx, phi = ref_step_inflow(gm, ogm, lin, qm, state, spec.inflow, 1e-12)
        T = np.maximum(physics.update_temperature(driver.dofs_to_cells(gm, phi), lin, -np.inf),
                       spec.t_floor)
        out.update({f"m{s}_X": state.X, f"m{s}_S": state.S, f"m{s}_W": state.W.values,
                    f"m{s}_T": T, f"m{s}_iters": it, f"m{s}_idx": idx, f"m{s}_phi": phi})
        print("marshak step", s, it, idx, T.max())
    save("inflow", **out)


def gen_edge_cases():
    """Cold-empty problem (tests/test_dlr_sn.py:127-136) and the full-rank
    step (tests/test_dlr_sn.py:91-109), outputs of the reference."""
    from helpers_ref import cell_step, random_state  # noqa: F401  (reference test helpers)

    out = {}
    g = mesh.build_grid(4, 4)
    quad = angular.build_quadrature(2, 4)
    mass = driver.assemble_mass(g)
    rng = np.random.default_rng(10)
    st = random_state(g, quad, 3, rng, mass=mass, scale=0.0)
    step = cell_step(g, 2.0, dt=0.2, T0=0.0)
    new, info = dlr_sn.step_collocation(g, step, quad, st)
    out.update(cold_X=st.X, cold_S=st.S, cold_W=st.W.values, cold_newX=new.X, cold_newS=new.S,
               cold_newW=new.W.values, cold_phi=info.phi, cold_sdef=info.spatial_deficiency,
               cold_adef=info.angular_deficiency, cold_idx=info.angle_indices,
               cold_iters=info.iterations)
    rng = np.random.default_rng(8)
    st = random_state(g, quad, quad.n_angles, rng, mass=mass, scale=0.05)
    step = cell_step(g, 2.0, dt=0.3, T0=0.6)
    new, info = dlr_sn.step_collocation(g, step, quad, st, si_tol=1e-13, si_max_iters=800, use_dsa=False)
    out.update(full_X=st.X, full_S=st.S, full_W=st.W.values, full_newX=new.X, full_newS=new.S,
               full_newW=new.W.values, full_phi=info.phi, full_idx=info.angle_indices,
               full_iters=info.iterations, full_sigma_t=step.sigma_t, full_sigma_s=step.sigma_s,
               full_q=step.q, full_inv_cdt=step.inv_cdt, full_psi=new.reconstruct())
    save("edge_cases", **out)


if __name__ == "__main__":
    sys.path.insert(0, "/root/reference/pkg/tests")
    import importlib

    sys.modules["helpers_ref"] = importlib.import_module("helpers")
    if len(sys.argv) > 1 and sys.argv[1] == "dlr_c2_50":
        # BASELINE config 2 itself, all 50 steps of the real reference (~35 min)
        run_c2_fifty()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "dlr_c1_20":
        # BASELINE config 1 itself, all 20 steps of the real reference
        run_c1_twenty()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "dlr_c2":
        # BASELINE config 2 itself, one step of the real reference (~1 min)
        run_checker("dlr_c2", per=40, r=16, nq=32, nsteps=1, seed=2, compact=True)
        sys.exit(0)
    gen_physics()
    gen_quadrature()
    gen_sweep()
    gen_source_iteration()
    gen_gram_schmidt()
    gen_deim()
    gen_projections()
    gen_edge_cases()
    gen_inflow()
    gen_sn()
    run_checker("dlr_small", per=2, r=4, nq=4, nsteps=4, seed=11)
    run_checker("dlr_c1", per=10, r=8, nq=16, nsteps=3, seed=1)
