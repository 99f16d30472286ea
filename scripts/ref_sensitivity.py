"""Sensitivity of the DLR step at ranks >= 32 (container only: imports the
reference read-only from /root/reference): the reference itself against the
oracle restatement, both CPU numpy, on the checkerboards used by
tests/test_gpu_dlr.py::test_wide_rank_steps_match_oracle.  Measured
(2026-10): X S W^T differs by 4.6e-10 (r=32) and 1.1e-10 (r=64) after one
step although both follow the same algorithm -- the spatial basis has
columns retaining ~1e-6 of their norm, so CGS2 round-off is amplified --
while r=16 agrees to 2e-15.  This sets the state tolerance of that test."""
import sys, numpy as np
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
from greytrt import angular, dlr_sn, driver, lowrank, mesh, physics
from paper_2601_18705_b200 import problems
from oracle import runner as R, port as P

def ref_run(spec, nsteps, nq_p, nq_a, r):
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    g = mesh.build_grid(spec.nx, spec.ny, spec.extent)
    quad = angular.build_quadrature(nq_p, nq_a)
    mass = driver.assemble_mass(g)
    comp = lowrank.spatial_monomials(mesh.dof_coordinates(g), g.extent, r + 8)
    X, _, _ = angular.gram_schmidt(Xr, lowrank.mass_inner(mass), comp)
    Wb, _, _ = angular.orthonormalize(Wr, quad)
    k = physics.PhysicsConstants(c=spec.c, a_r=spec.a_r)
    b0, _ = physics.planck(driver.cells_to_dofs(g, spec.T0), k)
    S = np.outer(X.T @ (mass @ b0), Wb.beta)
    state = lowrank.DlrState(X=X, S=S, W=Wb)
    T = spec.T0.copy(); out = []
    for s in range(nsteps):
        lin = physics.linearize(T, spec.sigma_a, spec.rho_cv, spec.dt, k)
        lin.sigma_t = lin.sigma_t + spec.sigma_s_phys
        lin.sigma_s = lin.sigma_s + spec.sigma_s_phys
        lin.q = lin.q + spec.q_ext
        state, info = dlr_sn.step_collocation(g, lin, quad, state, si_tol=1e-12, si_max_iters=400, use_dsa=False)
        T = np.maximum(physics.update_temperature(driver.dofs_to_cells(g, info.phi), lin, -np.inf), 1e-6)
        out.append((state.X.copy(), state.S.copy(), state.W.values.copy(), info.interpolation_condition))
    return out

for pb, r, npol, naz in [(6, 32, 8, 8), (4, 64, 8, 16), (8, 16, 16, 16)]:
    spec = problems.checkerboard(pb, rank=r, n_polar=npol, n_azimuthal=naz, seed=13, n_steps=3)
    rr = ref_run(spec, 3, npol, naz, r)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    ref = []
    R.run(spec, R.initial_state(spec, X, W), 3, record=lambda s, i, t: ref.append((s, i, t)))
    for k in range(3):
        s = ref[k][0]
        print(pb, r, k, "ref-vs-oracle", P.lowrank_rel_diff(rr[k][0], rr[k][1], rr[k][2], s.X, s.S, s.W), "cond", rr[k][3])
