"""GPU parity of the driver-level paths around the DLR step (SURVEY 8f-2,
8f-3): the full-SN method of the reference driver and its per-step energy
diagnostics, evaluated on the factors for the DLR method."""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_18705_b200.build import build

    build()


def _np(t):
    return t.detach().cpu().numpy()


def _check_rows(rows, g, key):
    for k, row in enumerate(rows):
        ref = g[key.format(k)]
        # (k, t, iterations, cond, discarded, e_mat, e_rad, outflow, residual)
        assert row[0] == k + 1
        got = np.array(row[5:8])
        assert np.allclose(got, ref[:3], rtol=1e-11, atol=0), (k, got, ref[:3])
        assert abs(row[8] - ref[3]) <= 1e-10, (k, row[8], ref[3])


@pytest.mark.parametrize("tag,dsa", [("plain", False), ("dsa", True)])
def test_full_sn_method_matches_reference(golden, tag, dsa):
    """driver.run_sn against the reference driver's "sn" branch: T, phi,
    SI counts and the energy rows every step, the final psi."""
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, run_sn

    g = golden("sn")
    spec = problems.checkerboard(2, rank=4, n_polar=4, n_azimuthal=4, seed=21, n_steps=3)
    dp = DeviceProblem.from_spec(spec)
    rows, recs = [], []
    psi, phi, T, iters = run_sn(dp, 3, si_tol=1e-12, si_max_iters=400, use_dsa=dsa,
                                diagnostics=rows,
                                record=lambda p, f, t, i: recs.append((_np(f).copy(),
                                                                       _np(t).copy(), i)))
    for k, (phi_k, T_k, it) in enumerate(recs):
        assert it == int(g[f"{tag}{k}_iters"]), k
        assert rel_l2(T_k, g[f"{tag}{k}_T"]) <= 1e-12
        assert rel_l2(phi_k, g[f"{tag}{k}_phi"]) <= 1e-11
    assert rel_l2(_np(psi), g[f"{tag}_psi"]) <= 1e-11
    _check_rows(rows, g, tag + "{}_diag")


@pytest.mark.parametrize("name", ["dlr_small", "dlr_c1"])
def test_dlr_energy_diagnostics_match_reference(golden, name):
    """The reference driver reconstructs X S W^T every step for e_rad and the
    outflow; run(..., diagnostics=rows) evaluates both on the factors."""
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state, run

    g = golden(name)
    per, r, nq, seed = int(g["per"]), int(g["rank"]), int(g["nq"]), int(g["seed"])
    spec = problems.checkerboard(per, rank=r, n_polar=nq, n_azimuthal=nq, seed=seed)
    dp = DeviceProblem.from_spec(spec)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    rows = []
    run(dp, initial_state(dp, X=X, W=W), int(g["nsteps"]), si_tol=1e-12, si_max_iters=400,
        diagnostics=rows)
    _check_rows(rows, g, "s{}_diag")
    for k, row in enumerate(rows):
        assert abs(row[3] - float(g[f"s{k}_cond"])) <= 1e-9 * float(g[f"s{k}_cond"])


def test_lowrank_outflow_equals_dense():
    """outflow_lowrank == outflow_dense(X S W^T) == transport.boundary_outflow."""
    from paper_2601_18705_b200 import transport
    from paper_2601_18705_b200.angular import AngularBasis, build_quadrature
    from paper_2601_18705_b200.diagnostics import outflow_dense, outflow_lowrank
    from paper_2601_18705_b200.lowrank import DlrState
    from paper_2601_18705_b200.mesh import build_grid

    rng = np.random.default_rng(5)
    grid = build_grid(13, 9, (0.0, 0.0, 2.0, 1.0))
    quad = build_quadrature(4, 8)
    r = 5
    st = DlrState(X=rng.standard_normal((grid.n_dofs, r)), S=rng.standard_normal((r, r)),
                  W=AngularBasis(values=rng.standard_normal((quad.n_angles, r))))
    psi = st.reconstruct()
    a = outflow_lowrank(grid, st, quad)
    b = outflow_dense(grid, psi, quad)
    c = transport.boundary_outflow(grid, psi, quad.omegas, quad.weights)
    assert abs(a - c) <= 1e-12 * abs(c) and abs(b - c) <= 1e-12 * abs(c)
