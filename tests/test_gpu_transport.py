"""GPU parity of the K1/K4 kernels (through the C ABI) against the oracle
and the reference's golden vectors."""

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


def _manual_step(n, sigma_t, sigma_s, q, inv_cdt):
    from paper_2601_18705_b200.physics import LinearizedStep

    sigma_t = np.asarray(sigma_t, float)
    return LinearizedStep(sigma_t=sigma_t, sigma_s=np.asarray(sigma_s, float),
                          sigma_a=sigma_t - inv_cdt, q=np.asarray(q, float), T0=np.zeros(n),
                          denom=np.ones(n), rho_cv=np.ones(n), dt=1.0, inv_cdt=float(inv_cdt))


def _grid(arr):
    from paper_2601_18705_b200.mesh import build_grid

    nx, ny, x0, y0, lx, ly = arr
    return build_grid(int(nx), int(ny), (x0, y0, lx, ly))


def test_physics_kernels_match_reference(golden):
    from paper_2601_18705_b200 import physics as Ph

    g = golden("physics")
    for tag in ("default", "unit"):
        k = Ph.PhysicsConstants(c=float(g[f"{tag}_c"]), a_r=float(g[f"{tag}_a_r"]))
        st = Ph.linearize(g["T"], g["sigma_a"], g["rho_cv"], float(g["dt"]), k)
        for f in ("sigma_t", "sigma_s", "q", "denom"):
            assert rel_l2(_np(getattr(st, f)), g[f"{tag}_{f}"]) <= 1e-15, f
        T = Ph.update_temperature(g[f"{tag}_phi"], st)
        assert rel_l2(_np(T), g[f"{tag}_Tnew"]) <= 1e-15


def test_physics_contract_violations():
    from paper_2601_18705_b200 import physics as Ph
    from paper_2601_18705_b200.errors import ContractViolation

    with pytest.raises(ContractViolation):
        Ph.linearize(np.ones(3), -np.ones(3), np.ones(3), 0.1)
    with pytest.raises(ContractViolation):
        Ph.linearize(-np.ones(3), np.ones(3), np.ones(3), 0.1)
    with pytest.raises(ContractViolation):
        Ph.linearize(np.ones(3), np.ones(3), np.ones(3), 0.0)


@pytest.mark.parametrize("tag", ["a", "b"])
def test_sweep_solve_matches_reference(golden, tag):
    from paper_2601_18705_b200 import transport as Tr

    g = golden("sweep")
    grid = _grid(g[f"{tag}_grid"])
    n = grid.n_cells
    sig = g[f"{tag}_sigma_t"]
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, 0 * sig, np.zeros(n), 0.5))
    om, rhs, ref = g[f"{tag}_omegas"], g[f"{tag}_rhs"], g[f"{tag}_psi"]
    for d in range(om.shape[0]):
        psi = _np(Tr.sweep_solve(ops, om[d], rhs[:, d]))
        assert rel_l2(psi, ref[:, d]) <= 1e-13, d


def test_source_iteration_matches_reference(golden):
    from paper_2601_18705_b200 import transport as Tr

    g = golden("source_iteration")
    grid = _grid(g["grid"])
    n = grid.n_cells
    ops = Tr.assemble_operators(grid, _manual_step(n, g["sigma_t"], g["sigma_s"], g["q"], float(g["inv_cdt"])))
    for dw in (1, 2, 4, 8):
        res = Tr.source_iteration(ops, g["omegas"], g["closure"], psi_time=g["psi_time"],
                                  use_dsa=False, tol=1e-12, max_iters=400, phi_start=g["phi_start"],
                                  extra_source=g["extra"], dw=dw)
        assert res.iterations == int(g["plain_iters"]), dw
        assert rel_l2(_np(res.psi), g["plain_psi"]) <= 1e-12
        assert rel_l2(_np(res.phi), g["plain_phi"]) <= 1e-12
    ops = Tr.assemble_operators(grid, _manual_step(n, g["sigma_t"], 0 * g["sigma_s"], g["q"], float(g["inv_cdt"])))
    res = Tr.source_iteration(ops, g["omegas"], g["closure"], psi_time=g["psi_time"], use_dsa=False, tol=1e-12)
    assert res.iterations == 1
    assert rel_l2(_np(res.psi), g["absorber_psi"]) <= 1e-13
    assert rel_l2(_np(res.phi), g["absorber_phi"]) <= 1e-13


def test_iteration_limit_error(golden):
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.errors import IterationLimitError
    from paper_2601_18705_b200.mesh import build_grid

    g = golden("source_iteration")
    grid = build_grid(8, 8)
    ops = Tr.assemble_operators(grid, _manual_step(64, np.full(64, 100.0), np.full(64, 99.99), np.ones(64), 0.0))
    q = build_quadrature(2, 4)
    with pytest.raises(IterationLimitError) as err:
        Tr.source_iteration(ops, q.omegas, q.weights, use_dsa=False, tol=1e-8, max_iters=10)
    assert err.value.iterations == 10
    assert abs(err.value.residual - float(g["limit_residual"])) <= 1e-9 * float(g["limit_residual"])


@pytest.mark.parametrize("nx,ny,ndir,dw", [(70, 70, 16, None), (3, 67, 9, 2), (45, 33, 24, 8),
                                            (64, 100, 40, 4), (1, 1, 4, 1), (50, 330, 32, 1),
                                            (40, 640, 32, 1), (33, 700, 30, 1)])
def test_source_iteration_matches_oracle_random(nx, ny, ndir, dw):
    """Multi-strip handoffs, partial strips, every group width, all quadrants.
    Single-direction groups above 4 x SM-count work items (strips x
    directions: 640 and 660 here) run the split-phase throughput kernel
    (sweep1s_kernel), below it the warp-specialised one (352 items)."""
    from oracle import port as P
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.mesh import build_grid

    rng = np.random.default_rng(nx * 1000 + ny)
    n = nx * ny
    sig = np.exp(rng.uniform(np.log(0.05), np.log(500.0), n))
    ss = sig * rng.uniform(0.0, 0.7, n)
    q = rng.uniform(0, 1, n)
    th = rng.uniform(0, 2 * np.pi, ndir)
    mu = rng.uniform(-0.95, 0.95, ndir)
    om = np.column_stack([np.sqrt(1 - mu**2) * np.cos(th), np.sqrt(1 - mu**2) * np.sin(th), mu])
    clo = rng.uniform(0.1, 1.0, ndir) * 4 * np.pi / ndir
    pt = rng.standard_normal((4 * n, ndir))
    grid = build_grid(nx, ny, (0.0, 0.0, 1.3, 0.9))
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, ss, q, 0.7))
    res = Tr.source_iteration(ops, om, clo, psi_time=pt, use_dsa=False, tol=1e-12, max_iters=500, dw=dw)
    pg = P.Grid(nx, ny, 0.0, 0.0, 1.3, 0.9)
    pst = P.Step(sig, ss, sig - 0.7, q, np.zeros(n), np.ones(n), np.ones(n), 1.0, 0.7)
    ref = P.source_iteration(P.assemble_operators(pg, pst), om, clo, psi_time=pt, use_dsa=False,
                             tol=1e-12, max_iters=500)
    assert res.iterations == ref.iterations
    assert rel_l2(_np(res.psi), ref.psi) <= 1e-12
    assert rel_l2(_np(res.phi), ref.phi) <= 1e-12


def test_sweep_is_deterministic():
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.mesh import build_grid

    rng = np.random.default_rng(5)
    nx, ny, D = 90, 75, 12
    n = nx * ny
    grid = build_grid(nx, ny)
    sig = rng.uniform(0.5, 30, n)
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, 0.5 * sig, rng.uniform(0, 1, n), 0.2))
    om = rng.standard_normal((D, 3))
    om /= np.linalg.norm(om, axis=1)[:, None]
    a = Tr.source_iteration(ops, om, np.full(D, 0.3), use_dsa=False, tol=1e-10)
    b = Tr.source_iteration(ops, om, np.full(D, 0.3), use_dsa=False, tol=1e-10)
    assert a.iterations == b.iterations
    assert torch.equal(a.psi, b.psi) and torch.equal(a.phi, b.phi)


# ---- isotropic inflow boundary (config 3), device kernel dlrsn_inflow_add


def test_inflow_constant_state_is_exact(golden):
    """psi_b on every wall, q = (sigma_t - sigma_s) psi_b: psi = psi_b."""
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature

    g = golden("inflow")
    grid = _grid(np.array([6, 5, 0.0, 0.0, 1.2, 1.0]))
    n = grid.n_cells
    psib = float(g["const_psib"])
    sig, ss = g["const_sigma_t"], g["const_sigma_s"]
    quad = build_quadrature(2, 6)
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, ss, (sig - ss) * psib, 0.0))
    for dw in (1, 2):
        res = Tr.source_iteration(ops, quad.omegas, quad.weights, use_dsa=False, tol=1e-14,
                                  max_iters=800, inflow=(psib,) * 4, dw=dw)
        assert res.iterations == int(g["const_iters"])
        assert np.abs(_np(res.psi) - psib).max() <= 1e-13
        assert rel_l2(_np(res.psi), g["const_psi"]) <= 1e-13


def test_inflow_source_iteration_matches_reference(golden):
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature

    g = golden("inflow")
    grid = _grid(np.array([6, 5, 0.0, 0.0, 1.2, 1.0]))
    n = grid.n_cells
    quad = build_quadrature(2, 6)
    inflow = {"left": 0.8, "top": 0.3}
    assert rel_l2(_np(Tr.inflow_source(grid, quad.omegas, inflow)), g["si_load"]) == 0.0
    ops = Tr.assemble_operators(grid, _manual_step(n, g["const_sigma_t"], g["const_sigma_s"],
                                                   g["si_q"], 0.4))
    for dw in (1, 4):
        res = Tr.source_iteration(ops, quad.omegas, quad.weights, psi_time=g["si_psi_time"],
                                  use_dsa=False, tol=1e-13, max_iters=800, inflow=inflow, dw=dw)
        assert res.iterations == int(g["si_iters"])
        assert rel_l2(_np(res.psi), g["si_psi"]) <= 1e-12
        assert rel_l2(_np(res.phi), g["si_phi"]) <= 1e-12


# ---- K6: diffusion synthetic acceleration (transport_sn.py:166-198, 325-367)


def test_dsa_source_iteration_matches_reference(golden):
    """use_dsa=True (the reference default) against the reference's own run."""
    from paper_2601_18705_b200 import transport as Tr

    g = golden("source_iteration")
    grid = _grid(g["grid"])
    n = grid.n_cells
    ops = Tr.assemble_operators(grid, _manual_step(n, g["sigma_t"], g["sigma_s"], g["q"],
                                                   float(g["inv_cdt"])))
    for dw in (1, 4):
        res = Tr.source_iteration(ops, g["omegas"], g["closure"], psi_time=g["psi_time"],
                                  use_dsa=True, tol=1e-12, max_iters=400,
                                  phi_start=g["phi_start"], extra_source=g["extra"], dw=dw)
        assert res.iterations == int(g["dsa_iters"]), dw
        assert rel_l2(_np(res.psi), g["dsa_psi"]) <= 1e-11
        assert rel_l2(_np(res.phi), g["dsa_phi"]) <= 1e-11


@pytest.mark.parametrize("nx,ny,penalty", [(40, 45, "simplified"), (7, 70, "collocation")])
def test_dsa_matches_oracle(nx, ny, penalty):
    """Full quadrature closure on multi-strip grids with thick scattering
    cells (where DSA matters): GPU vs oracle with the same DSA, both penalty
    variants; DSA must cut the iteration count."""
    from oracle import port as P
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.mesh import build_grid

    rng = np.random.default_rng(nx * 7 + ny)
    n = nx * ny
    sig = np.exp(rng.uniform(np.log(1.0), np.log(200.0), n))
    ss = sig * rng.uniform(0.8, 0.99, n)
    q = rng.uniform(0, 1, n)
    quad = build_quadrature(2, 8)
    om, w = quad.omegas, quad.weights
    grid = build_grid(nx, ny, (0.0, 0.0, 1.0, 1.1))
    pc = (om, w) if penalty == "collocation" else None
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, ss, q, 0.0), dsa_penalty=penalty,
                                penalty_closure=pc)
    res = Tr.source_iteration(ops, om, w, use_dsa=True, tol=1e-10, max_iters=500)
    plain = Tr.source_iteration(ops, om, w, use_dsa=False, tol=1e-10, max_iters=2000)
    pg = P.Grid(nx, ny, 0.0, 0.0, 1.0, 1.1)
    pst = P.Step(sig, ss, sig, q, np.zeros(n), np.ones(n), np.ones(n), 1.0, 0.0)
    pops = P.assemble_operators(pg, pst, dsa_penalty=penalty, penalty_closure=pc)
    ref = P.source_iteration(pops, om, w, use_dsa=True, tol=1e-10, max_iters=500)
    assert res.iterations == ref.iterations
    assert res.iterations < plain.iterations
    assert rel_l2(_np(res.phi), ref.phi) <= 1e-10
    assert rel_l2(_np(res.psi), ref.psi) <= 1e-10
    assert rel_l2(_np(res.phi), _np(plain.phi)) <= 1e-8  # same fixed point


def test_dsa_step_collocation_matches_reference(golden):
    """The cold-empty edge case ran through the reference with its default
    use_dsa=True (tests/test_dlr_sn.py:127-136)."""
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.lowrank import DlrState
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.physics import linearize

    g = golden("edge_cases")
    grid = build_grid(4, 4)
    quad = build_quadrature(2, 4)
    st = DlrState(X=g["cold_X"], S=g["cold_S"], W=g["cold_W"])
    st.W.bind(quad)
    n = grid.n_cells
    step = linearize(np.zeros(n), np.full(n, 2.0), np.ones(n), 0.2)
    new, info = step_collocation(grid, step, quad, st)  # use_dsa=True by default
    assert info.spatial_deficiency == int(g["cold_sdef"])
    assert list(info.angle_indices) == list(g["cold_idx"])
    assert info.iterations == int(g["cold_iters"])
    assert np.abs(_np(new.X) - g["cold_newX"]).max() <= 1e-12


@pytest.mark.parametrize("dedup", [True, False])
@pytest.mark.parametrize("nx,ny,npol,naz,dw", [(40, 70, 4, 8, 8), (33, 29, 2, 6, 2), (70, 40, 4, 8, 1)])
def test_closure_sweep_matches_oracle(nx, ny, npol, naz, dw, dedup):
    """Config 5's closure-only full-SN sweep (psi never stored, closure sums
    added with fp64 atomics): phi against the oracle's sweeps of EVERY
    direction with the shared rhs, to round-off (the atomic order varies);
    with ``dedup`` only the distinct (omega_x, omega_y) pairs are swept."""
    from oracle import port as P
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.mesh import build_grid

    rng = np.random.default_rng(nx + ny)
    n = nx * ny
    sig = np.exp(rng.uniform(np.log(0.1), np.log(100.0), n))
    q = rng.uniform(0, 1, n)
    grid = build_grid(nx, ny, (0.0, 0.0, float(nx), float(ny)))
    quad = build_quadrature(npol, naz)
    ops = Tr.assemble_operators(grid, _manual_step(n, sig, 0 * sig, q, 1.0))
    psi_old = rng.uniform(0, 1, 4 * n)  # isotropic previous intensity
    rhs = ops.source_vector(q) + 1.0 * ops.mass_apply(psi_old)
    phi = Tr.closure_sweep(ops, quad.omegas, quad.weights, rhs, dw=dw, ws_limit=1 << 13,
                           dedup=dedup)
    pg = P.Grid(nx, ny, 0.0, 0.0, float(nx), float(ny))
    pops = P.assemble_operators(pg, P.Step(sig, 0 * sig, sig - 1.0, q, np.zeros(n), np.ones(n),
                                           np.ones(n), 1.0, 1.0))
    rhs_np = pops.source_vector(q) + pops.mass_apply(psi_old)
    ref = P.sweep_many(pops, quad.omegas, np.tile(rhs_np[:, None], (1, quad.n_angles))) @ quad.weights
    assert rel_l2(_np(phi), ref) <= 1e-13
