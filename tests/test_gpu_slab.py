"""The row-slab DLR step ("Option B", slab.py) on one GPU with P virtual
ranks in lock step (no kernel of one rank waits on another's): against the
unsharded memory-lean step (the same kernels on the whole grid) and the
oracle, on config 5's medium at reduced sizes -- the first step from the
seeded state takes the exact slab-CGS2 path (rank-deficient swept columns,
completion), the later ones CholQR2 with all-reduced Grams."""

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


def _stress(n, r, nq, tile, seed=5):
    from paper_2601_18705_b200 import problems

    spec, fields = problems.stress(n=n, rank=r, n_polar=nq, n_azimuthal=nq, tile=tile, seed=seed)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    fields(rng)
    return spec, Xr, Wr


@pytest.mark.parametrize("n,r,nq,tile,P", [(48, 12, 6, 16, 2), (64, 20, 8, 16, 3),
                                           (70, 24, 12, 10, 4)])
def test_slab_steps_match_unsharded_and_oracle(n, r, nq, tile, P):
    from oracle import port as P_
    from oracle import runner as R
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state
    from paper_2601_18705_b200.slab import run_slabs_local

    spec, Xr, Wr = _stress(n, r, nq, tile)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    ref = []
    R.run(spec, R.initial_state(spec, X, W), 3, record=lambda s, i, t: ref.append((s, i, t)))
    dp = DeviceProblem.from_spec(spec)
    st = initial_state(dp, X=X, W=W)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for k, (rs, ri, rt) in enumerate(ref):
        st, infos, _ = run_slabs_local(P, dp.grid, dp.quad, lin, st)
        info = infos[0]
        assert all(list(i["angle_indices"]) == list(ri.angle_indices) for i in info), k
        assert all(i["spatial_deficiency"] == ri.spatial_deficiency for i in info), k
        phi = torch.cat([i["phi"] for i in info])
        assert rel_l2(phi.cpu().numpy(), ri.phi) <= 1e-11, k
        T = T.clone()
        lin = dp.advance(lin, phi, T)
        assert rel_l2(T.cpu().numpy(), rt) <= 1e-11, k
        Xg, Sg, Wg = st.to_numpy()
        assert P_.lowrank_rel_diff(Xg, Sg, Wg, rs.X, rs.S, rs.W) <= 1e-11, k
    assert any(i["gs_fallback"] for i in infos[0]) or k > 0


def test_slab_projections_sum_to_whole_grid():
    """dlrsn_project_slab over row slabs (halo = the row below, top wall
    only on the last slab) sums to dlrsn_project on the whole grid."""
    from paper_2601_18705_b200 import _lib
    from paper_2601_18705_b200._device import empty, stream
    from paper_2601_18705_b200.dlr_sn import project_operators
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.physics import LinearizedStep
    from paper_2601_18705_b200.slab import Slab, _slab_step_fields, slab_rows
    from paper_2601_18705_b200.transport import assemble_operators

    for nx, ny, r, P in [(13, 11, 8, 3), (20, 17, 40, 4), (9, 40, 64, 2)]:
        rng = np.random.default_rng(nx * ny + r)
        n = nx * ny
        sig = np.exp(rng.uniform(-1, 3, n))
        grid = build_grid(nx, ny, (0.0, 0.0, 1.3, 0.7))
        step = LinearizedStep(sigma_t=sig, sigma_s=0.4 * sig, sigma_a=sig - 0.3,
                              q=rng.uniform(0, 1, n), T0=np.zeros(n), denom=np.ones(n),
                              rho_cv=np.ones(n), dt=1.0, inv_cdt=0.3)
        X = torch.randn(4 * n, r, dtype=torch.float64, device="cuda")
        Xo = torch.randn(4 * n, r, dtype=torch.float64, device="cuda")
        whole, _ = project_operators(assemble_operators(grid, step), X, x_old=Xo)
        rows = slab_rows(ny, P)
        total = torch.zeros(7 * r * r + r, dtype=torch.float64, device="cuda")
        for p in range(P):
            sl = Slab(p, P, grid, rows)
            sops = assemble_operators(sl.sgrid, _slab_step_fields(step, sl), validate=False)
            out = empty(7 * r * r + r)
            part = empty(max(int(_lib.load().dlrsn_partials_len(sl.sgrid.n_cells, r, r, 1)), 1))
            halo = X[sl.d0 - 4 * nx:sl.d0].contiguous() if p > 0 else None
            _lib.call("dlrsn_project_slab", sops.cellops_ptr, r,
                      _lib.ptr(X[sl.d0:sl.d1].contiguous()), _lib.ptr(Xo[sl.d0:sl.d1].contiguous()),
                      _lib.ptr(halo), 1 if p == P - 1 else 0, _lib.ptr(sops.step.sigma_t),
                      _lib.ptr(sops.step.sigma_s), _lib.ptr(sops.step.q), _lib.ptr(out),
                      _lib.ptr(part), stream())
            total += out
        for i, k in enumerate(("px", "py", "jx", "jy", "mt", "ms", "mo")):
            a = total[i * r * r:(i + 1) * r * r].cpu().numpy()
            assert rel_l2(a, whole[k].cpu().numpy().ravel()) <= 1e-13, (nx, r, k)
        assert rel_l2(total[7 * r * r:].cpu().numpy(), whole["q"].cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("n,r,nq,P", [(40, 16, 8, 2), (48, 24, 12, 3)])
def test_slab_steps_with_scattering_match_oracle(n, r, nq, P):
    """Config 4's medium (sigma_s = 0.5 sigma_a: source iteration with the
    closure flux all-reduced every iteration) at reduced size: identical
    picks and iteration counts, 1e-11 on phi, T and X S W^T."""
    from oracle import port as P_
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state
    from paper_2601_18705_b200.slab import run_slabs_local

    spec, fields = problems.random_medium(n=n, rank=r, n_polar=nq, n_azimuthal=nq, seed=4)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    fields(rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    ref = []
    R.run(spec, R.initial_state(spec, X, W), 2, record=lambda s, i, t: ref.append((s, i, t)))
    dp = DeviceProblem.from_spec(spec)
    st = initial_state(dp, X=X, W=W)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for k, (rs, ri, rt) in enumerate(ref):
        st, infos, _ = run_slabs_local(P, dp.grid, dp.quad, lin, st, si_tol=1e-12,
                                       si_max_iters=400)
        info = infos[0]
        assert all(list(i["angle_indices"]) == list(ri.angle_indices) for i in info), k
        assert all(i["iterations"] == ri.iterations for i in info), k
        phi = torch.cat([i["phi"] for i in info])
        assert rel_l2(phi.cpu().numpy(), ri.phi) <= 1e-11, k
        T = T.clone()
        lin = dp.advance(lin, phi, T)
        assert rel_l2(T.cpu().numpy(), rt) <= 1e-11, k
        Xg, Sg, Wg = st.to_numpy()
        assert P_.lowrank_rel_diff(Xg, Sg, Wg, rs.X, rs.S, rs.W) <= 1e-11, k
