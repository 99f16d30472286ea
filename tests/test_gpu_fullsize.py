"""GPU checks at BASELINE.json's full sizes: config 2 against the
oracle step for step (the oracle finishes a C2 step in seconds), and
size-independent properties where the oracle cannot follow -- the global
particle balance of single-direction sweeps on the C4 (1024^2) and C5
(4096^2) media, and the orthonormality / DEIM contract of a full C4 step."""

import numpy as np
import pytest

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


def test_config2_two_steps_match_oracle():
    """Config 2 itself (280^2, r=16, 32x32 quadrature): identical DEIM picks
    and SI counts, rel-L2 <= 1e-11 on X S W^T and T after 2 steps."""
    from oracle import port as P
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state, run

    spec = problems.config2()
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    ref_state, ref_T, ref_infos = R.run(spec, R.initial_state(spec, X, W), 2, si_tol=1e-12)
    dp = DeviceProblem.from_spec(spec)
    state, T, infos = run(dp, initial_state(dp, X=X, W=W), 2, si_tol=1e-12, si_max_iters=400)
    Xg, Sg, Wg = state.to_numpy()
    assert [list(i.angle_indices) for i in infos] == [list(i.angle_indices) for i in ref_infos]
    assert [i.iterations for i in infos] == [i.iterations for i in ref_infos]
    assert P.lowrank_rel_diff(Xg, Sg, Wg, ref_state.X, ref_state.S, ref_state.W) <= 1e-11
    assert P.rel_l2(_np(T), ref_T) <= 1e-11


def _sweep_balance_case(spec, n_dirs_seed):
    from oracle import port as P
    from paper_2601_18705_b200 import transport
    from paper_2601_18705_b200.driver import DeviceProblem

    dp = DeviceProblem.from_spec(spec)
    T = torch.as_tensor(spec.T0, device="cuda")
    lin = dp.linearized(T)
    ops = transport.assemble_operators(dp.grid, lin)
    rhs = ops.source_vector(lin.q)
    if float(rhs.abs().sum()) == 0.0:  # cold medium: a seeded positive load
        g = torch.Generator(device="cuda").manual_seed(n_dirs_seed)
        rhs = torch.rand(dp.grid.n_dofs, dtype=torch.float64, device="cuda", generator=g)
    rhs_h = _np(rhs)
    sig = _np(lin.sigma_t)
    grid = P.Grid(spec.nx, spec.ny, *spec.extent)
    om = dp.quad.omegas
    rng = np.random.default_rng(n_dirs_seed)
    # one direction per quadrant plus the most grazing node of the set
    picks = [int(rng.choice(np.flatnonzero((np.sign(om[:, 0]) == sx) & (np.sign(om[:, 1]) == sy))))
             for sx in (1, -1) for sy in (1, -1)]
    picks.append(int(np.argmin(np.abs(om[:, 0]))))
    scale = float(np.abs(rhs_h).sum())
    for d in picks:
        psi = _np(transport.sweep_solve(ops, om[d], rhs))
        assert np.isfinite(psi).all()
        lhs, src = P.sweep_balance(grid, om[d], sig, rhs_h, psi)
        assert abs(lhs - src) <= 1e-11 * scale, (d, om[d], lhs, src)


def test_c4_sweep_balance_full_size():
    """Config 4's medium (1024^2 log-normal sigma): global balance of the
    GPU sweep to round-off for every quadrant and a grazing direction."""
    from paper_2601_18705_b200 import problems

    spec, fields = problems.random_medium()
    fields(np.random.default_rng(spec.seed))
    _sweep_balance_case(spec, 41)


def test_c5_sweep_balance_full_size():
    """Config 5's stress medium (4096^2, sigma_t in [0.1, 100] + 1/(c dt) on
    64^2 tiles): 16.8 M cells per sweep, balance to round-off."""
    from paper_2601_18705_b200 import problems

    spec, fields = problems.stress()
    fields(np.random.default_rng(spec.seed))
    _sweep_balance_case(spec, 51)


def test_c4_step_contract_full_size():
    """One full config-4 step (1024^2, r=64, 4096 directions): the DEIM
    picks equal the oracle's on the same W, and the new factors satisfy the
    reference's orthonormality contract (lowrank.py:68-81) checked on the
    host, independently of the device Grams."""
    from oracle import port as P
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec, fields = problems.random_medium()
    rng = np.random.default_rng(spec.seed)
    problems.draw_factors(spec, rng)
    fields(rng)
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    W_in = _np(state.W.values)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    new, lin2, T2, info = dp.step(state, lin, T, si_tol=1e-8)
    ref = P.deim_select(W_in)
    assert list(info.angle_indices) == list(ref.indices)
    assert info.iterations >= 1
    w = dp.quad.weights
    Wn = _np(new.W.values)
    assert np.abs(Wn.T @ (w[:, None] * Wn) - np.eye(spec.rank)).max() <= 1e-10
    mhat = P.q1_blocks()[0] * (dp.grid.dx * dp.grid.dy)
    G = np.zeros((spec.rank, spec.rank))
    Xn = new.X
    chunk = 1 << 18  # cells per host chunk
    for c0 in range(0, spec.n_cells, chunk):
        xc = _np(Xn[4 * c0:4 * min(spec.n_cells, c0 + chunk)]).reshape(-1, 4, spec.rank)
        G += np.einsum("cki,kl,clj->ij", xc, mhat, xc, optimize=True)
    assert np.abs(G - np.eye(spec.rank)).max() <= 1e-10
    Tn = _np(T2)
    assert np.isfinite(Tn).all() and Tn.min() >= 1e-6
