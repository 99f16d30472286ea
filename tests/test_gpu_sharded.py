"""The direction-sharded GPU code path on one GPU: two host threads act as
two ranks whose collectives go through shared memory (the kernels never
wait on each other; ranks only meet on the host), and the sharded source
iteration / DLR step must reproduce the unsharded one."""

import threading

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


class ThreadComm:
    """DirectionComm look-alike for ranks living in threads of one process."""

    def __init__(self, rank, world_size, shared):
        self.rank, self.world_size, self.shared = rank, world_size, shared

    def _exchange(self, t):
        sh = self.shared
        torch.cuda.synchronize()
        sh["slots"][self.rank] = t.clone()
        sh["barrier"].wait()
        out = [sh["slots"][p] for p in range(self.world_size)]
        sh["barrier"].wait()
        return out

    def allreduce_sum_(self, t):
        parts = self._exchange(t)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        t.copy_(acc)
        return t

    def allgather_columns(self, local, owners, n_total):
        parts = self._exchange(local)
        full = torch.empty(local.shape[0], n_total, dtype=local.dtype, device=local.device)
        for p, slots in enumerate(owners):
            if len(slots):
                full[:, torch.as_tensor(slots, device=local.device)] = parts[p]
        return full


def _run_ranks(fn, ws=2):
    shared = {"slots": [None] * ws, "barrier": threading.Barrier(ws)}
    results, errors = [None] * ws, []

    def body(rank):
        try:
            results[rank] = fn(ThreadComm(rank, ws, shared))
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(ws)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errors:
        raise errors[0]
    return results


def test_sharded_source_iteration_matches_unsharded():
    from paper_2601_18705_b200 import transport as Tr
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.physics import LinearizedStep

    rng = np.random.default_rng(3)
    nx, ny = 40, 70
    n = nx * ny
    sig = rng.uniform(0.5, 40.0, n)
    step = dict(sigma_t=sig, sigma_s=0.6 * sig, sigma_a=sig, q=rng.uniform(0, 1, n), T0=np.zeros(n),
                denom=np.ones(n), rho_cv=np.ones(n), dt=1.0, inv_cdt=0.4)
    grid = build_grid(nx, ny)
    quad = build_quadrature(4, 6)
    sel = [0, 1, 4, 7, 9, 12, 13, 17, 20, 22, 23]
    om, clo = quad.omegas[sel], quad.weights[sel]
    pt = rng.standard_normal((grid.n_dofs, len(sel)))
    ref = Tr.source_iteration(Tr.assemble_operators(grid, LinearizedStep(**step)), om, clo,
                              psi_time=pt, use_dsa=False, tol=1e-12)

    def rank_fn(comm):
        ops = Tr.assemble_operators(grid, LinearizedStep(**step))
        r = Tr.source_iteration(ops, om, clo, psi_time=pt, use_dsa=False, tol=1e-12, comm=comm)
        return r.iterations, r.psi.cpu().numpy(), r.phi.cpu().numpy()

    out = _run_ranks(rank_fn)
    rp = ref.psi.cpu().numpy()
    for it, psi, phi in out:
        assert it == ref.iterations
        assert np.linalg.norm(psi - rp) <= 1e-13 * np.linalg.norm(rp)
        assert np.linalg.norm(phi - ref.phi.cpu().numpy()) <= 1e-13 * np.linalg.norm(phi)
    assert np.array_equal(out[0][1], out[1][1])  # ranks hold identical results


@pytest.mark.parametrize("engine", ["native", "python"])
def test_sharded_dlr_steps_match_unsharded(engine):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.checkerboard(3, rank=6, n_polar=6, n_azimuthal=6, seed=4)

    def run(comm):
        dp = DeviceProblem.from_spec(spec)
        state = initial_state(dp)
        T = torch.as_tensor(spec.T0, device="cuda").clone()
        lin = dp.linearized(T)
        for _ in range(3):
            state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-12, use_dsa=False,
                                           comm=comm, engine=engine)
            lin = dp.advance(lin, info.phi, T)
        X, S, W = state.to_numpy()
        return X, S, W, T.cpu().numpy()

    ref = run(None)
    out = _run_ranks(run)
    from oracle.port import lowrank_rel_diff, rel_l2

    for X, S, W, T in out:
        assert lowrank_rel_diff(X, S, W, ref[0], ref[1], ref[2]) <= 1e-12
        assert rel_l2(T, ref[3]) <= 1e-12


def test_sharded_dsa_steps_match_unsharded():
    """use_dsa=True in the sharded native step: the diffusion correction runs
    replicated on every rank from the all-reduced flux.  The constant is put
    in span(W) so the reference's DSA converges."""
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.checkerboard(12, rank=6, n_polar=4, n_azimuthal=6, seed=9, blocks=3)
    spec.sigma_s_phys = np.where(spec.sigma_a > 0, 0.0, 30.0)
    Xr, Wr = problems.draw_factors(spec, np.random.default_rng(21))
    Wr[:, 0] = 1.0
    X0, W0 = R.orthonormal_factors(spec, Xr, Wr)

    def run(comm):
        dp = DeviceProblem.from_spec(spec)
        state = initial_state(dp, X=X0, W=W0)
        T = torch.as_tensor(spec.T0, device="cuda").clone()
        lin = dp.linearized(T)
        its = []
        for _ in range(2):
            state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-12,
                                           si_max_iters=400, use_dsa=True, comm=comm)
            its.append(info.iterations)
            lin = dp.advance(lin, info.phi, T)
        X, S, W = state.to_numpy()
        return X, S, W, T.cpu().numpy(), its

    ref = run(None)
    out = _run_ranks(run)
    from oracle.port import lowrank_rel_diff, rel_l2

    for X, S, W, T, its in out:
        assert its == ref[4]
        assert lowrank_rel_diff(X, S, W, ref[0], ref[1], ref[2]) <= 1e-12
        assert rel_l2(T, ref[3]) <= 1e-12
