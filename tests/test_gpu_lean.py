"""The memory-lean step for pure absorbers (engine="lean", lean.py): chunked
in-place sweeps and in-place CholQR2, the path that puts BASELINE config
5's DLR step on one GPU.  Checked against the one-call native step (same
kernels, full working set) and against the oracle, on config 5's medium
(random sigma_t on tiles, random source, sigma_s = 0) at reduced sizes."""

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


@pytest.mark.parametrize("n,r,nq,tile,chunk", [(48, 12, 6, 16, 5), (70, 20, 8, 10, 16),
                                               (64, 40, 8, 16, 7)])
def test_lean_step_matches_native_and_oracle(n, r, nq, tile, chunk):
    from oracle import port as P
    from oracle import runner as R
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state
    from paper_2601_18705_b200.lean import step_lean

    spec, Xr, Wr = _stress(n, r, nq, tile)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    dp = DeviceProblem.from_spec(spec)
    st0 = initial_state(dp, X=X, W=W)
    T = torch.as_tensor(spec.T0, device="cuda")
    lin = dp.linearized(T)
    a, ia = step_lean(dp.grid, lin, dp.quad, st0, si_tol=1e-12, si_max_iters=400,
                      check_state=True, chunk=chunk)
    b, ib = step_collocation(dp.grid, lin, dp.quad, st0, si_tol=1e-12, si_max_iters=400,
                             use_dsa=False)
    assert list(ia.angle_indices) == list(ib.angle_indices)
    assert ia.iterations == ib.iterations == 1
    assert rel_l2(ia.phi.cpu().numpy(), ib.phi.cpu().numpy()) <= 1e-13
    Xa, Sa, Wa = a.to_numpy()
    Xb, Sb, Wb = b.to_numpy()
    assert P.lowrank_rel_diff(Xa, Sa, Wa, Xb, Sb, Wb) <= 1e-13
    ref, rinfo = P.step_collocation(R.grid_of(spec), R.linearized(spec, spec.T0), R.quad_of(spec),
                                    R.initial_state(spec, X, W), si_tol=1e-12, use_dsa=False)
    assert list(ia.angle_indices) == list(rinfo.angle_indices)
    assert rel_l2(ia.phi.cpu().numpy(), rinfo.phi) <= 1e-11
    assert P.lowrank_rel_diff(Xa, Sa, Wa, ref.X, ref.S, ref.W) <= 1e-11


def test_lean_run_three_steps_matches_oracle():
    """The driver loop with engine="lean" (frozen coefficients, T update on
    the device) against the oracle's loop: 3 steps, 1e-11."""
    from oracle import port as P
    from oracle import runner as R
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec, Xr, Wr = _stress(64, 16, 8, 16)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    ref = []
    R.run(spec, R.initial_state(spec, X, W), 3, record=lambda s, i, t: ref.append((s, i, t)))
    dp = DeviceProblem.from_spec(spec)
    st = initial_state(dp, X=X, W=W)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for k, (rs, ri, rt) in enumerate(ref):
        st, lin, T, info = dp.step(st, lin, T, si_tol=1e-12, engine="lean")
        assert list(info.angle_indices) == list(ri.angle_indices), k
        assert rel_l2(info.phi.cpu().numpy(), ri.phi) <= 1e-11, k
        assert rel_l2(T.cpu().numpy(), rt) <= 1e-11, k
        Xg, Sg, Wg = st.to_numpy()
        assert P.lowrank_rel_diff(Xg, Sg, Wg, rs.X, rs.S, rs.W) <= 1e-11, k


def test_lean_rejects_scattering():
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state
    from paper_2601_18705_b200.errors import ContractViolation

    spec = problems.checkerboard(2, rank=4, n_polar=4, n_azimuthal=4, seed=3)
    dp = DeviceProblem.from_spec(spec)
    st = initial_state(dp)
    lin = dp.linearized(torch.as_tensor(spec.T0, device="cuda"))
    with pytest.raises(ContractViolation):
        step_collocation(dp.grid, lin, dp.quad, st, use_dsa=False, engine="lean")


def test_device_initial_state_is_orthonormal():
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state_device
    from paper_2601_18705_b200.transport import assemble_operators

    spec, _, _ = _stress(96, 24, 8, 16)
    dp = DeviceProblem.from_spec(spec)
    st = initial_state_device(dp)
    lin = dp.linearized(torch.as_tensor(spec.T0, device="cuda"))
    vals = st.check_values(assemble_operators(dp.grid, lin), dp.quad).cpu().numpy()
    assert vals.max() <= 1e-13
