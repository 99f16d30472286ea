"""The numpy-at-the-edges drop-in (paper_2601_18705_b200.compat) under a
reference-style time loop: objects shaped like greytrt's own (Grid,
LinearizedStep, QuadratureSet, DlrState / AngularBasis holding numpy
arrays) go in, the caller's own classes with numpy arrays come out, and a
restatement of the reference driver's dlr-sn loop (driver.py:485-539:
linearize -> step_collocation -> dofs_to_cells -> update_temperature ->
floor, all numpy on the host) with the B200 step swapped in reproduces the
REAL reference's config-1 run (tests/golden/dlr_c1.npz, made from greytrt)
to 1e-11."""

from dataclasses import dataclass

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


# stand-ins with greytrt's field names (lowrank.py:43-50, angular.py:163-183,
# mesh.py:76-83, angular.py:28-34, physics.py:78-91); numpy only
@dataclass(eq=False)
class RefBasis:
    values: np.ndarray
    beta: np.ndarray | None = None
    pinned: bool = False

    def bind(self, quad):
        self.beta = self.values.T @ quad.weights
        return self


@dataclass(eq=False)
class RefState:
    X: np.ndarray
    S: np.ndarray
    W: RefBasis

    def reconstruct(self):
        return self.X @ (self.S @ self.W.values.T)


@dataclass(frozen=True, eq=False)
class RefGrid:
    nx: int
    ny: int
    x0: float
    y0: float
    dx: float
    dy: float


@dataclass(frozen=True, eq=False)
class RefQuad:
    omegas: np.ndarray
    weights: np.ndarray
    antipode: np.ndarray
    n_polar: int
    n_azimuthal: int


def _ref_objects(spec):
    from oracle import port as P

    q = P.build_quadrature(spec.n_polar, spec.n_azimuthal)
    grid = RefGrid(spec.nx, spec.ny, spec.extent[0], spec.extent[1], spec.dx, spec.dy)
    anti = np.zeros(q.n_angles, dtype=int)
    return grid, RefQuad(q.omegas, q.weights, anti, spec.n_polar, spec.n_azimuthal)


def test_compat_types_and_numpy_edges():
    from oracle import runner as R
    from paper_2601_18705_b200 import compat, problems

    spec = problems.checkerboard(3, rank=5, n_polar=4, n_azimuthal=8, seed=23)
    grid, quad = _ref_objects(spec)
    rng = np.random.default_rng(spec.seed)
    X, W = R.orthonormal_factors(spec, *problems.draw_factors(spec, rng))
    ref0 = R.initial_state(spec, X, W)
    state = RefState(X=ref0.X, S=ref0.S, W=RefBasis(values=ref0.W).bind(quad))
    lin = R.linearized(spec, spec.T0)
    new, info = compat.step_collocation(grid, lin, quad, state, si_tol=1e-12, use_dsa=False)
    assert type(new) is RefState and type(new.W) is RefBasis
    for a in (new.X, new.S, new.W.values, new.W.beta, info.phi):
        assert isinstance(a, np.ndarray) and a.dtype == np.float64
    assert state.X is ref0.X  # the input state is not mutated
    ref_state, ref_info = __import__("oracle.port", fromlist=["x"]).step_collocation(
        R.grid_of(spec), lin, R.quad_of(spec), ref0, si_tol=1e-12, use_dsa=False)
    assert list(info.angle_indices) == list(ref_info.angle_indices)
    assert info.iterations == ref_info.iterations
    assert rel_l2(info.phi, ref_info.phi) <= 1e-11
    from oracle import port as P

    assert P.lowrank_rel_diff(new.X, new.S, new.W.values, ref_state.X, ref_state.S,
                              ref_state.W) <= 1e-11
    assert abs(info.interpolation_condition - ref_info.interpolation_condition) <= \
        1e-9 * ref_info.interpolation_condition


def test_reference_loop_with_b200_step_matches_real_reference(golden):
    """driver.py:485-539's dlr-sn branch restated on numpy objects, with
    step_collocation replaced by compat.step_collocation, against greytrt's
    own config-1 run (3 steps, golden)."""
    from oracle import port as P
    from oracle import runner as R
    from paper_2601_18705_b200 import compat, problems

    g = golden("dlr_c1")
    spec = problems.checkerboard(int(g["per"]), rank=int(g["rank"]), n_polar=int(g["nq"]),
                                 n_azimuthal=int(g["nq"]), seed=int(g["seed"]))
    grid, quad = _ref_objects(spec)
    rng = np.random.default_rng(spec.seed)
    X, W = R.orthonormal_factors(spec, *problems.draw_factors(spec, rng))
    st0 = R.initial_state(spec, X, W)
    state = RefState(X=st0.X, S=st0.S, W=RefBasis(values=st0.W).bind(quad))
    T = spec.T0.copy()
    for k in range(int(g["nsteps"])):
        lin = R.linearized(spec, T)                        # linearize (+ App. B adapters)
        state, info = compat.step_collocation(grid, lin, quad, state, si_tol=1e-12,
                                              si_max_iters=400, use_dsa=False)
        raw = P.update_temperature(P.dofs_to_cells(info.phi), lin, -np.inf)
        T = np.maximum(raw, spec.t_floor)                  # driver.py:532-534
        assert list(info.angle_indices) == list(g[f"s{k}_idx"]), k
        assert info.iterations == int(g[f"s{k}_iters"]), k
        assert rel_l2(info.phi, g[f"s{k}_phi"]) <= 1e-11, k
        assert rel_l2(T, g[f"s{k}_T"]) <= 1e-11, k
        rs = np.random.default_rng(9)
        phi_t = rs.standard_normal((state.X.shape[0], 12))
        om_t = rs.standard_normal((state.W.values.shape[0], 12))
        sk = (phi_t.T @ state.X) @ state.S @ (state.W.values.T @ om_t)
        assert rel_l2(sk, g[f"s{k}_sketch"]) <= 1e-11, k
