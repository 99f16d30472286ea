"""DEIM on the GPU: every kernel variant on every size class against the
oracle's restatement of lowrank.py:168-205 (picks, W_hat = Lhat U, the
per-pick top-2 residual gap), the near-tie guard, and the forced selection
(angle_indices) of a whole step."""

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


VARIANTS = {"register": lambda n, r: n <= 1024 and r <= 16, "cluster": lambda n, r: True,
            "block": lambda n, r: True, "grid": lambda n, r: True}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("n,r", [(32, 6), (257, 9), (1024, 16), (300, 16), (4096, 64),
                                 (5000, 40), (300, 128), (16384, 128)])
def test_deim_variants_match_oracle(variant, n, r):
    from oracle import port as P
    from paper_2601_18705_b200.lowrank import deim_select

    if not VARIANTS[variant](n, r):
        pytest.skip("size outside the variant's range")
    rng = np.random.default_rng(n * 131 + r)
    W = np.linalg.qr(rng.standard_normal((n, r)))[0]
    try:
        sel = deim_select(W, variant=variant)
    except Exception as e:  # cluster / block size limits are reported, not silent
        assert "does not fit" in str(e) or "work copy" in str(e) or "needs n" in str(e), e
        pytest.skip(str(e))
    ref = P.deim_select(W)
    assert list(sel.indices) == list(np.asarray(ref.indices))
    assert rel_l2((sel.lhat @ sel.u).cpu().numpy(), W[sel.indices]) <= 1e-12
    assert np.abs(sel.gaps - P.deim_gaps(W, ref.indices)).max() <= 1e-12


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_deim_all_nan_column_fails_without_duplicate(variant):
    """No finite candidate left: InterpolationError at that column, never a
    fallback to an already-picked row (lowrank.py:192-199)."""
    from paper_2601_18705_b200.errors import InterpolationError
    from paper_2601_18705_b200.lowrank import deim_select

    rng = np.random.default_rng(3)
    W = rng.standard_normal((64, 5))
    W[:, 2] = np.nan
    with pytest.raises(InterpolationError) as err:
        deim_select(W, variant=variant)
    assert err.value.column == 2


def test_deim_ties():
    """Exact tie (|W[:, 0]| has two bitwise-equal maxima): the lower row, as
    np.argmax and the reference's docstring rule (lowrank.py:176), gap 0,
    no error.  Near tie (2 ulp apart): the gap is reported and a positive
    tie_tol raises InterpolationTieError naming the column."""
    from paper_2601_18705_b200.errors import InterpolationTieError
    from paper_2601_18705_b200.lowrank import deim_select

    rng = np.random.default_rng(4)
    W = rng.standard_normal((50, 4)) * 0.1
    W[7, 0], W[31, 0] = -2.0, 2.0
    sel = deim_select(W, tie_tol=1e-12)
    assert sel.indices[0] == 7 and sel.gaps[0] == 0.0
    W[31, 0] = np.nextafter(np.nextafter(2.0, 3.0), 3.0)
    sel = deim_select(W)
    assert sel.indices[0] == 31 and 0.0 < sel.gaps[0] < 1e-15
    with pytest.raises(InterpolationTieError) as err:
        deim_select(W, tie_tol=1e-12)
    assert err.value.column == 0 and 0.0 < err.value.gap < 1e-15


def _small_problem():
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.checkerboard(3, rank=6, n_polar=6, n_azimuthal=8, seed=17)
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    dp = DeviceProblem.from_spec(spec)
    return spec, dp, initial_state(dp, X=X, W=W)


@pytest.mark.parametrize("engine", ["native", "python"])
def test_forced_selection_equals_deim(engine):
    """angle_indices = DEIM's own picks reproduces the unforced step."""
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.lowrank import deim_select

    spec, dp, st = _small_problem()
    lin = dp.linearized(torch.as_tensor(spec.T0, device="cuda"))
    a, ia = step_collocation(dp.grid, lin, dp.quad, st, si_tol=1e-12, use_dsa=False,
                             engine=engine)
    picks = deim_select(st.W.values).indices
    b, ib = step_collocation(dp.grid, lin, dp.quad, st, si_tol=1e-12, use_dsa=False,
                             engine=engine, angle_indices=picks)
    assert list(ia.angle_indices) == list(ib.angle_indices) == list(picks)
    assert ia.iterations == ib.iterations
    assert rel_l2(ib.phi.cpu().numpy(), ia.phi.cpu().numpy()) <= 1e-13
    assert rel_l2(b.X.cpu().numpy(), a.X.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("engine", ["native", "python"])
def test_forced_selection_other_nodes_and_errors(engine):
    """A different valid node set is honoured (the closure and rows follow
    it); a repeated node raises InterpolationError at its position."""
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.errors import InterpolationError

    spec, dp, st = _small_problem()
    lin = dp.linearized(torch.as_tensor(spec.T0, device="cuda"))
    picks = [3, 11, 20, 29, 37, 44]
    _, info = step_collocation(dp.grid, lin, dp.quad, st, si_tol=1e-12, use_dsa=False,
                               engine=engine, angle_indices=picks)
    assert list(info.angle_indices) == picks
    with pytest.raises(InterpolationError) as err:
        step_collocation(dp.grid, lin, dp.quad, st, si_tol=1e-12, use_dsa=False, engine=engine,
                         angle_indices=[3, 11, 20, 11, 37, 44])
    assert err.value.column == 3
