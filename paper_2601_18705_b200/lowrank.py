"""Low-rank state and the rank-manipulation kernels of the DLR-SN step
(mirror of lowrank.py:43-259 and the spatial Gram-Schmidt of
angular.py:104-160 as used by dlr_sn.py:124-125).

Factors live on the device (fp64 torch tensors); the arithmetic is in
``libdlrsn.so`` (csrc/dense.cu).  Names, arguments, return values and
exceptions follow the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from ._device import as_device, cached_upload, device, empty, stream, to_numpy, zeros
from .angular import AngularBasis
from .errors import ContractViolation, InterpolationError, InterpolationTieError, SolverError
from .mesh import cellops_struct

FOUR_PI = 4.0 * np.pi
# CholQR2 is used when every column keeps at least this fraction of its M-norm
# after projection (first-pass Cholesky); otherwise the exact CGS2 path with
# the reference's deficiency rule (1e-12, angular.py:137) decides.
CHOLQR_GUARD = 1e-6


def _i32(n):
    return zeros(n, dtype=torch.int32)


def _cellops_of(obj):
    """cellops struct from DiscreteOperators / Grid / cellops."""
    if isinstance(obj, _lib.CellOps):
        return obj
    if hasattr(obj, "cellops"):
        return obj.cellops
    return cellops_struct(obj)


def _addr(s):
    return ctypes.c_void_p(ctypes.addressof(s))


def mass_gram(ops, A, B=None, coeff=None):
    """sum_c coeff_c A_c^T M B_c (lowrank.py:23-25 for every column pair)."""
    co = _cellops_of(ops)
    A = as_device(A)
    B = A if B is None else as_device(B)
    ra, rb = A.shape[1], B.shape[1]
    nc = co.nx * co.ny
    part = empty(max(int(_lib.load().dlrsn_partials_len(nc, ra, rb, 0)), 1))
    G = empty(ra, rb)
    _lib.call("dlrsn_mgram", _addr(co), ra, rb, _lib.ptr(A), A.stride(0), _lib.ptr(B), B.stride(0),
              _lib.ptr(None if coeff is None else as_device(coeff)), _lib.ptr(G), _lib.ptr(part),
              stream())
    return G


def rowmix(X, K, out=None, beta=0.0):
    """out = X K (+ beta out) for tall X and small K."""
    X = as_device(X)
    K = as_device(K).contiguous()
    n, kx = X.shape
    ky = K.shape[1]
    if out is None:
        out = empty(n, ky)
    _lib.call("dlrsn_rowmix", n, kx, ky, _lib.ptr(X), X.stride(0), _lib.ptr(K), K.stride(0),
              float(beta), _lib.ptr(out), out.stride(0), stream())
    return out


def rowmix_upper(X, K, out=None):
    """out = X K for an upper-triangular square K (the CholQR2 factor R^-1:
    its zero blocks are skipped); out may be X itself (in place)."""
    X = as_device(X)
    K = as_device(K).contiguous()
    n, r = X.shape
    if out is None:
        out = empty(n, r)
    _lib.call("dlrsn_rowmix_upper", n, r, _lib.ptr(X), X.stride(0), _lib.ptr(K), K.stride(0),
              _lib.ptr(out), out.stride(0), stream())
    return out


def mass_inner(ops):
    """Inner product <u, v> = u^T M v on the device (lowrank.py:23-25)."""
    return lambda u, v: float(mass_gram(ops, as_device(u).reshape(-1, 1),
                                        as_device(v).reshape(-1, 1))[0, 0])


def spatial_monomials(coords, extent, count):
    """Scaled monomials x^a y^b of rising degree (lowrank.py:28-40), host."""
    x0, y0, lx, ly = extent
    xh = 2.0 * (coords[:, 0] - x0) / lx - 1.0
    yh = 2.0 * (coords[:, 1] - y0) / ly - 1.0
    return [xh**a * yh**b for a, b in spatial_monomial_exponents(count)]


def spatial_monomial_exponents(count):
    out = []
    deg = 0
    while len(out) < count:
        for a in range(deg, -1, -1):
            out.append((a, deg - a))
        deg += 1
    return out[:count]


def _chol(G):
    r = G.shape[0]
    R, Rinv, ratio = empty(r, r), empty(r, r), empty(2 * r)
    flag = _i32(1)
    _lib.call("dlrsn_chol_upper", r, _lib.ptr(G), _lib.ptr(R), _lib.ptr(Rinv), _lib.ptr(ratio),
              _lib.ptr(flag), stream())
    return R, Rinv, ratio, flag


def gram_schmidt_mass(ops, columns, completion_count=None, strict=True, method="cholqr2"):
    """M-orthonormal basis of ``columns`` (n_dofs, m): (Q, R, deficient).

    Same contract as ``angular.gram_schmidt(cols, mass_inner(M),
    spatial_monomials(...))`` (angular.py:104-160): columns = Q R with R
    upper triangular and positive diagonal, deficient columns (norm drop
    below 1e-12 relative, absolute for norms < 1) get R_kk = 0 and a
    completion monomial.  ``method="cholqr2"`` runs two Cholesky-QR passes
    when no column comes near that threshold (first-pass R_kk ratio >=
    CHOLQR_GUARD); otherwise, or with ``method="cgs2"``, the exact CGS2 kernel.
    """
    co = _cellops_of(ops)
    cols = as_device(columns)
    n, m = cols.shape
    if completion_count is None:
        completion_count = m + 8
    if method == "cholqr2":
        X, R, guard = cholqr2_speculative(co, cols)
        if cholqr_guard_ok(guard.cpu().numpy(), m):
            return X, R, []
    elif method != "cgs2":
        raise ContractViolation(f"unknown Gram-Schmidt method {method!r}")
    Q, R, defi, status = cgs2_spatial_async(co, cols, completion_count, strict)
    return Q, R, _cgs2_flags(defi.cpu().numpy(), status.cpu().numpy(), m)


def cholqr2_speculative(co, cols):
    """Two Cholesky-QR passes in the M inner product without a host sync;
    returns (X, R, guard) with guard = first-pass diag ratios (2m) + the
    non-positive-pivot flag, to be checked with cholqr_guard_ok."""
    G = mass_gram(co, cols)
    R1, R1inv, ratio, flag = _chol(G)
    X1 = rowmix(cols, R1inv)
    R2, R2inv, _, _ = _chol(mass_gram(co, X1))
    X = rowmix(X1, R2inv)
    return X, R2 @ R1, torch.cat([ratio, flag.to(torch.float64)])


def cholqr_guard_ok(host_guard, m):
    """CholQR's R_kk is accurate to ~eps/rel^2: trust it when every column
    keeps rel >= CHOLQR_GUARD of its norm and sits far (100x) above the
    reference's deficiency threshold 1e-12 * max(orig, 1) (angular.py:137)."""
    rel, dec = host_guard[:m], host_guard[m:2 * m]
    return (host_guard[-1] == 0 and float(rel.min(initial=np.inf)) >= CHOLQR_GUARD
            and float(dec.min(initial=np.inf)) >= 1e-10)


def cgs2_spatial_async(co, cols, completion_count, strict=True, out=None):
    """``out`` may be ``cols`` itself: column k is read before Q[:, k] is
    written and only Q[:, :k] is read at step k, so the kernel runs in place."""
    n, m = cols.shape
    return _cgs2_async(n, m, cols, metric=1, ops=co, comp_kind=1,
                       comp_exp=np.asarray(spatial_monomial_exponents(completion_count), np.int32),
                       coords=np.asarray([co.x0, co.y0, co.nx * co.dx, co.ny * co.dy]),
                       strict=strict, out=out)


def _cgs2_flags(defi, status, m):
    if int(status[0]) != 0:
        raise ContractViolation("ran out of completion vectors during orthonormalization")
    return [int(k) for k in np.flatnonzero(defi[:m])]


def _cgs2_async(n, m, cols, *, metric, ops=None, weights=None, comp_kind, comp_exp, coords,
                strict=True, out=None):
    """Exact CGS2 kernel without a host sync: (Q, R, deficient flags, status)."""
    Q = zeros(n, m) if out is None else out
    R = zeros(m, m)
    defi = _i32(max(m, 1))
    status = _i32(1)
    work = empty(int(_lib.load().dlrsn_cgs2_workspace_len(n)))
    ncomp = comp_exp.shape[0]
    exp_dev = (cached_upload(("exp", comp_exp.shape, comp_exp.tobytes()),
                             lambda: comp_exp.reshape(-1).astype(np.int32)) if ncomp else _i32(1))
    if not isinstance(coords, torch.Tensor):
        c = np.asarray(coords, dtype=np.float64)
        coords = cached_upload(("coords", c.shape, c.tobytes()), lambda: c)
    _lib.call("dlrsn_cgs2", n, m, _lib.ptr(cols), cols.stride(0), _lib.ptr(Q), Q.stride(0), _lib.ptr(R),
              _lib.ptr(defi), metric, _lib.ptr(weights), None if ops is None else _addr(ops),
              comp_kind, ncomp, _lib.ptr(exp_dev), _lib.ptr(coords), _lib.ptr(work),
              _lib.ptr(status), int(bool(strict)), stream())
    return Q, R, defi, status


def _cgs2(n, m, cols, **kw):
    Q, R, defi, status = _cgs2_async(n, m, cols, **kw)
    return Q, R, _cgs2_flags(defi.cpu().numpy(), status.cpu().numpy(), m)


@dataclass(eq=False)
class DlrState:
    """Rank-r factored intensity X S W^T (lowrank.py:43-81); device tensors."""

    X: torch.Tensor
    S: torch.Tensor
    W: AngularBasis

    def __post_init__(self):
        self.X = as_device(self.X)
        self.S = as_device(self.S)
        if not isinstance(self.W, AngularBasis):
            self.W = AngularBasis(values=self.W)

    @property
    def rank(self):
        return self.S.shape[0]

    def reconstruct(self, angle_indices=None):
        w = self.W.values if angle_indices is None else self.W.values[torch.as_tensor(angle_indices, device=device())]
        return rowmix(self.X, self.S @ w.T)

    def scalar_flux(self):
        return rowmix(self.X, (self.S @ self.W.beta).reshape(-1, 1))[:, 0]

    def angular_coefficients(self):
        return self.W.values @ self.S.T

    def check_values(self, ops, quad):
        """Device tensor [max|X^T M X - I|, max|W^T D W - I|(, pin drift)]."""
        gx = mass_gram(ops, self.X)
        eye = torch.eye(self.rank, dtype=torch.float64, device=device())
        w = quad.weights_device()
        gw = (self.W.values * w[:, None]).T @ self.W.values
        vals = [(gx - eye).abs().max(), (gw - eye).abs().max()]
        if self.W.pinned:
            vals.append((self.W.values[:, 0] - 1.0 / np.sqrt(FOUR_PI)).abs().max())
        return torch.stack(vals)

    def raise_check(self, host_vals, tol=1e-10):
        rx, rw = float(host_vals[0]), float(host_vals[1])
        if rx > tol or rw > tol:
            raise ContractViolation(f"factor orthonormality violated: spatial {rx:.2e}, angular {rw:.2e}")
        if self.W.pinned and float(host_vals[2]) > tol:
            raise ContractViolation(f"constant column drifted by {float(host_vals[2]):.2e}")
        return rx, rw

    def check(self, ops, quad, tol=1e-10):
        """Both factors orthonormal in their inner products (lowrank.py:68-81)."""
        return self.raise_check(self.check_values(ops, quad).cpu().numpy(), tol)

    def to_numpy(self):
        return to_numpy(self.X), to_numpy(self.S), to_numpy(self.W.values)


@dataclass(eq=False)
class DeimSelection:
    """Greedy interpolation points (lowrank.py:145-165): W_hat = W[idx] =
    Lhat U with Lhat unit lower triangular (pick order)."""

    indices: np.ndarray
    indices_dev: torch.Tensor
    w_hat: torch.Tensor
    lhat: torch.Tensor
    u: torch.Tensor
    gap_dev: torch.Tensor | None = None  # per pick relative top-2 residual gap (device)
    gaps: np.ndarray | None = None       # the same on the host, after deim_finish

    @property
    def rank(self):
        return self.indices_dev.numel()

    @cached_property
    def cond(self):
        """2-norm condition number of W_hat (np.linalg.cond, lowrank.py:204)."""
        return float(torch.linalg.cond(self.w_hat))

    def interpolation_coefficients(self, values):
        V = as_device(values)
        flat = V.ndim == 1
        V = V.reshape(self.rank, -1).contiguous()
        X = empty(*V.shape)
        _lib.call("dlrsn_what_solve", self.rank, V.shape[1], _lib.ptr(self.lhat), _lib.ptr(self.u),
                  _lib.ptr(V), _lib.ptr(X), 0, stream())
        return X[:, 0] if flat else X

    def closure_weights(self, beta):
        v = as_device(beta).reshape(self.rank, 1).contiguous()
        x = empty(self.rank, 1)
        _lib.call("dlrsn_what_solve", self.rank, 1, _lib.ptr(self.lhat), _lib.ptr(self.u),
                  _lib.ptr(v), _lib.ptr(x), 1, stream())
        return x[:, 0]


DEIM_VARIANTS = {"auto": 0, "register": 1, "cluster": 2, "block": 3, "grid": 4}


def deim_select(basis_values, *, variant="auto", tie_tol=0.0):
    """Greedy DEIM point selection over quadrature nodes (lowrank.py:168-205);
    ties take the lowest node index.  ``selection.gaps`` holds each pick's
    relative top-2 residual gap; ``tie_tol`` > 0 raises InterpolationTieError
    for a pick closer to a tie than that (an extension: the reference breaks
    every tie silently).  ``variant`` pins the kernel (tests)."""
    W = as_device(basis_values)
    if W.ndim != 2:
        raise ContractViolation("deim_select expects an (n_angles, rank) array")
    n, r = W.shape
    if r > n:
        raise ContractViolation(f"rank {r} exceeds the {n} available nodes")
    sel, err_idx = deim_launch(W, variant=variant)
    host = torch.cat([err_idx.to(torch.float64), sel.gap_dev]).cpu().numpy()
    sel = deim_finish(sel, host[:r + 1].astype(np.int64), host[r + 1:])
    check_ties(sel.gaps, tie_tol)
    return sel


def deim_launch(W, variant="auto"):
    """Launch DEIM without a host sync: (selection with device-side factors
    and top-2 gaps, int32 [err_col, idx...]) -- see deim_finish."""
    W = as_device(W).contiguous()
    n, r = W.shape
    work = empty(n, r)
    err_idx = _i32(r + 1)
    lhat, u = empty(r, r), empty(r, r)
    gap = empty(r)
    _lib.call("dlrsn_deim", n, r, _lib.ptr(work), _lib.ptr(W), _lib.ptr(err_idx[1:]),
              _lib.ptr(lhat), _lib.ptr(u), _lib.ptr(err_idx[:1]), _lib.ptr(gap),
              DEIM_VARIANTS[variant], stream())
    idx_dev = err_idx[1:].to(torch.int64)
    sel = DeimSelection(indices=None, indices_dev=idx_dev, w_hat=W[idx_dev].contiguous(),
                        lhat=lhat, u=u, gap_dev=gap)
    return sel, err_idx


def deim_forced_launch(W, indices):
    """DEIM factors for a forced selection (``angle_indices`` of a step):
    W_hat = W[indices] = Lhat U in the given order, err_col set when a pivot
    vanishes or an index repeats / is out of range (no host sync)."""
    W = as_device(W).contiguous()
    n, r = W.shape
    idx_h = np.ascontiguousarray(indices, dtype=np.int64).reshape(-1)
    if idx_h.shape != (r,):
        raise ContractViolation(f"angle_indices must hold {r} node indices")
    err_idx = _i32(r + 1)
    lhat, u = empty(r, r), empty(r, r)
    gap = empty(r)
    _lib.call("dlrsn_deim_forced", n, r, _lib.ptr(W), idx_h.ctypes.data, _lib.ptr(err_idx[1:]),
              _lib.ptr(lhat), _lib.ptr(u), _lib.ptr(err_idx[:1]), _lib.ptr(gap), stream())
    idx_dev = err_idx[1:].to(torch.int64)
    sel = DeimSelection(indices=None, indices_dev=idx_dev, w_hat=W[idx_dev].contiguous(),
                        lhat=lhat, u=u, gap_dev=gap)
    return sel, err_idx


def deim_finish(sel, host_err_idx, host_gaps=None):
    """Raise InterpolationError (lowrank.py:192-199) or attach host indices."""
    if host_err_idx[0] >= 0:
        raise InterpolationError("interpolation residual vanished; basis is rank deficient",
                                 column=int(host_err_idx[0]))
    sel.indices = np.asarray(host_err_idx[1:], dtype=np.int64)
    if host_gaps is not None:
        sel.gaps = np.asarray(host_gaps, dtype=float)
    return sel


def check_ties(gaps, tie_tol):
    """InterpolationTieError for the first pick whose relative top-2 gap is
    positive but below ``tie_tol`` (hazard (i) of SURVEY 8c: a near-tie is
    decided by round-off, so a GPU and a CPU run may pick different nodes).
    An exact tie (gap 0: bitwise-equal maxima, e.g. the constant completion
    column of a deficient angular basis) follows the reference's stated rule,
    the lowest node index (lowrank.py:176, np.argmax), as the kernels do."""
    if tie_tol and gaps is not None:
        g = np.asarray(gaps)
        bad = np.flatnonzero((g > 0.0) & (g < tie_tol))
        if bad.size:
            j = int(bad[0])
            raise InterpolationTieError("near-tie DEIM pick; pass angle_indices= to force the "
                                        "selection", column=j, gap=float(gaps[j]))


@dataclass(eq=False)
class CollocationFlux:
    values: torch.Tensor  # (n_dofs, r)
    selection: DeimSelection
    beta: torch.Tensor

    def scalar_flux(self):
        return rowmix(self.values, self.selection.closure_weights(self.beta).reshape(-1, 1))[:, 0]


def evaluate_rows(state, selection):
    """Psi at the selected angles, X (S W_sel^T) (lowrank.py:220-227)."""
    w_sel = state.W.values[selection.indices_dev]
    return CollocationFlux(values=rowmix(state.X, state.S @ w_sel.T), selection=selection,
                           beta=state.W.beta.clone())


def reconstruct_scalar_flux(flux):
    return flux.scalar_flux()


def _row_solve_async(n, r, proj_or_B, om_sel, ms, Q, weights):
    """Row solve without host sync: returns (L, lbar, status) with status
    (n + 1 ints) = per-node singular flags, then the coupled-system flag."""
    Binv = empty(n, r, r)
    status = _i32(n + 1)
    _lib.call("dlrsn_row_inverse", n, r, _lib.ptr(proj_or_B), _lib.ptr(om_sel), _lib.ptr(Binv),
              None, _lib.ptr(status), stream())
    L = empty(n, r)
    lbar = empty(r)
    _lib.call("dlrsn_row_combine", n, r, _lib.ptr(Binv), _lib.ptr(ms), _lib.ptr(Q),
              _lib.ptr(weights), _lib.ptr(L), _lib.ptr(lbar), _lib.ptr(status[n:]), stream())
    return L, lbar, status


def raise_row_status(flags, n):
    """SolverError naming the first singular node (lowrank.py:246-252)."""
    bad = np.flatnonzero(np.asarray(flags)[:n])
    if bad.size:
        raise SolverError(f"singular reduced transport operator at node {int(bad[0])}")
    if np.asarray(flags)[n]:
        raise SolverError("singular closure-coupled reduced system")


def _row_solve(n, r, proj_or_B, om_sel, ms, Q, weights):
    L, lbar, status = _row_solve_async(n, r, proj_or_B, om_sel, ms, Q, weights)
    raise_row_status(status.cpu().numpy(), n)
    return L, lbar


def solve_row_system(B_all, Ms_hat, Q_all, weights):
    """Direct solve of the angle-coupled reduced rows (lowrank.py:235-259)."""
    B = as_device(B_all).contiguous()
    n, r, _ = B.shape
    return _row_solve(n, r, B, None, as_device(Ms_hat).contiguous(),
                      as_device(Q_all).reshape(n, r).contiguous(), as_device(weights))
