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
from ._device import as_device, device, empty, stream, to_numpy, zeros
from .angular import AngularBasis
from .errors import ContractViolation, InterpolationError, SolverError
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
        G = mass_gram(co, cols)
        R1, R1inv, ratio, flag = _chol(G)
        host = torch.cat([ratio, flag.to(torch.float64)]).cpu().numpy()
        rel, dec = host[:m], host[m:2 * m]
        # CholQR's R_kk is accurate to ~eps/rel^2: trust it when every column
        # keeps rel >= CHOLQR_GUARD of its norm and sits far (100x) above the
        # reference's deficiency threshold 1e-12 * max(orig, 1)
        if (host[-1] == 0 and float(rel.min(initial=np.inf)) >= CHOLQR_GUARD
                and float(dec.min(initial=np.inf)) >= 1e-10):
            X1 = rowmix(cols, R1inv)
            R2, R2inv, _, _ = _chol(mass_gram(co, X1))
            X = rowmix(X1, R2inv)
            return X, R2 @ R1, []
    elif method != "cgs2":
        raise ContractViolation(f"unknown Gram-Schmidt method {method!r}")
    return _cgs2(n, m, cols, metric=1, ops=co, comp_kind=1,
                 comp_exp=np.asarray(spatial_monomial_exponents(completion_count), np.int32),
                 coords=np.asarray([co.x0, co.y0, co.nx * co.dx, co.ny * co.dy]), strict=strict)


def _cgs2(n, m, cols, *, metric, ops=None, weights=None, comp_kind, comp_exp, coords, strict=True):
    Q = zeros(n, m)
    R = zeros(m, m)
    defi = _i32(max(m, 1))
    status = _i32(1)
    work = empty(int(_lib.load().dlrsn_cgs2_workspace_len(n)))
    ncomp = comp_exp.shape[0]
    exp_dev = as_device(comp_exp.reshape(-1), dtype=torch.int32) if ncomp else _i32(1)
    _lib.call("dlrsn_cgs2", n, m, _lib.ptr(cols), cols.stride(0), _lib.ptr(Q), m, _lib.ptr(R),
              _lib.ptr(defi), metric, _lib.ptr(weights), None if ops is None else _addr(ops),
              comp_kind, ncomp, _lib.ptr(exp_dev), _lib.ptr(as_device(coords)), _lib.ptr(work),
              _lib.ptr(status), int(bool(strict)), stream())
    flags = defi[:m].cpu().numpy()
    if int(status.item()) != 0:
        raise ContractViolation("ran out of completion vectors during orthonormalization")
    return Q, R, [int(k) for k in np.flatnonzero(flags)]


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

    def check(self, ops, quad, tol=1e-10):
        """Both factors orthonormal in their inner products (lowrank.py:68-81)."""
        gx = mass_gram(ops, self.X)
        eye = torch.eye(self.rank, dtype=torch.float64, device=device())
        w = quad.weights_device()
        gw = (self.W.values * w[:, None]).T @ self.W.values
        vals = torch.stack([(gx - eye).abs().max(), (gw - eye).abs().max()])
        if self.W.pinned:
            pin = (self.W.values[:, 0] - 1.0 / np.sqrt(FOUR_PI)).abs().max()
            vals = torch.cat([vals, pin.reshape(1)])
        host = vals.cpu().numpy()
        rx, rw = float(host[0]), float(host[1])
        if rx > tol or rw > tol:
            raise ContractViolation(f"factor orthonormality violated: spatial {rx:.2e}, angular {rw:.2e}")
        if self.W.pinned and float(host[2]) > tol:
            raise ContractViolation(f"constant column drifted by {float(host[2]):.2e}")
        return rx, rw

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

    @property
    def rank(self):
        return self.indices.size

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


def deim_select(basis_values):
    """Greedy DEIM point selection over quadrature nodes (lowrank.py:168-205);
    ties take the lowest node index."""
    W = as_device(basis_values)
    if W.ndim != 2:
        raise ContractViolation("deim_select expects an (n_angles, rank) array")
    n, r = W.shape
    if r > n:
        raise ContractViolation(f"rank {r} exceeds the {n} available nodes")
    W = W.contiguous()
    work = empty(n, r)
    idx = _i32(r)
    lhat, u = empty(r, r), empty(r, r)
    err = _i32(1)
    _lib.call("dlrsn_deim", n, r, _lib.ptr(work), _lib.ptr(W), _lib.ptr(idx), _lib.ptr(lhat),
              _lib.ptr(u), _lib.ptr(err), stream())
    host = torch.cat([err, idx]).cpu().numpy()
    if host[0] >= 0:
        raise InterpolationError("interpolation residual vanished; basis is rank deficient",
                                 column=int(host[0]))
    indices = host[1:].astype(np.int64)
    idx_dev = idx.to(torch.int64)
    return DeimSelection(indices=indices, indices_dev=idx_dev, w_hat=W[idx_dev].contiguous(),
                         lhat=lhat, u=u)


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


def _row_solve(n, r, proj_or_B, om_sel, ms, Q, weights):
    Binv = empty(n, r, r)
    st = _i32(max(n, 1))
    _lib.call("dlrsn_row_inverse", n, r, _lib.ptr(proj_or_B), _lib.ptr(om_sel), _lib.ptr(Binv),
              None, _lib.ptr(st), stream())
    L = empty(n, r)
    lbar = empty(r)
    st2 = _i32(1)
    _lib.call("dlrsn_row_combine", n, r, _lib.ptr(Binv), _lib.ptr(ms), _lib.ptr(Q),
              _lib.ptr(weights), _lib.ptr(L), _lib.ptr(lbar), _lib.ptr(st2), stream())
    flags = torch.cat([st[:n], st2]).cpu().numpy()
    bad = np.flatnonzero(flags[:n])
    if bad.size:
        raise SolverError(f"singular reduced transport operator at node {int(bad[0])}")
    if flags[n]:
        raise SolverError("singular closure-coupled reduced system")
    return L, lbar


def solve_row_system(B_all, Ms_hat, Q_all, weights):
    """Direct solve of the angle-coupled reduced rows (lowrank.py:235-259)."""
    B = as_device(B_all).contiguous()
    n, r, _ = B.shape
    return _row_solve(n, r, B, None, as_device(Ms_hat).contiguous(),
                      as_device(Q_all).reshape(n, r).contiguous(), as_device(weights))
