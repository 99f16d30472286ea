"""Angular quadrature and orthonormal angular bases (mirror of angular.py).

The quadrature is input data and stays on the host (numpy, read-only arrays
as in the reference, angular.py:79-80).  Basis values live on the device;
``orthonormalize`` runs the weighted CGS2 of the reference
(angular.py:104-160,217-238) as a single-CTA CUDA kernel (csrc/dense.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._device import as_device
from .errors import ConfigurationError, ContractViolation

FOUR_PI = 4.0 * np.pi
DEFICIENCY_TOL = 1e-12


@dataclass(frozen=True, eq=False)
class QuadratureSet:
    omegas: np.ndarray
    weights: np.ndarray
    antipode: np.ndarray
    n_polar: int
    n_azimuthal: int

    @property
    def n_angles(self):
        return self.omegas.shape[0]

    def integrate(self, values):
        return np.asarray(values) @ self.weights

    def weights_device(self):
        w = getattr(self, "_wdev", None)
        if w is None:
            w = as_device(self.weights)
            object.__setattr__(self, "_wdev", w)
        return w

    def omegas_device(self):
        o = getattr(self, "_odev", None)
        if o is None:
            o = as_device(self.omegas)
            object.__setattr__(self, "_odev", o)
        return o


def build_quadrature(n_polar, n_azimuthal):
    """Gauss-Legendre polar cosines x half-offset uniform azimuths
    (angular.py:45-87); weights sum to 4 pi, closed under omega -> -omega."""
    if n_polar < 1 or n_azimuthal < 1:
        raise ConfigurationError("quadrature orders must be positive")
    if n_azimuthal % 2 != 0:
        raise ConfigurationError(f"n_azimuthal must be even for antipodal closure, got {n_azimuthal}")
    mu, wmu = np.polynomial.legendre.leggauss(n_polar)
    az = 2.0 * np.pi * (np.arange(n_azimuthal) + 0.5) / n_azimuthal
    s = np.sqrt(1.0 - mu**2)
    om = np.empty((n_polar, n_azimuthal, 3))
    om[..., 0] = s[:, None] * np.cos(az)[None, :]
    om[..., 1] = s[:, None] * np.sin(az)[None, :]
    om[..., 2] = mu[:, None]
    w = np.repeat(wmu * (2.0 * np.pi / n_azimuthal), n_azimuthal)
    p, a = np.divmod(np.arange(n_polar * n_azimuthal), n_azimuthal)
    anti = (n_polar - 1 - p) * n_azimuthal + (a + n_azimuthal // 2) % n_azimuthal
    om = om.reshape(-1, 3)
    for arr in (om, w, anti):
        arr.setflags(write=False)
    return QuadratureSet(om, w, anti, n_polar, n_azimuthal)


def inner_product(u, v, quad):
    """Weighted angular inner product (angular.py:90-101), on the device."""
    u = as_device(u)
    v = as_device(v)
    if u.shape[0] != quad.n_angles or v.shape[0] != quad.n_angles:
        raise ContractViolation(
            f"node-vector lengths {u.shape[0]}/{v.shape[0]} do not match the "
            f"{quad.n_angles}-angle quadrature")
    w = quad.weights_device()
    if u.ndim == 1 and v.ndim == 1:
        return float((w * u * v).sum())
    return (u * w[:, None]).T @ v if u.ndim > 1 else (u * w) @ v


@dataclass(eq=False)
class AngularBasis:
    """Columns orthonormal in the quadrature-weighted inner product
    (angular.py:163-191); ``values`` (n_angles, r) and ``beta`` = W^T w are
    device tensors."""

    values: torch.Tensor
    beta: torch.Tensor | None = None
    pinned: bool = False

    def __post_init__(self):
        self.values = as_device(self.values)
        if self.values.ndim != 2:
            raise ContractViolation("angular basis must be a 2D (n_angles, rank) array")
        if self.beta is not None:
            self.beta = as_device(self.beta)

    def bind(self, quad):
        self.beta = self.values.T @ quad.weights_device()
        return self

    @property
    def rank(self):
        return self.values.shape[1]

    def orthonormality_residual(self, quad):
        g = inner_product(self.values, self.values, quad)
        eye = torch.eye(self.rank, dtype=g.dtype, device=g.device)
        return float((g - eye).abs().max())


def constant_column(quad):
    return np.full(quad.n_angles, 1.0 / np.sqrt(FOUR_PI))


def angular_monomial_exponents(count):
    """(kx, ky, kz) of the first ``count`` candidates of angular_monomials."""
    out = [(0, 0, 0)]
    deg = 1
    while len(out) < count:
        for kx in range(deg, -1, -1):
            for ky in range(deg - kx, -1, -1):
                out.append((kx, ky, deg - kx - ky))
        deg += 1
    return out[:count]


def orthonormalize(columns, quad, pin_constant=False):
    """Weighted CGS2 with deterministic completion (angular.py:217-238), as
    one CUDA kernel.  Returns (AngularBasis, R, deficient)."""
    from .lowrank import _cgs2_flags

    basis, R, defi, status = orthonormalize_async(columns, quad, pin_constant)
    deficient = _cgs2_flags(defi.cpu().numpy(), status.cpu().numpy(), R.shape[0])
    if pin_constant:
        return basis, R, [d - 1 for d in deficient if d > 0]
    return basis, R, deficient


def orthonormalize_async(columns, quad, pin_constant=False):
    """orthonormalize without a host sync: (basis, R, deficient flags,
    status); R excludes the pinned constant's row... column (see above)."""
    from .lowrank import _cgs2_async

    cols = as_device(columns)
    if cols.ndim != 2 or cols.shape[0] != quad.n_angles:
        raise ContractViolation(
            f"basis rows ({cols.shape[0]}) must match quadrature size ({quad.n_angles})")
    if pin_constant:
        const = torch.full((quad.n_angles, 1), 1.0 / np.sqrt(FOUR_PI), dtype=torch.float64,
                           device=cols.device)
        cols = torch.cat([const, cols], dim=1)
    n, m = cols.shape
    ncomp = (m - (1 if pin_constant else 0)) + 8
    exps = np.asarray(angular_monomial_exponents(ncomp), dtype=np.int32)
    Q, R, defi, status = _cgs2_async(n, m, cols.contiguous(), metric=0,
                                     weights=quad.weights_device(), comp_kind=0, comp_exp=exps,
                                     coords=quad.omegas_device(), strict=True)
    basis = AngularBasis(values=Q, pinned=pin_constant).bind(quad)
    return basis, (R[:, 1:] if pin_constant else R), defi, status


def angular_monomials(quad, count):
    """Completion candidates: monomials in omega by rising degree, then unit
    vectors (angular.py:198-214).  Returned as an (n_angles, k) host array."""
    ox, oy, oz = quad.omegas.T
    cands = [np.ones_like(ox)]
    deg = 1
    while len(cands) < count:
        for kx in range(deg, -1, -1):
            for ky in range(deg - kx, -1, -1):
                cands.append(ox**kx * oy**ky * oz ** (deg - kx - ky))
        deg += 1
    return np.column_stack(cands[:count] + list(np.eye(quad.n_angles)))
