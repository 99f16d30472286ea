"""Grey physics on the device (mirror of physics.py:37-132).

``linearize`` / ``update_temperature`` keep the reference signatures and
error behaviour; the arithmetic runs in the fused K4 kernels of
``libdlrsn.so`` (csrc/physics.cu).  Arrays may be numpy or torch; results are
fp64 CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, stream, zeros
from .errors import ContractViolation

FOUR_PI = 4.0 * np.pi
DEFAULT_T_FLOOR = 1e-6


@dataclass(frozen=True)
class PhysicsConstants:
    c: float = 299.79
    a_r: float = 0.01372


@dataclass(frozen=True)
class Material:
    sigma_a: float
    c_v: float
    rho: float

    def __post_init__(self):
        if self.sigma_a < 0 or self.c_v <= 0 or self.rho <= 0:
            raise ContractViolation(f"material needs sigma_a >= 0, c_v > 0, rho > 0; got {self}")

    @property
    def rho_cv(self):
        return self.rho * self.c_v


def planck(T, constants=PhysicsConstants()):
    """B = a c T^4 / 4 pi and dB/dT = a c T^3 / pi (physics.py:63-75)."""
    T = as_device(T)
    if bool((T < 0).any()):
        raise ContractViolation("negative temperature passed to planck()")
    scale = constants.a_r * constants.c
    T2 = T * T
    return scale / FOUR_PI * (T2 * T2), scale / np.pi * (T2 * T)


@dataclass(eq=False)
class LinearizedStep:
    """Per-cell coefficients of one linearised step (physics.py:78-91);
    every field is an fp64 CUDA tensor."""

    sigma_t: torch.Tensor
    sigma_s: torch.Tensor
    sigma_a: torch.Tensor
    q: torch.Tensor
    T0: torch.Tensor
    denom: torch.Tensor
    rho_cv: torch.Tensor
    dt: float
    inv_cdt: float
    constants: PhysicsConstants = PhysicsConstants()

    def __post_init__(self):
        for name in ("sigma_t", "sigma_s", "sigma_a", "q", "T0", "denom", "rho_cv"):
            setattr(self, name, as_device(getattr(self, name)))


def linearize(T0, sigma_a, rho_cv, dt, constants=PhysicsConstants(), *, sigma_s_phys=None,
              q_ext=None, check=True):
    """Newton linearisation about T0 (physics.py:94-120).

    ``sigma_s_phys`` / ``q_ext`` optionally add physical scattering and an
    external source the way the reference's tests inject them
    (tests/test_transport_sn.py:22-36); both default to none.
    """
    if dt <= 0:
        raise ContractViolation(f"time step must be positive, got {dt}")
    T0 = as_device(T0)
    n = T0.numel()
    sa = as_device(sigma_a, n)
    rc = as_device(rho_cv, n)
    ssp = None if sigma_s_phys is None else as_device(sigma_s_phys, n)
    qe = None if q_ext is None else as_device(q_ext, n)
    st, ss, q, den = (torch.empty(n, dtype=torch.float64, device=device()) for _ in range(4))
    status = zeros(1, dtype=torch.int32)
    _lib.call("dlrsn_linearize", n, _lib.ptr(T0), _lib.ptr(sa), _lib.ptr(rc), float(dt),
              float(constants.c), float(constants.a_r), _lib.ptr(ssp), _lib.ptr(qe), _lib.ptr(st),
              _lib.ptr(ss), _lib.ptr(q), _lib.ptr(den), _lib.ptr(status), stream())
    if check and int(status.item()) != 0:
        if bool((T0 < 0).any()):
            raise ContractViolation("negative temperature passed to planck()")
        raise ContractViolation("need sigma_a >= 0 and rho*c_v > 0 in every cell")
    return LinearizedStep(sigma_t=st, sigma_s=ss, sigma_a=sa, q=q, T0=T0, denom=den, rho_cv=rc,
                          dt=float(dt), inv_cdt=1.0 / (constants.c * dt), constants=constants)


def update_temperature(phi, step, t_floor=DEFAULT_T_FLOOR):
    """Closed-form Newton temperature update (physics.py:123-132).  ``phi``
    is per cell, or per dof (then averaged per cell, driver.py:344-346)."""
    n = step.T0.numel()
    phi = as_device(phi)
    if phi.numel() == n:
        per_dof = 0
    elif phi.numel() == 4 * n:
        per_dof = 1
    else:
        raise ContractViolation(f"phi has {phi.numel()} entries for {n} cells")
    T = torch.empty(n, dtype=torch.float64, device=device())
    k = step.constants
    _lib.call("dlrsn_update_temperature", n, _lib.ptr(phi), per_dof, _lib.ptr(step.T0),
              _lib.ptr(step.sigma_a), _lib.ptr(step.denom), float(step.dt), float(k.c),
              float(k.a_r), float(t_floor), _lib.ptr(T), stream())
    return T
