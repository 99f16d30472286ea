"""Per-step energy diagnostics of the reference driver, factored for the
low-rank state.

The reference driver (driver.py:521-553) reconstructs the dense intensity
X S W^T (n_dofs x N_Omega) every step to evaluate

  e_mat    = sum rho_cv T * cell_area
  e_rad    = integrate_dofs(psi @ w) / c
  outflow  = boundary_outflow(grid, psi, omegas, weights)  (transport_sn.py:479-492)
  residual = (e_mat + e_rad - e_mat_prev - e_rad_prev + dt * outflow - floor_source) / |total|

which blocks configs 3-5 (the dense psi of config 4 is 137 GB).  Here every
term is evaluated on the factors: psi @ w = X (S beta); the outflow is, per
wall w, h_w^T S (W^T (w * max(omega.n_w, 0))) with h_w = X^T g_w the
trapezoid weights of the wall's edge dofs (0.5 * face length each; the
kernel dlrsn_inflow_project), so nothing of size n_dofs x N_Omega exists.
Rows follow the reference's DIAGNOSTIC_COLUMNS order (k, t, iterations,
interpolation condition, discarded, e_mat, e_rad, outflow, residual).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, empty, stream
from .mesh import cellops_struct

WALL_NORMALS = ((-1.0, 0.0), (1.0, 0.0), (0.0, -1.0), (0.0, 1.0))  # left right bottom top


def integrate_dofs(grid, values):
    """driver.py:349-350: cell means of a dof field times the cell area."""
    v = as_device(values).reshape(grid.n_cells, 4)
    return float(v.mean(dim=1).sum()) * grid.dx * grid.dy


def wall_traces(grid, cols):
    """(4, k) device tensor: h[w] = cols^T g_w, g_w = 0.5 * face length on
    the two edge dofs of every face of wall w (the trapezoid rule of
    transport_sn.py:486-488), for the columns of an (n_dofs, k) array."""
    cols = as_device(cols)
    if cols.ndim == 1:
        cols = cols.reshape(-1, 1)
    cols = cols.contiguous()
    k = cols.shape[1]
    co = cellops_struct(grid)
    h = empty(4 * k)
    walls = (ctypes.c_double * 4)(1.0, 1.0, 1.0, 1.0)
    _lib.call("dlrsn_inflow_project", ctypes.c_void_p(ctypes.addressof(co)), k, _lib.ptr(cols), k,
              walls, _lib.ptr(h), stream())
    return h.reshape(4, k)


def _outflow_weights(quad):
    """(4, N_Omega): w_d * max(omega_d . n_w, 0) per wall."""
    om = torch.as_tensor(np.array(quad.omegas[:, :2], dtype=float), device=device())
    w = torch.as_tensor(np.array(quad.weights, dtype=float), device=device())
    n = torch.tensor(WALL_NORMALS, dtype=torch.float64, device=device())
    return torch.clamp(n @ om.T, min=0.0) * w[None, :]


def outflow_dense(grid, psi, quad):
    """boundary_outflow (transport_sn.py:479-492) of a dense (n_dofs,
    N_Omega) device intensity."""
    h = wall_traces(grid, psi)
    return float((h * _outflow_weights(quad)).sum())


def outflow_lowrank(grid, state, quad):
    """boundary_outflow of X S W^T without forming it."""
    h = wall_traces(grid, state.X)                      # (4, r)
    a = _outflow_weights(quad) @ as_device(state.W.values)  # (4, r) = (W^T (w max(om.n,0)))^T
    s = a @ as_device(state.S).T                        # (4, r): row w = (S a_w)^T
    return float((h * s).sum())


@dataclass
class EnergyLedger:
    """Running energy balance of driver.run_problem (driver.py:476-553)."""

    grid: object
    quad: object
    rho_cv: torch.Tensor
    c: float
    dt: float
    e_mat: float = 0.0
    e_rad: float = 0.0

    @classmethod
    def start(cls, grid, quad, rho_cv, T, phi_dofs, c, dt):
        led = cls(grid, quad, as_device(rho_cv), float(c), float(dt))
        led.e_mat = led.material(T)
        led.e_rad = integrate_dofs(grid, phi_dofs) / led.c
        return led

    def material(self, T):
        return float((self.rho_cv * as_device(T)).sum()) * self.grid.dx * self.grid.dy

    def row(self, k, iterations, cond, T, raw_T, phi_quad, outflow, discarded=0.0):
        """One DIAGNOSTIC_COLUMNS row; phi_quad = psi @ w of the new state."""
        area = self.grid.dx * self.grid.dy
        floor_source = float((self.rho_cv * (as_device(T) - as_device(raw_T))).sum()) * area
        e_mat = self.material(T)
        e_rad = integrate_dofs(self.grid, phi_quad) / self.c
        total = e_mat + e_rad
        residual = (total - self.e_mat - self.e_rad + self.dt * outflow - floor_source) / max(
            abs(total), 1e-300)
        self.e_mat, self.e_rad = e_mat, e_rad
        return (k, k * self.dt, int(iterations), float(cond), float(discarded), e_mat, e_rad,
                float(outflow), residual)
