"""Numpy-at-the-edges drop-in for the reference's step API.

``step_collocation(grid, step, quad, state, ...)`` takes the reference's own
objects -- a greytrt ``Grid``, ``LinearizedStep``, ``QuadratureSet`` and
``DlrState`` holding numpy arrays (``dlr_sn.py:86-98``), or any object with
the same attributes -- runs the step on the B200 and returns a new state of
the caller's own ``DlrState`` / ``AngularBasis`` classes with numpy arrays,
plus a ``CollocationStepInfo`` whose ``phi`` is numpy (numpy at
``.X``, ``.S``, ``.W.values``, ``.W.beta``, ``info.phi``).  A greytrt time
loop (``driver.py:505-517``) runs unchanged with this function in place of
``greytrt.dlr_sn.step_collocation``.

Transfers: inputs are copied host -> device each call (directly by DMA when
the arrays are backed by pinned memory, which is the case for the arrays
this function returns, so a chained loop never stages through pageable
memory); outputs are read back into pinned blocks from torch's caching host
allocator, so a loop that drops its previous state recycles them.  The
device-resident API (``dlr_sn.step_collocation`` on ``lowrank.DlrState``)
avoids the copies altogether.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from ._device import device
from .angular import AngularBasis, QuadratureSet
from .lowrank import DlrState
from .mesh import build_grid
from .physics import LinearizedStep, PhysicsConstants

_GRIDS: dict = {}
_QUADS: dict = {}


def _cached(cache, obj, make):
    ent = cache.get(id(obj))
    if ent is None or ent[0] is not obj:
        if len(cache) > 32:
            cache.clear()
        ent = (obj, make(obj))
        cache[id(obj)] = ent
    return ent[1]


def device_grid(grid):
    """Our grid for a reference ``Grid`` (nx, ny, x0, y0, dx, dy; mesh.py:76-127)."""
    if hasattr(grid, "cellops_struct") or type(grid).__module__.startswith(__package__):
        return grid
    return _cached(_GRIDS, grid, lambda g: build_grid(
        int(g.nx), int(g.ny), (float(g.x0), float(g.y0), g.nx * float(g.dx), g.ny * float(g.dy))))


def device_quadrature(quad):
    """Our quadrature for a reference ``QuadratureSet`` (angular.py:28-42)."""
    if isinstance(quad, QuadratureSet):
        return quad

    def make(q):
        om = np.array(q.omegas, dtype=float)
        w = np.array(q.weights, dtype=float)
        anti = np.array(getattr(q, "antipode", np.arange(om.shape[0])))
        for a in (om, w, anti):
            a.setflags(write=False)
        return QuadratureSet(om, w, anti, int(getattr(q, "n_polar", 0)),
                             int(getattr(q, "n_azimuthal", 0)))

    return _cached(_QUADS, quad, make)


def _h2d(a):
    """Host array -> fp64 device tensor (async DMA when ``a`` is pinned)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=torch.float64).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to(device=device(), non_blocking=t.is_pinned())


def _pinned_like(t):
    return torch.empty(t.shape, dtype=t.dtype, pin_memory=True)


def device_step(step):
    """Our LinearizedStep for a reference one (physics.py:78-91)."""
    if isinstance(step, LinearizedStep):
        return step
    k = getattr(step, "constants", None)
    consts = PhysicsConstants(c=float(k.c), a_r=float(k.a_r)) if k is not None else PhysicsConstants()
    return LinearizedStep(
        sigma_t=_h2d(step.sigma_t), sigma_s=_h2d(step.sigma_s), sigma_a=_h2d(step.sigma_a),
        q=_h2d(step.q), T0=_h2d(step.T0), denom=_h2d(step.denom), rho_cv=_h2d(step.rho_cv),
        dt=float(step.dt), inv_cdt=float(step.inv_cdt), constants=consts)


def device_state(state):
    """Our DlrState for a reference one (lowrank.py:43-81)."""
    if isinstance(state, DlrState):
        return state
    W = state.W
    beta = getattr(W, "beta", None)
    basis = AngularBasis(values=_h2d(W.values), beta=None if beta is None else _h2d(beta),
                         pinned=bool(getattr(W, "pinned", False)))
    return DlrState(X=_h2d(state.X), S=_h2d(state.S), W=basis)


@dataclass(eq=False)
class CollocationStepInfo:
    """dlr_sn.py:40-47 with numpy ``phi`` and ``angle_indices``."""

    iterations: int
    angle_indices: np.ndarray
    phi: np.ndarray
    spatial_deficiency: int
    angular_deficiency: int
    _selection: object = None
    deim_gaps: np.ndarray | None = None

    @cached_property
    def interpolation_condition(self):
        return self._selection.cond


def to_host(new, info, like_state):
    """Read a device step result back as the caller's numpy types: returns
    (state of type(like_state), CollocationStepInfo)."""
    outs = [new.X, new.S, new.W.values, new.W.beta, info.phi]
    host = [_pinned_like(t) for t in outs]
    for h, t in zip(host, outs):
        h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(device()).synchronize()
    X, S, Wv, beta, phi = (h.numpy() for h in host)
    W_old = like_state.W
    basis_cls = type(W_old)
    try:
        basis = basis_cls(values=Wv, beta=beta, pinned=bool(getattr(W_old, "pinned", False)))
    except TypeError:
        basis = basis_cls(values=Wv, beta=beta)
    state = type(like_state)(X=X, S=S, W=basis)
    hinfo = CollocationStepInfo(
        iterations=int(info.iterations), angle_indices=np.asarray(info.angle_indices).copy(),
        phi=phi, spatial_deficiency=int(info.spatial_deficiency),
        angular_deficiency=int(info.angular_deficiency), _selection=info.selection,
        deim_gaps=getattr(info, "deim_gaps", None))
    return state, hinfo


def step_collocation(grid, step, quad, state, *, si_tol=1e-8, si_max_iters=200, use_dsa=True,
                     dsa_penalty="simplified", threads=0, check_state=True, **kw):
    """Drop-in for ``greytrt.dlr_sn.step_collocation`` (dlr_sn.py:86-151):
    reference objects in, reference-typed numpy results out; the step runs
    on the device (``dlr_sn.step_collocation``; extra keywords pass through,
    e.g. ``angle_indices``, ``deim_tie_tol``, ``inflow``)."""
    from .dlr_sn import step_collocation as device_step_collocation

    new, info = device_step_collocation(
        device_grid(grid), device_step(step), device_quadrature(quad), device_state(state),
        si_tol=si_tol, si_max_iters=si_max_iters, use_dsa=use_dsa, dsa_penalty=dsa_penalty,
        threads=threads, check_state=check_state, **kw)
    return to_host(new, info, state)
