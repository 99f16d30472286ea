"""Discrete-ordinates sweeps and source iteration on the B200
(mirror of transport_sn.py:38-450).

The reference assembles sparse N_x x N_x operators every step and sweeps
with cached per-cell inverses; here the structured stencil is implicit: the
per-step state is sigma_t / sigma_s / q per cell plus the constant reference
blocks, and one persistent CUDA launch sweeps every direction
(csrc/sweep.cu).  The public functions keep the reference names, arguments,
return types and exceptions.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, empty, stream, upload, zeros
from .errors import CgError, ConfigurationError, ContractViolation, IterationLimitError
from .mesh import DISCONTINUOUS, cellops_struct

FOUR_PI = 4.0 * np.pi
_WARPS_PER_SM_TARGET = 8


def quadrant_code(omega):
    """(sx<0) | 2*(sy<0); grazing components sweep as positive
    (transport_sn.py:38-42)."""
    return (0 if omega[0] >= 0.0 else 1) | (0 if omega[1] >= 0.0 else 2)


def plan_groups(omegas, closure, n_strips, dw=None, sm_count=148):
    """Partition the swept directions into warp groups (host logic).

    Directions of one quadrant share the traversal order, so a group holds
    up to ``dw`` directions of a single quadrant; the default width is 2 when
    that still yields enough warps (groups x strips) to fill the GPU, else 1.  Returns (groups structured array, dw, quad codes per slot).
    """
    om = np.asarray(omegas, dtype=float)
    clo = np.asarray(closure, dtype=float)
    D = om.shape[0]
    quads = np.array([quadrant_code(om[d]) for d in range(D)], dtype=np.int32)
    members = [np.flatnonzero(quads == q) for q in range(4)]
    if dw is None:
        # pairs of directions per warp when that still fills the GPU with
        # (group, strip) items (fastest on the config-2 full-SN sweep:
        # dw 2 > 4 > 1 > 8, scripts/full_sn.py), else one direction per warp
        target = _WARPS_PER_SM_TARGET * sm_count
        g2 = sum(math.ceil(len(m) / 2) for m in members)
        dw = 2 if g2 * n_strips >= target else 1
    biggest = max((len(m) for m in members), default=1)
    while dw > 1 and dw // 2 >= biggest:
        dw //= 2
    if dw not in (1, 2, 4, 8):
        raise ContractViolation(f"sweep group width must be 1, 2, 4 or 8, got {dw}")
    rows = []
    for q in range(4):
        m = members[q]
        for k in range(0, len(m), dw):
            rows.append((q, m[k:k + dw]))
    groups = np.zeros(len(rows), dtype=_lib.GROUP_DTYPE)
    for gi, (q, slots) in enumerate(rows):
        groups[gi]["quad"] = q
        groups[gi]["ndir"] = len(slots)
        groups[gi]["slot"][:len(slots)] = slots
        groups[gi]["ox"][:len(slots)] = np.abs(om[slots, 0])
        groups[gi]["oy"][:len(slots)] = np.abs(om[slots, 1])
        groups[gi]["cw"][:len(slots)] = clo[slots]
    return groups, dw, quads


def _groups_to_device(groups):
    return upload(np.frombuffer(groups.tobytes(), dtype=np.uint8).copy())


@dataclass(eq=False)
class DiscreteOperators:
    """Per-step operator data for the sweeps (transport_sn.py:78-97).

    Holds the grid, the linearised step (device tensors) and the scaled
    reference blocks; the sparse matrices of the reference are implicit.
    """

    grid: object
    step: object
    cellops: object
    dsa_penalty: str = "simplified"
    penalty_closure: tuple | None = None
    _sigma_sk4: torch.Tensor | None = None
    _scratch: dict = field(default_factory=dict)

    @property
    def n_cells(self):
        return self.grid.n_cells

    @property
    def vec_len(self):
        return int(_lib.load().dlrsn_sk_vec_len(self.grid.nx, self.grid.ny))

    @property
    def scalar_len(self):
        return int(_lib.load().dlrsn_sk_scalar_len(self.grid.nx, self.grid.ny))

    @property
    def cellops_ptr(self):
        import ctypes

        return ctypes.c_void_p(ctypes.addressof(self.cellops))

    def sigma_t_sk4(self):
        if self._sigma_sk4 is None:
            out = empty(4 * self.scalar_len)
            _lib.call("dlrsn_cells_to_sk4", self.cellops_ptr, _lib.ptr(self.step.sigma_t),
                      _lib.ptr(out), stream())
            self._sigma_sk4 = out
        return self._sigma_sk4

    def buffer(self, name, numel, dtype=torch.float64, zero=False):
        """Reusable device scratch (grows on demand)."""
        t = self._scratch.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = (torch.zeros if zero else torch.empty)(max(numel, 1), dtype=dtype, device=device())
            self._scratch[name] = t
        return t

    def mass_apply(self, u, coeff=None):
        """Block-diagonal mass times a dof vector / (n_dofs, k) block
        (transport_sn.py:107-116)."""
        m = torch.from_numpy(np.frombuffer(bytes(self.cellops.mass), dtype=np.float64)
                             .reshape(4, 4).copy()).to(device())
        u = as_device(u)
        flat = u.ndim == 1
        uc = u.reshape(self.n_cells, 4, -1)
        out = torch.einsum("ij,cjk->cik", m, uc)
        if coeff is not None:
            out = out * as_device(coeff)[:, None, None]
        out = out.reshape(self.grid.n_dofs, -1)
        return out[:, 0] if flat else out

    def source_vector(self, cell_values):
        row = torch.tensor(list(self.cellops.src_row), dtype=torch.float64, device=device())
        return (as_device(cell_values)[:, None] * row[None, :]).reshape(-1)


def assemble_operators(grid, step, dsa_penalty="simplified", penalty_closure=None, validate=True):
    """Per-step operator data (transport_sn.py:201-300); same checks
    (``validate=False`` defers the device-side sigma check to the caller)."""
    if grid.flavor != DISCONTINUOUS:
        raise ContractViolation("sweep transport needs the discontinuous dof layout")
    for name in ("sigma_t", "sigma_s", "q"):
        if tuple(getattr(step, name).shape) != (grid.n_cells,):
            raise ContractViolation(f"step field {name} must be per-cell")
    if validate and bool((step.sigma_t - step.sigma_s <= 0).any()):
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    if dsa_penalty not in ("simplified", "collocation"):
        raise ContractViolation(f"unknown dsa penalty variant {dsa_penalty!r}")
    return DiscreteOperators(grid=grid, step=step, cellops=cellops_struct(grid),
                             dsa_penalty=dsa_penalty, penalty_closure=penalty_closure)


@dataclass(eq=False)
class SourceIterationResult:
    psi: torch.Tensor  # (n_dofs, n_angles), canonical layout, on the device
    phi: torch.Tensor  # converged scattering scalar flux
    iterations: int


class _SweepPlan:
    """Device-side tables and buffers of one set of swept directions."""

    def __init__(self, ops, omegas, closure, dw=None):
        g = ops.grid
        sms = ctypes_int()
        _lib.call("dlrsn_device_sm_count", sms.ptr)
        ns = (g.ny + 31) // 32
        self.groups, self.dw, quads = plan_groups(omegas, closure, ns, dw=dw, sm_count=sms.value)
        self.G = len(self.groups)
        self.D = len(quads)
        self.groups_dev = _groups_to_device(self.groups)
        self.quads_dev = upload(quads)
        self.ws_bytes = int(_lib.load().dlrsn_sweep_workspace_bytes(g.nx, g.ny, self.G, self.dw))
        self.workspace = sweep_workspace(ops, self.ws_bytes)


class ctypes_int:
    def __init__(self):
        import ctypes

        self._v = ctypes.c_int(0)
        self.ptr = ctypes.byref(self._v)

    @property
    def value(self):
        return self._v.value


def sweep_workspace(ops, nbytes):
    """Sweep workspace (ticket, status, handoff slots), initialised once when
    (re)allocated; the kernel leaves it re-armed after every launch."""
    ws = ops._scratch.get("sweep_ws")
    if ws is None or ws.numel() < nbytes:
        ws = _shared_workspace(ops.grid, nbytes)
        ops._scratch["sweep_ws"] = ws
    return ws


_WS_CACHE = {}


def _shared_workspace(grid, nbytes):
    # one per (device, host thread): sweeps issued from different threads
    # (thread-ranks in the tests) must not share the ticket / handoff words
    key = (torch.cuda.current_device(), threading.get_ident())
    ws = _WS_CACHE.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device())
        _lib.call("dlrsn_sweep_workspace_init", _lib.ptr(ws), ws.numel(), stream())
        _WS_CACHE[key] = ws
    return ws


# Optional live timing of sweep launches (bench.py roofline): when set to a
# list, every launch appends (start_event, end_event, n_cells, n_dirs).
SWEEP_EVENTS = None


def _sweep(ops, plan, rhs_sk, psi_sk, scat_sk4=None, phi_part=None, max_ctas=0):
    sig = ops.sigma_t_sk4()
    ev = None
    if SWEEP_EVENTS is not None:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    _lib.call("dlrsn_sweep", ops.cellops_ptr, plan.G, _lib.ptr(plan.groups_dev), plan.dw,
              _lib.ptr(sig), _lib.ptr(scat_sk4), _lib.ptr(rhs_sk), _lib.ptr(psi_sk),
              _lib.ptr(phi_part), _lib.ptr(plan.workspace), plan.workspace.numel(), int(max_ctas),
              stream())
    if ev is not None:
        ev[1].record()
        SWEEP_EVENTS.append((ev[0], ev[1], ops.grid.n_cells, plan.D, plan.G))


def mirror_pairs(omegas):
    """z-mirror deduplication ("we need only
    solving for half the angles" in xy geometry): omega_z does not enter a
    2-D sweep, and the reference keys its per-direction operators on
    (omega_x, omega_y) (transport_sn.py:143), so nodes with bitwise-equal
    (omega_x, omega_y) sweep the same operator.  Returns (first index of each
    distinct pair, in node order; the pair index of every node)."""
    om = np.ascontiguousarray(np.asarray(omegas, dtype=float)[:, :2])
    key = om.view(np.dtype((np.void, om.dtype.itemsize * 2))).ravel()
    _, first, inverse = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")  # distinct pairs in node order
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return first[order], rank[inverse.ravel()]


def dedup_mirrors(omegas, closure):
    """(omegas of the distinct (omega_x, omega_y) pairs, their summed closure
    weights, pair index per node): the sweep of a z-symmetric problem (every
    node's rhs depends on (omega_x, omega_y) only) gives mirrored nodes the
    same psi, so one sweep per pair with the summed weight has the same
    closure flux (to round-off of the weight sum)."""
    om = np.asarray(omegas, dtype=float)
    clo = np.asarray(closure, dtype=float)
    first, inv = mirror_pairs(om)
    w = np.zeros(first.size)
    np.add.at(w, inv, clo)
    return om[first], w, inv


def closure_sweep(ops, omegas, closure, rhs, *, scat_phi=None, dw=4, ws_limit=8 << 30,
                  dedup=True):
    """One sweep of many directions that all see the same rhs, returning only
    the closure phi = sum_d closure_d psi_d (transport_sn.py:303-322 per
    direction, psi @ closure of :438) -- psi is never stored.  This is the
    full-SN stress sweep of config 5 (16384 directions on 4096^2: psi would
    be 8.8 TB).  ``rhs`` (n_dofs) is the shared right-hand side, e.g.
    source_vector(q) + inv_cdt M psi_old for an isotropic psi_old;
    ``scat_phi`` (n_dofs, optional) adds the scattering source
    M (sigma_s phi) / 4 pi.  Groups of ``dw`` directions add their closure
    sums with fp64 atomics (dlrsn_sweep_closure), so phi is reproducible to
    round-off only; the groups are launched in batches whose strip-handoff
    workspace stays under ``ws_limit`` bytes.  Every direction sees the same
    rhs, so z-mirrored nodes have the same psi: with ``dedup`` each distinct
    (omega_x, omega_y) is swept once with the summed closure weight (half of
    a product quadrature's nodes)."""
    g = ops.grid
    st = ops.step
    om = np.asarray(omegas.cpu() if isinstance(omegas, torch.Tensor) else omegas, dtype=float)
    clo = np.asarray(closure.cpu() if isinstance(closure, torch.Tensor) else closure, dtype=float)
    if clo.shape != (om.shape[0],):
        raise ContractViolation("closure vector must have one entry per swept angle")
    if dedup:
        om, clo, _ = dedup_mirrors(om, clo)
    vl = ops.vec_len
    rhs = as_device(rhs).reshape(g.n_dofs, 1)
    cols = rhs.expand(-1, 4).contiguous()  # the same rhs in the 4 quadrant orientations
    rhs4 = ops.buffer("rhs4", 4 * vl)
    quads4 = upload(np.arange(4, dtype=np.int32))
    zero_q = ops.buffer("zero_q", g.n_cells, zero=True)
    _lib.call("dlrsn_rhs_build", ops.cellops_ptr, 4, _lib.ptr(quads4), _lib.ptr(zero_q), 0.0,
              None, 1, _lib.ptr(cols), 4, _lib.ptr(rhs4), stream())
    del cols
    scat = None
    if scat_phi is not None:
        scat = ops.buffer("scat_sk4", 4 * vl)
        flags = zeros(1, dtype=torch.int32)
        _lib.call("dlrsn_scatter_source", ops.cellops_ptr, _lib.ptr(as_device(scat_phi)),
                  _lib.ptr(st.sigma_s), _lib.ptr(scat), _lib.ptr(flags), stream())
    ns = (g.ny + 31) // 32
    groups, dw, _ = plan_groups(om, clo, ns, dw=dw)
    G = len(groups)
    lib = _lib.load()
    per_group = int(lib.dlrsn_sweep_workspace_bytes(g.nx, g.ny, 1, dw))
    batch = max(1, min(G, ws_limit // max(per_group, 1)))
    ws_bytes = int(lib.dlrsn_sweep_workspace_bytes(g.nx, g.ny, batch, dw))
    ws = sweep_workspace(ops, ws_bytes)
    gdev = _groups_to_device(groups)
    gsize = _lib.GROUP_DTYPE.itemsize
    phi = zeros(g.n_dofs)
    sig = ops.sigma_t_sk4()
    for g0 in range(0, G, batch):
        nb = min(batch, G - g0)
        _lib.call("dlrsn_sweep_closure", ops.cellops_ptr, nb,
                  ctypes.c_void_p(gdev.data_ptr() + g0 * gsize), dw, _lib.ptr(sig),
                  _lib.ptr(scat), _lib.ptr(rhs4), _lib.ptr(phi), _lib.ptr(ws), ws.numel(), 0,
                  stream())
    return phi


def sweep_status_word(workspace):
    """Device view of the sweep workspace's sticky status (word 1; 2 = a
    strip handoff wait timed out, include/dlrsn.h)."""
    return workspace[4:8].view(torch.int32)


def raise_sweep_status(status, workspace):
    """A timed-out strip handoff leaves psi wrong: re-arm the workspace and
    fail loudly instead of returning it."""
    if int(status):
        _lib.call("dlrsn_sweep_workspace_init", _lib.ptr(workspace), workspace.numel(), stream())
        raise RuntimeError(f"dlrsn sweep strip handoff timed out (status {int(status)}); "
                           "workspace re-armed")


def _to_canonical(ops, plan, psi_sk, out=None):
    g = ops.grid
    psi = out if out is not None else empty(g.n_dofs, plan.D)
    _lib.call("dlrsn_sk_to_canonical", ops.cellops_ptr, plan.D, _lib.ptr(plan.quads_dev),
              _lib.ptr(psi_sk), _lib.ptr(psi), plan.D, stream())
    return psi


def sweep_solve(ops, omega, rhs, _key=None):
    """One direction's upwind solve by a single sweep (transport_sn.py:303-322)."""
    g = ops.grid
    omega = np.asarray(omega, dtype=float)
    rhs = as_device(rhs).reshape(g.n_dofs, 1).contiguous()
    plan = _SweepPlan(ops, omega[None, :], np.ones(1), dw=1)
    vl = ops.vec_len
    rhs_sk = empty(vl)
    psi_sk = empty(vl)
    zero_q = ops.buffer("zero_q", g.n_cells, zero=True)
    _lib.call("dlrsn_rhs_build", ops.cellops_ptr, 1, _lib.ptr(plan.quads_dev), _lib.ptr(zero_q),
              0.0, None, 1, _lib.ptr(rhs), 1, _lib.ptr(rhs_sk), stream())
    _sweep(ops, plan, rhs_sk, psi_sk)
    out = _to_canonical(ops, plan, psi_sk)[:, 0].contiguous()
    raise_sweep_status(sweep_status_word(plan.workspace).item(), plan.workspace)
    return out


def source_iteration(ops, omegas, closure, psi_time=None, *, use_dsa=True, tol=1e-8,
                     max_iters=200, phi_start=None, extra_source=None, threads=0, dw=None,
                     keep_sk=False, comm=None, inflow=None):
    """Lagged-scattering iteration over device sweeps (transport_sn.py:377-450).

    ``threads`` is accepted for API compatibility and ignored (the sweeps of
    all directions run in one launch).  ``psi_time`` / ``extra_source`` are
    (n_dofs, n_angles) arrays; results are device tensors.  With ``comm`` (a
    sharding.DirectionComm over > 1 rank) the directions are split across
    ranks and the closure flux is all-reduced every iteration.  ``inflow``
    (extension, see ``inflow_source``): isotropic inflow walls, added to the
    sweep rhs on the device (dlrsn_inflow_add) next to ``extra_source``.
    """
    omegas = np.asarray(omegas.cpu() if isinstance(omegas, torch.Tensor) else omegas, dtype=float)
    closure = np.asarray(closure.cpu() if isinstance(closure, torch.Tensor) else closure, dtype=float)
    nd = omegas.shape[0]
    if closure.shape != (nd,):
        raise ContractViolation("closure vector must have one entry per swept angle")
    g = ops.grid
    st = ops.step
    # direction sharding across ranks (sharding.py): this rank sweeps `mine`
    owners = None
    mine = np.arange(nd)
    if comm is not None and comm.world_size > 1:
        from .sharding import partition_directions

        owners = partition_directions(omegas, comm.world_size)
        mine = owners[comm.rank]
    nl = len(mine)
    plan = _SweepPlan(ops, omegas[mine], closure[mine], dw=dw) if nl else None
    vl = ops.vec_len
    rhs_sk = ops.buffer("rhs_sk", max(nl, 1) * vl)
    psi_sk = ops.buffer("psi_sk", max(nl, 1) * vl)
    # single-direction groups: the closure is read from psi itself (no partials)
    use_part = plan is not None and plan.dw > 1
    part = ops.buffer("phi_part", (plan.G if use_part else 1) * vl)
    part_arg = part if use_part else None
    scat = ops.buffer("scat_sk4", 4 * vl)

    def local_cols(a):
        if a is None:
            return None
        a = as_device(a).reshape(g.n_dofs, nd)
        if owners is not None:
            a = a[:, torch.as_tensor(mine, device=a.device)]
        return a.contiguous()

    pt, ex = local_cols(psi_time), local_cols(extra_source)
    if plan:
        _lib.call("dlrsn_rhs_build", ops.cellops_ptr, nl, _lib.ptr(plan.quads_dev), _lib.ptr(st.q),
                  float(st.inv_cdt), _lib.ptr(pt), nl, _lib.ptr(ex), nl, _lib.ptr(rhs_sk), stream())
        inflow4 = inflow_values(inflow)
        if inflow4 is not None:
            om_dev = upload(np.ascontiguousarray(omegas[mine], dtype=np.float64))
            vals = (ctypes.c_double * 4)(*inflow4)
            _lib.call("dlrsn_inflow_add", ops.cellops_ptr, nl, _lib.ptr(plan.quads_dev),
                      _lib.ptr(om_dev), None, vals, _lib.ptr(rhs_sk), stream())
    phi = zeros(g.n_dofs) if phi_start is None else as_device(phi_start).reshape(-1).clone()
    phi_new = empty(g.n_dofs)
    flags = zeros(1, dtype=torch.int32)
    _lib.call("dlrsn_scatter_source", ops.cellops_ptr, _lib.ptr(phi), _lib.ptr(st.sigma_s),
              _lib.ptr(scat), _lib.ptr(flags), stream())
    nb = (g.n_cells + 255) // 256
    red_ws = ops.buffer("red_ws", 256 // 8 + 2 * nb + 8, zero=True)
    norms = zeros(2)
    host = torch.empty(4, dtype=torch.float64, pin_memory=True)
    dsa = _DsaState(ops) if use_dsa else None
    change = math.inf
    for it in range(1, max_iters + 1):
        if owners is None and dsa is None:
            _sweep(ops, plan, rhs_sk, psi_sk, scat, part_arg)
            _lib.call("dlrsn_phi_combine", ops.cellops_ptr, plan.G, _lib.ptr(plan.groups_dev),
                      _lib.ptr(part_arg), _lib.ptr(psi_sk), _lib.ptr(phi), _lib.ptr(st.sigma_s),
                      _lib.ptr(phi_new), _lib.ptr(scat), _lib.ptr(norms), _lib.ptr(red_ws), stream())
        elif owners is None:
            # DSA: phi_half from the sweep, the diffusion correction, then the
            # norms and the next scattering source from phi_half + delta
            _sweep(ops, plan, rhs_sk, psi_sk, scat, part_arg)
            _lib.call("dlrsn_phi_combine", ops.cellops_ptr, plan.G, _lib.ptr(plan.groups_dev),
                      _lib.ptr(part_arg), _lib.ptr(psi_sk), _lib.ptr(phi), _lib.ptr(st.sigma_s),
                      _lib.ptr(phi_new), None, _lib.ptr(norms), _lib.ptr(red_ws), stream())
            dsa.correct(phi_new, phi)
            _lib.call("dlrsn_phi_finish", ops.cellops_ptr, _lib.ptr(phi_new), _lib.ptr(phi),
                      _lib.ptr(st.sigma_s), _lib.ptr(scat), _lib.ptr(norms), _lib.ptr(red_ws),
                      stream())
        else:
            # local partial closure flux -> allreduce over NVLink -> norms and
            # scattering source from the summed flux (identical on all ranks)
            if plan:
                _sweep(ops, plan, rhs_sk, psi_sk, scat, part_arg)
                _lib.call("dlrsn_phi_combine", ops.cellops_ptr, plan.G, _lib.ptr(plan.groups_dev),
                          _lib.ptr(part_arg), _lib.ptr(psi_sk), _lib.ptr(phi), _lib.ptr(st.sigma_s),
                          _lib.ptr(phi_new), None, _lib.ptr(norms), _lib.ptr(red_ws), stream())
            else:
                phi_new.zero_()
            comm.allreduce_sum_(phi_new)
            if dsa is not None:  # replicated on every rank from the summed flux
                dsa.correct(phi_new, phi)
            _lib.call("dlrsn_phi_finish", ops.cellops_ptr, _lib.ptr(phi_new), _lib.ptr(phi),
                      _lib.ptr(st.sigma_s), _lib.ptr(scat), _lib.ptr(norms), _lib.ptr(red_ws),
                      stream())
        host[:2].copy_(norms, non_blocking=True)
        if it == 1:
            host[2:3].copy_(flags.to(torch.float64), non_blocking=True)
        if plan:
            host[3:4].copy_(sweep_status_word(plan.workspace).to(torch.float64), non_blocking=True)
        if dsa is not None:
            dsa.stage_info()
        torch.cuda.current_stream(device()).synchronize()
        if plan:
            raise_sweep_status(host[3].item(), plan.workspace)
        if dsa is not None:
            dsa.raise_on_failure()
        phi, phi_new = phi_new, phi
        if it == 1 and host[2].item() == 0.0:  # pure absorber (transport_sn.py:410,430-432)
            return _finish(ops, plan, psi_sk, phi, 1, keep_sk, comm, owners, nd)
        d2, n2 = host[0].item(), host[1].item()
        change = math.sqrt(d2) / max(math.sqrt(n2), 1e-300)
        if change <= tol:
            return _finish(ops, plan, psi_sk, phi, it, keep_sk, comm, owners, nd)
    raise IterationLimitError("source iteration did not converge", max_iters, change)


class _DsaState:
    """Device state of the diffusion correction (transport_sn.py:353-367):
    dlrsn_dsa_correct solves the Jacobi-PCG system in one cooperative launch
    (tol 1e-10, at most 10 n_dofs iterations, the reference's pcg defaults)
    and writes phi_half + delta in place."""

    TOL = 1e-10
    HIST = 4096

    def __init__(self, ops):
        g = ops.grid
        st = ops.step
        if ops.dsa_penalty == "simplified":
            self.kx = self.ky = 0.25  # (1/2) <|omega.n|>, transport_sn.py:183-184
        else:
            om, cw = ops.penalty_closure
            om = np.asarray(om.cpu() if isinstance(om, torch.Tensor) else om, dtype=float)
            cw = np.asarray(cw.cpu() if isinstance(cw, torch.Tensor) else cw, dtype=float)
            self.kx = 0.5 * float(cw @ np.abs(om[:, 0])) / FOUR_PI  # :186-188
            self.ky = 0.5 * float(cw @ np.abs(om[:, 1])) / FOUR_PI
        self.ops = ops
        self.max_iters = 10 * g.n_dofs
        ln = int(_lib.load().dlrsn_dsa_workspace_len(g.nx, g.ny))
        self.ws = ops.buffer("dsa_ws", ln)
        self.ws_len = ln
        self.info = ops.buffer("dsa_info", 2, dtype=torch.int32)
        self.hist = ops.buffer("dsa_hist", self.HIST)
        self.host = torch.empty(2, dtype=torch.int32, pin_memory=True)
        self.sigma_t, self.sigma_s = st.sigma_t, st.sigma_s

    def correct(self, phi_half, phi_old):
        _lib.call("dlrsn_dsa_correct", self.ops.cellops_ptr, _lib.ptr(self.sigma_t),
                  _lib.ptr(self.sigma_s), self.kx, self.ky, _lib.ptr(phi_half),
                  _lib.ptr(phi_old), _lib.ptr(phi_half), self.TOL, self.max_iters,
                  _lib.ptr(self.ws), self.ws_len, _lib.ptr(self.info), _lib.ptr(self.hist),
                  self.HIST, stream())

    def stage_info(self):
        self.host.copy_(self.info[:2], non_blocking=True)

    def raise_on_failure(self):
        if int(self.host[1]):
            n = min(self.max_iters + 1, self.HIST)
            hist = self.hist[:n].cpu().numpy().tolist()
            raise CgError(f"dsa failed to reach tol {self.TOL:g}", self.max_iters, hist)


def _finish(ops, plan, psi_sk, phi, it, keep_sk, comm=None, owners=None, nd=0):
    if owners is None:
        psi = _to_canonical(ops, plan, psi_sk)
    else:
        local = _to_canonical(ops, plan, psi_sk) if plan else empty(ops.grid.n_dofs, 0)
        psi = comm.allgather_columns(local, owners, nd)
    res = SourceIterationResult(psi=psi, phi=phi, iterations=it)
    if keep_sk:
        res.psi_sk = psi_sk
        res.plan = plan
    return res


def boundary_outflow(grid, psi, omegas, weights, ref_edge=None):
    """Quadrature outflow through the boundary (transport_sn.py:479-492)."""
    psi = as_device(psi)
    cells, walls, normals, lengths = grid.boundary_faces
    e0 = np.array([{"left": 0, "right": 1, "bottom": 0, "top": 2}[w] for w in walls])
    e1 = np.array([{"left": 2, "right": 3, "bottom": 1, "top": 3}[w] for w in walls])
    i0 = torch.from_numpy(4 * cells + e0).to(device())
    i1 = torch.from_numpy(4 * cells + e1).to(device())
    vals = 0.5 * (psi[i0] + psi[i1]) * as_device(lengths)[:, None]
    on = as_device(normals) @ as_device(np.asarray(omegas)[:, :2]).T
    return float((torch.clamp(on, min=0.0) * vals @ as_device(weights)).sum())


def inflow_values(inflow):
    """None | {wall: psi_b} | (left, right, bottom, top) -> 4-tuple, or None
    when every wall is vacuum (ContractViolation for unknown walls or
    negative / non-finite intensities)."""
    if inflow is None:
        return None
    walls = ("left", "right", "bottom", "top")
    if isinstance(inflow, dict):
        bad = set(inflow) - set(walls)
        if bad:
            raise ContractViolation(f"unknown inflow walls {sorted(bad)}")
        vals = tuple(float(inflow.get(w, 0.0)) for w in walls)
    else:
        vals = tuple(float(v) for v in inflow)
        if len(vals) != 4:
            raise ContractViolation("inflow needs 4 values (left, right, bottom, top)")
    if any(not np.isfinite(v) or v < 0 for v in vals):
        raise ContractViolation("inflow intensities must be finite and non-negative")
    return vals if any(vals) else None

def inflow_source(grid, omegas, inflow):
    """(n_dofs, D) device load of isotropic inflow walls for the
    ``extra_source`` argument of ``source_iteration`` (transport_sn.py:387,
    406-407): column d gets max(-omega_d.n_w, 0) psi_b,w (e2 @ [1, 1]) on the
    edge dofs of the cells of wall w (mesh.py:34-39).  An extension: the
    reference is vacuum-only (transport_sn.py:11-13); restated in
    oracle/port.py ``inflow_load``."""
    vals = inflow_values(inflow)
    om = torch.as_tensor(np.array(np.atleast_2d(omegas), dtype=float), device=device())
    out = zeros(grid.n_dofs, om.shape[0])
    if vals is None:
        return out
    co = cellops_struct(grid)
    cid = torch.arange(grid.n_cells, device=out.device).reshape(grid.ny, grid.nx)
    walls = (("left", cid[:, 0], (-1.0, 0.0), (0, 2), co.e2x),
             ("right", cid[:, -1], (1.0, 0.0), (1, 3), co.e2x),
             ("bottom", cid[0, :], (0.0, -1.0), (0, 1), co.e2y),
             ("top", cid[-1, :], (0.0, 1.0), (2, 3), co.e2y))
    for (_, cells, n, locs, e2), psi_b in zip(walls, vals):
        if psi_b == 0.0:
            continue
        g = (e2[0] + e2[1], e2[2] + e2[3])
        coef = torch.clamp(-(om[:, 0] * n[0] + om[:, 1] * n[1]), min=0.0) * psi_b
        for k, l in enumerate(locs):
            out[4 * cells + l, :] += g[k] * coef[None, :]
    return out
