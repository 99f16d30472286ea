"""One implicit SN-like DLR step on the B200 (mirror of dlr_sn.py:40-151).

Algorithm 1 of the paper, same call signature and
results as the reference ``step_collocation``:

1. DEIM angles of the current angular basis, closure weights;
2. collocated source iteration over the selected directions (K1 sweeps);
3. new spatial basis from the swept columns (M-orthonormal, K2);
4. reduced row system from the fused projections (K3) solved at the nodes;
5. nodal rows -> angular functions through the old basis, orthonormalised.

All arrays stay on the device; the host only sees the r selected indices
and closure weights (to lay out the sweep groups) and the convergence
scalars of the source iteration.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, empty, stream
from .angular import AngularBasis, orthonormalize_async
from .errors import (
    CgError,
    ConfigurationError,
    ContractViolation,
    InterpolationError,
    IterationLimitError,
    SolverError,
)
from .lowrank import (
    DlrState,
    _addr,
    _cellops_of,
    _cgs2_flags,
    _row_solve_async,
    cgs2_spatial_async,
    check_ties,
    cholqr2_speculative,
    cholqr_guard_ok,
    deim_finish,
    deim_forced_launch,
    deim_launch,
    evaluate_rows,
    raise_row_status,
    rowmix,
)
from .transport import assemble_operators, inflow_values, source_iteration

FOUR_PI = 4.0 * np.pi
# DEIM picks closer to a tie than this (relative top-2 residual gap) raise
# InterpolationTieError unless the selection is forced (SURVEY 8c hazard (i)).
# The residuals of the GPU elimination and of the reference's solves agree to
# ~1e-15 relative (tests/test_gpu_deim.py), so a gap above 1e-12 cannot flip;
# gaps down to 2.6e-11 occur in ordinary runs (the interpolation property of
# the previous step's basis) and are picked identically.
DEIM_TIE_TOL = 1e-12


@dataclass(eq=False)
class CollocationStepInfo:
    """dlr_sn.py:40-47; ``phi`` is a device tensor, the condition number of
    W_hat is evaluated on first access."""

    iterations: int
    selection: object
    angle_indices: np.ndarray
    phi: torch.Tensor
    spatial_deficiency: int
    angular_deficiency: int
    si_phi: torch.Tensor | None = None

    @cached_property
    def interpolation_condition(self):
        return self.selection.cond


def project_operators(ops, x, x_old=None, no_scatter=False):
    """Fused reduced operators: dict px, py, jx, jy, mt, ms, mo (r x r) and q
    (project_row_operators dlr_sn.py:61-71; mo = X_old^T M x for
    project_initial :50-58).  Returns (dict, packed device buffer).
    no_scatter: the caller has checked sigma_s == 0, so ms = 0 and its MMAs
    are skipped (sigma_s passed as NULL)."""
    co = _cellops_of(ops)
    x = as_device(x).contiguous()
    r = x.shape[1]
    nc = co.nx * co.ny
    part = empty(max(int(_lib.load().dlrsn_partials_len(nc, r, r, 1)), 1))
    out = empty(7 * r * r + r)
    xo = None if x_old is None else as_device(x_old).contiguous()
    st = ops.step
    _lib.call("dlrsn_project", _addr(co), r, _lib.ptr(x), _lib.ptr(xo), _lib.ptr(st.sigma_t),
              None if no_scatter else _lib.ptr(st.sigma_s), _lib.ptr(st.q), _lib.ptr(out),
              _lib.ptr(part), stream())
    mats = out[:7 * r * r].reshape(7, r, r)
    names = ("px", "py", "jx", "jy", "mt", "ms", "mo")
    proj = {k: mats[i] for i, k in enumerate(names)}
    proj["q"] = out[7 * r * r:]
    return proj, out


def project_row_operators(ops, x):
    """dlr_sn.py:61-71."""
    proj, _ = project_operators(ops, x)
    proj.pop("mo")
    return proj


def row_matrices(proj, omegas):
    """dlr_sn.py:74-83."""
    om = as_device(np.asarray(omegas, dtype=float))
    return (om[:, 0, None, None] * proj["px"] + om[:, 1, None, None] * proj["py"]
            + om[:, 0].abs()[:, None, None] * proj["jx"] + om[:, 1].abs()[:, None, None] * proj["jy"]
            + proj["mt"][None])


def project_initial(state, x_new, ops):
    """Old factors against a new spatial basis (dlr_sn.py:50-58)."""
    from .lowrank import mass_gram

    mo = mass_gram(ops, state.X, x_new)
    return state.W.values @ (state.S.T @ mo)


def step_collocation(grid, step, quad, state, *, si_tol=1e-8, si_max_iters=200, use_dsa=True,
                     dsa_penalty="simplified", threads=0, check_state=True, gs_method="cholqr2",
                     sweep_dw=None, comm=None, engine="native", inflow=None, angle_indices=None,
                     deim_tie_tol=DEIM_TIE_TOL, _advance=None, _x_new_host=None):
    """Advance one linearised step; returns (new DlrState, CollocationStepInfo).

    ``engine="native"`` issues the whole step from C++ through the single
    C-ABI call ``dlrsn_step_collocation`` (include/dlrsn.h); ``"python"``
    orchestrates the same kernels from Python (kept as a cross-check and for
    the case the native call does not take: a pinned constant column).
    ``use_dsa=True`` (the reference default) runs inside the native call
    too: K6 (matrix-free Jacobi-PCG, one cooperative launch) after every
    sweep, skipped on the device once the iteration has converged.

    Host synchronisations: one before the source iteration (DEIM picks,
    closure weights and the input checks come back together), one per source
    iteration (convergence test) and one at the end (Gram-Schmidt guard,
    row-system status, angular deficiencies, output check).  Errors are raised
    in the reference's order (dlr_sn.py:99-141).

    ``inflow`` (an extension; the reference is vacuum-only,
    transport_sn.py:11-13): isotropic inflow intensities psi_b per wall, as
    ``{wall: psi_b}`` or (left, right, bottom, top).  The load
    |omega.n| psi_b (e2 row sums) on the wall edge dofs joins each selected
    direction's sweep rhs and, projected on X_new, its reduced row source
    (BASELINE config 3; restated in oracle/port.py ``inflow_load``).

    ``angle_indices`` (an extension) forces the DEIM selection (r node
    indices, in pick order) -- e.g. the reference's own picks for a basis
    with near-ties.  Otherwise each pick's relative top-2 residual gap is
    checked against ``deim_tie_tol`` (InterpolationTieError below it; 0
    disables) and reported as ``info.deim_gaps``.
    """
    if gs_method not in ("cholqr2", "cgs2"):
        raise ConfigurationError(f"unknown gs_method {gs_method!r}")
    if engine not in ("native", "python", "lean"):
        raise ConfigurationError(f"unknown engine {engine!r}")
    if engine == "lean":  # pure absorbers at config-5 size (lean.py)
        if use_dsa or inflow_values(inflow) is not None or comm is not None or _advance is not None \
                or gs_method != "cholqr2":
            raise ConfigurationError("the lean engine takes pure absorbers without DSA, inflow, "
                                     "sharding or the fused step boundary (CholQR2 only)")
        from .lean import step_lean

        return step_lean(grid, step, quad, state, si_tol=si_tol, si_max_iters=si_max_iters,
                         check_state=check_state, angle_indices=angle_indices,
                         deim_tie_tol=deim_tie_tol)
    if (engine == "native" and not state.W.pinned
            and state.rank <= _lib.MAX_RANK and (sweep_dw or 1) == 1
            and (comm is None or comm.world_size <= 8)):
        if dsa_penalty not in ("simplified", "collocation"):
            raise ContractViolation(f"unknown dsa penalty variant {dsa_penalty!r}")
        return _step_native(grid, step, quad, state, si_tol, si_max_iters, check_state,
                            gs_method, sweep_dw, comm, _advance, inflow_values(inflow),
                            angle_indices, deim_tie_tol, _x_new_host,
                            dsa=dsa_penalty if use_dsa else None)
    if inflow_values(inflow) is not None:
        raise ConfigurationError("inflow boundaries need the native engine")
    if _advance is not None:
        raise ConfigurationError("the fused step boundary needs the native engine")
    r = state.rank
    # ---- DEIM + closure + input checks: one readback ------------------------
    if angle_indices is not None:
        selection, err_idx = deim_forced_launch(state.W.values, angle_indices)
    else:
        selection, err_idx = deim_launch(state.W.values)
    closure = selection.closure_weights(state.W.beta)
    ops = assemble_operators(grid, step, dsa_penalty=dsa_penalty, validate=False)
    bad_sigma = (step.sigma_t - step.sigma_s <= 0).any().to(torch.float64).reshape(1)
    parts = [err_idx.to(torch.float64), closure, bad_sigma, selection.gap_dev]
    if check_state:
        parts.append(state.check_values(ops, quad))
    host = torch.cat(parts).cpu().numpy()
    deim_finish(selection, host[:r + 1], host[2 * r + 2:3 * r + 2])  # InterpolationError
    closure_host = host[r + 1:2 * r + 1].copy()
    if host[2 * r + 1]:                                        # transport_sn.py:208-209
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    if check_state:
        state.raise_check(host[3 * r + 2:])                    # lowrank.py:68-81
    if angle_indices is None:
        check_ties(selection.gaps, deim_tie_tol)
    omegas_sel = quad.omegas[selection.indices]
    if dsa_penalty == "collocation":
        ops.penalty_closure = (omegas_sel, closure_host)

    # ---- collocated source iteration (dlr_sn.py:110-121) ---------------------
    flux0 = evaluate_rows(state, selection)
    result = source_iteration(
        ops, omegas_sel, closure_host, psi_time=flux0.values, use_dsa=use_dsa, tol=si_tol,
        max_iters=si_max_iters, phi_start=state.scalar_flux(), threads=threads, dw=sweep_dw,
        comm=comm)

    # ---- Galerkin side, speculative CholQR2 (dlr_sn.py:123-141) --------------
    tail = _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result,
                          gs_method, check_state)
    if gs_method == "cholqr2" and not tail["gs_ok"]:
        tail = _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result,
                              "cgs2", check_state)
    new_state = tail["state"]
    info = CollocationStepInfo(
        iterations=result.iterations,
        selection=selection,
        angle_indices=selection.indices.copy(),
        phi=tail["phi"],
        spatial_deficiency=tail["sdef"],
        angular_deficiency=tail["adef"],
        si_phi=result.phi,
    )
    info.deim_gaps = selection.gaps
    return new_state, info


def _galerkin_tail(ops, step, quad, state, selection, closure, omegas_sel, result, gs_method,
                   check_state):
    r = state.rank
    co = _cellops_of(ops)
    if gs_method == "cholqr2":
        x_new, _, guard = cholqr2_speculative(co, result.psi)
        defi_x = status_x = None
    else:
        x_new, _, defi_x, status_x = cgs2_spatial_async(co, result.psi, r + 8, True)
        guard = None

    proj, packed = project_operators(ops, x_new, x_old=state.X)
    w_sel = state.W.values[selection.indices_dev]
    l_time = w_sel @ (state.S.T @ proj["mo"])
    q_all = (proj["q"][None, :] + step.inv_cdt * l_time).contiguous()
    om_sel = quad.omegas_device()[selection.indices_dev].contiguous()
    l_nodes, l_bar, row_status = _row_solve_async(r, r, packed, om_sel, proj["ms"].contiguous(),
                                                  q_all, closure)
    gamma = selection.interpolation_coefficients(l_nodes)
    l_full = rowmix(state.W.values, gamma)
    basis_new, r_ang, defi_w, status_w = orthonormalize_async(l_full, quad)
    new_state = DlrState(X=x_new, S=r_ang.T.contiguous(), W=basis_new)

    parts = [row_status.to(torch.float64), defi_w[:r].to(torch.float64),
             status_w.to(torch.float64)]
    if guard is not None:
        parts.append(guard)
    else:
        parts += [defi_x[:r].to(torch.float64), status_x.to(torch.float64)]
    if check_state:
        parts.append(new_state.check_values(ops, quad))
    host = torch.cat(parts).cpu().numpy()
    o = r + 1
    row_flags = host[:o]
    adef = host[o:o + r]
    st_w = host[o + r]
    o += r + 1
    if guard is not None:
        gs_ok = cholqr_guard_ok(host[o:o + 2 * r + 1], r)
        o += 2 * r + 1
        if not gs_ok:
            return {"gs_ok": False}
        sdef = 0
    else:
        sdef = len(_cgs2_flags(host[o:o + r], host[o + r:o + r + 1], r))
        o += r + 1
    raise_row_status(row_flags, r)                             # SolverError
    _cgs2_flags(adef, [st_w], r)                               # ContractViolation
    if check_state:
        new_state.raise_check(host[o:])
    return {"gs_ok": True, "state": new_state, "sdef": sdef,
            "adef": int(np.count_nonzero(adef)),
            "phi": rowmix(x_new, l_bar.reshape(-1, 1))[:, 0]}


# ---- native engine: the whole step in one C-ABI call ------------------------

class _NativeSelection:
    """DEIM picks of a native step (indices on the host; W_hat = W[idx] for
    the condition number, lowrank.py:204)."""

    def __init__(self, indices, w_values):
        self.indices = indices
        self._w = w_values

    @property
    def rank(self):
        return len(self.indices)

    @cached_property
    def indices_dev(self):
        return torch.as_tensor(self.indices, device=device())

    @cached_property
    def w_hat(self):
        return self._w[self.indices_dev]

    @cached_property
    def cond(self):
        return float(torch.linalg.cond(self.w_hat))


_STEP_WS = {}
_DSA_HIST = 4096
_DSA_MAX_ITERS = 0  # PCG cap of the native step (0: the reference's 10 n_dofs)


def release_workspaces():
    """Drop the cached per-problem step workspaces, native contexts and sweep
    workspaces (e.g. before a config-5 step that needs most of HBM)."""
    from . import transport

    _STEP_WS.clear()
    _CTX.clear()
    _HOOKS.clear()
    transport._WS_CACHE.clear()
    torch.cuda.empty_cache()


def _grid_cellops(grid):
    co = grid.__dict__.get("_cellops")
    if co is None:
        from .mesh import cellops_struct

        co = cellops_struct(grid)
        object.__setattr__(grid, "_cellops", co)
    return co


def _step_workspace(grid, r, no, world, rank):
    key = (torch.cuda.current_device(), grid.nx, grid.ny, r, no, world, rank)
    ws = _STEP_WS.get(key)
    if ws is None:
        nbytes = int(_lib.load().dlrsn_step_workspace_bytes(grid.nx, grid.ny, r, no, world))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device())
        _STEP_WS[key] = ws
    return ws


class _CommHooks:
    """C callbacks of dlrsn_comm over a DirectionComm-like object (anything
    with ``allreduce_sum_``; ``allgather_into_`` when it has one, else the
    gather is an allreduce of zero-padded blocks, which is exact)."""

    def __init__(self, comm, n, width):
        self.comm = comm
        self.n, self.width = n, width
        self.reduce_buf = empty(n)
        self.send = empty(n, width)
        self.recv = empty(comm.world_size, n, width)
        self.error = None
        self._ar = _lib.COMM_FN(self._allreduce)
        self._ag = _lib.COMM_FN(self._allgather)
        s = _lib.Comm()
        s.rank, s.world_size = comm.rank, comm.world_size
        s.user = None
        s.allreduce_sum, s.allgather = self._ar, self._ag
        s.reduce_buf = self.reduce_buf.data_ptr()
        s.gather_send = self.send.data_ptr()
        s.gather_recv = self.recv.data_ptr()
        s.gather_width = width
        self.struct = s

    def _allreduce(self, _user):
        try:
            self.comm.allreduce_sum_(self.reduce_buf)
            return 0
        except Exception as e:  # surfaced after the C call returns
            self.error = e
            return 1

    def _allgather(self, _user):
        try:
            if hasattr(self.comm, "allgather_into_"):
                self.comm.allgather_into_(self.recv, self.send)
            else:
                self.recv.zero_()
                self.recv[self.comm.rank].copy_(self.send)
                self.comm.allreduce_sum_(self.recv)
            return 0
        except Exception as e:
            self.error = e
            return 1


_HOOKS = {}


def _comm_hooks(comm, n, r):
    width = -(-r // comm.world_size) + 1
    key = (id(comm), comm.rank, n, width)
    h = _HOOKS.get(key)
    if h is None or h.comm is not comm:
        h = _CommHooks(comm, n, width)
        _HOOKS[key] = h
    return h


class _NativeCtx:
    """Per-(grid, quadrature, rank, sharding) state of the native step: the
    cellops struct, the parameter block, the step and sweep workspaces and
    the collective hooks, built once and reused by every step."""

    def __init__(self, grid, quad, r, comm):
        from .transport import _shared_workspace

        lib = _lib.load()
        self.grid, self.quad, self.comm = grid, quad, comm
        world = comm.world_size if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        self.co = _grid_cellops(grid)
        self.co_ptr = _addr(self.co)
        self.ws = _step_workspace(grid, r, quad.n_angles, world, rank)
        sw_bytes = int(lib.dlrsn_sweep_workspace_bytes(grid.nx, grid.ny, r, 1))
        self.sws = _shared_workspace(grid, sw_bytes)
        self.om_host = np.ascontiguousarray(quad.omegas, dtype=np.float64)
        p = _lib.StepParams()
        p.rank, p.n_omega = r, quad.n_angles
        p.omegas_host = self.om_host.ctypes.data
        p.omegas_dev = quad.omegas_device().data_ptr()
        p.weights_dev = quad.weights_device().data_ptr()
        p.sweep_dw = 1
        self.params = p
        self.params_ref = ctypes.byref(p)
        self.hooks = _comm_hooks(comm, grid.n_dofs, r) if world > 1 else None
        self.comm_ref = ctypes.byref(self.hooks.struct) if self.hooks else None
        n, no = grid.n_dofs, quad.n_angles
        # output block: X_new | S_new | W_new | beta_new | phi | si_phi, each
        # segment padded to an even length (16-byte aligned rows for X)
        sizes = [n * r, r * r, no * r, r, n, n]
        offs, o = [], 0
        for z in sizes:
            offs.append(o)
            o += z + (z & 1)
        self.x_slot = o  # spatial check of X_new (dlrsn_step_params.x_check_out)
        self.out_len, self.offs = o + 2, offs
        self.shapes = [(n, r), (r, r), (no, r), (r,), (n,), (n,)]
        self.strides = [(r, 1), (r, 1), (r, 1), (1,), (1,), (1,)]
        self.fn = lib.dlrsn_step_collocation
        # source iterations enqueued before the first readback: per problem,
        # so every rank of a sharded run (same steps, same ctx history) agrees
        self.si_hint = 0
        self.dsa_hist = None  # PCG residual history (device), allocated on first DSA step


_CTX = {}


def _native_ctx(grid, quad, r, comm):
    key = (id(grid), id(quad), r, id(comm), torch.cuda.current_device())
    ctx = _CTX.get(key)
    if ctx is None or ctx.grid is not grid or ctx.quad is not quad or ctx.comm is not comm:
        if len(_CTX) > 64:
            _CTX.clear()
        ctx = _NativeCtx(grid, quad, r, comm)
        _CTX[key] = ctx
    return ctx


def _step_native(grid, step, quad, state, si_tol, si_max_iters, check_state, gs_method, sweep_dw,
                 comm, advance=None, inflow=None, angle_indices=None, deim_tie_tol=DEIM_TIE_TOL,
                 x_new_host=None, dsa=None):
    r = state.rank
    no = quad.n_angles
    n = grid.n_dofs
    for name in ("sigma_t", "sigma_s", "q"):
        if getattr(step, name).shape[0] != grid.n_cells:
            raise ContractViolation(f"step field {name} must be per-cell")
    if tuple(state.W.values.shape) != (no, r) or tuple(state.X.shape) != (n, r):
        raise ContractViolation("factor shapes do not match the grid / quadrature")
    ctx = _native_ctx(grid, quad, r, comm if comm is not None and comm.world_size > 1 else None)
    X = state.X.contiguous()
    S = state.S.contiguous()
    W = state.W.values.contiguous()
    beta = state.W.beta if state.W.beta is not None else state.W.bind(quad).beta
    beta = beta.contiguous()
    out = torch.empty(ctx.out_len, dtype=torch.float64, device=X.device)
    X_new, S_new, W_new, beta_new, phi, si_phi = (
        out.as_strided(sh, st, o) for sh, st, o in zip(ctx.shapes, ctx.strides, ctx.offs))
    p = ctx.params
    p.inv_cdt = float(step.inv_cdt)
    p.si_tol, p.si_max_iters = float(si_tol), int(si_max_iters)
    p.check_state = 1 if check_state else 0
    p.gs_method = 0 if gs_method == "cholqr2" else 1
    p.advance = ctypes.addressof(advance) if advance is not None else None
    p.inflow[:] = inflow if inflow is not None else (0.0, 0.0, 0.0, 0.0)
    p.si_batch_hint = ctx.si_hint
    # DSA inside the call (K6 per source iteration, no host round trips)
    p.use_dsa = 0 if dsa is None else 1
    p.dsa_penalty = 1 if dsa == "collocation" else 0
    p.dsa_tol, p.dsa_max_iters = 0.0, int(_DSA_MAX_ITERS)  # 0: the reference's pcg defaults
    if dsa is not None:
        if ctx.dsa_hist is None:
            ctx.dsa_hist = torch.zeros(_DSA_HIST, dtype=torch.float64, device=X.device)
        p.dsa_history, p.dsa_hist_cap = ctx.dsa_hist.data_ptr(), _DSA_HIST
    else:
        p.dsa_history, p.dsa_hist_cap = None, 0
    if x_new_host is not None:
        if (not x_new_host.is_pinned() or x_new_host.dtype != torch.float64
                or tuple(x_new_host.shape) != (n, r) or not x_new_host.is_contiguous()):
            raise ContractViolation("x_new_host must be a contiguous pinned fp64 (n_dofs, r) tensor")
        p.x_new_host = x_new_host.data_ptr()
    else:
        p.x_new_host = None
    forced = None
    if angle_indices is not None:
        forced = np.ascontiguousarray(angle_indices, dtype=np.int64).reshape(-1)
        if forced.shape != (r,):
            raise ContractViolation(f"angle_indices must hold {r} node indices")
        p.angle_override, p.angle_indices_in = 1, forced.ctypes.data
    else:
        p.angle_override, p.angle_indices_in = 0, None
    # DlrState.check of an X this library produced and already checked (same
    # tensor, not modified since): the input Gram is not recomputed
    xc = getattr(state, "_xcheck", None)
    known = (check_state and xc is not None and xc[1] is state.X
             and xc[2] == state.X._version and X is state.X)
    p.x_check_in = xc[0].data_ptr() if known else None
    slot = out[ctx.x_slot:ctx.x_slot + 1]
    p.x_check_out = slot.data_ptr() if check_state else None
    info = _lib.StepInfo()
    hooks = ctx.hooks
    if hooks is not None:
        hooks.error = None
    ob = out.data_ptr()
    rc = ctx.fn(
        ctx.co_ptr, ctx.params_ref, X.data_ptr(), S.data_ptr(), W.data_ptr(), beta.data_ptr(),
        step.sigma_t.data_ptr(), step.sigma_s.data_ptr(), step.q.data_ptr(),
        ob + 8 * ctx.offs[0], ob + 8 * ctx.offs[1], ob + 8 * ctx.offs[2], ob + 8 * ctx.offs[3],
        ob + 8 * ctx.offs[4], ob + 8 * ctx.offs[5], ctx.ws.data_ptr(), ctx.ws.numel(),
        ctx.sws.data_ptr(), ctx.sws.numel(), ctx.comm_ref, ctypes.byref(info), stream())
    p.angle_override, p.angle_indices_in = 0, None
    p.x_new_host = None
    if rc == 0 or rc == -7:
        ctx.si_hint = max(ctx.si_hint, int(info.si_batch_hint))
    if hooks is not None and hooks.error is not None:
        raise hooks.error
    if rc != 0:
        lib = _lib.load()
        msg = lib.dlrsn_last_error().decode(errors="replace")
        if rc == -5:
            raise InterpolationError("interpolation residual vanished; basis is rank deficient",
                                     column=int(info.error_index))
        if rc == -7:
            raise IterationLimitError("source iteration did not converge", int(info.iterations),
                                      float(info.residual))
        if rc == -8:  # transport_sn.py:350
            cap = int(info.iterations)
            hist = ctx.dsa_hist[:min(cap + 1, _DSA_HIST)].cpu().numpy().tolist()
            raise CgError("dsa failed to reach tol 1e-10", cap, hist)
        if rc in (-2, -3):
            raise SolverError(msg)
        if rc in (-1, -6):
            raise ContractViolation(msg)
        raise RuntimeError(f"dlrsn CUDA failure ({rc}): {msg}")
    indices = np.frombuffer(info.angle_indices, dtype=np.int64, count=r).copy()
    gaps = np.frombuffer(info.deim_gap, dtype=np.float64, count=r).copy()
    if forced is None:
        try:
            check_ties(gaps, deim_tie_tol)
        except InterpolationError:
            import os
            import sys

            if os.environ.get("DLRSN_TIE_DEBUG"):
                w0 = W[:, 0].abs()
                top = torch.topk(w0, 3)
                print(f"dlrsn tie: gaps {gaps.tolist()} picks {indices.tolist()} |W[:,0]| top "
                      f"{top.values.tolist()} rows {top.indices.tolist()} it {info.iterations} "
                      f"X {X.data_ptr():#x} W {W.data_ptr():#x} out {ob:#x}", file=sys.stderr)
            raise
    basis = AngularBasis(values=W_new, beta=beta_new)
    new_state = DlrState(X=X_new, S=S_new, W=basis)
    if check_state:
        new_state._xcheck = (slot, X_new, X_new._version)
    res = CollocationStepInfo(
        iterations=int(info.iterations),
        selection=_NativeSelection(indices, W),
        angle_indices=indices.copy(),
        phi=phi,
        spatial_deficiency=int(info.spatial_deficiency),
        angular_deficiency=int(info.angular_deficiency),
        si_phi=si_phi,
    )
    res.gs_fallback = int(info.gs_fallback)
    res.deim_gaps = gaps
    if dsa is not None:
        res.dsa_iterations = int(info.dsa_iterations)
        res.dsa_solves = int(info.dsa_solves)
    return new_state, res
