"""Row-slab ("Option B" of SURVEY 8e) DLR-SN step over P ranks, for pure
absorbers (BASELINE config 5: sigma_s = 0, one sweep per step).

Direction sharding alone ("Option A", sharding.py) leaves the Galerkin side
of the step -- CholQR2, the projections, the Grams: ~95 % of a config-5 step
-- replicated on every rank.  Here the spatial factor is sharded by grid
rows: rank p owns the dof rows of the cell rows [j0_p, j1_p) of X, Psi and
X_new, and

1. DEIM, the closure weights and every r x r / N_Omega x r computation run
   replicated (deterministic kernels: identical results on all ranks);
2. psi_time = X (S W_sel^T) (lowrank.py:220-227) is formed on each slab for
   all directions, and one all-to-all hands rank q the columns of its
   directions (its sweep share, sharding.partition_directions) over all
   rows;
3. each rank sweeps its directions over the whole grid (K1; sigma_t and q of
   all cells are replicated inputs) and a second all-to-all returns the
   swept columns to the slabs, in selection order;
4. CholQR2 in the M inner product runs slab-locally with r x r all-reduced
   Grams (the guard decision is taken from the summed Gram, so all ranks
   agree); a failed guard runs the reference's exact CGS2 column by column
   with all-reduced inner products (same deficiency / completion rules);
5. the fused projections (K3, dlrsn_project_slab) run on each slab with the
   cell row below as a halo for the horizontal faces (one point-to-point
   exchange) and are all-reduced (7 r^2 + r doubles);
6. the T update is slab-local.

Collectives are yielded by a per-rank generator as request objects, so the
same step code runs (a) as P virtual ranks in one process -- ``run_local``,
lock-step, used by the tests on one GPU: no kernel of one rank waits on
another's -- and (b) on a torch.distributed group (NCCL over NVLink between
GPUs, gloo on CPU) -- ``run_dist``.  Sums over ranks are taken in rank order
(fixed for a fixed P), so results differ from the unsharded step only by
summation order.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import as_device, empty, stream, zeros
from .angular import orthonormalize_async
from .errors import ConfigurationError, ContractViolation, InterpolationError, SolverError
from .lowrank import (
    DlrState,
    _chol,
    _row_solve_async,
    _cgs2_flags,
    check_ties,
    cholqr_guard_ok,
    deim_finish,
    deim_launch,
    mass_gram,
    raise_row_status,
    rowmix,
    spatial_monomial_exponents,
)
from .mesh import build_grid, dof_coordinates
from .sharding import partition_directions
from .transport import _SweepPlan, _sweep, assemble_operators, raise_sweep_status, sweep_status_word

FOUR_PI = 4.0 * np.pi
DEFICIENCY_TOL = 1e-12  # angular.py:24


# ---- collectives as requests ----------------------------------------------

@dataclass
class AllReduce:
    """Sum ``t`` over ranks in place (rank order)."""

    t: torch.Tensor


@dataclass
class AllToAll:
    """send[q] goes to rank q; recv[q] receives rank q's send[me] (shapes
    agreed beforehand)."""

    send: list
    recv: list


def run_local(P, make_rank):
    """Run P virtual ranks in one process, in lock step: ``make_rank(p)``
    returns rank p's generator; each yields collective requests and returns
    its result.  Every rank must yield the same sequence of request kinds."""
    gens = [make_rank(p) for p in range(P)]
    reqs = [None] * P
    out = [None] * P
    done = [False] * P
    for p, g in enumerate(gens):
        try:
            reqs[p] = next(g)
        except StopIteration as e:
            done[p], out[p] = True, e.value
    while not all(done):
        if any(done):
            raise RuntimeError("virtual ranks diverged (one finished early)")
        kinds = {type(r) for r in reqs}
        if len(kinds) != 1:
            raise RuntimeError(f"virtual ranks diverged: {kinds}")
        if isinstance(reqs[0], AllReduce):
            total = reqs[0].t.clone()
            for r in reqs[1:]:
                total += r.t
            for r in reqs:
                r.t.copy_(total)
        elif isinstance(reqs[0], AllToAll):
            for p in range(P):
                for q in range(P):
                    reqs[q].recv[p].copy_(reqs[p].send[q])
        else:
            raise RuntimeError(f"unknown request {reqs[0]!r}")
        for p, g in enumerate(gens):
            try:
                reqs[p] = g.send(None)
            except StopIteration as e:
                done[p], out[p] = True, e.value
    return out


def run_dist(gen, group=None):
    """Drive one rank's generator on a torch.distributed group (NCCL / gloo)."""
    import torch.distributed as dist

    try:
        req = next(gen)
        while True:
            if isinstance(req, AllReduce):
                dist.all_reduce(req.t, op=dist.ReduceOp.SUM, group=group)
            elif isinstance(req, AllToAll):
                me = dist.get_rank(group)
                ops = []
                for q, (s, r) in enumerate(zip(req.send, req.recv)):
                    if q == me:
                        r.copy_(s)
                        continue
                    if s.numel():
                        ops.append(dist.P2POp(dist.isend, s.contiguous(), q, group))
                    if r.numel():
                        ops.append(dist.P2POp(dist.irecv, r, q, group))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
            else:
                raise RuntimeError(f"unknown request {req!r}")
            req = gen.send(None)
    except StopIteration as e:
        return e.value


# ---- the slab decomposition -----------------------------------------------

def slab_rows(ny, P):
    """Contiguous cell-row ranges [j0, j1) per rank, sizes differing by <= 1."""
    base, extra = divmod(ny, P)
    out, j = [], 0
    for p in range(P):
        k = base + (1 if p < extra else 0)
        out.append((j, j + k))
        j += k
    return out


@dataclass(eq=False)
class Slab:
    """Rank p's part of a grid: rows [j0, j1), its own grid object (the cell
    geometry of those rows) and the dof row range in the full grid."""

    rank: int
    P: int
    grid: object         # full grid
    rows: list           # (j0, j1) of every rank
    sgrid: object = None
    d0: int = 0
    d1: int = 0

    def __post_init__(self):
        j0, j1 = self.rows[self.rank]
        g = self.grid
        self.sgrid = build_grid(g.nx, j1 - j0, (g.x0, g.y0 + j0 * g.dy, g.nx * g.dx,
                                                (j1 - j0) * g.dy))
        self.d0, self.d1 = 4 * j0 * g.nx, 4 * j1 * g.nx

    def dof_range(self, q):
        j0, j1 = self.rows[q]
        return 4 * j0 * self.grid.nx, 4 * j1 * self.grid.nx

    def cell_range(self, q):
        j0, j1 = self.rows[q]
        return j0 * self.grid.nx, j1 * self.grid.nx


# ---- the three exchanges of a slab step (device-agnostic torch code, so the
# protocol is tested with gloo on CPU: tests/test_slab_protocol.py) --------

def rows_to_direction_columns(Y, owners, slab):
    """Generator: Y = this slab's rows (N_p x r) of a matrix whose columns are
    the selected directions; returns the FULL rows (N x |owners[me]|) of my
    directions' columns (one all-to-all)."""
    P, me = slab.P, slab.rank
    send = [Y[:, torch.as_tensor(owners[q], device=Y.device, dtype=torch.long)].contiguous()
            for q in range(P)]
    recv = [torch.empty(slab.dof_range(q)[1] - slab.dof_range(q)[0], len(owners[me]),
                        dtype=Y.dtype, device=Y.device) for q in range(P)]
    yield AllToAll(send, recv)
    return torch.cat(recv, dim=0)


def direction_columns_to_rows(C, owners, slab, r):
    """Generator: C = FULL rows (N x |owners[me]|) of my directions' columns;
    returns this slab's rows (N_p x r) of all columns in selection order."""
    P, me = slab.P, slab.rank
    send = [C[slice(*slab.dof_range(q))].contiguous() for q in range(P)]
    recv = [torch.empty(slab.d1 - slab.d0, len(owners[q]), dtype=C.dtype, device=C.device)
            for q in range(P)]
    yield AllToAll(send, recv)
    out = torch.empty(slab.d1 - slab.d0, r, dtype=C.dtype, device=C.device)
    for q in range(P):
        if len(owners[q]):
            out[:, torch.as_tensor(owners[q], device=C.device, dtype=torch.long)] = recv[q]
    return out


def halo_below(X, slab):
    """Generator: the X rows of the cell row just below my slab (from the
    rank below; None on the bottom slab).  My top row goes up."""
    P, me = slab.P, slab.rank
    nxr = 4 * slab.grid.nx
    r = X.shape[1]
    mk = lambda k: torch.empty(k, r, dtype=X.dtype, device=X.device)  # noqa: E731
    send = [mk(0) for _ in range(P)]
    recv = [mk(0) for _ in range(P)]
    halo = mk(nxr) if me > 0 else None
    if me + 1 < P:
        send[me + 1] = X[-nxr:].contiguous()
    if me > 0:
        recv[me - 1] = halo
    yield AllToAll(send, recv)
    return halo


def split_state(state, slab):
    """Rank's share of a full state: X rows of its slab (a copy), S, W."""
    return DlrState(X=state.X[slab.d0:slab.d1].contiguous(), S=state.S, W=state.W)


def _slab_step_fields(step, slab):
    """LinearizedStep restricted to the slab's cells (views)."""
    from .physics import LinearizedStep

    c0, c1 = slab.cell_range(slab.rank)
    return LinearizedStep(sigma_t=step.sigma_t[c0:c1], sigma_s=step.sigma_s[c0:c1],
                          sigma_a=step.sigma_a[c0:c1], q=step.q[c0:c1], T0=step.T0[c0:c1],
                          denom=step.denom[c0:c1], rho_cv=step.rho_cv[c0:c1], dt=step.dt,
                          inv_cdt=step.inv_cdt, constants=step.constants)


def step_slab(slab, step, quad, state, *, check_state=True, chunk=16, deim_tie_tol=1e-12,
              si_tol=1e-8, si_max_iters=200):
    """Generator: rank ``slab.rank``'s part of one DLR step (dlr_sn.py:86-151)
    on row slabs.  ``step`` holds the FULL per-cell fields (replicated),
    ``state`` the rank's slab rows of X with the replicated S and W.  With
    sigma_s = 0 one chunked in-place sweep; else the source iteration with
    the closure flux all-reduced every iteration.  Returns (new slab state,
    info dict)."""
    from .dlr_sn import project_operators  # noqa: F401 (documentation link)

    P, me = slab.P, slab.rank
    grid = slab.grid
    r = state.rank
    X, S, W = state.X, state.S, state.W.values
    beta = state.W.beta if state.W.beta is not None else state.W.bind(quad).beta
    ops = assemble_operators(grid, step, validate=False)  # full grid: the sweep
    sstep = _slab_step_fields(step, slab)
    sops = assemble_operators(slab.sgrid, sstep, validate=False)  # slab: Grams, K3
    # ---- 1. DEIM, closure, checks -----------------------------------------
    sel, err_idx = deim_launch(W)
    closure = sel.closure_weights(beta)
    st = ops.step
    flags = torch.stack([(st.sigma_t - st.sigma_s <= 0).any(), (st.sigma_s != 0).any()])
    parts = [err_idx.to(torch.float64), closure, flags.to(torch.float64), sel.gap_dev]
    gx = None
    if check_state:
        gx = mass_gram(sops, X)
        yield AllReduce(gx)
        eye = torch.eye(r, dtype=torch.float64, device=X.device)
        wq = quad.weights_device()
        gw = (W * wq[:, None]).T @ W
        parts.append(torch.stack([(gx - eye).abs().max(), (gw - eye).abs().max()]))
    host = torch.cat(parts).cpu().numpy()
    deim_finish(sel, host[:r + 1], host[2 * r + 3:3 * r + 3])
    cw = host[r + 1:2 * r + 1].copy()
    if host[2 * r + 1]:
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    pure = not host[2 * r + 2]  # sigma_s == 0: one sweep (transport_sn.py:410)
    if check_state:
        rx, rw = float(host[3 * r + 3]), float(host[3 * r + 4])
        if rx > 1e-10 or rw > 1e-10:
            raise ContractViolation(f"factor orthonormality violated: spatial {rx:.2e}, "
                                    f"angular {rw:.2e}")
    check_ties(sel.gaps, deim_tie_tol)
    om_sel = quad.omegas[sel.indices]
    owners = partition_directions(om_sel, P)  # sweep shares, selection positions
    mine = owners[me]
    # ---- 2. psi_time columns of my directions over all rows ---------------
    K = S @ W[sel.indices_dev].T
    Y = rowmix(X, K)  # (N_p, r): this slab's rows of psi_time for every direction
    pt = yield from rows_to_direction_columns(Y, owners, slab)  # (N, |mine|)
    del Y
    # ---- 3. sweep my directions over the whole grid -----------------------
    n = grid.n_dofs
    if pure:  # one sweep, in place, chunked (transport_sn.py:410,430-432)
        psi_mine = empty(n, len(mine))
        vl = ops.vec_len
        for c0 in range(0, len(mine), chunk):
            c1 = min(len(mine), c0 + chunk)
            D = c1 - c0
            cols = pt[:, c0:c1].contiguous()
            plan = _SweepPlan(ops, om_sel[mine[c0:c1]], cw[mine[c0:c1]], dw=1)
            sk = empty(D * vl)
            _lib.call("dlrsn_rhs_build", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev),
                      _lib.ptr(st.q), float(st.inv_cdt), _lib.ptr(cols), D, None, 1, _lib.ptr(sk),
                      stream())
            _sweep(ops, plan, sk, sk)
            _lib.call("dlrsn_sk_to_canonical", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev),
                      _lib.ptr(sk), ctypes.c_void_p(psi_mine.data_ptr() + 8 * c0), len(mine),
                      stream())
            raise_sweep_status(sweep_status_word(plan.workspace).item(), plan.workspace)
            del sk, cols
        iters = 1
    else:
        psi_mine, iters = yield from _source_iteration_slabs(ops, slab, om_sel, cw, mine, pt, X,
                                                            S, beta, si_tol, si_max_iters)
    del pt
    # ---- 4. swept columns back to the slabs, selection order ---------------
    psi = yield from direction_columns_to_rows(psi_mine, owners, slab, r)
    del psi_mine
    # ---- 5. K2: CholQR2 with all-reduced Grams (exact CGS2 if the guard fails)
    G1 = mass_gram(sops, psi)
    yield AllReduce(G1)
    R1, R1inv, ratio, flag = _chol(G1)
    guard = torch.cat([ratio, flag.to(torch.float64)]).cpu().numpy()
    sdef = 0
    fallback = not cholqr_guard_ok(guard, r)
    if not fallback:
        psi = rowmix(psi, R1inv)
        G2 = mass_gram(sops, psi)
        yield AllReduce(G2)
        _, R2inv, _, flag2 = _chol(G2)
        if int(flag2.item()):
            raise SolverError("second CholQR pass lost positive definiteness")
        x_new = rowmix(psi, R2inv)
        del psi
    else:
        x_new, sdef = yield from _cgs2_slabs(sops, psi, r, slab)
    # ---- 6. K3 on the slab with the halo row below, all-reduced -----------
    halo = yield from halo_below(x_new, slab)  # my top row is the next slab's halo
    out = empty(7 * r * r + r)
    part = empty(max(int(_lib.load().dlrsn_partials_len(slab.sgrid.n_cells, r, r, 1)), 1))
    _lib.call("dlrsn_project_slab", sops.cellops_ptr, r, _lib.ptr(x_new), _lib.ptr(X),
              _lib.ptr(halo), 1 if me == P - 1 else 0, _lib.ptr(sstep.sigma_t),
              _lib.ptr(sstep.sigma_s), _lib.ptr(sstep.q), _lib.ptr(out), _lib.ptr(part), stream())
    yield AllReduce(out)
    mats = out[:7 * r * r].reshape(7, r, r)
    proj = {k: mats[i] for i, k in enumerate(("px", "py", "jx", "jy", "mt", "ms", "mo"))}
    proj["q"] = out[7 * r * r:]
    # ---- 7. reduced rows, angular update: replicated (dlr_sn.py:126-141) --
    w_sel = W[sel.indices_dev]
    q_all = (proj["q"][None, :] + st.inv_cdt * (w_sel @ (S.T @ proj["mo"]))).contiguous()
    om_dev = quad.omegas_device()[sel.indices_dev].contiguous()
    l_nodes, l_bar, row_status = _row_solve_async(r, r, out, om_dev, proj["ms"].contiguous(),
                                                  q_all, closure)
    gamma = sel.interpolation_coefficients(l_nodes)
    basis_new, r_ang, defi_w, status_w = orthonormalize_async(rowmix(W, gamma), quad)
    new_state = DlrState(X=x_new, S=r_ang.T.contiguous(), W=basis_new)
    parts = [row_status.to(torch.float64), defi_w[:r].to(torch.float64),
             status_w.to(torch.float64)]
    if check_state:
        gx = mass_gram(sops, x_new)
        yield AllReduce(gx)
        eye = torch.eye(r, dtype=torch.float64, device=x_new.device)
        wq = quad.weights_device()
        Wn = basis_new.values
        parts.append(torch.stack([(gx - eye).abs().max(), ((Wn * wq[:, None]).T @ Wn - eye)
                                  .abs().max()]))
    host = torch.cat(parts).cpu().numpy()
    raise_row_status(host[:r + 1], r)
    adef = host[r + 1:2 * r + 1]
    _cgs2_flags(adef, [host[2 * r + 1]], r)
    if check_state:
        rx, rw = float(host[2 * r + 2]), float(host[2 * r + 3])
        if rx > 1e-10 or rw > 1e-10:
            raise ContractViolation(f"factor orthonormality violated: spatial {rx:.2e}, "
                                    f"angular {rw:.2e}")
    phi = rowmix(x_new, l_bar.reshape(-1, 1))[:, 0]  # slab rows of info.phi
    info = {"angle_indices": sel.indices.copy(), "iterations": iters, "phi": phi,
            "spatial_deficiency": sdef, "angular_deficiency": int(np.count_nonzero(adef)),
            "selection": sel, "deim_gaps": sel.gaps, "gs_fallback": int(fallback)}
    return new_state, info


def _source_iteration_slabs(ops, slab, om_sel, cw, mine, pt, X, S, beta, tol, max_iters):
    """Generator: the collocated source iteration (transport_sn.py:377-450)
    with my directions swept over the whole grid and the closure flux
    all-reduced each iteration (N_x doubles); the norms and the next
    scattering source come from the summed flux, so every rank takes the
    same convergence decision.  The starting flux phi_start = X S beta
    (lowrank.py:60-62) is assembled from the slabs.  Returns (psi of my
    directions, N_x x |mine|; iterations)."""
    import math

    from .errors import IterationLimitError

    g = ops.grid
    st = ops.step
    n = g.n_dofs
    phi = torch.zeros(n, dtype=torch.float64, device=X.device)
    phi[slab.d0:slab.d1] = rowmix(X, (S @ beta).reshape(-1, 1))[:, 0]
    yield AllReduce(phi)  # the slabs' rows of phi_start, every rank holds all
    vl = ops.vec_len
    D = len(mine)
    plan = _SweepPlan(ops, om_sel[mine], cw[mine], dw=1) if D else None
    rhs_sk = empty(max(D, 1) * vl)
    psi_sk = empty(max(D, 1) * vl)
    if D:
        cols = pt.contiguous()
        _lib.call("dlrsn_rhs_build", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev), _lib.ptr(st.q),
                  float(st.inv_cdt), _lib.ptr(cols), D, None, 1, _lib.ptr(rhs_sk), stream())
        del cols
    scat = empty(4 * vl)
    flags = zeros(1, dtype=torch.int32)
    _lib.call("dlrsn_scatter_source", ops.cellops_ptr, _lib.ptr(phi), _lib.ptr(st.sigma_s),
              _lib.ptr(scat), _lib.ptr(flags), stream())
    phi_new = empty(n)
    nb = (g.n_cells + 255) // 256
    red_ws = zeros(256 // 8 + 2 * nb + 8)
    norms = zeros(2)
    change = math.inf
    for it in range(1, max_iters + 1):
        if D:
            _sweep(ops, plan, rhs_sk, psi_sk, scat, None)
            _lib.call("dlrsn_phi_combine", ops.cellops_ptr, plan.G, _lib.ptr(plan.groups_dev), None,
                      _lib.ptr(psi_sk), _lib.ptr(phi), _lib.ptr(st.sigma_s), _lib.ptr(phi_new),
                      None, _lib.ptr(norms), _lib.ptr(red_ws), stream())
        else:
            phi_new.zero_()
        yield AllReduce(phi_new)
        _lib.call("dlrsn_phi_finish", ops.cellops_ptr, _lib.ptr(phi_new), _lib.ptr(phi),
                  _lib.ptr(st.sigma_s), _lib.ptr(scat), _lib.ptr(norms), _lib.ptr(red_ws), stream())
        host = norms.cpu().numpy()
        if D:
            raise_sweep_status(sweep_status_word(plan.workspace).item(), plan.workspace)
        phi, phi_new = phi_new, phi
        change = math.sqrt(host[0]) / max(math.sqrt(host[1]), 1e-300)
        if change <= tol:
            psi_mine = empty(n, D)
            if D:
                _lib.call("dlrsn_sk_to_canonical", ops.cellops_ptr, D, _lib.ptr(plan.quads_dev),
                          _lib.ptr(psi_sk), _lib.ptr(psi_mine), D, stream())
            return psi_mine, it
    raise IterationLimitError("source iteration did not converge", max_iters, change)


def _cgs2_slabs(sops, cols, m, slab, strict=True):
    """The reference's twice-projected classical Gram-Schmidt in the M inner
    product (angular.py:104-160, completion = spatial monomials,
    lowrank.py:28-40) on row slabs: every inner product is a slab Gram
    (dlrsn_mgram) all-reduced over the ranks, every update a slab rowmix.
    Column k is replaced by q_k in place.  Returns (Q, deficient count)."""
    Q = cols
    tol = DEFICIENCY_TOL
    exps = spatial_monomial_exponents(m + 8)
    coords = None
    next_cand = 0
    ndef = 0

    def mnorm2(v):
        g = mass_gram(sops, v, v)
        return g

    def project_twice(v, k):
        for _ in range(2):
            if k == 0:
                return v
            c = mass_gram(sops, Q[:, :k], v)  # (k, 1) slab part
            yield AllReduce(c)
            v = rowmix(Q[:, :k], -c, out=v.clone(), beta=1.0)  # v - Q c
        return v

    for k in range(m):
        v = Q[:, k:k + 1].contiguous()
        g0 = mnorm2(v)
        yield AllReduce(g0)
        orig = float(g0.item()) ** 0.5 if float(g0.item()) > 0 else 0.0
        v = yield from project_twice(v, k)
        g1 = mnorm2(v)
        yield AllReduce(g1)
        nrm = max(float(g1.item()), 0.0) ** 0.5
        if nrm <= tol * max(orig, 1.0):
            ndef += 1
            placed = False
            while next_cand < len(exps):
                a, b = exps[next_cand]
                next_cand += 1
                if coords is None:
                    g = sops.grid
                    xy = torch.as_tensor(dof_coordinates(g), device=Q.device)
                    full = slab.grid
                    xh = 2.0 * (xy[:, 0] - full.x0) / (full.nx * full.dx) - 1.0
                    yh = 2.0 * (xy[:, 1] - full.y0) / (full.ny * full.dy) - 1.0
                    coords = (xh, yh)
                cand = (coords[0] ** a * coords[1] ** b).reshape(-1, 1).contiguous()
                gc = mnorm2(cand)
                yield AllReduce(gc)
                c0 = max(float(gc.item()), 0.0) ** 0.5
                cand = yield from project_twice(cand, k)
                gc1 = mnorm2(cand)
                yield AllReduce(gc1)
                cn = max(float(gc1.item()), 0.0) ** 0.5
                if cn > 1e-6 * max(c0, 1.0):
                    Q[:, k] = cand[:, 0] / cn
                    placed = True
                    break
            if not placed and strict:
                raise ContractViolation("ran out of completion vectors during orthonormalization")
        else:
            Q[:, k] = v[:, 0] / nrm
    return Q, ndef


def run_slabs_local(P, grid, quad, step, state, n_steps=1, advance=None, **kw):  # noqa: D401
    """Convenience for tests: split a full state into P row slabs, run
    ``n_steps`` slab steps as virtual ranks in one process and gather the
    result (X rows concatenated; S, W from rank 0 -- identical on all)."""
    rows = slab_rows(grid.ny, P)
    slabs = [Slab(p, P, grid, rows) for p in range(P)]
    states = [split_state(state, s) for s in slabs]
    infos = []
    for _ in range(n_steps):
        res = run_local(P, lambda p: step_slab(slabs[p], step, quad, states[p], **kw))
        states = [s for s, _ in res]
        infos.append([i for _, i in res])
        if advance is not None:
            step = advance(step, torch.cat([i["phi"] for _, i in res]))
    X = torch.cat([s.X for s in states], dim=0)
    return DlrState(X=X, S=states[0].S, W=states[0].W), infos, step
