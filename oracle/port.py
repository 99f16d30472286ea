"""numpy/scipy restatement of the reference DLR-SN hot path (TEST ORACLE).

TEST INFRASTRUCTURE: only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU-baseline legs of ``bench.py`` may use this module.  It is the checker
and the timed CPU baseline ("port"), never the product path.

Every public function names the reference code it restates
(paths relative to ``/root/reference/pkg/src/greytrt``).  Semantics --
layouts, operation order where it matters for round-off, error types and
thresholds -- follow the reference; the implementation is our own
(vectorised across directions and cells where the reference loops).

Layout (reference convention, ``mesh.py:28-33,117-118,178-179``):
dof = 4*cell + local, local 0..3 = corners (0,0),(1,0),(0,1),(1,1),
cell = j*nx + i; psi / X are (n_dofs, k) row-major.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp

FOUR_PI = 4.0 * np.pi
DEFICIENCY_TOL = 1e-12  # angular.py:24
T_FLOOR = 1e-6  # physics.py:33

# edge dof pairs, mesh.py:34-39
EDGE = {"left": (0, 2), "right": (1, 3), "bottom": (0, 1), "top": (2, 3)}


# --------------------------------------------------------------------------
# error taxonomy (mirrors errors.py:4-41; the oracle raises the product's
# exception classes so tests can compare behaviour one-to-one)
from paper_2601_18705_b200.errors import (  # noqa: E402
    CgError,
    ContractViolation,
    InterpolationError,
    IterationLimitError,
    SolverError,
)


# --------------------------------------------------------------------------
# grid and reference-cell blocks


@dataclass(frozen=True)
class Grid:
    """Uniform structured grid (mesh.py:76-127, build_grid :130-210)."""

    nx: int
    ny: int
    x0: float = 0.0
    y0: float = 0.0
    lx: float = 1.0
    ly: float = 1.0

    @property
    def dx(self):
        return self.lx / self.nx

    @property
    def dy(self):
        return self.ly / self.ny

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def n_dofs(self):
        return 4 * self.nx * self.ny

    @property
    def extent(self):
        return (self.x0, self.y0, self.nx * self.dx, self.ny * self.dy)

    @property
    def cell_area(self):
        return self.dx * self.dy


def q1_blocks():
    """Q1 reference-cell integrals by 3-point Gauss, as mesh.py:285-313 does
    (so the fp64 bits of the blocks match the reference's)."""
    x, w = np.polynomial.legendre.leggauss(3)
    pts, wts = 0.5 * (x + 1.0), 0.5 * w
    mass = np.zeros((4, 4))
    gxi = np.zeros((4, 4))
    geta = np.zeros((4, 4))
    for xi, wx in zip(pts, wts):
        for eta, wy in zip(pts, wts):
            n = np.array([(1 - xi) * (1 - eta), xi * (1 - eta), (1 - xi) * eta, xi * eta])
            dxi = np.array([-(1 - eta), (1 - eta), -eta, eta])
            deta = np.array([-(1 - xi), -xi, (1 - xi), xi])
            ww = wx * wy
            mass += ww * np.outer(n, n)
            gxi += ww * np.outer(dxi, n)
            geta += ww * np.outer(deta, n)
    edge = np.array([[2.0, 1.0], [1.0, 2.0]]) / 6.0
    return mass, gxi, geta, edge


def dof_coordinates(grid):
    """Corner coordinates of every dof (mesh.py:251-265)."""
    c = np.arange(grid.n_cells)
    i, j = c % grid.nx, c // grid.nx
    off = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    cx = grid.x0 + i * grid.dx
    cy = grid.y0 + j * grid.dy
    out = np.empty((grid.n_cells, 4, 2))
    out[:, :, 0] = cx[:, None] + off[None, :, 0] * grid.dx
    out[:, :, 1] = cy[:, None] + off[None, :, 1] * grid.dy
    return out.reshape(-1, 2)


def cells_to_dofs(values):
    """driver.py:333-336 (discontinuous branch)."""
    return np.repeat(np.asarray(values, dtype=float), 4)


def dofs_to_cells(values):
    """driver.py:344-346."""
    return np.asarray(values, dtype=float).reshape(-1, 4).mean(axis=1)


# --------------------------------------------------------------------------
# angular quadrature and bases


@dataclass(frozen=True, eq=False)
class Quadrature:
    """angular.py:28-42."""

    omegas: np.ndarray
    weights: np.ndarray
    n_polar: int
    n_azimuthal: int

    @property
    def n_angles(self):
        return self.omegas.shape[0]


def build_quadrature(n_polar, n_azimuthal):
    """Gauss-Legendre(mu) x half-offset uniform azimuth (angular.py:45-87)."""
    mu, wmu = np.polynomial.legendre.leggauss(n_polar)
    az = 2.0 * np.pi * (np.arange(n_azimuthal) + 0.5) / n_azimuthal
    s = np.sqrt(1.0 - mu**2)
    om = np.empty((n_polar, n_azimuthal, 3))
    om[:, :, 0] = s[:, None] * np.cos(az)[None, :]
    om[:, :, 1] = s[:, None] * np.sin(az)[None, :]
    om[:, :, 2] = mu[:, None]
    wts = (wmu[:, None] * (2.0 * np.pi / n_azimuthal)) * np.ones((1, n_azimuthal))
    return Quadrature(om.reshape(-1, 3), wts.reshape(-1), n_polar, n_azimuthal)


def spatial_monomials(coords, extent, count):
    """Scaled monomials x^a y^b by rising degree (lowrank.py:28-40)."""
    x0, y0, lx, ly = extent
    xh = 2.0 * (coords[:, 0] - x0) / lx - 1.0
    yh = 2.0 * (coords[:, 1] - y0) / ly - 1.0
    out = []
    deg = 0
    while len(out) < count:
        for a in range(deg, -1, -1):
            out.append(xh**a * yh ** (deg - a))
        deg += 1
    return out[:count]


def angular_monomials(quad, count):
    """Monomials in omega then unit vectors (angular.py:198-214)."""
    ox, oy, oz = quad.omegas.T
    out = [np.ones_like(ox)]
    deg = 1
    while len(out) < count:
        for a in range(deg, -1, -1):
            for b in range(deg - a, -1, -1):
                out.append(ox**a * oy**b * oz ** (deg - a - b))
        deg += 1
    return out[:count] + list(np.eye(quad.n_angles))


def gram_schmidt(columns, dot_many, completion=None, strict=True):
    """Twice-projected classical Gram-Schmidt (angular.py:104-160).

    ``dot_many(Q, v)`` returns the vector of inner products <Q[:, i], v>
    (one fused product instead of the reference's per-column list; the
    values are the same inner products).  Returns (Q, R, deficient).
    """
    cols = np.array(columns, dtype=float)
    n, m = cols.shape
    q = np.zeros((n, m))
    r = np.zeros((m, m))
    deficient = []
    cand_iter = iter(completion) if completion is not None else iter(np.eye(n).T)

    def norm(v):
        return math.sqrt(max(float(dot_many(v[:, None], v)[0]), 0.0))

    def project_twice(v, k):
        tot = np.zeros(k)
        for _ in range(2):
            if k:
                cf = dot_many(q[:, :k], v)
                v = v - q[:, :k] @ cf
                tot = tot + cf
        return v, tot

    for k in range(m):
        v = cols[:, k]
        orig = norm(v)
        v, tot = project_twice(v, k)
        nrm = norm(v)
        r[:k, k] = tot
        if nrm <= DEFICIENCY_TOL * max(orig, 1.0):
            deficient.append(k)
            r[k, k] = 0.0
            while True:
                try:
                    cand = np.asarray(next(cand_iter), dtype=float)
                except StopIteration:
                    if not strict:
                        break
                    raise ContractViolation(
                        "ran out of completion vectors during orthonormalization"
                    ) from None
                c0 = norm(cand)
                cand, _ = project_twice(cand, k)
                c1 = norm(cand)
                if c1 > math.sqrt(DEFICIENCY_TOL) * max(c0, 1.0):
                    q[:, k] = cand / c1
                    break
        else:
            r[k, k] = nrm
            q[:, k] = v / nrm
    return q, r, deficient


def weighted_dot(weights):
    w = np.asarray(weights, dtype=float)
    return lambda Q, v: Q.T @ (w * v)


def orthonormalize(columns, quad):
    """Weighted CGS2 with angular-monomial completion (angular.py:217-238,
    pin_constant=False branch).  Returns (W, R, deficient)."""
    cols = np.asarray(columns, dtype=float)
    if cols.shape[0] != quad.n_angles:
        raise ContractViolation("basis rows must match quadrature size")
    comp = angular_monomials(quad, cols.shape[1] + 8)
    return gram_schmidt(cols, weighted_dot(quad.weights), comp)


# --------------------------------------------------------------------------
# physics (physics.py:63-132)


@dataclass(frozen=True)
class Constants:
    c: float = 299.79
    a_r: float = 0.01372


def planck(T, k=Constants()):
    T = np.asarray(T, dtype=float)
    if np.any(T < 0):
        raise ContractViolation("negative temperature passed to planck()")
    s = k.a_r * k.c
    return s / FOUR_PI * T**4, s / np.pi * T**3


@dataclass(eq=False)
class Step:
    """LinearizedStep (physics.py:78-91)."""

    sigma_t: np.ndarray
    sigma_s: np.ndarray
    sigma_a: np.ndarray
    q: np.ndarray
    T0: np.ndarray
    denom: np.ndarray
    rho_cv: np.ndarray
    dt: float
    inv_cdt: float
    constants: Constants = Constants()


def linearize(T0, sigma_a, rho_cv, dt, k=Constants()):
    """physics.py:94-120."""
    T0 = np.asarray(T0, dtype=float)
    sa = np.asarray(sigma_a, dtype=float)
    rc = np.asarray(rho_cv, dtype=float)
    if dt <= 0:
        raise ContractViolation(f"time step must be positive, got {dt}")
    if np.any(sa < 0) or np.any(rc <= 0):
        raise ContractViolation("need sigma_a >= 0 and rho*c_v > 0 in every cell")
    B, dB = planck(T0, k)
    den = rc + FOUR_PI * dt * sa * dB
    ss = sa * (FOUR_PI * dt * sa * dB) / den
    q = sa * B * rc / den
    icdt = 1.0 / (k.c * dt)
    return Step(sa + icdt, ss, sa, q, T0, den, rc, float(dt), icdt, k)


def update_temperature(phi_cells, step, t_floor=T_FLOOR):
    """physics.py:123-132."""
    B0, _ = planck(step.T0, step.constants)
    T = step.T0 + step.dt * step.sigma_a * (np.asarray(phi_cells, float) - FOUR_PI * B0) / step.denom
    return np.maximum(T, t_floor)


# --------------------------------------------------------------------------
# discrete operators (transport_sn.py:78-300)


def _embed(block, rows, cols):
    out = np.zeros((4, 4))
    out[np.ix_(rows, cols)] = block
    return out


@dataclass(eq=False)
class Operators:
    grid: Grid
    step: Step
    mass_cell: np.ndarray
    grad: tuple
    edge_mass: dict
    couple: dict
    Px: sp.csr_matrix = None
    Py: sp.csr_matrix = None
    Jx: sp.csr_matrix = None
    Jy: sp.csr_matrix = None
    dsa_penalty: str = "simplified"
    penalty_closure: tuple | None = None
    _dsa: tuple | None = None
    _cache: dict = field(default_factory=dict)

    def mass_apply(self, u, coeff=None):
        """transport_sn.py:107-116: per-cell mass block, then the coefficient."""
        u = np.asarray(u)
        flat = u.ndim == 1
        lib = _csweep_lib()
        if lib is not None and u.dtype == np.float64 and u.size >= (1 << 16):
            return _mass_apply_c(lib, self, u, coeff, flat)
        uc = u.reshape(self.grid.n_cells, 4, -1)
        out = np.einsum("ij,cjk->cik", self.mass_cell, uc)
        if coeff is not None:
            out = out * np.asarray(coeff)[:, None, None]
        out = out.reshape(self.grid.n_dofs, -1)
        return out[:, 0] if flat else out

    def mass_matrix(self, coeff=None):
        blocks = np.broadcast_to(self.mass_cell, (self.grid.n_cells, 4, 4)).copy()
        if coeff is not None:
            blocks *= np.asarray(coeff)[:, None, None]
        return _block_diag(blocks)

    def source_vector(self, cell_values):
        """transport_sn.py:124-127."""
        row = self.mass_cell.sum(axis=1)
        return (np.asarray(cell_values)[:, None] * row[None, :]).ravel()

    def streaming_matrix(self, omega):
        return (omega[0] * self.Px + omega[1] * self.Py
                + abs(omega[0]) * self.Jx + abs(omega[1]) * self.Jy).tocsr()


def _block_diag(blocks):
    n = blocks.shape[0]
    base = 4 * np.arange(n)
    rows = (base[:, None, None] + np.arange(4)[None, :, None]) * np.ones((1, 1, 4), int)
    cols = (base[:, None, None] + np.arange(4)[None, None, :]) * np.ones((1, 4, 1), int)
    return sp.csr_matrix((blocks.ravel(), (rows.ravel(), cols.ravel())), shape=(4 * n, 4 * n))


def _face_coo(rows_a, rows_b, e2, sign_pairs, n):
    """COO of 2x2 blocks e2 placed at (rows_a|rows_b) x (rows_a|rows_b)."""
    R, C, V = [], [], []
    for (ra, rb, s) in sign_pairs:
        ra_, rb_ = (rows_a if ra == "a" else rows_b), (rows_a if rb == "a" else rows_b)
        rr = np.repeat(ra_[:, :, None], 2, axis=2)
        cc = np.repeat(rb_[:, None, :], 2, axis=1)
        R.append(rr.ravel())
        C.append(cc.ravel())
        V.append(np.broadcast_to(s * e2, rr.shape).ravel())
    if not R:
        return sp.csr_matrix((n, n))
    return sp.csr_matrix((np.concatenate(V), (np.concatenate(R), np.concatenate(C))), shape=(n, n))


def assemble_operators(grid, step, dsa_penalty="simplified", penalty_closure=None,
                       with_matrices=True):
    """transport_sn.py:201-300 (vectorised COO assembly, vacuum walls)."""
    for name in ("sigma_t", "sigma_s", "q"):
        if np.asarray(getattr(step, name)).shape != (grid.n_cells,):
            raise ContractViolation(f"step field {name} must be per-cell")
    if np.any(step.sigma_t - step.sigma_s <= 0):
        raise ContractViolation("pseudo absorption sigma_t - sigma_s must stay positive")
    if dsa_penalty not in ("simplified", "collocation"):
        raise ContractViolation(f"unknown dsa penalty variant {dsa_penalty!r}")
    mhat, gxi, geta, ehat = q1_blocks()
    dx, dy = grid.dx, grid.dy
    mass_cell = mhat * dx * dy
    grad = (-dy * gxi, -dx * geta)
    e2x, e2y = dy * ehat, dx * ehat
    edge_mass = {w: _embed(e2x if w in ("left", "right") else e2y, EDGE[w], EDGE[w]) for w in EDGE}
    couple = {
        ("x", 1): _embed(e2x, EDGE["left"], EDGE["right"]),
        ("x", -1): _embed(e2x, EDGE["right"], EDGE["left"]),
        ("y", 1): _embed(e2y, EDGE["bottom"], EDGE["top"]),
        ("y", -1): _embed(e2y, EDGE["top"], EDGE["bottom"]),
    }
    ops = Operators(grid, step, mass_cell, grad, edge_mass, couple,
                    dsa_penalty=dsa_penalty, penalty_closure=penalty_closure)
    if not with_matrices:
        return ops
    n = grid.n_dofs
    nx, ny = grid.nx, grid.ny
    cid = np.arange(grid.n_cells).reshape(ny, nx)
    dofs = lambda cells, loc: 4 * cells[:, None] + np.asarray(loc)[None, :]  # noqa: E731
    gx = _block_diag(np.broadcast_to(grad[0], (grid.n_cells, 4, 4)).copy())
    gy = _block_diag(np.broadcast_to(grad[1], (grid.n_cells, 4, 4)).copy())
    # interior faces: average part n{u}[[v]] and jump (1/2)[[u]][[v]] (:230-244)
    fa_pairs = [("a", "a", 0.5), ("a", "b", 0.5), ("b", "a", -0.5), ("b", "b", -0.5)]
    j_pairs = [("a", "a", 0.5), ("a", "b", -0.5), ("b", "a", -0.5), ("b", "b", 0.5)]
    m_x = cid[:, :-1].ravel(); p_x = cid[:, 1:].ravel()
    m_y = cid[:-1, :].ravel(); p_y = cid[1:, :].ravel()
    ax, bx = dofs(m_x, EDGE["right"]), dofs(p_x, EDGE["left"])
    ay, by = dofs(m_y, EDGE["top"]), dofs(p_y, EDGE["bottom"])
    fax = _face_coo(ax, bx, e2x, fa_pairs, n)
    fay = _face_coo(ay, by, e2y, fa_pairs, n)
    jx_i = _face_coo(ax, bx, e2x, j_pairs, n)
    jy_i = _face_coo(ay, by, e2y, j_pairs, n)
    # boundary faces (:246-258): 0.5*n_k*e2 into P, 0.5*e2 into J
    lw = dofs(cid[:, 0], EDGE["left"]); rw = dofs(cid[:, -1], EDGE["right"])
    bw = dofs(cid[0, :], EDGE["bottom"]); tw = dofs(cid[-1, :], EDGE["top"])
    fbx = _face_coo(lw, lw, e2x, [("a", "a", -0.5)], n) + _face_coo(rw, rw, e2x, [("a", "a", 0.5)], n)
    fby = _face_coo(bw, bw, e2y, [("a", "a", -0.5)], n) + _face_coo(tw, tw, e2y, [("a", "a", 0.5)], n)
    jbx = _face_coo(lw, lw, e2x, [("a", "a", 0.5)], n) + _face_coo(rw, rw, e2x, [("a", "a", 0.5)], n)
    jby = _face_coo(bw, bw, e2y, [("a", "a", 0.5)], n) + _face_coo(tw, tw, e2y, [("a", "a", 0.5)], n)
    ops.Px = (gx + fax + fbx).tocsr()
    ops.Py = (gy + fay + fby).tocsr()
    ops.Jx = (jx_i + jbx).tocsr()
    ops.Jy = (jy_i + jby).tocsr()
    return ops


# --------------------------------------------------------------------------
# sweeps (transport_sn.py:38-69, 142-163, 303-322)


def quadrant_of(omega):
    """Grazing components sweep as positive (transport_sn.py:38-42)."""
    return (1 if omega[0] >= 0.0 else -1, 1 if omega[1] >= 0.0 else -1)


def _plan(nx, ny, sx, sy):
    """Anti-diagonal levels from the inflow corner (transport_sn.py:54-69)."""
    jj, ii = np.divmod(np.arange(nx * ny), nx)
    li = ii if sx > 0 else nx - 1 - ii
    lj = jj if sy > 0 else ny - 1 - jj
    level = li + lj
    order = np.argsort(level, kind="stable")
    cells = np.arange(nx * ny)[order]
    bounds = np.searchsorted(level[order], np.arange(nx + ny))
    levels = [cells[bounds[k]:bounds[k + 1]] for k in range(nx + ny - 1)]
    xi = ii - sx
    xn = np.where((xi >= 0) & (xi < nx), jj * nx + xi, -1)
    yi = jj - sy
    yn = np.where((yi >= 0) & (yi < ny), yi * nx + ii, -1)
    return levels, xn, yn


def _local_inverses(ops, omegas):
    """Per-direction, per-cell explicit inverses of the local operator
    (transport_sn.py:142-163).  omegas (D, >=2) all in one quadrant."""
    sx, sy = quadrant_of(omegas[0])
    out = np.empty((len(omegas), ops.grid.n_cells, 4, 4))
    for k, om in enumerate(omegas):
        key = (float(om[0]), float(om[1]))
        hit = ops._cache.get(key)
        if hit is None:
            ox, oy = abs(float(om[0])), abs(float(om[1]))
            stream = (om[0] * ops.grad[0] + om[1] * ops.grad[1]
                      + ox * ops.edge_mass["right" if sx > 0 else "left"]
                      + oy * ops.edge_mass["top" if sy > 0 else "bottom"])
            local = stream[None] + np.asarray(ops.step.sigma_t)[:, None, None] * ops.mass_cell[None]
            hit = np.linalg.inv(local)
            if len(ops._cache) < 64:
                ops._cache[key] = hit
        out[k] = hit
    return out


# --- plain-C restatement of the sweep (oracle/csweep.c), built on demand ---
_CSWEEP = None


def _csweep_lib():
    """ctypes handle of oracle/libcsweep.so (compiled with gcc -fopenmp on
    first use when missing or older than csweep.c); None if gcc fails."""
    global _CSWEEP
    if _CSWEEP is None:
        import ctypes
        import os
        import subprocess

        here = os.path.dirname(os.path.abspath(__file__))
        src = os.path.join(here, "csweep.c")
        so = os.path.join(here, "libcsweep.so")
        try:
            if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
                tmp = f"{so}.{os.getpid()}.tmp"
                subprocess.run(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src],
                               check=True, capture_output=True)
                os.replace(tmp, so)
            lib = ctypes.CDLL(so)
            f = lib.csweep_quadrant
            P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
            f.argtypes = [I, I, I, I, I, P, P, P, P, P, P, P, P, L, P, P, L, P, I]
            f.restype = None
            lib.cmass_apply.argtypes = [L, L, P, P, P, P, I]
            lib.cmass_apply.restype = None
            _CSWEEP = lib
        except Exception:
            _CSWEEP = False
    return _CSWEEP or None


def build_csweep():
    """Compile the C sweep restatement now (__graft_entry__.build)."""
    return _csweep_lib() is not None


def _mass_apply_c(lib, ops, u, coeff, flat):
    import os

    u = np.ascontiguousarray(u, dtype=np.float64)
    k = 1 if flat else u.shape[1]
    out = np.empty((ops.grid.n_dofs, k))
    mass = np.ascontiguousarray(ops.mass_cell, dtype=np.float64)
    cf = None if coeff is None else np.ascontiguousarray(coeff, dtype=np.float64)
    nthreads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 0
    lib.cmass_apply(ops.grid.n_cells, k, mass.ctypes.data, None if cf is None else cf.ctypes.data,
                    u.ctypes.data, out.ctypes.data, nthreads)
    return out[:, 0] if flat else out


def _sweep_many_c(lib, ops, omegas, rhs):
    import os

    g = ops.grid
    D = omegas.shape[0]
    rhs = np.ascontiguousarray(rhs, dtype=float)
    psi_out = np.empty((g.n_dofs, D))
    sig = np.ascontiguousarray(ops.step.sigma_t, dtype=float)
    mass = np.ascontiguousarray(ops.mass_cell, dtype=float)
    nthreads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 0
    quads = {}
    for d in range(D):
        quads.setdefault(quadrant_of(omegas[d]), []).append(d)
    for (sx, sy), idx in quads.items():
        om = omegas[idx]
        stream = np.empty((len(idx), 4, 4))
        for k, o in enumerate(om):
            stream[k] = (o[0] * ops.grad[0] + o[1] * ops.grad[1]
                         + abs(float(o[0])) * ops.edge_mass["right" if sx > 0 else "left"]
                         + abs(float(o[1])) * ops.edge_mass["top" if sy > 0 else "bottom"])
        cx = np.ascontiguousarray(ops.couple[("x", sx)], dtype=float)
        cy = np.ascontiguousarray(ops.couple[("y", sy)], dtype=float)
        ox = np.ascontiguousarray(np.abs(om[:, 0]))
        oy = np.ascontiguousarray(np.abs(om[:, 1]))
        cols = np.ascontiguousarray(idx, dtype=np.int32)
        lib.csweep_quadrant(g.nx, g.ny, sx, sy, len(idx), stream.ctypes.data, mass.ctypes.data,
                            sig.ctypes.data, cx.ctypes.data, cy.ctypes.data, ox.ctypes.data,
                            oy.ctypes.data, rhs.ctypes.data, D, cols.ctypes.data,
                            psi_out.ctypes.data, D, cols.ctypes.data, nthreads)
    return psi_out


def sweep_many(ops, omegas, rhs, chunk=16, use_c=True):
    """Upwind sweeps of many directions: rhs (n_dofs, D) -> psi (n_dofs, D).

    Same arithmetic per direction as ``sweep_solve`` (transport_sn.py:303-322);
    directions of one quadrant advance through the wavefront levels together
    (numpy), or run through the plain-C restatement (oracle/csweep.c, same
    per-cell arithmetic) when it builds.
    """
    omegas = np.asarray(omegas, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    lib = _csweep_lib() if use_c else None
    if lib is not None:
        return _sweep_many_c(lib, ops, omegas, rhs)
    g = ops.grid
    nc = g.n_cells
    D = omegas.shape[0]
    psi_out = np.empty((g.n_dofs, D))
    quads = {}
    for d in range(D):
        quads.setdefault(quadrant_of(omegas[d]), []).append(d)
    for (sx, sy), idx in quads.items():
        levels, xn, yn = _plan(g.nx, g.ny, sx, sy)
        cxT = ops.couple[("x", sx)].T
        cyT = ops.couple[("y", sy)].T
        for c0 in range(0, len(idx), chunk):
            sel = idx[c0:c0 + chunk]
            om = omegas[sel]
            ainv = _local_inverses(ops, om)
            ox = np.abs(om[:, 0])[:, None, None]
            oy = np.abs(om[:, 1])[:, None, None]
            acc = rhs[:, sel].T.reshape(len(sel), nc, 4)
            psi = np.zeros((len(sel), nc, 4))
            for cells in levels:
                local = acc[:, cells].copy()
                xc = xn[cells]
                m = xc >= 0
                if m.any():
                    local[:, m] += (psi[:, xc[m]] @ cxT) * ox
                yc = yn[cells]
                m = yc >= 0
                if m.any():
                    local[:, m] += (psi[:, yc[m]] @ cyT) * oy
                psi[:, cells] = np.einsum("dcij,dcj->dci", ainv[:, cells], local)
            psi_out[:, sel] = psi.reshape(len(sel), -1).T
    return psi_out


def sweep_solve(ops, omega, rhs):
    """transport_sn.py:303-322 (single direction)."""
    return sweep_many(ops, np.asarray(omega, float)[None, :], np.asarray(rhs, float)[:, None])[:, 0]



def sweep_balance(grid, omega, sigma_t, rhs, psi):
    """Global particle balance of one direction's upwind DG(Q1) solve, a
    size-independent property of the reference discretisation
    (transport_sn.py:142-163 local operator, :213-227 face couplings,
    :303-322 sweep; vacuum inflow).  Testing every cell equation with the
    constant 1 (the sum of its 4 rows): the volume streaming term vanishes
    (the columns of the reference gradient blocks sum to zero: sum_i dN_i = 0),
    each interior face's outflow term cancels the downwind cell's inflow
    coupling (upwind flux), and 1^T M_hat = 1/4.  What is left is
        sum_c sigma_t,c dx dy / 4 sum_l psi_{c,l}
      + sum_{outflow walls} |omega.n| len (psi_a + psi_b) / 2  =  sum(rhs)
    exactly, for any grid size.  Returns (left side, right side)."""
    nx, ny = grid.nx, grid.ny
    ox, oy = float(omega[0]), float(omega[1])
    p = np.asarray(psi, dtype=float).reshape(ny, nx, 4)
    st = np.asarray(sigma_t, dtype=float).reshape(ny, nx)
    absorbed = float(np.sum(st * p.sum(axis=2))) * grid.dx * grid.dy / 4.0
    out = 0.0
    if ox != 0.0:  # right wall (dofs 1, 3) for ox > 0, left wall (0, 2) otherwise
        col, e = (p[:, -1, :], EDGE["right"]) if ox > 0 else (p[:, 0, :], EDGE["left"])
        out += abs(ox) * grid.dy * 0.5 * float(np.sum(col[:, e[0]] + col[:, e[1]]))
    if oy != 0.0:
        row, e = (p[-1, :, :], EDGE["top"]) if oy > 0 else (p[0, :, :], EDGE["bottom"])
        out += abs(oy) * grid.dx * 0.5 * float(np.sum(row[:, e[0]] + row[:, e[1]]))
    return absorbed + out, float(np.sum(np.asarray(rhs, dtype=float)))

# --------------------------------------------------------------------------
# synthetic diffusion (transport_sn.py:166-198, 325-367)


def dsa_system(ops):
    if ops._dsa is not None:
        return ops._dsa
    st = ops.step
    blocks = np.linalg.inv(np.asarray(st.sigma_t)[:, None, None] * ops.mass_cell[None])
    mt_inv = _block_diag(blocks)
    if ops.dsa_penalty == "simplified":
        kx = ky = 0.25
    else:
        om, cw = ops.penalty_closure
        kx = 0.5 * float(cw @ np.abs(om[:, 0])) / FOUR_PI
        ky = 0.5 * float(cw @ np.abs(om[:, 1])) / FOUR_PI
    pen = kx * 2.0 * ops.Jx + ky * 2.0 * ops.Jy
    absorb = ops.mass_matrix(np.asarray(st.sigma_t) - np.asarray(st.sigma_s))
    a = ((ops.Px.T @ (mt_inv @ ops.Px) + ops.Py.T @ (mt_inv @ ops.Py)) / 3.0 + pen + absorb).tocsr()
    ops._dsa = (a, a.diagonal())
    return ops._dsa


def pcg(matvec, b, diag, tol=1e-10, max_iters=None, label="cg"):
    """Jacobi PCG (transport_sn.py:325-352)."""
    n = b.size
    max_iters = 10 * n if max_iters is None else max_iters
    x = np.zeros(n)
    r = b.copy()
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return x, 0
    minv = 1.0 / diag
    z = minv * r
    p = z.copy()
    rz = float(r @ z)
    hist = [float(np.linalg.norm(r))]
    for it in range(1, max_iters + 1):
        ap = matvec(p)
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        rn = float(np.linalg.norm(r))
        hist.append(rn)
        if rn <= tol * bn:
            return x, it
        z = minv * r
        rz2 = float(r @ z)
        p = z + (rz2 / rz) * p
        rz = rz2
    raise CgError(f"{label} failed to reach tol {tol:g}", max_iters, hist)


def dsa_correct(ops, residual_field, tol=1e-10):
    a, diag = dsa_system(ops)
    rhs = ops.mass_apply(np.asarray(residual_field, dtype=float))
    if not np.any(rhs):
        return np.zeros_like(rhs)
    delta, _ = pcg(lambda v: a @ v, rhs, diag, tol=tol, label="dsa")
    return delta


# --------------------------------------------------------------------------
# source iteration (transport_sn.py:370-450)


@dataclass(eq=False)
class SIResult:
    psi: np.ndarray
    phi: np.ndarray
    iterations: int


def source_iteration(ops, omegas, closure, psi_time=None, *, use_dsa=True, tol=1e-8,
                     max_iters=200, phi_start=None, extra_source=None, threads=0):
    omegas = np.asarray(omegas, dtype=float)
    closure = np.asarray(closure, dtype=float)
    nd = omegas.shape[0]
    if closure.shape != (nd,):
        raise ContractViolation("closure vector must have one entry per swept angle")
    st = ops.step
    base = np.tile(ops.source_vector(st.q), (nd, 1)).T
    if psi_time is not None:
        base = base + st.inv_cdt * ops.mass_apply(psi_time)
    if extra_source is not None:
        base = base + extra_source
    ss_dof = np.repeat(np.asarray(st.sigma_s), 4)
    phi = np.zeros(ops.grid.n_dofs) if phi_start is None else np.asarray(phi_start, float).copy()
    if not np.any(st.sigma_s):
        psi = sweep_many(ops, omegas, base)
        return SIResult(psi, psi @ closure, 1)
    change = np.inf
    for it in range(1, max_iters + 1):
        scatter = ops.mass_apply(ss_dof * phi) / FOUR_PI
        psi = sweep_many(ops, omegas, base + scatter[:, None])
        phi_half = psi @ closure
        phi_new = phi_half
        if use_dsa:
            phi_new = phi_half + dsa_correct(ops, ss_dof * (phi_half - phi))
        den = max(float(np.linalg.norm(phi_new)), 1e-300)
        change = float(np.linalg.norm(phi_new - phi)) / den
        phi = phi_new
        if change <= tol:
            return SIResult(psi, phi, it)
    raise IterationLimitError("source iteration did not converge", max_iters, change)


# --------------------------------------------------------------------------
# isotropic inflow boundary (BASELINE config 3) -- NOT in the reference, which
# is vacuum-only (transport_sn.py:11-13: "on the boundary the exterior state is
# zero").  Restatement: with a constant exterior state psi_b on an inflow wall
# the upwind face flux contributes the same coupling the interior faces use
# (|omega.n| * e2, the ``couple`` blocks of transport_sn.py:219-224) applied to
# psi_b [1, 1]: |omega.n| * psi_b * (e2 @ [1, 1]) on the wall's edge dofs.  It
# enters the sweep through the reference's ``extra_source`` slot
# (transport_sn.py:387,406-407) and the reduced rows through X^T of the same
# load.  With psi_b = 0 everything reduces to the reference.

WALLS = ("left", "right", "bottom", "top")
WALL_NORMALS = {"left": (-1.0, 0.0), "right": (1.0, 0.0), "bottom": (0.0, -1.0),
                "top": (0.0, 1.0)}


def inflow_tuple(inflow):
    """None | {wall: psi_b} | 4 values (left, right, bottom, top) -> 4-tuple or None."""
    if inflow is None:
        return None
    if isinstance(inflow, dict):
        bad = set(inflow) - set(WALLS)
        if bad:
            raise ContractViolation(f"unknown inflow walls {sorted(bad)}")
        vals = tuple(float(inflow.get(w, 0.0)) for w in WALLS)
    else:
        vals = tuple(float(v) for v in inflow)
        if len(vals) != 4:
            raise ContractViolation("inflow needs 4 values (left, right, bottom, top)")
    if any(not np.isfinite(v) or v < 0 for v in vals):
        raise ContractViolation("inflow intensities must be finite and non-negative")
    return vals if any(vals) else None


def inflow_load(grid, omegas, inflow):
    """(n_dofs, D) load of an isotropic inflow: column d gets
    max(-omega_d.n_w, 0) * psi_b,w * (e2 @ [1, 1]) on the edge dofs of every
    cell of each wall w."""
    vals = inflow_tuple(inflow)
    om = np.atleast_2d(np.asarray(omegas, dtype=float))
    out = np.zeros((grid.n_dofs, om.shape[0]))
    if vals is None:
        return out
    edge = q1_blocks()[3]
    cid = np.arange(grid.n_cells).reshape(grid.ny, grid.nx)
    cells = {"left": cid[:, 0], "right": cid[:, -1], "bottom": cid[0, :], "top": cid[-1, :]}
    for w, psi_b in zip(WALLS, vals):
        if psi_b == 0.0:
            continue
        e2 = (grid.dy if w in ("left", "right") else grid.dx) * edge
        g = e2 @ np.ones(2)
        n = WALL_NORMALS[w]
        coef = np.maximum(-(om[:, 0] * n[0] + om[:, 1] * n[1]), 0.0) * psi_b
        for k, l in enumerate(EDGE[w]):
            out[4 * cells[w] + l, :] += g[k] * coef[None, :]
    return out


def boundary_outflow(grid, psi, omegas, weights):
    """transport_sn.py:479-492 (trapezoid rule on the boundary traces)."""
    psi = np.asarray(psi)
    nx, ny = grid.nx, grid.ny
    cid = np.arange(grid.n_cells).reshape(ny, nx)
    walls = [("left", cid[:, 0], (-1.0, 0.0), grid.dy), ("right", cid[:, -1], (1.0, 0.0), grid.dy),
             ("bottom", cid[0, :], (0.0, -1.0), grid.dx), ("top", cid[-1, :], (0.0, 1.0), grid.dx)]
    om = np.asarray(omegas)[:, :2]
    total = 0.0
    for w, cells, nrm, length in walls:
        e = EDGE[w]
        vals = 0.5 * (psi[4 * cells + e[0]] + psi[4 * cells + e[1]]) * length
        on = np.maximum(om @ np.asarray(nrm), 0.0)
        total += float(np.sum(on[None, :] * vals @ np.asarray(weights)))
    return total


# --------------------------------------------------------------------------
# low-rank kernels (lowrank.py, dlr_sn.py)


@dataclass(eq=False)
class State:
    """DlrState (lowrank.py:43-81) with W stored as values + beta."""

    X: np.ndarray
    S: np.ndarray
    W: np.ndarray
    beta: np.ndarray

    @property
    def rank(self):
        return self.S.shape[0]

    def reconstruct(self, idx=None):
        w = self.W if idx is None else self.W[idx]
        return self.X @ (self.S @ w.T)

    def scalar_flux(self):
        return self.X @ (self.S @ self.beta)


def mass_dot(ops):
    """Q^T M v with M applied to the right argument (lowrank.py:23-25)."""
    return lambda Q, v: Q.T @ ops.mass_apply(v)


def state_check(state, ops, quad, tol=1e-10):
    """lowrank.py:68-81 (unpinned bases)."""
    gx = state.X.T @ ops.mass_apply(state.X)
    rx = float(np.abs(gx - np.eye(state.rank)).max())
    gw = (state.W * quad.weights[:, None]).T @ state.W
    rw = float(np.abs(gw - np.eye(state.rank)).max())
    if rx > tol or rw > tol:
        raise ContractViolation(f"factor orthonormality violated: spatial {rx:.2e}, angular {rw:.2e}")
    return rx, rw


@dataclass(eq=False)
class Deim:
    indices: np.ndarray
    w_hat: np.ndarray
    lu: tuple
    cond: float

    def interpolation_coefficients(self, values):
        return scipy.linalg.lu_solve(self.lu, values)

    def closure_weights(self, beta):
        return scipy.linalg.lu_solve(self.lu, beta, trans=1)


def deim_select(W):
    """Greedy DEIM over quadrature nodes (lowrank.py:168-205)."""
    w = np.asarray(W, dtype=float)
    if w.ndim != 2:
        raise ContractViolation("deim_select expects an (n_angles, rank) array")
    n, r = w.shape
    if r > n:
        raise ContractViolation(f"rank {r} exceeds the {n} available nodes")
    floor = 1e-14 * max(1.0, float(np.abs(w).max()))
    picks = []
    for j in range(r):
        if j == 0:
            res = w[:, 0]
        else:
            cf = np.linalg.solve(w[np.ix_(picks, range(j))], w[picks, j])
            res = w[:, j] - w[:, :j] @ cf
        p = int(np.argmax(np.abs(res)))
        if abs(res[p]) <= floor:
            raise InterpolationError("interpolation residual vanished; basis is rank deficient", column=j)
        if p in picks:
            raise InterpolationError("duplicate interpolation point; basis is rank deficient", column=j)
        picks.append(p)
    idx = np.asarray(picks, dtype=int)
    wh = w[idx, :]
    return Deim(idx, wh, scipy.linalg.lu_factor(wh), float(np.linalg.cond(wh)))


def deim_gaps(W, picks):
    """Relative top-2 gap of the |residual| at each pick of ``picks`` over the
    rows not picked before it (the near-tie diagnostic of the GPU DEIM; a
    restatement of the residuals of lowrank.py:186-191 with the picked rows
    excluded, whose residuals are zero up to round-off)."""
    w = np.asarray(W, dtype=float)
    picks = [int(p) for p in picks]
    gaps = []
    for j in range(len(picks)):
        if j == 0:
            res = w[:, 0].copy()
        else:
            cf = np.linalg.solve(w[np.ix_(picks[:j], range(j))], w[picks[:j], j])
            res = w[:, j] - w[:, :j] @ cf
        a = np.abs(res)
        a[picks[:j]] = -1.0
        top = np.sort(a)[::-1]
        second = max(top[1], 0.0) if top.size > 1 else 0.0
        gaps.append((top[0] - second) / top[0] if top[0] > 0 else 0.0)
    return np.asarray(gaps)


def project_row_operators(ops, x):
    """dlr_sn.py:61-71."""
    st = ops.step
    return {
        "px": x.T @ (ops.Px @ x),
        "py": x.T @ (ops.Py @ x),
        "jx": x.T @ (ops.Jx @ x),
        "jy": x.T @ (ops.Jy @ x),
        "mt": x.T @ ops.mass_apply(x, coeff=st.sigma_t),
        "ms": x.T @ ops.mass_apply(x, coeff=st.sigma_s),
        "q": x.T @ ops.source_vector(st.q),
    }


def row_matrices(proj, omegas):
    """dlr_sn.py:74-83."""
    om = np.asarray(omegas, dtype=float)
    return (om[:, 0, None, None] * proj["px"] + om[:, 1, None, None] * proj["py"]
            + np.abs(om[:, 0])[:, None, None] * proj["jx"]
            + np.abs(om[:, 1])[:, None, None] * proj["jy"] + proj["mt"][None])


def project_initial(state, x_new, ops):
    """dlr_sn.py:50-58 (mass applied matrix-free)."""
    return state.W @ (state.S.T @ (state.X.T @ ops.mass_apply(x_new)))


def solve_row_system(B, ms, Q, weights):
    """lowrank.py:235-259."""
    B = np.asarray(B, dtype=float)
    Q = np.asarray(Q, dtype=float)
    n, r, _ = B.shape
    try:
        Binv = np.linalg.inv(B)
    except np.linalg.LinAlgError:
        for d in range(n):
            c = np.linalg.cond(B[d])
            if not np.isfinite(c) or c > 1e15:
                raise SolverError(f"singular reduced transport operator at node {d}")
        raise
    cbar = np.einsum("d,dij->ij", weights, Binv)
    zeta = np.einsum("d,dij,dj->i", weights, Binv, Q)
    lbar = np.linalg.solve(np.eye(r) - cbar @ ms / FOUR_PI, zeta)
    rhs = Q + (ms @ lbar)[None, :] / FOUR_PI
    return np.einsum("dij,dj->di", Binv, rhs), lbar


def _lazy_spatial_monomials(grid, count):
    """The completion candidates of dlr_sn.py:124-125 (spatial_monomials,
    lowrank.py:28-40), generated only when a deficiency asks for one."""
    coords = None
    x0, y0, lx, ly = grid.extent
    k, deg = 0, 0
    while k < count:
        for a in range(deg, -1, -1):
            if k >= count:
                return
            if coords is None:
                coords = dof_coordinates(grid)
                xh = 2.0 * (coords[:, 0] - x0) / lx - 1.0
                yh = 2.0 * (coords[:, 1] - y0) / ly - 1.0
            yield xh**a * yh ** (deg - a)
            k += 1
        deg += 1


@dataclass(eq=False)
class StepInfo:
    """CollocationStepInfo (dlr_sn.py:40-47)."""

    iterations: int
    interpolation_condition: float
    angle_indices: np.ndarray
    phi: np.ndarray
    spatial_deficiency: int
    angular_deficiency: int
    si_phi: np.ndarray = None


def step_collocation(grid, step, quad, state, *, si_tol=1e-8, si_max_iters=200, use_dsa=True,
                     dsa_penalty="simplified", threads=0, check_state=True, inflow=None):
    """One implicit DLR-SN step, Algorithm 1 (dlr_sn.py:86-151).  ``inflow``
    (not in the reference): isotropic inflow walls, see ``inflow_load``."""
    sel = deim_select(state.W)
    closure = sel.closure_weights(state.beta)
    om_sel = quad.omegas[sel.indices]
    pc = (om_sel, closure) if dsa_penalty == "collocation" else None
    ops = assemble_operators(grid, step, dsa_penalty=dsa_penalty, penalty_closure=pc)
    if check_state:
        state_check(state, ops, quad)
    psi_time = state.X @ (state.S @ state.W[sel.indices].T)  # evaluate_rows, lowrank.py:220-227
    extra = inflow_load(grid, om_sel, inflow) if inflow_tuple(inflow) else None
    res = source_iteration(ops, om_sel, closure, psi_time=psi_time, use_dsa=use_dsa, tol=si_tol,
                           max_iters=si_max_iters, phi_start=state.scalar_flux(),
                           extra_source=extra)
    comp = _lazy_spatial_monomials(grid, state.rank + 8)
    x_new, _, dx_ = gram_schmidt(res.psi, mass_dot(ops), comp)
    proj = project_row_operators(ops, x_new)
    B = row_matrices(proj, om_sel)
    l_time = project_initial(state, x_new, ops)[sel.indices]
    q_all = proj["q"][None, :] + step.inv_cdt * l_time
    if extra is not None:  # Galerkin rows of the inflow load
        q_all = q_all + (x_new.T @ extra).T
    l_nodes, l_bar = solve_row_system(B, proj["ms"], q_all, closure)
    gamma = sel.interpolation_coefficients(l_nodes)
    l_full = state.W @ gamma
    w_new, r_ang, dw_ = orthonormalize(l_full, quad)
    new = State(x_new, r_ang.T.copy(), w_new, w_new.T @ quad.weights)
    if check_state:
        state_check(new, ops, quad)
    info = StepInfo(res.iterations, sel.cond, sel.indices.copy(), x_new @ l_bar, len(dx_), len(dw_),
                    si_phi=res.phi)
    return new, info


# --------------------------------------------------------------------------
# parity metrics (tests/helpers.py:48-51 and SURVEY 8c)


def rel_l2(a, b):
    a = np.asarray(a, dtype=float).ravel()
    b = np.asarray(b, dtype=float).ravel()
    return float(np.linalg.norm(a - b)) / max(float(np.linalg.norm(b)), 1e-300)


def lowrank_rel_diff(X1, S1, W1, X2, S2, W2):
    """||X1 S1 W1^T - X2 S2 W2^T||_F / ||X2 S2 W2^T||_F via stacked QR
    (no cancellation floor)."""
    Y = np.hstack([X1 @ S1, -(X2 @ S2)])
    Z = np.hstack([W1, W2])
    _, ry = np.linalg.qr(Y)
    _, rz = np.linalg.qr(Z)
    diff = np.linalg.norm(ry @ rz.T)
    _, ry2 = np.linalg.qr(X2 @ S2)
    _, rz2 = np.linalg.qr(W2)
    return float(diff) / max(float(np.linalg.norm(ry2 @ rz2.T)), 1e-300)
