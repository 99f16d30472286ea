"""Structured uniform grid for the DLR-SN path (mirror of mesh.py:76-210).

Only the broken bilinear ("discontinuous") layout is on the sweep path
(transport_sn.py:203-204 rejects anything else).  The grid is pure metadata:
the GPU kernels derive every neighbour relation from (i, j), so no face or
dof tables are materialised on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .errors import ConfigurationError

DISCONTINUOUS = "discontinuous"
CONTINUOUS = "continuous"

EDGE_LOCALS = {"left": (0, 2), "right": (1, 3), "bottom": (0, 1), "top": (2, 3)}
WALL_NORMALS = {"left": (-1.0, 0.0), "right": (1.0, 0.0), "bottom": (0.0, -1.0), "top": (0.0, 1.0)}


@dataclass(frozen=True, eq=False)
class Grid:
    nx: int
    ny: int
    x0: float
    y0: float
    dx: float
    dy: float
    flavor: str = DISCONTINUOUS

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def n_dofs(self):
        if self.flavor == DISCONTINUOUS:
            return 4 * self.nx * self.ny
        return (self.nx + 1) * (self.ny + 1)

    @property
    def cell_area(self):
        return self.dx * self.dy

    @property
    def extent(self):
        return (self.x0, self.y0, self.nx * self.dx, self.ny * self.dy)

    def cell_id(self, i, j):
        return j * self.nx + i

    @cached_property
    def cell_centers(self):
        jj, ii = np.divmod(np.arange(self.n_cells), self.nx)
        c = np.column_stack([self.x0 + (ii + 0.5) * self.dx, self.y0 + (jj + 0.5) * self.dy])
        c.setflags(write=False)
        return c

    @cached_property
    def cell_dofs(self):
        d = 4 * np.arange(self.n_cells)[:, None] + np.arange(4)[None, :]
        d.setflags(write=False)
        return d

    @cached_property
    def boundary_faces(self):
        """(cells, walls, normals, lengths) in the reference's order
        (mesh.py:166-178): per row left/right, then per column bottom/top."""
        cells, walls, lengths = [], [], []
        for j in range(self.ny):
            cells += [j * self.nx, j * self.nx + self.nx - 1]
            walls += ["left", "right"]
            lengths += [self.dy, self.dy]
        for i in range(self.nx):
            cells += [i, (self.ny - 1) * self.nx + i]
            walls += ["bottom", "top"]
            lengths += [self.dx, self.dx]
        normals = np.array([WALL_NORMALS[w] for w in walls])
        return np.asarray(cells), np.asarray(walls, dtype=object), normals, np.asarray(lengths)


def build_grid(nx, ny, extent=(0.0, 0.0, 1.0, 1.0), flavor=DISCONTINUOUS):
    """Uniform nx-by-ny grid over ``extent = (x0, y0, lx, ly)`` (mesh.py:130-140)."""
    if nx < 1 or ny < 1:
        raise ConfigurationError(f"grid needs at least one cell per direction, got {nx}x{ny}")
    if flavor not in (DISCONTINUOUS, CONTINUOUS):
        raise ConfigurationError(f"unknown dof flavor {flavor!r}")
    x0, y0, lx, ly = (float(v) for v in extent)
    if lx <= 0 or ly <= 0:
        raise ConfigurationError(f"domain extent must be positive, got lx={lx}, ly={ly}")
    return Grid(int(nx), int(ny), x0, y0, lx / nx, ly / ny, flavor)


def dof_coordinates(grid):
    """Corner coordinates per dof, (n_dofs, 2) (mesh.py:251-265)."""
    jj, ii = np.divmod(np.arange(grid.n_cells), grid.nx)
    off = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    out = np.empty((grid.n_cells, 4, 2))
    out[:, :, 0] = (grid.x0 + ii * grid.dx)[:, None] + off[None, :, 0] * grid.dx
    out[:, :, 1] = (grid.y0 + jj * grid.dy)[:, None] + off[None, :, 1] * grid.dy
    return out.reshape(-1, 2)


def q1_reference():
    """Q1 reference-cell integrals (mesh.py:285-313), evaluated by 3-point
    Gauss so the fp64 values equal the reference's bit for bit."""
    x, w = np.polynomial.legendre.leggauss(3)
    pts, wts = 0.5 * (x + 1.0), 0.5 * w
    mass = np.zeros((4, 4))
    grad = [np.zeros((4, 4)), np.zeros((4, 4))]
    for xi, wx in zip(pts, wts):
        for eta, wy in zip(pts, wts):
            n = np.array([(1 - xi) * (1 - eta), xi * (1 - eta), (1 - xi) * eta, xi * eta])
            g = (np.array([-(1 - eta), (1 - eta), -eta, eta]),
                 np.array([-(1 - xi), -xi, (1 - xi), xi]))
            mass += wx * wy * np.outer(n, n)
            grad[0] += wx * wy * np.outer(g[0], n)
            grad[1] += wx * wy * np.outer(g[1], n)
    edge = np.array([[2.0, 1.0], [1.0, 2.0]]) / 6.0
    return {"mass": mass, "grad": grad, "edge": edge}


def cell_blocks(grid):
    """Scaled per-cell blocks exactly as transport_sn.py:211-216 forms them."""
    ref = q1_reference()
    mass = ref["mass"] * grid.dx * grid.dy
    return {
        "mass": mass,
        "gx": -grid.dy * ref["grad"][0],
        "gy": -grid.dx * ref["grad"][1],
        "e2x": grid.dy * ref["edge"],
        "e2y": grid.dx * ref["edge"],
        "src_row": mass.sum(axis=1),
    }


def cellops_struct(grid):
    """Fill the C struct ``dlrsn_cellops`` (include/dlrsn.h) for ``grid``."""
    from ._lib import CellOps

    b = cell_blocks(grid)
    s = CellOps()
    s.nx, s.ny = grid.nx, grid.ny
    s.x0, s.y0, s.dx, s.dy = grid.x0, grid.y0, grid.dx, grid.dy
    for name in ("mass", "gx", "gy", "e2x", "e2y", "src_row"):
        arr = np.ascontiguousarray(b[name], dtype=np.float64).ravel()
        getattr(s, name)[:] = arr.tolist()
    return s
