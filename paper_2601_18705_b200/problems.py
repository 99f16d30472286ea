"""Seeded synthetic inputs for the BASELINE.json configurations.

Host-side input generation only (numpy); the reference has no such presets
for these configs, so the recipes follow SURVEY.md Appendix B and
BASELINE.md section 5.  Physical scattering and external sources are
injected into the linearised step exactly as the reference's own tests do
(``pkg/tests/test_transport_sn.py:22-36``): start from ``linearize`` and add
``sigma_s_phys`` to sigma_t and sigma_s and ``q_ext`` to q.

Seeds: ``numpy.random.default_rng(seed)``, draws in the order X, W, then the
random fields.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FOUR_PI = 4.0 * np.pi

# non-centre blocks of the reference lattice preset (driver.py:592-593)
CHECKER_ABSORBERS = frozenset({(1, 1), (1, 3), (1, 5), (2, 2), (2, 4), (3, 1), (3, 5),
                               (4, 2), (4, 4), (5, 1), (5, 3), (5, 5)})


@dataclass(eq=False)
class ProblemSpec:
    """Everything one DLR-SN run needs, as plain host arrays."""

    name: str
    nx: int
    ny: int
    extent: tuple  # (x0, y0, lx, ly)
    n_polar: int
    n_azimuthal: int
    rank: int
    dt: float
    n_steps: int
    T0: np.ndarray  # (n_cells,)
    rho_cv: np.ndarray
    sigma_a: np.ndarray  # opacity at T0 (constant unless ``opacity`` says otherwise)
    sigma_s_phys: np.ndarray
    q_ext: np.ndarray
    c: float = 1.0
    a_r: float = 1.0
    seed: int = 0
    opacity: tuple = ("constant",)  # or ("power", sigma0, p): sigma_a = sigma0 * T**p
    frozen: bool = False  # C5: coefficients fixed, not re-linearised each step
    frozen_sigma_t: np.ndarray | None = None
    frozen_q: np.ndarray | None = None
    t_floor: float = 1e-6
    inflow: tuple | None = None  # isotropic inflow psi_b (left, right, bottom, top); None: vacuum
    notes: dict = field(default_factory=dict)

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def n_dofs(self):
        return 4 * self.nx * self.ny

    @property
    def n_angles(self):
        return self.n_polar * self.n_azimuthal

    @property
    def dx(self):
        return self.extent[2] / self.nx

    @property
    def dy(self):
        return self.extent[3] / self.ny

    def opacity_at(self, T):
        if self.opacity[0] == "constant":
            return self.sigma_a
        _, s0, p = self.opacity
        return s0 * np.asarray(T, dtype=float) ** p

    def cell_centers(self):
        x0, y0, lx, ly = self.extent
        jj, ii = np.divmod(np.arange(self.n_cells), self.nx)
        return np.column_stack([x0 + (ii + 0.5) * self.dx, y0 + (jj + 0.5) * self.dy])


def draw_factors(spec, rng):
    """Raw (not yet orthonormal) factor draws, in the order X then W."""
    X = rng.standard_normal((spec.n_dofs, spec.rank))
    W = rng.standard_normal((spec.n_angles, spec.rank))
    return X, W


def checkerboard(per_block=10, rank=8, n_polar=16, n_azimuthal=16, dt=0.01, n_steps=20,
                 seed=1, name="C1", blocks=7):
    """C1/C2: 7x7-block checkerboard on [0,7]^2 (BASELINE configs[0..1])."""
    n = blocks * per_block
    spec = _empty(name, n, n, (0.0, 0.0, float(blocks), float(blocks)), n_polar, n_azimuthal,
                  rank, dt, n_steps, seed)
    cc = spec.cell_centers()
    bi = np.floor(cc[:, 0]).astype(int)
    bj = np.floor(cc[:, 1]).astype(int)
    absorber = np.array([(a, b) in CHECKER_ABSORBERS for a, b in zip(bi, bj)])
    centre = (bi == blocks // 2) & (bj == blocks // 2)
    spec.sigma_a = np.where(absorber, 10.0, 0.0)
    spec.sigma_s_phys = np.where(absorber, 0.0, 1.0)
    spec.q_ext = np.where(centre, 1.0 / FOUR_PI, 0.0)
    spec.T0 = np.full(spec.n_cells, 1e-3)
    return spec


def config1():
    return checkerboard(10, rank=8, n_polar=16, n_azimuthal=16, dt=0.01, n_steps=20, seed=1,
                        name="C1")


def config2():
    return checkerboard(40, rank=16, n_polar=32, n_azimuthal=32, dt=0.01, n_steps=50, seed=2,
                        name="C2")


def marshak(n=512, rank=32, n_polar=64, n_azimuthal=64, dt=1e-3, n_steps=100, seed=3,
            sigma0=300.0, T_b=1.0, T_init=1e-4, name="C3"):
    """C3: Marshak wave in [0,1]^2: sigma_a = sigma0 T^-3 (explicit in T, the
    linearisation point of each step), isotropic inflow at
    T_b on the left wall, psi_b = a c T_b^4 / (4 pi), vacuum
    elsewhere, T0 = 1e-4, c = a = rho c_v = 1, no physical scattering or
    external source."""
    spec = _empty(name, n, n, (0.0, 0.0, 1.0, 1.0), n_polar, n_azimuthal, rank, dt, n_steps,
                  seed)
    spec.T0 = np.full(spec.n_cells, float(T_init))
    spec.opacity = ("power", float(sigma0), -3.0)
    spec.sigma_a = spec.opacity_at(spec.T0)
    spec.inflow = (spec.a_r * spec.c * T_b ** 4 / FOUR_PI, 0.0, 0.0, 0.0)
    return spec


def config3():
    return marshak()


def random_medium(n=1024, rank=64, n_polar=64, n_azimuthal=64, dt=1e-2, n_steps=50, seed=4,
                  corr=8.0, name="C4"):
    """C4: log-normal smoothed opacity, sigma_s = 0.5 sigma_a, Gaussian hot spot."""
    from scipy.ndimage import gaussian_filter

    spec = _empty(name, n, n, (0.0, 0.0, 1.0, 1.0), n_polar, n_azimuthal, rank, dt, n_steps,
                  seed)
    spec.notes["corr_cells"] = corr
    return spec, (lambda rng: _random_medium_fields(spec, rng, corr, gaussian_filter))


def _random_medium_fields(spec, rng, corr, gaussian_filter):
    g = rng.standard_normal((spec.ny, spec.nx))
    g = gaussian_filter(g, sigma=corr, mode="wrap")
    g = (g - g.mean()) / g.std()
    sa = np.exp(1.5 * g).ravel()
    spec.sigma_a = sa
    spec.sigma_s_phys = 0.5 * sa
    spec.q_ext = np.zeros(spec.n_cells)
    cc = spec.cell_centers()
    r2 = (cc[:, 0] - 0.5) ** 2 + (cc[:, 1] - 0.5) ** 2
    w = 0.05
    spec.T0 = 1e-3 + (1.0 - 1e-3) * np.exp(-r2 / (2 * w * w))


def stress(n=4096, rank=128, n_polar=128, n_azimuthal=128, tile=64, n_steps=10, seed=5,
           name="C5"):
    """C5: piecewise-constant random sigma_t on tile x tile blocks, random
    source, pure absorber, dx = 1, dt = 1, c = 1 (fixed coefficients)."""
    spec = _empty(name, n, n, (0.0, 0.0, float(n), float(n)), n_polar, n_azimuthal, rank, 1.0,
                  n_steps, seed)
    spec.frozen = True
    return spec, (lambda rng: _stress_fields(spec, rng, tile))


def _stress_fields(spec, rng, tile):
    nt = spec.nx // tile
    tiles = np.exp(rng.uniform(np.log(0.1), np.log(100.0), (nt, nt)))
    sa = np.kron(tiles, np.ones((tile, tile))).ravel()
    q = rng.uniform(0.0, 1.0, spec.n_cells)
    spec.sigma_a = sa
    spec.sigma_s_phys = np.zeros(spec.n_cells)
    spec.q_ext = np.zeros(spec.n_cells)
    spec.frozen_sigma_t = sa + 1.0 / (spec.c * spec.dt)
    spec.frozen_q = q


def _empty(name, nx, ny, extent, n_polar, n_azimuthal, rank, dt, n_steps, seed):
    nc = nx * ny
    z = np.zeros(nc)
    return ProblemSpec(name=name, nx=nx, ny=ny, extent=extent, n_polar=n_polar,
                       n_azimuthal=n_azimuthal, rank=rank, dt=dt, n_steps=n_steps,
                       T0=np.full(nc, 1e-3), rho_cv=np.ones(nc), sigma_a=z.copy(),
                       sigma_s_phys=z.copy(), q_ext=z.copy(), seed=seed)
