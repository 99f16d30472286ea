"""Device-resident DLR-SN time loop for the BASELINE configurations.

Restates the dlr-sn branch of the reference driver's loop
(driver.py:485-539: linearize -> step_collocation -> dofs_to_cells ->
update_temperature -> floor) with every per-cell array on the device, plus
the SURVEY Appendix B adapters (physical scattering / external source added
to the linearised step, T-dependent opacity, frozen coefficients for C5).
Host I/O, CSV output and energy diagnostics of the reference driver are out
of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device, device, empty, stream, zeros
from .angular import AngularBasis, build_quadrature, orthonormalize
from .errors import ContractViolation
from .lowrank import DlrState, gram_schmidt_mass, mass_gram
from .mesh import build_grid, cellops_struct
from .physics import LinearizedStep, PhysicsConstants, linearize
from .problems import ProblemSpec, draw_factors

FOUR_PI = 4.0 * np.pi


@dataclass(eq=False)
class DeviceProblem:
    spec: ProblemSpec
    grid: object
    quad: object
    constants: PhysicsConstants
    sigma_a0: torch.Tensor
    rho_cv: torch.Tensor
    ss_phys: torch.Tensor
    q_ext: torch.Tensor

    @classmethod
    def from_spec(cls, spec):
        grid = build_grid(spec.nx, spec.ny, spec.extent)
        quad = build_quadrature(spec.n_polar, spec.n_azimuthal)
        sa0 = spec.sigma_a if spec.opacity[0] == "constant" else np.full(spec.n_cells, spec.opacity[1])
        return cls(spec, grid, quad, PhysicsConstants(c=spec.c, a_r=spec.a_r), as_device(sa0),
                   as_device(spec.rho_cv), as_device(spec.sigma_s_phys), as_device(spec.q_ext))

    @property
    def opacity_power(self):
        return 0.0 if self.spec.opacity[0] == "constant" else float(self.spec.opacity[2])

    def linearized(self, T):
        """Linearised step at temperature T (physics.py:94-120 + adapters)."""
        T = as_device(T)
        if self.spec.frozen:
            st = linearize(T, as_device(self.spec.frozen_sigma_t) - 1.0 / (self.spec.c * self.spec.dt),
                           self.rho_cv, self.spec.dt, self.constants, check=False)
            st.sigma_t = as_device(self.spec.frozen_sigma_t)
            st.sigma_s = zeros(self.spec.n_cells)
            st.q = as_device(self.spec.frozen_q)
            return st
        sa = self.sigma_a0 if self.opacity_power == 0.0 else self.sigma_a0 * T ** self.opacity_power
        return linearize(T, sa, self.rho_cv, self.spec.dt, self.constants,
                         sigma_s_phys=self.ss_phys, q_ext=self.q_ext, check=False)

    def advance(self, lin, phi_dofs, T):
        """Finish a step (T update + floor, driver.py:532-534) and linearise
        the next one in a single fused pass (K4).  Updates ``T`` in place and
        returns the next LinearizedStep."""
        n = self.spec.n_cells
        if self.spec.frozen:
            # coefficients stay frozen (sigma_t, q; sigma_s = 0) but the next
            # step linearises about the new T (T0, denom, sigma_a of the
            # update_temperature formula, physics.py:94-132), as oracle/runner.py
            from .physics import update_temperature

            T.copy_(update_temperature(phi_dofs, lin, self.spec.t_floor))
            return self.linearized(T.clone())
        # one allocation for the next step's coefficients; the kernel reads
        # this step's sigma_a / denom and writes the new ones out of place
        buf = empty(6, n)
        sa, den, st, ss, q, T0 = buf.unbind(0)
        k = self.constants
        _lib.call("dlrsn_advance_relinearize", n, _lib.ptr(as_device(phi_dofs)), _lib.ptr(T),
                  _lib.ptr(lin.sigma_a), _lib.ptr(lin.denom), _lib.ptr(sa), _lib.ptr(self.sigma_a0),
                  self.opacity_power, _lib.ptr(self.rho_cv), float(self.spec.dt), float(k.c),
                  float(k.a_r), float(self.spec.t_floor), _lib.ptr(self.ss_phys),
                  _lib.ptr(self.q_ext), _lib.ptr(st), _lib.ptr(ss), _lib.ptr(q), _lib.ptr(den),
                  _lib.ptr(T0), None, stream())
        return LinearizedStep(sigma_t=st, sigma_s=ss, sigma_a=sa, q=q, T0=T0, denom=den,
                              rho_cv=self.rho_cv, dt=float(self.spec.dt),
                              inv_cdt=1.0 / (k.c * self.spec.dt), constants=k)


    def step(self, state, lin, T, *, si_tol=1e-8, si_max_iters=200, check_state=True,
             gs_method="cholqr2", comm=None, engine="native", x_new_host=None, use_dsa=False,
             dsa_penalty="simplified"):
        """One DLR step and the step boundary (T update + re-linearisation)
        in a single native call (the fused form of step_collocation +
        advance, driver.py:486-487,532-534).  Returns (state, next
        LinearizedStep, new T tensor, info); T itself is not modified, so a
        step that raises leaves the caller's state as it was."""
        from .dlr_sn import step_collocation

        if self.spec.frozen or engine != "native":
            state, info = step_collocation(self.grid, lin, self.quad, state, si_tol=si_tol,
                                           si_max_iters=si_max_iters, use_dsa=use_dsa,
                                           dsa_penalty=dsa_penalty,
                                           check_state=check_state, gs_method=gs_method,
                                           comm=comm, inflow=self.spec.inflow, engine=engine)
            T = T.clone()
            return state, self.advance(lin, info.phi, T), T, info
        n = self.spec.n_cells
        buf = empty(6, n)
        sa, den, st, ss, q, T0 = buf.unbind(0)
        av = self.__dict__.get("_adv")
        if av is None:
            k = self.constants
            av = _lib.Advance()
            av.n = n
            av.sigma_a0 = self.sigma_a0.data_ptr()
            av.opacity_power = float(self.opacity_power)
            av.rho_cv = self.rho_cv.data_ptr()
            av.dt, av.c, av.a_r = float(self.spec.dt), float(k.c), float(k.a_r)
            av.t_floor = float(self.spec.t_floor)
            av.ss_phys = None if self.ss_phys is None else self.ss_phys.data_ptr()
            av.q_ext = None if self.q_ext is None else self.q_ext.data_ptr()
            self._adv = av
        av.T_in, av.sigma_a_in, av.denom_in = T.data_ptr(), lin.sigma_a.data_ptr(), lin.denom.data_ptr()
        av.T_out, av.sigma_a, av.sigma_t = T0.data_ptr(), sa.data_ptr(), st.data_ptr()
        av.sigma_s, av.q, av.denom = ss.data_ptr(), q.data_ptr(), den.data_ptr()
        state, info = step_collocation(self.grid, lin, self.quad, state, si_tol=si_tol,
                                       si_max_iters=si_max_iters, use_dsa=use_dsa,
                                       dsa_penalty=dsa_penalty,
                                       check_state=check_state, gs_method=gs_method, comm=comm,
                                       inflow=self.spec.inflow, _advance=av,
                                       _x_new_host=x_new_host)
        k = self.constants
        nxt = LinearizedStep(sigma_t=st, sigma_s=ss, sigma_a=sa, q=q, T0=T0, denom=den,
                             rho_cv=self.rho_cv, dt=float(self.spec.dt),
                             inv_cdt=1.0 / (k.c * self.spec.dt), constants=k)
        return state, nxt, T0, info


def initial_state(dp, X=None, W=None, seed=None, T=None):
    """Seeded random-orthonormal X (M inner product, spatial-monomial
    completion) and W (weighted), S = (X^T M b0) beta^T.
    ``X`` / ``W`` may be given already orthonormal (e.g. by a test oracle)."""
    spec = dp.spec
    if X is None or W is None:
        rng = np.random.default_rng(spec.seed if seed is None else seed)
        Xr, Wr = draw_factors(spec, rng)
        co = cellops_struct(dp.grid)
        X, _, dx = gram_schmidt_mass(co, as_device(Xr), spec.rank + 8, method="cgs2")
        basis, _, dw = orthonormalize(as_device(Wr), dp.quad)
        if dx or dw:
            raise ContractViolation("random initial factors are rank deficient")
        W = basis
    X = as_device(X)
    W = W if isinstance(W, AngularBasis) else AngularBasis(values=W).bind(dp.quad)
    T = as_device(spec.T0 if T is None else T)
    k = dp.constants
    b0 = (k.a_r * k.c / FOUR_PI) * (T * T) ** 2
    b0 = b0.repeat_interleave(4).reshape(-1, 1)
    xb = mass_gram(cellops_struct(dp.grid), X, b0)[:, 0]
    S = torch.outer(xb, W.beta)
    return DlrState(X=X, S=S, W=W)


def initial_state_device(dp, seed=None, block_rows=1 << 22):
    """Seeded random-orthonormal factors generated on the device, for sizes
    whose N_x x r draw does not fit host memory comfortably (config 5: X is
    68.7 GB): X ~ N(0, 1) from a CUDA generator seeded with the config seed,
    M-orthonormalised by two in-place Cholesky-QR passes (a Gaussian block is
    well conditioned); W from numpy's default_rng(seed) and the weighted
    orthonormalisation; S = (X^T M b0) beta^T as in ``initial_state``.  The
    draws differ from ``initial_state``'s host draws (stated in the bench)."""
    from .lean import rowmix_inplace
    from .lowrank import _chol

    spec = dp.spec
    seed = spec.seed if seed is None else seed
    co = cellops_struct(dp.grid)
    gen = torch.Generator(device=device()).manual_seed(int(seed))
    X = torch.randn(spec.n_dofs, spec.rank, dtype=torch.float64, device=device(), generator=gen)
    for _ in range(2):
        _, Rinv, _, flag = _chol(mass_gram(co, X))
        rowmix_inplace(X, Rinv, block_rows)
    if int(flag.item()):
        raise ContractViolation("random initial factors are rank deficient")
    Wr = np.random.default_rng(seed).standard_normal((spec.n_angles, spec.rank))
    W, _, dw = orthonormalize(as_device(Wr), dp.quad)
    if dw:
        raise ContractViolation("random initial factors are rank deficient")
    T = as_device(spec.T0)
    k = dp.constants
    b0 = ((k.a_r * k.c / FOUR_PI) * (T * T) ** 2).repeat_interleave(4).reshape(-1, 1)
    S = torch.outer(mass_gram(co, X, b0)[:, 0], W.beta)
    return DlrState(X=X, S=S, W=W)


def run(dp, state, n_steps, *, si_tol=1e-8, si_max_iters=200, check_state=True, T=None,
        record=None, gs_method="cholqr2", engine="native", comm=None, diagnostics=None,
        use_dsa=False, dsa_penalty="simplified"):
    """n_steps of the dlr-sn loop; returns (state, T, infos).  With a list
    as ``diagnostics``, the reference driver's energy rows (driver.py:
    521-553, DIAGNOSTIC_COLUMNS order) are appended to it, evaluated on the
    factors (diagnostics.py)."""
    from .dlr_sn import step_collocation
    from .physics import update_temperature

    T = as_device(dp.spec.T0 if T is None else T).clone()
    lin = dp.linearized(T)
    infos = []
    ledger = None
    if diagnostics is not None:
        from .diagnostics import EnergyLedger

        ledger = EnergyLedger.start(dp.grid, dp.quad, dp.rho_cv, T, state.scalar_flux(),
                                    dp.constants.c, dp.spec.dt)
    for step_no in range(1, n_steps + 1):
        lin_used = lin
        if engine == "native":  # step + boundary in one native call
            state, lin, T, info = dp.step(state, lin, T, si_tol=si_tol, si_max_iters=si_max_iters,
                                          check_state=check_state, gs_method=gs_method, comm=comm,
                                          use_dsa=use_dsa, dsa_penalty=dsa_penalty)
        else:
            state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=si_tol,
                                           si_max_iters=si_max_iters, use_dsa=use_dsa,
                                           dsa_penalty=dsa_penalty,
                                           check_state=check_state, gs_method=gs_method,
                                           engine=engine, comm=comm, inflow=dp.spec.inflow)
            lin = dp.advance(lin, info.phi, T)
        infos.append(info)
        if ledger is not None:
            from .diagnostics import outflow_lowrank

            raw = update_temperature(info.phi, lin_used, -np.inf)
            diagnostics.append(ledger.row(step_no, info.iterations, info.interpolation_condition,
                                          T, raw, state.scalar_flux(),
                                          outflow_lowrank(dp.grid, state, dp.quad)))
        if record is not None:
            record(state, info, T)
    return state, T, infos


def run_sn(dp, n_steps, *, si_tol=1e-8, si_max_iters=200, use_dsa=True, dsa_penalty="simplified",
           T=None, record=None, diagnostics=None, comm=None, dedup=True):
    """The reference driver's full discrete-ordinates method ("sn",
    driver.py:463-466, 492-504): psi0 = B(T0) on every quadrature node, then
    per step the source iteration over ALL directions with the previous
    intensity as psi_time (sweeps grouped DW directions per warp), the
    temperature update and the floor.  psi (n_dofs x N_Omega) stays on the
    device.  Returns (psi, phi, T, iterations per step); ``diagnostics``
    as in ``run``.

    ``dedup`` (z-mirror deduplication): psi0 is isotropic, so
    nodes with equal (omega_x, omega_y) start equal, sweep the same operator
    (omega_z does not enter, transport_sn.py:143) with equal rhs, and stay
    bitwise equal every step; only the distinct pairs (half the nodes) are
    swept, with summed closure weights, and psi is expanded to every node
    on output."""
    from . import transport
    from .physics import planck, update_temperature

    spec = dp.spec
    quad = dp.quad
    T = as_device(spec.T0 if T is None else T).clone()
    b0, _ = planck(T.repeat_interleave(4), dp.constants)
    w_full = np.array(quad.weights, dtype=float)
    if dedup:
        om_sw, w_sw, inv = transport.dedup_mirrors(quad.omegas, w_full)
        inv_dev = torch.as_tensor(inv, device=device())
    else:
        om_sw, w_sw, inv_dev = quad.omegas, w_full, None
    psi = b0[:, None].repeat(1, om_sw.shape[0]).contiguous()
    w = torch.as_tensor(w_sw, device=device())
    phi = psi @ w

    def expand(p):
        return p if inv_dev is None else p[:, inv_dev]
    ledger = None
    if diagnostics is not None:
        from .diagnostics import EnergyLedger, outflow_dense

        ledger = EnergyLedger.start(dp.grid, quad, dp.rho_cv, T, phi, dp.constants.c, spec.dt)
    iters = []
    for step_no in range(1, n_steps + 1):
        lin = dp.linearized(T)
        ops = transport.assemble_operators(dp.grid, lin, dsa_penalty=dsa_penalty)
        res = transport.source_iteration(ops, om_sw, w_sw, psi_time=psi,
                                         use_dsa=use_dsa, tol=si_tol, max_iters=si_max_iters,
                                         phi_start=phi, inflow=spec.inflow, comm=comm)
        psi, phi = res.psi, res.phi
        raw = update_temperature(phi, lin, -np.inf)
        T = torch.clamp(raw, min=spec.t_floor)
        iters.append(res.iterations)
        if ledger is not None:
            diagnostics.append(ledger.row(step_no, res.iterations, 0.0, T, raw, psi @ w,
                                          outflow_dense(dp.grid, expand(psi), quad)))
        if record is not None:
            record(expand(psi), phi, T, res.iterations)
    return expand(psi), phi, T, iters
