"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
multi-strip sweeps through every sweep kernel (warp-specialised latency
kernel, the multi-warp kernel with 1 and 2 directions per warp, the
closure-only sweep) and two native DLR steps.  Kept tiny: the tools replay
every access."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2601_18705_b200 import problems, transport
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state
    from paper_2601_18705_b200.physics import LinearizedStep

    nx, ny = 40, 70  # three 32-row strips: the strip handoff runs
    n = nx * ny
    rng = np.random.default_rng(1)
    sig = np.exp(rng.uniform(-1, 3, n))
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.angular import build_quadrature

    grid = build_grid(nx, ny, (0.0, 0.0, 2.0, 3.0))
    st = LinearizedStep(sigma_t=sig, sigma_s=0.3 * sig, sigma_a=0.7 * sig, q=np.ones(n),
                        T0=np.zeros(n), denom=np.ones(n), rho_cv=np.ones(n), dt=1.0, inv_cdt=1.0)
    ops = transport.assemble_operators(grid, st)
    quad = build_quadrature(4, 8)
    psi_t = torch.rand(4 * n, quad.n_angles, dtype=torch.float64, device="cuda")
    for dw in (1, 2):
        res = transport.source_iteration(ops, quad.omegas, quad.weights, psi_time=psi_t,
                                         use_dsa=False, tol=1e-10, dw=dw)
    os.environ.setdefault("DLRSN_SWEEP_WS", "1")
    transport.sweep_solve(ops, quad.omegas[3], torch.rand(4 * n, dtype=torch.float64, device="cuda"))
    transport.closure_sweep(ops, quad.omegas, quad.weights,
                            torch.rand(4 * n, dtype=torch.float64, device="cuda"), dw=2)
    spec = problems.checkerboard(5, rank=6, n_polar=4, n_azimuthal=8, seed=3)
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(2):
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-10)
    torch.cuda.synchronize()
    print("ok", res.iterations, info.iterations)


if __name__ == "__main__":
    main()
