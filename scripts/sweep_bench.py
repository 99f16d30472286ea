"""Sweep-only timing of D directions on an n x n grid for several group
widths (K1 tuning).  Usage: sweep_bench.py n D [dw ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2601_18705_b200 import transport
    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.physics import LinearizedStep

    n, D = int(sys.argv[1]), int(sys.argv[2])
    dws = [int(x) for x in sys.argv[3:]] or [1, 2, 4]
    grid = build_grid(n, n, (0.0, 0.0, 1.0, 1.0))
    nc = grid.n_cells
    rng = np.random.default_rng(0)
    sig = np.exp(rng.uniform(0, 4, nc))
    one = np.ones(nc)
    st = LinearizedStep(sigma_t=sig, sigma_s=0.5 * sig, sigma_a=sig, q=one, T0=one, denom=one,
                        rho_cv=one, dt=1.0, inv_cdt=0.0)
    ops = transport.assemble_operators(grid, st)
    quad = build_quadrature(64, 64)
    sel = rng.choice(quad.n_angles, D, replace=False)
    om, w = quad.omegas[sel], quad.weights[sel]
    vl = ops.vec_len
    rhs = torch.rand(D * vl, dtype=torch.float64, device="cuda")
    psi = torch.empty_like(rhs)
    scat = torch.rand(4 * vl, dtype=torch.float64, device="cuda")
    alg = nc * (D * 64 + 160)
    for dw in dws:
        plan = transport._SweepPlan(ops, om, w, dw=dw)
        for tag, part in (("psi", None),):
            for _ in range(2):
                transport._sweep(ops, plan, rhs, psi, scat, part)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 5
            for _ in range(reps):
                transport._sweep(ops, plan, rhs, psi, scat, part)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"n={n} D={D} dw={plan.dw} G={plan.G} {tag}: {ms:.3f} ms, "
                  f"{alg / ms / 1e6:.0f} GB/s alg, {nc * D / ms / 1e6:.3e} cell-angle/s", flush=True)


if __name__ == "__main__":
    main()
