"""Quick device timing of one sweep launch at several sizes (dev probe)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2601_18705_b200 import transport as Tr
from paper_2601_18705_b200.mesh import build_grid
from paper_2601_18705_b200.physics import LinearizedStep
from paper_2601_18705_b200.angular import build_quadrature

def run(n, D, dw=None, reps=5):
    rng = np.random.default_rng(0)
    nc = n * n
    sig = rng.uniform(0.5, 50, nc)
    st = LinearizedStep(sigma_t=sig, sigma_s=0.5 * sig, sigma_a=sig, q=rng.uniform(0, 1, nc), T0=np.zeros(nc),
                        denom=np.ones(nc), rho_cv=np.ones(nc), dt=1.0, inv_cdt=0.5)
    grid = build_grid(n, n, (0, 0, 1, 1))
    ops = Tr.assemble_operators(grid, st)
    quad = build_quadrature(4, 2 * ((D + 7) // 8))
    om = quad.omegas[:D]
    clo = quad.weights[:D]
    plan = Tr._SweepPlan(ops, om, clo, dw=dw)
    vl = ops.vec_len
    rhs = torch.rand(D * vl, dtype=torch.float64, device='cuda')
    psi = torch.empty_like(rhs)
    part = torch.empty(plan.G * vl, dtype=torch.float64, device='cuda')
    scat = torch.rand(4 * vl, dtype=torch.float64, device='cuda')
    for _ in range(2):
        Tr._sweep(ops, plan, rhs, psi, scat, part)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        Tr._sweep(ops, plan, rhs, psi, scat, part)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ca = nc * D
    gbs = ca * 64 / (ms * 1e-3) / 1e9
    print(f"n={n} D={D} dw={plan.dw} G={plan.G} ms={ms:.3f} cell-angle/s={ca/(ms*1e-3):.3e} alg GB/s={gbs:.0f}", flush=True)

for args in [(70, 8), (280, 16), (280, 16, 2), (280, 16, 4), (280, 1024), (280, 1024, 4), (280, 1024, 2), (1024, 64), (1024, 64, 2), (1024, 64, 4), (512, 32)]:
    run(*args)
