"""Quick device timing of one sweep launch at several sizes (dev probe)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2601_18705_b200 import transport as Tr
from paper_2601_18705_b200.mesh import build_grid
from paper_2601_18705_b200.physics import LinearizedStep
from paper_2601_18705_b200.angular import build_quadrature

def run(n, D, dw=None, reps=5, ny=None):
    rng = np.random.default_rng(0)
    ny = n if ny is None else ny
    nc = n * ny
    sig = rng.uniform(0.5, 50, nc)
    st = LinearizedStep(sigma_t=sig, sigma_s=0.5 * sig, sigma_a=sig, q=rng.uniform(0, 1, nc), T0=np.zeros(nc),
                        denom=np.ones(nc), rho_cv=np.ones(nc), dt=1.0, inv_cdt=0.5)
    grid = build_grid(n, ny, (0, 0, 1, 1))
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
    print(f"n={n}x{ny} D={D} dw={plan.dw} G={plan.G} ms={ms:.3f} cell-angle/s={ca/(ms*1e-3):.3e} alg GB/s={gbs:.0f}", flush=True)

if __name__ == "__main__" and len(sys.argv) > 1:
    a = [int(v) for v in sys.argv[1:]]
    run(a[0], a[1], a[2] if len(a) > 2 and a[2] > 0 else None, reps=a[3] if len(a) > 3 else 5,
        ny=a[4] if len(a) > 4 else None)
    sys.exit(0)
for args in [(4096, 1, 1, 3, 32), (4096, 4, 1, 3, 32), (4096, 148, 1, 3, 32), (4096, 592, 1, 3, 32), (4096, 8, 8, 3, 32), (4096, 64, 2, 3, 32), (70, 8), (280, 16), (280, 16, 2), (280, 16, 4), (280, 1024), (280, 1024, 4), (280, 1024, 2), (1024, 64), (1024, 64, 2), (1024, 64, 4), (512, 32)]:
    run(*args)
