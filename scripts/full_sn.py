"""One config-2 full-SN sweep (1024 directions) -- target for ncu / timing."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2601_18705_b200 import problems, transport
    from paper_2601_18705_b200.driver import DeviceProblem

    dp = DeviceProblem.from_spec(problems.config2())
    T = torch.as_tensor(dp.spec.T0, device="cuda")
    ops = transport.assemble_operators(dp.grid, dp.linearized(T))
    quad = dp.quad
    dw = int(os.environ.get("DW", "0")) or None
    plan = transport._SweepPlan(ops, quad.omegas, quad.weights, dw=dw)
    vl = ops.vec_len
    rhs = torch.rand(quad.n_angles * vl, dtype=torch.float64, device="cuda")
    psi = torch.empty_like(rhs)
    part = torch.empty(plan.G * vl, dtype=torch.float64, device="cuda")
    scat = torch.zeros(4 * vl, dtype=torch.float64, device="cuda")
    for _ in range(int(os.environ.get("REPS", "3"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        transport._sweep(ops, plan, rhs, psi, scat, part)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        nc = dp.grid.n_cells
        alg = nc * (quad.n_angles * 64 + 160)
        print(f"dw={plan.dw} G={plan.G} ms={ms:.3f} GB/s={alg / ms / 1e6:.0f}")


if __name__ == "__main__":
    main()
