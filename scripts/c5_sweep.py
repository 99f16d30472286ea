"""Config 5's full-SN stress sweep: 128x128 = 16384 directions on the
4096^2 tile medium, closure only (psi is never stored), one sweep.
Usage: c5_sweep.py [n] [n_polar]  (defaults 4096, 128)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2601_18705_b200 import problems, transport
    from paper_2601_18705_b200.driver import DeviceProblem

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    npol = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    spec, fields = problems.stress(n=n, n_polar=npol, n_azimuthal=npol)
    fields(np.random.default_rng(spec.seed))
    t0 = time.time()
    dp = DeviceProblem.from_spec(spec)
    T = torch.as_tensor(spec.T0, device="cuda")
    lin = dp.linearized(T)
    ops = transport.assemble_operators(dp.grid, lin)
    b0 = (spec.a_r * spec.c / (4 * np.pi)) * (T * T) ** 2  # isotropic psi_old = B(T0)
    rhs = ops.source_vector(lin.q) + lin.inv_cdt * ops.mass_apply(b0.repeat_interleave(4))
    quad = dp.quad
    torch.cuda.synchronize()
    print(f"setup {time.time() - t0:.1f} s, {quad.n_angles} directions, {spec.n_cells} cells", flush=True)
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        phi = transport.closure_sweep(ops, quad.omegas, quad.weights, rhs, dw=int(os.environ.get("DW", "4")))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ca = spec.n_cells * quad.n_angles
        print(f"sweep {ms:.1f} ms: {ca / ms / 1e6:.3e} cell-angle/s, phi sum {float(phi.sum()):.6e}",
              flush=True)


if __name__ == "__main__":
    main()
