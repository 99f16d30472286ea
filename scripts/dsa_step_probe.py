"""DSA inside the native step at scale: a BASELINE config whose angular
basis holds the constant (closure sum 4 pi, so the reference's DSA
converges) and whose scattering is scaled up, stepped with and without
use_dsa.  Prints per-step device time, source-iteration counts and PCG
iterations.  Usage: dsa_step_probe.py C2|C4 [steps] [scatter_scale]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(name, steps, scale):
    import bench
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = bench.make_spec(name)
    spec.sigma_s_phys = spec.sigma_s_phys * scale
    rng = np.random.default_rng(spec.seed)
    Xr, Wr = problems.draw_factors(spec, rng)
    Wr[:, 0] = 1.0
    dp = DeviceProblem.from_spec(spec)
    from paper_2601_18705_b200._device import as_device
    from paper_2601_18705_b200.angular import orthonormalize
    from paper_2601_18705_b200.lowrank import gram_schmidt_mass
    from paper_2601_18705_b200.mesh import cellops_struct

    X, _, _ = gram_schmidt_mass(cellops_struct(dp.grid), as_device(Xr), spec.rank + 8, method="cgs2")
    W, _, _ = orthonormalize(as_device(Wr), dp.quad)
    for dsa in (False, True):
        state = initial_state(dp, X=X, W=W)
        T = torch.as_tensor(spec.T0, device="cuda").clone()
        lin = dp.linearized(T)
        rows = []
        for k in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8, si_max_iters=2000, use_dsa=dsa)
            e1.record()
            torch.cuda.synchronize()
            rows.append((round(e0.elapsed_time(e1), 2), info.iterations,
                         getattr(info, "dsa_iterations", 0)))
        print(f"{name} scatter x{scale} use_dsa={dsa}: (ms, SI iterations, PCG iterations) per step {rows}",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 4,
         float(sys.argv[3]) if len(sys.argv) > 3 else 1.0)
