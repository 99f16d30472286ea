"""Run a few C2 DLR steps (native engine) -- target for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=int(os.environ.get("STEPS", "2"))):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(steps):
        state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-8, use_dsa=False)
        lin = dp.advance(lin, info.phi, T)
    torch.cuda.synchronize()
    print("ok", info.iterations)


if __name__ == "__main__":
    main()
