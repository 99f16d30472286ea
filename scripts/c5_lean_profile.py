"""Config 5's DLR step on one GPU (lean engine) with the per-phase device
timing of lean.py (DLRSN_LEAN_PROFILE=1, printed to stderr)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DLRSN_LEAN_PROFILE", "1")


def main(steps=2):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state_device

    spec, fields = problems.stress()
    fields(np.random.default_rng(spec.seed))
    dp = DeviceProblem.from_spec(spec)
    state = initial_state_device(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for k in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8, engine="lean")
        e1.record()
        torch.cuda.synchronize()
        print(f"step {k}: {e0.elapsed_time(e1):.1f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
