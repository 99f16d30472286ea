"""Run a few DLR steps of a BASELINE config (native engine, fused step
boundary) -- the target of the ncu launch lists in profiles/.
Usage: config_steps.py C4 [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(name, steps):
    import bench
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = bench.make_spec(name)
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(steps):
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
    torch.cuda.synchronize()
    print("ok", info.iterations)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C4", int(sys.argv[2]) if len(sys.argv) > 2 else 3)
