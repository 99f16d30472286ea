"""A/B timing of the chained C2 step (dp.step), with and without an L2
flush between steps.  Run once per library build (DLRSN_LIB=...)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(n=50):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(5):
        state, lin, T, _ = dp.step(state, lin, T, si_tol=1e-8)
    for mode in ("flush", "noflush", "flush", "noflush"):
        tot = 0.0
        for k in range(n):
            if mode == "flush":
                flush.fill_(float(k))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            state, lin, T, _ = dp.step(state, lin, T, si_tol=1e-8)
            e1.record()
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        print(os.environ.get("DLRSN_LIB", "new"), mode, round(tot / n, 4), flush=True)


if __name__ == "__main__":
    main()
