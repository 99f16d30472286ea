"""cProfile of the C2 step loop (native engine): where the host time goes
outside the one C-ABI call."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=20):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)

    def loop(k, state, lin):
        for _ in range(k):
            state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-8, use_dsa=False)
            lin = dp.advance(lin, info.phi, T)
        torch.cuda.synchronize()
        return state, lin

    state, lin = loop(3, state, lin)
    pr = cProfile.Profile()
    pr.enable()
    loop(steps, state, lin)
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
