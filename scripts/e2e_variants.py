"""Where bench.py's e2e time goes (config 2): the full e2e loop, the same
API loop without host copies, and the chained device loop."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(3):
        state, lin, T, _ = dp.step(state, lin, T, si_tol=1e-8)
    torch.cuda.synchronize()
    for rep in range(2):
        r = bench.measure_e2e(dp, state, T, lin, 20, None, warmup=3)
        print("e2e", round(r["ms_per_step"], 3), flush=True)

    def timed(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n

    box = {"s": state, "lin": lin, "T": T}

    def chained():
        box["s"], box["lin"], box["T"], _ = dp.step(box["s"], box["lin"], box["T"], si_tol=1e-8)

    print("chained dp.step", timed(chained), flush=True)
    s0, l0, T0 = box["s"], box["lin"], box["T"]

    def api_same_input():
        new, info = step_collocation(dp.grid, l0, dp.quad, s0, si_tol=1e-8, use_dsa=False)
        dp.advance(l0, info.phi, T0.clone())

    print("api same input (no copies)", timed(api_same_input), flush=True)

    def api_only():
        step_collocation(dp.grid, l0, dp.quad, s0, si_tol=1e-8, use_dsa=False)

    print("api step only", timed(api_only), flush=True)
    from paper_2601_18705_b200 import _lib
    t = []
    for _ in range(50):
        t0 = time.perf_counter()
        new, info = step_collocation(dp.grid, l0, dp.quad, s0, si_tol=1e-8, use_dsa=False)
        t.append(time.perf_counter() - t0)
    t.sort()
    print("api wall per call ms (median)", round(1e3 * t[len(t) // 2], 3), flush=True)


if __name__ == "__main__":
    main()
