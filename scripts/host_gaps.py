"""Host-side time per C2 step outside the native call: wall time of the
Python around dlrsn_step_collocation, the advance call and the loop."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=30):
    from paper_2601_18705_b200 import dlr_sn, problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    marks = []
    orig = dlr_sn._NativeCtx.__init__

    def wrap_ctx(self, *a, **k):
        orig(self, *a, **k)
        fn = self.fn

        def timed(*args):
            t0 = time.perf_counter()
            rc = fn(*args)
            marks.append((t0, time.perf_counter()))
            return rc
        self.fn = timed

    dlr_sn._NativeCtx.__init__ = wrap_ctx
    dlr_sn._CTX.clear()
    t_adv = []
    t_step = []
    for k in range(steps):
        a = time.perf_counter()
        state, info = dlr_sn.step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-8, use_dsa=False)
        b = time.perf_counter()
        lin = dp.advance(lin, info.phi, T)
        c = time.perf_counter()
        t_step.append((a, b))
        t_adv.append((b, c))
    torch.cuda.synchronize()
    sk = 5
    pre = [m[0] - s[0] for m, s in zip(marks[sk:], t_step[sk:])]
    call = [m[1] - m[0] for m in marks[sk:]]
    post = [s[1] - m[1] for m, s in zip(marks[sk:], t_step[sk:])]
    adv = [c - b for b, c in t_adv[sk:]]
    gap = [t_step[i + 1][0] - t_adv[i][1] for i in range(sk, steps - 1)]
    tot = [t_step[i + 1][0] - t_step[i][0] for i in range(sk, steps - 1)]
    us = lambda v: f"{1e6 * np.median(v):8.1f}"
    print("median us: pre-call", us(pre), "native call", us(call), "post-call", us(post),
          "advance", us(adv), "loop", us(gap), "total/step", us(tot))


if __name__ == "__main__":
    main()
