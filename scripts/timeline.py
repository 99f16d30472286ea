"""GPU timeline of a few C2 steps (torch.profiler / CUPTI): per-kernel device
time and the idle gaps between consecutive kernels, attributed to the kernel
that follows the gap.  Writes gpurun_out/timeline.json and prints a table."""

import json
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(steps=5):
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    engine = os.environ.get("ENGINE", "native")

    def one(state, lin):
        state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-8, use_dsa=False,
                                       engine=engine)
        return state, dp.advance(lin, info.phi, T), info

    for _ in range(3):
        state, lin, _ = one(state, lin)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            state, lin, _ = one(state, lin)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    rows = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda t: t[0])
    busy = defaultdict(float)
    gaps = defaultdict(float)
    cnt = defaultdict(int)
    prev_end = None
    for s, e, n in rows:
        busy[n] += e - s
        cnt[n] += 1
        if prev_end is not None and s > prev_end:
            gaps[n] += s - prev_end
        prev_end = max(prev_end or e, e)
    span = rows[-1][1] - rows[0][0]
    tot_busy = sum(busy.values())
    print(f"engine={engine} steps={steps} span={span / steps:.1f} us/step busy={tot_busy / steps:.1f} "
          f"idle={(span - tot_busy) / steps:.1f}")
    print(f"{'kernel':60s} {'n/step':>7s} {'us/step':>9s} {'gap-before us/step':>19s}")
    for n in sorted(busy, key=lambda k: -(busy[k] + gaps[k])):
        print(f"{n[:60]:60s} {cnt[n] / steps:7.1f} {busy[n] / steps:9.1f} {gaps[n] / steps:19.1f}")
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump({"rows": rows}, open(f"gpurun_out/timeline_{engine}.json", "w"))


if __name__ == "__main__":
    main()
