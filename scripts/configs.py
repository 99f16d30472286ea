"""Run a few native DLR steps of the BASELINE configurations that fit one
B200 (C1, C2, C3, C4; C5's 68.7 GB factors need space sharding) and print
per-step device time, source iterations and the sweep launch time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def spec_of(name):
    from paper_2601_18705_b200 import problems

    if name == "C1":
        return problems.config1()
    if name == "C2":
        return problems.config2()
    if name.startswith("C3"):
        n = int(name.split(":")[1]) if ":" in name else 512
        return problems.marshak(n=n)
    if name.startswith("C4"):
        n = int(name.split(":")[1]) if ":" in name else 1024
        spec, fields = problems.random_medium(n=n)
        rng = np.random.default_rng(spec.seed)
        problems.draw_factors(spec, rng)  # X, W first (SURVEY 8d draw order)
        fields(rng)
        return spec
    raise SystemExit(f"unknown config {name}")


def main():
    from paper_2601_18705_b200 import _lib
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    for name in sys.argv[1:] or ["C1", "C2", "C4"]:
        spec = spec_of(name)
        t0 = time.time()
        dp = DeviceProblem.from_spec(spec)
        state = initial_state(dp)
        T = torch.as_tensor(spec.T0, device="cuda").clone()
        lin = dp.linearized(T)
        setup = time.time() - t0
        steps = int(os.environ.get("STEPS", "12"))
        times, iters = [], []
        for k in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            iters.append(info.iterations)
        _lib.call("dlrsn_sweep_timing", 1)
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
        torch.cuda.synchronize()
        import ctypes
        cap = 256
        ms = (ctypes.c_float * cap)(); g = (ctypes.c_int * cap)(); dw = (ctypes.c_int * cap)()
        cnt = ctypes.c_int()
        _lib.call("dlrsn_sweep_timing_read", cap, ms, g, dw, ctypes.byref(cnt))
        _lib.call("dlrsn_sweep_timing", 0)
        if os.environ.get("PROFILE"):
            state, lin, T = profile_step(dp, state, lin, T)
        sweep = sum(ms[i] for i in range(min(cnt.value, cap))) / max(1, info.iterations)
        nc = spec.n_cells
        alg = nc * (spec.rank * 64 + 160)
        print(f"{name}: {spec.nx}x{spec.ny} r={spec.rank} N_omega={dp.quad.n_angles}: "
              f"step {np.median(times[steps // 2:]):.3f} ms (min {min(times):.3f}, first {times[0]:.1f}), "
              f"SI iters {iters}, sweep {sweep:.3f} ms = {nc * spec.rank / sweep * 1e3:.3e} "
              f"cell-direction/s, {alg / sweep / 1e6:.0f} GB/s alg; setup {setup:.1f} s; "
              f"peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")


def profile_step(dp, state, lin, T):
    from torch.profiler import ProfilerActivity, profile
    from collections import defaultdict

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
        torch.cuda.synchronize()
    busy, cnt = defaultdict(float), defaultdict(int)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            busy[e.name] += e.time_range.end - e.time_range.start
            cnt[e.name] += 1
    for n in sorted(busy, key=lambda k: -busy[k])[:14]:
        print(f"    {n[:56]:56s} {cnt[n] / 2:6.1f} {busy[n] / 2:10.1f} us/step")
    return state, lin, T


if __name__ == "__main__":
    main()
