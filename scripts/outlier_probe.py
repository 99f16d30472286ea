"""Chained C4 steps exactly as bench.py times them (L2 flush, CUDA events
around DeviceProblem.step), with the caching allocator's device-allocation
counters per step: finds the cause of occasional slow timed steps."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(n=40, lms=0):
    import bench
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = bench.make_spec("C4")
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    proc = None
    if lms:  # nvidia-smi polling as bench.ClockSampler does it
        import subprocess
        proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={bench.ClockSampler.Q}",
                                 "--format=csv,noheader,nounits", "-lms", str(lms)],
                                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        time.sleep(2.0)
    for k in range(n):
        flush.fill_(float(k))
        m0 = torch.cuda.memory_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        m1 = torch.cuda.memory_stats()
        print(f"step {k:2d}: {e0.elapsed_time(e1):7.2f} ms gpu, {1e3 * (t1 - t0):7.2f} ms host, "
              f"it {info.iterations}, device allocs +{m1['num_device_alloc'] - m0['num_device_alloc']}, "
              f"frees +{m1['num_device_free'] - m0['num_device_free']}, "
              f"retries +{m1['num_alloc_retries'] - m0['num_alloc_retries']}", flush=True)


    if proc is not None:
        proc.terminate()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
