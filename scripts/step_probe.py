"""Per-step device time, SI iterations and Gram-Schmidt path of a BASELINE
config (native engine): step_probe.py C3 [steps]"""
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
    for k in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
        e1.record()
        torch.cuda.synchronize()
        print(f"step {k}: {e0.elapsed_time(e1):8.3f} ms  it {info.iterations:3d}  "
              f"gs_fallback {getattr(info, 'gs_fallback', '?')}  "
              f"def {info.spatial_deficiency}/{info.angular_deficiency}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else 14)
