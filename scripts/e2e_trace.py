"""Timeline of bench.py's e2e loop (config 2 through the public API with host
buffers) under torch.profiler (CUPTI): writes a compact event list
(name, stream, start us, duration us) of kernels and memcpys for offline
analysis.  Usage: e2e_trace.py out.json [steps]"""
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main(out, steps=8):
    import bench
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(3):
        state, lin, T, _ = dp.step(state, lin, T, si_tol=1e-8)
    r = bench.measure_e2e(dp, state, T, lin, steps, None, warmup=3)
    print("untraced", json.dumps(r), flush=True)
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        r = bench.measure_e2e(dp, state, T, lin, steps, None, warmup=1)
    print("traced", json.dumps(r), flush=True)
    tmp = out + ".chrome.json"
    prof.export_chrome_trace(tmp)
    ev = json.load(open(tmp))["traceEvents"]
    keep = []
    for e in ev:
        if e.get("ph") != "X":
            continue
        cat = e.get("cat", "")
        if cat in ("kernel", "gpu_memcpy", "gpu_memset") or (
                cat == "cuda_runtime" and any(k in e["name"] for k in (
                    "Synchronize", "GraphLaunch", "Memcpy", "EventSynchronize"))):
            keep.append([e["name"][:60], cat, e.get("args", {}).get("stream", e.get("tid")),
                         round(float(e["ts"]), 2), round(float(e.get("dur", 0)), 2)])
    keep.sort(key=lambda x: x[3])
    json.dump(keep, open(out, "w"))
    os.remove(tmp)
    print("events", len(keep))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
