"""GPU vs the CPU oracle in lock step for the BASELINE configs' full step
counts (north_star: 1e-11 after the stated number of steps) -- too long for
the test suite, run once on the GPU box and committed as evidence
(profiles/r02_parity_long_*.json).  Same protocol as
tests/test_gpu_baseline_parity.py (si_tol 1e-12, identical picks / SI /
deficiency counts, rel-L2 on info.phi, T and X S W^T every step).

Usage: parity_long.py C3 100 out.json   (C3: Marshak 512^2 from T0 = 1e-4)
       parity_long.py C4 10 out.json"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "tests"))


def main(name, steps, out):
    from test_gpu_baseline_parity import TOL, _lockstep
    from paper_2601_18705_b200 import problems

    if name == "C3":
        spec = problems.marshak()
    elif name == "C4":
        spec, fields = problems.random_medium()
        rng = np.random.default_rng(spec.seed)
        problems.draw_factors(spec, rng)
        fields(rng)
    elif name == "C2":
        spec = problems.config2()
    else:
        raise SystemExit(f"unknown config {name}")
    t0 = time.time()
    recs = []
    try:
        _lockstep(spec, steps, check=lambda r: recs.append(r))
    finally:
        ok = all(r["picks"] and r["iters"][0] == r["iters"][1] and r["sdef"][0] == r["sdef"][1]
                 and r["adef"][0] == r["adef"][1] and max(r["phi"], r["T"], r["xsw"]) <= TOL
                 for r in recs)
        summary = {
            "config": name, "steps_run": len(recs), "steps_requested": steps, "all_within": ok,
            "tol": TOL, "max_phi": max((r["phi"] for r in recs), default=None),
            "max_T": max((r["T"] for r in recs), default=None),
            "max_xsw": max((r["xsw"] for r in recs), default=None),
            "picks_all_equal": all(r["picks"] for r in recs),
            "iters_all_equal": all(r["iters"][0] == r["iters"][1] for r in recs),
            "si_iterations": [r["iters"][0] for r in recs],
            "seconds": time.time() - t0, "records": recs,
        }
        with open(out, "w") as fh:
            json.dump(summary, fh, indent=1, default=str)
        print(json.dumps({k: v for k, v in summary.items() if k != "records"}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
