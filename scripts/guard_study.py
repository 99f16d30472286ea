"""CholQR2 guard study: native steps vs the oracle for a few ranks, printing
the state difference and the fallback bits (run with DLRSN_GUARD_RATIO /
DLRSN_GUARD_DEBUG set)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import port as P
    from oracle import runner as R
    from paper_2601_18705_b200 import problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state, run

    cases = [(4, 64, 8, 16, 3), (3, 40, 6, 12, 3), (6, 32, 8, 8, 3), (10, 8, 16, 16, 4), (8, 16, 16, 16, 3)]
    for pb, r, npol, naz, steps in cases:
        spec = problems.checkerboard(pb, rank=r, n_polar=npol, n_azimuthal=naz, seed=13, n_steps=steps)
        rng = np.random.default_rng(spec.seed)
        Xr, Wr = problems.draw_factors(spec, rng)
        X, W = R.orthonormal_factors(spec, Xr, Wr)
        ref = []
        R.run(spec, R.initial_state(spec, X, W), steps, record=lambda s, i, t: ref.append((s, i, t)))
        dp = DeviceProblem.from_spec(spec)
        got = []
        run(dp, initial_state(dp, X=X, W=W), steps, si_tol=1e-12, si_max_iters=400,
            record=lambda s, i, t: got.append((s, i)))
        for k, ((rs, ri, rt), (gs, gi)) in enumerate(zip(ref, got)):
            X2, S2, W2 = gs.to_numpy()
            d = P.lowrank_rel_diff(X2, S2, W2, rs.X, rs.S, rs.W)
            print(f"pb={pb} r={r} step {k}: fallback={gi.gs_fallback} diff={d:.2e}", flush=True)


if __name__ == "__main__":
    main()
