"""Timeline of one sweep launch: per work item (group, strip) chunk phases.
t0 chunk start, t1 after TMA issue, t2 after handoff, t3 after mbarrier wait."""
import os, sys, ctypes
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18705_b200 import transport as Tr, _lib
from paper_2601_18705_b200.mesh import build_grid
from paper_2601_18705_b200.physics import LinearizedStep
from paper_2601_18705_b200.angular import build_quadrature

n, D, dw = [int(v) for v in sys.argv[1:4]]
ny = int(sys.argv[4]) if len(sys.argv) > 4 else n
flags = int(sys.argv[5]) if len(sys.argv) > 5 else 0
rng = np.random.default_rng(0)
nc = n * ny
sig = rng.uniform(0.5, 50, nc)
st = LinearizedStep(sigma_t=sig, sigma_s=0.5 * sig, sigma_a=sig, q=rng.uniform(0, 1, nc), T0=np.zeros(nc),
                    denom=np.ones(nc), rho_cv=np.ones(nc), dt=1.0, inv_cdt=0.5)
ops = Tr.assemble_operators(build_grid(n, ny), st)
quad = build_quadrature(4, 2 * ((D + 7) // 8))
plan = Tr._SweepPlan(ops, quad.omegas[:D], quad.weights[:D], dw=dw)
vl = ops.vec_len
rhs = torch.rand(D * vl, dtype=torch.float64, device='cuda'); psi = torch.empty_like(rhs)
part = torch.empty(plan.G * vl, dtype=torch.float64, device='cuda'); scat = torch.rand(4 * vl, dtype=torch.float64, device='cuda')
_lib.call("dlrsn_debug_flags", flags)
Tr._sweep(ops, plan, rhs, psi, scat, part); torch.cuda.synchronize()
C = {1: 4, 2: 2, 4: 2, 8: 1}[plan.dw]
chunks = (n + 31 + C - 1) // C
ns = (ny + 31) // 32
buf = torch.zeros(ns * plan.G * chunks * 4, dtype=torch.int64, device='cuda')
_lib.call("dlrsn_debug_trace", ctypes.c_void_p(buf.data_ptr()), chunks)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); Tr._sweep(ops, plan, rhs, psi, scat, part); e1.record(); torch.cuda.synchronize()
print("flags", flags, "launch ms", e0.elapsed_time(e1))
_lib.call("dlrsn_debug_trace", None, 0)
t = buf.cpu().numpy().reshape(ns, plan.G, chunks, 4).astype(np.float64)
t = (t - t[t > 0].min()) / 1e3  # us
for s in list(range(min(ns, 3))) + ([ns - 1] if ns > 3 else []):
    x = t[s, 0]
    tma = x[:, 1] - x[:, 0]; hand = x[:, 2] - x[:, 1]; mb = x[:, 3] - x[:, 2]; comp = x[1:, 0] - x[:-1, 3]
    print(f"strip {s}: t0 {x[0,0]:7.1f} end {x[-1,3]:8.1f} us | median tma {np.median(tma):.2f} hand {np.median(hand):.2f} "
          f"mbar {np.median(mb):.2f} compute {np.median(comp):.2f} | sums tma {tma.sum():.0f} hand {hand.sum():.0f} mbar {mb.sum():.0f} comp {comp.sum():.0f}")
