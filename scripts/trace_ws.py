"""Timeline of the warp-specialised sweep: consumer wait/compute vs producers."""
import os, sys, ctypes
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18705_b200 import transport as Tr, _lib
from paper_2601_18705_b200.mesh import build_grid
from paper_2601_18705_b200.physics import LinearizedStep
from paper_2601_18705_b200.angular import build_quadrature
n, D, ny = [int(v) for v in sys.argv[1:4]]
C = 6
rng = np.random.default_rng(0)
nc = n * ny
sig = rng.uniform(0.5, 50, nc)
st = LinearizedStep(sigma_t=sig, sigma_s=0.5 * sig, sigma_a=sig, q=rng.uniform(0, 1, nc), T0=np.zeros(nc),
                    denom=np.ones(nc), rho_cv=np.ones(nc), dt=1.0, inv_cdt=0.5)
ops = Tr.assemble_operators(build_grid(n, ny), st)
quad = build_quadrature(4, 2 * ((D + 7) // 8))
plan = Tr._SweepPlan(ops, quad.omegas[:D], quad.weights[:D], dw=1)
vl = ops.vec_len
rhs = torch.rand(D * vl, dtype=torch.float64, device='cuda'); psi = torch.empty_like(rhs)
part = torch.empty(plan.G * vl, dtype=torch.float64, device='cuda'); scat = torch.rand(4 * vl, dtype=torch.float64, device='cuda')
Tr._sweep(ops, plan, rhs, psi, scat, None); torch.cuda.synchronize()
chunks = (n + 31 + C - 1) // C
ns = (ny + 31) // 32
buf = torch.zeros(ns * plan.G * chunks * 8, dtype=torch.int64, device='cuda')
_lib.call("dlrsn_debug_trace", ctypes.c_void_p(buf.data_ptr()), chunks)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); Tr._sweep(ops, plan, rhs, psi, scat, None); e1.record(); torch.cuda.synchronize()
_lib.call("dlrsn_debug_trace", None, 0)
print("launch ms", e0.elapsed_time(e1))
t = buf.cpu().numpy().reshape(ns * plan.G, chunks, 8).astype(np.float64)
t = (t - t[t > 0].min()) / 1e3
x = t[0]
cw = x[:, 1] - x[:, 0]; cc = x[:, 2] - x[:, 1]
pw = x[:, 4] - x[:, 3]; pc = x[:, 5] - x[:, 4]; pb = x[:, 6] - x[:, 5]
print(f"consumer: wait {np.median(cw):.3f} compute {np.median(cc):.3f} us/chunk (sum wait {cw.sum():.0f}, compute {cc.sum():.0f})")
print(f"producer: wait {np.median(pw):.3f} compute {np.median(pc):.3f} namedbar {np.median(pb):.3f} us/chunk (sums {pw.sum():.0f} {pc.sum():.0f} {pb.sum():.0f})")
# per-strip timeline of group 0 (items are strip-major: item = s * G + g)
G = plan.G
for s in range(ns):
    x = t[s * G]
    ok = x[:, 2] > 0
    if not ok.any():
        continue
    cw = x[ok, 1] - x[ok, 0]
    print(f"strip {s}: start {x[ok, 0].min():7.2f} end {x[ok, 2].max():7.2f} us, consumer wait sum {cw.sum():6.2f}"
          f" first-chunk wait {cw[0]:6.2f}")
for s in (0, 1, 4):
    x = t[s * G]
    cw = x[:, 1] - x[:, 0]; cc = x[:, 2] - x[:, 1]; gap = x[1:, 0] - x[:-1, 2]
    print(f"strip {s} per-chunk wait:", np.round(cw[:20], 2))
    print(f"strip {s} per-chunk comp:", np.round(cc[:20], 2))
    print(f"strip {s} gap to next   :", np.round(gap[:20], 2))
for s in (0, 4):
    x = t[s * G]
    pw = x[:, 4] - x[:, 3]; pc = x[:, 5] - x[:, 4]
    print(f"strip {s} producer wait:", np.round(pw[:16], 2))
    print(f"strip {s} producer comp:", np.round(pc[:16], 2))
    print(f"strip {s} prod ready(5) - cons wantstart(0):", np.round((x[:, 6] - x[:, 0])[:16], 2))
