"""Host-side timeline of C2 DLR steps: cProfile of the Python orchestration
plus per-phase CUDA-event timing (dev probe)."""
import cProfile, os, pstats, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_18705_b200 import problems
from paper_2601_18705_b200.dlr_sn import step_collocation
from paper_2601_18705_b200.driver import DeviceProblem, initial_state

spec = problems.config2()
dp = DeviceProblem.from_spec(spec)
state = initial_state(dp)
T = torch.as_tensor(spec.T0, device="cuda").clone()
lin = dp.linearized(T)
def one(state, lin):
    state, info = step_collocation(dp.grid, lin, dp.quad, state, si_tol=1e-8, use_dsa=False)
    lin = dp.advance(lin, info.phi, T)
    return state, lin
for _ in range(3):
    state, lin = one(state, lin)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    state, lin = one(state, lin)
torch.cuda.synchronize()
pr.disable()
print("wall per step ms", (time.perf_counter() - t0) / 5 * 1e3)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
