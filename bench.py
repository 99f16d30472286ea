"""Benchmark of the SN-like DLR hot path on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 2 -- 280x280 checkerboard on [0,7]^2,
rank 16, 32x32 product quadrature (1024 directions), dt=0.01, fp64,
seeded random-orthonormal initial factors, use_dsa=False, si_tol=1e-8.
A step is one DLR time step: step_collocation (DEIM -> collocated source
iteration -> spatial Gram-Schmidt -> fused projections -> row solve ->
angular re-orthonormalisation) plus the fused temperature update /
re-linearisation.  The value is sweep cell-angle updates per second over
whole steps (sum over steps of n_cells x r x SI iterations / device time);
``dlr_steps_per_s`` and the config-2 full-SN comparison sweep are reported
alongside.

``--impl reference`` times the CPU restatement of the reference (oracle/,
"port") on the same config on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "SN-sweep cell-angle updates/s and DLR steps/s, % of HBM roofline, 1/2/4/8 B200"
UNIT = "cell-angle updates/s"
SWEEP_BYTES_PER_CELL_ANGLE = 64  # rhs read + psi write
SWEEP_BYTES_PER_CELL = 160  # sigma_t + scatter source per quadrant batch (4 x 40 B)


def _peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # the timed region starts only once the sampler is producing, so
            # that it is sampled DURING the region (nvidia-smi starts slowly)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_step_rate(spec, n_steps, warmup):
    """Time the oracle port (the reference algorithm restated in numpy) on
    the host: returns (cell-angle updates/s, steps/s, seconds, iterations)."""
    from oracle import runner as R

    rng = np.random.default_rng(spec.seed)
    from paper_2601_18705_b200.problems import draw_factors

    Xr, Wr = draw_factors(spec, rng)
    X, W = R.orthonormal_factors(spec, Xr, Wr)
    state = R.initial_state(spec, X, W)
    T = spec.T0.copy()
    for _ in range(warmup):
        state, T, _ = R.run(spec, state, 1, si_tol=1e-8, T=T)
    t0 = time.perf_counter()
    state, T, infos = R.run(spec, state, n_steps, si_tol=1e-8, T=T)
    dt = time.perf_counter() - t0
    iters = sum(i.iterations for i in infos)
    return spec.n_cells * spec.rank * iters / dt, n_steps / dt, dt, iters


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from paper_2601_18705_b200 import problems

    spec = problems.config2()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    warm = min(args.warmup, 1)
    # bounded sample: at most 12 oracle steps (~40 s on 16 cores), rate per step
    n_run = max(1, min(args.steps, 12))
    rate, sps, sec, iters = cpu_reference_step_rate(spec, n_run, warm)
    sec = sec * args.steps / n_run
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "C2 checkerboard 280x280, r=16, 32x32 quadrature, dlr-sn step",
                   "si_tol": 1e-8, "use_dsa": False},
        "dlr_steps_per_s": sps,
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n_run} of the {args.steps} C2 DLR steps run ({iters} sweeps of "
                                   f"16 directions) after {warm} warm-up step(s), numpy/scipy, BLAS "
                                   f"on all cores; ms_per_step is the per-step mean"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # BASELINE config 2: 50 steps
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--full-sn", type=int, default=1, help="also time the config-2 full-SN sweep")
    ap.add_argument("--more-configs", default="C4,C3,C5dlr,C5",
                    help="also time a few steps of these BASELINE configs at N=1 ('' = none)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    from paper_2601_18705_b200 import _lib, problems, transport
    from paper_2601_18705_b200._device import set_device
    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    ws, rank, local = _dist()
    set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = problems.config2()
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)

    from paper_2601_18705_b200.sharding import DirectionComm

    comm = DirectionComm.from_default_group()  # None at N=1; NCCL direction sharding at N>1

    Tbox = [T]

    def one_step(state, lin):
        # step_collocation + the step boundary (T update, re-linearisation)
        # in one native call (DeviceProblem.step)
        state, lin, Tbox[0], info = dp.step(state, lin, Tbox[0], si_tol=1e-8, check_state=True,
                                            comm=comm)
        return state, lin, info

    # setup (untimed, before the W warm-up steps): the step's CUDA graphs are
    # captured per buffer set on first sighting and the sticky iteration
    # batch settles within the first few steps of a chain
    for _ in range(10):
        state, lin, _ = one_step(state, lin)
    for _ in range(args.warmup):
        state, lin, _ = one_step(state, lin)
    torch.cuda.synchronize()

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    iters = []
    launches0 = _lib.launch_count()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))  # evict L2 between timed steps (outside the events)
            starts[k].record()
            state, lin, info = one_step(state, lin)
            ends[k].record()
            iters.append(info.iterations)
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = _lib.launch_count() - launches0
    if ws > 1:
        torch.distributed.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # roofline pass (after the timed region): CUDA events around every sweep
    # launch of a few more steps (sweep timing turns the step's graph replay
    # off, so it is kept out of the timed steps; kernel times are the same)
    _lib.call("dlrsn_sweep_timing", 1)
    r_iters = []
    for _ in range(3):
        state, lin, info = one_step(state, lin)
        r_iters.append(info.iterations)
    torch.cuda.synchronize()
    sweep_ms, sweep_groups = _sweep_timings(_lib)
    n_cells, D = spec.n_cells, int(sweep_groups[0])  # single-direction groups: D = G
    updates = sum(spec.n_cells * spec.rank * it for it in iters)
    value = updates / (ms * 1e-3)
    peak, peak_kind = _peaks()
    alg_bytes = n_cells * (D * SWEEP_BYTES_PER_CELL_ANGLE + SWEEP_BYTES_PER_CELL)
    # launches past convergence (speculative, return at once) are counted in
    # the time but not as sweeps: time per real sweep = all sweep time / iterations
    sweep_avg_ms = float(np.sum(sweep_ms)) / max(1, sum(r_iters))
    achieved = alg_bytes / (sweep_avg_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(HERE, "profiles", "sweep_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("C2_dlr_sweep_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end-to-end: public API with HOST (pinned) buffers each step -------
    # (untimed warm-up long enough for every step graph of the rotation to be
    # captured: 2 input sets x 3 output blocks cycling through the caching
    # allocator = 6 buffer keys, each captured on its second sighting)
    e2e = measure_e2e(dp, state, Tbox[0], lin, max(1, min(args.steps, 20)), comm,
                      warmup=max(args.warmup, 14))

    # ---- full-SN comparison sweep (config 2: all 1024 directions) ----------
    full = measure_full_sn(dp, comm) if args.full_sn else None

    # ---- larger BASELINE configs at N=1 (not the headline: step time and
    # the DLR sweep's HBM fraction where the sweep is bandwidth-bound) -------
    more = []
    if ws == 1 and args.more_configs:
        del state, lin, Tbox, dp
        torch.cuda.empty_cache()
        for name in args.more_configs.split(","):
            more.append(measure_config(name.strip()))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config 2 checkerboard, random-orthonormal factors)",
        "config": {"workload": "C2 checkerboard 280x280, r=16, 32x32 quadrature, dlr-sn step",
                   "si_tol": 1e-8, "use_dsa": False, "parallelism": f"dp{ws} (directions)",
                   "l2": "512 MB buffer written between timed steps (outside the step events)"},
        "dlr_steps_per_s": args.steps / (ms * 1e-3),
        "si_iterations_per_step": float(np.mean(iters)),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "sweep_ws_kernel", "launch_ms": sweep_avg_ms,
                     "sweep_launches": len(sweep_ms), "sweeps_converging": int(sum(r_iters)),
                     "alg_bytes_per_launch": alg_bytes,
                     "sweep_share_of_step": (sum(sweep_ms) / len(r_iters)) / (ms / args.steps)},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "wall_s_timed_region": wall,
    }
    if full is not None:
        line["full_sn_sweep"] = full
    if more:
        line["more_configs"] = more
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        rate, sps, sec, it = cpu_reference_step_rate(spec, args.cpu_steps, 0)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{args.cpu_steps} full C2 DLR steps of the oracle port "
                                          f"({it} sweeps of 16 directions, {sec:.1f} s)",
                                "dlr_steps_per_s": sps}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def measure_e2e(dp, state, T, lin, n, comm=None, warmup=3):
    """Same step through the public API with the state and per-cell fields
    in pinned HOST memory: every step copies X, S, W, T and the step
    coefficients host->device, runs step_collocation + the T update, and
    copies the new X, S, W and T device->host.  Steps are independent
    problems streamed through the API, so the copies are pipelined: the H2D
    of step k+1 (copy stream) and the D2H of step k-1 (second copy stream)
    overlap step k's compute; everything is inside the timed region."""
    import torch

    from paper_2601_18705_b200.dlr_sn import step_collocation
    from paper_2601_18705_b200.lowrank import DlrState
    from paper_2601_18705_b200.angular import AngularBasis
    from paper_2601_18705_b200.physics import LinearizedStep

    def pin(t):
        return t.detach().cpu().pin_memory()

    host = {"X": pin(state.X), "S": pin(state.S), "W": pin(state.W.values), "T": pin(T)}
    fields = ("sigma_t", "sigma_s", "sigma_a", "q", "T0", "denom", "rho_cv")
    host.update({f: pin(getattr(lin, f)) for f in fields})
    outs = [{k: torch.empty_like(host[k]).pin_memory() for k in ("X", "S", "W", "T")}
            for _ in range(2)]
    h2d = sum(v.numel() * 8 for v in host.values())
    d2h = sum(v.numel() * 8 for v in outs[0].values())
    dev = [{k: torch.empty_like(v, device="cuda") for k, v in host.items()} for _ in range(2)]
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    loaded = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    for e in freed + copied:
        e.record(comp)
    keep = [None, None]

    def upload(k):
        b = k % 2
        with torch.cuda.stream(up):
            up.wait_event(freed[b])
            for name, v in host.items():
                dev[b][name].copy_(v, non_blocking=True)
            loaded[b].record(up)

    def compute(k):
        b = k % 2
        d = dev[b]
        comp.wait_event(loaded[b])
        st = DlrState(X=d["X"], S=d["S"], W=AngularBasis(values=d["W"]).bind(dp.quad))
        step = LinearizedStep(dt=lin.dt, inv_cdt=lin.inv_cdt, constants=lin.constants,
                              **{f: d[f] for f in fields})
        new, info = step_collocation(dp.grid, step, dp.quad, st, si_tol=1e-8, use_dsa=False,
                                     comm=comm)
        # T update in place on this step's input slot (re-filled by the upload of step k+2)
        Tn = dp.advance(step, info.phi, d["T0"])
        freed[b].record(comp)  # the input set may be overwritten from here on
        res = {"X": new.X, "S": new.S, "W": new.W.values, "T": Tn.T0}
        done[b].record(comp)
        comp.wait_event(copied[b])  # outputs of step k-2 read back before reuse
        keep[b] = res
        with torch.cuda.stream(down):
            down.wait_event(done[b])
            for name, v in res.items():
                outs[b][name].copy_(v, non_blocking=True)
            copied[b].record(down)
        for v in res.values():
            v.record_stream(down)
        return info.iterations

    def run(count):
        it = 0
        up.wait_stream(comp)  # the first upload starts inside the timed region
        upload(0)
        for k in range(count):
            if k + 1 < count:
                upload(k + 1)
            it += compute(k)
        comp.wait_stream(down)
        return it

    run(warmup)  # untimed: first-sighting setup of both buffer sets
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    iters = run(n)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if comm is not None:
        ms = comm.max_scalar(ms)
    spec = dp.spec
    return {"value": spec.n_cells * spec.rank * iters / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": n, "warmup": warmup, "ms_per_step": ms / n,
            "pipelined": "H2D of step k+1 and D2H of step k-1 overlap step k (2 copy streams)"}


def measure_config(name, steps=6, warmup=6):
    """A few DLR steps of a larger BASELINE config (C3 Marshak 512^2 r=32
    from its initial state, C4 random medium 1024^2 r=64): device time per
    step (inputs resident, L2 flushed between steps) and the DLR sweep's
    algorithmic HBM fraction from per-launch CUDA events."""
    import torch

    from paper_2601_18705_b200 import _lib, problems
    from paper_2601_18705_b200.driver import DeviceProblem, initial_state

    if name == "C5":
        return measure_c5_sweep()
    if name == "C5dlr":
        return measure_c5_dlr_sweep()
    if name == "C3":
        spec = problems.marshak()
        label = "C3 Marshak 512x512, r=32, 64x64 quadrature, inflow T_b=1, dlr-sn step"
    elif name == "C4":
        spec, fields = problems.random_medium()
        rng = np.random.default_rng(spec.seed)
        problems.draw_factors(spec, rng)  # X, W first (SURVEY 8d draw order)
        fields(rng)
        label = "C4 random medium 1024x1024, r=64, 64x64 quadrature, dlr-sn step"
    else:
        raise SystemExit(f"unknown config {name}")
    dp = DeviceProblem.from_spec(spec)
    state = initial_state(dp)
    T = torch.as_tensor(spec.T0, device="cuda").clone()
    lin = dp.linearized(T)
    for _ in range(warmup):
        state, lin, T, _ = dp.step(state, lin, T, si_tol=1e-8)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ms, iters, per = 0.0, [], []
    for k in range(steps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
        e1.record()
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
        ms += per[-1]
        iters.append(info.iterations)
    _lib.call("dlrsn_sweep_timing", 1)
    state, lin, T, info = dp.step(state, lin, T, si_tol=1e-8)
    torch.cuda.synchronize()
    sw, _ = _sweep_timings(_lib)
    sweep_ms = float(np.sum(sw)) / max(1, info.iterations)
    alg = spec.n_cells * (spec.rank * SWEEP_BYTES_PER_CELL_ANGLE + SWEEP_BYTES_PER_CELL)
    peak, _ = _peaks()
    out = {"workload": label, "steps": steps, "ms_per_step": ms / steps,
           "ms_per_step_each": [round(x, 3) for x in per],
           "dlr_steps_per_s": steps / (ms * 1e-3), "si_iterations": iters,
           "cell_angle_per_s": spec.n_cells * spec.rank * sum(iters) / (ms * 1e-3),
           "sweep": {"kernel": "sweep_kernel<1>", "launch_ms": sweep_ms,
                     "alg_bytes_per_launch": alg, "achieved_GBs": alg / (sweep_ms * 1e-3) / 1e9,
                     "frac_of_hbm": alg / (sweep_ms * 1e-3) / 1e9 / peak}}
    del state, lin, T, dp, flush
    torch.cuda.empty_cache()
    return out


def measure_c5_dlr_sweep(reps=3):
    """Config 5's DLR sweep on one GPU: the r = 128 directions DEIM selects
    from a seeded random orthonormal W (16384 x 128, lowrank.py:168-205),
    swept over the 4096^2 tile medium with psi STORED for every direction
    (rhs and psi are 69 GB each in the SK layout, both in HBM), i.e. the
    per-iteration sweep of the C5 DLR step (sigma_s = 0: one sweep per step,
    no scattering source).  The rhs of every direction is the step's
    source_vector(q) + inv_cdt M psi_old for the isotropic psi_old = B(T0)
    (forming X S W_sel^T needs the 68.7 GB X, which with rhs and psi does
    not fit one GPU; the sweep's traffic and arithmetic do not depend on
    the rhs values).  Algorithmic bytes: 64 per cell-angle + 32 per cell
    (sigma_t in 4 quadrant orientations)."""
    import torch

    from paper_2601_18705_b200 import _lib, problems, transport
    from paper_2601_18705_b200.driver import DeviceProblem
    from paper_2601_18705_b200.lowrank import deim_select

    spec, fields = problems.stress()
    rng = np.random.default_rng(spec.seed)
    fields(rng)
    dp = DeviceProblem.from_spec(spec)
    T = torch.as_tensor(spec.T0, device="cuda")
    lin = dp.linearized(T)
    ops = transport.assemble_operators(dp.grid, lin)
    quad = dp.quad
    W0 = torch.randn(quad.n_angles, spec.rank, dtype=torch.float64, device="cuda",
                     generator=torch.Generator(device="cuda").manual_seed(spec.seed))
    W = torch.linalg.qr(W0 * torch.sqrt(quad.weights_device())[:, None])[0] / \
        torch.sqrt(quad.weights_device())[:, None]
    sel = deim_select(W)
    idx = sel.indices
    om = quad.omegas[idx]
    cw = np.ones(len(idx))
    plan = transport._SweepPlan(ops, om, cw)
    b0 = (spec.a_r * spec.c / (4 * np.pi)) * (T * T) ** 2
    rhs = ops.source_vector(lin.q) + lin.inv_cdt * ops.mass_apply(b0.repeat_interleave(4))
    vl = ops.vec_len
    rhs4 = torch.empty(4 * vl, dtype=torch.float64, device="cuda")
    cols = rhs.reshape(-1, 1).expand(-1, 4).contiguous()
    quads4 = torch.arange(4, dtype=torch.int32, device="cuda")
    zero_q = torch.zeros(spec.n_cells, dtype=torch.float64, device="cuda")
    _lib.call("dlrsn_rhs_build", ops.cellops_ptr, 4, _lib.ptr(quads4), _lib.ptr(zero_q), 0.0,
              None, 1, _lib.ptr(cols), 4, _lib.ptr(rhs4), transport.stream())
    del cols, W0, W
    D = len(idx)
    quads = plan.quads_dev.cpu().numpy()
    rhs_sk = torch.empty(D * vl, dtype=torch.float64, device="cuda")
    for d in range(D):
        rhs_sk[d * vl:(d + 1) * vl].copy_(rhs4[int(quads[d]) * vl:(int(quads[d]) + 1) * vl])
    del rhs4
    psi_sk = torch.empty_like(rhs_sk)
    transport._sweep(ops, plan, rhs_sk, psi_sk)  # warm-up
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for e0, e1 in evs:  # 138 GB touched per sweep: inputs far larger than L2
        e0.record()
        transport._sweep(ops, plan, rhs_sk, psi_sk)
        e1.record()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    n_sel_quads = np.bincount(quads, minlength=4).tolist()
    chk = float(psi_sk[:vl].sum())
    alg = spec.n_cells * (D * SWEEP_BYTES_PER_CELL_ANGLE + 32)
    peak, _ = _peaks()
    out = {"workload": "C5 stress 4096x4096, r=128 DEIM-selected of 128x128 directions, "
                       "DLR sweep with psi stored (sigma_s = 0: one sweep per step)",
           "kernel": f"sweep_kernel<{plan.dw}>", "groups": plan.G, "directions_per_quadrant":
           n_sel_quads, "ms_per_sweep": ms, "cell_angle_per_s": spec.n_cells * D / (ms * 1e-3),
           "alg_bytes_per_launch": alg, "achieved_GBs": alg / (ms * 1e-3) / 1e9,
           "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / peak, "psi_checksum": chk,
           "note": "rhs = source + inv_cdt M B(T0) per direction (X S W_sel^T needs the "
                   "68.7 GB X); l2: inputs 138 GB >> L2"}
    del rhs_sk, psi_sk, ops, lin, T, rhs, dp, plan
    torch.cuda.empty_cache()
    return out


def measure_c5_sweep(reps=1):
    """Config 5's full-SN stress sweep on one GPU: 16384 directions on the
    4096^2 tile medium (sigma_a log-uniform [0.1, 100] per 64x64 tile, q ~
    U[0,1], dt = dx = 1, pure absorber => one sweep per step), closure only:
    psi (8.8 TB) is never stored, so there are no per-cell-angle HBM bytes
    and the sweep is FP64-issue bound (report cell-angle/s).  The fields
    are drawn from seed 5 directly (the 68.7 GB X draw of the DLR factors
    is skipped: config 5's DLR step needs the space-sharded layout)."""
    import torch

    from paper_2601_18705_b200 import problems, transport
    from paper_2601_18705_b200.driver import DeviceProblem

    spec, fields = problems.stress()
    fields(np.random.default_rng(spec.seed))
    dp = DeviceProblem.from_spec(spec)
    T = torch.as_tensor(spec.T0, device="cuda")
    lin = dp.linearized(T)
    ops = transport.assemble_operators(dp.grid, lin)
    b0 = (spec.a_r * spec.c / (4 * np.pi)) * (T * T) ** 2  # isotropic psi_old = B(T0)
    rhs = ops.source_vector(lin.q) + lin.inv_cdt * ops.mass_apply(b0.repeat_interleave(4))
    quad = dp.quad
    phi = transport.closure_sweep(ops, quad.omegas, quad.weights, rhs)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        phi = transport.closure_sweep(ops, quad.omegas, quad.weights, rhs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ca = spec.n_cells * quad.n_angles
    out = {"workload": "C5 stress 4096x4096, 128x128 = 16384 directions, full-SN closure-only sweep",
           "ms_per_sweep": ms, "cell_angle_per_s": ca / (ms * 1e-3), "cell_angles": ca,
           "bound": "fp64 issue (no per-cell-angle HBM traffic: psi not stored)",
           "phi_checksum": float(phi.sum())}
    del ops, lin, T, rhs, phi, dp
    torch.cuda.empty_cache()
    return out


def _sweep_timings(_lib):
    """Per-launch sweep times recorded by the library (dlrsn_sweep_timing)."""
    import ctypes

    cap = 4096
    ms = (ctypes.c_float * cap)()
    groups = (ctypes.c_int * cap)()
    dw = (ctypes.c_int * cap)()
    cnt = ctypes.c_int()
    _lib.call("dlrsn_sweep_timing_read", cap, ms, groups, dw, ctypes.byref(cnt))
    _lib.call("dlrsn_sweep_timing", 0)
    n = min(cnt.value, cap)
    if n == 0 or any(dw[k] != 1 for k in range(n)):
        raise RuntimeError("sweep timing: expected single-direction groups")
    return [ms[k] for k in range(n)], [groups[k] for k in range(n)]


def measure_full_sn(dp, comm=None, reps=3):
    """Config 2's full-SN comparison sweep: one source-iteration sweep over
    all 1024 quadrature directions (closure = quadrature weights) on the
    280x280 grid, psi stored (64 B/cell-angle algorithmic)."""
    import torch

    from paper_2601_18705_b200 import transport

    T = torch.as_tensor(dp.spec.T0, device="cuda")
    lin = dp.linearized(T)
    ops = transport.assemble_operators(dp.grid, lin)
    quad = dp.quad
    D = quad.n_angles
    mine = np.arange(D)
    if comm is not None:
        from paper_2601_18705_b200.sharding import partition_directions

        mine = partition_directions(quad.omegas, comm.world_size)[comm.rank]
    plan = transport._SweepPlan(ops, quad.omegas[mine], quad.weights[mine])
    vl = ops.vec_len
    Dl = len(mine)
    rhs = torch.rand(Dl * vl, dtype=torch.float64, device="cuda")
    psi = torch.empty_like(rhs)
    part = torch.empty(plan.G * vl, dtype=torch.float64, device="cuda")
    scat = torch.zeros(4 * vl, dtype=torch.float64, device="cuda")
    for _ in range(2):
        transport._sweep(ops, plan, rhs, psi, scat, part)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        transport._sweep(ops, plan, rhs, psi, scat, part)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if comm is not None:
        ms = comm.max_scalar(ms)
    nc = dp.grid.n_cells
    alg = nc * (D * SWEEP_BYTES_PER_CELL_ANGLE + SWEEP_BYTES_PER_CELL)
    peak, _ = _peaks()
    return {"directions": D, "ms_per_sweep": ms, "cell_angle_per_s": nc * D / (ms * 1e-3),
            "achieved_GBs": alg / (ms * 1e-3) / 1e9, "frac_of_hbm": alg / (ms * 1e-3) / 1e9 / peak,
            "group_width": plan.dw, "groups": plan.G}


if __name__ == "__main__":
    main()
