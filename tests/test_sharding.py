"""Direction sharding (multi-GPU path) on CPU: partition logic and the
per-iteration allreduce / final allgather protocol, world_size 2 with gloo.

The sharded source iteration below uses exactly the helpers the GPU path
uses (paper_2601_18705_b200.sharding) with the oracle's sweeps standing in
for the CUDA kernels, and must reproduce the unsharded iteration.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_18705_b200.sharding import DirectionComm, partition_directions


def test_partition_is_balanced_and_complete():
    rng = np.random.default_rng(0)
    om = rng.standard_normal((37, 3))
    for ws in (1, 2, 3, 4, 8):
        parts = partition_directions(om, ws)
        allslots = np.sort(np.concatenate(parts))
        assert np.array_equal(allslots, np.arange(37))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
        # per quadrant balance within one direction
        q = (om[:, 0] < 0).astype(int) | 2 * (om[:, 1] < 0).astype(int)
        for qq in range(4):
            per = [int(np.sum(q[p] == qq)) for p in parts]
            assert max(per) - min(per) <= 1
        assert all(np.all(np.diff(p) > 0) for p in parts)
        assert [list(p) for p in partition_directions(om, ws)] == [list(p) for p in parts]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from oracle import port as P

    rng = np.random.default_rng(12)
    nx, ny = 9, 7
    n = nx * ny
    sig = rng.uniform(1.0, 20.0, n)
    ss = sig * rng.uniform(0.2, 0.8, n)
    q = rng.uniform(0, 1, n)
    grid = P.Grid(nx, ny, 0.0, 0.0, 1.0, 0.8)
    st = P.Step(sig, ss, sig - 0.3, q, np.zeros(n), np.ones(n), np.ones(n), 1.0, 0.3)
    ops = P.assemble_operators(grid, st)
    quad = P.build_quadrature(2, 6)
    om = quad.omegas[[0, 2, 3, 5, 6, 8, 9, 11]]
    clo = rng.uniform(0.5, 2.0, om.shape[0])
    pt = rng.standard_normal((grid.n_dofs, om.shape[0]))
    ps = rng.standard_normal(grid.n_dofs)
    return P, ops, om, clo, pt, ps


def _sharded_si(rank, ws, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        P, ops, om, clo, pt, ps = _problem()
        comm = DirectionComm(rank=rank, world_size=ws)
        nd = om.shape[0]
        owners = partition_directions(om, ws)
        mine = owners[rank]
        st = ops.step
        base = np.tile(ops.source_vector(st.q), (nd, 1)).T + st.inv_cdt * ops.mass_apply(pt)
        ss_dof = np.repeat(st.sigma_s, 4)
        phi = ps.copy()
        for it in range(1, 200):
            scatter = ops.mass_apply(ss_dof * phi) / (4 * np.pi)
            psi_loc = P.sweep_many(ops, om[mine], base[:, mine] + scatter[:, None])
            phi_part = torch.from_numpy(psi_loc @ clo[mine])
            phi_new = comm.allreduce_sum_(phi_part).numpy()
            change = np.linalg.norm(phi_new - phi) / max(np.linalg.norm(phi_new), 1e-300)
            phi = phi_new
            if change <= 1e-12:
                break
        psi = comm.allgather_columns(torch.from_numpy(psi_loc), owners, nd).numpy()
        if rank == 0:
            np.savez(out, psi=psi, phi=phi, it=it)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2])
def test_sharded_source_iteration_matches_unsharded(tmp_path, ws):
    out = str(tmp_path / "sharded.npz")
    mp.spawn(_sharded_si, args=(ws, _free_port(), out), nprocs=ws, join=True)
    got = np.load(out)
    P, ops, om, clo, pt, ps = _problem()
    ref = P.source_iteration(ops, om, clo, psi_time=pt, use_dsa=False, tol=1e-12, phi_start=ps)
    assert int(got["it"]) == ref.iterations
    assert np.linalg.norm(got["psi"] - ref.psi) <= 1e-13 * np.linalg.norm(ref.psi)
    assert np.linalg.norm(got["phi"] - ref.phi) <= 1e-13 * np.linalg.norm(ref.phi)


def _gather_check(rank, ws, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        comm = DirectionComm(rank=rank, world_size=ws)
        owners = [np.array([0, 3, 4]), np.array([1, 2])] if ws == 2 else None
        full_ref = torch.arange(6 * 5, dtype=torch.float64).reshape(6, 5)
        local = full_ref[:, torch.as_tensor(owners[rank])]
        full = comm.allgather_columns(local, owners, 5)
        t = torch.tensor([float(rank + 1)])
        mx = comm.max_scalar(rank + 1.0)
        if rank == 0:
            np.savez(out, ok=bool(torch.equal(full, full_ref)), mx=mx)
    finally:
        dist.destroy_process_group()


def test_allgather_columns_places_uneven_shards():
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "g.npz")
        mp.spawn(_gather_check, args=(2, _free_port(), out), nprocs=2, join=True)
        r = np.load(out)
        assert bool(r["ok"]) and float(r["mx"]) == 2.0


def test_mirror_pairs_halve_product_quadratures():
    """z-mirror dedup (transport.mirror_pairs): a Gauss-Legendre x uniform
    azimuth product set has exactly two nodes per (omega_x, omega_y), the
    pair index maps every node onto a pair with bitwise-equal components,
    and the summed closure weights keep the total (4 pi)."""
    import numpy as np

    from paper_2601_18705_b200.angular import build_quadrature
    from paper_2601_18705_b200.transport import dedup_mirrors, mirror_pairs

    for n in (4, 16, 32, 128):
        q = build_quadrature(n, n)
        first, inv = mirror_pairs(q.omegas)
        assert first.size * 2 == q.n_angles
        assert np.array_equal(q.omegas[first[inv], :2], q.omegas[:, :2])
        assert np.all(np.diff(first) > 0)
        om, w, inv2 = dedup_mirrors(q.omegas, q.weights)
        assert np.array_equal(inv, inv2) and abs(w.sum() - 4 * np.pi) <= 1e-12
