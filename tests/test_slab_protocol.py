"""The exchanges of the row-slab step (slab.py, "Option B" of SURVEY 8e) on
CPU: two gloo ranks (torch.distributed, the same driver NCCL uses on GPUs)
and the in-process virtual-rank driver, against direct indexing of the full
matrices.  Device-agnostic torch code: no CUDA needed."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _case(P, me, nx=6, ny=7, r=9, seed=3):
    from paper_2601_18705_b200.mesh import build_grid
    from paper_2601_18705_b200.sharding import partition_directions
    from paper_2601_18705_b200.slab import Slab, slab_rows

    grid = build_grid(nx, ny)
    slab = Slab(me, P, grid, slab_rows(ny, P))
    rng = np.random.default_rng(seed)
    Y = torch.as_tensor(rng.standard_normal((grid.n_dofs, r)))
    om = rng.standard_normal((r, 3))
    owners = partition_directions(om, P)
    return grid, slab, Y, owners


def _protocol(P, me):
    """One rank's generator: the three exchanges; returns what it checked."""
    from paper_2601_18705_b200.slab import direction_columns_to_rows, halo_below, rows_to_direction_columns

    grid, slab, Y, owners = _case(P, me)
    mine = owners[me]
    cols = yield from rows_to_direction_columns(Y[slab.d0:slab.d1].contiguous(), owners, slab)
    assert torch.equal(cols, Y[:, torch.as_tensor(mine)])
    rows = yield from direction_columns_to_rows(Y[:, torch.as_tensor(mine)].contiguous(), owners,
                                                slab, Y.shape[1])
    assert torch.equal(rows, Y[slab.d0:slab.d1])
    halo = yield from halo_below(Y[slab.d0:slab.d1].contiguous(), slab)
    if me == 0:
        assert halo is None
    else:
        nxr = 4 * grid.nx
        assert torch.equal(halo, Y[slab.d0 - nxr:slab.d0])
    return len(mine)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_slab_exchanges_virtual_ranks(P):
    from paper_2601_18705_b200.slab import run_local

    counts = run_local(P, lambda p: _protocol(P, p))
    assert sum(counts) == 9


def _worker(rank, world, port, errs):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_18705_b200.slab import run_dist

        run_dist(_protocol(world, rank))
    except Exception as e:  # surfaced to the parent
        errs.put(repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchanges_gloo(world):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    errs = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(k, world, port, errs)) for k in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert errs.empty(), errs.get()


def test_slab_rows_cover_the_grid():
    from paper_2601_18705_b200.slab import slab_rows

    for ny, P in [(7, 3), (4096, 8), (5, 5), (9, 2)]:
        rows = slab_rows(ny, P)
        assert rows[0][0] == 0 and rows[-1][1] == ny
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        sizes = [b - a for a, b in rows]
        assert max(sizes) - min(sizes) <= 1
