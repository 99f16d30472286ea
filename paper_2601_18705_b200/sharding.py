"""Direction sharding across the GPUs of one node.

Given a frozen scattering source the per-direction sweeps of one source
iteration are independent (transport_sn.py:419-427), so the r
swept directions are split across ranks.  Per source iteration each rank
sweeps its directions and forms its partial closure flux
phi_p = sum_{d in p} c_d psi_d; one allreduce(sum) over NVLink gives every
rank the same phi, from which the convergence norm and the next scattering
source are computed redundantly (identical on all ranks).  After the
iteration the swept columns are all-gathered in selection order and the
Galerkin side of the step (Gram-Schmidt, projections, row solve, angular
update) runs replicated, so every rank holds the same state ("Option A";
the all-to-all re-layout of "Option B" is the next step for the largest
configs).

Everything here is device-agnostic torch code so that the protocol is tested
on CPU with the gloo backend (tests/test_sharding.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


def quadrant_code(omega):
    return (0 if omega[0] >= 0.0 else 1) | (0 if omega[1] >= 0.0 else 2)


def partition_directions(omegas, world_size):
    """Deterministic, quadrant-balanced partition of direction slots.

    Directions are dealt round-robin within each quadrant (so every rank
    gets the same wavefront work per quadrant up to one direction), with the
    deal order rotating between quadrants so that totals stay balanced.
    Returns a list of sorted slot arrays, one per rank.
    """
    om = np.asarray(omegas, dtype=float)
    quads = np.array([quadrant_code(o) for o in om], dtype=int)
    owners = [[] for _ in range(world_size)]
    nxt = 0
    for q in range(4):
        for slot in np.flatnonzero(quads == q):
            owners[nxt % world_size].append(int(slot))
            nxt += 1
    return [np.asarray(sorted(o), dtype=np.int64) for o in owners]


@dataclass
class DirectionComm:
    """Collectives of the sharded step on a torch.distributed process group
    (NCCL on the GPUs, gloo in the CPU tests)."""

    group: object = None
    rank: int = 0
    world_size: int = 1

    @classmethod
    def from_default_group(cls):
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            return None
        ws = dist.get_world_size()
        if ws == 1:
            return None
        return cls(group=None, rank=dist.get_rank(), world_size=ws)

    def allreduce_sum_(self, t):
        """In-place sum over ranks (the partial closure flux, N_x doubles)."""
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allgather_columns(self, local, owners, n_total):
        """Assemble (n, n_total) from each rank's (n, |owners[p]|) columns,
        placing rank p's columns at slots owners[p] (selection order)."""
        import torch.distributed as dist

        n = local.shape[0]
        width = max(len(o) for o in owners)
        send = torch.zeros(width, n, dtype=local.dtype, device=local.device)
        if local.shape[1]:
            send[:local.shape[1]] = local.T
        recv = [torch.empty_like(send) for _ in range(self.world_size)]
        dist.all_gather(recv, send.contiguous(), group=self.group)
        full = torch.empty(n, n_total, dtype=local.dtype, device=local.device)
        for p, slots in enumerate(owners):
            if len(slots):
                idx = torch.as_tensor(slots, device=local.device)
                full[:, idx] = recv[p][:len(slots)].T
        return full

    def allgather_into_(self, recv, send):
        """recv[p] = send of rank p (recv: (world_size, *send.shape)); the
        native step's gather of the swept columns (include/dlrsn.h dlrsn_comm)."""
        import torch.distributed as dist

        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(recv.reshape(-1), send.contiguous().reshape(-1),
                                        group=self.group)
        else:
            dist.all_gather(list(recv.unbind(0)), send.contiguous(), group=self.group)
        return recv

    def max_scalar(self, x):
        import torch.distributed as dist

        t = torch.tensor([float(x)], dtype=torch.float64)
        if dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())
