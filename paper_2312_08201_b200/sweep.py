"""Multi-GPU sweep over a parameter grid: shard, solve, all-gather, argmin.

Every v is independent (north star (c)): the seed state is replicated, each rank solves its shard,
and the only collective is an all-gather of the traces (nv x 8 bytes), followed by an argmin with
the smallest-flat-index tie-break (reading R16).

Sharding (strong scaling, one grid split over the ranks):
  * with a per-row cost (the engine's proxy sum_t |v_t| ||B~l_t|| ||B^r_t||, Problem.cost_proxy):
    rows sorted by cost, largest first, dealt to ranks in a snake (0..N-1, N-1..0, ...), so every
    rank gets the same number of rows (+-1) and the same cost (within the largest single row);
  * without: chunks of `chunk` consecutive rows dealt round-robin.
The solver is a callable, so the same code runs the CUDA engine over NCCL in bench.py and a fake
analytic solver over gloo in the CPU tests.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

CHUNK = 64


def shard_indices(nv: int, rank: int, world: int, chunk: int = CHUNK, cost=None) -> np.ndarray:
    """Rows of V owned by `rank` (sorted ascending)."""
    if cost is not None:
        cost = np.asarray(cost, dtype=np.float64).reshape(-1)
        assert cost.shape[0] == nv
        order = np.argsort(-cost, kind="stable")  # largest first; ties in row order
        pos = np.arange(nv)
        rnd, off = pos // world, pos % world
        owner = np.where(rnd % 2 == 0, off, world - 1 - off)  # snake
        return np.sort(order[owner == rank]).astype(np.int64)
    starts = range(rank * chunk, nv, world * chunk)
    parts = [np.arange(s, min(nv, s + chunk)) for s in starts]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)


def shard_balance(nv: int, world: int, cost, chunk: int = CHUNK, balanced: bool = True) -> float:
    """max over ranks / mean of the summed cost of each shard (1.0 = perfect)."""
    cost = np.asarray(cost, dtype=np.float64).reshape(-1)
    tot = [cost[shard_indices(nv, r, world, chunk, cost if balanced else None)].sum() for r in range(world)]
    return float(max(tot) / (sum(tot) / world))


class Sweep:
    """Pre-computed gather layout for one (nv, world) so the timed step allocates nothing on the host.

    solve(shard_rows) -> traces for those rows (a torch tensor on `device`)."""

    def __init__(self, nv: int, rank: int, world: int, device, group=None, chunk: int = CHUNK,
                 scaling: str = "strong", cost=None):
        """strong: one grid of nv rows sharded over the ranks (cost-balanced when `cost` is given);
        weak: every rank owns nv rows of its own (rows [rank*nv, (rank+1)*nv) of the global
        world*nv batch)."""
        import torch
        self.rank, self.world, self.device, self.group = rank, world, device, group
        if scaling == "weak":
            shards = [np.arange(r * nv, (r + 1) * nv) for r in range(world)]
            nv = nv * world
        else:
            shards = [shard_indices(nv, r, world, chunk, cost) for r in range(world)]
        self.nv = nv
        self.mine = shards[rank]
        self.nmax = max((len(s) for s in shards), default=0)
        pad = [np.pad(s, (0, self.nmax - len(s)), constant_values=-1) for s in shards]
        idx = torch.tensor(np.concatenate(pad) if pad else np.zeros(0, np.int64), device=device)
        self.valid = idx >= 0
        self.dest = idx[self.valid]
        self.gathered = torch.empty(world * self.nmax, dtype=torch.float64, device=device)
        self.buf = torch.empty(self.nmax, dtype=torch.float64, device=device)
        self.full = torch.empty(self.nv, dtype=torch.float64, device=device)

    def run(self, solve: Callable):
        """One sweep step: local solve, all-gather (world > 1), argmin. Returns (traces[nv], argmin)."""
        import torch
        import torch.distributed as dist
        tau = solve(self.mine)
        if self.world == 1:
            full = tau
        else:
            self.buf.fill_(float("inf"))
            self.buf[: tau.numel()] = tau
            dist.all_gather_into_tensor(self.gathered, self.buf, group=self.group)
            full = self.full
            full[self.dest] = self.gathered[self.valid]
        return full, torch.argmin(full)  # torch.argmin returns the first index among ties
