"""Multi-GPU SpMV: one process per GPU, row shards = whole plan partitions.

SURVEY.md §8e: the SpMV plan's partitions are contiguous nnz-balanced row
ranges (scheduler.cpp:67-89) and windows never cross them (miner.cpp:298-300),
so rank r executes partitions [r*P/N, (r+1)*P/N) -- an exact slice of the one
bit-exact plan -- and owns the x entries of its rows. A step gathers the full
x (NCCL all-gather over NVLink; gloo on CPU for tests) and multiplies. Results
are bitwise those of the single-GPU executor because every row is computed by
the same code on the same operands. The solve does not shard (replicas only).
"""
from __future__ import annotations

from typing import List, Tuple

from .psc import CodeletPlan, partition_rows


def shard_partitions(n_partitions: int, world: int, rank: int) -> Tuple[int, int]:
    """Partitions [p0, p1) owned by `rank` (contiguous, as even as possible)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_partitions: bad rank/world")
    return rank * n_partitions // world, (rank + 1) * n_partitions // world


def shard_row_ranges(plan: CodeletPlan, world: int) -> List[Tuple[int, int]]:
    """Row range of every rank's shard."""
    n_parts = plan.counts().n_partitions
    out = []
    for r in range(world):
        p0, p1 = shard_partitions(n_parts, world, r)
        out.append(partition_rows(plan, p0, p1) if p1 > p0 else (0, 0))
    return out


class XExchange:
    """All-gather of the distributed x: rank r holds x[rows_r]; every rank
    receives the full vector. Slices are padded to the largest one so the
    collective is a single all-gather (NCCL all_gather_into_tensor on GPU)."""

    def __init__(self, ranges: List[Tuple[int, int]], n_cols: int, device, dtype=None):
        import torch

        self.ranges = ranges
        self.sizes = [e - b for b, e in ranges]
        self.pad = max(self.sizes) if self.sizes else 0
        self.world = len(ranges)
        dtype = dtype or torch.float64
        self.local = torch.zeros(max(self.pad, 1), dtype=dtype, device=device)
        self.gathered = torch.empty(max(self.pad, 1) * self.world, dtype=dtype, device=device)
        self.full = torch.empty(n_cols, dtype=dtype, device=device)
        if sum(self.sizes) != n_cols or any(b != (ranges[i - 1][1] if i else 0) for i, (b, _) in enumerate(ranges)):
            raise ValueError("XExchange: row shards must tile x contiguously")

    def exchange(self, x_local, group=None):
        """x_local: this rank's slice (len = its rows). Returns the full x."""
        import torch
        import torch.distributed as dist

        n = x_local.numel()
        self.local[:n].copy_(x_local)
        if self.local.is_cuda:
            dist.all_gather_into_tensor(self.gathered, self.local, group=group)
        else:  # gloo
            parts = list(self.gathered.view(self.world, -1).unbind(0))
            dist.all_gather(parts, self.local, group=group)
        g = self.gathered.view(self.world, -1)
        for r, (b, e) in enumerate(self.ranges):
            if e > b:
                self.full[b:e].copy_(g[r, : e - b])
        return self.full
