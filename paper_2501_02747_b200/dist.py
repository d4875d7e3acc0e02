"""Multi-GPU plumbing (one process per GPU, torch.distributed).

The hot path shards without any data-path exchange:
independent cities / snapshot ranges / pair row-blocks per rank. The only
collectives are the timing reductions of bench.py (max over ranks of the
device time, sum of the work units) and, for a row-sharded matrix, one
all-gather of bit rows. These helpers work on any backend (gloo on CPU in the
tests, nccl on the B200 box).
"""
from __future__ import annotations

from typing import Tuple


def shard(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [start, stop) of `total` items for `rank`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pair_row_blocks(n: int, world: int):
    """Row ranges [r0, r1) of the i<j pair triangle with near-equal pair
    counts (row i holds n-1-i pairs)."""
    total = n * (n - 1) // 2
    cum = [0]
    for i in range(n):
        cum.append(cum[-1] + n - 1 - i)   # pairs in rows [0, i+1)
    bounds = [0]
    row = 0
    for r in range(1, world):
        goal = r * total / world
        while row < n and cum[row] < goal:
            row += 1
        # pick the nearer of row-1 / row to the goal
        if row > 0 and abs(cum[row - 1] - goal) < abs(cum[row] - goal):
            row -= 1
        bounds.append(max(row, bounds[-1]))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def reduce_step_metrics(local_ms: float, local_units: float, device=None):
    """(max over ranks of the step time, sum over ranks of the work units)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([local_ms], dtype=torch.float64, device=device)
    u = torch.tensor([local_units], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t[0]), float(u[0])


def gather_bit_rows(rows, device=None):
    """All-gather equally shaped uint64 bit-row blocks (as int64 tensors)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [rows]
    out = [torch.empty_like(rows) for _ in range(dist.get_world_size())]
    dist.all_gather(out, rows)
    return out


def merge_bit_blocks(bits, device=None):
    """The full (B) matrix from the ranks' row blocks (Scene.pair_visibility(rows=...)):
    every rank holds a full-size uint64 matrix that is zero outside its own pairs, so an
    integer SUM all-reduce of the words is their OR (disjoint bits never carry) — one
    collective of N x ceil(N/64) x 8 bytes (config 4: 61 MB) over NVLink. `bits` is a
    numpy uint64 array; returns the merged array."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return bits
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int64).copy())
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy().view(np.uint64).reshape(bits.shape)
