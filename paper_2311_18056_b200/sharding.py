"""Multi-GPU sharding of the batched path: independent QPs are split by column across ranks
(one process per GPU), every rank holds the full W ladder, and nothing crosses GPUs during the
solve; only the result columns are gathered.

`torch.distributed` is plumbing here: any initialised backend works ("nccl" on GPUs, "gloo" in
the CPU tests).  The per-rank solve is a callable so that the host logic can be exercised
without a GPU; on a GPU box it is `BatchSolver.solve`.
"""
from __future__ import annotations

from typing import Callable, Dict, Tuple

import numpy as np


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous column range [lo, hi) of `rank`: sizes differ by at most one, earlier ranks
    take the larger shards, empty shards are allowed (total < world)."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


RESULT_KEYS = ("y", "z", "lam", "status", "iterations", "final_index", "n_switches", "r_prim", "r_dual")


def solve_sharded(solve_fn: Callable[[np.ndarray, np.ndarray, np.ndarray], Dict[str, np.ndarray]],
                  g: np.ndarray, c: np.ndarray, d: np.ndarray, dst: int = 0):
    """Every rank passes the SAME global (g, c, d) (n x B, m x B, m x B); each solves its own
    column shard with `solve_fn`; rank `dst` receives the results re-assembled in the original
    column order (other ranks get None)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    B = g.shape[1]
    lo, hi = shard_range(B, world, rank)
    local = None
    if hi > lo:
        local = solve_fn(np.asfortranarray(g[:, lo:hi]), np.asfortranarray(c[:, lo:hi]),
                         np.asfortranarray(d[:, lo:hi]))
    payload = None if local is None else {k: np.ascontiguousarray(local[k]) for k in RESULT_KEYS}
    gathered = [None] * world if rank == dst else None
    dist.gather_object(payload, gathered, dst=dst)   # result gather: the only inter-rank traffic
    if rank != dst:
        return None
    out: Dict[str, np.ndarray] = {}
    for k in RESULT_KEYS:
        parts = [p[k] for p in gathered if p is not None]
        out[k] = np.concatenate(parts, axis=1 if parts[0].ndim == 2 else 0)
    assert out["iterations"].shape[0] == B
    return out
