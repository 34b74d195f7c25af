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
    if B == 0:   # every shard is empty: nothing was solved, return empty results of the right shapes
        n, m = g.shape[0], c.shape[0]
        empty = {"y": np.zeros((n, 0)), "z": np.zeros((m, 0)), "lam": np.zeros((m, 0)),
                 "r_prim": np.zeros(0), "r_dual": np.zeros(0)}
        return {k: empty.get(k, np.zeros(0, dtype=np.int32)) for k in RESULT_KEYS}
    for k in RESULT_KEYS:
        parts = [p[k] for p in gathered if p is not None]
        out[k] = np.concatenate(parts, axis=1 if parts[0].ndim == 2 else 0)
    assert out["iterations"].shape[0] == B
    return out


def solve_sharded_device(batch, g: np.ndarray, c: np.ndarray, d: np.ndarray, dst: int = 0, pinned=None):
    """The GPU path of `solve_sharded` (one process per GPU, backend "nccl"): every rank passes the
    SAME global (g, c, d); rank r solves columns shard_range(B, world, r) with its `BatchSolver`
    (`batch`, capacity >= the largest shard), the results stay in device memory and are gathered
    to rank `dst` with NCCL (`dist.gather`; shards are padded to the largest one), which copies
    them to the host.  No other inter-GPU traffic.  Returns (results on `dst` | None, timing dict).

    `pinned`: optional (g, c, d) page-locked copies of this rank's shard, column-major, to upload
    from (bench.py); otherwise the shard is sliced from the global arrays."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    n, m, B = g.shape[0], c.shape[0], g.shape[1]
    lo, hi = shard_range(B, world, rank)
    cnt, per = hi - lo, shard_range(B, world, 0)[1] - shard_range(B, world, 0)[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    y = torch.zeros((max(per, 1), n), **f64); z = torch.zeros((max(per, 1), m), **f64)
    lam = torch.zeros((max(per, 1), m), **f64)
    ints = torch.zeros((4, max(per, 1)), dtype=torch.int32, device=dev)     # status, iterations, final_index, n_switches
    res = torch.zeros((2, max(per, 1)), **f64)                             # r_prim, r_dual
    timing = {"compute_ms": 0.0, "device_ms": 0.0, "launches": 0, "gemm_ms": 0.0, "gemm_flops": 0.0, "rounds": 0}
    if cnt > 0:
        if pinned is not None:
            gl, cl, dl = pinned
        else:
            gl, cl, dl = (np.asfortranarray(a[:, lo:hi]) for a in (g, c, d))
        ip = ints.data_ptr()
        timing = batch.solve_into(cnt, gl.ctypes.data, cl.ctypes.data, dl.ctypes.data, y.data_ptr(), z.data_ptr(),
                                  lam.data_ptr(), ip, ip + 4 * per, ip + 8 * per, res.data_ptr(),
                                  res.data_ptr() + 8 * per, ip + 12 * per)
        keep = (gl, cl, dl)  # noqa: F841  (alive until the call returned: it synchronises its stream)
    parts = {}
    for name, t in (("y", y), ("z", z), ("lam", lam), ("ints", ints), ("res", res)):
        if world > 1:
            bucket = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
            dist.gather(t, bucket, dst=dst)       # result gather over NCCL: the only inter-GPU traffic
        else:
            bucket = [t]
        parts[name] = bucket
    if rank != dst:
        return None, timing
    out: Dict[str, np.ndarray] = {}
    sizes = [shard_range(B, world, r)[1] - shard_range(B, world, r)[0] for r in range(world)]
    cat = lambda name, sl: torch.cat([sl(t, k) for t, k in zip(parts[name], sizes)], dim=0).cpu().numpy()  # noqa: E731
    out["y"] = cat("y", lambda t, k: t[:k]).T
    out["z"] = cat("z", lambda t, k: t[:k]).T
    out["lam"] = cat("lam", lambda t, k: t[:k]).T
    for i, key in enumerate(("status", "iterations", "final_index", "n_switches")):
        out[key] = cat("ints", lambda t, k, i=i: t[i, :k])
    for i, key in enumerate(("r_prim", "r_dual")):
        out[key] = cat("res", lambda t, k, i=i: t[i, :k])
    assert out["iterations"].shape[0] == B
    return out, timing
