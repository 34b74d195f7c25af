"""CPU, world_size 2, gloo: the column-sharding host logic of the batched path.  The per-rank
solve is the CPU oracle here (test infrastructure); on GPUs it is BatchSolver.solve."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def test_shard_range_covers_everything():
    from paper_2311_18056_b200.sharding import shard_range
    for total in (0, 1, 2, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for a, b in zip(ranges, ranges[1:]):
                assert a[1] == b[0]
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _oracle_solve_fn(base):
    from oracle import oracle as O
    solver = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d), variant="v3")

    def fn(g, c, d):
        B = g.shape[1]
        out = {"y": np.empty((base.n, B)), "z": np.empty((base.m, B)), "lam": np.empty((base.m, B)),
               "status": np.empty(B, np.int32), "iterations": np.empty(B, np.int32),
               "final_index": np.empty(B, np.int32), "n_switches": np.empty(B, np.int32),
               "r_prim": np.empty(B), "r_dual": np.empty(B)}
        for j in range(B):
            solver.update_vectors(g[:, j], c[:, j], d[:, j]); solver.cold_start()
            s = solver.solve().solution
            out["y"][:, j], out["z"][:, j], out["lam"][:, j] = s.y, s.z, s.lam
            out["status"][j], out["iterations"][j] = s.status, s.iterations
            out["final_index"][j], out["n_switches"][j] = s.rho_trace[-1][1], len(s.rho_trace) - 1
            out["r_prim"][j], out["r_dual"][j] = s.r_prim, s.r_dual
        return out
    return fn


def _worker(rank, world, port, B, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_18056_b200 import problems
    from paper_2311_18056_b200.sharding import solve_sharded
    wl = problems.config2(4, seed=2)
    g, c, d, _ = problems.batch_instances(wl, B)
    out = solve_sharded(_oracle_solve_fn(wl.base_problem()), g, c, d, dst=0)
    if rank == 0:
        q.put({k: v for k, v in out.items()})
    else:
        assert out is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 1])
def test_solve_sharded_world2_matches_single_process(B):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    [p.start() for p in procs]
    got = q.get(timeout=180)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    from paper_2311_18056_b200 import problems
    wl = problems.config2(4, seed=2)
    g, c, d, _ = problems.batch_instances(wl, B)
    ref = _oracle_solve_fn(wl.base_problem())(g, c, d)
    for k in ref:
        assert np.array_equal(got[k], ref[k]), k
