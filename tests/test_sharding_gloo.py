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
    from workloads import problems
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


@pytest.mark.parametrize("B", [7, 1, 0])
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
    from workloads import problems
    wl = problems.config2(4, seed=2)
    g, c, d, _ = problems.batch_instances(wl, B)
    if B == 0:      # every shard is empty: empty results of the right shapes, no IndexError
        assert got["y"].shape == (wl.n, 0) and got["lam"].shape == (wl.m, 0) and got["iterations"].shape == (0,)
        return
    ref = _oracle_solve_fn(wl.base_problem())(g, c, d)
    for k in ref:
        assert np.array_equal(got[k], ref[k]), k


def test_bench_refuses_to_time_fewer_gpus_than_claimed():
    """`python bench.py --gpus N` spawns the N ranks itself; on a box with fewer than N devices it
    must fail loudly instead of timing one GPU under an N-GPU label."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 8:
        pytest.skip("8 CUDA devices are present")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "8", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2 and "only" in r.stderr and not r.stdout.strip()
