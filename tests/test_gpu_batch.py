"""GPU parity tests of the batched path (FP64 DMMA grouped GEMM) vs the CPU oracle, column by
column: identical iteration counts, final ladder index and switch counts; y, lambda within 1e-6."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2311_18056_b200 import solver as S
    from paper_2311_18056_b200 import _lib
    if _lib.load().cqp_device_count() < 1:
        pytest.fail("no CUDA device: the solve path has no CPU fallback")
    return S


@pytest.fixture(scope="module")
def P():
    from workloads import problems
    return problems


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def oracle_columns(O, base, g, c, d):
    s = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d), variant="v3")
    out = []
    for j in range(g.shape[1]):
        s.update_vectors(g[:, j], c[:, j], d[:, j])
        s.cold_start()
        out.append(s.solve().solution)
    return s, out


@pytest.mark.parametrize("nu,B,unstable", [(10, 200, False), (10, 131, True), (4, 1, False), (20, 300, False)])
def test_batch_matches_per_column_oracle(G, oracle, P, nu, B, unstable):
    wl = P.config2(nu, seed=5, unstable=unstable)
    base = wl.base_problem()
    g, c, d, _ = P.batch_instances(wl, B, lo=0.3, hi=10.0)
    cpu, ref = oracle_columns(oracle, base, g, c, d)
    layers = {"W": [cpu.cache.W(k) for k in range(cpu.cache.L)], "D": [cpu.cache.D(k) for k in range(cpu.cache.L)],
              "GD": [cpu.cache.GD(k) for k in range(cpu.cache.L)], "grid": cpu.cache.grid,
              "initial_index": cpu.cache.initial_index, "Gs": cpu.cache.Gs, "E": cpu.cache.E,
              "F": cpu.cache.F, "cost_scale": cpu.cache.cost_scale}
    single = G.Solver(base.H, base.g, base.G, base.c, base.d, layers=layers)
    batch = G.BatchSolver(single, capacity=B)
    out = batch.solve(g, c, d)
    iters_ref = np.array([s.iterations for s in ref])
    assert np.array_equal(out["iterations"], iters_ref)
    assert np.array_equal(out["status"], np.array([s.status for s in ref]))
    assert np.array_equal(out["final_index"], np.array([s.rho_trace[-1][1] for s in ref]))
    assert np.array_equal(out["n_switches"], np.array([len(s.rho_trace) - 1 for s in ref]))
    assert len(set(iters_ref.tolist())) > 1 or B == 1      # the batch really is heterogeneous
    for j, s in enumerate(ref):
        assert rel_err(out["y"][:, j], s.y) <= 1e-6
        assert rel_err(out["lam"][:, j], s.lam) <= 1e-6
        assert rel_err(out["z"][:, j], s.z) <= 1e-6
        assert abs(out["r_prim"][j] - s.r_prim) <= 2e-3 * s.r_prim + 1e-9
        assert abs(out["r_dual"][j] - s.r_dual) <= 2e-3 * s.r_dual + 1e-9
        assert np.all(out["z"][:, j] >= c[:, j]) and np.all(out["z"][:, j] <= d[:, j])
    # second call on the same batch object (buffers are reused) and the single-QP kernel agree
    out = {k: np.array(v, copy=True) if isinstance(v, np.ndarray) else v for k, v in out.items()}  # (views of reused pinned buffers)
    out2 = batch.solve(g, c, d)
    assert np.array_equal(out2["iterations"], out["iterations"]) and np.array_equal(out2["y"], out["y"])
    single.update_vectors(g[:, 0], c[:, 0], d[:, 0]); single.cold_start()
    r = single.solve()
    assert r.solution.iterations == out["iterations"][0]
    assert rel_err(out["y"][:, 0], r.solution.y) <= 1e-9


def test_batch_max_iters_and_capacity(G, oracle, P):
    wl = P.config2(4, seed=1)
    base = wl.base_problem()
    g, c, d, _ = P.batch_instances(wl, 40, lo=5.0, hi=10.0)
    st = G.SolverSettings(eps_prim=1e-13, eps_dual=1e-13, max_iters=60)   # 2 checks + 10 trailing iterations
    so = oracle.SolverSettings(eps_prim=1e-13, eps_dual=1e-13, max_iters=60)
    single = G.Solver(base.H, base.g, base.G, base.c, base.d, st)
    batch = G.BatchSolver(single, capacity=64)
    out = batch.solve(g, c, d)
    cpu = oracle.Solver(oracle.QProblem(base.H, base.g, base.G, base.c, base.d), so)
    for j in range(40):
        cpu.update_vectors(g[:, j], c[:, j], d[:, j]); cpu.cold_start()
        s = cpu.solve().solution
        assert out["iterations"][j] == 60 == s.iterations
        assert out["status"][j] == s.status == G.MAX_ITERS
        assert out["n_switches"][j] == len(s.rho_trace) - 1
        assert rel_err(out["y"][:, j], s.y) <= 1e-6
    with pytest.raises(MemoryError):
        batch.solve(np.zeros((base.n, 65)), np.zeros((base.m, 65)), np.ones((base.m, 65)))


def test_structured_layer_matches_dense_layer(G, P, monkeypatch):
    """The batched layer skips the zeros of W's blocks (3,2) = -diag(rho), (3,3) = I
    (layers.cpp:159-161) and adds the two diagonal terms in the accumulator's start value.
    CQP_BATCH_DENSE=1 multiplies the full dense W instead: counts, traces and statuses must be
    identical, solutions equal to rounding -- on a batch with heterogeneous iteration counts and
    rho switches, and with n + m not a multiple of the tile sizes."""
    wl = P.config2(10, seed=5)
    base = wl.base_problem()
    B = 700
    g, c, d, _ = P.batch_instances(wl, B, lo=0.3, hi=10.0)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CQP_BATCH_DENSE", flag)
        single = G.Solver(base.H, base.g, base.G, base.c, base.d)
        batch = G.BatchSolver(single, capacity=B)
        outs.append({k: np.array(v, copy=True) if isinstance(v, np.ndarray) else v for k, v in batch.solve(g, c, d).items()})
        batch.close(); single.close()
    monkeypatch.delenv("CQP_BATCH_DENSE", raising=False)
    a, b = outs
    assert b["gemm_flops"] < 0.85 * a["gemm_flops"]            # the structured layer really ran
    assert len(set(a["iterations"].tolist())) > 3 and a["n_switches"].max() >= 1
    for key in ("iterations", "status", "final_index", "n_switches"):
        assert np.array_equal(a[key], b[key]), key
    for key in ("y", "z", "lam"):
        assert rel_err(a[key], b[key]) <= 1e-9, key


def test_lanes_match_one_batch(G, oracle, P, monkeypatch):
    """Batches of >= 1024 columns are cut into two sub-batches that run concurrently on their own
    streams (their GEMM launches fill each other's wave tails).  Columns are independent QPs, so
    counts, traces and statuses must equal the single-lane run; values agree to rounding only
    (the tile shape / k-split of a round follows the lane's active-column count, which changes
    the summation order).  A sample of columns is checked against the oracle as well."""
    wl = P.config2(10, seed=5)
    base = wl.base_problem()
    B = 1100
    g, c, d, _ = P.batch_instances(wl, B, lo=0.3, hi=10.0)
    outs = []
    for lanes in ("1", "2", "3"):
        monkeypatch.setenv("CQP_BATCH_LANES", lanes)
        single = G.Solver(base.H, base.g, base.G, base.c, base.d)
        batch = G.BatchSolver(single, capacity=B)
        outs.append({k: np.array(v, copy=True) if isinstance(v, np.ndarray) else v for k, v in batch.solve(g, c, d).items()})
        small = batch.solve(g[:, :500], c[:, :500], d[:, :500])     # < 512 columns: one lane if it has the capacity (not with 3)
        assert np.array_equal(small["iterations"], outs[0]["iterations"][:500])
        small = batch.solve(g[:, :100], c[:, :100], d[:, :100])     # small batch on a multi-lane object: one lane
        assert np.array_equal(small["iterations"], outs[0]["iterations"][:100])
        assert rel_err(small["y"], outs[0]["y"][:, :100]) <= 1e-9
        batch.close(); single.close()
    monkeypatch.delenv("CQP_BATCH_LANES", raising=False)
    a = outs[0]
    assert len(set(a["iterations"].tolist())) > 3 and a["n_switches"].max() >= 1
    for b in outs[1:]:
        for key in ("iterations", "status", "final_index", "n_switches"):
            assert np.array_equal(a[key], b[key]), key
        for key in ("y", "z", "lam"):
            assert rel_err(a[key], b[key]) <= 1e-9, key
        assert b["compute_ms"] > 0 and b["gemm_ms"] > 0 and b["gemm_flops"] == a["gemm_flops"]
    cpu = oracle.Solver(oracle.QProblem(base.H, base.g, base.G, base.c, base.d), variant="v3")
    for j in list(range(0, B, 97)) + [B - 1]:
        cpu.update_vectors(g[:, j], c[:, j], d[:, j]); cpu.cold_start()
        s = cpu.solve().solution
        assert outs[1]["iterations"][j] == s.iterations and outs[1]["status"][j] == s.status
        assert rel_err(outs[1]["y"][:, j], s.y) <= 1e-6 and rel_err(outs[1]["lam"][:, j], s.lam) <= 1e-6


def test_solve_sharded_paths_at_world_one(G, P):
    """The multi-GPU host logic with the real BatchSolver as the per-rank solve, at world size 1
    (one GPU box): `solve_sharded` (object gather) and `solve_sharded_device` (results stay in
    device memory until the NCCL gather) both reproduce a plain `BatchSolver.solve`."""
    import torch.distributed as dist
    from paper_2311_18056_b200 import sharding
    wl = P.config2(6, seed=3)
    base = wl.base_problem()
    B = 150
    g, c, d, _ = P.batch_instances(wl, B)
    single = G.Solver(base.H, base.g, base.G, base.c, base.d)
    batch = G.BatchSolver(single, capacity=B)
    ref = batch.solve(g, c, d)
    out_dev, timing = sharding.solve_sharded_device(batch, g, c, d)       # no process group: world 1
    assert timing["compute_ms"] > 0 and timing["launches"] > 0
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        out_obj = sharding.solve_sharded(lambda a, b_, c_: batch.solve(a, b_, c_), g, c, d)
    finally:
        dist.destroy_process_group()
    for out in (out_dev, out_obj):
        for key in sharding.RESULT_KEYS:
            assert np.array_equal(out[key], ref[key]), key
    batch.close(); single.close()


def _nccl_worker(rank, world, port, B, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from workloads import problems
    from paper_2311_18056_b200 import sharding, solver as S
    wl = problems.config2(6, seed=3)
    base = wl.base_problem()
    g, c, d, _ = problems.batch_instances(wl, B)
    single = S.Solver(base.H, base.g, base.G, base.c, base.d, device=rank)
    lo, hi = sharding.shard_range(B, world, rank)
    batch = S.BatchSolver(single, capacity=max(hi - lo, 1))
    out, _ = sharding.solve_sharded_device(batch, g, c, d, dst=0)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_solve_sharded_device_two_gpus(G, P):
    """World size 2 over NCCL (needs two GPUs; the 1-GPU boxes skip it)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 CUDA devices")
    B = 151
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, B, q)) for r in range(2)]
    [p.start() for p in procs]
    got = q.get(timeout=600)
    [p.join(timeout=120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    wl = P.config2(6, seed=3)
    base = wl.base_problem()
    g, c, d, _ = P.batch_instances(wl, B)
    single = G.Solver(base.H, base.g, base.G, base.c, base.d)
    ref = G.BatchSolver(single, capacity=B).solve(g, c, d)
    for key in ("iterations", "status", "final_index", "n_switches"):
        assert np.array_equal(got[key], ref[key]), key
    for key in ("y", "z", "lam"):
        assert rel_err(got[key], ref[key]) <= 1e-9, key


def test_batch_traces_and_histories_match_single_solver(G, oracle, P):
    """cqp_batch_get_traces / cqp_batch_get_history: column j's records equal what the oracle's
    `solve()` reports for that column (problem.hpp:57-70, solver.hpp:56-67), also through the lanes."""
    wl = P.config2(10, seed=5)
    base = wl.base_problem()
    B = 1100                                                     # >= 1024: two lanes
    g, c, d, _ = P.batch_instances(wl, B, lo=0.3, hi=10.0)
    cpu = oracle.Solver(oracle.QProblem(base.H, base.g, base.G, base.c, base.d), variant="ref")
    layers = {"W": [cpu.cache.W(k) for k in range(cpu.cache.L)], "D": [cpu.cache.D(k) for k in range(cpu.cache.L)],
              "GD": [cpu.cache.GD(k) for k in range(cpu.cache.L)], "grid": cpu.cache.grid,
              "initial_index": cpu.cache.initial_index, "Gs": cpu.cache.Gs, "E": cpu.cache.E,
              "F": cpu.cache.F, "cost_scale": cpu.cache.cost_scale}
    single = G.Solver(base.H, base.g, base.G, base.c, base.d, layers=layers)
    batch = G.BatchSolver(single, capacity=B)
    out = batch.solve(g, c, d)
    traces, hists = batch.traces(), batch.histories()
    assert max(len(t) for t in traces) >= 2
    for j in list(range(0, B, 13)) + [B - 1]:
        cpu.update_vectors(g[:, j], c[:, j], d[:, j]); cpu.cold_start()
        ro = cpu.solve()
        assert traces[j] == ro.solution.rho_trace, j
        assert [(h[0], h[3]) for h in hists[j]] == [(h[0], h[3]) for h in ro.residual_history], j
        for hg, ho in zip(hists[j], ro.residual_history):
            assert abs(hg[1] - ho[1]) <= 2e-3 * abs(ho[1]) + 1e-9 and abs(hg[2] - ho[2]) <= 2e-3 * abs(ho[2]) + 1e-9
        assert out["iterations"][j] == ro.solution.iterations
    small = batch.solve(g[:, :40], c[:, :40], d[:, :40])         # one lane of the same object
    assert batch.traces() == traces[:40] and len(batch.histories()) == 40
    assert np.array_equal(small["iterations"], out["iterations"][:40])
    with pytest.raises(ValueError):                              # results are copies: closing is safe
        batch.close(); batch.solve(g, c, d)
    assert out["y"].flags.owndata or out["y"].base is not None
    single.close()


@pytest.mark.parametrize("nu,B", [(10, 200), (20, 333)])
def test_round_kernel_matches_per_iteration_kernel(G, P, monkeypatch, nu, B):
    """The persistent TMA round kernel (one launch per check round, dataflow dependencies between the
    iterations of a column tile, cqp_batch_round.cuh) against the per-iteration cp.async kernel
    (CQP_BATCH_LEGACY=1) on the same slot-ordered iterate, for EVERY tile configuration of the round
    kernel.  The per-element summation order (k-tiles, then k-steps, ascending) is the same in both
    kernels unless warp groups split k, so: bit-identical results for the plain configurations, and
    counts / statuses / final indices / switch counts identical with values equal to rounding for
    the k-split ones.  nu = 10 has n + m = 200: 32-row tiles leave a row tile of padding only between
    the two parts of the structured layer (the skipped tile must not count as a completion)."""
    wl = P.config2(nu, seed=5)
    base = wl.base_problem()
    g, c, d, _ = P.batch_instances(wl, B, lo=0.3, hi=10.0)

    def run(env):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        single = G.Solver(base.H, base.g, base.G, base.c, base.d)
        batch = G.BatchSolver(single, capacity=B)
        out = {k: np.array(v, copy=True) if isinstance(v, np.ndarray) else v for k, v in batch.solve(g, c, d).items()}
        out["traces"] = batch.traces()
        batch.close(); single.close()
        for k in env:
            monkeypatch.delenv(k, raising=False)
        return out

    ref = run({"CQP_BATCH_LEGACY": "1", "CQP_BATCH_FORCE_CFG": "3"})
    assert len(set(ref["iterations"].tolist())) > 3 and ref["n_switches"].max() >= 1
    assert ref["launches"] > 25 * ref["rounds"]                       # one launch per iteration
    ksplit = {4, 5, 7, 8}
    for cfg in range(1, 10):
        # (CQP_BATCH_KX=1,0: no K split over CTAs, which adds a tile's products up in another order)
        out = run({"CQP_BATCH_FORCE_CFG": str(cfg), "CQP_BATCH_KX": "1,0"})
        assert out["launches"] < 16 * out["rounds"], cfg              # one launch per ROUND
        for key in ("iterations", "status", "final_index", "n_switches"):
            assert np.array_equal(ref[key], out[key]), (cfg, key)
        assert ref["traces"] == out["traces"], cfg
        for key in ("y", "z", "lam"):
            if cfg in ksplit:
                assert rel_err(out[key], ref[key]) <= 1e-9, (cfg, key)
            else:
                assert np.array_equal(out[key], ref[key]), (cfg, key)
    # K loops split over 2 ... 8 CTAs in EVERY round (threshold above B; the default plan uses 4 and 6): the last split to arrive adds the
    # partial tiles up in split order, so the result does not depend on the arrival order: two runs agree bit
    # for bit, and with the unsplit kernel to rounding
    for kx in ("2", "3", "4", "6", "8"):
        a = run({"CQP_BATCH_FORCE_CFG": "6", "CQP_BATCH_KX": kx + ",100000"})
        b = run({"CQP_BATCH_FORCE_CFG": "6", "CQP_BATCH_KX": kx + ",100000"})
        for key in ("iterations", "status", "final_index", "n_switches"):
            assert np.array_equal(ref[key], a[key]), (kx, key)
        assert ref["traces"] == a["traces"], kx
        for key in ("y", "z", "lam"):
            assert rel_err(a[key], ref[key]) <= 1e-9, (kx, key)
            assert np.array_equal(a[key], b[key]), (kx, key)
    out = run({})                                                      # the default plan
    for key in ("iterations", "status", "final_index", "n_switches"):
        assert np.array_equal(ref[key], out[key]), key
