"""Frozen vectors (tests/golden/solve_vectors.json, made by tests/golden/make_golden.py).

CPU (`-m "not gpu"`): the oracle still reproduces them (counts and rho_trace exactly, vectors to 1e-12:
an edit of the oracle that moves a result shows up against committed numbers).
GPU (`-m gpu`): the CUDA path through the C ABI against the same numbers, at north_star's bar: identical
iteration counts / status / rho-switch sequence (/root/reference/proj/src/solver.cpp:43-105), y, z,
lambda within 1e-6 relative; the warm-started solve (solver.cpp:144-156) and fixed_iters(30) too.
The batched path solves all instances of one workload as columns and must give the same per-column
counts and traces.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REL_SOL = 1e-6  # north_star tolerance


def _load():
    with open(os.path.join(HERE, "golden", "solve_vectors.json")) as f:
        return json.load(f)["cases"]


CASES = _load()
IDS = [f"{c['config']}-nu{c['nu']}-seed{c['seed']}" for c in CASES]


def vec(h):
    return np.array([float.fromhex(x) for x in h])


def trace(t):
    return [tuple(x) for x in t]


def rel_err(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(1.0, np.abs(np.asarray(b)).max()))


def workload(case):
    from workloads import problems
    return problems.config1(seed=case["seed"]) if case["config"] == "config1" else problems.config2(case["nu"], case["seed"])


def run_case(make_solver, case):
    """Cold solve, warm-started solve of the neighbouring instance, fixed_iters(30) from cold."""
    wl = workload(case)
    base = wl.base_problem()
    assert (base.n, base.m) == (case["n"], case["m"])
    q = wl.problem_at(wl.x0(case["x0_scale"]))
    s = make_solver(base)
    s.update_vectors(q.g, q.c, q.d)
    s.cold_start()
    rep = s.solve()
    q2 = wl.problem_at(wl.x0(case["warm"]["x0_scale"]))
    s.update_vectors(q2.g, q2.c, q2.d)
    s.warm_start(rep.solution)
    warm = s.solve().solution
    s.cold_start()
    fixed = s.fixed_iters(30).solution
    return rep, warm, fixed


def check(case, rep, warm, fixed, tol):
    sol = rep.solution
    assert sol.iterations == case["iterations"]
    assert int(sol.status) == case["status"]
    assert sol.rho_trace == trace(case["rho_trace"])
    assert [(h[0], h[3]) for h in rep.residual_history] == trace(case["history"])
    for name in ("y", "z", "lam"):
        assert rel_err(getattr(sol, name), vec(case[name])) <= tol, name
    assert warm.iterations == case["warm"]["iterations"]
    assert warm.rho_trace == trace(case["warm"]["rho_trace"])
    assert rel_err(warm.y, vec(case["warm"]["y"])) <= tol
    assert fixed.iterations == case["fixed30"]["iterations"] == 30
    assert rel_err(fixed.y, vec(case["fixed30"]["y"])) <= tol
    assert rel_err(fixed.lam, vec(case["fixed30"]["lam"])) <= tol


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_reproduces_golden(case):
    from oracle import oracle as O
    rep, warm, fixed = run_case(lambda b: O.Solver(O.QProblem(b.H, b.g, b.G, b.c, b.d)), case)
    check(case, rep, warm, fixed, 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_gpu_matches_golden(case):
    from paper_2311_18056_b200 import _lib, solver as S
    if _lib.load().cqp_device_count() < 1:
        pytest.fail("no CUDA device: the solve path has no CPU fallback")
    holder = []

    def make(b):
        holder.append(S.Solver(b.H, b.g, b.G, b.c, b.d))  # offline stage on the device
        return holder[0]
    rep, warm, fixed = run_case(make, case)
    check(case, rep, warm, fixed, REL_SOL)
    holder[0].close()


@pytest.mark.gpu
def test_gpu_batch_matches_golden_config1():
    """The config1 instances of seed 0 as columns of one batch next to the golden column."""
    from paper_2311_18056_b200 import _lib, solver as S
    if _lib.load().cqp_device_count() < 1:
        pytest.fail("no CUDA device: the solve path has no CPU fallback")
    case = CASES[0]
    wl = workload(case)
    base = wl.base_problem()
    scales = [case["x0_scale"], 1.0, 3.0, 0.3, case["x0_scale"]]
    qs = [wl.problem_at(wl.x0(sc)) for sc in scales]
    g, c, d = (np.asfortranarray(np.stack([getattr(q, k) for q in qs], axis=1)) for k in ("g", "c", "d"))
    single = S.Solver(base.H, base.g, base.G, base.c, base.d)
    batch = S.BatchSolver(single, capacity=len(qs))
    out = batch.solve(g, c, d)
    tr = batch.traces()
    for j in (0, len(qs) - 1):  # the golden instance sits in the first and the last column
        assert out["iterations"][j] == case["iterations"]
        assert out["status"][j] == case["status"]
        assert tr[j] == trace(case["rho_trace"])
        for name in ("y", "z", "lam"):
            assert rel_err(out[name][:, j], vec(case[name])) <= REL_SOL, name
    batch.close(); single.close()
