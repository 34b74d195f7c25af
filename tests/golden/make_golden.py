"""Generates the frozen vectors under tests/golden/ (run once, commit the output):

    python tests/golden/make_golden.py

The reference (C++ / Eigen) cannot be built in this image and ships no vector files; what pins the
solve path are its known-answer tests, re-asserted on the oracle in tests/test_oracle_known_answers.py.
These fixtures freeze the outputs of THAT oracle (oracle/clampqp_oracle.c, reference flags) on the
BASELINE.json workloads, so that (a) a later edit of the oracle that moves an iteration count, a
rho_trace or a solution shows up as a diff against committed numbers (tests/test_golden.py, CPU), and
(b) the GPU path is also compared with numbers that do not come from the same process
(tests/test_golden.py -m gpu).  Inputs are regenerated from (config, nu, seed, x0 scale) by
workloads/problems.py; floats are stored as C99 hex strings, i.e. bit for bit.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from workloads import problems  # noqa: E402

# (name, nu, seed, x0 scale): configs[0] and points of the configs[1] sweep (nx = 2 nu, N = 10)
CASES = [("config1", 10, 0, 10.0), ("config1", 10, 1, 3.0), ("config1", 10, 2, 0.5),
         ("config2", 14, 0, 10.0), ("config2", 18, 3, 5.0), ("config2", 22, 1, 10.0), ("config2", 30, 0, 10.0)]


def workload(name, nu, seed):
    return problems.config1(seed=seed) if name == "config1" else problems.config2(nu, seed)


def hexes(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def main():
    out = []
    for name, nu, seed, scale in CASES:
        wl = workload(name, nu, seed)
        base = wl.base_problem()
        q = wl.problem_at(wl.x0(scale))
        s = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d))
        s.update_vectors(q.g, q.c, q.d)
        s.cold_start()
        rep = s.solve()
        sol = rep.solution
        # a second, warm-started solve of a neighbouring instance (solver.cpp:144-156) and a fixed_iters(30)
        q2 = wl.problem_at(wl.x0(0.9 * scale))
        s.update_vectors(q2.g, q2.c, q2.d)
        s.warm_start(sol)
        warm = s.solve().solution
        s.cold_start()
        fixed = s.fixed_iters(30).solution
        out.append({
            "config": name, "nu": nu, "seed": seed, "x0_scale": scale, "n": base.n, "m": base.m,
            "status": int(sol.status), "iterations": int(sol.iterations),
            "rho_trace": [[int(a), int(b)] for a, b in sol.rho_trace],
            "history": [[int(h[0]), int(h[3])] for h in rep.residual_history],
            "r_prim": float(sol.r_prim).hex(), "r_dual": float(sol.r_dual).hex(),
            "y": hexes(sol.y), "z": hexes(sol.z), "lam": hexes(sol.lam),
            "warm": {"x0_scale": 0.9 * scale, "iterations": int(warm.iterations),
                     "rho_trace": [[int(a), int(b)] for a, b in warm.rho_trace], "y": hexes(warm.y)},
            "fixed30": {"iterations": int(fixed.iterations), "y": hexes(fixed.y), "lam": hexes(fixed.lam)},
        })
        print(name, nu, seed, scale, "->", sol.iterations, sol.rho_trace, "warm", warm.iterations)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "solve_vectors.json")
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "oracle": "oracle/clampqp_oracle.c (-O3 -DNDEBUG)",
                   "cases": out}, f, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
