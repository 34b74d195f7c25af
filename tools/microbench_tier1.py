"""Scratch (GPU box): per-iteration time of the L2/HBM tier at robot-sized configs.
usage: microbench_tier1.py [atlas:N | quad:N ...]   (default atlas:30 quad:30)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import problems
from paper_2311_18056_b200 import solver as S
specs = sys.argv[1:] or ["atlas:30", "quad:30"]
for spec in specs:
    kind, N = spec.split(":"); N = int(N)
    wl = problems.config3_atlas(N, 0) if kind == "atlas" else problems.config4_quadruped(N, 0)
    base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
    res = {}
    for k in (2, 15, 200, 600):
        ts = []
        for _ in range(3):
            s.cold_start(); r = s.fixed_iters(k); ts.append(r.kernel_us)
        res[k] = sorted(ts)[1]
    D = base.n + 2 * base.m
    info = s.launch_info()
    per = (res[600] - res[200]) / 400.0
    print(spec, "D", D, info, {k: round(v, 1) for k, v in res.items()}, "us/iter %.2f" % per,
          "W MB/iter %.1f" % (info["w_bytes_per_iteration"] / 1e6), "W stream GB/s %.0f" % (info["w_bytes_per_iteration"] / per * 1e-3), flush=True)
    s.close()
