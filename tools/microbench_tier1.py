"""Scratch (GPU box): per-iteration time of the L2/HBM tier at the robot-sized configs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_18056_b200 import problems, solver as S
for name, wl in (("atlas30", problems.config3_atlas(30, 0)), ("quad30", problems.config4_quadruped(30, 0))):
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
    per = (res[600] - res[200]) / 400.0
    print(name, "D", D, s.launch_info(), {k: round(v, 1) for k, v in res.items()}, "us/iter %.2f" % per, "W stream GB/s %.0f" % (8.0 * D * D / per * 1e-3), flush=True)
    s.close()
