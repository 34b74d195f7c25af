"""Scratch (GPU box): one single-QP solve at nu=50 (D=1500) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import problems
from paper_2311_18056_b200 import solver as S
nu = int(sys.argv[1]) if len(sys.argv) > 1 else 50
wl = problems.config2(nu, 0); base = wl.base_problem()
s = S.Solver(base.H, base.g, base.G, base.c, base.d)
q = wl.problem_at(wl.x0(10.0)); s.update_vectors(q.g, q.c, q.d)
for _ in range(2):
    s.cold_start(); r = s.solve()
print("iterations", r.solution.iterations, "kernel_us", r.kernel_us)
