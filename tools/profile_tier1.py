"""Scratch (GPU box): one solve at the quadruped-sized config (D = 4080, L2/HBM tier) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import problems
from paper_2311_18056_b200 import solver as S
wl = problems.config4_quadruped(30, 0) if (len(sys.argv) < 2 or sys.argv[1] == "quad") else problems.config3_atlas(30, 0)
base = wl.base_problem()
s = S.Solver(base.H, base.g, base.G, base.c, base.d)
q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
for _ in range(2):
    s.cold_start(); r = s.fixed_iters(100)
print("iterations", r.solution.iterations, "kernel_us", r.kernel_us, s.launch_info())
