"""Scratch (GPU box): the same problem in several Solver instances of one process (all kept alive, so their
device buffers sit at different addresses): per-iteration time of each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import problems
from paper_2311_18056_b200 import solver as S
nu = int(sys.argv[1]) if len(sys.argv) > 1 else 30
count = int(sys.argv[2]) if len(sys.argv) > 2 else 6
wl = problems.config2(nu, 0)
base = wl.base_problem()
q = wl.problem_at(wl.x0(10.0))
keep = []
for k in range(count):
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000, check_interval=int(os.environ.get("CHECK", "25"))))
    keep.append(s)
    s.update_vectors(q.g, q.c, q.d)
    t = {}
    for it in (1000, 4000):
        ts = []
        for _ in range(3):
            s.cold_start(); ts.append(s.fixed_iters(it).kernel_us)
        t[it] = sorted(ts)[1]
    print("nu", nu, "instance", k, "us/iter %.3f" % ((t[4000] - t[1000]) / 3000.0), flush=True)
# and once more on the first instance
s = keep[0]
t = {}
for it in (1000, 4000):
    ts = []
    for _ in range(3):
        s.cold_start(); ts.append(s.fixed_iters(it).kernel_us)
    t[it] = sorted(ts)[1]
print("nu", nu, "instance 0 again", "us/iter %.3f" % ((t[4000] - t[1000]) / 3000.0))
