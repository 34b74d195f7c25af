for sl in 0 200 500 800 1200; do for nu in 30 50; do CQP_IDLE_SLEEP_NS=$sl python - <<PY
import sys, os; sys.path.insert(0,'.')
from paper_2311_18056_b200 import problems, solver as S
wl = problems.config2($nu, 0); base = wl.base_problem()
s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
q = wl.problem_at(wl.x0(10.0)); s.update_vectors(q.g, q.c, q.d)
ts = {}
for k in (1000, 4000):
    v = []
    for _ in range(3):
        s.cold_start(); v.append(s.fixed_iters(k).kernel_us)
    ts[k] = sorted(v)[1]
print("sleep", $sl, "nu", $nu, "D", 3*base.n, "us/iter %.3f" % ((ts[4000]-ts[1000])/3000), flush=True)
PY
done; done
