python - <<'PY'
import time, sys
sys.path.insert(0, ".")
from paper_2311_18056_b200 import problems, solver as S
for name, make in (("nu10", lambda: problems.config2(10, 0)), ("nu50", lambda: problems.config2(50, 0)), ("atlas30", lambda: problems.config3_atlas(30, 0)), ("quad30", lambda: problems.config4_quadruped(30, 0))):
    wl = make(); base = wl.base_problem()
    for rep in range(2):
        t0 = time.time(); s = S.Solver(base.H, base.g, base.G, base.c, base.d); t1 = time.time()
        q = wl.problem_at(wl.x0(10.0)); s.update_vectors(q.g, q.c, q.d); s.cold_start(); r = s.solve()
        print(name, "n", base.n, "m", base.m, "setup_s", round(t1 - t0, 3), "iters", r.solution.iterations, "status", r.solution.status, flush=True)
        s.close()
PY
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
