"""Scratch (GPU box): per-iteration time of the shared-memory-resident tier for the nu sweep under the
environment's knobs (CQP_COFETCH / CQP_WREG / CQP_DIRECT_WAIT_GO / CQP_POLL_DELAY_NS), plus a hash of the
iterate after 1000 iterations so that runs under different knobs can be compared bit for bit."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from workloads import problems
from paper_2311_18056_b200 import solver as S

nus = [int(a) for a in sys.argv[1:]] or [22, 30, 38, 50]
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("CQP_") and k != "CQP_B200_LIB")
for nu in nus:
    wl = problems.config2(nu, 0)
    base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    q = wl.problem_at(wl.x0(10.0))
    s.update_vectors(q.g, q.c, q.d)
    t = {}
    for k in (1000, 4000):
        ts = []
        for _ in range(5):
            s.cold_start()
            r = s.fixed_iters(k)
            ts.append(r.kernel_us)
        t[k] = sorted(ts)[2]
    s.cold_start()
    r = s.fixed_iters(1000)
    h = hashlib.sha1(np.concatenate([r.solution.y, r.solution.z, r.solution.lam]).tobytes()).hexdigest()[:12]
    s.cold_start()
    rs = s.solve()
    print(json.dumps({"knobs": tag, "nu": nu, "D": 3 * base.n, "us_per_iter": round((t[4000] - t[1000]) / 3000.0, 4),
                      "hash1000": h, "solve_iters": rs.solution.iterations, "solve_us": round(rs.kernel_us, 1),
                      "launch": s.launch_info()}), flush=True)
