"""Scratch (GPU box): small solves through every kernel tier, for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from workloads import problems
from paper_2311_18056_b200 import solver as S
which = sys.argv[1] if len(sys.argv) > 1 else "all"
def run(tag, wl, env=None, k=60):
    for kk, v in (env or {}).items(): os.environ[kk] = v
    base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d)
    q = wl.problem_at(wl.x0(3.0)); s.update_vectors(q.g, q.c, q.d); s.cold_start()
    r = s.fixed_iters(k)
    s.set_mpc_template(wl.tmpl, wl.limits)
    u0, r2 = s.mpc_step_x0(wl.x0(1.0), 2)
    print(tag, s.launch_info(), r.solution.iterations, float(np.abs(r.solution.y).max()), u0[:2], flush=True)
    s.close()
    for kk in (env or {}): os.environ.pop(kk, None)
if which in ("all", "cluster"):
    run("cluster-reg", problems.config2(6, 1))                       # D = 180: register mode
    run("cluster-smem", problems.config2(6, 1), {"CQP_CLUSTER_MODE": "smem"})
if which in ("all", "grid"):
    run("grid-resident", problems.config2(6, 1), {"CQP_FORCE_TIER": "0"})                      # direct fetch, W in registers
    run("grid-resident-wsmem", problems.config2(6, 1), {"CQP_FORCE_TIER": "0", "CQP_WREG": "0"})  # direct fetch, W in shared memory
    run("grid-resident-staged", problems.config2(6, 1), {"CQP_FORCE_TIER": "0", "CQP_COFETCH": "1"})
    run("grid-resident-540", problems.config2(18, 1), k=30)                                       # D = 540: the default grid size class
    run("grid-stream", problems.config2(6, 1), {"CQP_FORCE_TIER": "1", "CQP_SINGLE_DENSE": "1"})
    run("grid-stream-structured", problems.config2(6, 1), {"CQP_FORCE_TIER": "1", "CQP_FORCE_STRUCTURED": "1"})
    run("grid-stream-structured-odd", problems.config2(7, 1), {"CQP_FORCE_TIER": "1", "CQP_FORCE_STRUCTURED": "1"})
if which in ("all", "batch"):
    wl = problems.config2(6, 1); base = wl.base_problem()
    g, c, d, _ = problems.batch_instances(wl, 96)
    s = S.Solver(base.H, base.g, base.G, base.c, base.d)
    b = S.BatchSolver(s, 96)
    out = b.solve(g, c, d)
    print("batch", out["iterations"][:8], flush=True)
    b.close()
    os.environ["CQP_BATCH_KX"] = "1,0"             # no K split over CTAs
    b = S.BatchSolver(s, 96)
    out = b.solve(g, c, d)
    print("batch-nosplit", out["iterations"][:8], flush=True)
    b.close()
    os.environ.pop("CQP_BATCH_KX")
    os.environ["CQP_BATCH_LANES"] = "2"           # two concurrent lanes (sub-batches on their own streams)
    g, c, d, _ = problems.batch_instances(wl, 640)
    b = S.BatchSolver(s, 640)
    out = b.solve(g, c, d)
    print("batch-lanes", out["iterations"][:8], out["launches"], flush=True)
    b.close()
    os.environ["CQP_BATCH_DENSE"] = "1"           # dense layer (A/B switch)
    b = S.BatchSolver(s, 96)
    out = b.solve(g[:, :96], c[:, :96], d[:, :96])
    print("batch-dense", out["iterations"][:8], flush=True)
