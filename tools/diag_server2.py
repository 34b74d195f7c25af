"""Scratch (GPU box): which entries of the first served step differ from the launch-per-step path."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_18056_b200 import problems, solver as S  # noqa: E402
name, k = sys.argv[1], int(sys.argv[2])
make = {"nu30": lambda: problems.config2(30, seed=0), "nu50": lambda: problems.config2(50, seed=0),
        "nu40": lambda: problems.config2(40, seed=0),
        "nu30nx80": lambda: problems.make_mpc_workload(30, 80, 10, 0), "nu45nx60": lambda: problems.make_mpc_workload(45, 60, 10, 0)}[name]
wl = make(); base = wl.base_problem()
gpu = S.Solver(base.H, base.g, base.G, base.c, base.d)
gpu.set_mpc_template(wl.tmpl, wl.limits)
n, m = base.n, base.m
def run(server):
    q = wl.problem_at(wl.x0(1.0))
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve()
    v_before = gpu.state.copy()
    if server: gpu.mpc_server_start(k)
    x = np.ascontiguousarray(wl.x0(1.0)) * float(os.environ.get('XSCALE', '1.0'))
    u0, rep = gpu.mpc_step_x0(x, k)
    if server: gpu.mpc_server_stop()
    s = rep.solution
    return dict(v0=v_before, u0=u0.copy(), y=s.y.copy(), z=s.z.copy(), lam=s.lam.copy(), v=gpu.state.copy(), layer=np.array([gpu.layer_index]),
                res=np.array([s.r_prim, s.r_dual]))
a, b = run(False), run(True)
for key in a:
    bad = np.where(a[key] != b[key])[0]
    print(key, len(a[key]), "n_bad", len(bad), "idx", bad[:12], "...", bad[-4:] if len(bad) else "", "max", np.abs(a[key]-b[key]).max())
R = gpu.launch_info()["rows_per_cta"]
bad = np.where(a["v"] != b["v"])[0]
bad = bad[(bad < n) | (bad >= n + m)]          # y and lambda rows (z rows differ by the early refresh)
ctas = {}
for i in bad: ctas.setdefault(int(i) // R, []).append(int(i) % R)
allc = (n + 2 * m + R - 1) // R
print("R", R, "CTAs with bad y/lam rows:", len(ctas), "of", allc)
print("good CTAs:", [c for c in range(allc) if c not in ctas and not (n <= c * R < n + m - R)])
print({c: r for c, r in list(ctas.items())[:40]})
