"""Scratch (GPU box): per-step comparison of the closed loop, launch per step vs resident server.
  python tools/diag_server.py nu50 2 400"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_18056_b200 import problems, solver as S  # noqa: E402
name, k, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
fast = os.environ.get("FAST", "1") == "1"
make = {"nu30": lambda: problems.config2(30, seed=0), "nu50": lambda: problems.config2(50, seed=0),
        "nu40": lambda: problems.config2(40, seed=0), "atlas30": lambda: problems.config3_atlas(30, seed=0)}[name]
wl = make(); base = wl.base_problem()
gpu = S.Solver(base.H, base.g, base.G, base.c, base.d)
gpu.set_mpc_template(wl.tmpl, wl.limits)
print(gpu.launch_info())
A, B = wl.sys.A, wl.sys.B
def run(server):
    q = wl.problem_at(wl.x0(1.0))
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve()
    if server: gpu.mpc_server_start(k)
    x = np.ascontiguousarray(wl.x0(1.0)); us = []
    for t in range(steps):
        if fast:
            u0 = np.zeros(wl.sys.nu); gpu.mpc_step_x0_fast(x, k, u0)
        else:
            u0, rep = gpu.mpc_step_x0(x, k)
        us.append(u0.copy()); x = np.ascontiguousarray(A @ x + B @ u0)
    if server: gpu.mpc_server_stop()
    return np.array(us)
runs = [("launch", run(False)), ("launch", run(False)), ("server", run(True)), ("server", run(True)), ("server", run(True))]
ref = runs[0][1]
for nm, u in runs[1:]:
    bad = np.where((u != ref).any(axis=1))[0]
    print(nm, "identical" if len(bad) == 0 else f"first diff at step {bad[0]} of {steps}, n_bad={len(bad)}, max|du| at first={np.abs(u[bad[0]]-ref[bad[0]]).max():.3e}", flush=True)
