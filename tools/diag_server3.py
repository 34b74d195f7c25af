"""Scratch (GPU box): dump W, v_0 (refreshed) and v_1 of both paths for an offline look at the summation order."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_18056_b200 import problems, solver as S  # noqa: E402
wl = problems.config2(50, seed=0); base = wl.base_problem()
gpu = S.Solver(base.H, base.g, base.G, base.c, base.d)
gpu.set_mpc_template(wl.tmpl, wl.limits)
n, m = base.n, base.m
out = {}
def run(server, k):
    q = wl.problem_at(wl.x0(1.0))
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve()
    if server: gpu.mpc_server_start(k)
    x = np.ascontiguousarray(wl.x0(1.0))
    u0, rep = gpu.mpc_step_x0(x, k)
    if server: gpu.mpc_server_stop()
    return gpu.state.copy(), gpu.layer_index
v0, li = run(False, 0)
out["v0"] = v0; out["layer"] = np.array([li])
out["v1_launch"], _ = run(False, 1)
out["v1_server"], _ = run(True, 1)
# fixed_iters path
q = wl.problem_at(wl.x0(1.0)); gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve(); gpu.refresh_z(); gpu.fixed_iters(1)
out["v1_fixed"] = gpu.state.copy()
out["W"] = gpu.layer(li)["W"]
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/diag3.npz", **out)
print("saved", li)
