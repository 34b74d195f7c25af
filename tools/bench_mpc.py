"""Receding-horizon MPC step benchmark (BASELINE.json configs[0], [2], [3]): per control step
{instantiate (host), update_vectors, refresh_z, fixed_iters(k)} -- the protocol of
/root/reference/proj/src/bench.cpp:157-185 -- through cqp_mpc_step on the GPU, next to the CPU
oracle on the same closed loop.  Writes profiles/<tag>_mpc_steps.json (run on a B200 box)."""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from workloads import problems  # noqa: E402
from paper_2311_18056_b200 import solver as S  # noqa: E402

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["config1", "atlas30", "quad30"]
CASES = {
    "config1": (lambda: problems.config1(seed=0), 1, 1.0),
    "config1_k2": (lambda: problems.config1(seed=0), 2, 1.0),
    "nu50": (lambda: problems.config2(50, seed=0), 2, 1.0),
    "atlas30": (lambda: problems.config3_atlas(30, seed=0), 2, 1.0),
    "atlas50": (lambda: problems.config3_atlas(50, seed=0), 2, 1.0),
    "quad30": (lambda: problems.config4_quadruped(30, seed=0), 15, 1.0),
}
out = {}
for name in which:
    make, k, hard = CASES[name]
    t0 = time.time(); wl = make(); t_gen = time.time() - t0
    base = wl.base_problem()
    n, m = base.n, base.m
    t0 = time.time(); gpu = S.Solver(base.H, base.g, base.G, base.c, base.d); t_setup = time.time() - t0
    x0 = wl.x0(hard)
    A, B, K, nu = wl.sys.A, wl.sys.B, wl.tmpl.K, wl.sys.nu
    u_lo, u_hi = wl.limits.u_lo, wl.limits.u_hi
    # initial solve to tolerance, then the receding-horizon loop
    q = wl.problem_at(x0)
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start()
    r0 = gpu.solve()
    steps = 300
    x = x0.copy(); wall, ker, ys, cwall = [], [], [], []
    for t in range(steps):
        q = wl.problem_at(x)                      # host instantiate (mpc.cpp:260-270)
        t1 = time.perf_counter()
        rep = gpu.mpc_step(q.g, q.c, q.d, k)
        wall.append((time.perf_counter() - t1) * 1e6); ker.append(rep.kernel_us); cwall.append(rep.wall_ms * 1e3)
        if t < 20:
            ys.append(rep.solution.y.copy())
        u = np.clip(-K @ x + rep.solution.y[:nu], u_lo, u_hi)
        x = A @ x + B @ u
    rec = {"n": n, "m": m, "D": n + 2 * m, "k": k, "launch": gpu.launch_info(), "gen_s": t_gen, "gpu_setup_s": t_setup,
           "initial_solve": {"iterations": r0.solution.iterations, "kernel_us": r0.kernel_us, "status": r0.solution.status,
                             "rho_trace": r0.solution.rho_trace},
           "gpu_step_wall_us_p50": statistics.median(wall[20:]), "gpu_step_kernel_us_p50": statistics.median(ker[20:]),
           "gpu_step_cabi_wall_us_p50": statistics.median(cwall[20:]),
           "gpu_hz": 1e6 / statistics.median(wall[20:]), "final_state_norm": float(np.abs(x).max())}
    # CPU oracle on the same loop (first 20 steps), best-effort build for setup speed, ref build timed
    if n <= 900:
        t0 = time.time(); cpu = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d), variant="ref"); rec["cpu_setup_s"] = time.time() - t0
        q = wl.problem_at(x0)
        cpu.update_vectors(q.g, q.c, q.d); cpu.cold_start()
        c0 = cpu.solve()
        rec["initial_solve"]["cpu_iterations"] = c0.solution.iterations
        rec["initial_solve"]["cpu_ms"] = c0.wall_ms
        rec["initial_solve"]["trace_equal"] = c0.solution.rho_trace == r0.solution.rho_trace
        x = x0.copy(); cw = []; worst = 0.0
        for t in range(20):
            q = wl.problem_at(x)
            t1 = time.perf_counter()
            cpu.update_vectors(q.g, q.c, q.d); cpu.refresh_z(); rc = cpu.fixed_iters(k)
            cw.append((time.perf_counter() - t1) * 1e6)
            worst = max(worst, float(np.abs(rc.solution.y - ys[t]).max() / max(1.0, np.abs(rc.solution.y).max())))
            u = np.clip(-K @ x + rc.solution.y[:nu], u_lo, u_hi)
            x = A @ x + B @ u
        rec["cpu_step_us_p50"] = statistics.median(cw)
        rec["cpu_hz"] = 1e6 / statistics.median(cw)
        rec["speedup"] = rec["cpu_step_us_p50"] / rec["gpu_step_wall_us_p50"]
        rec["max_rel_diff_y_first20"] = worst
    out[name] = rec
    print(name, json.dumps(rec), flush=True)
    gpu.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"{TAG}_mpc_steps.json"), "w"), indent=1)
