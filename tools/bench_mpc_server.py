"""Scratch (GPU box): control-step latency of the closed loop (bench.cpp:157-185), launch per step
vs the resident server, through the C ABI call cqp_mpc_step_x0 (x0 in, u0 out).
  python tools/bench_mpc_server.py config1,atlas30,quad30"""
import json, os, statistics, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads import problems  # noqa: E402
from paper_2311_18056_b200 import solver as S  # noqa: E402

CASES = {
    "config1": (lambda: problems.config1(seed=0), 1),
    "config1_k2": (lambda: problems.config1(seed=0), 2),
    "nu30": (lambda: problems.config2(30, seed=0), 2),
    "nu50": (lambda: problems.config2(50, seed=0), 2),
    "atlas30": (lambda: problems.config3_atlas(30, seed=0), 2),
    "atlas50": (lambda: problems.config3_atlas(50, seed=0), 2),
    "quad30": (lambda: problems.config4_quadruped(30, seed=0), 15),
}
which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["config1", "atlas30"]
steps = int(os.environ.get("STEPS", "400"))
out = {}
for name in which:
    make, k = CASES[name]
    wl = make(); base = wl.base_problem()
    gpu = S.Solver(base.H, base.g, base.G, base.c, base.d)
    gpu.set_mpc_template(wl.tmpl, wl.limits)
    A, B = wl.sys.A, wl.sys.B
    rec = {"n": base.n, "m": base.m, "D": base.n + 2 * base.m, "k": k, "launch": gpu.launch_info()}
    finals = {}
    for mode in ("launch_per_step", "server"):
        q = wl.problem_at(wl.x0(1.0))
        gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.solve()
        if mode == "server":
            gpu.mpc_server_start(k)
        x = np.ascontiguousarray(wl.x0(1.0)); u0 = np.zeros(wl.sys.nu)
        wall, cwall, dev = [], [], []
        for t in range(steps):
            t1 = time.perf_counter()
            gpu.mpc_step_x0_fast(x, k, u0)
            wall.append((time.perf_counter() - t1) * 1e6)
            if mode == "server":
                w, d = gpu.mpc_server_last_timing(); cwall.append(w); dev.append(d)
            x = np.ascontiguousarray(A @ x + B @ u0)
        _, rep = gpu.mpc_step_x0(x, k)          # one step with the report: device-side duration
        if mode == "server":
            gpu.mpc_server_stop()
        finals[mode] = (x.copy(), u0.copy())
        w = sorted(wall[20:])
        rec[mode] = {"wall_us_p50": statistics.median(w), "wall_us_p90": w[int(0.9 * len(w))], "wall_us_min": w[0],
                     "device_step_us_with_report": rep.kernel_us, "hz": 1e6 / statistics.median(w)}
        if cwall:
            rec[mode]["cabi_wall_us_p50"] = statistics.median(cwall[20:])
            rec[mode]["device_step_us_p50"] = statistics.median(dev[20:])
    rec["bit_identical_closed_loop"] = bool(np.array_equal(finals["launch_per_step"][0], finals["server"][0]) and
                                            np.array_equal(finals["launch_per_step"][1], finals["server"][1]))
    rec["speedup"] = rec["launch_per_step"]["wall_us_p50"] / rec["server"]["wall_us_p50"]
    out[name] = rec
    print(name, json.dumps(rec), flush=True)
    gpu.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "mpc_server_bench.json"), "w") as f:
    json.dump(out, f, indent=1)
