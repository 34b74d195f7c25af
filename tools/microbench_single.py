"""Scratch micro-benchmark (GPU box): per-iteration time of the persistent single-QP kernel for
several sizes, and the FP64 matmul rate cuBLAS reaches (denominator of the batched roofline)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads import problems  # noqa: E402
from paper_2311_18056_b200 import solver as S  # noqa: E402

out = {}
for nu in (10, 30, 50):
    wl = problems.config2(nu, 0)
    base = wl.base_problem()
    t = time.time()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    t_setup = time.time() - t
    q = wl.problem_at(wl.x0(10.0))
    s.update_vectors(q.g, q.c, q.d)
    res = {}
    for k in (1, 2, 25, 1000, 4000):
        times = []
        for _ in range(5):
            s.cold_start()
            r = s.fixed_iters(k)
            times.append((r.kernel_us, r.wall_ms * 1e3))
        times.sort()
        res[k] = {"kernel_us": times[2][0], "wall_us": sorted(t[1] for t in times)[2]}
    s.cold_start()
    r = s.solve()
    D = 3 * base.n
    per_iter = (res[4000]["kernel_us"] - res[1000]["kernel_us"]) / 3000.0
    out[f"nu{nu}"] = {"D": D, "setup_s": t_setup, "launch": s.launch_info(), "fixed": res,
                      "us_per_iter": per_iter, "smem_GBs": 8.0 * D * D / per_iter * 1e-3,
                      "solve_iters": r.solution.iterations, "solve_kernel_us": r.kernel_us,
                      "solve_wall_us": r.wall_ms * 1e3, "trace": r.solution.rho_trace}
    print(nu, json.dumps(out[f"nu{nu}"]), flush=True)

try:
    import torch
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        (a @ b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["dgemm_fp64_tflops_8192"] = 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    a = torch.randn(1536, 1536, dtype=torch.float64, device="cuda")
    b = torch.randn(1536, 4096, dtype=torch.float64, device="cuda")
    for _ in range(2):
        (a @ b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["dgemm_fp64_tflops_1536x1536x4096"] = 2 * 1536 * 1536 * 4096 / (best * 1e-3) / 1e12
    print("dgemm", out["dgemm_fp64_tflops_8192"], out["dgemm_fp64_tflops_1536x1536x4096"])
except Exception as e:  # noqa: BLE001
    out["dgemm_error"] = repr(e)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "microbench_single.json"), "w"), indent=1)
