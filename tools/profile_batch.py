"""Scratch (GPU box): one batched solve (B columns, nu=50) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_18056_b200 import problems, solver as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
wl = problems.config2(50, 0); base = wl.base_problem()
g, c, d, _ = problems.batch_instances(wl, B)
s = S.Solver(base.H, base.g, base.G, base.c, base.d)
b = S.BatchSolver(s, B)
out = b.solve(g, c, d)
print("B", B, "compute_ms", out["compute_ms"], "gemm_ms", out["gemm_ms"], "TF", out["gemm_flops"] / out["gemm_ms"] / 1e9, "launches", out["launches"])
import numpy as np
print("rounds", out["rounds"])
print("active", out["round_active"].tolist())
print("ms", [round(float(x), 2) for x in out["round_ms"]])
print("iters hist", np.bincount(out["iterations"] // 25).tolist(), "final idx", np.bincount(out["final_index"]).tolist())
