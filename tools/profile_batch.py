"""Scratch (GPU box): one batched solve (B columns, nu=50) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import problems
from paper_2311_18056_b200 import solver as S
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
wl = problems.config2(50, 0); base = wl.base_problem()
g, c, d, _ = problems.batch_instances(wl, B)
if len(sys.argv) > 2 and sys.argv[2] == "oracle_layers":
    # offline stage on the CPU oracle: the only dmma_gemm launches left are the batch's own
    from oracle import oracle as O
    oc = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d), variant="v3").cache
    layers = {"W": [oc.W(k) for k in range(oc.L)], "D": [oc.D(k) for k in range(oc.L)],
              "GD": [oc.GD(k) for k in range(oc.L)], "grid": oc.grid, "initial_index": oc.initial_index,
              "Gs": oc.Gs, "E": oc.E, "F": oc.F, "cost_scale": oc.cost_scale}
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, layers=layers)
else:
    s = S.Solver(base.H, base.g, base.G, base.c, base.d)
b = S.BatchSolver(s, B)
out = b.solve(g, c, d)
print("B", B, "compute_ms", out["compute_ms"], "gemm_ms", out["gemm_ms"], "TF", out["gemm_flops"] / out["gemm_ms"] / 1e9, "launches", out["launches"])
import numpy as np
print("rounds", out["rounds"])
print("active", out["round_active"].tolist())
print("ms", [round(float(x), 2) for x in out["round_ms"]])
print("iters hist", np.bincount(out["iterations"] // 25).tolist(), "final idx", np.bincount(out["final_index"]).tolist())
