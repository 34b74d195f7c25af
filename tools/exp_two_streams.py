"""Scratch (GPU box): does splitting the 4096-column batch into K independent sub-batches on K streams
(one host thread each) hide the per-launch wave tails?  Prints ms per full solve for K = 1, 2, 3."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_18056_b200 import problems, solver as S
B = 4096
wl = problems.config2(50, 0); base = wl.base_problem()
g, c, d, _ = problems.batch_instances(wl, B)
s = S.Solver(base.H, base.g, base.G, base.c, base.d)
for K in (1, 2, 3, 4):
    per = (B + K - 1) // K
    parts = [(i * per, min(B, (i + 1) * per)) for i in range(K)]
    bs = [S.BatchSolver(s, hi - lo) for lo, hi in parts]
    ins = [(np.ascontiguousarray(g[:, lo:hi]), np.ascontiguousarray(c[:, lo:hi]), np.ascontiguousarray(d[:, lo:hi])) for lo, hi in parts]
    outs = [None] * K
    def work(i):
        outs[i] = bs[i].solve(*ins[i])
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        ts = [threading.Thread(target=work, args=(i,)) for i in range(K)]
        [t.start() for t in ts]; [t.join() for t in ts]
        best = min(best, time.perf_counter() - t0)
    its = np.concatenate([o["iterations"] for o in outs])
    print("K", K, "wall_ms", round(best * 1e3, 1), "sum compute_ms", [round(o["compute_ms"], 1) for o in outs], "mean iters", its.mean())
    for b in bs:
        b.close()
