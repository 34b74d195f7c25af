"""Scratch (GPU box): timeline of CTA 0's warp roles in the L2/HBM tier, iterations 100..103, from a
-DCQP_TRACE build (CQP_B200_LIB=build/trace/libcqp_b200.so).  Times in us relative to the first stamp."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from workloads import problems
from paper_2311_18056_b200 import solver as S, _lib
NAMES = {0: "cmp:v_i landed", 1: "cmp:v landed", 10: "cmp15:v landed", 2: "cmp:done", 11: "cmp15:done", 4: "pub:start",
         5: "pub:full", 6: "pub:published", 7: "pub:rearmed", 8: "ldr:go", 9: "ldr:fetched",
         3: "cmp:dot done", 12: "cmp:row ready", 13: "cmp:rearm ok"}
which = sys.argv[1] if len(sys.argv) > 1 else "quad"
if which == "quad":
    wl = problems.config4_quadruped(30, 0)
elif which == "atlas":
    wl = problems.config3_atlas(30, 0)
else:
    wl = problems.config2(int(which[2:]), 0)   # "nu30": the resident tier at D = 900
base = wl.base_problem()
s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
for _ in range(2):
    s.cold_start(); r = s.fixed_iters(120)
if len(sys.argv) > 2 and sys.argv[2] == "step":
    # prologue / epilogue stamps (slots 48..54, -DCQP_TRACE build) of one fused MPC step of k iterations
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    for _ in range(3):
        r = s.mpc_step(q.g, q.c, q.d, k)
    words = (C.c_int * 256)()
    _lib.load().cqp_debug_words(s._h, words)
    st = np.frombuffer(bytes(words), dtype=np.int64)[32 + 48:32 + 48 + 7]
    names = ["entry", "bounds+refresh_z", "bias rows", "v0 loaded", "iterations", "final residual pass", "results written"]
    print(which, "k", k, "kernel_us", r.kernel_us, " ".join(f"{nm}@{(int(t) - int(st[0])) / 1965.0:.2f}" for nm, t in zip(names, st)))
    sys.exit(0)
print(which, s.launch_info(), "kernel_us", r.kernel_us, "us/iter", r.kernel_us / 120)
if len(sys.argv) > 2 and sys.argv[2] == "check":
    # stamps of the third residual pass of the launch (iteration 75), thread 0 of CTA 0
    words = (C.c_int * 256)()
    _lib.load().cqp_debug_words(s._h, words)
    st = np.frombuffer(bytes(words), dtype=np.int64)[32 + 64:32 + 64 + 8]
    names = ["entered", "CTA assembled", "unscaled", "row dots", "CTA maxima", "grid barrier", "all-CTA maxima", "decision"]
    print("check pass:", " ".join(f"{nm}@{(int(t) - int(st[0])) / 1965.0:.2f}" for nm, t in zip(names, st)))
    sys.exit(0)
words = (C.c_int * 256)()
_lib.load().cqp_debug_words(s._h, words)
st = np.frombuffer(bytes(words), dtype=np.int64)[32:32 + 64].reshape(4, 16)
t0 = st[0][0]
two = len(sys.argv) > 2 and sys.argv[2] == "two"   # -DCQP_TRACE_TWO build: rows = (CTA 0: it, it+1), (last CTA: it, it+1), ns
for it in range(4):
    ev = sorted((int(st[it][k]), NAMES[k]) for k in NAMES if st[it][k] > 0)
    label = (("cta0", "ctaLast")[it // 2] + f" iter {100 + it % 2}") if two else f"iter {100 + it}"
    print(label, " ".join(f"{n}@{(t - t0) / (1000.0 if two else 1965.0):.2f}" for t, n in ev))
