"""Scratch: staged sanity runs of the persistent kernel (each stage under its own timeout)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_18056_b200 import problems, solver as S

stage = sys.argv[1]
import faulthandler
faulthandler.dump_traceback_later(240, exit=True)
if stage == "1d_fixed1":
    print("creating", flush=True)
    s = S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])
    print("created", flush=True)
    r = s.fixed_iters(1); print(stage, r.solution.iterations, s.state, r.kernel_us)
elif stage == "1d_fixed3":
    print("creating", flush=True)
    s = S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])
    print("created", flush=True)
    r = s.fixed_iters(3); print(stage, r.solution.iterations, s.state, r.kernel_us)
elif stage == "1d_fixed30":
    s = S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])
    r = s.fixed_iters(30); print(stage, r.solution.iterations, s.state, r.kernel_us, r.residual_history)
elif stage == "1d_solve":
    s = S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])
    r = s.solve(); print(stage, r.solution.iterations, r.solution.y, r.solution.lam, r.kernel_us)
elif stage.startswith("mpc"):
    nu = int(stage[3:])
    wl = problems.config2(nu, 0); base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d)
    q = wl.problem_at(wl.x0(10.0)); s.update_vectors(q.g, q.c, q.d)
    print(s.launch_info(), flush=True)
    for k in (1, 2, 3, 4, 5, 8, 26, 100, 1000):
        s.cold_start(); r = s.fixed_iters(k); print(stage, k, r.solution.iterations, r.kernel_us, r.solution.r_prim, flush=True)
    s.cold_start(); r = s.solve(); print(stage, "solve", r.solution.iterations, r.solution.rho_trace, r.kernel_us)
elif stage.startswith("perf"):
    nu = int(stage[4:])
    wl = problems.config2(nu, 0); base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    q = wl.problem_at(wl.x0(10.0)); s.update_vectors(q.g, q.c, q.d)
    res = {}
    for k in (1000, 3000):
        ts = []
        for _ in range(3):
            s.cold_start(); r = s.fixed_iters(k); ts.append(r.kernel_us)
        res[k] = sorted(ts)[1]
    print(stage, "fence_mode", os.environ.get("CQP_FENCE_MODE", "0"), "us/iter", (res[3000] - res[1000]) / 2000.0, res, flush=True)
elif stage.startswith("watch"):
    import threading, time, ctypes as C
    k = int(stage[5:])
    print("creating", flush=True)
    s = S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])
    print("created", s.launch_info(), flush=True)
    def watch():
        time.sleep(4)
        w = (C.c_int * 256)()
        s._L.cqp_debug_words(s._h, w)
        print("dbg", list(w)[:8], "progress(cta x [compute,publisher,loader,epilogue])", [list(w)[16 + 4 * c:20 + 4 * c] for c in range(3)], flush=True)
        os._exit(3)
    threading.Thread(target=watch, daemon=True).start()
    r = s.fixed_iters(k); print(stage, r.solution.iterations, s.state, r.kernel_us, flush=True)
    os._exit(0)
elif stage.startswith("fixed"):
    import ctypes as C
    wl = problems.config1(0); base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d)
    q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
    s.cold_start(); s.solve()
    for _ in range(3):
        r = s.mpc_step(q.g, q.c, q.d, int(stage[5:]))
    w = (C.c_int * 256)()
    s._L.cqp_debug_words(s._h, w)
    al = np.frombuffer(bytes(w), dtype=np.int64)[32 + 48:32 + 64]
    names = ["entry", "vectors+rows cached", "cluster sync 1", "refresh_z done", "layer + W regs", "v0 + cluster sync", "loop done", "final v arrived", "residual pass", "outputs written", "exit sync"]
    print(s.launch_info(), "kernel_us", r.kernel_us)
    print("  ".join(f"{names[i]}@{int(al[i] - al[0])}" for i in range(11) if al[i]))
elif stage.startswith("chunks"):
    import ctypes as C
    wl = problems.config3_atlas(30, 0) if stage[6:] == "atlas" else problems.config4_quadruped(30, 0)
    base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
    for _ in range(2):
        s.cold_start(); r = s.fixed_iters(300)
    w = (C.c_int * 256)()
    s._L.cqp_debug_words(s._h, w)
    al = np.frombuffer(bytes(w), dtype=np.int64)
    ll = al[32:80]; ll = ll[ll != 0]
    pl = al[80:128]; pl = pl[pl != 0]
    print(s.launch_info(), "consumer chunk-ready stamps (cycles since the first):", [int(x - ll[0]) for x in ll])
    print("producer issue stamps (same origin):", [int(x - ll[0]) for x in pl])
    print("us/iter", r.kernel_us / 300)
elif stage.startswith("trace"):
    import ctypes as C
    if stage[5:] == "quad":
        wl = problems.config4_quadruped(30, 0)
    elif stage[5:] == "atlas":
        wl = problems.config3_atlas(30, 0)
    else:
        wl = problems.config2(int(stage[5:]), 0)
    base = wl.base_problem()
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=100000))
    q = wl.problem_at(wl.x0(1.0)); s.update_vectors(q.g, q.c, q.d)
    print(s.launch_info())
    for _ in range(2):
        s.cold_start(); r = s.fixed_iters(1000)
    w = (C.c_int * 256)()
    s._L.cqp_debug_words(s._h, w)
    ll = np.frombuffer(bytes(w), dtype=np.int64)[32:]
    names = {0: "c:start", 1: "c:x ready", 3: "c:fma done", 2: "c:dots done", 10: "c15:x ready", 11: "c15:done", 4: "p:start|check begin", 5: "p:partials ready|pass done", 6: "p:published", 7: "p:done|check end", 8: "l:go seen", 9: "l:fetched"}
    t00 = ll[0]
    for it in range(4):
        row = ll[it * 16:(it + 1) * 16]
        ev = sorted((int(row[k] - t00), names[k]) for k in names if row[k] != 0)
        print("iter", 100 + it, "  ".join(f"{n}@{t}" for t, n in ev))
    print("us/iter", r.kernel_us / 1000)
