"""Scratch (GPU box): A/B of the batched path.  Runs one batched solve per environment setting in
its own process (the knobs are read at handle creation), prints the timing profile of each and
compares the results bit for bit against the first setting.

  python tools/ab_batch.py 4096 "CQP_BATCH_LEGACY=1" "" "CQP_BATCH_LANES=1"
"""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    from workloads import problems
    from paper_2311_18056_b200 import solver as S
    B, nu, out_path, reps = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
    wl = problems.config2(nu, 0); base = wl.base_problem()
    g, c, d, _ = problems.batch_instances(wl, B)
    mi = int(os.environ.get("AB_MAX_ITERS", "4000"))
    s = S.Solver(base.H, base.g, base.G, base.c, base.d, S.SolverSettings(max_iters=mi, check_interval=int(os.environ.get("AB_CHECK", "25"))))
    b = S.BatchSolver(s, B)
    best = None
    for _ in range(reps):
        out = b.solve(g, c, d)
        if best is None or out["compute_ms"] < best["compute_ms"]:
            best = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in out.items()}
    tr = b.traces()
    np.savez(out_path, y=best["y"], lam=best["lam"], z=best["z"], iterations=best["iterations"], status=best["status"],
             final_index=best["final_index"], trace_len=np.array([len(t) for t in tr]))
    if os.environ.get("AB_BRIEF"):
        print(json.dumps({"compute_ms": round(best["compute_ms"], 3), "TF": round(best["gemm_flops"] / best["gemm_ms"] / 1e9, 2),
                          "rounds": int(best["rounds"]), "launches": int(best["launches"])}))
        sys.exit(0)
    print(json.dumps({"compute_ms": best["compute_ms"], "gemm_ms": best["gemm_ms"],
                      "TF": best["gemm_flops"] / best["gemm_ms"] / 1e9, "launches": int(best["launches"]),
                      "rounds": int(best["rounds"]), "active": best["round_active"].tolist(),
                      "round_ms": [round(float(x), 3) for x in best["round_ms"]]}))
    sys.exit(0)

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
settings = sys.argv[2:] or ["CQP_BATCH_LEGACY=1", ""]
nu = int(os.environ.get("AB_NU", "50"))
reps = int(os.environ.get("AB_REPS", "3"))
ref = None
for i, setting in enumerate(settings):
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=", 1)
        env[k] = v
    path = f"/tmp/ab_batch_{i}.npz"
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", str(B), str(nu), path, str(reps)], env=env,
                       capture_output=True, text=True, timeout=1500)
    print(f"== [{setting or 'default'}] rc={r.returncode}")
    print(r.stdout.strip()[-3000:])
    if "[verify]" in r.stderr:
        print("\n".join(l for l in r.stderr.splitlines() if "[verify]" in l)[:6000])
    if r.returncode != 0:
        print(r.stderr[-3000:])
        continue
    out = dict(np.load(path))
    if ref is None:
        ref = out
        continue
    same_counts = bool((out["iterations"] == ref["iterations"]).all() and (out["status"] == ref["status"]).all()
                       and (out["final_index"] == ref["final_index"]).all() and (out["trace_len"] == ref["trace_len"]).all())
    dy = float(np.abs(out["y"] - ref["y"]).max()); dl = float(np.abs(out["lam"] - ref["lam"]).max())
    print(f"   vs first: counts/status/index/trace_len equal={same_counts} max|dy|={dy:.3e} max|dlam|={dl:.3e} "
          f"bit_identical={bool((out['y'] == ref['y']).all() and (out['lam'] == ref['lam']).all() and (out['z'] == ref['z']).all())}")
