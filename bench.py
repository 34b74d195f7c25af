#!/usr/bin/env python
"""Benchmark of the ReLU-QP solve path on B200 (contract: see the task statement / DESIGN.md 6).

  python bench.py --gpus N --steps K --warmup W            # GPU arm (this repo's CUDA path)
  python bench.py --impl reference --gpus N --steps K ...  # reference arm: the CPU implementation

Headline workload (BASELINE.json configs[4]): a batch of 4096 random linear-MPC instances
(nu = 50, nx = 100, horizon 10 -> n = m = 500, D = 1500) that share one W ladder and differ in
x0 (hence g, c, d); every instance is a cold-start `solve()` to 1e-6.  One "step" = one solve of
the whole batch.  With N > 1 the 4096 columns are SHARDED over the ranks (strong scaling, as the
config says: "sharded across 1/2/4/8 B200"): rank r solves columns shard_range(4096, N, r), no
inter-GPU traffic during the solve, the result columns are gathered to rank 0 with NCCL inside
the e2e region.  A weak-scaling run (4096 columns per rank) is reported under "weak_scaling".
Run without torchrun, `--gpus N` spawns the N ranks itself.

  value  = QPs/s with the batch inputs already resident in HBM (CUDA events around the solve)
  e2e    = QPs/s through the C-ABI call cqp_batch_solve with HOST buffers: host->device copy of
           (g, c, d), the solve, device->host copy of (y, z, lambda, status, ...) all inside the
           timed region
  roofline = the iteration kernel (round_kernel: one persistent launch per check round, TMA-staged
           operands, FP64 DMMA): EXECUTED flop per active column per iteration
           (2 ((n+m) D + m n): the zero blocks (3,2), (3,3) of W are skipped, so less than the
           dense 2 D^2) / CUDA-event time of those launches, against the FP64 GEMM rate cuBLAS
           reaches on this GPU measured in the same run (MEASURED_PEAKS.json has no FP64 entry)
  cpu_baseline = the CPU oracle (a restatement of the reference solver, compiled like the
           reference: -O3 -DNDEBUG, no -march) on a bounded sample of the same instances
  single_qp = configs[1]: single-QP solve time (p50 us) per size through cqp_solve, next to the
           CPU oracle, with the achieved shared-memory streaming rate 8 D^2 bytes / iteration
  mpc_steps = configs[0], [2], [3]: receding-horizon control step (fused cqp_mpc_step) wall/kernel
           p50 and the W streaming rate next to the HBM peak
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NU, NX, HORIZON, BATCH = 50, 100, 10, 4096
WORKLOAD = f"batched {BATCH} random linear-MPC QPs, nu={NU} nx={NX} N={HORIZON} (n=m=500, D=1500), shared W, x0 scale log-uniform in [0.3,10]x LQR push, sharded by column over the GPUs"
# identical in both arms (the driver compares the arms' `config`); run-specific facts go elsewhere
CONFIG = {"workload": WORKLOAD, "batch": BATCH, "nu": NU, "nx": NX, "horizon": HORIZON, "n": 500, "m": 500, "D": 1500,
          "check_interval": 25, "eps": 1e-6, "max_iters": 4000, "start": "cold", "seed": 0,
          "l2_policy": "working set per step (S ping-pong 98 MB + bias/bounds 66 MB + W ladder) exceeds the 126 MB L2; inputs re-uploaded every step"}
METRIC = "batched QP solves per second (cold-start solve to 1e-6, FP64)"


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(path)), "measured (MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
        sm, mx, reasons = [], 0.0, set()
        for r in self.rows:
            try:
                sm.append(float(r[0])); mx = max(mx, float(r[1]))
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(first: int = 0):
    from workloads import problems
    wl = problems.config2(NU, seed=0)
    g, c, d, _ = problems.batch_instances(wl, BATCH, first=first)
    return wl, g, c, d


_ORACLE_POOL = {}


def oracle_solve_columns(wl, g, c, d, cols, threads: int, variant: str = "ref"):
    """CPU path: one oracle Solver per thread (the reference has no threading of its own; a
    caller parallelises over instances), returns (seconds, iterations list).  The per-thread
    solvers (offline stage, untimed) are built once and reused."""
    from oracle import oracle as O
    key = (id(wl), threads, variant)
    if key not in _ORACLE_POOL:
        base = wl.base_problem()
        p = O.QProblem(base.H, base.g, base.G, base.c, base.d)
        solvers = [None] * threads

        def setup(i):
            solvers[i] = O.Solver(p, variant=variant)
        ts = [threading.Thread(target=setup, args=(i,)) for i in range(threads)]
        [t.start() for t in ts]; [t.join() for t in ts]
        _ORACLE_POOL[key] = solvers
    solvers = _ORACLE_POOL[key]
    iters = [0] * len(cols)
    chunks = [list(range(i, len(cols), threads)) for i in range(threads)]

    def work(i):
        s = solvers[i]
        for k in chunks[i]:
            j = cols[k]
            s.update_vectors(g[:, j], c[:, j], d[:, j]); s.cold_start()
            iters[k] = s.solve().solution.iterations
    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    [t.start() for t in ts]; [t.join() for t in ts]
    return time.perf_counter() - t0, iters


def reference_arm(args, rank: int, world: int):
    """The reference's own CPU implementation of the path (oracle/_ref cannot be built: Eigen is
    absent, so the restated port is timed), all host threads, a bounded sample of the workload per
    step: 4 instances per core per step (one oracle Solver per thread), i.e. 80 per core over the
    driver's 20 steps."""
    if rank != 0:
        return
    wl, g, c, d = make_workload(0)
    cores = os.cpu_count() or 1
    sample = 4 * cores
    cols = list(range(sample))
    for _ in range(min(args.warmup, 1)):
        oracle_solve_columns(wl, g, c, d, cols[:cores], cores)
    per_step = []
    for _ in range(args.steps):
        sec, _ = oracle_solve_columns(wl, g, c, d, cols, cores)
        per_step.append(sec)
    qps = sample * len(per_step) / sum(per_step)
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "QP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(per_step) / len(per_step),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": CONFIG,
            "cpu_baseline": {"value": qps, "unit": "QP/s", "cores": cores, "kind": "port",
                             "sample": f"{sample} of the {BATCH} instances per step ({sample // cores} per core) x {args.steps} steps, one oracle Solver per thread, -O3 -DNDEBUG build (the reference's flags)"},
            "e2e": {"value": qps, "unit": "QP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def read_stream_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "stream_traffic.json"))).get("dram_bytes_per_iteration")
    except Exception:  # noqa: BLE001
        return None


def measure_dgemm_peak():
    import torch
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def measure_hbm_copy_peak():
    """STREAM-style device copy (read + write bytes / time), the HBM denominator when the driver's
    MEASURED_PEAKS.json is absent: 2 GiB buffers, best of 5."""
    import torch
    n = 1 << 28  # doubles: 2 GiB
    a = torch.empty(n, dtype=torch.float64, device="cuda").normal_()
    b = torch.empty_like(a)
    for _ in range(2):
        b.copy_(a)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8 * n / (best * 1e-3) / 1e9


def measure_read_peaks(device: int):
    """(HBM read GB/s, L2 read GB/s) with the library's own read kernel (cqp_measure_read_bandwidth):
    a 2 GiB buffer read 3 times, and a 48 MB buffer (fits the 126 MB L2) read 60 times."""
    import ctypes as C
    from paper_2311_18056_b200 import _lib
    L = _lib.load()
    out = []
    for nbytes, passes in ((2 << 30, 3), (48 << 20, 60)):
        v = C.c_double()
        rc = L.cqp_measure_read_bandwidth(device, nbytes, passes, C.byref(v))
        out.append(v.value if rc == 0 else None)
    return tuple(out)


def single_qp_sweep(S, problems, repeats: int = 21, seeds=tuple(range(10)), nus=tuple(range(10, 51, 4)),
                    cpu_seeds=(0, 1, 2)):
    """configs[0..1], protocol of SURVEY 8(d): for every nu in {10, 14, ..., 50} (tools/main.cpp:243,
    nx = 2 nu, N = 10) and every seed 0..9, `repeats` timed cold-start solves from the hard start
    (x0 = 10 x the LQR push scale, bench.cpp:35); p50 over all seeds x repeats of the kernel-only
    (CUDA events) and through-the-C-ABI wall time (the reference's wall_ms region).  Beside it the
    CPU oracle on ONE core (the reference has no threading): the reference-flags build on seeds
    `cpu_seeds` and the -march=x86-64-v3 "best-effort CPU" build on seed 0, same inputs, iteration
    counts and rho traces compared with the GPU's."""
    import concurrent.futures as cf
    from oracle import oracle as O
    out = []
    for nu in nus:
        ker, wall, iters, bytes_it = [], [], [], 0.0
        gpu_by_seed, info = {}, None
        for seed in seeds:
            wl = problems.config2(nu, seed=seed)
            base = wl.base_problem()
            q = wl.problem_at(wl.x0(10.0))
            gs = S.Solver(base.H, base.g, base.G, base.c, base.d)        # offline stage on the device
            gs.update_vectors(q.g, q.c, q.d)
            rep = None
            k_s, w_s = [], []
            for r in range(repeats + 2):
                gs.cold_start()
                rep = gs.solve()
                if r >= 2:
                    k_s.append(rep.kernel_us); w_s.append(rep.wall_ms * 1e3)
            ker += k_s; wall += w_s
            iters.append(rep.solution.iterations)
            gpu_by_seed[seed] = (rep.solution.iterations, rep.solution.rho_trace, statistics.median(w_s), wl, base, q)
            info = gs.launch_info()
            bytes_it = info["w_bytes_per_iteration"]
            gs.close()

        def cpu_setup(job):
            seed, variant = job
            _, _, _, wl, base, q = gpu_by_seed[seed]
            cpu = O.Solver(O.QProblem(base.H, base.g, base.G, base.c, base.d), variant=variant)
            cpu.update_vectors(q.g, q.c, q.d)
            return cpu
        jobs = [(sd, "ref") for sd in cpu_seeds if sd in gpu_by_seed] + [(min(gpu_by_seed), "v3")]
        with cf.ThreadPoolExecutor(min(len(jobs), os.cpu_count() or 1)) as pool:   # untimed setups in parallel
            cpus = list(pool.map(cpu_setup, jobs))
        cpu_ms = {"ref": [], "v3": []}
        gpu_wall_same = []
        match = True
        for (seed, variant), cpu in zip(jobs, cpus):                                # timed solves: one at a time
            ts = []
            for _ in range(3):
                cpu.cold_start()
                ro = cpu.solve()
                ts.append(ro.wall_ms)
            cpu_ms[variant].append(statistics.median(ts))
            if variant == "ref":
                gpu_wall_same.append(gpu_by_seed[seed][2])
                match = match and ro.solution.iterations == gpu_by_seed[seed][0] and ro.solution.rho_trace == gpu_by_seed[seed][1]
        D = 30 * nu
        k50, w50 = statistics.median(ker), statistics.median(wall)
        c_ref, c_v3 = statistics.median(cpu_ms["ref"]) * 1e3, statistics.median(cpu_ms["v3"]) * 1e3
        us_it = sum(ker) / (repeats * sum(iters))
        out.append({"nu": nu, "D": D, "seeds": len(seeds), "repeats": repeats,
                    "iterations_by_seed": iters, "gpu_kernel_us_p50": k50, "gpu_wall_us_p50": w50,
                    "us_per_iteration": us_it, "smem_stream_GBs": bytes_it / (us_it * 1e-6) / 1e9,
                    "cpu_1core_us_p50_ref_flags": c_ref, "cpu_1core_us_p50_march_v3": c_v3, "cpu_seeds": list(cpu_seeds),
                    "speedup_wall_vs_cpu_ref_same_seeds": c_ref / statistics.median(gpu_wall_same),
                    "iterations_and_rho_trace_equal_cpu": bool(match), "launch": info})
    return out


def mpc_step_section(S, problems, peaks):
    """configs[0], [2], [3]: receding-horizon step {instantiate, update_vectors, refresh_z,
    fixed_iters(k), control extraction} (bench.cpp:157-185) through cqp_mpc_step_x0 (template on the
    device: upload x0, one launch, download u0): host wall p50 per step through the Python wrapper
    and through the C ABI alone, kernel p50, and the W streaming rate 8 D^2 k / kernel time
    next to the HBM peak (the robot-sized W levels, 54 and 133 MB, are L2/HBM streamed)."""
    out = []
    for name, make, k in (("config1 nu=10 N=10", lambda: problems.config1(seed=0), 1),
                          ("atlas-sized nx=58 nu=29 N=30", lambda: problems.config3_atlas(30, seed=0), 2),
                          ("atlas-sized nx=58 nu=29 N=40", lambda: problems.config3_atlas(40, seed=0), 2),
                          ("atlas-sized nx=58 nu=29 N=50", lambda: problems.config3_atlas(50, seed=0), 2),
                          ("quadruped-sized nx=52 nu=32 N=30", lambda: problems.config4_quadruped(30, seed=0), 15)):
        wl = make()
        base = wl.base_problem()
        gs = S.Solver(base.H, base.g, base.G, base.c, base.d)
        x = wl.x0(1.0)
        q = wl.problem_at(x)
        gs.update_vectors(q.g, q.c, q.d); gs.cold_start()
        r0 = gs.solve()                                   # initial solve to tolerance
        A, B, K, nu = wl.sys.A, wl.sys.B, wl.tmpl.K, wl.sys.nu
        # (a) template on the device: a step uploads x0 and downloads u0 (cqp_mpc_step_x0)
        gs.set_mpc_template(wl.tmpl, wl.limits)
        wall, ker, cabi = [], [], []
        for t in range(120):
            t1 = time.perf_counter()
            u, rep = gs.mpc_step_x0(x, k)
            wall.append((time.perf_counter() - t1) * 1e6); ker.append(rep.kernel_us); cabi.append(rep.wall_ms * 1e3)
            x = A @ x + B @ u
        # (a') the same closed loop served by the resident kernel (cqp_mpc_server_start): u0-only steps
        # through the C ABI (no CUDA call per step), and steps that also return the report
        x = wl.x0(1.0)
        srv_c, srv_d, srv_cr = [], [], []
        gs.cold_start(); gs.update_vectors(q.g, q.c, q.d); gs.solve()
        gs.mpc_server_start(k)
        u_buf = np.zeros(nu)
        for t in range(200):
            gs.mpc_step_x0_fast(np.ascontiguousarray(x), k, u_buf)
            wsrv, dsrv = gs.mpc_server_last_timing()
            srv_c.append(wsrv); srv_d.append(dsrv)
            x = A @ x + B @ u_buf
        for t in range(60):
            u, rep = gs.mpc_step_x0(x, k)
            srv_cr.append(rep.wall_ms * 1e3)
            x = A @ x + B @ u
        gs.mpc_server_stop()
        # (b) host-side instantiate (untimed), step uploads g, c, d (cqp_mpc_step)
        x = wl.x0(1.0)
        wall_gcd = []
        for t in range(60):
            q = wl.problem_at(x)
            t1 = time.perf_counter()
            rep = gs.mpc_step(q.g, q.c, q.d, k)
            wall_gcd.append((time.perf_counter() - t1) * 1e6)
            u = np.clip(-K @ x + rep.solution.y[:nu], wl.limits.u_lo, wl.limits.u_hi)
            x = A @ x + B @ u
        D = base.n + 2 * base.m
        info = gs.launch_info()
        wbytes = info["w_bytes_per_iteration"]      # bytes of W one iteration reads (structured: < 8 D^2)
        w50, k50 = statistics.median(wall[20:]), statistics.median(ker[20:])
        out.append({"workload": name, "n": base.n, "m": base.m, "D": D, "iters_per_step": k,
                    "initial_solve_iterations": r0.solution.iterations, "initial_solve_kernel_us": r0.kernel_us,
                    "step_wall_us_p50": w50, "step_kernel_us_p50": k50, "step_hz": 1e6 / w50,
                    "step_cabi_wall_us_p50": statistics.median(cabi[20:]),
                    "step_wall_us_p50_host_instantiate": statistics.median(wall_gcd[10:]),
                    "server_step_cabi_wall_us_p50": statistics.median(srv_c[20:]),
                    "server_step_device_us_p50": statistics.median(srv_d[20:]),
                    "server_step_hz": 1e6 / statistics.median(srv_c[20:]),
                    "server_step_with_report_cabi_wall_us_p50": statistics.median(srv_cr[10:]),
                    "server_note": "resident kernel + host-mapped mailbox (cqp_mpc_server_start); u0-only steps skip the final residual pass whose results the caller does not take; bit-identical iterate and u0 (tests/test_gpu_mpc_server.py)",
                    "W_bytes_per_iteration": wbytes, "dense_W_bytes_per_iteration": 8.0 * D * D,
                    "W_stream_GBs": wbytes * k / (k50 * 1e-6) / 1e9,
                    "cold_solve_W_GBs": wbytes * r0.solution.iterations / (r0.kernel_us * 1e-6) / 1e9,
                    "W_stream_frac_of_hbm_peak": wbytes * k / (k50 * 1e-6) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                    "launch": info})
        gs.close()
    return out


def gpu_arm(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from workloads import problems
    from paper_2311_18056_b200 import sharding, solver as S

    wl, g, c, d = make_workload(0)                       # every rank builds the same global batch
    base = wl.base_problem()
    n, m = base.n, base.m
    lo, hi = sharding.shard_range(BATCH, world, rank)    # strong scaling: this rank's columns
    cnt = hi - lo
    single = S.Solver(base.H, base.g, base.G, base.c, base.d, device=local_rank)   # offline stage on the device
    batch = S.BatchSolver(single, capacity=BATCH if world > 1 else max(cnt, 1))     # (N > 1: also the weak-scaling run)
    # pinned host staging of this rank's step inputs (e2e copies start from pinned memory)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, lo:hi].T)).pin_memory().numpy().T  # noqa: E731
    gp, cp, dp = pin(g), pin(c), pin(d)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        """One step through the public API: host inputs -> results on the host of rank 0."""
        if world == 1:
            o = batch.solve(gp, cp, dp, zero_copy=True)
            return o, o
        return sharding.solve_sharded_device(batch, g, c, d, dst=0, pinned=(gp, cp, dp))

    for _ in range(max(args.warmup, 3)):
        out, tm = step()
    sampler = ClockSampler(local_rank)
    barrier()
    sampler.start()
    t0 = time.perf_counter()
    comp_ms = tot_ms = gemm_ms = gemm_fl = 0.0
    launches = 0
    for _ in range(args.steps):
        out, tm = step()
        comp_ms += tm["compute_ms"]; tot_ms += tm["device_ms"]
        gemm_ms += tm["gemm_ms"]; gemm_fl += tm["gemm_flops"]; launches += tm["launches"]
    barrier()
    wall_s = time.perf_counter() - t0
    clocks = sampler.stop()

    stats = torch.tensor([comp_ms, tot_ms, wall_s * 1e3, gemm_ms], dtype=torch.float64, device="cuda")
    sums = torch.tensor([gemm_fl, float(launches)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)      # device time: max over ranks
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    comp_ms_max, tot_ms_max, wall_ms_max, gemm_ms_max = [float(x) for x in stats.tolist()]
    gemm_fl_all, launches_all = float(sums[0]), int(sums[1])

    # weak scaling (N > 1 only): every rank solves its own 4096 columns, nothing is gathered
    weak = None
    if world > 1:
        gw, cw, dw, _ = problems.batch_instances(wl, BATCH, first=rank * BATCH)
        pinw = lambda a: torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory().numpy().T  # noqa: E731
        gw, cw, dw = pinw(gw), pinw(cw), pinw(dw)
        wsteps = max(1, min(args.steps, 3))
        batch.solve(gw, cw, dw, zero_copy=True)
        barrier()
        wms = 0.0
        for _ in range(wsteps):
            wms += batch.solve(gw, cw, dw, zero_copy=True)["compute_ms"]
        barrier()
        wt = torch.tensor([wms], dtype=torch.float64, device="cuda")
        dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        weak = {"value": world * BATCH * wsteps / (float(wt[0]) * 1e-3), "unit": "QP/s", "per_gpu_batch": BATCH,
                "steps": wsteps, "scaling": "weak"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    total_qps = BATCH * args.steps
    value = total_qps / (comp_ms_max * 1e-3)
    e2e = total_qps / (wall_ms_max * 1e-3)
    peaks, peak_src = read_peaks()
    dgemm_peak = measure_dgemm_peak()
    achieved = gemm_fl_all / world / (gemm_ms_max * 1e-3) / 1e12      # per-GPU rate of the iteration GEMM
    D = n + 2 * m
    flop_col = 2 * ((n + m) * D + m * n) + 4 * m     # executed per active column per iteration
    dense_equiv = achieved * (2 * D * D) / flop_col   # what a dense-W kernel would need for the same solves
    traffic = None
    # (ncu --set full on two full-batch round_kernel launches, tools/summarize_profiles.py: dram read + write
    # bytes per LAUNCH = per check round of 25 layers over 4096 columns)
    prof = os.path.join(ROOT, "profiles", "round_kernel_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    mean_iterations = float(np.mean(out["iterations"]))
    solved = int((out["status"] == 0).sum())

    # CPU baseline on this box's host cores: bounded samples of the same instances (about 20 s)
    cores = os.cpu_count() or 1
    sample = 4 * cores
    sec, cpu_iters = oracle_solve_columns(wl, g, c, d, list(range(sample)), cores)
    cpu_qps = sample / sec
    # parity spot check inside the bench: the sampled columns' iteration counts
    parity_ok = bool(np.array_equal(np.array(cpu_iters), out["iterations"][:sample]))
    sec1, _ = oracle_solve_columns(wl, g, c, d, list(range(8)), 1)                     # the reference as shipped: one thread
    sec1v3, _ = oracle_solve_columns(wl, g, c, d, list(range(8)), 1, variant="v3")      # "best-effort CPU" flags
    secv3, _ = oracle_solve_columns(wl, g, c, d, list(range(sample)), cores, variant="v3")

    # secondary sections: a failure there must not cost the headline line
    section_errors = {}

    def guarded(name, fn):
        try:
            return fn()
        except Exception as e:  # noqa: BLE001
            section_errors[name] = repr(e)
            return None

    extra = world == 1 and not args.no_single
    sweep_kw = {"repeats": 21} if not args.quick else {"repeats": 5, "seeds": (0, 1), "nus": (10, 30, 50), "cpu_seeds": (0,)}
    single_qp = guarded("single_qp", lambda: single_qp_sweep(S, problems, **sweep_kw)) if extra else None
    hbm_measured = guarded("hbm_copy_peak", measure_hbm_copy_peak) if extra else None
    if hbm_measured is not None and "measured" not in peak_src:
        peaks = dict(peaks, hbm_gbs=hbm_measured)
        peak_src = "device copy measured in this run (MEASURED_PEAKS.json absent)"
    mpc_steps = guarded("mpc_steps", lambda: mpc_step_section(S, problems, peaks)) if extra else None
    rd_peaks = guarded("read_peaks", lambda: measure_read_peaks(local_rank)) if extra else None
    hbm_read, l2_read = rd_peaks if rd_peaks else (None, None)

    def small_batch_section(cols=512, reps=3):
        """The per-GPU share of the batch at N = 8 (512 columns), solved alone on this GPU: the small-batch
        regime that strong scaling runs into (device-resident timing, same accounting as `roofline`)."""
        sb = S.BatchSolver(single, capacity=cols)
        pin2 = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, :cols].T)).pin_memory().numpy().T  # noqa: E731
        g2, c2, d2 = pin2(g), pin2(c), pin2(d)
        sb.solve(g2, c2, d2, zero_copy=True)
        ms = gms = gfl = 0.0
        for _ in range(reps):
            o = sb.solve(g2, c2, d2, zero_copy=True)
            ms += o["compute_ms"]; gms += o["gemm_ms"]; gfl += o["gemm_flops"]
        its = float(np.mean(o["iterations"]))
        sb.close()
        return {"columns": cols, "steps": reps, "ms_per_step": ms / reps, "value": cols * reps / (ms * 1e-3), "unit": "QP/s",
                "mean_iterations": its, "round_kernel_tflops": gfl / (gms * 1e-3) / 1e12, "frac": gfl / (gms * 1e-3) / 1e12 / dgemm_peak,
                "frac_of_whole_step": gfl / (ms * 1e-3) / 1e12 / dgemm_peak,
                "note": "columns 0..511 of the same batch; what one of 8 GPUs solves under strong scaling"}

    batched_small = guarded("batched_small", small_batch_section) if extra else None

    line = {
        "metric": METRIC, "value": value, "unit": "QP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": comp_ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CONFIG,
        "results": {"mean_iterations": mean_iterations, "solved": solved, "columns_per_gpu": [sharding.shard_range(BATCH, world, r)[1] - sharding.shard_range(BATCH, world, r)[0] for r in range(world)],
                    "gather": "none (one GPU)" if world == 1 else "NCCL dist.gather of y, z, lambda, status/iterations/index/switches, residuals to rank 0, inside e2e"},
        "e2e": {"value": e2e, "unit": "QP/s", "h2d_bytes_per_step": 8 * (n + 2 * m) * BATCH,
                "d2h_bytes_per_step": 8 * (n + 2 * m) * BATCH + BATCH * (4 * 4 + 2 * 8),
                "device_ms_per_step": tot_ms_max / args.steps, "host_ms_per_step": wall_ms_max / args.steps},
        "gpu_launches": int(launches_all),
        "clocks": clocks,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": dgemm_peak, "unit": "TFLOP/s",
                     "frac": achieved / dgemm_peak, "traffic": traffic,
                     "kernel": "round_kernel (persistent launch = one check round of 25 ADMM layers of every active column; operands staged by TMA cp.async.bulk.tensor, FP64 DMMA.8x8x4)",
                     "frac_of_whole_step": (gemm_fl_all / world / (comp_ms_max * 1e-3) / 1e12 / dgemm_peak) if comp_ms_max else None,
                     "algorithmic": f"executed 2*((n+m)*D + m*n) + 4*m = {flop_col} flop per active column per iteration (the zero blocks (3,2), (3,3) of W are skipped; dense W would be 2*D^2 = {2 * D * D}); {gemm_fl_all:.4g} flop in {gemm_ms_max:.1f} ms over {args.steps} steps" + (f" on each of {world} GPUs (per-GPU rate)" if world > 1 else ""),
                     "dense_equivalent_tflops": dense_equiv,
                     "peak_source": "cuBLAS DGEMM 8192^3 via torch.matmul, best of 5, measured in this run (no FP64 entry in MEASURED_PEAKS.json)",
                     "peak_theoretical": f"148 SMs x 64 FP64 FMA/clk x 2 x {peaks.get('sm_max_mhz', 1965.0):.0f} MHz = {148 * 64 * 2 * peaks.get('sm_max_mhz', 1965.0) * 1e-6:.1f} TFLOP/s",
                     "gemm_share_of_step": gemm_ms_max / comp_ms_max if comp_ms_max else None,
                     "timing": "achieved = executed flop of all round_kernel launches / the sum of their durations (CUDA events around every launch on the solve's stream); frac_of_whole_step divides the same flop by the whole device-timed step (check rounds, re-bucketing and setup included)"},
        "cpu_baseline": {"value": cpu_qps, "unit": "QP/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} of the {BATCH} instances ({sample // cores} per core), one oracle Solver per thread (-O3 -DNDEBUG build = the reference's flags)",
                         "iteration_counts_match_gpu": parity_ok,
                         "one_core_qps": 8 / sec1, "one_core_qps_march_v3": 8 / sec1v3, "one_core_sample": "the first 8 instances, one thread (the reference has no threading)",
                         "all_cores_qps_march_v3": sample / secv3},
        "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "source": peak_src, "hbm_copy_gbs_this_run": hbm_measured},
    }
    if weak is not None:
        line["weak_scaling"] = weak
    if section_errors:
        line["section_errors"] = section_errors
    if mpc_steps is not None:
        a50 = [r for r in mpc_steps if "N=50" in r["workload"]]
        if a50:
            # Atlas-sized N = 50: the structured level (n+m)*D*8 + m*n*8 = 118 MB + vectors no longer
            # fits the 126 MB L2 next to everything else: the stream is HBM-bound
            r50 = a50[0]
            line["roofline_single_qp_hbm"] = {
                "bound": "hbm", "achieved": r50["cold_solve_W_GBs"], "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": r50["cold_solve_W_GBs"] / peaks.get("hbm_gbs", 6650.0), "traffic": None,
                "kernel": "run_kernel<16, true> at D = 4350 (W level 151 MB dense, structured 118 MB)",
                "algorithmic": f"{r50['W_bytes_per_iteration']:.0f} bytes of W per iteration x {r50['initial_solve_iterations']} iterations of the cold solve / its kernel time",
                "peak_source": peak_src}
    if batched_small is not None:
        line["batched_512_columns"] = batched_small
    if single_qp is not None:
        line["single_qp"] = single_qp
    if mpc_steps is not None:
        line["mpc_steps"] = mpc_steps
        big = mpc_steps[-1]      # quadruped-sized: the HBM-streamed tier of the single-QP kernel
        # The structured level of this config (94 MB) fits the 126 MB L2: ncu shows about a third of
        # the bytes coming from DRAM, the rest is served by L2.  The ceiling is therefore the L2 read
        # rate (measured above with an L2-resident reduction), not the HBM copy rate.
        l2_peak = l2_read if l2_read else 12400.0
        line["roofline_single_qp_stream"] = {
            "bound": "l2", "achieved": big["W_stream_GBs"], "peak": l2_peak, "unit": "GB/s",
            "frac": big["W_stream_GBs"] / l2_peak, "traffic": read_stream_traffic(),
            "kernel": "run_kernel<16, true> (persistent single-QP kernel, W through the cp.async.bulk ring)",
            "algorithmic": f"{big['W_bytes_per_iteration']:.0f} bytes of W per iteration (lambda rows streamed as rho*G only; dense 8*D^2 = {8 * big['D'] ** 2}) x {big['iters_per_step']} iterations per step / step kernel time (includes refresh_z, bias and epilogue residual passes)",
            "peak_source": ("cqp_measure_read_bandwidth: all SMs read an L2-resident 48 MB buffer 60 times (16-byte loads, 8 in flight per thread), measured in this run" if l2_read
                            else "fallback: ~6300 B/clk LTS cap x 1.965 GHz (B300_MICROARCH.md)"),
            "hbm_read_gbs": hbm_read,
            "hbm_copy_gbs": peaks.get("hbm_gbs"), "frac_of_hbm_copy_rate": big["W_stream_frac_of_hbm_peak"],
            "traffic_source": "ncu dram__bytes_read + write per iteration (profiles/stream_traffic.json): DRAM supplies that much of the algorithmic bytes, L2 the rest",
            "note": "frac_of_hbm_copy_rate can exceed 1 because most of W is re-read from L2 every iteration; with the dense layer (133 MB, session 2) the same kernel was HBM-bound at 92 % of the copy rate"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without torchrun: start the N ranks (one per GPU) ourselves."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible; refusing to time fewer GPUs "
              "under an N-GPU label", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO" if args.nccl_log else "WARN")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    ap.add_argument("--no-single", action="store_true", help="skip the single-QP / MPC-step sections")
    ap.add_argument("--quick", action="store_true", help="shortened single-QP sweep (3 sizes, 2 seeds, 5 repeats)")
    ap.add_argument("--nccl-log", action="store_true", help="NCCL_DEBUG=INFO for the spawned ranks")
    args = ap.parse_args()
    if args.impl == "gpu" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
