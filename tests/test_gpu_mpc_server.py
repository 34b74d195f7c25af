"""GPU tests of the resident control-step server (cqp_mpc_server_start): the closed loop of
bench.cpp:157-185 served by ONE persistent kernel from a host-mapped mailbox must reproduce the
launch-per-step path (cqp_mpc_step_x0 without the server) bit for bit, in every kernel tier."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2311_18056_b200 import solver as S
    from paper_2311_18056_b200 import _lib
    if _lib.load().cqp_device_count() < 1:
        pytest.fail("no CUDA device: the solve path has no CPU fallback")
    return S


@pytest.fixture(scope="module")
def P():
    from workloads import problems
    return problems


def closed_loop(gs, wl, k, steps, use_server, idle_ms=100.0, pause_at=(), pause_s=0.0, poke_at=(), fast=False):
    """Runs the receding-horizon loop; returns per step (u0, y, z, lam, r_prim, r_dual, status)."""
    gs.cold_start()
    gs.update_vectors(*[getattr(wl.problem_at(wl.x0(1.0)), a) for a in ("g", "c", "d")])
    gs.solve()                                   # converge once: the loop continues from here (warm)
    if use_server:
        gs.mpc_server_start(k, idle_ms)
    A, B = wl.sys.A, wl.sys.B
    x = wl.x0(1.0)
    out = []
    for step in range(steps):
        if step in pause_at:
            time.sleep(pause_s)                  # let the idle timeout retire the kernel
        if step in poke_at:
            assert gs.layer_index >= 0           # any other entry point retires the resident kernel
        if fast and step % 3 != 0:               # u0-only steps (no report, no final residual pass) in between
            u0 = np.zeros(wl.sys.nu)
            gs.mpc_step_x0_fast(np.ascontiguousarray(x), k, u0)
            out.append((u0.copy(),))
        else:
            u0, rep = gs.mpc_step_x0(x, k)
            s = rep.solution
            out.append((u0.copy(), s.y.copy(), s.z.copy(), s.lam.copy(), s.r_prim, s.r_dual, s.status, s.iterations))
        x = A @ x + B @ u0
    if use_server:
        gs.mpc_server_stop()
    return out


def same(a, b):
    for sa, sb in zip(a, b):
        for va, vb in zip(sa, sb):
            if isinstance(va, np.ndarray):
                assert np.array_equal(va, vb)
            else:
                assert va == vb
    assert len(a) == len(b)


@pytest.mark.parametrize("tier", ["cluster", "grid_resident", "grid_streamed"])
@pytest.mark.parametrize("k", [1, 2, 15])
def test_server_matches_launch_per_step(G, P, monkeypatch, tier, k):
    if tier == "grid_resident":
        monkeypatch.setenv("CQP_FORCE_TIER", "0")
    elif tier == "grid_streamed":
        monkeypatch.setenv("CQP_FORCE_TIER", "1")
    wl = P.config1(seed=3)
    base = wl.base_problem()
    gs = G.Solver(base.H, base.g, base.G, base.c, base.d)
    want = {"cluster": 2, "grid_resident": 0, "grid_streamed": 1}[tier]
    assert gs.launch_info()["tier"] == want
    gs.set_mpc_template(wl.tmpl, wl.limits)
    ref = closed_loop(gs, wl, k, 40, use_server=False)
    got = closed_loop(gs, wl, k, 40, use_server=True)
    same(ref, got)
    # u0-only steps mixed in: the same controls and, at the reporting steps, the same reports
    ref_f = closed_loop(gs, wl, k, 40, use_server=False, fast=True)
    got_f = closed_loop(gs, wl, k, 40, use_server=True, fast=True)
    same(ref_f, got_f)
    same([r[:1] for r in ref], [r[:1] for r in got_f])
    assert any(np.any(np.isclose(r[0], wl.limits.u_lo) | np.isclose(r[0], wl.limits.u_hi)) for r in ref)  # limits hit
    gs.close()


def test_server_idle_timeout_and_interleaved_calls(G, P):
    """The resident kernel leaves after the idle timeout and the next step restarts it; any other
    entry point of the handle retires it; results do not change."""
    wl = P.config1(seed=3)
    base = wl.base_problem()
    gs = G.Solver(base.H, base.g, base.G, base.c, base.d)
    gs.set_mpc_template(wl.tmpl, wl.limits)
    ref = closed_loop(gs, wl, 2, 30, use_server=False)
    got = closed_loop(gs, wl, 2, 30, use_server=True, idle_ms=5.0, pause_at=(7, 19), pause_s=0.05, poke_at=(11, 12))
    same(ref, got)
    # a plain solve still works after the server (and equals a solve without it)
    q = wl.problem_at(wl.x0(10.0))
    gs.mpc_server_start(2)
    gs.update_vectors(q.g, q.c, q.d); gs.cold_start()
    a = gs.solve().solution
    gs.update_vectors(q.g, q.c, q.d); gs.cold_start()
    b = gs.solve().solution
    assert a.iterations == b.iterations and np.array_equal(a.y, b.y)
    gs.close()


def test_server_mid_size_streamed_tier(G, P):
    """An Atlas-like size (streamed tier by itself, structured layer, n = m = 290): server == launch per step."""
    wl = P.config3_atlas(horizon=10)
    base = wl.base_problem()
    gs = G.Solver(base.H, base.g, base.G, base.c, base.d)
    gs.set_mpc_template(wl.tmpl, wl.limits)
    ref = closed_loop(gs, wl, 2, 12, use_server=False)
    got = closed_loop(gs, wl, 2, 12, use_server=True)
    same(ref, got)
    gs.close()


@pytest.mark.parametrize("nu,k", [(40, 1), (50, 2)])
def test_server_resident_tier_large_slices(G, P, nu, k):
    """Resident tier with 9..11 rows per CTA (16-row blocks; D = 1200 / 1500): server == launch per
    step.  (A launch of k < 4 iterations used to stream W instead of holding it in shared memory, which
    adds a row's products up in another order: the two paths then differed in the last bits.)"""
    wl = P.config2(nu, seed=0)
    base = wl.base_problem()
    gs = G.Solver(base.H, base.g, base.G, base.c, base.d)
    assert gs.launch_info()["tier"] == 0 and gs.launch_info()["rows_per_cta"] > 8
    gs.set_mpc_template(wl.tmpl, wl.limits)
    ref = closed_loop(gs, wl, k, 25, use_server=False, fast=True)
    got = closed_loop(gs, wl, k, 25, use_server=True, fast=True)
    same(ref, got)
    gs.close()
