"""GPU parity on the robot-sized BASELINE.json configs ([2] Atlas-sized, [3] quadruped + arm sized).

These are the sizes whose W level (54 - 133 MB) no longer fits shared memory: the persistent
kernel streams W from L2/HBM (tier 1).  Checked through the C ABI against the CPU oracle where the
oracle finishes in seconds (Atlas N = 30, quadruped N = 15), and through size-independent
properties at the full quadruped size (N = 30, D = 4080): KKT residual bounds, z inside its box,
`fixed_iters(a + b)` == `fixed_iters(a); fixed_iters(b)` bit for bit, fused MPC step == 3 calls.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from test_gpu_single import assert_report_parity, oracle_layers, rel_err  # noqa: E402


@pytest.fixture(scope="module")
def G():
    from paper_2311_18056_b200 import _lib
    from paper_2311_18056_b200 import solver as S
    if _lib.load().cqp_device_count() < 1:
        pytest.fail("no CUDA device: the solve path has no CPU fallback")
    return S


@pytest.fixture(scope="module")
def P():
    from workloads import problems
    return problems


def closed_loop(wl, gpu, cpu, k, steps, x):
    """bench.cpp:157-185: instantiate -> update_vectors -> refresh_z -> fixed_iters(k) -> plant."""
    A, B, K, nu = wl.sys.A, wl.sys.B, wl.tmpl.K, wl.sys.nu
    for _ in range(steps):
        q = wl.problem_at(x)
        cpu.update_vectors(q.g, q.c, q.d); cpu.refresh_z(); ro = cpu.fixed_iters(k)
        rg = gpu.mpc_step(q.g, q.c, q.d, k)
        assert rg.solution.iterations == k == ro.solution.iterations
        assert rg.solution.rho_trace == ro.solution.rho_trace
        assert rel_err(rg.solution.y, ro.solution.y) <= 1e-9
        assert rel_err(rg.solution.lam, ro.solution.lam) <= 1e-9
        assert rel_err(rg.solution.z, ro.solution.z) <= 1e-9
        u = np.clip(-K @ x + ro.solution.y[:nu], wl.limits.u_lo, wl.limits.u_hi)
        x = A @ x + B @ u
    return x


@pytest.mark.parametrize("name,k,hard", [("atlas30", 2, 3.0), ("quad15", 15, 3.0)])
def test_robot_sized_parity_with_oracle(G, oracle, P, name, k, hard):
    wl = P.config3_atlas(30, seed=0) if name == "atlas30" else P.config4_quadruped(15, seed=0)
    base = wl.base_problem()
    cpu = oracle.Solver(oracle.QProblem(base.H, base.g, base.G, base.c, base.d), variant="v3")
    gpu = G.Solver(base.H, base.g, base.G, base.c, base.d, layers=oracle_layers(cpu.cache))
    info = gpu.launch_info()
    assert info["tier"] == 1 and info["structured"] == 1   # W streamed from L2/HBM, lambda rows as rho G only
    # initial solve to tolerance from a hard start, then the receding-horizon loop
    x0 = wl.x0(hard)
    q = wl.problem_at(x0)
    for s in (gpu, cpu):
        s.update_vectors(q.g, q.c, q.d)
        s.cold_start()
    rg, ro = gpu.solve(), cpu.solve()
    assert ro.solution.status == oracle.SOLVED
    assert_report_parity(rg, ro)
    x5 = closed_loop(wl, gpu, cpu, k, 5, x0)
    # the same loop with instantiate + control extraction on the device (upload x0, download u0)
    gpu.set_mpc_template(wl.tmpl, wl.limits)
    A, B, K, nu = wl.sys.A, wl.sys.B, wl.tmpl.K, wl.sys.nu
    x = x5
    for _ in range(3):
        q = wl.problem_at(x)
        cpu.update_vectors(q.g, q.c, q.d); cpu.refresh_z(); ro = cpu.fixed_iters(k)
        u_ref = np.clip(-K @ x + ro.solution.y[:nu], wl.limits.u_lo, wl.limits.u_hi)
        u0, rg = gpu.mpc_step_x0(x, k)
        assert rel_err(rg.solution.y, ro.solution.y) <= 1e-9 and rel_err(rg.solution.lam, ro.solution.lam) <= 1e-9
        assert np.abs(u0 - u_ref).max() <= 1e-9 * max(1.0, np.abs(u_ref).max())
        x = A @ x + B @ u_ref


def test_quadruped_full_size_properties(G, P):
    """configs[3] at N = 30 (n = 960, m = 1560, D = 4080, W level 133 MB), device offline stage."""
    wl = P.config4_quadruped(30, seed=0)
    base = wl.base_problem()
    gpu = G.Solver(base.H, base.g, base.G, base.c, base.d)
    info = gpu.launch_info()
    assert info["tier"] == 1 and info["ctas"] >= 140
    q = wl.problem_at(wl.x0(3.0))
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start()
    rep = gpu.solve()
    sol = rep.solution
    assert sol.status == G.SOLVED and sol.iterations % 25 == 0
    assert [h[0] for h in rep.residual_history] == list(range(25, sol.iterations + 1, 25))
    # the returned point satisfies the reference's own stopping rule on the ORIGINAL problem
    assert np.abs(q.G @ sol.y - sol.z).max() <= 1e-6
    assert np.abs(q.H @ sol.y + q.g + q.G.T @ sol.lam).max() <= 1e-6
    assert np.all(sol.z >= q.c) and np.all(sol.z <= q.d)
    # complementarity sign: multipliers push only against active bounds
    inner = (sol.z > q.c + 1e-7) & (sol.z < q.d - 1e-7)
    assert np.abs(sol.lam[inner]).max() <= 1e-4
    # fixed_iters composes bit for bit (tests/test_solver.cpp:211-233 at full size)
    gpu.cold_start(); gpu.fixed_iters(7); va = gpu.state
    gpu.cold_start(); gpu.fixed_iters(3); gpu.fixed_iters(4); vb = gpu.state
    assert np.array_equal(va, vb)
    # fused MPC step == update_vectors + refresh_z + fixed_iters, bit for bit
    q2 = wl.problem_at(0.5 * wl.x0(3.0))
    gpu.cold_start(); gpu.fixed_iters(5)
    v0 = gpu.state
    r_fused = gpu.mpc_step(q2.g, q2.c, q2.d, 15)
    v_fused = gpu.state
    gpu.update_vectors(q.g, q.c, q.d); gpu.cold_start(); gpu.fixed_iters(5)
    assert np.array_equal(gpu.state, v0)
    gpu.update_vectors(q2.g, q2.c, q2.d); gpu.refresh_z(); r_three = gpu.fixed_iters(15)
    assert np.array_equal(gpu.state, v_fused)
    assert np.array_equal(r_fused.solution.y, r_three.solution.y)
