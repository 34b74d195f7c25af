"""Soak / litmus test of the iterate exchange of the persistent single-QP kernels (data-as-flag L2
ring of cqp_single.cu, st.async + mbarrier exchange of cqp_cluster.cu): 10^6 iterations in ONE launch
per tier and fence mode.  A lost or stale word would trip the in-kernel watchdog (a CUDA error) or
change the iterate; the final state must be bit-identical from run to run and across the fence modes
(the publish order does not change the arithmetic)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITERS = 1_000_000


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


@pytest.mark.parametrize("nu,tier_env,want_tier", [(10, None, 2), (30, None, 0), (14, "1", 1), (10, "0", 0)])
def test_million_iterations_per_launch(G, P, monkeypatch, nu, tier_env, want_tier):
    wl = P.config2(nu, seed=1)
    base = wl.base_problem()
    q = wl.problem_at(wl.x0(10.0))
    states = []
    for fence in ("0", "2", "0"):
        monkeypatch.setenv("CQP_FENCE_MODE", fence)
        if tier_env is not None:
            monkeypatch.setenv("CQP_FORCE_TIER", tier_env)
        # adaptive_rho off: the iterate keeps moving for longer and no layer switch hides a bad word
        gs = G.Solver(base.H, base.g, base.G, base.c, base.d, G.SolverSettings(adaptive_rho=(fence == "2")))
        assert gs.launch_info()["tier"] == want_tier
        gs.update_vectors(q.g, q.c, q.d)
        gs.cold_start()
        rep = gs.fixed_iters(ITERS)                       # one launch, 10^6 exchanges of the iterate
        assert rep.solution.iterations == ITERS
        assert len(rep.residual_history) == ITERS // 25
        assert np.all(np.isfinite(rep.solution.y)) and rep.solution.r_prim <= 1e-6 and rep.solution.r_dual <= 1e-6
        states.append((gs.state.copy(), gs.layer_index, rep.solution.y.copy()))
        gs.close()
    assert np.array_equal(states[0][0], states[2][0]) and states[0][1] == states[2][1]   # run to run
    # adaptive run (fence mode 2) ends at the same KKT point
    assert np.abs(states[1][2] - states[0][2]).max() <= 1e-6 * max(1.0, np.abs(states[0][2]).max())
