"""GPU parity tests of the single-QP path, through the C ABI (libcqp_b200.so) vs the CPU oracle.

Bar (BASELINE.json north_star): identical iteration counts and rho-switch sequence in FP64;
primal and dual solutions within 1e-6 relative.  Residual samples are compared to 2e-3
relative (sums of O(n) FP64 terms in a different order, amplified near convergence).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_SOL = 1e-6     # north_star tolerance on y and lambda
REL_RES = 2e-3     # residual samples: a different FP64 summation order is amplified by the
                   # x1e3 equality penalties near convergence (observed up to 2e-4 at n = 200)


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


def oracle_layers(cache):
    return {"W": [cache.W(k) for k in range(cache.L)], "D": [cache.D(k) for k in range(cache.L)],
            "GD": [cache.GD(k) for k in range(cache.L)], "grid": cache.grid,
            "initial_index": cache.initial_index, "Gs": cache.Gs, "E": cache.E, "F": cache.F,
            "cost_scale": cache.cost_scale}


def settings_pair(O, S, **kw):
    return O.SolverSettings(**kw), S.SolverSettings(**kw)


def rel_err(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(1.0, np.abs(np.asarray(b)).max()))


def assert_report_parity(rg, ro, sol_tol=REL_SOL, res_rel=REL_RES, res_abs=1e-9):
    sg, so = rg.solution, ro.solution
    assert sg.iterations == so.iterations
    assert sg.status == so.status
    assert sg.rho_trace == so.rho_trace
    assert [(h[0], h[3]) for h in rg.residual_history] == [(h[0], h[3]) for h in ro.residual_history]
    for hg, ho in zip(rg.residual_history, ro.residual_history):
        # residuals are differences of O(1) sums: absolute floor ~1e-10, else relative
        assert abs(hg[1] - ho[1]) <= res_rel * abs(ho[1]) + res_abs
        assert abs(hg[2] - ho[2]) <= res_rel * abs(ho[2]) + res_abs
    assert rel_err(sg.y, so.y) <= sol_tol
    assert rel_err(sg.lam, so.lam) <= sol_tol
    assert rel_err(sg.z, so.z) <= sol_tol


def make_pair(O, S, p, so=None, sg=None, from_layers=True):
    """(gpu solver, oracle solver) on the same problem; with from_layers the GPU gets the
    oracle's ladder so the ONLY difference is the online loop."""
    so = so or O.SolverSettings()
    sg = sg or S.SolverSettings()
    osolver = O.Solver(O.QProblem(p.H, p.g, p.G, p.c, p.d), so, variant="ref")
    layers = oracle_layers(osolver.cache) if from_layers else None
    gsolver = S.Solver(p.H, p.g, p.G, p.c, p.d, sg, layers=layers)
    return gsolver, osolver


# ---- known answers of the reference, on the GPU path --------------------------------------------
def test_1d_hand_worked_iterate(G, oracle):
    # tests/test_solver.cpp:58-72 / SPEC.md:212: sigma = 0, rho = 1: one iterate from 0 = [2/3, .5, 0]
    O = oracle
    D = O.build_kkt_inverse([[2.0]], [[1.0]], 0.0, [1.0])
    W, GD, b = O.build_layer([[2.0]], [[1.0]], [-2.0], 0.0, [1.0], D)
    layers = {"W": [W, W], "D": [D, D], "GD": [GD, GD], "grid": [1.0, 10.0], "initial_index": 0,
              "Gs": [[1.0]], "E": [1.0], "F": [1.0], "cost_scale": 1.0}
    s = G.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5], G.SolverSettings(adaptive_rho=False),
                 layers=layers)
    got = s.layer(0)
    expected = np.array([[-1 / 3, 2 / 3, -1 / 3], [2 / 3, -1 / 3, 2 / 3], [1.0, -1.0, 1.0]])
    assert np.abs(got["W"] - expected).max() < 1e-15          # tests/test_layers.cpp:191-207
    assert np.abs(got["b"] - np.array([2 / 3, 2 / 3, 0.0])).max() < 1e-15
    s.fixed_iters(1)
    v = s.state
    assert v[0] == pytest.approx(2.0 / 3.0, rel=1e-14)
    assert v[1] == 0.5
    assert v[2] == 0.0


def test_three_1d_kkt_solves(G):
    # tests/test_solver.cpp:175-209
    st = G.SolverSettings(eps_prim=1e-8, eps_dual=1e-8, max_iters=20000)
    sol = G.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5], st).solve().solution
    assert sol.status == G.SOLVED
    assert sol.y[0] == pytest.approx(0.5, rel=1e-6) and sol.lam[0] == pytest.approx(1.0, rel=1e-6)
    sol = G.Solver([[1.0]], [0.0], [[1.0]], [1.0], [1.0], st).solve().solution
    assert sol.status == G.SOLVED
    assert sol.y[0] == pytest.approx(1.0, rel=1e-6) and sol.lam[0] == pytest.approx(-1.0, rel=1e-6)
    sol = G.Solver([[2.0]], [-2.0], [[1.0]], [-10.0], [10.0], st).solve().solution
    assert sol.status == G.SOLVED
    assert sol.y[0] == pytest.approx(1.0, rel=1e-6) and abs(sol.lam[0]) < 1e-6


def test_1d_solves_match_oracle_exactly_in_counts(G, oracle):
    for (H, g, c, d) in [(2.0, -2.0, 0.0, 0.5), (1.0, 0.0, 1.0, 1.0), (2.0, -2.0, -10.0, 10.0)]:
        kw = dict(eps_prim=1e-8, eps_dual=1e-8, max_iters=20000)
        so, sg = settings_pair(oracle, G, **kw)
        p = oracle.QProblem([[H]], [g], [[1.0]], [c], [d])
        gs, os_ = make_pair(oracle, G, p, so, sg, from_layers=False)
        assert_report_parity(gs.solve(), os_.solve())


# ---- parity on the reference's random dense QP family (equality rows -> rho switches) -----------
@pytest.mark.parametrize("n,seeds", [(8, range(4)), (20, range(4)), (50, range(3)), (200, range(2))])
def test_dense_qp_parity_with_oracle_ladder(G, oracle, n, seeds):
    for seed in seeds:
        p = oracle.gen_random_dense_qp(n, seed)
        gs, os_ = make_pair(oracle, G, p, from_layers=True)
        assert_report_parity(gs.solve(), os_.solve())


@pytest.mark.parametrize("n,seeds", [(12, range(3)), (50, range(2)), (200, range(1))])
def test_dense_qp_parity_with_device_offline_stage(G, oracle, n, seeds):
    for seed in seeds:
        p = oracle.gen_random_dense_qp(n, seed)
        gs, os_ = make_pair(oracle, G, p, from_layers=False)
        # offline stage: every W / D / GD against the oracle (tests/test_layers.cpp:265-274);
        # the two stiffest grid points are ill-conditioned (see test_oracle_known_answers.py)
        sc = gs.scaling()
        assert np.array_equal(sc["E"], os_.cache.E) and np.array_equal(sc["F"], os_.cache.F)
        assert sc["cost_scale"] == os_.cache.cost_scale
        assert sc["initial_index"] == os_.cache.initial_index
        assert np.array_equal(sc["grid"], os_.cache.grid)
        assert np.array_equal(sc["c_tilde"], os_.cache.c_tilde)
        for k in range(gs.L):
            lay = gs.layer(k)
            tol = 1e-10 if os_.cache.grid[k] <= 1.0 else 1e-7
            assert np.abs(lay["W"] - os_.cache.W(k)).max() <= tol * max(1.0, np.abs(os_.cache.W(k)).max())
            assert np.abs(lay["D"] - os_.cache.D(k)).max() <= tol * max(1.0, np.abs(os_.cache.D(k)).max())
            assert np.array_equal(lay["rho_vec"], os_.cache.rho_vec(k))
            assert np.abs(lay["b"] - os_.cache.b(k)).max() <= tol * max(1.0, np.abs(os_.cache.b(k)).max())
        # Two FP64 offline stages (the blocked device Cholesky + substitution of cqp_setup.cu here, the oracle's there) differ
        # by ~cond(KKT)*eps in W (up to 1e-10 at these sizes); the x1e3 equality penalties
        # amplify that into the 1e-7 digits of the residual SAMPLES near convergence.  Counts,
        # traces and solutions must still agree.
        assert_report_parity(gs.solve(), os_.solve(), res_rel=0.5, res_abs=1e-7)


def test_cluster_kernel_layouts(G, oracle, P, monkeypatch):
    """(CQP_FORCE_TIER=2 keeps the cluster kernel above D = 512, where the default is the all-SM grid.)
    The cluster tier picks its layout from D: register mode with NPT = 2..16 column pairs per
    lane (D <= 512), shared-memory mode with 1-4 rows per warp above, residual rows cached in shared
    memory or read through L2 when they do not fit.  One parity solve per layout, odd D included."""
    cases = [("dense", 35), ("dense", 90), ("dense", 130), ("dense", 200), ("mpc", 21)]
    monkeypatch.setenv("CQP_FORCE_TIER", "2")
    for kind, size in cases:
        if kind == "dense":
            p = oracle.gen_random_dense_qp(size, 7)
            q = p
        else:
            wl = P.config2(size, seed=1)
            p = wl.base_problem()
            q = wl.problem_at(wl.x0(3.0))
        gs, os_ = make_pair(oracle, G, p, from_layers=True)
        assert gs.launch_info()["tier"] == 2, (kind, size, gs.launch_info())
        for s in (gs, os_):
            s.update_vectors(q.g, q.c, q.d)
            s.cold_start()
        assert_report_parity(gs.solve(), os_.solve())
        # fixed_iters composes bit for bit in this tier too (tests/test_solver.cpp:211-233)
        gs.cold_start(); gs.fixed_iters(7); va = gs.state
        gs.cold_start(); gs.fixed_iters(3); gs.fixed_iters(4)
        assert np.array_equal(gs.state, va)


# ---- the BASELINE.json MPC configs ---------------------------------------------------------------
@pytest.mark.parametrize("nu,hard,unstable", [(10, 1.0, False), (10, 10.0, False), (10, 10.0, True),
                                             (30, 1.0, False), (30, 10.0, False), (50, 10.0, False)])
def test_random_mpc_parity(G, oracle, P, nu, hard, unstable):
    wl = P.config2(nu, seed=0, unstable=unstable)
    base = wl.base_problem()
    gs, os_ = make_pair(oracle, G, base, from_layers=True)
    q = wl.problem_at(wl.x0(hard))
    for s in (gs, os_):
        s.update_vectors(q.g, q.c, q.d)
        s.cold_start()
    rg, ro = gs.solve(), os_.solve()
    assert ro.solution.status == oracle.SOLVED
    assert_report_parity(rg, ro)
    # size-independent property: the returned point satisfies the KKT residual bound itself
    y, z, lam = rg.solution.y, rg.solution.z, rg.solution.lam
    assert np.abs(q.G @ y - z).max() <= 1e-6 and np.abs(q.H @ y + q.g + q.G.T @ lam).max() <= 1e-6
    assert np.all(z >= q.c) and np.all(z <= q.d)


def test_mpc_device_offline_stage_counts(G, oracle, P):
    wl = P.config2(30, seed=1)
    base = wl.base_problem()
    gs, os_ = make_pair(oracle, G, base, from_layers=False)
    q = wl.problem_at(wl.x0(10.0))
    for s in (gs, os_):
        s.update_vectors(q.g, q.c, q.d)
        s.cold_start()
    assert_report_parity(gs.solve(), os_.solve())


# ---- structural tests of the reference ----------------------------------------------------------
def test_fixed_iters_composes_and_history(G, oracle):
    # tests/test_solver.cpp:211-233, 378-388
    p = oracle.gen_random_dense_qp(8, 6)
    kw = dict(adaptive_rho=False, eq_enabled=False)
    so, sg = settings_pair(oracle, G, **kw)
    gs, os_ = make_pair(oracle, G, p, so, sg)
    cache = os_.cache
    k0 = cache.initial_index
    W, b = cache.W(k0), cache.b(k0)
    one = gs.fixed_iters(1)
    v1 = oracle.iterate(np.zeros(16), W, b, cache.c_tilde, cache.d_tilde)
    assert rel_err(one.solution.y, v1[:8]) <= 1e-13 and one.solution.iterations == 1
    gs.cold_start()
    many = gs.fixed_iters(25)
    assert many.solution.iterations == 25 and len(many.residual_history) == 1
    # k calls of fixed_iters(1) == one call of fixed_iters(k), bit for bit (persistent iterate)
    gs.cold_start()
    for _ in range(25):
        gs.fixed_iters(1)
    v_steps = gs.state
    gs.cold_start()
    gs.fixed_iters(25)
    assert np.array_equal(gs.state, v_steps)
    p13 = oracle.gen_random_dense_qp(8, 13)
    gs2, _ = make_pair(oracle, G, p13, oracle.SolverSettings(adaptive_rho=False),
                       G.SolverSettings(adaptive_rho=False))
    rep = gs2.fixed_iters(100)
    assert [h[0] for h in rep.residual_history] == [25, 50, 75, 100]


@pytest.mark.parametrize("nu", [30, 40, 50])
def test_iteration_split_is_bitwise_neutral_at_mpc_sizes(G, P, nu):
    """fixed_iters(1) + fixed_iters(2) + fixed_iters(5) == fixed_iters(8) bit for bit at the sizes of the
    nu sweep (resident tier, 7..11 rows per CTA): the summation order of a layer is a property of the
    handle, not of how many iterations one launch runs."""
    wl = P.config2(nu, seed=1)
    base = wl.base_problem()
    gs = G.Solver(base.H, base.g, base.G, base.c, base.d, G.SolverSettings(adaptive_rho=False))
    q = wl.problem_at(wl.x0(1.0))
    gs.update_vectors(q.g, q.c, q.d)
    gs.cold_start()
    for k in (1, 2, 5):
        gs.fixed_iters(k)
    split = gs.state.copy()
    gs.cold_start()
    gs.fixed_iters(8)
    assert np.array_equal(gs.state, split)
    gs.close()


def test_rho_trace_structure_and_persistent_index(G, oracle):
    # tests/test_solver.cpp:390-401 + semantics 2/6 of SURVEY.md section 8(a)
    p = oracle.gen_random_dense_qp(16, 14)
    gs, os_ = make_pair(oracle, G, p)
    rg, ro = gs.solve(), os_.solve()
    tr = rg.solution.rho_trace
    assert tr[0] == (0, os_.cache.initial_index)
    for i in range(1, len(tr)):
        assert tr[i][0] % 25 == 0 and tr[i][1] != tr[i - 1][1]
    assert gs.layer_index == os_.layer_index == tr[-1][1]
    # a second solve() continues from the persistent state (solver.cpp:202-205)
    assert_report_parity(gs.solve(), os_.solve())


def test_identical_solves_bit_for_bit(G, oracle):
    # tests/test_solver.cpp:318-334
    p = oracle.gen_random_dense_qp(20, 11)
    a, _ = make_pair(oracle, G, p)
    b, _ = make_pair(oracle, G, p)
    ra, rb = a.solve(), b.solve()
    assert np.array_equal(ra.solution.y, rb.solution.y)
    assert np.array_equal(ra.solution.z, rb.solution.z)
    assert np.array_equal(ra.solution.lam, rb.solution.lam)
    assert ra.solution.iterations == rb.solution.iterations
    assert ra.residual_history == rb.residual_history
    a.cold_start()
    rc = a.solve()
    assert np.array_equal(ra.solution.y, rc.solution.y) and ra.residual_history == rc.residual_history


def test_warm_start_mapping(G, oracle):
    # tests/test_solver.cpp:139-173
    p = oracle.gen_random_dense_qp(8, 4)
    gs, os_ = make_pair(oracle, G, p, oracle.SolverSettings(grid_points=7), G.SolverSettings(grid_points=7))
    rng = oracle.Rng(5)
    prev_o = oracle.Solution(y=rng.normal_vector(8), lam=rng.normal_vector(4), z=np.full(4, 123.0),
                             rho_trace=[(0, 2), (50, 4)])
    prev_g = G.Solution(prev_o.y, prev_o.z, prev_o.lam, rho_trace=prev_o.rho_trace)
    gs.warm_start(prev_g)
    os_.warm_start(prev_o)
    assert gs.layer_index == 4 == os_.layer_index
    assert rel_err(gs.state, os_.state) <= 1e-14
    with pytest.raises(ValueError):
        gs.warm_start(G.Solution(np.zeros(3), np.zeros(4), np.zeros(4)))
    gs.warm_start(G.Solution(np.zeros(8), np.zeros(4), np.zeros(4), rho_trace=[(0, 2)]))
    assert np.all(gs.state == 0.0) and gs.layer_index == 2


def test_validation_and_argument_errors(G):
    # tests/test_problem.cpp validate codes; tests/test_solver.cpp:362-376
    with pytest.raises(G.ProblemError) as e:
        G.Solver([[1.0, 0.5], [0.0, 1.0]], [0.0, 0.0], [[1.0, 0.0]], [0.0], [1.0])
    assert e.value.code == "NonSymmetricH"
    with pytest.raises(G.ProblemError) as e:
        G.Solver([[-1.0]], [0.0], [[1.0]], [0.0], [1.0])
    assert e.value.code == "NonPositiveDefiniteH"
    with pytest.raises(G.ProblemError) as e:
        G.Solver([[1.0]], [0.0], [[1.0]], [1.0], [0.0])
    assert e.value.code == "InvertedBounds"
    with pytest.raises(G.ProblemError) as e:
        G.Solver([[1.0]], [float("nan")], [[1.0]], [0.0], [1.0])
    assert e.value.code == "NonFiniteEntry"
    with pytest.raises(G.ProblemError) as e:
        G.Solver([[1.0]], [0.0, 1.0], [[1.0]], [0.0], [1.0])
    assert e.value.code == "DimensionMismatch"
    with pytest.raises(ValueError):
        G.Solver([[1.0]], [0.0], [[1.0]], [0.0], [1.0], G.SolverSettings(check_interval=0))
    with pytest.raises(ValueError):
        G.Solver([[1.0]], [0.0], [[1.0]], [0.0], [1.0], G.SolverSettings(max_iters=10))
    with pytest.raises(ValueError):
        G.Solver([[1.0]], [0.0], [[1.0]], [0.0], [1.0], G.SolverSettings(grid_points=1))
    s = G.Solver([[1.0]], [0.0], [[1.0]], [0.0], [1.0])
    with pytest.raises(ValueError):
        s.fixed_iters(0)
    with pytest.raises(ValueError):
        s.update_vectors([0.0, 1.0], [0.0], [1.0])


def test_infinite_bounds_pass_through(G, oracle):
    # +-inf bounds survive scaling and the clamp
    p = oracle.gen_random_dense_qp(12, 3)
    p.c[3] = -np.inf
    p.d[4] = np.inf
    p.c[5], p.d[5] = -np.inf, np.inf
    gs, os_ = make_pair(oracle, G, p)
    assert_report_parity(gs.solve(), os_.solve())


def test_max_iters_status(G, oracle):
    p = oracle.gen_random_dense_qp(50, 1)
    kw = dict(eps_prim=1e-13, eps_dual=1e-13, max_iters=100)
    so, sg = settings_pair(oracle, G, **kw)
    gs, os_ = make_pair(oracle, G, p, so, sg)
    rg, ro = gs.solve(), os_.solve()
    assert rg.solution.status == G.MAX_ITERS == ro.solution.status
    assert rg.solution.iterations == 100 and len(rg.residual_history) == 4
    assert rg.solution.rho_trace == ro.solution.rho_trace


# ---- MPC step protocol (bench.cpp:157-185): update_vectors + refresh_z + fixed_iters(k) ---------
@pytest.mark.parametrize("k", [1, 2, 15])
def test_closed_loop_protocol_matches_oracle(G, oracle, P, k):
    wl = P.config1(seed=3)
    base = wl.base_problem()
    gs, os_ = make_pair(oracle, G, base)
    gs2, _ = make_pair(oracle, G, base)
    x = wl.x0(1.0)
    A, B, K = wl.sys.A, wl.sys.B, wl.tmpl.K
    nu = wl.sys.nu
    for step in range(25):
        q = wl.problem_at(x)
        os_.update_vectors(q.g, q.c, q.d); os_.refresh_z(); ro = os_.fixed_iters(k)
        gs.update_vectors(q.g, q.c, q.d); gs.refresh_z(); rg = gs.fixed_iters(k)
        rf = gs2.mpc_step(q.g, q.c, q.d, k)          # fused single-launch step
        assert rg.solution.iterations == k == ro.solution.iterations
        assert rel_err(rg.solution.y, ro.solution.y) <= 1e-9
        assert rel_err(rg.solution.lam, ro.solution.lam) <= 1e-9
        assert abs(rg.solution.r_prim - ro.solution.r_prim) <= 1e-9 * max(1.0, ro.solution.r_prim)
        assert abs(rg.solution.r_dual - ro.solution.r_dual) <= 1e-9 * max(1.0, ro.solution.r_dual)
        assert np.array_equal(rf.solution.y, rg.solution.y)      # fused == 3 calls, bit for bit
        assert np.array_equal(rf.solution.lam, rg.solution.lam)
        assert rf.solution.r_prim == rg.solution.r_prim
        u = np.clip(-K @ x + ro.solution.y[:nu], -1.0, 1.0)
        x = A @ x + B @ u


@pytest.mark.parametrize("k", [1, 15])
def test_closed_loop_from_x0_on_device(G, oracle, P, k):
    """cqp_mpc_set_template + cqp_mpc_step_x0: instantiate (mpc.cpp:260-270) and the control
    extraction (bench.cpp:169-175) on the device; the step uploads x0 and downloads u0.  Against
    the oracle driven by the host-side instantiate, over a closed loop that hits the limits."""
    wl = P.config1(seed=3)
    base = wl.base_problem()
    gs, os_ = make_pair(oracle, G, base)
    gs.set_mpc_template(wl.tmpl, wl.limits)
    x = wl.x0(1.0)
    A, B, K, nu = wl.sys.A, wl.sys.B, wl.tmpl.K, wl.sys.nu
    clipped = 0
    for step in range(25):
        q = wl.problem_at(x)
        os_.update_vectors(q.g, q.c, q.d); os_.refresh_z(); ro = os_.fixed_iters(k)
        u_ref_raw = -K @ x + ro.solution.y[:nu]
        u_ref = np.clip(u_ref_raw, wl.limits.u_lo, wl.limits.u_hi)
        clipped += int(np.any(u_ref != u_ref_raw))
        u0, rg = gs.mpc_step_x0(x, k)
        assert rg.solution.iterations == k
        assert rel_err(rg.solution.y, ro.solution.y) <= 1e-9
        assert rel_err(rg.solution.lam, ro.solution.lam) <= 1e-9
        assert rel_err(rg.solution.z, ro.solution.z) <= 1e-9
        assert abs(rg.solution.r_prim - ro.solution.r_prim) <= 1e-9 * max(1.0, ro.solution.r_prim)
        assert np.abs(u0 - u_ref).max() <= 1e-9 * max(1.0, np.abs(u_ref).max())
        assert np.all(u0 >= wl.limits.u_lo) and np.all(u0 <= wl.limits.u_hi)
        x = A @ x + B @ u_ref
    assert clipped > 0                                   # the clamp in the control law was exercised
    # the device-side c, d are what the host-side instantiate produces
    sc = gs.scaling()
    Fv = os_.cache.F
    assert np.abs(sc["c_tilde"][base.n:base.n + base.m] - Fv * q.c).max() <= 1e-12 * max(1.0, np.abs(q.c).max())
    with pytest.raises(ValueError):
        gs.mpc_step_x0(np.zeros(3), k)


# ---- tiers ---------------------------------------------------------------------------------------
def test_all_kernel_modes_agree(G, oracle, P, monkeypatch):
    """tier 0 (all-SM grid, W in shared memory), tier 1 (W streamed from L2/HBM through a
    cp.async.bulk ring) and tier 2 (one thread-block cluster, DSMEM exchange;
    the default for small problems) sums each row in a different order: same counts, traces and
    history indices, values within rounding."""
    wl = P.config2(14, seed=2)
    base = wl.base_problem()
    q = wl.problem_at(wl.x0(10.0))
    reports = []
    for env, tier in (({"CQP_FORCE_TIER": "0"}, 0), ({"CQP_FORCE_TIER": "1"}, 1), ({}, 2),
                      ({"CQP_CLUSTER_SIZE": "8"}, 2)):
        monkeypatch.delenv("CQP_FORCE_TIER", raising=False)
        monkeypatch.delenv("CQP_CLUSTER_SIZE", raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s, os_ = make_pair(oracle, G, base)
        assert s.launch_info()["tier"] == tier
        s.update_vectors(q.g, q.c, q.d); s.cold_start()
        reports.append(s.solve())
        s.cold_start()
        s.fixed_iters(3)                       # few iterations: the W slice is streamed, same bits
        v3 = s.state
        s.cold_start()
        for _ in range(3):
            s.fixed_iters(1)
        assert np.array_equal(s.state, v3)
    monkeypatch.delenv("CQP_FORCE_TIER", raising=False)
    monkeypatch.delenv("CQP_CLUSTER_SIZE", raising=False)
    a, b, c, c8 = reports
    assert c8.solution.iterations == c.solution.iterations and rel_err(c8.solution.y, c.solution.y) <= 1e-9
    # tier 1 streams W through a shared-memory ring: each row is summed as 4 partials instead of 16
    assert b.solution.iterations == a.solution.iterations and b.solution.rho_trace == a.solution.rho_trace
    assert rel_err(b.solution.y, a.solution.y) <= 1e-9 and rel_err(b.solution.lam, a.solution.lam) <= 1e-9
    assert c.solution.iterations == a.solution.iterations and c.solution.rho_trace == a.solution.rho_trace
    assert [(h[0], h[3]) for h in c.residual_history] == [(h[0], h[3]) for h in a.residual_history]
    assert rel_err(c.solution.y, a.solution.y) <= 1e-9 and rel_err(c.solution.lam, a.solution.lam) <= 1e-9
    os_.update_vectors(q.g, q.c, q.d); os_.cold_start()
    ro = os_.solve()
    assert_report_parity(a, ro)
    assert_report_parity(b, ro)
    assert_report_parity(c, ro)


@pytest.mark.parametrize("n", [51, 201])
def test_structured_stream_layer_matches_dense_and_oracle(G, oracle, monkeypatch, n):
    """L2/HBM tier, structured layer: the lambda rows of W, [rho G, -diag(rho), I]
    (layers.cpp:159-161), are streamed as their first n columns and the two diagonal terms are
    added by the publisher.  Forced here on small problems (odd n: a column pair straddles the
    y / z boundary; equality rows: rho differs per row) and compared with the dense layer and the
    oracle: identical counts, traces, history indices; values within rounding."""
    p = oracle.gen_random_dense_qp(n, 3)
    monkeypatch.setenv("CQP_FORCE_TIER", "1")
    reports = []
    for env, want in ((("CQP_SINGLE_DENSE", "1"), 0), (("CQP_FORCE_STRUCTURED", "1"), 1)):
        monkeypatch.delenv("CQP_SINGLE_DENSE", raising=False)
        monkeypatch.delenv("CQP_FORCE_STRUCTURED", raising=False)
        monkeypatch.setenv(*env)
        gs, os_ = make_pair(oracle, G, p, from_layers=True)
        info = gs.launch_info()
        assert info["tier"] == 1 and info["structured"] == want
        D = p.n + 2 * p.m
        assert info["w_bytes_per_iteration"] == (8.0 * ((p.n + p.m) * D + p.m * p.n) if want else 8.0 * D * D)
        reports.append(gs.solve())
        gs.cold_start(); gs.fixed_iters(7); va = gs.state
        gs.cold_start(); gs.fixed_iters(3); gs.fixed_iters(4)
        assert np.array_equal(gs.state, va)
        gs.close()
    for k in ("CQP_FORCE_TIER", "CQP_SINGLE_DENSE", "CQP_FORCE_STRUCTURED"):
        monkeypatch.delenv(k, raising=False)
    dense, struct = reports
    ro = os_.solve()
    assert len(ro.solution.rho_trace) > 1 or n < 100   # the larger one switches rho
    assert_report_parity(dense, ro)
    assert_report_parity(struct, ro)
    assert struct.solution.iterations == dense.solution.iterations
    assert rel_err(struct.solution.y, dense.solution.y) <= 1e-9
    assert rel_err(struct.solution.lam, dense.solution.lam) <= 1e-9


def test_rho_rule_without_log10_takes_the_same_decisions(G, oracle, P, monkeypatch):
    """nearest_grid_index (layers.cpp:38-50) compares |log10(grid[k]) - log10(rho)|.  The kernels count the
    bounds sqrt(grid[k] grid[k+1]) below rho instead and fall back to the log10 comparison within 1e-9 of a
    bound or for a rho that is not a positive finite number; CQP_EXACT_LOG=1 always takes log10.  Same
    rho_trace, iteration count and bits on the rho-switching dense family and an MPC problem, in the
    cluster tier and on the all-SM grid."""
    cases = [(oracle.gen_random_dense_qp(120, seed), None) for seed in (1, 3)]      # 4 -> 2, 4 -> 1 at iteration 75
    for seed in range(4):                                                          # 4 -> 5 (-> 6) at 50 ... 550
        wl = P.config2(10, seed=seed)
        cases.append((wl.base_problem(), wl.problem_at(wl.x0(10.0))))
    switches = 0
    for tier in (None, "0"):
        for prob, q in cases:
            reps = []
            for exact in ("0", "1"):
                monkeypatch.setenv("CQP_EXACT_LOG", exact)
                if tier is not None:
                    monkeypatch.setenv("CQP_FORCE_TIER", tier)
                s = G.Solver(prob.H, prob.g, prob.G, prob.c, prob.d)
                if q is not None:
                    s.update_vectors(q.g, q.c, q.d)
                s.cold_start()
                reps.append(s.solve())
                s.close()
            a, b = reps
            assert a.solution.iterations == b.solution.iterations and a.solution.rho_trace == b.solution.rho_trace
            assert np.array_equal(a.solution.y, b.solution.y) and np.array_equal(a.solution.lam, b.solution.lam)
            switches += len(a.solution.rho_trace) - 1
    monkeypatch.delenv("CQP_EXACT_LOG", raising=False)
    monkeypatch.delenv("CQP_FORCE_TIER", raising=False)
    assert switches >= 12


@pytest.mark.parametrize("nu", [22, 30, 42])
def test_resident_tier_fetch_modes_are_bit_identical(G, oracle, P, monkeypatch, nu):
    """The shared-memory-resident tier can bring the iterate into a CTA three ways (CQP_COFETCH=0: loader
    warps, 1: loaders + compute warps, 2 = default: every compute thread polls for its own column pairs
    and keeps them -- and, where they fit, its columns of W_k -- in registers).  Same products, same
    summation order: the iterate after a fixed number of layers, a full solve with rho switches (which
    reload the register copy of W_k) and fused MPC steps are the same bits; the default also matches the
    oracle.  nu = 22 / 30: W_k in registers (4 / 8 rows per CTA); nu = 42: two column pairs per thread,
    W_k in shared memory."""
    wl = P.config2(nu, seed=1)
    base = wl.base_problem()
    q = wl.problem_at(wl.x0(10.0))
    q2 = wl.problem_at(wl.x0(3.0, seed=5))
    outs = []
    os_ = oracle.Solver(oracle.QProblem(base.H, base.g, base.G, base.c, base.d), oracle.SolverSettings(), variant="ref")
    layers = oracle_layers(os_.cache)
    for mode in ("2", "1", "0", "2w"):
        monkeypatch.setenv("CQP_COFETCH", mode[0])
        monkeypatch.setenv("CQP_WREG", "0" if mode.endswith("w") else "1")
        s = G.Solver(base.H, base.g, base.G, base.c, base.d, G.SolverSettings(), layers=layers)
        assert s.launch_info()["tier"] == 0
        s.update_vectors(q.g, q.c, q.d); s.cold_start()
        r = s.solve()
        s.cold_start(); s.fixed_iters(60)
        v60 = s.state.copy()
        steps = [s.mpc_step(q2.g, q2.c, q2.d, 2).solution.y.copy() for _ in range(3)]
        outs.append((r, v60, steps))
        s.close()
    monkeypatch.delenv("CQP_COFETCH", raising=False)
    monkeypatch.delenv("CQP_WREG", raising=False)
    r0, v0, st0 = outs[0]
    for r, v, st in outs[1:]:
        assert r.solution.iterations == r0.solution.iterations and r.solution.rho_trace == r0.solution.rho_trace
        assert np.array_equal(r.solution.y, r0.solution.y) and np.array_equal(r.solution.lam, r0.solution.lam)
        assert np.array_equal(v, v0)
        assert all(np.array_equal(a, b) for a, b in zip(st, st0))
    os_.update_vectors(q.g, q.c, q.d); os_.cold_start()
    assert_report_parity(r0, os_.solve())


@pytest.mark.parametrize("shape", ["odd_n_odd_m", "even_n_odd_m"])
def test_odd_dimensions_in_every_grid_mode(G, oracle, P, monkeypatch, shape):
    """n and m whose separately padded scratch vectors [uy; uz; ul] need MORE room than the padded
    iterate (npad + 2 mpad > Dpad): they alias the idle copy of the iterate in the grid kernel, so
    the copies are spaced by max(Dpad, npad + 2 mpad).  Checked against the oracle in the resident
    tier, the streamed tier with the dense and with the structured layer, and the cluster tier:
    cold solve (14 residual passes), then fused MPC steps (refresh_z + bias + iterations)."""
    import numpy as np
    from workloads import mpc
    if shape == "odd_n_odd_m":
        wl = P.make_mpc_workload(3, 6, 5, seed=2)                       # n = m = 15, D = 45
    else:
        lim = mpc.BoxLimits(np.full(2, -1.0), np.full(2, 1.0), np.full(5, -20.0), np.full(5, 20.0), x_rows=[0])
        wl = P.make_mpc_workload(2, 5, 5, seed=2, limits=lim)           # n = 10, m = 15, D = 40
    base = wl.base_problem()
    assert (base.n + base.n % 2) + 2 * (base.m + base.m % 2) > (base.n + 2 * base.m + (base.n + 2 * base.m) % 2)
    q = wl.problem_at(wl.x0(3.0))
    q2 = wl.problem_at(wl.x0(2.0, seed=7))
    envs = ({"CQP_FORCE_TIER": "0"}, {"CQP_FORCE_TIER": "1", "CQP_SINGLE_DENSE": "1"},
            {"CQP_FORCE_TIER": "1", "CQP_FORCE_STRUCTURED": "1"}, {})
    keys = ("CQP_FORCE_TIER", "CQP_SINGLE_DENSE", "CQP_FORCE_STRUCTURED")
    for env in envs:
        for k in keys:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        gs, os_ = make_pair(oracle, G, base)
        for s in (gs, os_):
            s.update_vectors(q.g, q.c, q.d); s.cold_start()
        assert_report_parity(gs.solve(), os_.solve())
        for _ in range(3):
            os_.update_vectors(q2.g, q2.c, q2.d); os_.refresh_z(); ro = os_.fixed_iters(3)
            rg = gs.mpc_step(q2.g, q2.c, q2.d, 3)
            assert rg.solution.iterations == 3 and rel_err(rg.solution.y, ro.solution.y) <= 1e-9
            assert rel_err(rg.solution.lam, ro.solution.lam) <= 1e-9 and rel_err(rg.solution.z, ro.solution.z) <= 1e-9
        gs.close()
    for k in keys:
        monkeypatch.delenv(k, raising=False)
