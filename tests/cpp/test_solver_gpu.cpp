// C++ host-side mirror of the reference's solver tests, run against the GPU Solver
// (paper_2311_18056_b200/csrc/host/clampqp_gpu.hpp over libcqp_b200.so).
// Each block names the reference test it restates (/root/reference/proj/tests/test_solver.cpp).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "clampqp_gpu.hpp"

using namespace clampqp;

static int failures = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) { std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); ++failures; } \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool ok__ = false;                                                       \
    try { expr; } catch (const type&) { ok__ = true; } catch (...) {}        \
    if (!ok__) { std::printf("FAIL %s:%d  %s should throw %s\n", __FILE__, __LINE__, #expr, #type); ++failures; } \
  } while (0)

static bool approx(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::fmax(std::fabs(a), std::fabs(b)); }

static QProblem box_1d() {  // test_solver.cpp:28-36
  QProblem p;
  p.H = Mat{{2.0}};
  p.g = Vec{-2.0};
  p.G = Mat{{1.0}};
  p.c = Vec{0.0};
  p.d = Vec{0.5};
  return p;
}

static SolverSettings tight_settings() {  // test_solver.cpp:38-44
  SolverSettings s;
  s.eps_prim = 1e-8;
  s.eps_dual = 1e-8;
  s.max_iters = 20000;
  return s;
}

int main() {
  // "solve reaches the KKT point of the three 1-D benchmarks"  test_solver.cpp:175-209
  {
    Solver solver(box_1d(), tight_settings());
    const Solution sol = solver.solve().solution;
    CHECK(sol.status == SolveStatus::Solved);
    CHECK(approx(sol.y[0], 0.5, 1e-6));
    CHECK(approx(sol.lambda[0], 1.0, 1e-6));
  }
  {
    QProblem p = box_1d();
    p.H = Mat{{1.0}}; p.g = Vec{0.0}; p.c = Vec{1.0}; p.d = Vec{1.0};
    Solver solver(p, tight_settings());
    const Solution sol = solver.solve().solution;
    CHECK(sol.status == SolveStatus::Solved);
    CHECK(approx(sol.y[0], 1.0, 1e-6));
    CHECK(approx(sol.lambda[0], -1.0, 1e-6));
  }
  {
    QProblem p = box_1d();
    p.c = Vec{-10.0}; p.d = Vec{10.0};
    Solver solver(p, tight_settings());
    const Solution sol = solver.solve().solution;
    CHECK(sol.status == SolveStatus::Solved);
    CHECK(approx(sol.y[0], 1.0, 1e-6));
    CHECK(std::fabs(sol.lambda[0]) < 1e-6);
  }
  // "residual history has one sample per check"  test_solver.cpp:378-388
  {
    SolverSettings s;
    s.adaptive_rho = false;
    Solver solver(box_1d(), s);
    const SolveReport report = solver.fixed_iters(100);
    CHECK(report.residual_history.size() == 4);
    for (size_t i = 0; i < report.residual_history.size(); ++i)
      CHECK(report.residual_history[i].iteration == 25 * static_cast<int>(i + 1));
    CHECK(report.solution.iterations == 100);
  }
  // "rho trace records the starting index and every switch"  test_solver.cpp:390-401
  {
    Solver solver(box_1d(), SolverSettings{});
    const Solution sol = solver.solve().solution;
    CHECK(!sol.rho_trace.empty());
    CHECK(sol.rho_trace.front().iteration == 0);
    CHECK(sol.rho_trace.front().grid_index == 4);  // 13-point grid starts at 0.1 (test_layers.cpp:89)
    for (size_t i = 1; i < sol.rho_trace.size(); ++i) {
      CHECK(sol.rho_trace[i].iteration % 25 == 0);
      CHECK(sol.rho_trace[i].grid_index != sol.rho_trace[i - 1].grid_index);
    }
    CHECK(solver.layer_index() == sol.rho_trace.back().grid_index);
  }
  // "identical solves are bit-for-bit identical"  test_solver.cpp:318-334
  {
    Solver a(box_1d(), SolverSettings{}), b(box_1d(), SolverSettings{});
    const SolveReport ra = a.solve(), rb = b.solve();
    CHECK(ra.solution.y[0] == rb.solution.y[0]);
    CHECK(ra.solution.lambda[0] == rb.solution.lambda[0]);
    CHECK(ra.solution.iterations == rb.solution.iterations);
    CHECK(ra.residual_history.size() == rb.residual_history.size());
    for (size_t i = 0; i < ra.residual_history.size() && i < rb.residual_history.size(); ++i) {
      CHECK(ra.residual_history[i].r_prim == rb.residual_history[i].r_prim);
      CHECK(ra.residual_history[i].r_dual == rb.residual_history[i].r_dual);
    }
  }
  // "settings and argument validation"  test_solver.cpp:362-376 (through the Solver)
  {
    SolverSettings bad;
    bad.check_interval = 0;
    CHECK_THROWS_AS(Solver(box_1d(), bad), std::invalid_argument);
    bad = SolverSettings{};
    bad.max_iters = 10;
    CHECK_THROWS_AS(Solver(box_1d(), bad), std::invalid_argument);
    Solver solver(box_1d());
    CHECK_THROWS_AS(solver.fixed_iters(0), std::invalid_argument);
    CHECK_THROWS_AS(solver.update_vectors(Vec{0.0, 1.0}, Vec{0.0}, Vec{1.0}), std::invalid_argument);
  }
  // validate error codes (tests/test_problem.cpp)
  {
    QProblem p = box_1d();
    p.H = Mat{{-1.0}};
    bool ok = false;
    try { Solver s(p); } catch (const ProblemError& e) { ok = e.code() == ProblemError::Code::NonPositiveDefiniteH; }
    CHECK(ok);
    p = box_1d();
    p.c = Vec{1.0}; p.d = Vec{0.0};
    ok = false;
    try { Solver s(p); } catch (const ProblemError& e) { ok = e.code() == ProblemError::Code::InvertedBounds; }
    CHECK(ok);
  }
  // MPC protocol: update_vectors + refresh_z + fixed_iters(k) == mpc_step, bit for bit
  {
    Solver a(box_1d()), b(box_1d());
    for (int t = 0; t < 5; ++t) {
      const Vec g{-2.0 + 0.1 * t}, c{0.0}, d{0.5 + 0.05 * t};
      a.update_vectors(g, c, d); a.refresh_z();
      const SolveReport ra = a.fixed_iters(2);
      const SolveReport rb = b.mpc_step(g, c, d, 2);
      CHECK(ra.solution.y[0] == rb.solution.y[0]);
      CHECK(ra.solution.lambda[0] == rb.solution.lambda[0]);
      CHECK(ra.solution.iterations == 2 && rb.solution.iterations == 2);
    }
  }
  // instantiate + control extraction on the device: a 1-D "template" with nx = 2
  //   g = offset_g x0, c = c_base - offset_c x0, d = d_base - offset_c x0, u0 = clamp(-K x0 + y)
  {
    Solver a(box_1d()), b(box_1d());
    const Mat og{{-1.0, 0.5}}, oc{{0.25, -0.125}}, K{{0.5, 0.25}};
    const Vec cb{0.0}, db{0.5}, ulo{-0.2}, uhi{0.3};
    b.set_mpc_template(og, oc, cb, db, K, ulo, uhi);
    for (int t = 0; t < 5; ++t) {
      const Vec x0{1.0 + 0.25 * t, -0.5 + 0.125 * t};   // dyadic values: the tiny dots are exact
      const double shift = 0.25 * x0[0] - 0.125 * x0[1];
      const Vec g{-1.0 * x0[0] + 0.5 * x0[1]}, c{0.0 - shift}, d{0.5 - shift};
      a.update_vectors(g, c, d); a.refresh_z();
      const SolveReport ra = a.fixed_iters(3);
      Vec u0;
      const SolveReport rb = b.mpc_step(x0, 3, &u0);
      CHECK(ra.solution.y[0] == rb.solution.y[0]);
      CHECK(ra.solution.lambda[0] == rb.solution.lambda[0]);
      double u = -(0.5 * x0[0] + 0.25 * x0[1]) + ra.solution.y[0];
      u = u < -0.2 ? -0.2 : (u > 0.3 ? 0.3 : u);
      CHECK(std::fabs(u0[0] - u) <= 1e-15);
    }
    CHECK_THROWS_AS(b.mpc_step(Vec{1.0}, 1, nullptr), std::invalid_argument);
  }
  // Solver::cache() read-back (solver.hpp:124) against the 1-D layer of test_layers.cpp:191-207:
  // H = 2, g = -2, G = 1, sigma = 0, rho = 1  =>  W = [[-1/3, 2/3, -1/3], [2/3, -1/3, 2/3], [1, -1, 1]], b = [2/3, 2/3, 0]
  {
    SolverSettings s;
    s.sigma = 0.0;
    s.equilibration.enabled = false;
    s.grid_points = 7;                      // decade grid 1e-3 .. 1e3: index 3 is rho = 1 (test_layers.cpp:62-91)
    Solver solver(box_1d(), s);
    const LayerCache cache = solver.cache();
    CHECK(cache.n() == 1 && cache.m() == 1 && cache.num_layers() == 7);
    CHECK(cache.initial_index() == 2);
    const std::vector<double> grid = cache.grid_values();
    CHECK(grid.size() == 7 && grid[0] == 1e-3 && grid[6] == 1e3 && approx(grid[3], 1.0, 1e-15));
    const Layer l = cache.layer(3);
    const double W[3][3] = {{-1.0 / 3, 2.0 / 3, -1.0 / 3}, {2.0 / 3, -1.0 / 3, 2.0 / 3}, {1.0, -1.0, 1.0}};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) CHECK(std::fabs(l.W(i, j) - W[i][j]) <= 1e-15);
    CHECK(std::fabs(l.b[0] - 2.0 / 3) <= 1e-15 && std::fabs(l.b[1] - 2.0 / 3) <= 1e-15 && l.b[2] == 0.0);
    CHECK(std::fabs(l.D(0, 0) - 1.0 / 3) <= 1e-15 && l.rho_vec[0] == grid[3] && l.rho_base == grid[3]);
    const Scaling sc = cache.scaling();
    CHECK(sc.E[0] == 1.0 && sc.F[0] == 1.0 && sc.cost_scale == 1.0);
    const Vec ct = cache.c_tilde(), dt = cache.d_tilde();  // test_layers.cpp:223-245: [-inf; c; -inf], [+inf; d; +inf]
    CHECK(ct[0] == -kInf && ct[1] == 0.0 && ct[2] == -kInf && dt[0] == kInf && dt[1] == 0.5 && dt[2] == kInf);
  }
  // free-standing solve / fixed_iters / warm_start on a cache (solver.hpp:81-97) == the Solver's own,
  // bit for bit, and a Solver that shares the cache keeps its iterate and vectors
  {
    const SolverSettings s = tight_settings();
    Solver solver(box_1d(), s);
    const SolveReport own = solver.solve();
    const Vec state_before = solver.state();
    const int index_before = solver.layer_index();
    const LayerCache cache = solver.cache();
    const SolveReport free_cold = solve(box_1d(), cache, s);
    CHECK(free_cold.solution.status == SolveStatus::Solved);
    CHECK(free_cold.solution.iterations == own.solution.iterations);
    CHECK(free_cold.solution.y[0] == own.solution.y[0] && free_cold.solution.lambda[0] == own.solution.lambda[0]);
    CHECK(free_cold.solution.rho_trace.size() == own.solution.rho_trace.size());
    // another problem on the same ladder (same H, G; other vectors), warm-started from the first solution
    QProblem q = box_1d();
    q.g = Vec{-1.5}; q.d = Vec{0.4};
    const SolveReport free_warm = solve(q, cache, s, &own.solution);
    Solver ref(q, s);
    ref.warm_start(own.solution);
    const SolveReport ref_warm = ref.solve();
    CHECK(free_warm.solution.iterations == ref_warm.solution.iterations);
    CHECK(free_warm.solution.y[0] == ref_warm.solution.y[0] && free_warm.solution.lambda[0] == ref_warm.solution.lambda[0]);
    CHECK(approx(free_warm.solution.y[0], 0.4, 1e-6));
    const SolveReport fi = fixed_iters(q, cache, s, 50);
    Solver ref2(q, s);
    const SolveReport fi_ref = ref2.fixed_iters(50);
    CHECK(fi.solution.iterations == 50 && fi.solution.y[0] == fi_ref.solution.y[0] && fi.residual_history.size() == 2);
    CHECK_THROWS_AS(fixed_iters(q, cache, s, 0), std::invalid_argument);
    // dims mismatch: a status, not an exception (solver.cpp:161)
    QProblem bad;
    bad.H = Mat{{1.0, 0.0}, {0.0, 1.0}}; bad.g = Vec{0.0, 0.0}; bad.G = Mat{{1.0, 0.0}}; bad.c = Vec{0.0}; bad.d = Vec{1.0};
    CHECK(solve(bad, cache, s).solution.status == SolveStatus::Invalid);
    // the Solver that shares the cache is where it was
    const Vec state_after = solver.state();
    CHECK(solver.layer_index() == index_before);
    for (Index i = 0; i < state_after.size(); ++i) CHECK(state_after[i] == state_before[i]);
    const SolveReport again = solver.fixed_iters(25);       // continues from its own iterate, own vectors
    Solver twin(box_1d(), s);
    twin.solve();
    const SolveReport twin_again = twin.fixed_iters(25);
    CHECK(again.solution.y[0] == twin_again.solution.y[0] && again.solution.lambda[0] == twin_again.solution.lambda[0]);
    // warm_start(prev, cache): the mapped iterate [y / E; G_s y_s; cost_scale lambda / F] and the last index
    const std::pair<Vec, int> ws = warm_start(own.solution, cache);
    CHECK(ws.second == own.solution.rho_trace.back().grid_index);
    ref.warm_start(own.solution);
    const Vec ref_state = ref.state();
    for (Index i = 0; i < ref_state.size(); ++i) CHECK(ws.first[i] == ref_state[i]);
  }
  // precompute_all + BatchSolver: column j == solve(p_j, cache, s)
  {
    const SolverSettings s = tight_settings();
    const LayerCache cache = precompute_all(box_1d(), s);
    const int B = 5;
    Mat g(1, B), c(1, B), d(1, B);
    for (int j = 0; j < B; ++j) { g(0, j) = -2.0 + 0.3 * j; c(0, j) = 0.0; d(0, j) = 0.5 + 0.1 * j; }
    BatchSolver batch(cache, 8);
    const BatchSolver::Result r = batch.solve(g, c, d);
    for (int j = 0; j < B; ++j) {
      QProblem q = box_1d();
      q.g = Vec{g(0, j)}; q.c = Vec{c(0, j)}; q.d = Vec{d(0, j)};
      const SolveReport one = solve(q, cache, s);
      CHECK(r.status[static_cast<size_t>(j)] == one.solution.status);
      CHECK(r.iterations[static_cast<size_t>(j)] == one.solution.iterations);
      CHECK(approx(r.y(0, j), one.solution.y[0], 1e-9) || std::fabs(r.y(0, j) - one.solution.y[0]) <= 1e-12);
      CHECK(r.rho_trace[static_cast<size_t>(j)].size() == one.solution.rho_trace.size());
      for (size_t i = 0; i < one.solution.rho_trace.size() && i < r.rho_trace[static_cast<size_t>(j)].size(); ++i) {
        CHECK(r.rho_trace[static_cast<size_t>(j)][i].iteration == one.solution.rho_trace[i].iteration);
        CHECK(r.rho_trace[static_cast<size_t>(j)][i].grid_index == one.solution.rho_trace[i].grid_index);
      }
    }
    CHECK_THROWS_AS(batch.solve(Mat(2, 1), c, d), std::invalid_argument);
  }
  if (failures == 0) std::printf("ALL C++ HOST-MIRROR CHECKS PASSED\n");
  return failures == 0 ? 0 : 1;
}
