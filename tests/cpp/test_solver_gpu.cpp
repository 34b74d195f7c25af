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
  if (failures == 0) std::printf("ALL C++ HOST-MIRROR CHECKS PASSED\n");
  return failures == 0 ? 0 : 1;
}
