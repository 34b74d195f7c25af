// clampqp_gpu.hpp -- the reference's public solver API (clampqp::Solver and its value types,
// /root/reference/proj/include/clampqp/solver.hpp:29-135, problem.hpp:31-92) re-hosted on the
// B200 C ABI (include/cqp_b200.h).  Same class, method names, argument meaning and exception
// behaviour; the private part is an opaque GPU handle instead of a LayerCache + iterate.
//
// With Eigen available (`-DCLAMPQP_GPU_USE_EIGEN`, as in the reference's own build) Mat/Vec are
// the reference's aliases (types.hpp:22-24) and this header is source compatible with code
// written against clampqp/solver.hpp.  Without Eigen (this image) a minimal column-major
// Mat/Vec pair with the same element access is used.
//
// Header only; link with libcqp_b200.so.
#pragma once

#include <cmath>
#include <cstddef>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "cqp_b200.h"

#ifdef CLAMPQP_GPU_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace clampqp {

#ifdef CLAMPQP_GPU_USE_EIGEN
using Mat = Eigen::MatrixXd;
using Vec = Eigen::VectorXd;
using Index = Eigen::Index;
#else
using Index = std::ptrdiff_t;

/// Minimal stand-in for Eigen::VectorXd.
class Vec {
 public:
  Vec() = default;
  explicit Vec(Index n) : d_(static_cast<size_t>(n), 0.0) {}
  Vec(std::initializer_list<double> v) : d_(v) {}
  static Vec Zero(Index n) { return Vec(n); }
  static Vec Constant(Index n, double v) { Vec r(n); for (auto& x : r.d_) x = v; return r; }
  Index size() const { return static_cast<Index>(d_.size()); }
  double& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return d_[static_cast<size_t>(i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  void resize(Index n) { d_.assign(static_cast<size_t>(n), 0.0); }
 private:
  std::vector<double> d_;
};

/// Minimal stand-in for Eigen::MatrixXd (column-major, types.hpp:22).
class Mat {
 public:
  Mat() = default;
  Mat(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  Mat(std::initializer_list<std::initializer_list<double>> rows) {
    r_ = static_cast<Index>(rows.size());
    c_ = r_ ? static_cast<Index>(rows.begin()->size()) : 0;
    d_.assign(static_cast<size_t>(r_ * c_), 0.0);
    Index i = 0;
    for (const auto& row : rows) { Index j = 0; for (double v : row) (*this)(i, j++) = v; ++i; }
  }
  static Mat Zero(Index r, Index c) { return Mat(r, c); }
  static Mat Identity(Index r, Index c) { Mat m(r, c); for (Index i = 0; i < (r < c ? r : c); ++i) m(i, i) = 1.0; return m; }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};
#endif

inline constexpr double kInf = std::numeric_limits<double>::infinity();  // types.hpp:26

/// problem.hpp:31-40
struct QProblem {
  Mat H;
  Vec g;
  Mat G;
  Vec c;
  Vec d;
  Index num_vars() const { return H.rows(); }
  Index num_constraints() const { return G.rows(); }
};

enum class SolveStatus { Solved, MaxIters, Invalid };  // problem.hpp:51

/// problem.hpp:57-60
struct RhoSwitch {
  int iteration = 0;
  int grid_index = 0;
};

/// problem.hpp:62-71
struct Solution {
  Vec y;
  Vec z;
  Vec lambda;
  SolveStatus status = SolveStatus::Invalid;
  int iterations = 0;
  double r_prim = 0.0;
  double r_dual = 0.0;
  std::vector<RhoSwitch> rho_trace;
};

/// problem.hpp:73-92
class ProblemError : public std::runtime_error {
 public:
  enum class Code { DimensionMismatch, NonSymmetricH, NonPositiveDefiniteH, InvertedBounds, NonFiniteEntry, MalformedDocument, MissingField };
  ProblemError(Code code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Code code() const { return code_; }
 private:
  Code code_;
};

/// layers.hpp:100-104
struct Equilibration {
  bool enabled = true;
  int max_passes = 10;
  double tol = 1e-3;
};

/// solver.hpp:43-53
struct SolverSettings {
  double eps_prim = 1e-6;
  double eps_dual = 1e-6;
  int check_interval = 25;
  int max_iters = 4000;
  double sigma = 1e-6;
  int grid_points = 13;
  double rho_switch_threshold = 5.0;
  bool adaptive_rho = true;
  Equilibration equilibration{};
};

/// solver.hpp:56-61
struct ResidualSample {
  int iteration = 0;
  double r_prim = 0.0;
  double r_dual = 0.0;
  int grid_index = 0;
};

/// solver.hpp:63-67 (+ the CUDA-event time of the persistent kernel)
struct SolveReport {
  Solution solution;
  double wall_ms = 0.0;
  std::vector<ResidualSample> residual_history;
  double kernel_us = 0.0;
};

/// Error thrown when the CUDA runtime fails; there is no CPU fallback to fall back to.
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
/// cqp_status -> the reference's exception types.
inline void check(int rc) {
  if (rc == CQP_OK) return;
  const std::string msg = cqp_last_error();
  switch (rc) {
    case CQP_ERR_DIMENSION: throw ProblemError(ProblemError::Code::DimensionMismatch, msg);
    case CQP_ERR_NONSYMMETRIC_H: throw ProblemError(ProblemError::Code::NonSymmetricH, msg);
    case CQP_ERR_NOT_PD_H: throw ProblemError(ProblemError::Code::NonPositiveDefiniteH, msg);
    case CQP_ERR_INVERTED_BOUNDS: throw ProblemError(ProblemError::Code::InvertedBounds, msg);
    case CQP_ERR_NONFINITE: throw ProblemError(ProblemError::Code::NonFiniteEntry, msg);
    case CQP_ERR_SETTINGS:
    case CQP_ERR_ARGUMENT: throw std::invalid_argument(msg);
    case CQP_ERR_FACTORIZATION: throw std::runtime_error(msg);
    default: throw CudaError(msg);
  }
}
inline cqp_settings to_c(const SolverSettings& s) {
  cqp_settings c;
  c.eps_prim = s.eps_prim; c.eps_dual = s.eps_dual;
  c.check_interval = s.check_interval; c.max_iters = s.max_iters;
  c.sigma = s.sigma; c.grid_points = s.grid_points;
  c.rho_switch_threshold = s.rho_switch_threshold; c.adaptive_rho = s.adaptive_rho ? 1 : 0;
  c.eq_enabled = s.equilibration.enabled ? 1 : 0; c.eq_max_passes = s.equilibration.max_passes;
  c.eq_tol = s.equilibration.tol;
  return c;
}
}  // namespace detail

/// GPU clampqp::Solver (solver.hpp:107-135).  Build once, then solve() or, per MPC step,
/// update_vectors + refresh_z + fixed_iters (or the fused mpc_step).
class Solver {
 public:
  explicit Solver(QProblem p, SolverSettings settings = {}, int device = -1)
      : problem_(std::move(p)), settings_(settings) {
    const Index n = problem_.H.rows(), m = problem_.G.rows();
    if (n < 1 || m < 1 || problem_.H.cols() != n || problem_.g.size() != n || problem_.G.cols() != n ||
        problem_.c.size() != m || problem_.d.size() != m) {
      throw ProblemError(ProblemError::Code::DimensionMismatch, "inconsistent problem dimensions");
    }
    const cqp_settings cs = detail::to_c(settings_);
    detail::check(cqp_create(&h_, static_cast<int>(n), static_cast<int>(m), problem_.H.data(),
                             problem_.g.data(), problem_.G.data(), problem_.c.data(),
                             problem_.d.data(), &cs, device));
  }
  ~Solver() { cqp_destroy(h_); }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  Solver(Solver&& o) noexcept : problem_(std::move(o.problem_)), settings_(o.settings_), h_(o.h_) { o.h_ = nullptr; }

  void cold_start() { detail::check(cqp_cold_start(h_)); }
  void warm_start(const Solution& prev) {
    if (prev.y.size() != problem_.num_vars() || prev.lambda.size() != problem_.num_constraints()) {
      throw std::invalid_argument("warm_start: dimension mismatch");
    }
    const int last = prev.rho_trace.empty() ? -1 : prev.rho_trace.back().grid_index;
    detail::check(cqp_warm_start(h_, prev.y.data(), prev.lambda.data(), last));
  }
  void refresh_z() { detail::check(cqp_refresh_z(h_)); }

  SolveReport solve() { return run(0, nullptr, nullptr, nullptr); }
  SolveReport fixed_iters(int k) {
    if (k < 1) throw std::invalid_argument("fixed_iters: k must be >= 1");
    return run(k, nullptr, nullptr, nullptr);
  }
  void update_vectors(const Vec& g, const Vec& c, const Vec& d) {
    if (g.size() != problem_.num_vars() || c.size() != problem_.num_constraints() ||
        d.size() != problem_.num_constraints()) {
      throw std::invalid_argument("update_vectors: dimension mismatch");
    }
    detail::check(cqp_update_vectors(h_, g.data(), c.data(), d.data()));
    problem_.g = g; problem_.c = c; problem_.d = d;
  }
  /// update_vectors + refresh_z + fixed_iters(k) as one upload and one launch (bench.cpp:157-167).
  SolveReport mpc_step(const Vec& g, const Vec& c, const Vec& d, int k) {
    if (k < 1) throw std::invalid_argument("mpc_step: k must be >= 1");
    if (g.size() != problem_.num_vars() || c.size() != problem_.num_constraints() ||
        d.size() != problem_.num_constraints()) {
      throw std::invalid_argument("mpc_step: dimension mismatch");
    }
    problem_.g = g; problem_.c = c; problem_.d = d;
    return run(k, g.data(), c.data(), d.data());
  }

  const QProblem& problem() const { return problem_; }
  const SolverSettings& settings() const { return settings_; }
  /// state(): the stacked iterate v = [y; z; lambda] in the cache's space (solver.hpp:126).
  Vec state() const {
    Vec v(problem_.num_vars() + 2 * problem_.num_constraints());
    detail::check(cqp_get_state(h_, v.data(), nullptr));
    return v;
  }
  int layer_index() const {
    int idx = 0;
    detail::check(cqp_get_state(h_, nullptr, &idx));
    return idx;
  }
  cqp_handle* native_handle() { return h_; }

  /// Condensed-MPC template on the device (mpc.hpp CondensedTemplate fields + BoxLimits):
  /// afterwards mpc_step(x0, k, &u0) instantiates the step QP (mpc.cpp:260-270) and extracts the
  /// control (bench.cpp:169-175) on the device; a step uploads x0 and downloads u0.
  void set_mpc_template(const Mat& offset_g, const Mat& offset_c, const Vec& c_base, const Vec& d_base,
                        const Mat& K, const Vec& u_lo, const Vec& u_hi) {
    const Index nx = offset_g.cols(), nu = K.rows();
    if (offset_g.rows() != problem_.num_vars() || offset_c.rows() != problem_.num_constraints() ||
        offset_c.cols() != nx || K.cols() != nx || c_base.size() != problem_.num_constraints() ||
        d_base.size() != c_base.size() || u_lo.size() != nu || u_hi.size() != nu) {
      throw std::invalid_argument("set_mpc_template: dimension mismatch");
    }
    detail::check(cqp_mpc_set_template(h_, static_cast<int>(nx), static_cast<int>(nu), offset_g.data(),
                                       offset_c.data(), c_base.data(), d_base.data(), K.data(), u_lo.data(),
                                       u_hi.data()));
    mpc_nx_ = nx; mpc_nu_ = nu;
  }
  SolveReport mpc_step(const Vec& x0, int k, Vec* u0) {
    if (k < 1) throw std::invalid_argument("mpc_step: k must be >= 1");
    if (mpc_nx_ == 0 || x0.size() != mpc_nx_) throw std::invalid_argument("mpc_step: x0 dimension mismatch");
    if (u0) *u0 = Vec(mpc_nu_);
    return run(k, nullptr, nullptr, nullptr, x0.data(), u0 ? u0->data() : nullptr);
  }

 private:
  SolveReport run(int k, const double* g, const double* c, const double* d, const double* x0 = nullptr,
                  double* u0 = nullptr) {
    const Index n = problem_.num_vars(), m = problem_.num_constraints();
    const int total = k > 0 ? k : settings_.max_iters;
    const int cap = total / settings_.check_interval + 2;
    SolveReport rep;
    rep.solution.y = Vec(n); rep.solution.z = Vec(m); rep.solution.lambda = Vec(m);
    std::vector<cqp_rho_switch> trace(static_cast<size_t>(cap));
    std::vector<cqp_residual_sample> hist(static_cast<size_t>(cap));
    cqp_result r{};
    r.y = rep.solution.y.data(); r.z = rep.solution.z.data(); r.lambda = rep.solution.lambda.data();
    r.rho_trace = trace.data(); r.rho_trace_cap = cap;
    r.history = hist.data(); r.history_cap = cap;
    if (x0) detail::check(cqp_mpc_step_x0(h_, x0, k, u0, &r));
    else if (g) detail::check(cqp_mpc_step(h_, g, c, d, k, &r));
    else if (k > 0) detail::check(cqp_fixed_iters(h_, k, &r));
    else detail::check(cqp_solve(h_, &r));
    rep.solution.status = r.status == CQP_SOLVED ? SolveStatus::Solved
                          : r.status == CQP_MAX_ITERS ? SolveStatus::MaxIters : SolveStatus::Invalid;
    rep.solution.iterations = r.iterations;
    rep.solution.r_prim = r.r_prim; rep.solution.r_dual = r.r_dual;
    for (int i = 0; i < r.rho_trace_len && i < cap; ++i) rep.solution.rho_trace.push_back({trace[i].iteration, trace[i].grid_index});
    for (int i = 0; i < r.history_len && i < cap; ++i) rep.residual_history.push_back({hist[i].iteration, hist[i].r_prim, hist[i].r_dual, hist[i].grid_index});
    rep.wall_ms = r.wall_ms; rep.kernel_us = r.kernel_us;
    return rep;
  }

  QProblem problem_;
  SolverSettings settings_;
  cqp_handle* h_ = nullptr;
  Index mpc_nx_ = 0, mpc_nu_ = 0;
};

}  // namespace clampqp
