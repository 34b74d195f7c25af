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
#include <memory>
#include <mutex>
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

/// layers.hpp:87-98: one ladder point as `Solver::cache().layer(k)` hands it back (host copies).
struct Layer {
  Mat W;        // (n+2m) x (n+2m)
  Mat D;        // n x n
  Mat GD;       // m x n
  Vec b;        // n+2m, for the cache's current g
  Vec rho_vec;  // m
  double rho_base = 0.0;
};

/// layers.hpp:52-60
struct Scaling {
  Vec E, F;
  double cost_scale = 1.0;
};

/// layers.hpp:111-127 on the device.  The ladder (13 x W_k, D_k, G D_k, scaling, grid) lives in HBM
/// inside a cqp_handle; this object shares that handle (with the Solver it came from, or on its own
/// when built by precompute_all) and reads pieces back on demand.  Calls that use the handle are
/// serialised by a mutex, so concurrent free-standing solves on one cache are safe.
class LayerCache {
 public:
  LayerCache() = default;
  Index n() const { return sh_ ? sh_->n : 0; }
  Index m() const { return sh_ ? sh_->m : 0; }
  int num_layers() const { return sh_ ? sh_->L : 0; }
  Layer layer(int k) const {
    require();
    if (k < 0 || k >= sh_->L) throw std::out_of_range("LayerCache::layer");
    const Index nn = sh_->n, mm = sh_->m, D = nn + 2 * mm;
    Layer l;
    l.W = Mat(D, D); l.D = Mat(nn, nn); l.GD = Mat(mm, nn); l.b = Vec(D); l.rho_vec = Vec(mm);
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_get_layer(sh_->h, k, l.W.data(), l.D.data(), l.GD.data(), l.b.data(), l.rho_vec.data()));
    l.rho_base = grid_values_locked()[static_cast<size_t>(k)];
    return l;
  }
  Scaling scaling() const {
    require();
    Scaling sc;
    sc.E = Vec(sh_->n); sc.F = Vec(sh_->m);
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_get_scaling(sh_->h, sc.E.data(), sc.F.data(), &sc.cost_scale, nullptr, nullptr, nullptr, nullptr));
    return sc;
  }
  /// PenaltyGrid (layers.hpp:27-50): values and the index a cold start uses
  std::vector<double> grid_values() const { require(); std::lock_guard<std::mutex> lock(sh_->mu); return grid_values_locked(); }
  int initial_index() const {
    require();
    int idx = 0;
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_get_scaling(sh_->h, nullptr, nullptr, nullptr, nullptr, &idx, nullptr, nullptr));
    return idx;
  }
  Vec c_tilde() const { return bounds(true); }
  Vec d_tilde() const { return bounds(false); }

  struct Shared {
    cqp_handle* h = nullptr;
    std::mutex mu;
    Index n = 0, m = 0;
    int L = 0;
    Vec g, c, d;               // the vectors the handle currently holds (original units) ...
    bool vectors_known = true;  // ... unless the device-side instantiate (mpc_step from x0) set them
    ~Shared() { cqp_destroy(h); }
  };
  explicit LayerCache(std::shared_ptr<Shared> sh) : sh_(std::move(sh)) {}
  const std::shared_ptr<Shared>& shared() const { return sh_; }

 private:
  void require() const { if (!sh_ || !sh_->h) throw std::invalid_argument("LayerCache: empty"); }
  std::vector<double> grid_values_locked() const {
    std::vector<double> g(static_cast<size_t>(sh_->L));
    detail::check(cqp_get_scaling(sh_->h, nullptr, nullptr, nullptr, g.data(), nullptr, nullptr, nullptr));
    return g;
  }
  Vec bounds(bool lower) const {
    require();
    Vec v(sh_->n + 2 * sh_->m);
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_get_scaling(sh_->h, nullptr, nullptr, nullptr, nullptr, nullptr, lower ? v.data() : nullptr, lower ? nullptr : v.data()));
    return v;
  }
  std::shared_ptr<Shared> sh_;
};

namespace detail {
inline std::shared_ptr<LayerCache::Shared> make_shared_handle(const QProblem& p, const SolverSettings& s, int device) {
  const Index n = p.H.rows(), m = p.G.rows();
  if (n < 1 || m < 1 || p.H.cols() != n || p.g.size() != n || p.G.cols() != n || p.c.size() != m || p.d.size() != m) {
    throw ProblemError(ProblemError::Code::DimensionMismatch, "inconsistent problem dimensions");
  }
  auto sh = std::make_shared<LayerCache::Shared>();
  const cqp_settings cs = to_c(s);
  check(cqp_create(&sh->h, static_cast<int>(n), static_cast<int>(m), p.H.data(), p.g.data(), p.G.data(), p.c.data(),
                   p.d.data(), &cs, device));
  sh->n = n; sh->m = m;
  sh->g = p.g; sh->c = p.c; sh->d = p.d;
  int nn = 0, mm = 0;
  check(cqp_dims(sh->h, &nn, &mm, &sh->L));
  return sh;
}
}  // namespace detail

/// Offline stage on the device (layers.cpp:189-228): equilibrate, then every grid point's (W, b, D).
inline LayerCache precompute_all(const QProblem& p, const SolverSettings& s = {}, int device = -1) {
  return LayerCache(detail::make_shared_handle(p, s, device));
}

/// GPU clampqp::Solver (solver.hpp:107-135).  Build once, then solve() or, per MPC step,
/// update_vectors + refresh_z + fixed_iters (or the fused mpc_step).
class Solver {
 public:
  explicit Solver(QProblem p, SolverSettings settings = {}, int device = -1)
      : problem_(std::move(p)), settings_(settings) {
    sh_ = detail::make_shared_handle(problem_, settings_, device);
    h_ = sh_->h;
  }
  ~Solver() = default;  // (the handle goes with the last owner: this Solver or a cache() copy)
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  Solver(Solver&& o) noexcept
      : problem_(std::move(o.problem_)), settings_(o.settings_), sh_(std::move(o.sh_)), h_(o.h_), mpc_nx_(o.mpc_nx_), mpc_nu_(o.mpc_nu_) {
    o.h_ = nullptr;
  }

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
    sh_->g = g; sh_->c = c; sh_->d = d; sh_->vectors_known = true;
  }
  /// update_vectors + refresh_z + fixed_iters(k) as one upload and one launch (bench.cpp:157-167).
  SolveReport mpc_step(const Vec& g, const Vec& c, const Vec& d, int k) {
    if (k < 1) throw std::invalid_argument("mpc_step: k must be >= 1");
    if (g.size() != problem_.num_vars() || c.size() != problem_.num_constraints() ||
        d.size() != problem_.num_constraints()) {
      throw std::invalid_argument("mpc_step: dimension mismatch");
    }
    problem_.g = g; problem_.c = c; problem_.d = d;
    sh_->g = g; sh_->c = c; sh_->d = d; sh_->vectors_known = true;
    return run(k, g.data(), c.data(), d.data());
  }

  const QProblem& problem() const { return problem_; }
  const SolverSettings& settings() const { return settings_; }
  /// cache() (solver.hpp:124): the ladder this Solver iterates on, shared (not copied: 13 levels of
  /// W are 0.2 - 2 GB); read pieces back with layer(k), scaling(), grid_values(), c_tilde()...
  LayerCache cache() const { return LayerCache(sh_); }
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
    sh_->vectors_known = false;  // (g, c, d now come from the device-side instantiate)
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
  std::shared_ptr<LayerCache::Shared> sh_;
  cqp_handle* h_ = nullptr;
  Index mpc_nx_ = 0, mpc_nu_ = 0;
};

// ---- free-standing online stage (solver.hpp:81-97) ----------------------------------------------
namespace detail {
/// Runs `k` iterations (k == 0: solve to tolerance) on the cache's device ladder from a cold start
/// or from `warm`, for the problem vectors of `p`.  The handle's own iterate, ladder index and
/// vectors (a Solver may share it) are saved before and restored afterwards.
inline SolveReport run_on_cache(const QProblem& p, const LayerCache& cache, const SolverSettings& s, int k,
                                const Solution* warm) {
  SolveReport rep;
  const auto& sh = cache.shared();
  const Index n = cache.n(), m = cache.m();
  if (!sh || p.H.rows() != n || p.G.rows() != m || p.g.size() != n || p.c.size() != m || p.d.size() != m ||
      (warm && (warm->y.size() != n || warm->lambda.size() != m))) {
    rep.solution.status = SolveStatus::Invalid;  // solver.cpp:161: a status, not an exception
    return rep;
  }
  std::lock_guard<std::mutex> lock(sh->mu);
  cqp_handle* h = sh->h;
  const Index D = n + 2 * m;
  Vec saved(D);
  int saved_idx = 0;
  check(cqp_get_state(h, saved.data(), &saved_idx));
  check(cqp_update_vectors(h, p.g.data(), p.c.data(), p.d.data()));
  if (warm) {
    const int last = warm->rho_trace.empty() ? -1 : warm->rho_trace.back().grid_index;
    check(cqp_warm_start(h, warm->y.data(), warm->lambda.data(), last));
  } else {
    check(cqp_cold_start(h));
  }
  const int total = k > 0 ? k : s.max_iters;
  const int cap = total / s.check_interval + 2;
  rep.solution.y = Vec(n); rep.solution.z = Vec(m); rep.solution.lambda = Vec(m);
  std::vector<cqp_rho_switch> trace(static_cast<size_t>(cap));
  std::vector<cqp_residual_sample> hist(static_cast<size_t>(cap));
  cqp_result r{};
  r.y = rep.solution.y.data(); r.z = rep.solution.z.data(); r.lambda = rep.solution.lambda.data();
  r.rho_trace = trace.data(); r.rho_trace_cap = cap; r.history = hist.data(); r.history_cap = cap;
  check(k > 0 ? cqp_fixed_iters(h, k, &r) : cqp_solve(h, &r));
  rep.solution.status = r.status == CQP_SOLVED ? SolveStatus::Solved : r.status == CQP_MAX_ITERS ? SolveStatus::MaxIters : SolveStatus::Invalid;
  rep.solution.iterations = r.iterations; rep.solution.r_prim = r.r_prim; rep.solution.r_dual = r.r_dual;
  for (int i = 0; i < r.rho_trace_len && i < cap; ++i) rep.solution.rho_trace.push_back({trace[i].iteration, trace[i].grid_index});
  for (int i = 0; i < r.history_len && i < cap; ++i) rep.residual_history.push_back({hist[i].iteration, hist[i].r_prim, hist[i].r_dual, hist[i].grid_index});
  rep.wall_ms = r.wall_ms; rep.kernel_us = r.kernel_us;
  // put the shared handle back: vectors (unless a device-side instantiate owns them), iterate, index
  if (sh->vectors_known) check(cqp_update_vectors(h, sh->g.data(), sh->c.data(), sh->d.data()));
  check(cqp_set_state(h, saved.data(), saved_idx));
  return rep;
}
}  // namespace detail

/// solver.hpp:86-88.  The settings that shaped the ladder (sigma, grid, equilibration) are the
/// cache's; eps / max_iters / check_interval / adaptive_rho of `s` must equal the ones the cache was
/// built with (they live in the handle): pass the same SolverSettings.
inline SolveReport solve(const QProblem& p, const LayerCache& cache, const SolverSettings& s,
                         const Solution* warm = nullptr) {
  return detail::run_on_cache(p, cache, s, 0, warm);
}
/// solver.hpp:92-94
inline SolveReport fixed_iters(const QProblem& p, const LayerCache& cache, const SolverSettings& s, int k,
                               const Solution* warm = nullptr) {
  if (k < 1) throw std::invalid_argument("fixed_iters: k must be >= 1");
  return detail::run_on_cache(p, cache, s, k, warm);
}
/// solver.hpp:81: v = [y / E; G_s (y / E); cost_scale * lambda / F] in the cache's space and the grid
/// index the previous solve ended on (the cache's initial index when prev has no trace).
inline std::pair<Vec, int> warm_start(const Solution& prev, const LayerCache& cache) {
  const auto& sh = cache.shared();
  if (!sh || prev.y.size() != cache.n() || prev.lambda.size() != cache.m()) throw std::invalid_argument("warm_start: dimension mismatch");
  std::lock_guard<std::mutex> lock(sh->mu);
  const Index D = cache.n() + 2 * cache.m();
  Vec saved(D), v(D);
  int saved_idx = 0, idx = 0;
  detail::check(cqp_get_state(sh->h, saved.data(), &saved_idx));
  const int last = prev.rho_trace.empty() ? -1 : prev.rho_trace.back().grid_index;
  detail::check(cqp_warm_start(sh->h, prev.y.data(), prev.lambda.data(), last));
  detail::check(cqp_get_state(sh->h, v.data(), &idx));
  detail::check(cqp_set_state(sh->h, saved.data(), saved_idx));
  return {v, idx};
}

/// Batched path (include/cqp_b200.h cqp_batch_*): B QPs that share (H, G) -- hence the cache's ladder --
/// and differ in (g, c, d); column j of the result is what solve(p_j, cache, s) returns.
class BatchSolver {
 public:
  BatchSolver(const LayerCache& cache, int capacity) : sh_(cache.shared()), capacity_(capacity) {
    if (!sh_) throw std::invalid_argument("BatchSolver: empty cache");
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_batch_create(&b_, sh_->h, capacity));
  }
  ~BatchSolver() { cqp_batch_destroy(b_); }
  BatchSolver(const BatchSolver&) = delete;
  BatchSolver& operator=(const BatchSolver&) = delete;

  struct Result {
    Mat y, z, lambda;                       // n x B, m x B, m x B
    std::vector<SolveStatus> status;
    std::vector<int> iterations;
    std::vector<double> r_prim, r_dual;
    std::vector<std::vector<RhoSwitch>> rho_trace;
    double device_ms = 0.0;
  };
  /// g: n x B, c / d: m x B (column-major, original units)
  Result solve(const Mat& g, const Mat& c, const Mat& d, int max_trace = 0) {
    const Index n = sh_->n, m = sh_->m, B = g.cols();
    if (g.rows() != n || c.rows() != m || d.rows() != m || c.cols() != B || d.cols() != B || B < 1 || B > capacity_) {
      throw std::invalid_argument("BatchSolver::solve: dimension mismatch");
    }
    Result r;
    r.y = Mat(n, B); r.z = Mat(m, B); r.lambda = Mat(m, B);
    std::vector<int> st(static_cast<size_t>(B)), fin(static_cast<size_t>(B)), nsw(static_cast<size_t>(B));
    r.iterations.assign(static_cast<size_t>(B), 0); r.r_prim.assign(static_cast<size_t>(B), 0.0); r.r_dual.assign(static_cast<size_t>(B), 0.0);
    std::lock_guard<std::mutex> lock(sh_->mu);
    detail::check(cqp_batch_solve(b_, static_cast<int>(B), g.data(), c.data(), d.data(), r.y.data(), r.z.data(), r.lambda.data(),
                                  st.data(), r.iterations.data(), fin.data(), r.r_prim.data(), r.r_dual.data(), nsw.data(), &r.device_ms));
    for (int v : st) r.status.push_back(v == CQP_SOLVED ? SolveStatus::Solved : v == CQP_MAX_ITERS ? SolveStatus::MaxIters : SolveStatus::Invalid);
    int cap = max_trace;
    if (cap <= 0) { cap = 2; for (int v : nsw) cap = v + 2 > cap ? v + 2 : cap; }
    std::vector<cqp_rho_switch> tr(static_cast<size_t>(B) * cap);
    std::vector<int> len(static_cast<size_t>(B));
    detail::check(cqp_batch_get_traces(b_, static_cast<int>(B), cap, tr.data(), len.data()));
    r.rho_trace.resize(static_cast<size_t>(B));
    for (Index j = 0; j < B; ++j)
      for (int i = 0; i < len[static_cast<size_t>(j)] && i < cap; ++i)
        r.rho_trace[static_cast<size_t>(j)].push_back({tr[static_cast<size_t>(j) * cap + i].iteration, tr[static_cast<size_t>(j) * cap + i].grid_index});
    return r;
  }

 private:
  std::shared_ptr<LayerCache::Shared> sh_;
  cqp_batch* b_ = nullptr;
  int capacity_ = 0;
};

}  // namespace clampqp
