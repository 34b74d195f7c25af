/*
 * cqp_b200.h -- C ABI of the B200-native ReLU-QP ("clampqp") solve path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types.  Each entry
 * point names the reference interface it replaces (paths under /root/reference/proj).  The
 * reference has no FFI of its own; its boundary for this path is the public C++ `Solver`
 * API (include/clampqp/solver.hpp:107-135), so the entry points are exactly what a
 * `clampqp::Solver` whose private part is a GPU handle has to call.  INTEGRATION.md shows that
 * binding; paper_2311_18056_b200/csrc/clampqp_gpu.hpp is a worked copy of it.
 *
 * Conventions
 *   - All matrices are column-major doubles (Eigen::MatrixXd layout, types.hpp:22).
 *   - The caller owns every host buffer; a handle owns its device memory and one stream.
 *   - Return value: CQP_OK or a cqp_status error; cqp_last_error() gives the message.
 *     The C++ wrapper maps them onto the reference's exception types.
 *   - One handle = one mutable iterate (like clampqp::Solver it is not thread-safe);
 *     separate handles may be driven from separate threads.
 *   - There is NO CPU fallback behind this boundary: without a CUDA device every call that
 *     needs one returns CQP_ERR_CUDA.
 */
#ifndef CQP_B200_H_
#define CQP_B200_H_

#ifdef __cplusplus
extern "C" {
#endif

#define CQP_API __attribute__((visibility("default")))

typedef enum {
  CQP_OK = 0,
  CQP_ERR_DIMENSION = 1,        /* -> ProblemError::DimensionMismatch / std::invalid_argument */
  CQP_ERR_NONSYMMETRIC_H = 2,   /* -> ProblemError::NonSymmetricH        (problem.cpp:140-144) */
  CQP_ERR_NOT_PD_H = 3,         /* -> ProblemError::NonPositiveDefiniteH (problem.cpp:146-149) */
  CQP_ERR_INVERTED_BOUNDS = 4,  /* -> ProblemError::InvertedBounds       (problem.cpp:157-161) */
  CQP_ERR_NONFINITE = 5,        /* -> ProblemError::NonFiniteEntry       (problem.cpp:136-138) */
  CQP_ERR_SETTINGS = 6,         /* -> std::invalid_argument              (solver.cpp:29-34)    */
  CQP_ERR_FACTORIZATION = 7,    /* -> std::runtime_error                 (layers.cpp:127-129)  */
  CQP_ERR_ARGUMENT = 8,         /* -> std::invalid_argument (k < 1, null pointers, ...)        */
  CQP_ERR_CUDA = 9,             /* CUDA runtime failure or no device: there is no CPU path    */
  CQP_ERR_CAPACITY = 10         /* problem does not fit the device / batch capacity            */
} cqp_status;

/* SolveStatus, problem.hpp:51 */
enum { CQP_SOLVED = 0, CQP_MAX_ITERS = 1, CQP_INVALID = 2 };

/* SolverSettings + Equilibration, solver.hpp:43-53 / layers.hpp:100-104 (same defaults). */
typedef struct {
  double eps_prim;
  double eps_dual;
  int check_interval;
  int max_iters;
  double sigma;
  int grid_points;
  double rho_switch_threshold;
  int adaptive_rho;
  int eq_enabled;
  int eq_max_passes;
  double eq_tol;
} cqp_settings;

/* RhoSwitch, problem.hpp:57-60 */
typedef struct {
  int iteration;
  int grid_index;
} cqp_rho_switch;

/* ResidualSample, solver.hpp:56-61 */
typedef struct {
  int iteration;
  double r_prim;
  double r_dual;
  int grid_index;
} cqp_residual_sample;

/* SolveReport + Solution, solver.hpp:63-67 / problem.hpp:62-71.
 * The caller provides y (n), z (m), lambda (m) and the two record arrays with their
 * capacities; *_len receive the number of records the solve produced (records beyond the
 * capacity are dropped, the length still counts them). */
typedef struct {
  double *y;
  double *z;
  double *lambda;
  cqp_rho_switch *rho_trace;
  int rho_trace_cap;
  int rho_trace_len;
  cqp_residual_sample *history;
  int history_cap;
  int history_len;
  int status;      /* CQP_SOLVED / CQP_MAX_ITERS / CQP_INVALID */
  int iterations;
  double r_prim;
  double r_dual;
  double wall_ms;   /* host clock around the call: launch + kernel + result download; the
                       reference's wall_ms region (solver.cpp:46,101-103) */
  double kernel_us; /* CUDA-event time of the persistent solve kernel alone */
} cqp_result;

typedef struct cqp_handle cqp_handle;

CQP_API void cqp_default_settings(cqp_settings *s);
CQP_API const char *cqp_last_error(void);
CQP_API int cqp_device_count(void);

/* Solver::Solver(QProblem, SolverSettings), solver.cpp:180-186: validate, check settings,
 * build the 13-point grid, run the offline stage (layers.cpp:189-228: Ruiz equilibration,
 * per-grid-point D = (H + sigma I + G' rho G)^-1 and W) ON THE DEVICE, cold-start.
 * `device` is the CUDA ordinal (-1: current device). */
CQP_API int cqp_create(cqp_handle **out, int n, int m, const double *H, const double *g,
                       const double *G, const double *c, const double *d,
                       const cqp_settings *settings, int device);

/* Same, but with the offline stage already done by the caller (e.g. the reference's own
 * precompute_all on the host): a LayerCache (layers.hpp:108-127) handed over field by field.
 * W[k]: (n+2m)^2, Dk[k]: n x n, GDk[k]: m x n for k < L; grid_values: L; H, g, G, c, d: the
 * ORIGINAL (unscaled) problem; Gs: cache.problem.G (scaled, m x n); E (n), F (m), cost_scale:
 * cache.scaling. */
CQP_API int cqp_create_from_layers(cqp_handle **out, int n, int m, int L,
                                   const double *const *W, const double *const *Dk,
                                   const double *const *GDk, const double *grid_values,
                                   int initial_index, const double *H, const double *g,
                                   const double *G, const double *c, const double *d,
                                   const double *Gs, const double *E, const double *F,
                                   double cost_scale, const cqp_settings *settings, int device);

CQP_API void cqp_destroy(cqp_handle *h);

/* Solver::update_vectors, solver.cpp:213-218 -> LayerCache::update_vectors, layers.cpp:177-187.
 * g (n), c (m), d (m) in ORIGINAL units.  Rescaling and the bias rebuild run on the device. */
CQP_API int cqp_update_vectors(cqp_handle *h, const double *g, const double *c, const double *d);

/* Solver::cold_start, solver.cpp:188-191 */
CQP_API int cqp_cold_start(cqp_handle *h);

/* Solver::warm_start(prev), solver.cpp:193-195 -> warm_start(), solver.cpp:144-156.
 * y (n), lambda (m) in original units; layer_index = prev.rho_trace.back().grid_index, or -1
 * for an empty trace (-> grid.initial_index). */
CQP_API int cqp_warm_start(cqp_handle *h, const double *y, const double *lambda,
                           int layer_index);

/* Solver::refresh_z, solver.cpp:197-200 */
CQP_API int cqp_refresh_z(cqp_handle *h);

/* Solver::solve, solver.cpp:202-205: run_loop(early_exit = true, total = max_iters) as ONE
 * persistent cooperative kernel; continues from the handle's iterate. */
CQP_API int cqp_solve(cqp_handle *h, cqp_result *out);

/* Solver::fixed_iters(k), solver.cpp:207-211: run_loop(early_exit = false, total = k). */
CQP_API int cqp_fixed_iters(cqp_handle *h, int k, cqp_result *out);

/* One receding-horizon control step (bench.cpp:157-167) as a single upload + single launch:
 * update_vectors(g, c, d); refresh_z(); fixed_iters(k).  Results are identical to the three
 * separate calls. */
CQP_API int cqp_mpc_step(cqp_handle *h, const double *g, const double *c, const double *d,
                         int k, cqp_result *out);

/* Condensed-MPC template on the device: mpc::instantiate (mpc.cpp:260-270) and the control
 * extraction of the closed loop (bench.cpp:169-175) move behind the boundary, so that a control
 * step uploads x0 (nx doubles) instead of g, c, d (n + 2m doubles) and downloads u0.
 * offset_g: n x nx, offset_c: m x nx, K: nu x nx (column-major, CondensedTemplate fields,
 * mpc.hpp); c_base, d_base: m; u_lo, u_hi: nu (BoxLimits).  nu <= n. */
CQP_API int cqp_mpc_set_template(cqp_handle *h, int nx, int nu, const double *offset_g,
                                 const double *offset_c, const double *c_base,
                                 const double *d_base, const double *K, const double *u_lo,
                                 const double *u_hi);

/* One receding-horizon control step from the measured state (bench.cpp:157-175):
 *   p = instantiate(tmpl, x0); update_vectors(p.g, p.c, p.d); refresh_z(); fixed_iters(k);
 *   u0 = clamp(-K x0 + y[0:nu], u_lo, u_hi)
 * all on the device.  u0 (nu) and out may be NULL. */
CQP_API int cqp_mpc_step_x0(cqp_handle *h, const double *x0, int k, double *u0, cqp_result *out);

/* Resident control-step server for the closed loop of bench.cpp:157-185 (the reference calls
 * instantiate / update_vectors / refresh_z / fixed_iters(k) once per control step; at kHz rates the
 * GPU port of that loop is bound by launch and synchronisation overhead, not by the step itself).
 * cqp_mpc_server_start launches ONE persistent kernel that keeps W_k, the scaling vectors and the
 * residual rows on the SMs and serves steps from a host-mapped mailbox; while it is enabled,
 * cqp_mpc_step_x0(h, x0, k, ...) posts x0 there and spins on the answer: no CUDA call per step, results
 * bit-identical to the launch-per-step path.  The kernel leaves by itself when idle for
 * idle_timeout_ms (<= 0: 100 ms) -- the next step restarts it -- and every other entry point of the
 * handle retires it first, so the API keeps its meaning; it occupies the SMs it runs on (one 16-CTA
 * cluster for small QPs, every SM otherwise) while it is resident.  nx <= 128. */
CQP_API int cqp_mpc_server_start(cqp_handle *h, int k, double idle_timeout_ms);
CQP_API int cqp_mpc_server_stop(cqp_handle *h);
/* Last step served by the resident kernel: wall time inside cqp_mpc_step_x0 and the device-side
 * duration (request seen -> answer written), both in microseconds.  With out == NULL the step
 * returns u0 only and skips the final residual evaluation of solver.cpp:94-95 (its results would not
 * be observable); the iterate and u0 are the same bits either way. */
CQP_API int cqp_mpc_server_last_timing(const cqp_handle *h, double *wall_us, double *device_us);

/* Solver::state() / layer_index(), solver.hpp:126-127: v (n+2m, cache space) and the index. */
CQP_API int cqp_get_state(cqp_handle *h, double *v, int *layer_index);

/* The inverse of cqp_get_state: the persistent iterate (cache space, n+2m) and the ladder index a
 * free-standing solve(p, cache, s, warm) / fixed_iters(...) of solver.hpp:86-97 starts from or hands
 * back (the host mirror saves and restores a Solver's iterate around those calls). */
CQP_API int cqp_set_state(cqp_handle *h, const double *v, int layer_index);

/* Solver::cache() read-back (solver.hpp:124) for one grid point; any pointer may be NULL.
 * W (n+2m)^2, Dk n*n, GDk m*n column-major; b (n+2m) for the CURRENT g; rho_vec (m). */
CQP_API int cqp_get_layer(cqp_handle *h, int k, double *W, double *Dk, double *GDk, double *b,
                          double *rho_vec);

/* cache().scaling / grid / clamp bounds: E (n), F (m), cost_scale (1), grid (L), c_tilde and
 * d_tilde (n+2m); any pointer may be NULL. */
CQP_API int cqp_get_scaling(cqp_handle *h, double *E, double *F, double *cost_scale,
                            double *grid, int *initial_index, double *c_tilde,
                            double *d_tilde);

CQP_API int cqp_dims(const cqp_handle *h, int *n, int *m, int *L);

/* Diagnostics: the 256-int host-mapped watchdog record of the persistent kernel (word 0 != 0
 * after a watchdog trap: 1 = where, 2 = iteration, 3 = CTA, 4 = thread; words 64.. hold the
 * optional -DCQP_TRACE timeline). */
CQP_API int cqp_debug_words(const cqp_handle *h, int *out256);

/* How the persistent kernel was configured: CTAs, rows of W per CTA, tier (0: all-SM grid, W
 * slice resident in shared memory; 1: all-SM grid, W streamed from L2/HBM; 2: one thread-block
 * cluster, W resident, iterate exchanged through distributed shared memory), dynamic shared
 * memory bytes. */
CQP_API int cqp_launch_info(const cqp_handle *h, int *ctas, int *rows_per_cta, int *tier,
                            int *smem_bytes);

/* Bytes of W_k one iteration of the persistent kernel reads (the roofline numerator of the
 * matvec path): 8 D^2 for the dense layer (solver.cpp:60); the L2/HBM tier streams the lambda rows
 * [rho G, -diag(rho), I] (layers.cpp:159-161) as their first n columns only, 8 ((n+m) D + m n),
 * and reports structured = 1. */
CQP_API int cqp_layer_traffic(const cqp_handle *h, double *w_bytes_per_iteration, int *structured);

/* Measurement helper for roofline denominators (bench.py): rate at which all SMs read a device
 * buffer of `bytes` bytes `passes` times with 16-byte loads, 8 in flight per thread.  A buffer
 * much larger than the 126 MB L2 gives the HBM read rate, one that fits it the L2 read rate. */
CQP_API int cqp_measure_read_bandwidth(int device, unsigned long long bytes, int passes,
                                       double *gb_per_s);

/* Page-locked host memory for the caller's input / output buffers (cudaMallocHost / cudaFreeHost):
 * copies from and to pinned buffers run at full PCIe rate and asynchronously; pageable buffers
 * are staged by the driver.  Optional: every entry point accepts any host pointer. */
CQP_API int cqp_pinned_alloc(void **out, unsigned long long bytes);
CQP_API void cqp_pinned_free(void *p);

/* ---- batched path: many QPs sharing (H, G) and therefore the W ladder ---------------------
 * (MPC instances that differ in x0, i.e. in g, c, d).  Semantically B independent
 * `solve()` calls from a cold start (solver.cpp:158-166), one per column. */
typedef struct cqp_batch cqp_batch;

CQP_API int cqp_batch_create(cqp_batch **out, cqp_handle *shared, int capacity);
CQP_API void cqp_batch_destroy(cqp_batch *b);

/* g_cols: n x B, c_cols/d_cols: m x B (column-major, original units).  Outputs, any may be
 * NULL: y_cols n x B, z_cols m x B, lambda_cols m x B, status/iterations/final_index (B),
 * r_prim/r_dual (B), n_switches (B).  device_ms: CUDA-event time of the whole batch solve.
 * Every input / output array may live in host memory (pageable or pinned) OR in the handle's
 * device memory (unified addressing decides): a caller that gathers results across GPUs passes
 * device buffers and hands them to its collective without a host round trip. */
CQP_API int cqp_batch_solve(cqp_batch *b, int B, const double *g_cols, const double *c_cols,
                            const double *d_cols, double *y_cols, double *z_cols,
                            double *lambda_cols, int *status, int *iterations,
                            int *final_index, double *r_prim, double *r_dual, int *n_switches,
                            double *device_ms);

/* Per-column Solution::rho_trace (problem.hpp:57-70; entry 0 is {0, start index}, solver.cpp:50)
 * of the LAST cqp_batch_solve (B must equal that call's B).  trace: B x cap records, column j at
 * trace + j * cap; trace_len (B): records column j produced (records beyond `cap` are dropped, the
 * length still counts them).  Either pointer may be NULL.  cap >= max_iters / check_interval + 2
 * holds every possible trace. */
CQP_API int cqp_batch_get_traces(cqp_batch *b, int B, int cap, cqp_rho_switch *trace,
                                 int *trace_len);

/* Per-column SolveReport::residual_history (solver.hpp:56-67: one sample per convergence check,
 * grid_index = the index BEFORE that check's switch) of the last cqp_batch_solve; same layout. */
CQP_API int cqp_batch_get_history(cqp_batch *b, int B, int cap, cqp_residual_sample *history,
                                  int *history_len);

/* CUDA-event times of the last cqp_batch_solve: compute_ms = from "inputs resident in HBM" to
 * "results ready in HBM"; total_ms additionally covers the host->device and device->host
 * copies; launches = kernels launched by the solve. */
CQP_API int cqp_batch_last_timing(const cqp_batch *b, double *compute_ms, double *total_ms,
                                  long long *launches);

/* Iteration-GEMM profile of the last cqp_batch_solve: gemm_ms = CUDA-event time spent in the
 * iteration GEMM launches, gemm_flops = the algorithmic flops they carried (2 D^2 per active
 * column per iteration), rounds = check rounds executed. */
CQP_API int cqp_batch_last_profile(const cqp_batch *b, double *gemm_ms, double *gemm_flops,
                                   int *rounds);

/* Per check round of the last solve (up to `cap` rounds): active columns during the round and
 * the CUDA-event time of its iteration GEMM launches. */
CQP_API int cqp_batch_round_profile(const cqp_batch *b, int cap, int *active, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* CQP_B200_H_ */
