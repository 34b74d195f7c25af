/*
 * clampqp_oracle.c -- CPU restatement of the reference ReLU-QP ("clampqp") solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2311_18056_b200/ links, loads or calls this
 * file.  It is used by tests/, by __graft_entry__.smoke() as the checker, and by bench.py's
 * cpu_baseline / --impl reference leg as the CPU implementation that is timed.
 *
 * PARITY STATUS: the reference cannot be compiled in this image (Eigen and its vendor/
 * headers are absent), so this restatement is pinned against every known-answer value the
 * reference's own tests hold for this path (tests/test_oracle_known_answers.py lists them with
 * reference file:line).  Iteration counts and rho-switch sequences on non-trivial problems are
 * not pinned by any reference test ("parity unpinned" for those two quantities).
 *
 * Every function cites the reference file:line it follows (paths under /root/reference/proj).
 * Storage is column-major, like Eigen::MatrixXd (include/clampqp/types.hpp:22):
 *   A(i,j) == a[i + j*rows].
 *
 * Plain C11, no dependencies beyond libm.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------------
 * small dense helpers (stand-ins for the Eigen expressions the reference uses)
 * ---------------------------------------------------------------------------------------- */

static double *dalloc(size_t count) {
  double *p = (double *)calloc(count ? count : 1, sizeof(double));
  return p;
}

/* C(rows x cols) += A(rows x inner) * B(inner x cols), all column-major. */
static void gemm_nn_acc(int rows, int inner, int cols, const double *A, const double *B,
                        double *C) {
  for (int j = 0; j < cols; ++j) {
    double *cj = C + (size_t)j * rows;
    for (int k = 0; k < inner; ++k) {
      const double bkj = B[k + (size_t)j * inner];
      if (bkj == 0.0) continue;
      const double *ak = A + (size_t)k * rows;
      for (int i = 0; i < rows; ++i) cj[i] += ak[i] * bkj;
    }
  }
}

/* C(rows x cols) = A * B */
static void gemm_nn(int rows, int inner, int cols, const double *A, const double *B, double *C) {
  memset(C, 0, sizeof(double) * (size_t)rows * cols);
  gemm_nn_acc(rows, inner, cols, A, B, C);
}

/* At(cols x rows) = A(rows x cols)^T */
static void transpose(int rows, int cols, const double *A, double *At) {
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) At[j + (size_t)i * cols] = A[i + (size_t)j * rows];
}

/* y(rows) = A(rows x cols) * x, column-axpy order (the order a column-major GEMV walks). */
static void gemv_n(int rows, int cols, const double *A, const double *x, double *y) {
  for (int i = 0; i < rows; ++i) y[i] = 0.0;
  for (int j = 0; j < cols; ++j) {
    const double xj = x[j];
    const double *aj = A + (size_t)j * rows;
    for (int i = 0; i < rows; ++i) y[i] += aj[i] * xj;
  }
}

/* y(cols) = A(rows x cols)^T * x, one dot product per column. */
static void gemv_t(int rows, int cols, const double *A, const double *x, double *y) {
  for (int j = 0; j < cols; ++j) {
    const double *aj = A + (size_t)j * rows;
    double acc = 0.0;
    for (int i = 0; i < rows; ++i) acc += aj[i] * x[i];
    y[j] = acc;
  }
}

/* types.hpp:34-37  inf_norm(Vec): max |v_i|, 0 for empty. */
static double vec_inf_norm(int len, const double *v) {
  double best = 0.0;
  for (int i = 0; i < len; ++i) {
    const double a = fabs(v[i]);
    if (a > best) best = a;
    if (a != a) return a; /* NaN propagates like Eigen's maxCoeff on NaN input (unspecified) */
  }
  return best;
}

/* types.hpp:29-32  inf_norm(Mat): max absolute row sum. */
static double mat_inf_norm(int rows, int cols, const double *a) {
  double best = 0.0;
  for (int i = 0; i < rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < cols; ++j) s += fabs(a[i + (size_t)j * rows]);
    if (s > best) best = s;
  }
  return best;
}

/* In-place lower Cholesky of a (n x n, column-major). Returns 0 on success, 1 when a pivot is
 * not strictly positive (Eigen::LLT reports NumericalIssue in that case; layers.cpp:126-129,
 * problem.cpp:146-149). */
static int cholesky_lower(int n, double *a) {
  for (int j = 0; j < n; ++j) {
    double diag = a[j + (size_t)j * n];
    for (int k = 0; k < j; ++k) {
      const double l = a[j + (size_t)k * n];
      diag -= l * l;
    }
    if (!(diag > 0.0)) return 1;
    const double ljj = sqrt(diag);
    a[j + (size_t)j * n] = ljj;
    /* column j below the diagonal: a[i,j] = (a[i,j] - sum_k l[i,k] l[j,k]) / ljj */
    for (int k = 0; k < j; ++k) {
      const double ljk = a[j + (size_t)k * n];
      if (ljk == 0.0) continue;
      const double *colk = a + (size_t)k * n;
      double *colj = a + (size_t)j * n;
      for (int i = j + 1; i < n; ++i) colj[i] -= colk[i] * ljk;
    }
    const double inv = 1.0 / ljj;
    for (int i = j + 1; i < n; ++i) a[i + (size_t)j * n] *= inv;
  }
  return 0;
}

/* X = (L L^T)^{-1} given the lower factor L (only the lower triangle of l is read). */
static void cholesky_inverse(int n, const double *l, double *x) {
  /* Solve L Y = I column by column, then L^T X = Y. */
  for (int c = 0; c < n; ++c) {
    double *col = x + (size_t)c * n;
    for (int i = 0; i < n; ++i) col[i] = (i == c) ? 1.0 : 0.0;
    /* forward substitution (column-oriented); entries above c stay zero */
    for (int k = c; k < n; ++k) {
      const double yk = col[k] / l[k + (size_t)k * n];
      col[k] = yk;
      if (yk == 0.0) continue;
      const double *lk = l + (size_t)k * n;
      for (int i = k + 1; i < n; ++i) col[i] -= lk[i] * yk;
    }
    /* back substitution with L^T (row-oriented dot products over column k of L) */
    for (int k = n - 1; k >= 0; --k) {
      const double *lk = l + (size_t)k * n;
      double acc = col[k];
      for (int i = k + 1; i < n; ++i) acc -= lk[i] * col[i];
      col[k] = acc / lk[k];
    }
  }
}

/* ------------------------------------------------------------------------------------------
 * bench::Rng  (include/clampqp/bench.hpp:29-47, src/bench.cpp:58-87)
 * std::mt19937_64 is bit-specified by the C++ standard; restated here so that streams match.
 * ---------------------------------------------------------------------------------------- */

#define MT_NN 312
#define MT_MM 156

typedef struct {
  uint64_t mt[MT_NN];
  int idx;
  int has_spare;
  double spare;
} orc_rng;

ORC_API void orc_rng_seed(orc_rng *r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_NN;
  r->has_spare = 0;
  r->spare = 0.0;
}

ORC_API uint64_t orc_rng_next_u64(orc_rng *r) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < MT_NN - 1; ++i) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (r->mt[MT_NN - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* bench.hpp:36  uniform(): top 53 bits scaled by 2^-53. */
ORC_API double orc_rng_uniform(orc_rng *r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* bench.hpp:37 */
ORC_API double orc_rng_uniform_range(orc_rng *r, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_uniform(r);
}

/* bench.cpp:58-73  Box-Muller with a cached spare. */
ORC_API double orc_rng_normal(orc_rng *r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  do {
    u1 = orc_rng_uniform(r);
  } while (u1 <= 0.0);
  const double u2 = orc_rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 6.283185307179586 * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}

/* bench.cpp:75-79 */
ORC_API void orc_rng_normal_vector(orc_rng *r, int len, double *out) {
  for (int i = 0; i < len; ++i) out[i] = orc_rng_normal(r);
}

/* bench.cpp:81-87  filled row by row (i outer, j inner) into a column-major matrix. */
ORC_API void orc_rng_normal_matrix(orc_rng *r, int rows, int cols, double *out) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out[i + (size_t)j * rows] = orc_rng_normal(r);
}

ORC_API int orc_rng_sizeof(void) { return (int)sizeof(orc_rng); }

/* bench.cpp:89-118  gen_random_dense_qp.  m = 2*floor(n/4) rows: first half equalities.
 * Outputs: H(n x n), g(n), G(m x n), c(m), d(m), witness(n, may be NULL). Returns m, or -1. */
ORC_API int orc_gen_random_dense_qp(int n, uint64_t seed, double *H, double *g, double *G,
                                    double *c, double *d, double *witness) {
  if (n < 4) return -1;
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  double *M = dalloc((size_t)n * n);
  double *Mt = dalloc((size_t)n * n);
  orc_rng_normal_matrix(&rng, n, n, M);
  transpose(n, n, M, Mt);
  gemm_nn(n, n, n, Mt, M, H); /* M'M */
  for (int i = 0; i < n; ++i) H[i + (size_t)i * n] += 0.1;
  /* p.H = 0.5 * (p.H + p.H') */
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < j; ++i) {
      const double s = 0.5 * (H[i + (size_t)j * n] + H[j + (size_t)i * n]);
      H[i + (size_t)j * n] = s;
      H[j + (size_t)i * n] = s;
    }
  orc_rng_normal_vector(&rng, n, g);
  const int n_side = n / 4;
  const int m = 2 * n_side;
  double *y0 = dalloc((size_t)n);
  double *gy0 = dalloc((size_t)m);
  orc_rng_normal_vector(&rng, n, y0);
  orc_rng_normal_matrix(&rng, m, n, G);
  gemv_n(m, n, G, y0, gy0);
  for (int i = 0; i < n_side; ++i) {
    c[i] = gy0[i];
    d[i] = gy0[i];
  }
  for (int i = n_side; i < m; ++i) {
    const double slack = fabs(orc_rng_normal(&rng)) + 0.1;
    c[i] = gy0[i] - slack;
    d[i] = gy0[i] + slack;
  }
  if (witness) memcpy(witness, y0, sizeof(double) * (size_t)n);
  free(M);
  free(Mt);
  free(y0);
  free(gy0);
  return m;
}

/* ------------------------------------------------------------------------------------------
 * problem.cpp:121-164  validate.  Returns 0 when valid, else 1 + ProblemError::Code
 * (problem.hpp:75-83): 1 DimensionMismatch, 2 NonSymmetricH, 3 NonPositiveDefiniteH,
 * 4 InvertedBounds, 5 NonFiniteEntry.
 * ---------------------------------------------------------------------------------------- */
static int all_finite(size_t count, const double *a) {
  for (size_t i = 0; i < count; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

ORC_API int orc_validate(int n, int m, const double *H, const double *g, const double *G,
                         const double *c, const double *d) {
  if (n < 1) return 1;
  if (m < 1) return 1;
  if (!all_finite((size_t)n * n, H)) return 5;
  if (!all_finite((size_t)n, g)) return 5;
  if (!all_finite((size_t)m * n, G)) return 5;
  const double h_norm = mat_inf_norm(n, n, H);
  const double h_scale = h_norm > 1.0 ? h_norm : 1.0;
  double asym = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double a = fabs(H[i + (size_t)j * n] - H[j + (size_t)i * n]);
      if (a > asym) asym = a;
    }
  if (asym > 1e-12 * h_scale) return 2;
  double *l = dalloc((size_t)n * n);
  memcpy(l, H, sizeof(double) * (size_t)n * n);
  const int bad = cholesky_lower(n, l);
  free(l);
  if (bad) return 3;
  for (int i = 0; i < m; ++i) {
    const double lo = c[i], hi = d[i];
    if (isnan(lo) || isnan(hi)) return 5;
    if (lo == INFINITY || hi == -INFINITY || lo > hi) return 4;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * layers.cpp:22-50  penalty grid
 * ---------------------------------------------------------------------------------------- */

/* layers.cpp:38-50 */
ORC_API int orc_nearest_grid_index(const double *values, int L, double rho) {
  const double target = log10(rho);
  int best = 0;
  double best_dist = INFINITY;
  for (int k = 0; k < L; ++k) {
    const double dist = fabs(log10(values[k]) - target);
    if (dist < best_dist - 1e-15) {
      best = k;
      best_dist = dist;
    }
  }
  return best;
}

/* layers.cpp:22-36.  Returns initial_index, or -1 when n_points < 2 (reference throws). */
ORC_API int orc_build_penalty_grid(int n_points, double *values) {
  if (n_points < 2) return -1;
  const double lo = -3.0, hi = 3.0;
  for (int k = 0; k < n_points; ++k) {
    const double t = lo + (hi - lo) * k / (n_points - 1);
    values[k] = pow(10.0, t);
  }
  values[0] = 1e-3;
  values[n_points - 1] = 1e3;
  return orc_nearest_grid_index(values, n_points, 0.1);
}

/* ------------------------------------------------------------------------------------------
 * layers.cpp:52-120  Scaling + Ruiz
 * ---------------------------------------------------------------------------------------- */

/* layers.cpp:60-69  Scaling::apply. */
static void scaling_apply(int n, int m, const double *E, const double *F, double cs,
                          const double *H, const double *g, const double *G, const double *c,
                          const double *d, double *Hs, double *gs, double *Gs, double *cs_out,
                          double *ds_out) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      Hs[i + (size_t)j * n] = cs * ((E[i] * H[i + (size_t)j * n]) * E[j]);
  for (int i = 0; i < n; ++i) gs[i] = cs * (E[i] * g[i]);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) Gs[i + (size_t)j * m] = (F[i] * G[i + (size_t)j * m]) * E[j];
  for (int i = 0; i < m; ++i) {
    cs_out[i] = F[i] * c[i];
    ds_out[i] = F[i] * d[i];
  }
}

/* layers.cpp:82-120  ruiz_equilibrate: computes E, F, cost_scale from H and G only. */
ORC_API void orc_ruiz_scaling(int n, int m, const double *H_in, const double *G_in,
                              int max_passes, double tol, double *E, double *F,
                              double *cost_scale) {
  double *H = dalloc((size_t)n * n);
  double *G = dalloc((size_t)m * n);
  double *delta = dalloc((size_t)n + m);
  memcpy(H, H_in, sizeof(double) * (size_t)n * n);
  memcpy(G, G_in, sizeof(double) * (size_t)m * n);
  for (int i = 0; i < n; ++i) E[i] = 1.0;
  for (int i = 0; i < m; ++i) F[i] = 1.0;

  for (int pass = 0; pass < max_passes; ++pass) {
    for (int i = 0; i < n; ++i) {
      double rh = 0.0, rg = 0.0;
      for (int j = 0; j < n; ++j) {
        const double a = fabs(H[i + (size_t)j * n]);
        if (a > rh) rh = a;
      }
      for (int k = 0; k < m; ++k) {
        const double a = fabs(G[k + (size_t)i * m]);
        if (a > rg) rg = a;
      }
      const double r = rh > rg ? rh : rg;
      delta[i] = r > 0.0 ? 1.0 / sqrt(r) : 1.0;
    }
    for (int i = 0; i < m; ++i) {
      double r = 0.0;
      for (int j = 0; j < n; ++j) {
        const double a = fabs(G[i + (size_t)j * m]);
        if (a > r) r = a;
      }
      delta[n + i] = r > 0.0 ? 1.0 / sqrt(r) : 1.0;
    }
    const double *dE = delta, *dF = delta + n;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        H[i + (size_t)j * n] = (dE[i] * H[i + (size_t)j * n]) * dE[j];
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i)
        G[i + (size_t)j * m] = (dF[i] * G[i + (size_t)j * m]) * dE[j];
    for (int i = 0; i < n; ++i) E[i] = E[i] * dE[i];
    for (int i = 0; i < m; ++i) F[i] = F[i] * dF[i];

    double change = 0.0;
    for (int i = 0; i < n + m; ++i) {
      const double a = fabs(delta[i] - 1.0);
      if (a > change) change = a;
    }
    if (change < tol) break;
  }

  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = 0.0;
    for (int j = 0; j < n; ++j) {
      const double a = fabs(H[i + (size_t)j * n]);
      if (a > r) r = a;
    }
    sum += r;
  }
  const double row_mean = sum / (double)n;
  *cost_scale = 1.0 / (row_mean > 1.0 ? row_mean : 1.0);
  free(H);
  free(G);
  free(delta);
}

/* ------------------------------------------------------------------------------------------
 * layers.cpp:122-175  D, W, b
 * ---------------------------------------------------------------------------------------- */

/* layers.cpp:122-131.  D(n x n) = (H + sigma I + G' diag(rho) G)^{-1}. Returns 1 on
 * factorisation failure (the reference throws std::runtime_error). */
ORC_API int orc_build_kkt_inverse(int n, int m, const double *H, const double *G, double sigma,
                                  const double *rho_vec, double *D) {
  double *kkt = dalloc((size_t)n * n);
  double *rG = dalloc((size_t)m * n);
  double *Gt = dalloc((size_t)n * m);
  memcpy(kkt, H, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) kkt[i + (size_t)i * n] += sigma;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) rG[i + (size_t)j * m] = rho_vec[i] * G[i + (size_t)j * m];
  transpose(m, n, G, Gt);
  gemm_nn_acc(n, m, n, Gt, rG, kkt);
  const int bad = cholesky_lower(n, kkt);
  if (!bad) cholesky_inverse(n, kkt, D);
  free(kkt);
  free(rG);
  free(Gt);
  return bad;
}

/* layers.cpp:168-175  layer_bias: b = [-D g; -GD g; 0]. */
ORC_API void orc_layer_bias(int n, int m, const double *D, const double *GD, const double *g,
                            double *b) {
  gemv_n(n, n, D, g, b);
  gemv_n(m, n, GD, g, b + n);
  for (int i = 0; i < n + m; ++i) b[i] = -b[i];
  for (int i = 0; i < m; ++i) b[n + m + i] = 0.0;
}

/* layers.cpp:133-166  build_layer: W((n+2m)^2), GD(m x n), b(n+2m). */
ORC_API void orc_build_layer(int n, int m, const double *H, const double *G, const double *g,
                             double sigma, const double *rho_vec, const double *D, double *W,
                             double *GD, double *b) {
  (void)H;
  const int dim = n + 2 * m;
  double *Gt = dalloc((size_t)n * m);
  double *DGt = dalloc((size_t)n * m);
  double *GDGt = dalloc((size_t)m * m);
  double *rG = dalloc((size_t)m * n);
  double *T = dalloc((size_t)n * n);
  double *blk = dalloc((size_t)(n > m ? n : m) * (n > m ? n : m));

  gemm_nn(m, n, n, G, D, GD);       /* layer.GD = G * D              :140 */
  transpose(m, n, G, Gt);
  gemm_nn(n, n, m, D, Gt, DGt);     /* DGt = D * G'                  :144 */
  gemm_nn(m, n, m, G, DGt, GDGt);   /* GDGt = G * DGt                :145 */
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) rG[i + (size_t)j * m] = rho_vec[i] * G[i + (size_t)j * m];
  gemm_nn(n, m, n, Gt, rG, T);      /* G' r G                        :147 */
  for (size_t k = 0; k < (size_t)n * n; ++k) T[k] = -T[k];
  for (int i = 0; i < n; ++i) T[i + (size_t)i * n] += sigma; /* sI - G'rG :146-147 */

  memset(W, 0, sizeof(double) * (size_t)dim * dim);
#define WAT(i, j) W[(size_t)(i) + (size_t)(j) * dim]
  /* (0,0) = D*T  :151 */
  gemm_nn(n, n, n, D, T, blk);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) WAT(i, j) = blk[i + (size_t)j * n];
  /* (0,1) = 2 DGt r ; (0,2) = -DGt  :152-153 */
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) {
      const double v = DGt[i + (size_t)j * n];
      WAT(i, n + j) = (2.0 * v) * rho_vec[j];
      WAT(i, n + m + j) = -v;
    }
  /* (1,0) = GD*T + G  :154-155 */
  gemm_nn(m, n, n, GD, T, blk);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) WAT(n + i, j) = blk[i + (size_t)j * m] + G[i + (size_t)j * m];
  /* (1,1) = 2 GDGt r - I ; (1,2) = -GDGt + r^-1  :156-159 */
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      const double v = GDGt[i + (size_t)j * m];
      WAT(n + i, n + j) = (2.0 * v) * rho_vec[j] - (i == j ? 1.0 : 0.0);
      WAT(n + i, n + m + j) = -v + (i == j ? 1.0 / rho_vec[j] : 0.0);
    }
  /* (2,0) = r G ; (2,1) = -r ; (2,2) = I  :160-162 */
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) WAT(n + m + i, j) = rG[i + (size_t)j * m];
  for (int i = 0; i < m; ++i) {
    WAT(n + m + i, n + i) = -rho_vec[i];
    WAT(n + m + i, n + m + i) = 1.0;
  }
#undef WAT
  orc_layer_bias(n, m, D, GD, g, b);
  free(Gt);
  free(DGt);
  free(GDGt);
  free(rG);
  free(T);
  free(blk);
}

/* ------------------------------------------------------------------------------------------
 * LayerCache (layers.hpp:108-127) and precompute_all (layers.cpp:189-228)
 * ---------------------------------------------------------------------------------------- */

typedef struct {
  int n, m, L;
  double *Hs, *gs, *Gs, *cs, *ds; /* cache.problem (scaled when equilibration is on) */
  double *E, *F;
  double cost_scale;
  double *grid;
  int initial_index;
  double eq_scale;
  double sigma;
  double **W, **D, **GD, **rho_vec, **b;
  double *c_tilde, *d_tilde;
} orc_cache;

typedef struct {
  double eps_prim, eps_dual;
  int check_interval, max_iters;
  double sigma;
  int grid_points;
  double rho_switch_threshold;
  int adaptive_rho;
  int eq_enabled, eq_max_passes;
  double eq_tol;
} orc_settings;

/* solver.hpp:43-53 defaults */
ORC_API void orc_default_settings(orc_settings *s) {
  s->eps_prim = 1e-6;
  s->eps_dual = 1e-6;
  s->check_interval = 25;
  s->max_iters = 4000;
  s->sigma = 1e-6;
  s->grid_points = 13;
  s->rho_switch_threshold = 5.0;
  s->adaptive_rho = 1;
  s->eq_enabled = 1;
  s->eq_max_passes = 10;
  s->eq_tol = 1e-3;
}

ORC_API void orc_cache_free(orc_cache *c) {
  if (!c) return;
  free(c->Hs); free(c->gs); free(c->Gs); free(c->cs); free(c->ds);
  free(c->E); free(c->F); free(c->grid);
  for (int k = 0; k < c->L; ++k) {
    if (c->W) free(c->W[k]);
    if (c->D) free(c->D[k]);
    if (c->GD) free(c->GD[k]);
    if (c->rho_vec) free(c->rho_vec[k]);
    if (c->b) free(c->b[k]);
  }
  free(c->W); free(c->D); free(c->GD); free(c->rho_vec); free(c->b);
  free(c->c_tilde); free(c->d_tilde);
  free(c);
}

/* layers.cpp:189-228.  `grid_points` builds the grid (solver.cpp:183). Returns NULL and sets
 * *err = 1 on KKT factorisation failure, 2 on a bad grid size. */
ORC_API orc_cache *orc_precompute_all(int n, int m, const double *H, const double *g,
                                      const double *G, const double *c, const double *d,
                                      int grid_points, double sigma, int eq_enabled,
                                      int eq_max_passes, double eq_tol, int *err) {
  *err = 0;
  orc_cache *cache = (orc_cache *)calloc(1, sizeof(orc_cache));
  const int dim = n + 2 * m;
  cache->n = n; cache->m = m; cache->L = grid_points;
  cache->sigma = sigma;
  cache->eq_scale = 1e3; /* layers.hpp:29 */
  cache->grid = dalloc((size_t)(grid_points > 0 ? grid_points : 1));
  cache->initial_index = orc_build_penalty_grid(grid_points, cache->grid);
  if (cache->initial_index < 0) {
    cache->L = 0;
    orc_cache_free(cache);
    *err = 2;
    return NULL;
  }
  cache->Hs = dalloc((size_t)n * n); cache->gs = dalloc((size_t)n);
  cache->Gs = dalloc((size_t)m * n); cache->cs = dalloc((size_t)m); cache->ds = dalloc((size_t)m);
  cache->E = dalloc((size_t)n); cache->F = dalloc((size_t)m);
  if (eq_enabled) {
    orc_ruiz_scaling(n, m, H, G, eq_max_passes, eq_tol, cache->E, cache->F, &cache->cost_scale);
    scaling_apply(n, m, cache->E, cache->F, cache->cost_scale, H, g, G, c, d, cache->Hs,
                  cache->gs, cache->Gs, cache->cs, cache->ds);
  } else {
    for (int i = 0; i < n; ++i) cache->E[i] = 1.0;
    for (int i = 0; i < m; ++i) cache->F[i] = 1.0;
    cache->cost_scale = 1.0;
    memcpy(cache->Hs, H, sizeof(double) * (size_t)n * n);
    memcpy(cache->gs, g, sizeof(double) * (size_t)n);
    memcpy(cache->Gs, G, sizeof(double) * (size_t)m * n);
    memcpy(cache->cs, c, sizeof(double) * (size_t)m);
    memcpy(cache->ds, d, sizeof(double) * (size_t)m);
  }
  const int L = grid_points;
  cache->W = (double **)calloc((size_t)L, sizeof(double *));
  cache->D = (double **)calloc((size_t)L, sizeof(double *));
  cache->GD = (double **)calloc((size_t)L, sizeof(double *));
  cache->rho_vec = (double **)calloc((size_t)L, sizeof(double *));
  cache->b = (double **)calloc((size_t)L, sizeof(double *));
  for (int k = 0; k < L; ++k) {
    cache->W[k] = dalloc((size_t)dim * dim);
    cache->D[k] = dalloc((size_t)n * n);
    cache->GD[k] = dalloc((size_t)m * n);
    cache->rho_vec[k] = dalloc((size_t)m);
    cache->b[k] = dalloc((size_t)dim);
    for (int i = 0; i < m; ++i) {
      /* problem.hpp:45-47 row_kind on the cache's (scaled) bounds; layers.cpp:206-215 */
      const double scale = (cache->cs[i] == cache->ds[i]) ? cache->eq_scale : 1.0;
      cache->rho_vec[k][i] = scale * cache->grid[k];
    }
    if (orc_build_kkt_inverse(n, m, cache->Hs, cache->Gs, sigma, cache->rho_vec[k],
                              cache->D[k])) {
      orc_cache_free(cache);
      *err = 1;
      return NULL;
    }
    orc_build_layer(n, m, cache->Hs, cache->Gs, cache->gs, sigma, cache->rho_vec[k],
                    cache->D[k], cache->W[k], cache->GD[k], cache->b[k]);
  }
  cache->c_tilde = dalloc((size_t)dim);
  cache->d_tilde = dalloc((size_t)dim);
  for (int i = 0; i < dim; ++i) {
    cache->c_tilde[i] = -INFINITY;
    cache->d_tilde[i] = INFINITY;
  }
  memcpy(cache->c_tilde + n, cache->cs, sizeof(double) * (size_t)m);
  memcpy(cache->d_tilde + n, cache->ds, sizeof(double) * (size_t)m);
  return cache;
}

/* layers.cpp:177-187  LayerCache::update_vectors (original units in). */
ORC_API void orc_cache_update_vectors(orc_cache *cache, const double *g, const double *c,
                                      const double *d) {
  const int n = cache->n, m = cache->m;
  for (int i = 0; i < n; ++i) cache->gs[i] = cache->cost_scale * (cache->E[i] * g[i]);
  for (int i = 0; i < m; ++i) {
    cache->cs[i] = cache->F[i] * c[i];
    cache->ds[i] = cache->F[i] * d[i];
  }
  for (int k = 0; k < cache->L; ++k)
    orc_layer_bias(n, m, cache->D[k], cache->GD[k], cache->gs, cache->b[k]);
  memcpy(cache->c_tilde + n, cache->cs, sizeof(double) * (size_t)m);
  memcpy(cache->d_tilde + n, cache->ds, sizeof(double) * (size_t)m);
}

/* accessors used by the Python wrapper */
ORC_API int orc_cache_n(const orc_cache *c) { return c->n; }
ORC_API int orc_cache_m(const orc_cache *c) { return c->m; }
ORC_API int orc_cache_L(const orc_cache *c) { return c->L; }
ORC_API int orc_cache_initial_index(const orc_cache *c) { return c->initial_index; }
ORC_API double orc_cache_cost_scale(const orc_cache *c) { return c->cost_scale; }
ORC_API double orc_cache_sigma(const orc_cache *c) { return c->sigma; }
ORC_API const double *orc_cache_ptr(const orc_cache *c, int what, int k) {
  switch (what) {
    case 0: return c->W[k];
    case 1: return c->D[k];
    case 2: return c->GD[k];
    case 3: return c->rho_vec[k];
    case 4: return c->b[k];
    case 5: return c->Hs;
    case 6: return c->gs;
    case 7: return c->Gs;
    case 8: return c->cs;
    case 9: return c->ds;
    case 10: return c->E;
    case 11: return c->F;
    case 12: return c->grid;
    case 13: return c->c_tilde;
    case 14: return c->d_tilde;
    default: return NULL;
  }
}

/* ------------------------------------------------------------------------------------------
 * solver.cpp:109-156  free functions
 * ---------------------------------------------------------------------------------------- */

/* solver.cpp:109-117  iterate: out = clamp(W v + b, c~, d~). out must not alias v. */
ORC_API void orc_iterate(int dim, const double *v, const double *W, const double *b,
                         const double *c_tilde, const double *d_tilde, double *out) {
  gemv_n(dim, dim, W, v, out);
  for (int i = 0; i < dim; ++i) {
    double x = out[i] + b[i];
    x = x < c_tilde[i] ? c_tilde[i] : x; /* cwiseMax(c~) */
    x = x > d_tilde[i] ? d_tilde[i] : x; /* cwiseMin(d~) */
    out[i] = x;
  }
}

/* solver.cpp:119-124  residuals on the problem as given. */
ORC_API void orc_residuals(int n, int m, const double *y, const double *z, const double *lam,
                           const double *H, const double *g, const double *G, double *r_prim,
                           double *r_dual) {
  double *t = dalloc((size_t)(n > m ? n : m));
  double *u = dalloc((size_t)n);
  gemv_n(m, n, G, y, t);
  for (int i = 0; i < m; ++i) t[i] -= z[i];
  *r_prim = vec_inf_norm(m, t);
  gemv_n(n, n, H, y, t);
  gemv_t(m, n, G, lam, u);
  for (int i = 0; i < n; ++i) t[i] = t[i] + g[i] + u[i];
  *r_dual = vec_inf_norm(n, t);
  free(t);
  free(u);
}

static double max2(double a, double b) { return a > b ? a : b; }

/* solver.cpp:126-134  rho_nominal. */
ORC_API double orc_rho_nominal(int n, int m, double r_prim, double r_dual, const double *y,
                               const double *z, const double *lam, const double *H,
                               const double *g, const double *G, double current_rho) {
  if (r_prim == 0.0 || r_dual == 0.0) return current_rho;
  double *t = dalloc((size_t)(n > m ? n : m));
  gemv_n(n, n, H, y, t);
  const double hy = vec_inf_norm(n, t);
  gemv_t(m, n, G, lam, t);
  const double gtl = vec_inf_norm(n, t);
  gemv_n(m, n, G, y, t);
  const double gy = vec_inf_norm(m, t);
  free(t);
  const double num_scale = max2(max2(hy, gtl), max2(vec_inf_norm(n, g), 1e-4));
  const double den_scale = max2(max2(gy, vec_inf_norm(m, z)), 1e-4);
  return current_rho * sqrt((r_prim * num_scale) / (r_dual * den_scale));
}

/* solver.cpp:136-142  select_layer. */
ORC_API int orc_select_layer(double rho_nom, const double *grid, int L, int current_index,
                             double threshold) {
  const int candidate = orc_nearest_grid_index(grid, L, rho_nom);
  const double rho_cur = grid[current_index];
  const double ratio = max2(rho_nom / rho_cur, rho_cur / rho_nom);
  return ratio >= threshold ? candidate : current_index;
}

/* solver.cpp:144-156  warm_start: v = [y/E; G_s (y/E); cost_scale*lambda/F].  `last_index` is
 * prev.rho_trace.back().grid_index, or -1 for an empty trace (-> initial_index). */
ORC_API int orc_warm_start(const orc_cache *cache, const double *y, const double *lam,
                           int last_index, double *v) {
  const int n = cache->n, m = cache->m;
  for (int i = 0; i < n; ++i) v[i] = y[i] / cache->E[i];
  gemv_n(m, n, cache->Gs, v, v + n);
  for (int i = 0; i < m; ++i) v[n + m + i] = cache->cost_scale * (lam[i] / cache->F[i]);
  return last_index < 0 ? cache->initial_index : last_index;
}

/* solver.cpp:197-200  Solver::refresh_z: z_s <- G_s y_s, y and lambda untouched. */
ORC_API void orc_refresh_z(const orc_cache *cache, double *v) {
  gemv_n(cache->m, cache->n, cache->Gs, v, v + cache->n);
}

/* ------------------------------------------------------------------------------------------
 * solver.cpp:43-105  run_loop
 * ---------------------------------------------------------------------------------------- */

typedef struct {
  /* Solution (problem.hpp:62-71); status: 0 Solved, 1 MaxIters, 2 Invalid */
  int status;
  int iterations;
  double r_prim, r_dual;
  int n_trace;  /* rho_trace entries written */
  int n_hist;   /* residual_history entries written */
  double wall_ms;
} orc_report_head;

/* Unscale helpers, layers.hpp:57-59. */
static void unscale(const orc_cache *c, const double *v, double *y, double *z, double *lam) {
  const int n = c->n, m = c->m;
  for (int i = 0; i < n; ++i) y[i] = c->E[i] * v[i];
  for (int i = 0; i < m; ++i) z[i] = v[n + i] / c->F[i];
  for (int i = 0; i < m; ++i) lam[i] = (c->F[i] * v[n + m + i]) / c->cost_scale;
}

/* run_loop.  p_* is the problem handed to the loop (the unscaled Solver::problem_).
 * state v (n+2m) and *layer_index are updated in place.  Arrays: y(n) z(m) lam(m);
 * trace_iter/trace_idx and hist_iter/hist_rp/hist_rd/hist_idx have capacity `cap` each
 * (cap >= total_iters / check_interval + 2 always suffices). */
ORC_API void orc_run_loop(const orc_cache *cache, const orc_settings *s, const double *pH,
                          const double *pg, const double *pG, const double *pc,
                          const double *pd, double *v, int *layer_index, int early_exit,
                          int total_iters, orc_report_head *head, double *y, double *z,
                          double *lam, int *trace_iter, int *trace_idx, int *hist_iter,
                          double *hist_rp, double *hist_rd, int *hist_idx, int cap) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const int n = cache->n, m = cache->m, dim = n + 2 * m;
  double *next = dalloc((size_t)dim);
  int n_trace = 0, n_hist = 0;
  if (n_trace < cap) { trace_iter[n_trace] = 0; trace_idx[n_trace] = *layer_index; }
  ++n_trace;

  int converged = 0, iters_done = 0;
  for (int i = 1; i <= total_iters; ++i) {
    const int k = *layer_index;
    orc_iterate(dim, v, cache->W[k], cache->b[k], cache->c_tilde, cache->d_tilde, next);
    memcpy(v, next, sizeof(double) * (size_t)dim);
    iters_done = i;
    if (i % s->check_interval != 0) continue;

    unscale(cache, v, y, z, lam);
    double rp, rd;
    orc_residuals(n, m, y, z, lam, pH, pg, pG, &rp, &rd);
    if (n_hist < cap) {
      hist_iter[n_hist] = i; hist_rp[n_hist] = rp; hist_rd[n_hist] = rd; hist_idx[n_hist] = k;
    }
    ++n_hist;

    if (s->adaptive_rho) {
      const double rho_cur = cache->grid[k];
      const double rho_nom = orc_rho_nominal(n, m, rp, rd, y, z, lam, pH, pg, pG, rho_cur);
      const int cand = orc_select_layer(rho_nom, cache->grid, cache->L, k,
                                        s->rho_switch_threshold);
      if (cand != k) {
        *layer_index = cand;
        if (n_trace < cap) { trace_iter[n_trace] = i; trace_idx[n_trace] = cand; }
        ++n_trace;
      }
    }
    if (early_exit && rp <= s->eps_prim && rd <= s->eps_dual) {
      converged = 1;
      break;
    }
  }

  unscale(cache, v, y, z, lam);
  for (int i = 0; i < m; ++i) {
    double x = z[i];
    x = x < pc[i] ? pc[i] : x;
    x = x > pd[i] ? pd[i] : x;
    z[i] = x;
  }
  orc_residuals(n, m, y, z, lam, pH, pg, pG, &head->r_prim, &head->r_dual);
  head->iterations = iters_done;
  head->status =
      (converged || (head->r_prim <= s->eps_prim && head->r_dual <= s->eps_dual)) ? 0 : 1;
  head->n_trace = n_trace;
  head->n_hist = n_hist;
  free(next);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  head->wall_ms = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;
}

/* solver.cpp:29-34  check_settings: 0 ok, 1 -> std::invalid_argument. */
ORC_API int orc_check_settings(const orc_settings *s) {
  if (s->check_interval < 1) return 1;
  if (s->max_iters < s->check_interval) return 1;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * oracle.cpp:63-74  admm_step_reordered -- the independent sequential step used to check W.
 * state (y, z, lam) -> (y+, z+, lam+) on the given (scaled) problem.
 * ---------------------------------------------------------------------------------------- */
ORC_API int orc_admm_step_reordered(int n, int m, const double *H, const double *g,
                                    const double *G, const double *c, const double *d,
                                    double sigma, const double *rho_vec, const double *y,
                                    const double *z, const double *lam, double *y_out,
                                    double *z_out, double *lam_out) {
  double *D = dalloc((size_t)n * n);
  if (orc_build_kkt_inverse(n, m, H, G, sigma, rho_vec, D)) {
    free(D);
    return 1;
  }
  double *t = dalloc((size_t)m);
  double *rhs = dalloc((size_t)n);
  gemv_n(m, n, G, y, t);
  for (int i = 0; i < m; ++i) lam_out[i] = lam[i] + rho_vec[i] * (t[i] - z[i]);
  for (int i = 0; i < m; ++i) t[i] = rho_vec[i] * z[i] - lam_out[i];
  gemv_t(m, n, G, t, rhs);
  for (int i = 0; i < n; ++i) rhs[i] = -g[i] + sigma * y[i] + rhs[i];
  gemv_n(n, n, D, rhs, y_out);
  gemv_n(m, n, G, y_out, t);
  for (int i = 0; i < m; ++i) {
    double x = t[i] + (1.0 / rho_vec[i]) * lam_out[i];
    x = x < c[i] ? c[i] : x;
    x = x > d[i] ? d[i] : x;
    z_out[i] = x;
  }
  free(D);
  free(t);
  free(rhs);
  return 0;
}
