// Offline stage on the device: Solver::Solver -> validate + precompute_all
// (/root/reference/proj/src/solver.cpp:180-186, src/problem.cpp:121-164,
//  src/layers.cpp:22-36 grid, :82-120 Ruiz, :122-131 D, :133-166 W, :189-228 precompute_all).
//
// Setup work, off the hot path, but still hand-written CUDA with no library dependency (an
// earlier cuSOLVER/cuBLAS version pulled 1.7 GB of shared objects into every process, minutes
// of cold-load time on a fresh box):
//   * D = (H + sigma I + G' rho G)^-1 by a right-looking Cholesky (one scale + one rank-1
//     update kernel per column) followed by forward and backward substitution on the identity
//     (layers.cpp:126-130 does LLT + solve(I)); a non-positive pivot is reported like
//     Eigen::LLT's NumericalIssue (-> ProblemError::NonPositiveDefiniteH / std::runtime_error);
//   * the five dense products of build_layer (layers.cpp:140-155) on the FP64 tensor-core GEMM
//     of cqp_batch.cu;
//   * the Ruiz equilibration (O(passes * n(n+m)) elementwise work on H and G) on the host,
//     exactly in the reference's operation order, so E, F and cost_scale are bit-identical to a
//     host implementation.
// The result is the same device layout cqp_create_from_layers produces: W_k row-major padded,
// [D_k; G D_k] row-major padded.
#include <algorithm>
#include <cmath>
#include <vector>

#include "cqp_internal.h"

namespace cqp {

// from cqp_capi.cu
int handle_alloc(cqp_handle** out, int n, int m, int L, const cqp_settings& s, int device);
int upload_small(cqp_handle* h, const double* grid, const double* E, const double* F);
int upload_vectors(cqp_handle* h, const double* g, const double* c, const double* d);
int cold_start(cqp_handle* h);

namespace {

// All offline-stage matrices are column-major with a padded leading dimension (multiple of 16)
// so that they can feed the DMMA GEMM directly (K contiguous, zero padded).

// rG = diag(rho) G   (m x n, leading dimension ld)
__global__ void scale_rows_kernel(const double* __restrict__ G, const double* __restrict__ rho,
                                  int m, int n, int ld, double* __restrict__ out) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)m * n) return;
  const int i = (int)(idx % m), j = (int)(idx / m);
  out[i + (size_t)j * ld] = rho[i] * G[i + (size_t)j * ld];
}

// kkt = H + sigma I + M ;  T = sigma I - M   (n x n, leading dimension ld)
__global__ void kkt_and_t_kernel(const double* __restrict__ H, const double* __restrict__ M,
                                 double sigma, int n, int ld, double* __restrict__ kkt,
                                 double* __restrict__ T) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  const size_t at = i + (size_t)j * ld;
  const double s = (i == j) ? sigma : 0.0;
  kkt[at] = (H[at] + s) + M[at];
  T[at] = s - M[at];
}

// ---- Cholesky + inverse (LLT, then solve(I)), blocked ---------------------------------------
// Block size 64: per block column one diagonal-block kernel (one CTA, the block in shared memory),
// one panel / row-block solve (a thread per row or column, its 64 unknowns in registers) and one
// tiled rank-64 update of everything behind it: ~7 n / 64 launches per ladder level instead of 4 n
// (n = 870: 98 instead of 3480), and the update runs as 64 x 64 x 64 shared-memory tiles instead of
// rank-1 sweeps over the whole trailing matrix.  Same algorithm as before and as the reference
// (layers.cpp:126-130: LLT, then forward and backward substitution on the identity); only the
// summation order inside a block differs.
constexpr int kNB = 64;

// Diagonal block A[j0 : j0+nb, j0 : j0+nb] -> its Cholesky factor, in place.  A non-positive pivot is
// recorded (first one wins, 1-based global column) and replaced by 1 so that the rest stays finite.
__global__ void __launch_bounds__(256) chol_diag_kernel(double* __restrict__ A, int ld, int j0, int nb, int* fail) {
  __shared__ double S[kNB][kNB + 1];
  const int t = threadIdx.x;
  for (int e = t; e < nb * nb; e += 256) {
    const int r = e % nb, c = e / nb;
    S[r][c] = (r >= c) ? A[(j0 + r) + (size_t)(j0 + c) * ld] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (t == 0) {
      double a = S[j][j];
      if (!(a > 0.0)) {
        atomicCAS(fail, 0, j0 + j + 1);
        a = 1.0;
      }
      S[j][j] = sqrt(a);
    }
    __syncthreads();
    const double l = S[j][j];
    for (int r = j + 1 + t; r < nb; r += 256) S[r][j] /= l;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int e = t; e < rem * rem; e += 256) {
      const int r = j + 1 + e % rem, c = j + 1 + e / rem;
      if (r >= c) S[r][c] -= S[r][j] * S[c][j];
    }
    __syncthreads();
  }
  for (int e = t; e < nb * nb; e += 256) {
    const int r = e % nb, c = e / nb;
    if (r >= c) A[(j0 + r) + (size_t)(j0 + c) * ld] = S[r][c];
  }
}

// Panel below the diagonal block: row i of A[i, j0 : j0+nb] <- row i . L11^-T (one thread per row).
__global__ void __launch_bounds__(128) chol_panel_kernel(double* __restrict__ A, int ld, int n, int j0, int nb) {
  __shared__ double L[kNB][kNB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += 128) {
    const int r = e % nb, c = e / nb;
    L[r][c] = (r >= c) ? A[(j0 + r) + (size_t)(j0 + c) * ld] : 0.0;
  }
  __syncthreads();
  const int i = j0 + nb + blockIdx.x * 128 + threadIdx.x;
  if (i >= n) return;
  double x[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    if (c < nb) {
      double v = A[i + (size_t)(j0 + c) * ld];
#pragma unroll
      for (int k = 0; k < kNB; ++k)
        if (k < c) v -= x[k] * L[c][k];
      x[c] = v / L[c][c];
      A[i + (size_t)(j0 + c) * ld] = x[c];
    }
  }
}

// C[i, c] -= sum_{q < nb} P(i, q) Q(q, c)  over rows [i0, i1) and columns [c0, c1), 64 x 64 tiles:
//   P(i, q) = PT ? Pm[(p0 + q) + i ld] : Pm[i + (p0 + q) ld]     (PT: the factor read transposed)
//   Q(q, c) = QT ? Qm[c + (p0 + q) ld] : Qm[(p0 + q) + c ld]
//   LOWER: only entries with i >= c (the trailing update of the Cholesky factor)
template <bool PT, bool QT, bool LOWER>
__global__ void __launch_bounds__(256) tile_update_kernel(double* __restrict__ C, const double* __restrict__ Pm,
                                                          const double* __restrict__ Qm, int ld, int i0, int i1, int c0,
                                                          int c1, int p0, int nb) {
  const int ti = i0 + blockIdx.x * 64, tc = c0 + blockIdx.y * 64;
  if (LOWER && tc > ti + 63) return;  // tile strictly above the diagonal
  constexpr int KH = 32;              // q is walked in halves: two 32 x 65 tiles fit the static 48 KB
  __shared__ double Ps[KH][65];       // [q][row]
  __shared__ double Qs[KH][65];       // [q][col]
  const int t = threadIdx.x;
  const int tr = (t & 15) * 4, tcol = (t >> 4) * 4;
  double acc[4][4] = {};
  for (int qh = 0; qh < nb; qh += KH) {
    const int nq = min(KH, nb - qh);
    for (int e = t; e < 64 * nq; e += 256) {
      int r, q;
      if (PT) { q = e % nq; r = e / nq; } else { r = e % 64; q = e / 64; }
      const int i = ti + r;
      Ps[q][r] = (i < i1) ? (PT ? Pm[(p0 + qh + q) + (size_t)i * ld] : Pm[i + (size_t)(p0 + qh + q) * ld]) : 0.0;
    }
    for (int e = t; e < 64 * nq; e += 256) {
      int cc, q;
      if (QT) { cc = e % 64; q = e / 64; } else { q = e % nq; cc = e / nq; }
      const int c = tc + cc;
      Qs[q][cc] = (c < c1) ? (QT ? Qm[c + (size_t)(p0 + qh + q) * ld] : Qm[(p0 + qh + q) + (size_t)c * ld]) : 0.0;
    }
    __syncthreads();
    for (int q = 0; q < nq; ++q) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = Ps[q][tr + u]; b[u] = Qs[q][tcol + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int c = tc + tcol + v;
    if (c >= c1) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = ti + tr + u;
      if (i < i1 && (!LOWER || i >= c)) C[i + (size_t)c * ld] -= acc[u][v];
    }
  }
}

// Row block k0 of the forward substitution L Y = I:  Y[k0 : k0+nb, c] <- L11^-1 Y[k0 : k0+nb, c] for the
// columns c < ncols (a thread per column).  BWD: the backward substitution L' X = Y (L11^-T instead).
template <bool BWD>
__global__ void __launch_bounds__(128) tri_block_solve_kernel(const double* __restrict__ Lm, double* __restrict__ Y, int ld,
                                                              int k0, int nb, int ncols) {
  __shared__ double L[kNB][kNB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += 128) {
    const int r = e % nb, c = e / nb;
    L[r][c] = (r >= c) ? Lm[(k0 + r) + (size_t)(k0 + c) * ld] : 0.0;
  }
  __syncthreads();
  const int c = blockIdx.x * 128 + threadIdx.x;
  if (c >= ncols) return;
  double* y = Y + (size_t)c * ld + k0;
  double x[kNB];
  if (!BWD) {
#pragma unroll
    for (int r = 0; r < kNB; ++r) {
      if (r < nb) {
        double v = y[r];
#pragma unroll
        for (int q = 0; q < kNB; ++q)
          if (q < r) v -= L[r][q] * x[q];
        x[r] = v / L[r][r];
        y[r] = x[r];
      }
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < kNB; ++rr) {
      const int r = kNB - 1 - rr;
      if (r < nb) {
        double v = y[r];
#pragma unroll
        for (int q = 0; q < kNB; ++q)
          if (q > r && q < nb) v -= L[q][r] * x[q];
        x[r] = v / L[r][r];
        y[r] = x[r];
      }
    }
  }
}

__global__ void set_identity_kernel(double* __restrict__ Y, int ld, int n) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  Y[i + (size_t)j * ld] = (i == j) ? 1.0 : 0.0;
}

// make the computed inverse exactly symmetric (upper <- lower)
__global__ void mirror_lower_kernel(double* __restrict__ A, int ld, int n) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  if (i < j) A[i + (size_t)j * ld] = A[j + (size_t)i * ld];
}

// Assemble W (row-major, ld = Dpad, pad zero) from its blocks (layers.cpp:149-162):
//   [ DT          2 DGt r         -DGt        ]      DT  = D T        (n x n, ld_n)
//   [ GDT + G     2 GDGt r - I    -GDGt + 1/r ]      GD  = G D        (m x n, ld_m)  DGt = GD'
//   [ r G         -r              I           ]      GDT = GD T (m x n, ld_m), GDGt (m x m, ld_m)
__global__ void assemble_w_kernel(int n, int m, int Dpad, int ld_n, int ld_m,
                                  const double* __restrict__ DT, const double* __restrict__ GD,
                                  const double* __restrict__ GDT, const double* __restrict__ GDGt,
                                  const double* __restrict__ Gs, const double* __restrict__ rho,
                                  double* __restrict__ W) {
  const int D = n + 2 * m;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)D * Dpad) return;
  const int r = (int)(idx / Dpad), c = (int)(idx % Dpad);
  double v = 0.0;
  if (c < D) {
    if (r < n) {
      if (c < n) v = DT[r + (size_t)c * ld_n];
      else if (c < n + m) v = (2.0 * GD[(c - n) + (size_t)r * ld_m]) * rho[c - n];
      else v = -GD[(c - n - m) + (size_t)r * ld_m];
    } else if (r < n + m) {
      const int i = r - n;
      if (c < n) v = GDT[i + (size_t)c * ld_m] + Gs[i + (size_t)c * ld_m];
      else if (c < n + m) {
        const int j = c - n;
        v = (2.0 * GDGt[i + (size_t)j * ld_m]) * rho[j] - (i == j ? 1.0 : 0.0);
      } else {
        const int j = c - n - m;
        v = -GDGt[i + (size_t)j * ld_m] + (i == j ? 1.0 / rho[j] : 0.0);
      }
    } else {
      const int i = r - n - m;
      if (c < n) v = rho[i] * Gs[i + (size_t)c * ld_m];
      else if (c < n + m) v = (c - n == i) ? -rho[i] : 0.0;
      else v = (c - n - m == i) ? 1.0 : 0.0;
    }
  }
  W[idx] = v;
}

int blocks_for(size_t count) { return (int)((count + 255) / 256); }

}  // namespace

// layers.cpp:38-50 (host)
static int nearest_grid_index_host(const std::vector<double>& grid, double rho) {
  const double target = std::log10(rho);
  int best = 0;
  double best_dist = INFINITY;
  for (int k = 0; k < (int)grid.size(); ++k) {
    const double dist = std::fabs(std::log10(grid[k]) - target);
    if (dist < best_dist - 1e-15) {
      best = k;
      best_dist = dist;
    }
  }
  return best;
}

// layers.cpp:82-120 on the host, same operation order as the reference.
static void ruiz_host(int n, int m, const double* H_in, const double* G_in, int max_passes,
                      double tol, std::vector<double>& E, std::vector<double>& F,
                      double& cost_scale) {
  std::vector<double> H(H_in, H_in + (size_t)n * n), G(G_in, G_in + (size_t)m * n);
  std::vector<double> delta((size_t)n + m);
  E.assign(n, 1.0);
  F.assign(m, 1.0);
  for (int pass = 0; pass < max_passes; ++pass) {
    for (int i = 0; i < n; ++i) {
      double rh = 0.0, rg = 0.0;
      for (int j = 0; j < n; ++j) rh = std::max(rh, std::fabs(H[i + (size_t)j * n]));
      for (int k = 0; k < m; ++k) rg = std::max(rg, std::fabs(G[k + (size_t)i * m]));
      const double r = std::max(rh, rg);
      delta[i] = r > 0.0 ? 1.0 / std::sqrt(r) : 1.0;
    }
    for (int i = 0; i < m; ++i) {
      double r = 0.0;
      for (int j = 0; j < n; ++j) r = std::max(r, std::fabs(G[i + (size_t)j * m]));
      delta[n + i] = r > 0.0 ? 1.0 / std::sqrt(r) : 1.0;
    }
    const double* dE = delta.data();
    const double* dF = delta.data() + n;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) H[i + (size_t)j * n] = (dE[i] * H[i + (size_t)j * n]) * dE[j];
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) G[i + (size_t)j * m] = (dF[i] * G[i + (size_t)j * m]) * dE[j];
    for (int i = 0; i < n; ++i) E[i] *= dE[i];
    for (int i = 0; i < m; ++i) F[i] *= dF[i];
    double change = 0.0;
    for (size_t i = 0; i < delta.size(); ++i) change = std::max(change, std::fabs(delta[i] - 1.0));
    if (change < tol) break;
  }
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = 0.0;
    for (int j = 0; j < n; ++j) r = std::max(r, std::fabs(H[i + (size_t)j * n]));
    sum += r;
  }
  const double row_mean = sum / (double)n;
  cost_scale = 1.0 / std::max(1.0, row_mean);
}

}  // namespace cqp

using namespace cqp;

extern "C" int cqp_create(cqp_handle** out, int n, int m, const double* H, const double* g,
                          const double* G, const double* c, const double* d,
                          const cqp_settings* settings, int device) {
  if (!out) return CQP_ERR_ARGUMENT;
  *out = nullptr;
  // ---- validate, host part (problem.cpp:121-144) ----
  if (n < 1 || m < 1 || !H || !g || !G || !c || !d) {
    set_error("n and m must be >= 1 (use a row with infinite bounds for an unconstrained problem)");
    return CQP_ERR_DIMENSION;
  }
  for (size_t i = 0; i < (size_t)n * n; ++i)
    if (!std::isfinite(H[i])) { set_error("H contains a non-finite entry"); return CQP_ERR_NONFINITE; }
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(g[i])) { set_error("g contains a non-finite entry"); return CQP_ERR_NONFINITE; }
  for (size_t i = 0; i < (size_t)m * n; ++i)
    if (!std::isfinite(G[i])) { set_error("G contains a non-finite entry"); return CQP_ERR_NONFINITE; }
  {
    double h_norm = 0.0, asym = 0.0;
    for (int i = 0; i < n; ++i) {
      double srow = 0.0;
      for (int j = 0; j < n; ++j) {
        srow += std::fabs(H[i + (size_t)j * n]);
        asym = std::max(asym, std::fabs(H[i + (size_t)j * n] - H[j + (size_t)i * n]));
      }
      h_norm = std::max(h_norm, srow);
    }
    if (asym > 1e-12 * std::max(1.0, h_norm)) { set_error("H is not symmetric"); return CQP_ERR_NONSYMMETRIC_H; }
  }
  cqp_settings s;
  if (settings) s = *settings; else cqp_default_settings(&s);

  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    set_error("no CUDA device available: libcqp_b200 has no CPU fallback");
    return CQP_ERR_CUDA;
  }
  if (device < 0) CQP_CUDA(cudaGetDevice(&device));
  CQP_CUDA(cudaSetDevice(device));

  cqp_handle* h = nullptr;
  DenseGemm* gemm_n = nullptr;  // N = n output columns
  DenseGemm* gemm_m = nullptr;  // N = m output columns
  cudaStream_t st0 = nullptr;
  std::vector<void*> temps;
  auto cleanup = [&](int code) {
    for (void* p : temps) cudaFree(p);
    dense_gemm_destroy(gemm_n);
    dense_gemm_destroy(gemm_m);
    if (st0) cudaStreamDestroy(st0);
    if (code != CQP_OK) { cqp_destroy(h); h = nullptr; }
    return code;
  };
  auto talloc = [&](double** p, size_t cnt) -> int {
    if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(double) * (cnt ? cnt : 1)) != cudaSuccess) return (int)CQP_ERR_CUDA;
    if (cudaMemset(*p, 0, sizeof(double) * (cnt ? cnt : 1)) != cudaSuccess) return (int)CQP_ERR_CUDA;
    // cudaMemset runs on the legacy default stream, which does NOT order against the
    // cudaStreamNonBlocking streams the kernels below use: wait for it here
    if (cudaStreamSynchronize(0) != cudaSuccess) return (int)CQP_ERR_CUDA;
    temps.push_back(*p);
    return (int)CQP_OK;
  };
#define TRY(expr) do { int rc__ = (expr); if (rc__) return cleanup(rc__); } while (0)
#define TRYCUDA(expr) do { cudaError_t e__ = (expr); if (e__ != cudaSuccess) return cleanup(cuda_fail(e__, #expr)); } while (0)

  const int ld_n = (n + 15) / 16 * 16, ld_m = (m + 15) / 16 * 16;      // K-padded leading dimensions
  const int n128 = (n + 127) / 128 * 128, m128 = (m + 127) / 128 * 128;  // row-padded A operands
  int* dfail = nullptr;
  TRYCUDA(cudaMalloc(reinterpret_cast<void**>(&dfail), sizeof(int)));
  temps.push_back(dfail);
  TRYCUDA(cudaStreamCreateWithFlags(&st0, cudaStreamNonBlocking));

  // In-place lower Cholesky of the n x n matrix A (leading dimension ld_n); fail flag on device.
  auto cholesky = [&](double* A, cudaStream_t st) -> int {
    CQP_CUDA(cudaMemsetAsync(dfail, 0, sizeof(int), st));
    for (int j0 = 0; j0 < n; j0 += kNB) {
      const int nb = std::min(kNB, n - j0), rem = n - j0 - nb;
      chol_diag_kernel<<<1, 256, 0, st>>>(A, ld_n, j0, nb, dfail);
      if (rem > 0) {
        chol_panel_kernel<<<(rem + 127) / 128, 128, 0, st>>>(A, ld_n, n, j0, nb);
        const int tiles = (rem + 63) / 64;
        tile_update_kernel<false, true, true><<<dim3(tiles, tiles), 256, 0, st>>>(A, A, A, ld_n, j0 + nb, n, j0 + nb, n, j0, nb);
      }
    }
    CQP_CUDA(cudaGetLastError());
    return CQP_OK;
  };
  auto read_fail = [&](cudaStream_t st, int* out_flag) -> int {
    CQP_CUDA(cudaMemcpyAsync(out_flag, dfail, sizeof(int), cudaMemcpyDeviceToHost, st));
    CQP_CUDA(cudaStreamSynchronize(st));
    return CQP_OK;
  };

  // ---- PD check of H: LLT (problem.cpp:146-149) ----
  double* dH = nullptr;
  TRY(talloc(&dH, (size_t)n * ld_n));
  TRYCUDA(cudaMemcpy2D(dH, sizeof(double) * ld_n, H, sizeof(double) * n, sizeof(double) * n, n, cudaMemcpyHostToDevice));
  // (a synchronous copy from pageable memory may return before its DMA has landed, and the legacy
  // stream does not order against st0: without this wait the factorisation could read a partial H
  // and report a spurious non-positive pivot)
  TRYCUDA(cudaStreamSynchronize(0));
  TRY(cholesky(dH, st0));
  int info = 0;
  TRY(read_fail(st0, &info));
  if (info != 0) { set_error("H is not positive-definite"); return cleanup(CQP_ERR_NOT_PD_H); }

  // ---- bounds (problem.cpp:151-162) ----
  for (int i = 0; i < m; ++i) {
    const double lo = c[i], hi = d[i];
    if (std::isnan(lo) || std::isnan(hi)) { set_error("bound row contains NaN"); return cleanup(CQP_ERR_NONFINITE); }
    if (lo == INFINITY || hi == -INFINITY || lo > hi) { set_error("row has inverted bounds"); return cleanup(CQP_ERR_INVERTED_BOUNDS); }
  }
  // ---- settings (solver.cpp:29-34) and grid (layers.cpp:22-36) ----
  if (s.check_interval < 1) { set_error("check_interval must be >= 1"); return cleanup(CQP_ERR_SETTINGS); }
  if (s.max_iters < s.check_interval) { set_error("max_iters must be >= check_interval"); return cleanup(CQP_ERR_SETTINGS); }
  if (s.grid_points < 2) { set_error("penalty grid needs at least 2 points"); return cleanup(CQP_ERR_SETTINGS); }
  const int L = s.grid_points;
  std::vector<double> grid(L);
  for (int k = 0; k < L; ++k) grid[k] = std::pow(10.0, -3.0 + (3.0 - -3.0) * k / (L - 1));
  grid.front() = 1e-3;
  grid.back() = 1e3;
  const int initial_index = nearest_grid_index_host(grid, 0.1);

  // ---- equilibration (layers.cpp:195-203) ----
  std::vector<double> E, F;
  double cost_scale = 1.0;
  if (s.eq_enabled) ruiz_host(n, m, H, G, s.eq_max_passes, s.eq_tol, E, F, cost_scale);
  else { E.assign(n, 1.0); F.assign(m, 1.0); }
  std::vector<double> Hs((size_t)n * n), Gs((size_t)m * n), cs(m), ds(m);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      Hs[i + (size_t)j * n] = s.eq_enabled ? cost_scale * ((E[i] * H[i + (size_t)j * n]) * E[j]) : H[i + (size_t)j * n];
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i)
      Gs[i + (size_t)j * m] = s.eq_enabled ? (F[i] * G[i + (size_t)j * m]) * E[j] : G[i + (size_t)j * m];
  for (int i = 0; i < m; ++i) { cs[i] = F[i] * c[i]; ds[i] = F[i] * d[i]; }

  TRY(handle_alloc(&h, n, m, L, s, device));
  h->initial_index = initial_index;
  h->cost_scale = cost_scale;
  cudaStream_t st = h->stream;
  TRY(dense_gemm_create(&gemm_n, n, h->num_sms));
  TRY(dense_gemm_create(&gemm_m, m, h->num_sms));

  const int D = h->D;
  const size_t nm = (size_t)n + m;
  // column-major, K-padded; matrices that also serve as a row-major A operand get padded rows
  double *dHs, *dGs, *dGsrm, *dRho, *drG, *dM, *dKkt, *dY, *dT, *dGD, *dGDrm, *dGDGt, *dDT, *dGDT, *dscr;
  TRY(talloc(&dHs, (size_t)n * ld_n));
  TRY(talloc(&dGs, (size_t)n128 * ld_m));      // Gs (m x n, ld_m); as A operand it is Gs' row-major
  TRY(talloc(&dGsrm, (size_t)m128 * ld_n));    // Gs row-major (m x n, ld_n)
  TRY(talloc(&dRho, (size_t)m));
  TRY(talloc(&drG, (size_t)n * ld_m));
  TRY(talloc(&dM, (size_t)n * ld_n));
  TRY(talloc(&dKkt, (size_t)n * ld_n));
  TRY(talloc(&dY, (size_t)n128 * ld_n));       // D (symmetric: also its own row-major image)
  TRY(talloc(&dT, (size_t)n * ld_n));
  TRY(talloc(&dGD, (size_t)n * ld_m));
  TRY(talloc(&dGDrm, (size_t)m128 * ld_n));
  TRY(talloc(&dGDGt, (size_t)m * ld_m));
  TRY(talloc(&dDT, (size_t)n * ld_n));
  TRY(talloc(&dGDT, (size_t)n * ld_m));
  TRY(talloc(&dscr, std::max((size_t)n * n, (size_t)m * n)));
  TRYCUDA(cudaMemcpy2DAsync(dHs, sizeof(double) * ld_n, Hs.data(), sizeof(double) * n, sizeof(double) * n, n, cudaMemcpyHostToDevice, st));
  TRYCUDA(cudaMemcpy2DAsync(dGs, sizeof(double) * ld_m, Gs.data(), sizeof(double) * m, sizeof(double) * m, n, cudaMemcpyHostToDevice, st));
  TRY(launch_transpose_pad(st, dGs, m, n, dGsrm, ld_n, ld_m));

  std::vector<double> rho_all((size_t)L * m);
  for (int k = 0; k < L; ++k) {
    // per-row penalties (layers.cpp:210-215; row_kind on the SCALED bounds, problem.hpp:45-47)
    double* rho = rho_all.data() + (size_t)k * m;
    for (int i = 0; i < m; ++i) rho[i] = ((cs[i] == ds[i]) ? 1e3 : 1.0) * grid[k];
    TRYCUDA(cudaMemcpyAsync(dRho, rho, sizeof(double) * m, cudaMemcpyHostToDevice, st));
    scale_rows_kernel<<<blocks_for((size_t)m * n), 256, 0, st>>>(dGs, dRho, m, n, ld_m, drG);
    // M = Gs' (rho Gs): A = Gs' row-major == Gs column-major (n rows of length m)
    TRY(dense_gemm_run(gemm_n, st, dGs, ld_m, n, n128, drG, ld_m, dM, ld_n, 1.0));
    kkt_and_t_kernel<<<blocks_for((size_t)n * n), 256, 0, st>>>(dHs, dM, s.sigma, n, ld_n, dKkt, dT);
    // D = kkt^-1: Cholesky, then L Y = I and L' D = Y (layers.cpp:126-130)
    TRY(cholesky(dKkt, st));
    set_identity_kernel<<<blocks_for((size_t)n * n), 256, 0, st>>>(dY, ld_n, n);
    // L Y = I, block row by block row: only the columns c < k0 + nb of row block k0 are non-zero
    for (int k0 = 0; k0 < n; k0 += kNB) {
      const int nb = std::min(kNB, n - k0), ncols = k0 + nb, rem = n - k0 - nb;
      tri_block_solve_kernel<false><<<(ncols + 127) / 128, 128, 0, st>>>(dKkt, dY, ld_n, k0, nb, ncols);
      if (rem > 0)
        tile_update_kernel<false, false, false><<<dim3((rem + 63) / 64, (ncols + 63) / 64), 256, 0, st>>>(
            dY, dKkt, dY, ld_n, k0 + nb, n, 0, ncols, k0, nb);
    }
    // L' D = Y, from the last block row up
    for (int k0 = (n - 1) / kNB * kNB; k0 >= 0; k0 -= kNB) {
      const int nb = std::min(kNB, n - k0);
      tri_block_solve_kernel<true><<<(n + 127) / 128, 128, 0, st>>>(dKkt, dY, ld_n, k0, nb, n);
      if (k0 > 0)
        tile_update_kernel<true, false, false><<<dim3((k0 + 63) / 64, (n + 63) / 64), 256, 0, st>>>(
            dY, dKkt, dY, ld_n, 0, k0, 0, n, k0, nb);
    }
    mirror_lower_kernel<<<blocks_for((size_t)n * n), 256, 0, st>>>(dY, ld_n, n);  // dY = D
    TRY(read_fail(st, &info));
    if (info != 0) {
      set_error("KKT factorization failed: H + sigma I + G'rho G is not positive-definite");
      return cleanup(CQP_ERR_FACTORIZATION);
    }
    // GD = Gs D ; GDGt = Gs (GD)' ; DT = D T ; GDT = GD T   (layers.cpp:140-155)
    TRY(dense_gemm_run(gemm_n, st, dGsrm, ld_n, m, m128, dY, ld_n, dGD, ld_m, 1.0));
    TRY(launch_transpose_pad(st, dGD, m, n, dGDrm, ld_n, ld_m));
    TRY(dense_gemm_run(gemm_m, st, dGsrm, ld_n, m, m128, dGDrm, ld_n, dGDGt, ld_m, 1.0));
    TRY(dense_gemm_run(gemm_n, st, dY, ld_n, n, n128, dT, ld_n, dDT, ld_n, 1.0));
    TRY(dense_gemm_run(gemm_n, st, dGDrm, ld_n, m, m128, dT, ld_n, dGDT, ld_m, 1.0));
    assemble_w_kernel<<<blocks_for((size_t)D * h->Dpad), 256, 0, st>>>(
        n, m, h->Dpad, ld_n, ld_m, dDT, dGD, dGDT, dGDGt, dGs, dRho, h->W + (size_t)k * D * h->Dpad);
    double* dg = h->Dk + (size_t)k * nm * h->npad;
    TRY(launch_transpose_pad(st, dY, n, n, dg, h->npad, ld_n));
    TRY(launch_transpose_pad(st, dGD, m, n, dg + (size_t)n * h->npad, h->npad, ld_m));
    TRYCUDA(cudaGetLastError());
  }
  TRYCUDA(cudaMemcpyAsync(h->rho_vec, rho_all.data(), sizeof(double) * rho_all.size(), cudaMemcpyHostToDevice, st));

  // unscaled H, G, G' and scaled G in the solve kernel's row-major layout
  TRYCUDA(cudaMemcpyAsync(dscr, H, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, st));
  TRY(launch_transpose_pad(st, dscr, n, n, h->H, h->npad));
  TRY(launch_transpose_pad(st, dGs, m, n, h->Gs, h->npad, ld_m));
  TRYCUDA(cudaStreamSynchronize(st));
  TRYCUDA(cudaMemcpyAsync(dscr, G, sizeof(double) * (size_t)m * n, cudaMemcpyHostToDevice, st));
  TRY(launch_transpose_pad(st, dscr, m, n, h->Gr, h->npad));
  {
    // G' (n x m) in the kernel's row-major padded layout
    std::vector<double> Gt_host((size_t)n * m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < n; ++i) Gt_host[i + (size_t)j * n] = G[j + (size_t)i * m];
    TRYCUDA(cudaStreamSynchronize(st));
    TRYCUDA(cudaMemcpyAsync(dscr, Gt_host.data(), sizeof(double) * Gt_host.size(), cudaMemcpyHostToDevice, st));
    TRY(launch_transpose_pad(st, dscr, n, m, h->Gt, h->mpad));
    TRYCUDA(cudaStreamSynchronize(st));
  }
  TRY(upload_small(h, grid.data(), E.data(), F.data()));
  TRY(upload_vectors(h, g, c, d));
  TRY(prepare_streaming(h));
  TRY(cold_start(h));
  TRYCUDA(cudaStreamSynchronize(st));
  *out = h;
  return cleanup(CQP_OK);
#undef TRY
#undef TRYCUDA
}
