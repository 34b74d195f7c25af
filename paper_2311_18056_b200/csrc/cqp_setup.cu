// Offline stage on the device: Solver::Solver -> validate + precompute_all
// (/root/reference/proj/src/solver.cpp:180-186, src/problem.cpp:121-164,
//  src/layers.cpp:22-36 grid, :82-120 Ruiz, :122-131 D, :133-166 W, :189-228 precompute_all).
//
// This is setup work, off the hot path: the O(L n^3) dense algebra goes through cuSOLVER
// (potrf/potri) and cuBLAS (dgemm); the Ruiz equilibration (O(passes * n(n+m)) elementwise
// work on H and G) runs on the host exactly in the reference's operation order so that E, F
// and cost_scale are bit-identical to a host implementation.  The result is the same device
// layout cqp_create_from_layers produces: W_k row-major padded, [D_k; G D_k] row-major padded.
#include <cublas_v2.h>
#include <cusolverDn.h>

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

#define CQP_BLAS(call)                                                    \
  do {                                                                    \
    cublasStatus_t st__ = (call);                                         \
    if (st__ != CUBLAS_STATUS_SUCCESS) {                                  \
      set_error(std::string("cuBLAS error ") + std::to_string((int)st__) + " in " #call); \
      return cleanup(CQP_ERR_CUDA);                                              \
    }                                                                     \
  } while (0)
#define CQP_SOLVER(call)                                                  \
  do {                                                                    \
    cusolverStatus_t st__ = (call);                                       \
    if (st__ != CUSOLVER_STATUS_SUCCESS) {                                \
      set_error(std::string("cuSOLVER error ") + std::to_string((int)st__) + " in " #call); \
      return cleanup(CQP_ERR_CUDA);                                              \
    }                                                                     \
  } while (0)

// rG = diag(rho) G   (m x n column-major)
__global__ void scale_rows_kernel(const double* __restrict__ G, const double* __restrict__ rho,
                                  int m, int n, double* __restrict__ out) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < (size_t)m * n) out[idx] = rho[idx % m] * G[idx];
}

// kkt = H + sigma I + M ;  T = sigma I - M   (n x n column-major)
__global__ void kkt_and_t_kernel(const double* __restrict__ H, const double* __restrict__ M,
                                 double sigma, int n, double* __restrict__ kkt,
                                 double* __restrict__ T) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  const double s = (i == j) ? sigma : 0.0;
  kkt[idx] = (H[idx] + s) + M[idx];
  T[idx] = s - M[idx];
}

// potri leaves the inverse in the lower triangle: mirror it.
__global__ void mirror_lower_kernel(double* __restrict__ A, int n) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  if (i < j) A[idx] = A[(size_t)j + (size_t)i * n];
}

// Assemble W (row-major, ld = Dpad, pad zero) from its blocks (layers.cpp:149-162):
//   [ DT          2 DGt r         -DGt        ]      DT  = D T        (n x n, col-major)
//   [ GDT + G     2 GDGt r - I    -GDGt + 1/r ]      GD  = G D        (m x n)  DGt = GD'
//   [ r G         -r              I           ]      GDT = GD T (m x n), GDGt (m x m)
__global__ void assemble_w_kernel(int n, int m, int Dpad, const double* __restrict__ DT,
                                  const double* __restrict__ GD, const double* __restrict__ GDT,
                                  const double* __restrict__ GDGt, const double* __restrict__ Gs,
                                  const double* __restrict__ rho, double* __restrict__ W) {
  const int D = n + 2 * m;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)D * Dpad) return;
  const int r = (int)(idx / Dpad), c = (int)(idx % Dpad);
  double v = 0.0;
  if (c < D) {
    if (r < n) {
      if (c < n) v = DT[r + (size_t)c * n];
      else if (c < n + m) v = (2.0 * GD[(c - n) + (size_t)r * m]) * rho[c - n];
      else v = -GD[(c - n - m) + (size_t)r * m];
    } else if (r < n + m) {
      const int i = r - n;
      if (c < n) v = GDT[i + (size_t)c * m] + Gs[i + (size_t)c * m];
      else if (c < n + m) {
        const int j = c - n;
        v = (2.0 * GDGt[i + (size_t)j * m]) * rho[j] - (i == j ? 1.0 : 0.0);
      } else {
        const int j = c - n - m;
        v = -GDGt[i + (size_t)j * m] + (i == j ? 1.0 / rho[j] : 0.0);
      }
    } else {
      const int i = r - n - m;
      if (c < n) v = rho[i] * Gs[i + (size_t)c * m];
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

  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cqp_handle* h = nullptr;
  std::vector<double*> temps;
  auto cleanup = [&](int code) {
    for (double* p : temps) cudaFree(p);
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
    if (code != CQP_OK) { cqp_destroy(h); h = nullptr; }
    return code;
  };
  auto talloc = [&](double** p, size_t cnt) -> int {
    if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(double) * (cnt ? cnt : 1)) != cudaSuccess) return (int)CQP_ERR_CUDA;
    temps.push_back(*p);
    return (int)CQP_OK;
  };
#define TRY(expr) do { int rc__ = (expr); if (rc__) return cleanup(rc__); } while (0)
#define TRYCUDA(expr) do { cudaError_t e__ = (expr); if (e__ != cudaSuccess) return cleanup(cuda_fail(e__, #expr)); } while (0)

  if (cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS || cusolverDnCreate(&solver) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cuBLAS/cuSOLVER initialisation failed");
    return cleanup(CQP_ERR_CUDA);
  }

  // ---- PD check of H: LLT (problem.cpp:146-149) ----
  double *dH = nullptr, *dwork = nullptr;
  int* dinfo = nullptr;
  TRY(talloc(&dH, (size_t)n * n));
  TRYCUDA(cudaMalloc(reinterpret_cast<void**>(&dinfo), sizeof(int)));
  temps.push_back(reinterpret_cast<double*>(dinfo));
  int lwork_f = 0, lwork_i = 0;
  if (cusolverDnDpotrf_bufferSize(solver, CUBLAS_FILL_MODE_LOWER, n, dH, n, &lwork_f) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri_bufferSize(solver, CUBLAS_FILL_MODE_LOWER, n, dH, n, &lwork_i) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cuSOLVER workspace query failed");
    return cleanup(CQP_ERR_CUDA);
  }
  const int lwork = std::max(lwork_f, lwork_i);
  TRY(talloc(&dwork, (size_t)lwork));
  TRYCUDA(cudaMemcpy(dH, H, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice));
  int info = 0;
  if (cusolverDnDpotrf(solver, CUBLAS_FILL_MODE_LOWER, n, dH, n, dwork, lwork, dinfo) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cusolverDnDpotrf failed");
    return cleanup(CQP_ERR_CUDA);
  }
  TRYCUDA(cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
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
  CQP_BLAS(cublasSetStream(blas, h->stream));
  CQP_SOLVER(cusolverDnSetStream(solver, h->stream));

  const int D = h->D;
  const size_t nm = (size_t)n + m;
  double *dHs, *dGs, *dRho, *drG, *dM, *dKkt, *dT, *dGD, *dGDGt, *dDT, *dGDT, *dscr;
  TRY(talloc(&dHs, (size_t)n * n)); TRY(talloc(&dGs, (size_t)m * n)); TRY(talloc(&dRho, (size_t)m));
  TRY(talloc(&drG, (size_t)m * n)); TRY(talloc(&dM, (size_t)n * n)); TRY(talloc(&dKkt, (size_t)n * n));
  TRY(talloc(&dT, (size_t)n * n)); TRY(talloc(&dGD, (size_t)m * n)); TRY(talloc(&dGDGt, (size_t)m * m));
  TRY(talloc(&dDT, (size_t)n * n)); TRY(talloc(&dGDT, (size_t)m * n));
  TRY(talloc(&dscr, std::max((size_t)n * n, (size_t)m * n)));
  TRYCUDA(cudaMemcpyAsync(dHs, Hs.data(), sizeof(double) * Hs.size(), cudaMemcpyHostToDevice, h->stream));
  TRYCUDA(cudaMemcpyAsync(dGs, Gs.data(), sizeof(double) * Gs.size(), cudaMemcpyHostToDevice, h->stream));

  std::vector<double> rho_all((size_t)L * m);
  const double one = 1.0, zero = 0.0;
  for (int k = 0; k < L; ++k) {
    // per-row penalties (layers.cpp:210-215; row_kind on the SCALED bounds, problem.hpp:45-47)
    double* rho = rho_all.data() + (size_t)k * m;
    for (int i = 0; i < m; ++i) rho[i] = ((cs[i] == ds[i]) ? 1e3 : 1.0) * grid[k];
    TRYCUDA(cudaMemcpyAsync(dRho, rho, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream));
    scale_rows_kernel<<<blocks_for((size_t)m * n), 256, 0, h->stream>>>(dGs, dRho, m, n, drG);
    // M = Gs' (rho Gs)
    CQP_BLAS(cublasDgemm(blas, CUBLAS_OP_T, CUBLAS_OP_N, n, n, m, &one, dGs, m, drG, m, &zero, dM, n));
    kkt_and_t_kernel<<<blocks_for((size_t)n * n), 256, 0, h->stream>>>(dHs, dM, s.sigma, n, dKkt, dT);
    // D = kkt^-1 via Cholesky (layers.cpp:126-130)
    if (cusolverDnDpotrf(solver, CUBLAS_FILL_MODE_LOWER, n, dKkt, n, dwork, lwork, dinfo) != CUSOLVER_STATUS_SUCCESS) {
      set_error("cusolverDnDpotrf failed"); return cleanup(CQP_ERR_CUDA);
    }
    TRYCUDA(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TRYCUDA(cudaStreamSynchronize(h->stream));
    if (info != 0) {
      set_error("KKT factorization failed: H + sigma I + G'rho G is not positive-definite");
      return cleanup(CQP_ERR_FACTORIZATION);
    }
    if (cusolverDnDpotri(solver, CUBLAS_FILL_MODE_LOWER, n, dKkt, n, dwork, lwork, dinfo) != CUSOLVER_STATUS_SUCCESS) {
      set_error("cusolverDnDpotri failed"); return cleanup(CQP_ERR_CUDA);
    }
    mirror_lower_kernel<<<blocks_for((size_t)n * n), 256, 0, h->stream>>>(dKkt, n);  // dKkt = D
    // GD = Gs D ; GDGt = Gs (GD)' ; DT = D T ; GDT = GD T
    CQP_BLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, m, n, n, &one, dGs, m, dKkt, n, &zero, dGD, m));
    CQP_BLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_T, m, m, n, &one, dGs, m, dGD, m, &zero, dGDGt, m));
    CQP_BLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, dKkt, n, dT, n, &zero, dDT, n));
    CQP_BLAS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_N, m, n, n, &one, dGD, m, dT, n, &zero, dGDT, m));
    assemble_w_kernel<<<blocks_for((size_t)D * h->Dpad), 256, 0, h->stream>>>(
        n, m, h->Dpad, dDT, dGD, dGDT, dGDGt, dGs, dRho, h->W + (size_t)k * D * h->Dpad);
    double* dg = h->Dk + (size_t)k * nm * h->npad;
    TRY(launch_transpose_pad(h->stream, dKkt, n, n, dg, h->npad));
    TRY(launch_transpose_pad(h->stream, dGD, m, n, dg + (size_t)n * h->npad, h->npad));
    TRYCUDA(cudaGetLastError());
  }
  TRYCUDA(cudaMemcpyAsync(h->rho_vec, rho_all.data(), sizeof(double) * rho_all.size(), cudaMemcpyHostToDevice, h->stream));

  // unscaled H, G, G' and scaled G in the solve kernel's row-major layout
  TRYCUDA(cudaMemcpyAsync(dscr, H, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice, h->stream));
  TRY(launch_transpose_pad(h->stream, dscr, n, n, h->H, h->npad));
  TRY(launch_transpose_pad(h->stream, dGs, m, n, h->Gs, h->npad));
  TRYCUDA(cudaMemcpyAsync(drG, G, sizeof(double) * (size_t)m * n, cudaMemcpyHostToDevice, h->stream));
  TRY(launch_transpose_pad(h->stream, drG, m, n, h->Gr, h->npad));
  {
    // G' (n x m) in the kernel's row-major padded layout
    std::vector<double> Gt_host((size_t)n * m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < n; ++i) Gt_host[i + (size_t)j * n] = G[j + (size_t)i * m];
    TRYCUDA(cudaMemcpyAsync(dGDT, Gt_host.data(), sizeof(double) * Gt_host.size(), cudaMemcpyHostToDevice, h->stream));
    TRY(launch_transpose_pad(h->stream, dGDT, n, m, h->Gt, h->mpad));
    TRYCUDA(cudaStreamSynchronize(h->stream));
  }
  TRY(upload_small(h, grid.data(), E.data(), F.data()));
  TRY(upload_vectors(h, g, c, d));
  TRY(cold_start(h));
  TRYCUDA(cudaStreamSynchronize(h->stream));
  *out = h;
  return cleanup(CQP_OK);
#undef TRY
#undef TRYCUDA
}
