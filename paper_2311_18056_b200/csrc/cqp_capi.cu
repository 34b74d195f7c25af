// C ABI of libcqp_b200.so (include/cqp_b200.h): handle management, uploads, result download.
// Mirrors the reference's Solver lifecycle (/root/reference/proj/src/solver.cpp:180-218).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>

#include "cqp_internal.h"

namespace cqp {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what;
  return CQP_ERR_CUDA;
}

namespace {

template <typename T>
int dev_alloc(T** p, size_t count) {
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1)));
  return CQP_OK;
}

size_t result_bytes(int n, int m, int cap) {
  return sizeof(DevResultHead) + sizeof(int) * 4 * (size_t)cap + sizeof(double) * 2 * (size_t)cap +
         sizeof(double) * ((size_t)n + 2 * (size_t)m) + sizeof(double) * (size_t)n /* u0, nu <= n */;
}

int ensure_result_capacity(cqp_handle* h, int cap) {
  if (cap <= h->res_cap) return CQP_OK;
  // The result record lives in host-mapped pinned memory: the kernel writes it straight over PCIe
  // (posted writes, a few KB), so a solve needs no device->host copy after the launch.
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->hres) cudaFreeHost(h->hres);
  h->dres = h->hres = nullptr;
  h->res_cap = cap;
  h->res_bytes = result_bytes(h->n, h->m, cap);
  CQP_CUDA(cudaHostAlloc(&h->hres, h->res_bytes, cudaHostAllocMapped));
  CQP_CUDA(cudaHostGetDevicePointer(&h->dres, h->hres, 0));
  return CQP_OK;
}

// solver.cpp:29-34
int check_settings(const cqp_settings& s) {
  if (s.check_interval < 1) {
    set_error("check_interval must be >= 1");
    return CQP_ERR_SETTINGS;
  }
  if (s.max_iters < s.check_interval) {
    set_error("max_iters must be >= check_interval");
    return CQP_ERR_SETTINGS;
  }
  return CQP_OK;
}

// Upload a column-major host matrix as a row-major, even-padded device matrix.
int upload_transposed(cqp_handle* h, const double* host, int rows, int cols, double* dst, int ld,
                      double* scratch) {
  CQP_CUDA(cudaMemcpyAsync(scratch, host, sizeof(double) * (size_t)rows * cols,
                           cudaMemcpyHostToDevice, h->stream));
  return launch_transpose_pad(h->stream, scratch, rows, cols, dst, ld);
}

}  // namespace

// Allocates everything whose size depends only on (n, m, L) and fills the fields shared by both
// creation paths.  Device buffers for the ladder are allocated here and filled by the caller.
int handle_alloc(cqp_handle** out, int n, int m, int L, const cqp_settings& s, int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    set_error("no CUDA device available: libcqp_b200 has no CPU fallback");
    return CQP_ERR_CUDA;
  }
  if (device < 0) CQP_CUDA(cudaGetDevice(&device));
  CQP_CUDA(cudaSetDevice(device));
  cqp_handle* h = new cqp_handle();
  *out = h;
  h->n = n; h->m = m; h->D = n + 2 * m; h->L = L;
  h->npad = pad2(n); h->mpad = pad2(m); h->Dpad = pad2(h->D);
  h->s = s;
  h->device = device;
  cudaDeviceProp prop;
  CQP_CUDA(cudaGetDeviceProperties(&prop, device));
  h->num_sms = prop.multiProcessorCount;
  int coop = 0;
  CQP_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) {
    set_error("device does not support cooperative launch");
    return CQP_ERR_CUDA;
  }
  CQP_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CQP_CUDA(cudaEventCreate(&h->ev0));
  CQP_CUDA(cudaEventCreate(&h->ev1));
  const size_t D = h->D, nm = (size_t)n + m;
  int rc;
  if ((rc = dev_alloc(&h->W, (size_t)L * D * h->Dpad))) return rc;
  if ((rc = dev_alloc(&h->Dk, (size_t)L * nm * h->npad))) return rc;
  if ((rc = dev_alloc(&h->H, (size_t)n * h->npad))) return rc;
  if ((rc = dev_alloc(&h->Gr, (size_t)m * h->npad))) return rc;
  if ((rc = dev_alloc(&h->Gt, (size_t)n * h->mpad))) return rc;
  if ((rc = dev_alloc(&h->Gs, (size_t)m * h->npad))) return rc;
  if ((rc = dev_alloc(&h->E, (size_t)n))) return rc;
  if ((rc = dev_alloc(&h->F, (size_t)m))) return rc;
  if ((rc = dev_alloc(&h->dgrid, (size_t)L))) return rc;
  if ((rc = dev_alloc(&h->dlog_grid, 2 * (size_t)L))) return rc;  // log10(grid), then the bounds between neighbours
  if ((rc = dev_alloc(&h->g, nm + m))) return rc;
  h->c = h->g + n;
  h->d = h->c + m;
  h->ring_ld = (h->Dpad + 15) / 16 * 16;  // ring slots start on their own 128-byte L2 lines
  if ((rc = dev_alloc(&h->vq, 4 * (size_t)h->ring_ld))) return rc;
  if ((rc = dev_alloc(&h->state, 2))) return rc;
  if ((rc = dev_alloc(&h->barrier, 2))) return rc;
  CQP_CUDA(cudaMemset(h->barrier, 0, 2 * sizeof(unsigned)));
  CQP_CUDA(cudaStreamSynchronize(0));  // legacy-stream memset vs the handle's non-blocking stream
  if ((rc = dev_alloc(&h->partial, 2 * 8 * (size_t)(h->num_sms + 1)))) return rc;  // [pass parity][CTA][8]
  if ((rc = dev_alloc(&h->rho_vec, (size_t)L * m))) return rc;
  if ((rc = dev_alloc(&h->dtmp, (size_t)h->Dpad))) return rc;
  CQP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->hstage), sizeof(double) * (nm + m)));
  CQP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h->dbg_host), sizeof(int) * 256, cudaHostAllocMapped));
  std::memset(h->dbg_host, 0, sizeof(int) * 256);
  CQP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dbg_dev), h->dbg_host, 0));
  if ((rc = ensure_result_capacity(h, s.max_iters / s.check_interval + 2))) return rc;
  if ((rc = configure_launch(h))) return rc;
  return CQP_OK;
}

// grid values + their log10 (host libm, so the table equals what the reference recomputes at
// every selection, layers.cpp:43), E, F.
int upload_small(cqp_handle* h, const double* grid, const double* E, const double* F) {
  h->grid.assign(grid, grid + h->L);
  h->E_host.assign(E, E + h->n);
  h->F_host.assign(F, F + h->m);
  std::vector<double> lg(2 * (size_t)h->L, 0.0);
  for (int k = 0; k < h->L; ++k) lg[k] = std::log10(grid[k]);
  // bounds between neighbours for nearest_grid_index_fast (cqp_device.cuh); only for an ascending grid
  h->grid_bounds = true;
  for (int k = 0; k + 1 < h->L; ++k) {
    if (!(grid[k] > 0.0) || !(grid[k + 1] > grid[k])) h->grid_bounds = false;
    lg[h->L + k] = std::sqrt(grid[k] * grid[k + 1]);
  }
  CQP_CUDA(cudaMemcpyAsync(h->dgrid, grid, sizeof(double) * h->L, cudaMemcpyHostToDevice, h->stream));
  CQP_CUDA(cudaMemcpyAsync(h->dlog_grid, lg.data(), sizeof(double) * 2 * h->L, cudaMemcpyHostToDevice, h->stream));
  CQP_CUDA(cudaMemcpyAsync(h->E, E, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->stream));
  CQP_CUDA(cudaMemcpyAsync(h->F, F, sizeof(double) * h->m, cudaMemcpyHostToDevice, h->stream));
  CQP_CUDA(cudaStreamSynchronize(h->stream));  // lg is a local
  return CQP_OK;
}

int upload_vectors(cqp_handle* h, const double* g, const double* c, const double* d) {
  const int n = h->n, m = h->m;
  std::memcpy(h->hstage, g, sizeof(double) * n);
  std::memcpy(h->hstage + n, c, sizeof(double) * m);
  std::memcpy(h->hstage + n + m, d, sizeof(double) * m);
  h->c_host.assign(c, c + m);
  h->d_host.assign(d, d + m);
  h->vectors_device_only = false;
  CQP_CUDA(cudaMemcpyAsync(h->g, h->hstage, sizeof(double) * ((size_t)n + 2 * (size_t)m),
                           cudaMemcpyHostToDevice, h->stream));
  return CQP_OK;
}

// ---- resident MPC server (cqp_mpc_server_start) ------------------------------------------------
// One persistent kernel keeps W (registers / shared memory), the scaling vectors and the residual
// rows on the SMs and serves control steps from a host-mapped mailbox: the host writes x0 and a
// request number, the kernel instantiates, refreshes z, iterates, extracts u0, writes the result
// record (host-mapped) and answers with the request number.  No CUDA call on the per-step path.
// The kernel leaves by itself when told to stop or when idle for srv_idle_ns (a crashed host never
// leaves a spinning kernel behind); the next step relaunches it.
int server_stop(cqp_handle* h) {
  if (!h->srv_running) return CQP_OK;
  reinterpret_cast<volatile unsigned long long*>(h->mb_host)[kMbStop] = 1ull;
  const cudaError_t e = cudaStreamSynchronize(h->stream);
  h->srv_running = false;
  if (e != cudaSuccess) return cuda_fail(e, "mpc server kernel");
  return CQP_OK;
}

static int server_launch_from(cqp_handle* h, int k, unsigned long long served) {
  int rc = server_stop(h);
  if (rc) return rc;
  if (!h->mb_host) {
    CQP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h->mb_host), sizeof(unsigned long long) * kMbWords, cudaHostAllocMapped));
    CQP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->mb_dev), h->mb_host, 0));
    std::memset(h->mb_host, 0, sizeof(unsigned long long) * kMbWords);
    if ((rc = dev_alloc(&h->srv_seq, 1))) return rc;
  }
  if ((rc = ensure_result_capacity(h, k / h->s.check_interval + 2))) return rc;
  volatile unsigned long long* mb = h->mb_host;
  mb[kMbStop] = 0ull; mb[kMbExited] = 0ull;
  if (served == h->srv_req) { mb[kMbReq] = served; mb[kMbResp] = served; }  // (else a request is pending: keep it)
  CQP_CUDA(cudaMemcpyAsync(h->srv_seq, &served, sizeof(unsigned long long), cudaMemcpyHostToDevice, h->stream));
  CQP_CUDA(cudaStreamSynchronize(h->stream));  // (pageable source)
  h->srv_k = k;
  h->srv_running = true;
  h->mpc_extract = true;
  h->vectors_device_only = true;
  const unsigned long long newest = h->srv_req;
  h->srv_req = served;  // (launch_run hands RunParams::served = srv_req to the kernel)
  rc = launch_run(h, false, k, true);
  h->srv_req = newest;
  h->mpc_extract = false;
  if (rc) { h->srv_running = false; return rc; }
  return CQP_OK;
}

int server_launch(cqp_handle* h, int k) { return server_launch_from(h, k, h->srv_req); }

// One control step through the resident kernel: post x0, wait for the answer, read the record.
static int server_step(cqp_handle* h, const double* x0, int k, double* u0, cqp_result* out) {
  const auto t0 = std::chrono::steady_clock::now();
  int rc;
  if (h->srv_running && h->srv_k != k && (rc = server_stop(h))) return rc;
  if (h->srv_running && h->mb_host[kMbExited] != 0ull && (rc = server_stop(h))) return rc;  // idle timeout
  if (!h->srv_running && (rc = server_launch(h, k))) return rc;
  volatile unsigned long long* mb = h->mb_host;
  std::memcpy(h->mb_host + kMbX0, x0, sizeof(double) * h->mpc_nx);
  mb[kMbWantFull] = (out && (out->y || out->z || out->lambda)) ? 1ull : 0ull;
  std::atomic_thread_fence(std::memory_order_release);
  const unsigned long long seq = ++h->srv_req;
  mb[kMbReq] = seq;
  unsigned spins = 0;
  while (mb[kMbResp] != seq) {
    if ((++spins & 0x3FF) != 0) continue;
    if (mb[kMbExited] != 0ull) {
      // the kernel left its loop (idle timeout) around the time this request was posted
      if ((rc = server_stop(h))) return rc;
      if (mb[kMbResp] == seq) break;                        // it had answered before leaving
      if ((rc = server_launch_from(h, k, seq - 1))) return rc;  // run it again: it finds the request
    } else if ((spins & 0xFFFFF) == 0) {
      const cudaError_t q = cudaStreamQuery(h->stream);
      if (q != cudaErrorNotReady && mb[kMbResp] != seq && mb[kMbExited] == 0ull) {
        // the kernel is gone without an answer and without the exit mark: a fault (watchdog trap)
        h->srv_running = false;
        const int* d = h->dbg_host;
        set_error(std::string("mpc server kernel failed: ") + cudaGetErrorString(q) +
                  (d && d[0] ? " (watchdog: where=" + std::to_string(d[1]) + " iter=" + std::to_string(d[2]) + ")" : std::string()));
        return CQP_ERR_CUDA;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  h->srv_last_device_us = 1e-3 * (double)mb[kMbStepNs];
  const unsigned char* base = static_cast<const unsigned char*>(h->hres);
  const DevResultHead* head = reinterpret_cast<const DevResultHead*>(base);
  const int cap = h->res_cap;
  size_t off = sizeof(DevResultHead) + sizeof(int) * 4 * (size_t)cap + sizeof(double) * 2 * (size_t)cap;
  const double* y = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->n;
  const double* z = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->m;
  const double* lam = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->m;
  if (u0) std::memcpy(u0, base + off, sizeof(double) * (size_t)h->mpc_nu);
  if (out) {
    out->status = head->status; out->iterations = head->iterations;
    out->r_prim = head->r_prim; out->r_dual = head->r_dual;
    if (out->y) std::memcpy(out->y, y, sizeof(double) * h->n);
    if (out->z) std::memcpy(out->z, z, sizeof(double) * h->m);
    if (out->lambda) std::memcpy(out->lambda, lam, sizeof(double) * h->m);
    out->rho_trace_len = head->n_trace; out->history_len = head->n_hist;
    const int* trace = reinterpret_cast<const int*>(base + sizeof(DevResultHead));
    if (out->rho_trace)
      for (int i = 0; i < std::min(std::min(head->n_trace, out->rho_trace_cap), cap); ++i) out->rho_trace[i] = {trace[2 * i], trace[2 * i + 1]};
    out->kernel_us = h->srv_last_device_us;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  h->srv_last_wall_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  return CQP_OK;
}

int cold_start(cqp_handle* h) {
  // ring invariant between launches: slot 0 = iterate (zero), slots 1..3 = sentinel (all ones)
  CQP_CUDA(cudaMemsetAsync(h->vq, 0, sizeof(double) * (size_t)h->Dpad, h->stream));
  CQP_CUDA(cudaMemsetAsync(h->vq + h->ring_ld, 0xFF, sizeof(double) * 3 * (size_t)h->ring_ld, h->stream));
  return launch_set_state(h, h->initial_index);
}

}  // namespace cqp

using namespace cqp;

// ---- measurement helper: read bandwidth of a device buffer -----------------------------------
static __global__ void __launch_bounds__(512) read_bw_kernel(const double2* __restrict__ buf, size_t n2, int passes,
                                                      double* __restrict__ sink) {
  double acc = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int pass = 0; pass < passes; ++pass) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n2; i += 8 * stride) {  // 8 independent 16-byte loads in flight per thread
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(buf + i + u * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) {
      const double2 v = __ldcg(buf + i);
      acc += v.x + v.y;
    }
  }
  if (acc == 123.456) *sink = acc;  // keeps the loads alive
}


extern "C" {

void cqp_default_settings(cqp_settings* s) {
  // solver.hpp:43-53, layers.hpp:100-104
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

const char* cqp_last_error(void) { return g_last_error.c_str(); }

int cqp_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  return count;
}

int cqp_create_from_layers(cqp_handle** out, int n, int m, int L, const double* const* W,
                           const double* const* Dk, const double* const* GDk,
                           const double* grid_values, int initial_index, const double* H,
                           const double* g, const double* G, const double* c, const double* d,
                           const double* Gs, const double* E, const double* F, double cost_scale,
                           const cqp_settings* settings, int device) {
  if (!out) return CQP_ERR_ARGUMENT;
  *out = nullptr;
  if (n < 1 || m < 1 || L < 2 || initial_index < 0 || initial_index >= L) {
    set_error("cqp_create_from_layers: bad dimensions");
    return CQP_ERR_DIMENSION;
  }
  cqp_settings s;
  if (settings) s = *settings; else cqp_default_settings(&s);
  int rc = check_settings(s);
  if (rc) return rc;
  cqp_handle* h = nullptr;
  rc = handle_alloc(&h, n, m, L, s, device);
  if (rc) { cqp_destroy(h); return rc; }
  h->initial_index = initial_index;
  h->cost_scale = cost_scale;
  const size_t D = h->D, nm = (size_t)n + m;
  double* scratch = nullptr;
  if ((rc = dev_alloc(&scratch, D * D))) { cqp_destroy(h); return rc; }
  auto fail = [&](int code) { cudaFree(scratch); cqp_destroy(h); return code; };
  for (int k = 0; k < L; ++k) {
    if ((rc = upload_transposed(h, W[k], (int)D, (int)D, h->W + (size_t)k * D * h->Dpad, h->Dpad, scratch))) return fail(rc);
    double* dg = h->Dk + (size_t)k * nm * h->npad;
    if ((rc = upload_transposed(h, Dk[k], n, n, dg, h->npad, scratch))) return fail(rc);
    if ((rc = upload_transposed(h, GDk[k], m, n, dg + (size_t)n * h->npad, h->npad, scratch))) return fail(rc);
  }
  if ((rc = upload_transposed(h, H, n, n, h->H, h->npad, scratch))) return fail(rc);
  if ((rc = upload_transposed(h, G, m, n, h->Gr, h->npad, scratch))) return fail(rc);
  if ((rc = upload_transposed(h, Gs, m, n, h->Gs, h->npad, scratch))) return fail(rc);
  {
    // G' (n x m) in the kernel's row-major padded layout
    std::vector<double> Gt_host((size_t)n * m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < n; ++i) Gt_host[i + (size_t)j * n] = G[j + (size_t)i * m];
    if ((rc = upload_transposed(h, Gt_host.data(), n, m, h->Gt, h->mpad, scratch))) return fail(rc);
    CQP_CUDA(cudaStreamSynchronize(h->stream));
  }
  // per-row penalties (layers.cpp:210-215): equality rows (scaled c == d) get eq_scale = 1e3
  {
    std::vector<double> rho((size_t)L * m);
    for (int k = 0; k < L; ++k)
      for (int i = 0; i < m; ++i) {
        const bool eq = (F[i] * c[i]) == (F[i] * d[i]);
        rho[(size_t)k * m + i] = (eq ? 1e3 : 1.0) * grid_values[k];
      }
    CQP_CUDA(cudaMemcpy(h->rho_vec, rho.data(), sizeof(double) * rho.size(), cudaMemcpyHostToDevice));
    CQP_CUDA(cudaStreamSynchronize(0));  // (pageable source: the DMA may outlive the call)
  }
  if ((rc = upload_small(h, grid_values, E, F))) return fail(rc);
  if ((rc = upload_vectors(h, g, c, d))) return fail(rc);
  if ((rc = prepare_streaming(h))) return fail(rc);
  if ((rc = cold_start(h))) return fail(rc);
  CQP_CUDA(cudaStreamSynchronize(h->stream));
  cudaFree(scratch);
  *out = h;
  return CQP_OK;
}

// Every entry point that touches the handle's state or stream first retires the resident MPC kernel
// (it owns the SMs and the iterate while it runs).
#define CQP_QUIESCE(h)                                  \
  do {                                                  \
    if ((h)->srv_running) {                             \
      if (int rc__ = ::cqp::server_stop(h)) return rc__; \
    }                                                   \
  } while (0)

void cqp_destroy(cqp_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  server_stop(h);
  if (h->mb_host) cudaFreeHost(h->mb_host);
  cudaFree(h->srv_seq);
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->W); cudaFree(h->Wt); cudaFree(h->Dk); cudaFree(h->H); cudaFree(h->Gr); cudaFree(h->Gt);
  cudaFree(h->Gs); cudaFree(h->E); cudaFree(h->F); cudaFree(h->dgrid); cudaFree(h->dlog_grid);
  cudaFree(h->g); cudaFree(h->vq); cudaFree(h->state); cudaFree(h->barrier);
  cudaFree(h->partial); cudaFree(h->rho_vec); cudaFree(h->dtmp);  // (dres aliases the mapped hres)
  if (h->hres) cudaFreeHost(h->hres);
  if (h->hstage) cudaFreeHost(h->hstage);
  if (h->hx0) cudaFreeHost(h->hx0);
  cudaFree(h->mpc_og); cudaFree(h->mpc_oc); cudaFree(h->mpc_cb); cudaFree(h->mpc_db);
  cudaFree(h->mpc_K); cudaFree(h->mpc_ulo); cudaFree(h->mpc_uhi); cudaFree(h->mpc_x0);
  if (h->dbg_host) cudaFreeHost(h->dbg_host);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int cqp_update_vectors(cqp_handle* h, const double* g, const double* c, const double* d) {
  if (!h || !g || !c || !d) { set_error("update_vectors: null argument"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  return upload_vectors(h, g, c, d);
}

int cqp_cold_start(cqp_handle* h) {
  if (!h) return CQP_ERR_ARGUMENT;
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  return cold_start(h);
}

int cqp_warm_start(cqp_handle* h, const double* y, const double* lambda, int layer_index) {
  if (!h || !y || !lambda) { set_error("warm_start: null argument"); return CQP_ERR_ARGUMENT; }
  if (layer_index >= h->L) { set_error("warm_start: layer index out of range"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  const int n = h->n, m = h->m;
  CQP_CUDA(cudaStreamSynchronize(h->stream));  // hstage may still feed an update_vectors copy
  double* hs = h->hstage;
  double* ds = h->dtmp;
  std::memcpy(hs, y, sizeof(double) * n);
  std::memcpy(hs + n, lambda, sizeof(double) * m);
  CQP_CUDA(cudaMemcpyAsync(ds, hs, sizeof(double) * ((size_t)n + m), cudaMemcpyHostToDevice, h->stream));
  int rc = launch_warm_start(h, ds, ds + n, layer_index < 0 ? h->initial_index : layer_index);
  if (rc) return rc;
  CQP_CUDA(cudaStreamSynchronize(h->stream));  // hstage is reused by update_vectors
  return CQP_OK;
}

int cqp_refresh_z(cqp_handle* h) {
  if (!h) return CQP_ERR_ARGUMENT;
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  // Same device code as the fused step's prologue (run kernel, zero iterations), so that
  // update_vectors + refresh_z + fixed_iters(k) and cqp_mpc_step agree bit for bit.
  return launch_run(h, false, 0, true);
}

static int run_and_fetch(cqp_handle* h, bool early_exit, int total, bool refresh, cqp_result* out,
                         std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(),
                         double* u0 = nullptr) {
  int rc = ensure_result_capacity(h, total / h->s.check_interval + 2);
  if (rc) return rc;
  CQP_CUDA(cudaEventRecord(h->ev0, h->stream));
  if ((rc = launch_run(h, early_exit, total, refresh))) return rc;
  CQP_CUDA(cudaEventRecord(h->ev1, h->stream));
  {
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
      const int* d = h->dbg_host;
      set_error(std::string("solve kernel failed: ") + cudaGetErrorString(e) +
                (d && d[0] ? " (watchdog: where=" + std::to_string(d[1]) + " iter=" + std::to_string(d[2]) +
                                 " cta=" + std::to_string(d[3]) + " thread=" + std::to_string(d[4]) + ")"
                           : std::string()));
      return CQP_ERR_CUDA;
    }
  }
  const unsigned char* base = static_cast<const unsigned char*>(h->hres);
  const DevResultHead* head = reinterpret_cast<const DevResultHead*>(base);
  size_t off = sizeof(DevResultHead);
  const int cap = h->res_cap;
  const int* trace = reinterpret_cast<const int*>(base + off); off += sizeof(int) * 2 * (size_t)cap;
  const int* hist_i = reinterpret_cast<const int*>(base + off); off += sizeof(int) * 2 * (size_t)cap;
  const double* hist_r = reinterpret_cast<const double*>(base + off); off += sizeof(double) * 2 * (size_t)cap;
  const double* y = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->n;
  const double* z = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->m;
  const double* lam = reinterpret_cast<const double*>(base + off); off += sizeof(double) * (size_t)h->m;
  if (u0) std::memcpy(u0, base + off, sizeof(double) * (size_t)h->mpc_nu);
  if (out) {
    out->status = head->status;
    out->iterations = head->iterations;
    out->r_prim = head->r_prim;
    out->r_dual = head->r_dual;
    if (out->y) std::memcpy(out->y, y, sizeof(double) * h->n);
    if (out->z) std::memcpy(out->z, z, sizeof(double) * h->m);
    if (out->lambda) std::memcpy(out->lambda, lam, sizeof(double) * h->m);
    out->rho_trace_len = head->n_trace;
    out->history_len = head->n_hist;
    if (out->rho_trace) {
      const int cnt = std::min(std::min(head->n_trace, out->rho_trace_cap), cap);
      for (int i = 0; i < cnt; ++i) out->rho_trace[i] = {trace[2 * i], trace[2 * i + 1]};
    }
    if (out->history) {
      const int cnt = std::min(std::min(head->n_hist, out->history_cap), cap);
      for (int i = 0; i < cnt; ++i)
        out->history[i] = {hist_i[2 * i], hist_r[2 * i], hist_r[2 * i + 1], hist_i[2 * i + 1]};
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    out->kernel_us = 1e3 * (double)ms;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return CQP_OK;
}

int cqp_solve(cqp_handle* h, cqp_result* out) {
  if (!h) return CQP_ERR_ARGUMENT;
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  return run_and_fetch(h, true, h->s.max_iters, false, out);
}

int cqp_fixed_iters(cqp_handle* h, int k, cqp_result* out) {
  if (!h) return CQP_ERR_ARGUMENT;
  if (k < 1) { set_error("fixed_iters: k must be >= 1"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  return run_and_fetch(h, false, k, false, out);
}

int cqp_mpc_step(cqp_handle* h, const double* g, const double* c, const double* d, int k,
                 cqp_result* out) {
  if (!h || !g || !c || !d) { set_error("mpc_step: null argument"); return CQP_ERR_ARGUMENT; }
  if (k < 1) { set_error("mpc_step: k must be >= 1"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  const auto t0 = std::chrono::steady_clock::now();  // wall_ms of a fused step includes the upload
  int rc = upload_vectors(h, g, c, d);
  if (rc) return rc;
  return run_and_fetch(h, false, k, true, out, t0);
}

int cqp_mpc_set_template(cqp_handle* h, int nx, int nu, const double* offset_g, const double* offset_c,
                         const double* c_base, const double* d_base, const double* K, const double* u_lo,
                         const double* u_hi) {
  if (!h || !offset_g || !offset_c || !c_base || !d_base || !K || !u_lo || !u_hi) {
    set_error("mpc_set_template: null argument");
    return CQP_ERR_ARGUMENT;
  }
  if (nx < 1 || nu < 1 || nu > h->n) { set_error("mpc_set_template: bad dimensions"); return CQP_ERR_DIMENSION; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  CQP_CUDA(cudaStreamSynchronize(h->stream));
  const int n = h->n, m = h->m;
  cudaFree(h->mpc_og); cudaFree(h->mpc_oc); cudaFree(h->mpc_cb); cudaFree(h->mpc_db);
  cudaFree(h->mpc_K); cudaFree(h->mpc_ulo); cudaFree(h->mpc_uhi); cudaFree(h->mpc_x0);
  if (h->hx0) cudaFreeHost(h->hx0);
  h->mpc_og = h->mpc_oc = h->mpc_cb = h->mpc_db = h->mpc_K = h->mpc_ulo = h->mpc_uhi = h->mpc_x0 = h->hx0 = nullptr;
  h->mpc_nx = nx; h->mpc_nu = nu; h->mpc_nxpad = pad2(nx);
  int rc;
  if ((rc = dev_alloc(&h->mpc_og, (size_t)n * h->mpc_nxpad))) return rc;
  if ((rc = dev_alloc(&h->mpc_oc, (size_t)m * h->mpc_nxpad))) return rc;
  if ((rc = dev_alloc(&h->mpc_cb, (size_t)m))) return rc;
  if ((rc = dev_alloc(&h->mpc_db, (size_t)m))) return rc;
  if ((rc = dev_alloc(&h->mpc_K, (size_t)nu * h->mpc_nxpad))) return rc;
  if ((rc = dev_alloc(&h->mpc_ulo, (size_t)nu))) return rc;
  if ((rc = dev_alloc(&h->mpc_uhi, (size_t)nu))) return rc;
  if ((rc = dev_alloc(&h->mpc_x0, (size_t)nx))) return rc;
  CQP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->hx0), sizeof(double) * nx));
  double* scratch = nullptr;
  const size_t big = (size_t)std::max(std::max(n, m), nu) * nx;
  if ((rc = dev_alloc(&scratch, big))) return rc;
  auto done = [&](int code) { cudaStreamSynchronize(h->stream); cudaFree(scratch); return code; };
  if ((rc = upload_transposed(h, offset_g, n, nx, h->mpc_og, h->mpc_nxpad, scratch))) return done(rc);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
  if ((rc = upload_transposed(h, offset_c, m, nx, h->mpc_oc, h->mpc_nxpad, scratch))) return done(rc);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
  if ((rc = upload_transposed(h, K, nu, nx, h->mpc_K, h->mpc_nxpad, scratch))) return done(rc);
  if (cudaMemcpyAsync(h->mpc_cb, c_base, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
      cudaMemcpyAsync(h->mpc_db, d_base, sizeof(double) * m, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
      cudaMemcpyAsync(h->mpc_ulo, u_lo, sizeof(double) * nu, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
      cudaMemcpyAsync(h->mpc_uhi, u_hi, sizeof(double) * nu, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "mpc_set_template upload"));
  return done(CQP_OK);
}

int cqp_mpc_step_x0(cqp_handle* h, const double* x0, int k, double* u0, cqp_result* out) {
  if (!h || !x0) { set_error("mpc_step_x0: null argument"); return CQP_ERR_ARGUMENT; }
  if (!h->mpc_og) { set_error("mpc_step_x0: no template (call cqp_mpc_set_template first)"); return CQP_ERR_ARGUMENT; }
  if (k < 1) { set_error("mpc_step_x0: k must be >= 1"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  if (h->srv_enabled && h->mpc_nx <= kMaxInlineX0) return server_step(h, x0, k, u0, out);
  const auto t0 = std::chrono::steady_clock::now();
  int rc = launch_instantiate(h, x0);
  if (rc) return rc;
  h->vectors_device_only = true;
  h->mpc_extract = true;
  rc = run_and_fetch(h, false, k, true, out, t0, u0);
  h->mpc_extract = false;
  return rc;
}

int cqp_mpc_server_start(cqp_handle* h, int k, double idle_timeout_ms) {
  if (!h) return CQP_ERR_ARGUMENT;
  if (!h->mpc_og) { set_error("mpc_server_start: no template (call cqp_mpc_set_template first)"); return CQP_ERR_ARGUMENT; }
  if (k < 1) { set_error("mpc_server_start: k must be >= 1"); return CQP_ERR_ARGUMENT; }
  if (h->mpc_nx > kMaxInlineX0) { set_error("mpc_server_start: nx exceeds the mailbox (128 states)"); return CQP_ERR_CAPACITY; }
  CQP_CUDA(cudaSetDevice(h->device));
  h->srv_idle_ns = (long long)((idle_timeout_ms > 0.0 ? idle_timeout_ms : 100.0) * 1e6);
  h->srv_enabled = true;
  return server_launch(h, k);
}

int cqp_mpc_server_last_timing(const cqp_handle* h, double* wall_us, double* device_us) {
  if (!h) return CQP_ERR_ARGUMENT;
  if (wall_us) *wall_us = h->srv_last_wall_us;
  if (device_us) *device_us = h->srv_last_device_us;
  return CQP_OK;
}

int cqp_mpc_server_stop(cqp_handle* h) {
  if (!h) return CQP_ERR_ARGUMENT;
  CQP_CUDA(cudaSetDevice(h->device));
  h->srv_enabled = false;
  return server_stop(h);
}

int cqp_get_state(cqp_handle* h, double* v, int* layer_index) {
  if (!h) return CQP_ERR_ARGUMENT;
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  int st[1];
  CQP_CUDA(cudaMemcpyAsync(st, h->state, sizeof(st), cudaMemcpyDeviceToHost, h->stream));
  CQP_CUDA(cudaStreamSynchronize(h->stream));
  if (layer_index) *layer_index = st[0];
  if (v) {
    CQP_CUDA(cudaMemcpyAsync(v, h->vq, sizeof(double) * h->D,
                             cudaMemcpyDeviceToHost, h->stream));
    CQP_CUDA(cudaStreamSynchronize(h->stream));
  }
  return CQP_OK;
}

int cqp_set_state(cqp_handle* h, const double* v, int layer_index) {
  if (!h || !v) { set_error("set_state: null argument"); return CQP_ERR_ARGUMENT; }
  if (layer_index < 0 || layer_index >= h->L) { set_error("set_state: layer index out of range"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  // ring invariant between launches: slot 0 = iterate, slots 1..3 = sentinel
  CQP_CUDA(cudaMemsetAsync(h->vq, 0, sizeof(double) * (size_t)h->Dpad, h->stream));
  CQP_CUDA(cudaMemsetAsync(h->vq + h->ring_ld, 0xFF, sizeof(double) * 3 * (size_t)h->ring_ld, h->stream));
  CQP_CUDA(cudaMemcpyAsync(h->vq, v, sizeof(double) * (size_t)h->D, cudaMemcpyHostToDevice, h->stream));
  int rc = launch_set_state(h, layer_index);
  if (rc) return rc;
  CQP_CUDA(cudaStreamSynchronize(h->stream));  // (v may be pageable)
  return CQP_OK;
}

int cqp_get_layer(cqp_handle* h, int k, double* W, double* Dk, double* GDk, double* b,
                  double* rho_vec) {
  if (!h || k < 0 || k >= h->L) { set_error("get_layer: bad index"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
  const int n = h->n, m = h->m, D = h->D;
  const size_t nm = (size_t)n + m;
  double* scratch = nullptr;
  int rc = dev_alloc(&scratch, (size_t)D * D);
  if (rc) return rc;
  auto done = [&](int code) { cudaStreamSynchronize(h->stream); cudaFree(scratch); return code; };
  if (W) {
    if ((rc = launch_untranspose(h->stream, h->W + (size_t)k * D * h->Dpad, D, D, h->Dpad, scratch))) return done(rc);
    if (cudaMemcpyAsync(W, scratch, sizeof(double) * (size_t)D * D, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
    cudaStreamSynchronize(h->stream);
  }
  const double* dg = h->Dk + (size_t)k * nm * h->npad;
  if (Dk) {
    if ((rc = launch_untranspose(h->stream, dg, n, n, h->npad, scratch))) return done(rc);
    if (cudaMemcpyAsync(Dk, scratch, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
    cudaStreamSynchronize(h->stream);
  }
  if (GDk) {
    if ((rc = launch_untranspose(h->stream, dg + (size_t)n * h->npad, m, n, h->npad, scratch))) return done(rc);
    if (cudaMemcpyAsync(GDk, scratch, sizeof(double) * (size_t)m * n, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
    cudaStreamSynchronize(h->stream);
  }
  if (b) {
    if ((rc = launch_bias(h, k, scratch))) return done(rc);
    if (cudaMemcpyAsync(b, scratch, sizeof(double) * (size_t)D, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
    cudaStreamSynchronize(h->stream);
  }
  if (rho_vec) {
    if (cudaMemcpyAsync(rho_vec, h->rho_vec + (size_t)k * m, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) return done(CQP_ERR_CUDA);
  }
  return done(CQP_OK);
}

int cqp_get_scaling(cqp_handle* h, double* E, double* F, double* cost_scale, double* grid,
                    int* initial_index, double* c_tilde, double* d_tilde) {
  if (!h) return CQP_ERR_ARGUMENT;
  const int n = h->n, m = h->m;
  if (h->vectors_device_only && (c_tilde || d_tilde)) {  // c, d came from the device-side instantiate
    CQP_CUDA(cudaSetDevice(h->device));
  CQP_QUIESCE(h);
    h->c_host.resize(m); h->d_host.resize(m);
    CQP_CUDA(cudaMemcpyAsync(h->c_host.data(), h->c, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream));
    CQP_CUDA(cudaMemcpyAsync(h->d_host.data(), h->d, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream));
    CQP_CUDA(cudaStreamSynchronize(h->stream));
  }
  if (E) std::memcpy(E, h->E_host.data(), sizeof(double) * n);
  if (F) std::memcpy(F, h->F_host.data(), sizeof(double) * m);
  if (cost_scale) *cost_scale = h->cost_scale;
  if (grid) std::memcpy(grid, h->grid.data(), sizeof(double) * h->L);
  if (initial_index) *initial_index = h->initial_index;
  for (int i = 0; i < h->D; ++i) {
    const bool zrow = i >= n && i < n + m;
    if (c_tilde) c_tilde[i] = zrow ? h->F_host[i - n] * h->c_host[i - n] : -INFINITY;
    if (d_tilde) d_tilde[i] = zrow ? h->F_host[i - n] * h->d_host[i - n] : INFINITY;
  }
  return CQP_OK;
}

int cqp_pinned_alloc(void** out, unsigned long long bytes) {
  if (!out) return CQP_ERR_ARGUMENT;
  *out = nullptr;
  CQP_CUDA(cudaMallocHost(out, bytes ? (size_t)bytes : 1));
  return CQP_OK;
}

void cqp_pinned_free(void* p) {
  if (p) cudaFreeHost(p);
}

int cqp_debug_words(const cqp_handle* h, int* out256) {
  if (!h || !out256) return CQP_ERR_ARGUMENT;
  for (int i = 0; i < 256; ++i) out256[i] = ((volatile int*)h->dbg_host)[i];
  return CQP_OK;
}

int cqp_dims(const cqp_handle* h, int* n, int* m, int* L) {
  if (!h) return CQP_ERR_ARGUMENT;
  if (n) *n = h->n;
  if (m) *m = h->m;
  if (L) *L = h->L;
  return CQP_OK;
}

int cqp_launch_info(const cqp_handle* h, int* ctas, int* rows_per_cta, int* tier, int* smem_bytes) {
  if (!h) return CQP_ERR_ARGUMENT;
  if (ctas) *ctas = h->G;
  if (rows_per_cta) *rows_per_cta = h->R;
  if (tier) *tier = h->cluster ? 2 : (h->w_smem ? 0 : 1);
  if (smem_bytes) *smem_bytes = h->smem_bytes;
  return CQP_OK;
}

int cqp_measure_read_bandwidth(int device, unsigned long long bytes, int passes, double* gb_per_s) {
  if (!gb_per_s || bytes < 4096 || passes < 1) { set_error("measure_read_bandwidth: bad argument"); return CQP_ERR_ARGUMENT; }
  CQP_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CQP_CUDA(cudaGetDeviceProperties(&prop, device));
  double2* buf = nullptr;
  double* sink = nullptr;
  const size_t n2 = (size_t)bytes / sizeof(double2);
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&buf), n2 * sizeof(double2)));
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&sink), sizeof(double)));
  CQP_CUDA(cudaMemset(buf, 0, n2 * sizeof(double2)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = prop.multiProcessorCount * 4;
  read_bw_kernel<<<grid, 512>>>(buf, n2, 2, sink);  // warm-up (also brings an L2-sized buffer into L2)
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    read_bw_kernel<<<grid, 512>>>(buf, n2, passes, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(buf); cudaFree(sink);
  if (err != cudaSuccess) return cuda_fail(err, "read_bw_kernel");
  *gb_per_s = (double)n2 * sizeof(double2) * passes / (best * 1e-3) / 1e9;
  return CQP_OK;
}

int cqp_layer_traffic(const cqp_handle* h, double* w_bytes_per_iteration, int* structured) {
  if (!h) return CQP_ERR_ARGUMENT;
  const double D = h->D, n = h->n, m = h->m;
  if (w_bytes_per_iteration) *w_bytes_per_iteration = h->structured ? 8.0 * ((n + m) * D + m * n) : 8.0 * D * D;
  if (structured) *structured = h->structured;
  return CQP_OK;
}

}  // extern "C"
