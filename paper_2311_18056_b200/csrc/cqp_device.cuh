// Device-side helpers shared by the persistent single-QP kernels (cqp_single.cu: all-SM grid with
// an L2 ring exchange; cqp_cluster.cu: one thread-block cluster with a DSMEM exchange).
#pragma once

#include <cfloat>
#include <cmath>

#include "cqp_internal.h"

namespace cqp {
namespace {

constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ double nanmax(double best, double a) {
  // max that keeps NaN once seen (the oracle's inf_norm propagates NaN the same way)
  return (a > best || a != a) ? a : best;
}

// Watchdog: a spin that lasts longer than ~2 s records where it was stuck in host-mapped memory
// and traps, so a protocol bug or a lost CTA becomes a CUDA error instead of a hung GPU.
constexpr long long kSpinLimitCycles = 4000000000ll;

__device__ __noinline__ void watchdog_fire(int* d, int where, int iter) {
  if (d && atomicCAS(d, 0, 1) == 0) {
    d[1] = where;
    d[2] = iter;
    d[3] = (int)blockIdx.x;
    d[4] = (int)threadIdx.x;
    __threadfence_system();
  }
#ifdef CQP_DEBUG_PROGRESS
  // debug builds: the first 47 threads that time out leave a record each, and the trap waits a while
  // so that the others get there (tools/deadlock_probe.py)
  if (d) {
    const int idx = atomicAdd(d + 5, 1);
    if (idx < 47) {
      volatile int* r = d + 64 + 4 * idx;
      r[0] = where; r[1] = iter; r[2] = (int)blockIdx.x; r[3] = (int)threadIdx.x;
      __threadfence_system();
    }
    const long long t0 = clock64();
    while (clock64() - t0 < 40000000ll) {}
  }
#endif
  __trap();
}

__device__ __forceinline__ void progress(int* d, int role, int value) {
#ifdef CQP_DEBUG_PROGRESS
  if (d && blockIdx.x < 12) {
    *((volatile int*)(d + 16 + blockIdx.x * 4 + role)) = value;
  }
#endif
}

// Optional timeline trace (-DCQP_TRACE): clock64() stamps of CTA 0's roles for iterations
// 100..103, 16 slots per iteration, into the host-mapped debug record (as long long, from word 64).
#if defined(CQP_TRACE_TWO)
// Two-CTA variant (tools/trace_tier1.py two): CTA 0 and the LAST CTA (a lambda-row CTA of the
// structured partition) stamp iterations AT, AT+1 with %globaltimer (ns, common to all SMs).
#ifndef CQP_TRACE_AT
#define CQP_TRACE_AT 100
#endif
__device__ __forceinline__ long long cqp_globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CQP_STAMP(dbg, it, slot)                                                                          \
  do {                                                                                                    \
    if ((blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (it) >= CQP_TRACE_AT && (it) < CQP_TRACE_AT + 2) \
      reinterpret_cast<volatile long long*>((dbg) + 64)[(blockIdx.x == 0 ? 0 : 32) + ((it)-CQP_TRACE_AT) * 16 + (slot)] = \
          cqp_globaltimer();                                                                              \
  } while (0)
#define CQP_STAMP0(dbg, slot) do {} while (0)
#define CQP_STAMPR(dbg, pass, slot) do {} while (0)
#elif defined(CQP_TRACE)
#ifndef CQP_TRACE_AT
#define CQP_TRACE_AT 100
#endif
#define CQP_STAMP(dbg, it, slot)                                                        \
  do {                                                                                  \
    if (blockIdx.x == 0 && (it) >= CQP_TRACE_AT && (it) < CQP_TRACE_AT + 4)                                   \
      reinterpret_cast<volatile long long*>((dbg) + 64)[((it)-CQP_TRACE_AT) * 16 + (slot)] = clock64(); \
  } while (0)
// prologue / epilogue stamps of CTA 0 (fixed slots 48..63 of the same record)
#define CQP_STAMP0(dbg, slot)                                                                   \
  do {                                                                                          \
    if (blockIdx.x == 0 && threadIdx.x == 0)                                                    \
      reinterpret_cast<volatile long long*>((dbg) + 64)[48 + (slot)] = clock64();               \
  } while (0)
// residual pass number 2 of the launch (the third check), thread 0 of CTA 0: slots 64.. of the same array
#define CQP_STAMPR(dbg, pass, slot)                                                                    \
  do {                                                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (pass) == 2)                                            \
      reinterpret_cast<volatile long long*>((dbg) + 64)[64 + (slot)] = clock64();                      \
  } while (0)
#else
#define CQP_STAMP(dbg, it, slot) do {} while (0)
#define CQP_STAMP0(dbg, slot) do {} while (0)
#define CQP_STAMPR(dbg, pass, slot) do {} while (0)
#endif

__device__ __forceinline__ bool is_sentinel(double x) {
  return (unsigned long long)__double_as_longlong(x) == kSentinel;
}

__device__ __forceinline__ void publish(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void publish_release(double* p, double v) {
  asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int parity, int* dbg, int where, int iter) {
  unsigned ok;
  long long t0 = 0;
  unsigned spins = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && (++spins & 0xFF) == 0) {
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, where, iter);
    }
  } while (!ok);
}

// ---- thread-block-cluster helpers (small problems: the whole W ladder slice set fits the shared
// memory of one cluster, and the iterate is exchanged through distributed shared memory) ----
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned map_to_cta(unsigned local_smem_addr, unsigned cta_rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(cta_rank));
  return r;
}
__device__ __forceinline__ void st_remote(unsigned cluster_addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(cluster_addr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, int parity, int* dbg, int where, int iter) {
  unsigned ok;
  long long t0 = 0;
  unsigned spins = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!ok && (++spins & 0xFF) == 0) {
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, where, iter);
    }
  } while (!ok);
}

__device__ __forceinline__ double2 load_pair(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p)
               : "memory");
  return v;
}

// layers.cpp:38-50 with log10(grid) tabulated on the host.
__device__ __forceinline__ int nearest_grid_index(const double* log_grid, int L, double rho) {
  const double target = log10(rho);
  int best = 0;
  double best_dist = INFINITY;
  for (int k = 0; k < L; ++k) {
    const double dist = fabs(log_grid[k] - target);
    if (dist < best_dist - 1e-15) {
      best = k;
      best_dist = dist;
    }
  }
  return best;
}


// The same index without log10 where that is safe.  `bound[k] = sqrt(grid[k] grid[k+1])` is the value whose
// log10 lies midway between two neighbours of an ascending grid (host-computed; bound == nullptr: no fast
// path), so the nearest index is the number of bounds below rho.  Within 1e-9 (relative) of a bound, and
// for rho that is not a positive finite number, the comparison in log space above decides, exactly as
// before: the fast path only skips the FP64 log10 (about 1 us for the single deciding thread).
__device__ __forceinline__ int nearest_grid_index_fast(const double* log_grid, const double* bound, int L, double rho) {
  if (bound == nullptr || !(rho > 0.0) || !(rho < 1.0e300)) return nearest_grid_index(log_grid, L, rho);
  int k = 0;
  for (int j = 0; j + 1 < L; ++j) k += (rho > bound[j]) ? 1 : 0;
  const double lo = k > 0 ? bound[k - 1] : 0.0;
  const double hi = k + 1 < L ? bound[k] : 1.0e308;
  if (rho - lo <= 1e-9 * lo || hi - rho <= 1e-9 * hi) return nearest_grid_index(log_grid, L, rho);
  return k;
}

// One warp: M[row, :] . x with M row-major in global memory and x in shared memory (pad entries of
// both zero), U 16-byte loads per lane in flight: an n = 870 row (14 column pairs per lane) costs
// two L2 round trips instead of one per pair.  Fixed order: lane l takes pairs l, l + 32, ...
template <int U>
__device__ __forceinline__ double warp_row_dot_mlp(const double* __restrict__ Mrow, const double* __restrict__ x,
                                                   int ncols_pad, int lane) {
  const double2* m2 = reinterpret_cast<const double2*>(Mrow);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int nc2 = ncols_pad >> 1;
  double a0 = 0.0, a1 = 0.0;
  for (int base = lane; base < nc2; base += 32 * U) {
    double2 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c2 = base + 32 * u;
      w[u] = c2 < nc2 ? __ldg(m2 + c2) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c2 = base + 32 * u;
      if (c2 < nc2) {
        const double2 xv = x2[c2];
        if (u & 1) {
          a1 = fma(w[u].x, xv.x, a1);
          a1 = fma(w[u].y, xv.y, a1);
        } else {
          a0 = fma(w[u].x, xv.x, a0);
          a0 = fma(w[u].y, xv.y, a0);
        }
      }
    }
  }
  double v = a0 + a1;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
  return v;
}

__device__ __forceinline__ void mbar_inval(unsigned long long* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One row of mpc::instantiate (mpc.cpp:260-270) by one warp: row < n: g[row] = offset_g[row, :] . x0;
// else c / d [row - n] = base - offset_c[row - n, :] . x0.  The standalone kernel and the resident
// server share this, so both produce the same bits.
__device__ __forceinline__ void instantiate_row(int row, int lane, const double* __restrict__ og,
                                                const double* __restrict__ oc, const double* __restrict__ cb,
                                                const double* __restrict__ db, const double* x0, int n, int nx,
                                                int nxpad, double* g, double* c, double* d, bool x0_in_global = true) {
  const double* M = row < n ? og + (size_t)row * nxpad : oc + (size_t)(row - n) * nxpad;
  double acc = 0.0;
  for (int j = lane; j < nx; j += 32) acc = fma(M[j], x0_in_global ? __ldcg(x0 + j) : x0[j], acc);  // (x0 changes per server step: not through L1)
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
  if (lane == 0) {
    if (row < n) {
      g[row] = acc;
    } else {
      c[row - n] = cb[row - n] - acc;
      d[row - n] = db[row - n] - acc;
    }
  }
}

// Resident MPC server, request side.  Warp 0 of the FIRST CTA polls the host-mapped mailbox; on a new
// request it fetches x0 with all lanes at once (one PCIe round trip), stores it to the device copy and
// republishes the request number in device memory for the other CTAs (release).  Returns the request
// number, or kSrvExit when told to stop / idle for too long.  Call with the whole warp.
// `stage` (shared memory, optional): x0 is also left at stage[2 ...] for a caller that forwards the request
// itself (the cluster kernel pushes it through distributed shared memory); the device-memory relay and
// its fence are then skipped.
__device__ __forceinline__ unsigned long long server_fetch_request(const RunParams& p, unsigned long long served, int lane,
                                                                   int& want_full, double* stage = nullptr) {
  unsigned long long seq = served;
  if (lane == 0) {
    const long long t0 = globaltimer_ns();
    unsigned spins = 0;
    for (;;) {
      seq = p.mb[kMbReq];
      if (seq != served) break;
      if (p.mb[kMbStop] != 0ull) { seq = kSrvExit; break; }
      if ((++spins & 0x3F) == 0 && globaltimer_ns() - t0 > p.idle_ns) { seq = kSrvExit; break; }
    }
  }
  seq = __shfl_sync(0xffffffffu, seq, 0);
  if (seq != kSrvExit) {
    const volatile double* src = reinterpret_cast<const volatile double*>(p.mb + kMbX0);
    double v[kMaxInlineX0 / 32];
    const unsigned long long wf = (lane == 0) ? p.mb[kMbWantFull] : 0ull;  // (in flight together with x0)
#pragma unroll
    for (int u = 0; u < kMaxInlineX0 / 32; ++u) v[u] = (lane + 32 * u < p.mpc_nx) ? src[lane + 32 * u] : 0.0;
    want_full = (int)__shfl_sync(0xffffffffu, wf, 0);
#pragma unroll
    for (int u = 0; u < kMaxInlineX0 / 32; ++u)
      if (lane + 32 * u < p.mpc_nx) {
        p.mpc_x0_w[lane + 32 * u] = v[u];
        if (stage) stage[2 + lane + 32 * u] = v[u];
      }
    if (!stage) __threadfence();
    __syncwarp();
  }
  // (the relay word carries "full report wanted" in bit 62: every CTA must take the same path)
  if (lane == 0 && !stage) st_release_gpu_u64(p.srv_seq, seq == kSrvExit ? seq : (seq | ((unsigned long long)(want_full != 0) << 62)));
  return seq;
}

// The other CTAs: wait until the first CTA has republished a request newer than `served`.
__device__ __forceinline__ unsigned long long server_wait_relay(const RunParams& p, unsigned long long served, int& want_full) {
  unsigned long long w;
  do { w = ld_acquire_gpu_u64(p.srv_seq); } while (w != kSrvExit && (w & ~(1ull << 62)) == served);
  if (w == kSrvExit) return w;
  want_full = (int)((w >> 62) & 1ull);
  return w & ~(1ull << 62);
}

// Control extraction of the closed loop (bench.cpp:169-175): u0 = clamp(-K x + y[0:nu], u_lo, u_hi).
// `y` is the unscaled primal solution in shared memory; executed by one CTA (thread `t0` takes
// controls t0, t0 + blockDim.x, ...).
__device__ __forceinline__ void mpc_extract_control(const RunParams& p, const double* y, int t0, const double* x0_smem = nullptr) {
  if (!p.mpc_K) return;
  for (int t = t0; t < p.mpc_nu; t += (int)blockDim.x) {
    const double* Krow = p.mpc_K + (size_t)t * p.mpc_nxpad;
    double kx = 0.0;
    for (int j = 0; j < p.mpc_nx; ++j) kx = fma(Krow[j], x0_smem ? x0_smem[j] : __ldcg(p.mpc_x0 + j), kx);
    double u = -kx + y[t];
    const double lo = p.mpc_ulo[t], hi = p.mpc_uhi[t];
    u = u < lo ? lo : u;
    u = u > hi ? hi : u;
    p.out_u[t] = u;
  }
}

}  // namespace
}  // namespace cqp
