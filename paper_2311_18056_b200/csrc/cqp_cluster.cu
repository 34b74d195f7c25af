// Single-QP solve path for SMALL problems: one thread-block cluster, iterate exchanged through
// distributed shared memory.  Same contract as run_kernel in cqp_single.cu (it replaces the
// reference's run_loop, /root/reference/proj/src/solver.cpp:43-105, with its helpers :109-142,
// layers.cpp:38-50,168-187 and refresh_z solver.cpp:197-200); chosen by configure_launch when one
// ladder level W_k (8 D^2 bytes) fits the shared memory of a single cluster (D <~ 650 with 16 CTAs).
//
// Why a second kernel: for D <= ~650 the all-SM grid spends > 90 % of an iteration on the
// L2-mediated all-to-all of v (publish -> L2 -> poll, ~2.3 us).  Inside a cluster the exchange is
// a DSMEM store (~215 cycles) that carries its own completion signal:
//   * CTA r of the C-CTA cluster keeps rows [r R, r R + R) of W_k resident in shared memory and a
//     full double-buffered copy of the iterate (xs[2][Dpad]).
//   * All 16 warps are compute warps and own WHOLE rows, so there is no cross-warp reduction, no
//     publisher warp and no CTA-wide barrier in the iteration loop.  Two layouts:
//       - register mode (R <= 32, D <= 512): 16 lanes per row, 2 rows per warp; every lane keeps
//         its NPT column pairs of W_k in REGISTERS for the whole solve (a rho switch reloads
//         them), so an iteration reads only x from shared memory (both half-warps read the same
//         16 addresses: one 256-byte broadcast wavefront per LDS) and needs a 4-step butterfly;
//       - shared-memory mode (larger R): W slice resident in shared memory, warp w owns local rows
//         [w RPW, w RPW + RPW), lanes stride over column pairs (16-byte LDS, conflict-free), two
//         FMA chains per row, a 5-step butterfly.
//   * The warp that finished a row adds the bias, clamps and pushes the value into every CTA's
//     copy with st.async.shared::cluster ... mbarrier::complete_tx::bytes (lane -> peer lane % C).
//     Each CTA's xready[parity] mbarrier expects exactly 8 D bytes per iteration, so "v_i is
//     complete here" is one mbarrier phase: no flags, no polling of memory, no fences.
//   * Residual checks (every check_interval iterations) split the rows of H, G', G over the CTAs
//     (warp per row), exchange the seven max-norms with the same st.async + mbarrier pattern and
//     every CTA takes the identical rho decision.
// Summation order differs from the grid kernel (and from Eigen), which the parity contract allows:
// identical iteration counts / rho traces, solutions within 1e-6 relative (tests/test_gpu_single.py).
#include <cstdlib>

#include "cqp_device.cuh"
#include "cqp_internal.h"

namespace cqp {
namespace {

constexpr int kClThreads = 512;
constexpr int kClWarps = kClThreads / 32;
constexpr int kClMaxRpw = 4;  // rows of W per warp (R <= 64 rows per CTA)

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// st.async: remote 8-byte store whose completion is counted (in bytes) on the destination CTA's
// mbarrier.  Both addresses are shared::cluster addresses of the SAME destination CTA.
__device__ __forceinline__ void st_async_f64(unsigned dst_cluster_addr, double v, unsigned mbar_cluster_addr) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(dst_cluster_addr),
               "l"(__double_as_longlong(v)), "r"(mbar_cluster_addr)
               : "memory");
}

// (Re-)arm a single-arrival mbarrier for its next phase: that phase completes once `bytes` of
// st.async traffic have landed.  A complete_tx that overtakes the arm only drives the tx-count
// negative for a moment; the phase cannot complete before this (its only) arrival.
__device__ __forceinline__ void mbar_arm(unsigned long long* bar, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
  return v;
}

// One warp: M[row, :] . x with M row-major in global memory (read through L1/L2), x in shared
// memory, pad entries of both zero.  Fixed order: lane l takes column pairs l, l + 32, ...
template <bool LDG = true>
__device__ __forceinline__ double warp_row_dot(const double* __restrict__ Mrow, const double* __restrict__ x,
                                               int ncols_pad, int lane) {
  const double2* m2 = reinterpret_cast<const double2*>(Mrow);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int nc2 = ncols_pad >> 1;
  double a0 = 0.0, a1 = 0.0;
  int c2 = lane;
  for (; c2 + 32 < nc2; c2 += 64) {
    const double2 w0 = LDG ? __ldg(m2 + c2) : m2[c2], w1 = LDG ? __ldg(m2 + c2 + 32) : m2[c2 + 32];
    const double2 x0 = x2[c2], x1 = x2[c2 + 32];
    a0 = fma(w0.x, x0.x, a0);
    a0 = fma(w0.y, x0.y, a0);
    a1 = fma(w1.x, x1.x, a1);
    a1 = fma(w1.y, x1.y, a1);
  }
  if (c2 < nc2) {
    const double2 w0 = LDG ? __ldg(m2 + c2) : m2[c2];
    const double2 x0 = x2[c2];
    a0 = fma(w0.x, x0.x, a0);
    a0 = fma(w0.y, x0.y, a0);
  }
  return warp_sum(a0 + a1);
}

// Three row dots of one residual step at once: H[rh, :] . y, G'[rh, :] . lambda, G[rg, :] . y (a
// null row pointer yields 0).  Each sum has the same fixed order as warp_row_dot; all global loads
// of a trip are issued before the first FMA and the three butterflies interleave.  The rows may
// live in shared memory (hg_smem) or in global memory: generic loads.
__device__ __forceinline__ void warp_row_dot3(const double* __restrict__ Hrow, const double* __restrict__ Gtrow,
                                              const double* __restrict__ Grow, const double* __restrict__ y,
                                              const double* __restrict__ lam, int npad, int mpad, int lane,
                                              double& hy, double& gtl, double& gy) {
  const double2* h2 = reinterpret_cast<const double2*>(Hrow);
  const double2* t2 = reinterpret_cast<const double2*>(Gtrow);
  const double2* g2 = reinterpret_cast<const double2*>(Grow);
  const double2* y2 = reinterpret_cast<const double2*>(y);
  const double2* l2 = reinterpret_cast<const double2*>(lam);
  const int nn2 = npad >> 1, nm2 = mpad >> 1, top = max(nn2, nm2);
  const double2 zero = make_double2(0.0, 0.0);
  double a[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  for (int c2 = lane; c2 < top; c2 += 64) {
    const int d2 = c2 + 32;
    const bool n0 = c2 < nn2, n1 = d2 < nn2, m0 = c2 < nm2, m1 = d2 < nm2;
    const double2 wh0 = (Hrow && n0) ? h2[c2] : zero, wh1 = (Hrow && n1) ? h2[d2] : zero;
    const double2 wt0 = (Gtrow && m0) ? t2[c2] : zero, wt1 = (Gtrow && m1) ? t2[d2] : zero;
    const double2 wg0 = (Grow && n0) ? g2[c2] : zero, wg1 = (Grow && n1) ? g2[d2] : zero;
    const double2 y0 = n0 ? y2[c2] : zero, y1 = n1 ? y2[d2] : zero;
    const double2 l0 = m0 ? l2[c2] : zero, l1 = m1 ? l2[d2] : zero;
    a[0][0] = fma(wh0.x, y0.x, a[0][0]); a[0][0] = fma(wh0.y, y0.y, a[0][0]);
    a[0][1] = fma(wh1.x, y1.x, a[0][1]); a[0][1] = fma(wh1.y, y1.y, a[0][1]);
    a[1][0] = fma(wt0.x, l0.x, a[1][0]); a[1][0] = fma(wt0.y, l0.y, a[1][0]);
    a[1][1] = fma(wt1.x, l1.x, a[1][1]); a[1][1] = fma(wt1.y, l1.y, a[1][1]);
    a[2][0] = fma(wg0.x, y0.x, a[2][0]); a[2][0] = fma(wg0.y, y0.y, a[2][0]);
    a[2][1] = fma(wg1.x, y1.x, a[2][1]); a[2][1] = fma(wg1.y, y1.y, a[2][1]);
  }
  double v0 = a[0][0] + a[0][1], v1 = a[1][0] + a[1][1], v2 = a[2][0] + a[2][1];
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, w);
    v1 += __shfl_xor_sync(0xffffffffu, v1, w);
    v2 += __shfl_xor_sync(0xffffffffu, v2, w);
  }
  hy = v0; gtl = v1; gy = v2;
}

struct ClSmem {
  double* sW;     // R * Dpad  this CTA's rows of W_k (shared-memory mode only)
  double* xs;     // 2 * xs_stride  full iterate, double buffered by iteration parity (peers write here)
  double* sH;     // pern * npad   this CTA's rows of H   (hg_smem only; else read from global)
  double* sGt;    // pern * mpad   ... of G'
  double* sG;     // perm * npad   ... of G
  double* uy;     // npad      unscaled y (also scratch for g_s)
  double* uz;     // mpad
  double* ul;     // mpad
  double* sE;     // npad      scaling.E   (constant for the launch)
  double* sF;     // mpad      scaling.F
  double* sg;     // npad      unscaled g
  double* sb;     // Rp  bias rows
  double* slo;    // Rp
  double* shi;    // Rp
  double* sgrid;  // 3 * 16   grid values, log10(grid), bounds between neighbours (L <= 16; else read from global)
  double* wmax;   // kClWarps * 8   per-warp partial maxima
  double* cmax;   // 8              this CTA's maxima / the cluster-wide result
  double* norms;  // 2 * 16 * 8     per-CTA maxima of a residual pass, by pass parity (peers write here)
  unsigned long long* bars;  // xready[2], nbar[2], (server: request word, report flag), cbar, gbar
  double* sx0;    // 2 + kMaxInlineX0   resident server: {request number, report flag, x0} pushed by CTA 0
};

// Shared-memory doubles: `wrows` rows of W (0 in register mode), the iterate copies, and the
// (optional) rows of H, G', G a CTA needs for the residual checks.
__host__ __device__ inline size_t cl_smem_doubles(int R, int wrows, int Dpad, int xs_stride, int npad, int mpad,
                                                  int hg_rows_n, int hg_rows_m) {
  const int Rp = (R + 1) & ~1;
  return (size_t)wrows * Dpad + 2 * (size_t)xs_stride + 3 * (size_t)npad + 3 * (size_t)mpad + 3 * (size_t)Rp +
         (size_t)hg_rows_n * (npad + mpad) + (size_t)hg_rows_m * npad + 48 + kClWarps * 8 + 8 + 2 * 16 * 8 + 8 +
         2 + kMaxInlineX0;
}

__device__ __forceinline__ ClSmem cl_carve(unsigned char* raw, const RunParams& p) {
  ClSmem s;
  double* base = reinterpret_cast<double*>(raw);
  const int Rp = (p.R + 1) & ~1;
  const int pern = p.hg_smem ? (p.n + p.G - 1) / p.G : 0, perm = p.hg_smem ? (p.m + p.G - 1) / p.G : 0;
  s.sW = base;
  s.xs = s.sW + (p.w_smem ? (size_t)p.R * p.Dpad : 0);
  s.sH = s.xs + 2 * p.xs_stride;
  s.sGt = s.sH + (size_t)pern * p.npad;
  s.sG = s.sGt + (size_t)pern * p.mpad;
  s.uy = s.sG + (size_t)perm * p.npad;
  s.uz = s.uy + p.npad;
  s.ul = s.uz + p.mpad;
  s.sE = s.ul + p.mpad;
  s.sF = s.sE + p.npad;
  s.sg = s.sF + p.mpad;
  s.sb = s.sg + p.npad;
  s.slo = s.sb + Rp;
  s.shi = s.slo + Rp;
  s.sgrid = s.shi + Rp;
  s.wmax = s.sgrid + 48;
  s.cmax = s.wmax + kClWarps * 8;
  s.norms = s.cmax + 8;
  s.bars = reinterpret_cast<unsigned long long*>(s.norms + 2 * 16 * 8);
  s.sx0 = reinterpret_cast<double*>(s.bars + 8);
  return s;
}

// Makes layer k current: W slice -> shared memory, bias rows b = -[D_k; G D_k] g_s for the rows
// this CTA owns, 0 on the lambda rows (layers.cpp:168-175).  s.uy is scratch for
// g_s = cost_scale * E o g (layers.cpp:181).
// `dg_cache` (resident server): this CTA's rows of [D_k; G D_k] for level k, in shared memory.
__device__ void cl_load_layer(const RunParams& p, const ClSmem& s, int k, int row0, int nrows, bool copy_w = true,
                              const double* dg_cache = nullptr) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __syncthreads();
  if (p.w_smem && copy_w) {
    const double2* src = reinterpret_cast<const double2*>(p.W + ((size_t)k * p.D + row0) * p.Dpad);
    double2* dst = reinterpret_cast<double2*>(s.sW);
    const int count = nrows * (p.Dpad >> 1);
    int i = t;
    for (; i + 3 * kClThreads < count; i += 4 * kClThreads) {
      const double2 a = __ldg(src + i), b = __ldg(src + i + kClThreads), c = __ldg(src + i + 2 * kClThreads),
                    d = __ldg(src + i + 3 * kClThreads);
      dst[i] = a;
      dst[i + kClThreads] = b;
      dst[i + 2 * kClThreads] = c;
      dst[i + 3 * kClThreads] = d;
    }
    for (; i < count; i += kClThreads) dst[i] = __ldg(src + i);
  }
  for (int i = t; i < p.npad; i += kClThreads) s.uy[i] = (i < p.n) ? p.cost_scale * (s.sE[i] * s.sg[i]) : 0.0;
  __syncthreads();
  const int nm = p.n + p.m;
  const double* DG = p.Dk + (size_t)k * nm * p.npad;  // [D_k; G D_k], (n+m) x npad
  for (int r = warp; r < nrows; r += kClWarps) {
    const int row = row0 + r;
    double bias = 0.0;
    if (row < nm) bias = dg_cache ? -warp_row_dot<false>(dg_cache + (size_t)r * p.npad, s.uy, p.npad, lane)
                                  : -warp_row_dot(DG + (size_t)row * p.npad, s.uy, p.npad, lane);
    if (lane == 0) s.sb[r] = bias;
  }
  __syncthreads();
}

// Residual pass on the unscaled problem (solver.cpp:67-70,119-134; epilogue :90-95 when `final`).
// `xs` is this CTA's copy of the iterate.  On return every thread of every CTA holds the same
// seven norms: 0 ||Gy - z||  1 ||Hy + g + G'lam||  2 ||Hy||  3 ||G'lam||  4 ||Gy||  5 ||z||  6 ||g||
__device__ void cl_residual_pass(const RunParams& p, const ClSmem& s, const double* xs, bool final, int pass,
                                 unsigned rank, int C, double (&out)[7]) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = p.n, m = p.m;
  unsigned long long* nbar = s.bars + 2;
  asm volatile("cp.async.wait_all;" ::: "memory");  // the cached rows of H, G', G (first pass only: a no-op later)
  __syncthreads();
  // unscale (layers.hpp:57-59)
  for (int i = t; i < p.npad; i += kClThreads) s.uy[i] = (i < n) ? s.sE[i] * xs[i] : 0.0;
  for (int i = t; i < p.mpad; i += kClThreads) {
    double z = 0.0, l = 0.0;
    if (i < m) {
      z = xs[n + i] / s.sF[i];
      if (final) {  // solver.cpp:94  z = clamp(z, p.c, p.d) in original units
        const double lo = __ldcg(p.c + i), hi = __ldcg(p.d + i);  // (rewritten by every server step: not through L1)
        z = z < lo ? lo : z;
        z = z > hi ? hi : z;
      }
      l = (s.sF[i] * xs[n + m + i]) / p.cost_scale;
    }
    s.uz[i] = z;
    s.ul[i] = l;
  }
  __syncthreads();

  double mx[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  {
    // CTA `rank` owns rows [h0, h1) of H and G' and rows [g0, g1) of G; warp w takes the j-th row
    // of both ranges together (j = w, w + 16, ...) so that the three row reads are in flight at
    // once and the three butterflies interleave.
    const int pern = (n + C - 1) / C, perm = (m + C - 1) / C;
    const int h0 = (int)rank * pern, h1 = min(n, h0 + pern);
    const int g0 = (int)rank * perm, g1 = min(m, g0 + perm);
    const int trips = max(pern, perm);
    for (int j = warp; j < trips; j += kClWarps) {
      const int rh = h0 + j, rg = g0 + j;
      const bool vh = rh < h1, vg = rg < g1;
      if (!vh && !vg) break;
      double hy, gtl, gy;
      const double* Hrow = p.hg_smem ? s.sH + (size_t)j * p.npad : p.H + (size_t)rh * p.npad;
      const double* Trow = p.hg_smem ? s.sGt + (size_t)j * p.mpad : p.Gt + (size_t)rh * p.mpad;
      const double* Grow = p.hg_smem ? s.sG + (size_t)j * p.npad : p.Gr + (size_t)rg * p.npad;
      warp_row_dot3(vh ? Hrow : nullptr, vh ? Trow : nullptr, vg ? Grow : nullptr, s.uy, s.ul, p.npad, p.mpad,
                    lane, hy, gtl, gy);
      if (vh) {
        const double gi = s.sg[rh];
        const double dual = (hy + gi) + gtl;  // (H y + g) + G' lambda
        mx[6] = nanmax(mx[6], fabs(gi));
        mx[1] = nanmax(mx[1], fabs(dual));
        mx[2] = nanmax(mx[2], fabs(hy));
        mx[3] = nanmax(mx[3], fabs(gtl));
      }
      if (vg) {
        const double z = s.uz[rg];
        mx[0] = nanmax(mx[0], fabs(gy - z));
        mx[4] = nanmax(mx[4], fabs(gy));
        mx[5] = nanmax(mx[5], fabs(z));
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 7; ++k) s.wmax[warp * 8 + k] = mx[k];
  }
  __syncthreads();
  const int pp = pass & 1;
  if (t < 7 * C) {
    // thread (peer, k): CTA maximum of norm k -> peer's norms[pp][rank][k]
    const int peer = t / 7, k = t - 7 * peer;
    double best = 0.0;
    for (int w = 0; w < kClWarps; ++w) best = nanmax(best, s.wmax[w * 8 + k]);
    st_async_f64(map_to_cta(smem_u32(s.norms + (pp * 16 + (int)rank) * 8 + k), (unsigned)peer), best,
                 map_to_cta(smem_u32(&nbar[pp]), (unsigned)peer));
  }
  mbar_wait_cluster(&nbar[pp], (pass >> 1) & 1, p.dbg, 6, pass);
  if (t < 7) {
    double best = 0.0;
    for (int c = 0; c < C; ++c) best = nanmax(best, s.norms[(pp * 16 + c) * 8 + t]);
    s.cmax[t] = best;
  }
  __syncthreads();  // also: every thread is past the wait, so the barrier may be re-armed
  if (t == 0) mbar_arm(&nbar[pp], 7u * 8u * (unsigned)C);
#pragma unroll
  for (int k = 0; k < 7; ++k) out[k] = s.cmax[k];
  __syncthreads();
}

// NPT == 0: shared-memory mode with RPW rows per warp; NPT > 0: register mode (RPW unused), each
// lane keeps NPT column pairs of its row in registers.
template <int RPW, int NPT>
__global__ void __launch_bounds__(kClThreads, 1) cluster_kernel(const RunParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool kReg = NPT > 0;
  const ClSmem s = cl_carve(smem_raw, p);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int C = p.G;  // cluster size == grid size
  const unsigned rank = cluster_rank();
  unsigned long long* xready = s.bars;  // [2]: v_i is complete in xs[i & 1]
  unsigned long long* nbar = s.bars + 2;  // [2]: the norms of residual pass `pass` are complete
  const int n = p.n, m = p.m, D = p.D;
  const unsigned xbytes = 8u * (unsigned)D;
  CQP_STAMP0(p.dbg, 0);
  // balanced row split: every CTA owns >= 1 row (D >= C), at most p.R = ceil(D / C)
  const int row0 = (int)(((long long)rank * D) / C);
  const int nrows = (int)(((long long)(rank + 1) * D) / C) - row0;
  int layer = p.state[0];

  for (int i = t; i < p.npad; i += kClThreads) s.sE[i] = (i < n) ? p.E[i] : 1.0;
  for (int i = t; i < p.mpad; i += kClThreads) s.sF[i] = (i < m) ? p.F[i] : 1.0;
  for (int i = n + t; i < p.npad; i += kClThreads) s.sg[i] = 0.0;  // (pad entries; the resident server never rewrites them)
  const bool grid_smem = p.L <= 16;
  if (grid_smem && t < p.L) {
    s.sgrid[t] = p.grid[t];
    s.sgrid[16 + t] = p.log_grid[t];
    s.sgrid[32 + t] = p.grid_bound ? p.grid_bound[t] : 0.0;
  }
  const double* grid_v = grid_smem ? s.sgrid : p.grid;
  const double* grid_log = grid_smem ? s.sgrid + 16 : p.log_grid;
  const double* grid_bnd = p.grid_bound ? (grid_smem ? s.sgrid + 32 : p.grid_bound) : nullptr;
  if (p.hg_smem) {  // the rows of H, G', G this CTA needs at every residual check
    const int pern = (n + C - 1) / C, perm = (m + C - 1) / C;
    const int h0 = (int)rank * pern, g0 = (int)rank * perm;
    const int cn = max(0, min(pern, n - h0)), cm = max(0, min(perm, m - g0));
    // asynchronous (cp.async, 16 B): the rows are first needed at the first residual pass, which
    // waits for them; the prologue does not
    auto copy_async = [&](double* dst, const double* src, int doubles) {
      for (int i = 2 * t; i < doubles; i += 2 * kClThreads)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + i)), "l"(src + i) : "memory");
    };
    copy_async(s.sH, p.H + (size_t)h0 * p.npad, cn * p.npad);
    copy_async(s.sGt, p.Gt + (size_t)h0 * p.mpad, cn * p.mpad);
    copy_async(s.sG, p.Gr + (size_t)g0 * p.npad, cm * p.npad);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  // ---- work split inside the CTA ----
  const int nc2 = p.Dpad >> 1;
  const int XS = p.xs_stride;
  // register mode: lanes [0,16) of warp w own local row 2w, lanes [16,32) row 2w + 1; lane `sub` of a
  // row covers column pairs sub, sub + 16, ...  and pushes the finished row to peer `sub`.
  // shared-memory mode: warp w owns local rows [w RPW, w RPW + RPW); lane (peer = lane % C,
  // lane / C) pushes rows lane / C, lane / C + 32 / C, ... of the warp to `peer`.
  const int sub = kReg ? (lane & 15) : lane / C;
  const int peer = kReg ? (lane & 15) : (lane & (C - 1));
  const int wr0 = kReg ? 2 * warp : warp * RPW;                               // first local row of this warp
  const int nr = max(0, min(kReg ? 2 : RPW, nrows - wr0));                    // rows this warp owns
  const int lr = wr0 + (lane >> 4);                                           // register mode: this lane's row
  const bool has_row = kReg && lr < nrows;
  const bool pusher = kReg && has_row && peer < C;
  unsigned push_mask = 0;  // shared-memory mode, bit r: this lane pushes the warp's r-th row
  if (!kReg) {
    const int step = 32 / C;  // C is 8 or 16: a power of two
    for (int r = 0; r < nr; ++r)
      if (((r - sub) & (step - 1)) == 0) push_mask |= 1u << r;
  }
  const unsigned peer_xs = map_to_cta(smem_u32(s.xs), (unsigned)(peer < C ? peer : 0));
  const unsigned peer_bar = map_to_cta(smem_u32(&xready[0]), (unsigned)(peer < C ? peer : 0));

  double2 wreg[kReg ? NPT : 1];
  auto load_registers = [&](int k) {  // register mode: this lane's column pairs of W_k[row0 + lr, :]
    if (kReg) {
      const double2* src = reinterpret_cast<const double2*>(p.W + ((size_t)k * D + row0 + (has_row ? lr : 0)) * p.Dpad);
#pragma unroll
      for (int j = 0; j < (kReg ? NPT : 1); ++j) {
        const int c2 = (lane & 15) + 16 * j;
        wreg[j] = (has_row && c2 < nc2) ? __ldg(src + c2) : make_double2(0.0, 0.0);
      }
    }
  };

  load_registers(layer);  // (global loads into registers: their latency overlaps refresh_z and the bias rows)

  // Resident MPC server (p.server): everything above is loaded ONCE; the loop below is one control
  // step per request { x0 from the mailbox -> instantiate -> refresh_z -> total_iters layers -> final
  // pass -> answer }.  W stays in registers / shared memory between steps.  A plain launch runs the
  // body once.
  // Resident server, shared-memory caches of what a step reads besides W (srv_cache: when they fit): this
  // CTA's rows of the bias operator [D_k; G D_k] of the current level, of offset_g / offset_c, c_base,
  // d_base, and (CTA 0) K, u_lo, u_hi.  From L2 each of these reads is a dependent 0.7 us round trip.
  double* const c_dg = s.sx0 + 2 + kMaxInlineX0;                 // [R][npad]
  const int perg = (n + C - 1) / C;
  double* const c_og = c_dg + (size_t)p.R * p.npad;                // [perg][nxpad]  g rows [rank perg, ...)
  double* const c_oc = c_og + (size_t)perg * p.mpc_nxpad;          // [R][nxpad]     the z rows this CTA owns
  double* const c_cb = c_oc + (size_t)p.R * p.mpc_nxpad;           // [R]
  double* const c_db = c_cb + p.R;                                 // [R]
  double* const c_K = c_db + p.R;                                  // [nu][nxpad]
  double* const c_ul = c_K + (size_t)p.mpc_nu * p.mpc_nxpad;       // [nu]
  double* const c_uh = c_ul + p.mpc_nu;                            // [nu]
  const bool cached = p.server && p.srv_cache;
  const int zlo = max(row0, n) - n, zhi = max(zlo, min(row0 + nrows, n + m) - n);  // z rows of this CTA: [zlo, zhi)
  int cached_dg_layer = -1;
  auto cache_dg = [&](int k) {  // (all threads; callers synchronise afterwards)
    const double* DG = p.Dk + (size_t)k * (n + m) * p.npad;
    for (int e = t; e < nrows * p.npad; e += kClThreads) {
      const int r = e / p.npad, cidx = e - r * p.npad;
      c_dg[e] = (row0 + r < n + m) ? __ldg(DG + (size_t)(row0 + r) * p.npad + cidx) : 0.0;
    }
    cached_dg_layer = k;
  };
  if (cached) {
    cache_dg(layer);
    const int ga = (int)rank * perg, gb = min(n, ga + perg);
    for (int e = t; e < max(0, gb - ga) * p.mpc_nxpad; e += kClThreads) c_og[e] = p.mpc_og[(size_t)ga * p.mpc_nxpad + e];
    for (int e = t; e < (zhi - zlo) * p.mpc_nxpad; e += kClThreads) c_oc[e] = p.mpc_oc[(size_t)zlo * p.mpc_nxpad + e];
    for (int e = t; e < zhi - zlo; e += kClThreads) { c_cb[e] = p.mpc_cb[zlo + e]; c_db[e] = p.mpc_db[zlo + e]; }
    if (rank == 0) {
      for (int e = t; e < p.mpc_nu * p.mpc_nxpad; e += kClThreads) c_K[e] = p.mpc_K[e];
      for (int e = t; e < p.mpc_nu; e += kClThreads) { c_ul[e] = p.mpc_ulo[e]; c_uh[e] = p.mpc_uhi[e]; }
    }
    __syncthreads();
  }
  unsigned long long served = p.served;
  int resident_layer = -1;  // ladder level whose W slice is in shared memory (shared-memory mode)
  // (two spare words of the barrier block: the kernel may not own static shared memory, its dynamic
  // allocation is the full 227 KB)
  unsigned long long& cmd_s = s.bars[4];
  unsigned long long& want_full_s = s.bars[5];
  unsigned long long* cbar = s.bars + 6;  // resident server: the request has landed in s.sx0
  unsigned long long* gbar = s.bars + 7;  // resident server: g is complete in s.sg
  // The pieces of a step's prologue.  A plain launch runs them in the reference's order; the resident
  // server moves everything that does not depend on the request (barriers, refresh_z, v_0) in FRONT of the
  // wait for it, so that it overlaps the host's turnaround instead of sitting on the step's critical path.
  bool first_step = true;
  auto init_barriers = [&]() {  // no peer pushes into this CTA between its final residual pass of the previous
    if (t == 0) {               // step and the next cluster barrier
      if (!first_step) {
        for (int k = 0; k < 4; ++k) mbar_inval(&s.bars[k]);
        mbar_inval(cbar); mbar_inval(gbar);
      }
      for (int k = 0; k < 4; ++k) mbar_init(&s.bars[k], 1);
      mbar_init(cbar, 1); mbar_init(gbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(&xready[0], xbytes);  // first use: v_2
      mbar_arm(&xready[1], xbytes);  // first use: v_1
      mbar_arm(&nbar[0], 7u * 8u * (unsigned)C);
      mbar_arm(&nbar[1], 7u * 8u * (unsigned)C);
      if (p.server) {
        mbar_arm(cbar, 8u * (unsigned)(2 + p.mpc_nx));  // the request: {number, report flag, x0} from CTA 0
        mbar_arm(gbar, 8u * (unsigned)n);               // g = offset_g x0: every CTA pushes its rows to every CTA
      }
    }
  };
  auto step_vectors = [&]() {  // g and the clamp bounds of the rows this CTA owns (layers.cpp:182-186, 223-226)
    for (int i = t; i < p.npad; i += kClThreads) s.sg[i] = (i < n) ? __ldcg(p.g + i) : 0.0;
    for (int r = t; r < nrows; r += kClThreads) {
      const int row = row0 + r;
      double lo = -INFINITY, hi = INFINITY;  // c~ = [-inf; F o c; -inf], d~ = [+inf; F o d; +inf]
      if (row >= n && row < n + m) {
        lo = s.sF[row - n] * __ldcg(p.c + row - n);
        hi = s.sF[row - n] * __ldcg(p.d + row - n);
      }
      s.slo[r] = lo;
      s.shi[r] = hi;
    }
    __syncthreads();
  };
  auto refresh_z = [&]() {  // Solver::refresh_z (solver.cpp:197-200): z_s <- G_s y_s, in place in p.vq (slot 0)
    for (int i = t; i < p.npad; i += kClThreads) s.uy[i] = (i < n) ? __ldcg(p.vq + i) : 0.0;
    __syncthreads();
    const int per = (m + C - 1) / C;
    const int g0 = (int)rank * per;
    const int g1 = min(m, g0 + per);
    for (int row = g0 + warp; row < g1; row += kClWarps) {
      const double zs = warp_row_dot(p.Gs + (size_t)row * p.npad, s.uy, p.npad, lane);
      if (lane == 0) __stcg(p.vq + n + row, zs);
    }
    __syncthreads();
    cluster_sync_all();  // release/acquire at cluster scope: the peers' rows of z_s are visible
  };
  auto load_v0 = [&]() {  // v_0 -> xs[0]; pad slots of both copies stay zero for the whole step
    for (int i = t; i < XS; i += kClThreads) {
      s.xs[i] = (i < D) ? __ldcg(p.vq + i) : 0.0;
      s.xs[XS + i] = 0.0;
    }
    __syncthreads();
    cluster_sync_all();  // peers write into xs[1] as soon as they finish iteration 1 (and: every peer's
                         // mbarrier initialisation is ordered before the pushes)
  };
  for (;;) {
  unsigned long long req = 0;
  long long t_step = 0;
  if (p.server) {
    // before the request: everything of the step that only needs the previous step's result
    init_barriers();
    refresh_z();
    load_v0();
    // The request.  Warp 0 of CTA 0 polls the host-mapped mailbox, then pushes {number, report flag, x0}
    // into every CTA's shared memory with st.async (completion counted on the receiver's cbar): no L2
    // relay, and x0 is where instantiate needs it.
    if (rank == 0 && warp == 0) {
      int want = 1;
      double* stage = s.norms;  // (2 * 16 * 8 doubles, idle between residual passes)
      const unsigned long long r = server_fetch_request(p, served, lane, want, stage);  // (x0 -> stage[2 ...] and the device copy)
      if (lane == 0) {
        stage[0] = __longlong_as_double((long long)r);
        stage[1] = (double)want;
      }
      __syncwarp();
      const int words = 2 + p.mpc_nx;
      for (int idx = lane; idx < words * C; idx += 32) {
        const int peer_c = idx % C, word = idx / C;
        st_async_f64(map_to_cta(smem_u32(s.sx0 + word), (unsigned)peer_c), stage[word], map_to_cta(smem_u32(cbar), (unsigned)peer_c));
      }
    }
    mbar_wait_cluster(cbar, 0, p.dbg, 7, 0);
    req = (unsigned long long)__double_as_longlong(s.sx0[0]);
    if (t == 0) { cmd_s = req; want_full_s = (unsigned long long)(s.sx0[1] != 0.0); }
    __syncthreads();
    if (req == kSrvExit) break;
    t_step = globaltimer_ns();
    // mpc::instantiate (mpc.cpp:260-270).  g rows: this CTA's share, pushed to every CTA's s.sg (gbar);
    // c, d rows: exactly the z rows this CTA owns in the iterate, so the clamp bounds need no exchange.
    // All of g, c, d also go to global memory (the report's final clamp and later plain calls read them).
    {
      const double* x0s = s.sx0 + 2;
      const int ga = (int)rank * perg, gb = min(n, ga + perg);
      for (int row = ga + warp; row < gb; row += kClWarps) {
        const double* M = cached ? c_og + (size_t)(row - ga) * p.mpc_nxpad : p.mpc_og + (size_t)row * p.mpc_nxpad;
        double acc = 0.0;
        for (int j = lane; j < p.mpc_nx; j += 32) acc = fma(M[j], x0s[j], acc);
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
        if (lane < C) st_async_f64(map_to_cta(smem_u32(s.sg + row), (unsigned)lane), acc, map_to_cta(smem_u32(gbar), (unsigned)lane));
        if (lane == 0) p.g_w[row] = acc;
      }
      for (int j = zlo + warp; j < zhi; j += kClWarps) {
        const double* M = cached ? c_oc + (size_t)(j - zlo) * p.mpc_nxpad : p.mpc_oc + (size_t)j * p.mpc_nxpad;
        double acc = 0.0;
        for (int q = lane; q < p.mpc_nx; q += 32) acc = fma(M[q], x0s[q], acc);
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
        if (lane == 0) {
          const double cj = (cached ? c_cb[j - zlo] : p.mpc_cb[j]) - acc, dj = (cached ? c_db[j - zlo] : p.mpc_db[j]) - acc;
          p.c_w[j] = cj;
          p.d_w[j] = dj;
          s.slo[n + j - row0] = s.sF[j] * cj;   // c~, d~ of this row (layers.cpp:182-186)
          s.shi[n + j - row0] = s.sF[j] * dj;
        }
      }
      for (int r = t; r < nrows; r += kClThreads)
        if (row0 + r < n || row0 + r >= n + m) { s.slo[r] = -INFINITY; s.shi[r] = INFINITY; }
    }
#ifdef CQP_SRV_TRACE
#define SRV_STAMP(k) do { if (p.server && rank == 0 && t == 0) p.mb[kMbX0 + 100 + (k)] = (unsigned long long)(globaltimer_ns() - t_step); } while (0)
#else
#define SRV_STAMP(k) do {} while (0)
#endif
    SRV_STAMP(0);  // instantiate rows pushed
    mbar_wait_cluster(gbar, 0, p.dbg, 8, 0);
    __syncthreads();
    SRV_STAMP(1);  // g complete
    CQP_STAMP0(p.dbg, 3);
    if (cached && cached_dg_layer != layer) { cache_dg(layer); __syncthreads(); }
    cl_load_layer(p, s, layer, row0, nrows, resident_layer != layer, cached ? c_dg : nullptr);  // (bias rows; W only when it changed)
    resident_layer = layer;
    SRV_STAMP(2);  // bias rows done
  } else {
    init_barriers();
    step_vectors();
    CQP_STAMP0(p.dbg, 1);
    if (p.do_refresh) refresh_z();
    CQP_STAMP0(p.dbg, 3);
    cl_load_layer(p, s, layer, row0, nrows, resident_layer != layer);  // (bias rows; the W slice only when it changed)
    resident_layer = layer;
    CQP_STAMP0(p.dbg, 4);
    load_v0();
  }
  first_step = false;
  CQP_STAMP0(p.dbg, 5);

  int n_trace = 1, n_hist = 0, pass = 0;
  if (rank == 0 && t == 0) {
    p.trace[0] = 0;
    p.trace[1] = layer;
  }

  bool converged = false;
  int until_check = p.check_interval;
  int iters_done = 0;
  int have = 0;  // v_have has been awaited (and its barrier re-armed) already
  for (int i = 1; i <= p.total_iters; ++i) {
    // ---- one fused layer: v <- clamp(W v + b, c~, d~)  (solver.cpp:59-63) ----
    const int b = i & 1;
    // Warps without rows (nr == 0) skip the loop's waits: a warp that pushes nothing does not hold
    // the cluster back, so the barrier could run two phases ahead of it; they rejoin at the checks.
    // Warp 0 always owns rows (nrows >= 1), so thread 0 re-arms every phase.
    if (t == 0) CQP_STAMP(p.dbg, i, 0);
    if (i > 1 && have != i - 1 && nr > 0) {
      mbar_wait_cluster(&xready[b ^ 1], ((i - 2) >> 1) & 1, p.dbg, 1, i);  // v_{i-1} landed
      // Safe to re-arm without a CTA barrier: the next phase of this barrier carries v_{i+1}, which
      // no peer sends before it has ALL of v_i, i.e. before every row-owning warp here (each past
      // this wait) pushed its rows of v_i.
      if (t == 0) mbar_arm(&xready[b ^ 1], xbytes);
    }
    if (t == 0) CQP_STAMP(p.dbg, i, 1);
    if (nr > 0) {
      const double2* x2 = reinterpret_cast<const double2*>(s.xs + (size_t)(b ^ 1) * XS);
      if constexpr (kReg) {
        double a0 = 0.0, a1 = 0.0;
        const double2* xl = x2 + (lane & 15);
#pragma unroll
        for (int j = 0; j < NPT; j += 2) {
          const double2 x0 = xl[16 * j];
          a0 = fma(wreg[j].x, x0.x, a0);
          a0 = fma(wreg[j].y, x0.y, a0);
          if (j + 1 < NPT) {
            const double2 x1 = xl[16 * (j + 1)];
            a1 = fma(wreg[j + 1].x, x1.x, a1);
            a1 = fma(wreg[j + 1].y, x1.y, a1);
          }
        }
        if (t == 0) CQP_STAMP(p.dbg, i, 3);
        double tot = a0 + a1;
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, w);
        if (t == 0) CQP_STAMP(p.dbg, i, 2);
        if (pusher) {
          double x = tot + s.sb[lr];
          const double lo = s.slo[lr], hi = s.shi[lr];
          x = x < lo ? lo : x;
          x = x > hi ? hi : x;
          st_async_f64(peer_xs + 8u * (unsigned)(b * XS + row0 + lr), x, peer_bar + 8u * (unsigned)b);
        }
      } else {
        const double2* w2 = reinterpret_cast<const double2*>(s.sW);
        size_t roff[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) roff[r] = (size_t)min(wr0 + r, nrows - 1) * nc2;  // duplicates are not pushed
        double a0[RPW], a1[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) a0[r] = a1[r] = 0.0;
        int c2 = lane;
        for (; c2 + 32 < nc2; c2 += 64) {
          const double2 x0 = x2[c2], x1 = x2[c2 + 32];
#pragma unroll
          for (int r = 0; r < RPW; ++r) {
            const double2 w0 = w2[roff[r] + c2], w1 = w2[roff[r] + c2 + 32];
            a0[r] = fma(w0.x, x0.x, a0[r]);
            a0[r] = fma(w0.y, x0.y, a0[r]);
            a1[r] = fma(w1.x, x1.x, a1[r]);
            a1[r] = fma(w1.y, x1.y, a1[r]);
          }
        }
        if (c2 < nc2) {
          const double2 x0 = x2[c2];
#pragma unroll
          for (int r = 0; r < RPW; ++r) {
            const double2 w0 = w2[roff[r] + c2];
            a0[r] = fma(w0.x, x0.x, a0[r]);
            a0[r] = fma(w0.y, x0.y, a0[r]);
          }
        }
        if (t == 0) CQP_STAMP(p.dbg, i, 3);
        double tot[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) tot[r] = a0[r] + a1[r];
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
          for (int r = 0; r < RPW; ++r) tot[r] += __shfl_xor_sync(0xffffffffu, tot[r], w);
        }
        if (t == 0) CQP_STAMP(p.dbg, i, 2);
        // every lane holds the RPW row sums; lane (peer, sub) pushes rows sub, sub + step, ...
        const unsigned xdst = peer_xs + 8u * (unsigned)(b * XS + row0 + wr0);
        const unsigned bdst = peer_bar + 8u * (unsigned)b;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          if ((push_mask >> r) & 1u) {
            double x = tot[r] + s.sb[wr0 + r];
            const double lo = s.slo[wr0 + r], hi = s.shi[wr0 + r];
            x = x < lo ? lo : x;
            x = x > hi ? hi : x;
            st_async_f64(xdst + 8u * (unsigned)r, x, bdst);
          }
        }
      }
      if (t == 0) CQP_STAMP(p.dbg, i, 6);
    }
    iters_done = i;
    if (--until_check != 0) continue;
    until_check = p.check_interval;

    // ---- convergence check + penalty adaptation (solver.cpp:65-87) ----
    mbar_wait_cluster(&xready[b], ((i - 1) >> 1) & 1, p.dbg, 2, i);  // v_i
    have = i;
    double nrm[7];
    if (t == 0) CQP_STAMP(p.dbg, i, 4);
    cl_residual_pass(p, s, s.xs + (size_t)b * XS, false, pass++, rank, C, nrm);
    if (t == 0) CQP_STAMP(p.dbg, i, 5);
    // (the pass begins with a CTA barrier, so every warp is past its wait on xready[b])
    if (t == 0) mbar_arm(&xready[b], xbytes);
    const double r_prim = nrm[0], r_dual = nrm[1];
    if (rank == 0 && t == 0 && n_hist < p.cap) {
      p.hist_i[2 * n_hist] = i;
      p.hist_i[2 * n_hist + 1] = layer;
      p.hist_r[2 * n_hist] = r_prim;
      p.hist_r[2 * n_hist + 1] = r_dual;
    }
    ++n_hist;
    if (p.adaptive) {
      // one thread evaluates the rule (FP64 sqrt, divisions, log10, the scan of the grid) and hands the
      // result to the others: 512 threads doing it took about a third of the check step
      int* cand_s = reinterpret_cast<int*>(s.cmax + 7);
      if (t == 0) {
        const double rho_cur = grid_v[layer];
        double rho_nom = rho_cur;
        if (!(r_prim == 0.0 || r_dual == 0.0)) {
          const double g_norm = nrm[6];
          double num = nrm[2] < nrm[3] ? nrm[3] : nrm[2];  // std::max({hy, gtl, ||g||, 1e-4})
          num = num < g_norm ? g_norm : num;
          num = num < 1e-4 ? 1e-4 : num;
          double den = nrm[4] < nrm[5] ? nrm[5] : nrm[4];  // std::max({gy, ||z||, 1e-4})
          den = den < 1e-4 ? 1e-4 : den;
          rho_nom = rho_cur * sqrt((r_prim * num) / (r_dual * den));
        }
        const int cand_near = nearest_grid_index_fast(grid_log, grid_bnd, p.L, rho_nom);
        const double qa = rho_nom / rho_cur, qb = rho_cur / rho_nom;
        const double ratio = qa < qb ? qb : qa;
        *cand_s = ratio >= p.threshold ? cand_near : layer;
      }
      __syncthreads();
      const int cand = *cand_s;
      if (cand != layer) {
        layer = cand;
        if (rank == 0 && t == 0 && n_trace < p.cap) {
          p.trace[2 * n_trace] = i;
          p.trace[2 * n_trace + 1] = cand;
        }
        ++n_trace;
        if (cached) { __syncthreads(); cache_dg(layer); __syncthreads(); }
        cl_load_layer(p, s, layer, row0, nrows, true, cached ? c_dg : nullptr);
        resident_layer = layer;
        load_registers(layer);
      }
    }
    if (t == 0) CQP_STAMP(p.dbg, i, 7);
    if (p.early_exit && r_prim <= p.eps_prim && r_dual <= p.eps_dual) {
      converged = true;
      break;
    }
  }

  // ---- epilogue (solver.cpp:90-99) ----
  SRV_STAMP(3);  // iterations issued
  CQP_STAMP0(p.dbg, 6);
  const int bf = iters_done & 1;
  if (iters_done >= 1 && have != iters_done)
    mbar_wait_cluster(&xready[bf], ((iters_done - 1) >> 1) & 1, p.dbg, 3, iters_done);
  double nrm[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double* xfinal = s.xs + (size_t)bf * XS;
  CQP_STAMP0(p.dbg, 7);
  // Server step whose caller takes only u0 (cqp_mpc_step_x0 with out == NULL): the report is not
  // observable, so the final residual evaluation (solver.cpp:94-95) is skipped; iterate and u0 are
  // the same bits.  Only the unscaled controls y[0:nu] are formed, for the extraction.
  const bool fast = p.server && want_full_s == 0ull;
  if (fast) {
    __syncthreads();  // (every warp is past its wait for v_k)
    if (rank == 0) {
      for (int i = t; i < p.mpc_nu; i += kClThreads) s.uy[i] = s.sE[i] * xfinal[i];
      __syncthreads();
    }
  } else {
    if (p.server) {  // the final clamp reads every CTA's rows of c, d from global memory
      __threadfence();
      __syncthreads();
      cluster_sync_all();
    }
    cl_residual_pass(p, s, xfinal, true, pass++, rank, C, nrm);
  }
  CQP_STAMP0(p.dbg, 8);
  // between-launch invariant: p.vq slot 0 = iterate (slots 1..3 keep the grid kernel's sentinel)
  for (int r = t; r < nrows; r += kClThreads) p.vq[row0 + r] = xfinal[row0 + r];
  if (rank == 0) {
    if (cached) {
      // u0 = clamp(-K x0 + y[0:nu], u_lo, u_hi) (bench.cpp:169-175) from the shared-memory copies of K and
      // x0; same operation order as mpc_extract_control
      const double* x0s = s.sx0 + 2;
      for (int c = t; c < p.mpc_nu; c += kClThreads) {
        const double* Krow = c_K + (size_t)c * p.mpc_nxpad;
        double kx = 0.0;
        for (int j = 0; j < p.mpc_nx; ++j) kx = fma(Krow[j], x0s[j], kx);
        double u = -kx + s.uy[c];
        u = u < c_ul[c] ? c_ul[c] : u;
        u = u > c_uh[c] ? c_uh[c] : u;
        p.out_u[c] = u;
      }
    } else {
      mpc_extract_control(p, s.uy, t, p.server ? s.sx0 + 2 : nullptr);
    }
    if (p.Dpad != D && t == 0) p.vq[D] = 0.0;
    if (!p.server || want_full_s) {
      for (int i = t; i < n; i += kClThreads) p.out_y[i] = s.uy[i];
      for (int i = t; i < m; i += kClThreads) {
        p.out_z[i] = s.uz[i];
        p.out_lam[i] = s.ul[i];
      }
    }
    if (t == 0 && fast) p.state[0] = layer;  // (u0-only step: the host does not read the record's head)
    if (t == 0 && !fast) {
      DevResultHead h;
      h.r_prim = nrm[0];
      h.r_dual = nrm[1];
      h.iterations = iters_done;
      h.status = (converged || (nrm[0] <= p.eps_prim && nrm[1] <= p.eps_dual)) ? CQP_SOLVED : CQP_MAX_ITERS;
      h.n_trace = n_trace;
      h.n_hist = n_hist;
      h.final_layer = layer;
      h.final_buf = 0;
      *p.head = h;
      p.state[0] = layer;
    }
  }
  if (!p.server) break;
  SRV_STAMP(4);  // results written
  // answer: the result record is host-mapped; every writer fences system-wide, then one thread
  // publishes the request number.  The cluster barrier also keeps the next step's instantiate /
  // relay from overwriting g, c, d, x0 while a peer still reads them.
  // (a u0-only step wrote nu <= 32 words from warp 0 of CTA 0: only that warp fences)
  if (rank == 0 && t == 0) p.mb[kMbStepNs] = (unsigned long long)(globaltimer_ns() - t_step);  // (up to the fence)
  if (!fast || (rank == 0 && warp == 0)) __threadfence_system();
  if (!fast) __syncthreads(); else __syncwarp();
  SRV_STAMP(5);  // system fence done
  if (rank == 0 && t == 0) p.mb[kMbResp] = req;
  served = req;
  cluster_sync_all();
  }  // server loop
  __syncthreads();
  CQP_STAMP0(p.dbg, 9);
  cluster_sync_all();  // no CTA leaves while a peer could still address its shared memory
  if (p.server && rank == 0 && t == 0) {
    __threadfence_system();
    p.mb[kMbExited] = 1ull;
  }
  CQP_STAMP0(p.dbg, 10);
}

// `set_attrs`: opt the kernel into the full dynamic shared memory and 16-CTA clusters.  Done when
// the handle is configured (ClOp::Fits), never on the launch path; the attributes are per function
// and device, so they are set to the maximum (handles of different sizes share the functions).
template <int RPW, int NPT>
int cluster_launch_cfg(cqp_handle* h, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr, bool set_attrs, size_t extra_smem = 0) {
  auto fn = cluster_kernel<RPW, NPT>;
  if (set_attrs) {
    CQP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
    CQP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3(h->G);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = (size_t)h->smem_bytes + extra_smem;
  cfg.stream = h->stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)h->G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return CQP_OK;
}

enum class ClOp { Launch, Fits };

// Shared memory of the resident server's caches (see the kernel): rows of the bias operator, of the MPC
// template and of K, for one CTA.
size_t server_cache_bytes(const cqp_handle* h) {
  const size_t R = (size_t)h->R, perg = (size_t)(h->n + h->G - 1) / h->G, nxp = (size_t)h->mpc_nxpad, nu = (size_t)h->mpc_nu;
  return sizeof(double) * (R * h->npad + perg * nxp + R * nxp + 2 * R + nu * nxp + 2 * nu);
}

// Launch, or ask whether the device schedules one cluster of h->G CTAs with h->smem_bytes each.
template <int RPW, int NPT>
int cluster_do(ClOp op, cqp_handle* h, const RunParams* p) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  const size_t extra = (op == ClOp::Launch && p && p->server && p->srv_cache) ? server_cache_bytes(h) : 0;
  int rc = cluster_launch_cfg<RPW, NPT>(h, cfg, attr, op == ClOp::Fits, extra);
  if (op == ClOp::Fits) {
    int clusters = 0;
    if (rc != CQP_OK || cudaOccupancyMaxActiveClusters(&clusters, cluster_kernel<RPW, NPT>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return clusters >= 1;
  }
  if (rc) return rc;
  CQP_CUDA(cudaLaunchKernelEx(&cfg, cluster_kernel<RPW, NPT>, *p));
  return CQP_OK;
}

int cluster_dispatch(ClOp op, cqp_handle* h, const RunParams* p) {
  switch (h->npt) {
    case 2: return cluster_do<1, 2>(op, h, p);
    case 4: return cluster_do<1, 4>(op, h, p);
    case 6: return cluster_do<1, 6>(op, h, p);
    case 8: return cluster_do<1, 8>(op, h, p);
    case 10: return cluster_do<1, 10>(op, h, p);
    case 12: return cluster_do<1, 12>(op, h, p);
    case 14: return cluster_do<1, 14>(op, h, p);
    case 16: return cluster_do<1, 16>(op, h, p);
    default: break;
  }
  switch (h->rpw) {
    case 1: return cluster_do<1, 0>(op, h, p);
    case 2: return cluster_do<2, 0>(op, h, p);
    case 3: return cluster_do<3, 0>(op, h, p);
    default: return cluster_do<4, 0>(op, h, p);
  }
}

}  // namespace

int configure_cluster(cqp_handle* h) {
  h->cluster = 0;
  const int D = h->D;
  if (D < 32) return CQP_OK;  // the balanced row split needs D >= C; tiny problems use the grid kernel
  const char* only = std::getenv("CQP_CLUSTER_SIZE");  // test hooks: pin the cluster size (16 or 8),
  const char* mode = std::getenv("CQP_CLUSTER_MODE");  // "smem" forbids the register mode
  const bool allow_reg = !(mode && mode[0] == 's');
  for (int C : {16, 8}) {
    if (only && std::atoi(only) != C) continue;
    const int R = (D + C - 1) / C;
    const int pern = (h->n + C - 1) / C, perm = (h->m + C - 1) / C;
    // register mode: 2 rows per warp (R <= 32), 16 lanes per row, NPT = ceil(nc2 / 16) <= 16 pairs per lane
    const int np = ((h->Dpad >> 1) + 15) / 16;
    for (int reg = allow_reg ? 1 : 0; reg >= 0; --reg) {
      int npt = 0, rpw = 0, xs_stride = h->Dpad;
      if (reg) {
        if (R > 2 * kClWarps || np > 16) continue;
        npt = (np + 1) / 2 * 2;
        xs_stride = 32 * npt;
      } else {
        rpw = (R + kClWarps - 1) / kClWarps;
        if (rpw > kClMaxRpw) continue;
      }
      const int wrows = reg ? 0 : R;
      size_t need = cl_smem_doubles(R, wrows, h->Dpad, xs_stride, h->npad, h->mpad, pern, perm) * sizeof(double);
      int hg = 1;
      if (need > (size_t)kMaxSmemBytes) {  // no room to cache the residual rows: read them through L2
        hg = 0;
        need = cl_smem_doubles(R, wrows, h->Dpad, xs_stride, h->npad, h->mpad, 0, 0) * sizeof(double);
      }
      if (need > (size_t)kMaxSmemBytes) continue;
      h->R = R; h->G = C; h->rpw = rpw; h->npt = npt; h->xs_stride = xs_stride; h->hg_smem = hg;
      h->smem_bytes = (int)need; h->w_smem = reg ? 0 : 1; h->rb = 0;
      if (!cluster_dispatch(ClOp::Fits, h, nullptr)) continue;
      h->cluster = 1;
      return CQP_OK;
    }
  }
  return CQP_OK;
}

int launch_cluster(cqp_handle* h, const RunParams& p0) {
  RunParams p = p0;
  p.w_smem = h->w_smem;
  p.xs_stride = h->xs_stride;
  p.hg_smem = h->hg_smem;
  p.srv_cache = (p.server && (size_t)h->smem_bytes + server_cache_bytes(h) <= (size_t)kMaxSmemBytes) ? 1 : 0;
  return cluster_dispatch(ClOp::Launch, h, &p);
}

}  // namespace cqp
