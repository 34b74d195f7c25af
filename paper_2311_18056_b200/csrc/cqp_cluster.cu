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
//   * All 16 warps are compute warps and own WHOLE rows (warp w: local rows [w RPW, w RPW + RPW)),
//     lanes stride over column pairs (16-byte LDS, conflict-free), two FMA chains per row, a
//     5-step xor butterfly; there is no cross-warp reduction, no publisher warp and no CTA-wide
//     barrier in the iteration loop.
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
__device__ __forceinline__ double warp_row_dot(const double* __restrict__ Mrow, const double* __restrict__ x,
                                               int ncols_pad, int lane) {
  const double2* m2 = reinterpret_cast<const double2*>(Mrow);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int nc2 = ncols_pad >> 1;
  double a0 = 0.0, a1 = 0.0;
  int c2 = lane;
  for (; c2 + 32 < nc2; c2 += 64) {
    const double2 w0 = __ldg(m2 + c2), w1 = __ldg(m2 + c2 + 32);
    const double2 x0 = x2[c2], x1 = x2[c2 + 32];
    a0 = fma(w0.x, x0.x, a0);
    a0 = fma(w0.y, x0.y, a0);
    a1 = fma(w1.x, x1.x, a1);
    a1 = fma(w1.y, x1.y, a1);
  }
  if (c2 < nc2) {
    const double2 w0 = __ldg(m2 + c2);
    const double2 x0 = x2[c2];
    a0 = fma(w0.x, x0.x, a0);
    a0 = fma(w0.y, x0.y, a0);
  }
  return warp_sum(a0 + a1);
}

struct ClSmem {
  double* sW;     // R * Dpad  this CTA's rows of W_k
  double* xs;     // 2 * Dpad  full iterate, double buffered by iteration parity (peers write here)
  double* uy;     // npad      unscaled y (also scratch for g_s)
  double* uz;     // mpad
  double* ul;     // mpad
  double* sb;     // Rp  bias rows
  double* slo;    // Rp
  double* shi;    // Rp
  double* wmax;   // kClWarps * 8   per-warp partial maxima
  double* cmax;   // 8              this CTA's maxima / the cluster-wide result
  double* norms;  // 2 * 16 * 8     per-CTA maxima of a residual pass, by pass parity (peers write here)
  unsigned long long* bars;  // xready[2], nbar[2]
};

__host__ __device__ inline size_t cl_smem_doubles(int R, int Dpad, int npad, int mpad) {
  const int Rp = (R + 1) & ~1;
  return (size_t)R * Dpad + 2 * (size_t)Dpad + npad + 2 * (size_t)mpad + 3 * (size_t)Rp + kClWarps * 8 + 8 +
         2 * 16 * 8 + 8;
}

__device__ __forceinline__ ClSmem cl_carve(unsigned char* raw, const RunParams& p) {
  ClSmem s;
  double* base = reinterpret_cast<double*>(raw);
  const int Rp = (p.R + 1) & ~1;
  s.sW = base;
  s.xs = s.sW + (size_t)p.R * p.Dpad;
  s.uy = s.xs + 2 * p.Dpad;
  s.uz = s.uy + p.npad;
  s.ul = s.uz + p.mpad;
  s.sb = s.ul + p.mpad;
  s.slo = s.sb + Rp;
  s.shi = s.slo + Rp;
  s.wmax = s.shi + Rp;
  s.cmax = s.wmax + kClWarps * 8;
  s.norms = s.cmax + 8;
  s.bars = reinterpret_cast<unsigned long long*>(s.norms + 2 * 16 * 8);
  return s;
}

// Makes layer k current: W slice -> shared memory, bias rows b = -[D_k; G D_k] g_s for the rows
// this CTA owns, 0 on the lambda rows (layers.cpp:168-175).  s.uy is scratch for
// g_s = cost_scale * E o g (layers.cpp:181).
__device__ void cl_load_layer(const RunParams& p, const ClSmem& s, int k, int row0, int nrows) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __syncthreads();
  {
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
  for (int i = t; i < p.npad; i += kClThreads) s.uy[i] = (i < p.n) ? p.cost_scale * (p.E[i] * p.g[i]) : 0.0;
  __syncthreads();
  const int nm = p.n + p.m;
  const double* DG = p.Dk + (size_t)k * nm * p.npad;  // [D_k; G D_k], (n+m) x npad
  for (int r = warp; r < nrows; r += kClWarps) {
    const int row = row0 + r;
    double bias = 0.0;
    if (row < nm) bias = -warp_row_dot(DG + (size_t)row * p.npad, s.uy, p.npad, lane);
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
  __syncthreads();
  // unscale (layers.hpp:57-59)
  for (int i = t; i < p.npad; i += kClThreads) s.uy[i] = (i < n) ? p.E[i] * xs[i] : 0.0;
  for (int i = t; i < p.mpad; i += kClThreads) {
    double z = 0.0, l = 0.0;
    if (i < m) {
      z = xs[n + i] / p.F[i];
      if (final) {  // solver.cpp:94  z = clamp(z, p.c, p.d) in original units
        const double lo = p.c[i], hi = p.d[i];
        z = z < lo ? lo : z;
        z = z > hi ? hi : z;
      }
      l = (p.F[i] * xs[n + m + i]) / p.cost_scale;
    }
    s.uz[i] = z;
    s.ul[i] = l;
  }
  __syncthreads();

  double mx[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  {  // rows of H and G' owned by this CTA (warp per row)
    const int per = (n + C - 1) / C;
    const int h0 = (int)rank * per;
    const int h1 = min(n, h0 + per);
    for (int row = h0 + warp; row < h1; row += kClWarps) {
      const double hy = warp_row_dot(p.H + (size_t)row * p.npad, s.uy, p.npad, lane);
      const double gtl = warp_row_dot(p.Gt + (size_t)row * p.mpad, s.ul, p.mpad, lane);
      const double gi = p.g[row];
      const double dual = (hy + gi) + gtl;  // (H y + g) + G' lambda
      mx[6] = nanmax(mx[6], fabs(gi));
      mx[1] = nanmax(mx[1], fabs(dual));
      mx[2] = nanmax(mx[2], fabs(hy));
      mx[3] = nanmax(mx[3], fabs(gtl));
    }
  }
  {  // rows of G owned by this CTA
    const int per = (m + C - 1) / C;
    const int g0 = (int)rank * per;
    const int g1 = min(m, g0 + per);
    for (int row = g0 + warp; row < g1; row += kClWarps) {
      const double gy = warp_row_dot(p.Gr + (size_t)row * p.npad, s.uy, p.npad, lane);
      const double z = s.uz[row];
      mx[0] = nanmax(mx[0], fabs(gy - z));
      mx[4] = nanmax(mx[4], fabs(gy));
      mx[5] = nanmax(mx[5], fabs(z));
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

template <int RPW>
__global__ void __launch_bounds__(kClThreads, 1) cluster_kernel(const RunParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const ClSmem s = cl_carve(smem_raw, p);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int C = p.G;  // cluster size == grid size
  const unsigned rank = cluster_rank();
  unsigned long long* xready = s.bars;  // [2]: v_i is complete in xs[i & 1]
  unsigned long long* nbar = s.bars + 2;  // [2]: the norms of residual pass `pass` are complete
  const int n = p.n, m = p.m, D = p.D;
  const unsigned xbytes = 8u * (unsigned)D;
  if (t == 0) {
    for (int k = 0; k < 4; ++k) mbar_init(&s.bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(&xready[0], xbytes);  // first use: v_2
    mbar_arm(&xready[1], xbytes);  // first use: v_1
    mbar_arm(&nbar[0], 7u * 8u * (unsigned)C);
    mbar_arm(&nbar[1], 7u * 8u * (unsigned)C);
  }
  // balanced row split: every CTA owns >= 1 row (D >= C), at most p.R = ceil(D / C)
  const int row0 = (int)(((long long)rank * D) / C);
  const int nrows = (int)(((long long)(rank + 1) * D) / C) - row0;
  int layer = p.state[0];

  // clamp bounds of the rows this CTA owns: c~ = [-inf; F o c; -inf], d~ = [+inf; F o d; +inf]
  // (layers.cpp:182-186, 223-226)
  for (int r = t; r < nrows; r += kClThreads) {
    const int row = row0 + r;
    double lo = -INFINITY, hi = INFINITY;
    if (row >= n && row < n + m) {
      lo = p.F[row - n] * p.c[row - n];
      hi = p.F[row - n] * p.d[row - n];
    }
    s.slo[r] = lo;
    s.shi[r] = hi;
  }
  __syncthreads();
  cluster_sync_all();  // every peer's barriers are initialised and armed before anyone pushes

  // optional Solver::refresh_z (solver.cpp:197-200): z_s <- G_s y_s, in place in p.vq (slot 0)
  if (p.do_refresh) {
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
  }

  cl_load_layer(p, s, layer, row0, nrows);

  // v_0 -> xs[0]; pad slots of both copies stay zero for the whole launch
  for (int i = t; i < p.Dpad; i += kClThreads) {
    s.xs[i] = (i < D) ? __ldcg(p.vq + i) : 0.0;
    s.xs[p.Dpad + i] = 0.0;
  }
  __syncthreads();
  cluster_sync_all();  // peers write into xs[1] as soon as they finish iteration 1

  int n_trace = 1, n_hist = 0, pass = 0;
  if (rank == 0 && t == 0) {
    p.trace[0] = 0;
    p.trace[1] = layer;
  }

  // per-lane push target: peer = lane % C gets rows {lane / C, lane / C + 32 / C, ...} of this warp
  const int peer = lane & (C - 1);
  const int sub = lane / C, step = 32 / C;
  const unsigned peer_xs = map_to_cta(smem_u32(s.xs), (unsigned)peer);
  const unsigned peer_bar = map_to_cta(smem_u32(&xready[0]), (unsigned)peer);
  const int wr0 = warp * RPW;                       // first local row of this warp
  const int nr = max(0, min(RPW, nrows - wr0));     // rows this warp owns
  const int nc2 = p.Dpad >> 1;

  bool converged = false;
  int iters_done = 0;
  int have = 0;  // v_have has been awaited (and its barrier re-armed) already
  for (int i = 1; i <= p.total_iters; ++i) {
    // ---- one fused layer: v <- clamp(W v + b, c~, d~)  (solver.cpp:59-63) ----
    const int b = i & 1;
    // Warps without rows (nr == 0) skip the loop's waits: a warp that pushes nothing does not hold
    // the cluster back, so the barrier could run two phases ahead of it; they rejoin at the checks.
    // Warp 0 always owns rows (nrows >= 1), so thread 0 re-arms every phase.
    if (i > 1 && have != i - 1 && nr > 0) {
      mbar_wait_cluster(&xready[b ^ 1], ((i - 2) >> 1) & 1, p.dbg, 1, i);  // v_{i-1} landed
      // Safe to re-arm without a CTA barrier: the next phase of this barrier carries v_{i+1}, which
      // no peer sends before it has ALL of v_i, i.e. before every row-owning warp here (each past
      // this wait) pushed its rows of v_i.
      if (t == 0) mbar_arm(&xready[b ^ 1], xbytes);
    }
    if (nr > 0) {
      const double2* x2 = reinterpret_cast<const double2*>(s.xs + (size_t)(b ^ 1) * p.Dpad);
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
      double tot[RPW];
#pragma unroll
      for (int r = 0; r < RPW; ++r) tot[r] = a0[r] + a1[r];
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
        for (int r = 0; r < RPW; ++r) tot[r] += __shfl_xor_sync(0xffffffffu, tot[r], w);
      }
      // every lane holds the RPW row sums; lane (peer, sub) pushes rows sub, sub + step, ...
      const unsigned xdst = peer_xs + 8u * (unsigned)(b * p.Dpad + row0 + wr0);
      const unsigned bdst = peer_bar + 8u * (unsigned)b;
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        if (r < nr && ((r - sub) % step) == 0 && r >= sub) {
          double x = tot[r] + s.sb[wr0 + r];
          const double lo = s.slo[wr0 + r], hi = s.shi[wr0 + r];
          x = x < lo ? lo : x;
          x = x > hi ? hi : x;
          st_async_f64(xdst + 8u * (unsigned)r, x, bdst);
        }
      }
    }
    iters_done = i;
    if (i % p.check_interval != 0) continue;

    // ---- convergence check + penalty adaptation (solver.cpp:65-87) ----
    mbar_wait_cluster(&xready[b], ((i - 1) >> 1) & 1, p.dbg, 2, i);  // v_i
    have = i;
    double nrm[7];
    cl_residual_pass(p, s, s.xs + (size_t)b * p.Dpad, false, pass++, rank, C, nrm);
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
      const double rho_cur = p.grid[layer];
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
      const int cand_near = nearest_grid_index(p.log_grid, p.L, rho_nom);
      const double qa = rho_nom / rho_cur, qb = rho_cur / rho_nom;
      const double ratio = qa < qb ? qb : qa;
      const int cand = ratio >= p.threshold ? cand_near : layer;
      if (cand != layer) {
        layer = cand;
        if (rank == 0 && t == 0 && n_trace < p.cap) {
          p.trace[2 * n_trace] = i;
          p.trace[2 * n_trace + 1] = cand;
        }
        ++n_trace;
        cl_load_layer(p, s, layer, row0, nrows);
      }
    }
    if (p.early_exit && r_prim <= p.eps_prim && r_dual <= p.eps_dual) {
      converged = true;
      break;
    }
  }

  // ---- epilogue (solver.cpp:90-99) ----
  const int bf = iters_done & 1;
  if (iters_done >= 1 && have != iters_done)
    mbar_wait_cluster(&xready[bf], ((iters_done - 1) >> 1) & 1, p.dbg, 3, iters_done);
  double nrm[7];
  const double* xfinal = s.xs + (size_t)bf * p.Dpad;
  cl_residual_pass(p, s, xfinal, true, pass++, rank, C, nrm);
  // between-launch invariant: p.vq slot 0 = iterate (slots 1..3 keep the grid kernel's sentinel)
  for (int r = t; r < nrows; r += kClThreads) p.vq[row0 + r] = xfinal[row0 + r];
  if (rank == 0) {
    if (p.Dpad != D && t == 0) p.vq[D] = 0.0;
    for (int i = t; i < n; i += kClThreads) p.out_y[i] = s.uy[i];
    for (int i = t; i < m; i += kClThreads) {
      p.out_z[i] = s.uz[i];
      p.out_lam[i] = s.ul[i];
    }
    if (t == 0) {
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
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer could still address its shared memory
}

template <int RPW>
int cluster_launch_cfg(cqp_handle* h, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr) {
  auto fn = cluster_kernel<RPW>;
  CQP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_bytes));
  if (h->G > 8) CQP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3(h->G);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = (size_t)h->smem_bytes;
  cfg.stream = h->stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)h->G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return CQP_OK;
}

template <int RPW>
int cluster_launch_rpw(cqp_handle* h, const RunParams& p) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  int rc = cluster_launch_cfg<RPW>(h, cfg, attr);
  if (rc) return rc;
  CQP_CUDA(cudaLaunchKernelEx(&cfg, cluster_kernel<RPW>, p));
  return CQP_OK;
}

// Does the device schedule one cluster of h->G CTAs with h->smem_bytes each?
template <int RPW>
bool cluster_fits(cqp_handle* h) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  if (cluster_launch_cfg<RPW>(h, cfg, attr) != CQP_OK) { cudaGetLastError(); return false; }
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, cluster_kernel<RPW>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return clusters >= 1;
}

}  // namespace

int configure_cluster(cqp_handle* h) {
  h->cluster = 0;
  const int D = h->D;
  if (D < 32) return CQP_OK;  // the balanced row split needs D >= C; tiny problems use the grid kernel
  const char* only = std::getenv("CQP_CLUSTER_SIZE");  // test hook: pin the cluster size (16 or 8)
  for (int C : {16, 8}) {
    if (only && std::atoi(only) != C) continue;
    const int R = (D + C - 1) / C;
    const int rpw = (R + kClWarps - 1) / kClWarps;
    if (rpw > kClMaxRpw) continue;
    const size_t need = cl_smem_doubles(R, h->Dpad, h->npad, h->mpad) * sizeof(double);
    if (need > (size_t)kMaxSmemBytes) continue;
    h->R = R; h->G = C; h->rpw = rpw; h->smem_bytes = (int)need; h->w_smem = 1; h->rb = 0;
    const bool ok = rpw == 1 ? cluster_fits<1>(h) : rpw == 2 ? cluster_fits<2>(h) : rpw == 3 ? cluster_fits<3>(h) : cluster_fits<4>(h);
    if (!ok) continue;
    h->cluster = 1;
    return CQP_OK;
  }
  return CQP_OK;
}

int launch_cluster(cqp_handle* h, const RunParams& p) {
  switch (h->rpw) {
    case 1: return cluster_launch_rpw<1>(h, p);
    case 2: return cluster_launch_rpw<2>(h, p);
    case 3: return cluster_launch_rpw<3>(h, p);
    default: return cluster_launch_rpw<4>(h, p);
  }
}

}  // namespace cqp
