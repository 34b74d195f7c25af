// Single-QP solve path, all-SM tiers: one persistent cooperative sm_100a kernel per
// solve() / fixed_iters() / mpc_step().  (Problems whose ladder level fits ONE thread-block
// cluster's shared memory, D <~ 650, run the cluster kernel of cqp_cluster.cu instead.)
//
// Replaces the reference's run_loop (/root/reference/proj/src/solver.cpp:43-105) and the
// helpers it calls (iterate :109-117, residuals :119-124, rho_nominal :126-134,
// select_layer :136-142 + nearest_grid_index layers.cpp:38-50), plus the per-MPC-step
// vector update (layers.cpp:177-187), z refresh (solver.cpp:197-200), mpc::instantiate
// (mpc.cpp:260-270) and the control extraction of the closed loop (bench.cpp:169-175).
//
// Design:
//   * W_k (D x D, D = n + 2m) is stored row-major; CTA b owns rows [b*R, b*R + R) and either keeps
//     that slice resident in shared memory (tier 0, run_kernel<RB, false>) or streams it from
//     L2/HBM through a shared-memory ring of cp.async.bulk stages fed from a re-tiled copy of the
//     ladder (tier 1, run_kernel<RB, true>; one contiguous <= 32 KB block per stage).
//   * The iterate is exchanged through L2 WITHOUT a grid barrier: four D-vectors q[0..3] form a
//     ring; iteration i reads v_{i-1} from q[(i-1)&3] and writes v_i to q[i&3].  A slot that has
//     not been written yet holds a sentinel bit pattern (all ones, a NaN no arithmetic
//     produces), so the data word is its own "ready" flag (8-byte accesses are single-copy
//     atomic).
//   * Warp roles inside a CTA (no CTA-wide barrier in the iteration loop):
//       - 16 compute warps form the R dot products (x from shared memory, 16-byte LDS of W,
//         FP64 FMA), reduce them with a shuffle butterfly and hand per-warp partials to
//       - 1 publisher warp, which sums the partials in a FIXED order (bit-reproducible run to
//         run), adds the bias, clamps, stores the rows to q[i&3], wakes the loaders, re-arms
//         its rows of q[(i+2)&3] with the sentinel and fences (off the critical path); in tier 1
//         it is also the producer of the W ring and runs ahead of the compute warps, across
//         iterations too (W does not depend on v);
//       - 3 loader warps poll L2 for v_i into a double-buffered shared-memory copy: all loads in
//         flight, every re-poll round re-issues ALL still-armed entries back to back (one L2 round
//         trip per round); the compute warps, idle during the exchange, fetch along.
//     Hand-offs use parity-split mbarriers (full[2], xready[2], go, wfull[], wempty[]), so a role
//     can run at most one phase ahead and arrivals of different iterations never mix.
//   * Shared-memory-resident tier, default ("direct fetch", run_kernel<.., FETCH = 2, .., WREG>): a compute
//     thread multiplies the same column pairs of every row, so it polls the ring for ITS OWN pairs of
//     v_i and keeps them -- and, where they fit, its columns of W_k -- in registers: no loader warps, no
//     shared-memory staging and no xready hand-off in the loop.  The publisher gates the first poll
//     (a per-CTA adaptive spin in front of `go`), and a warp vote reconverges the warp behind the
//     polling loop.  Same products, same summation order as the staged fetch: bit-identical.
//   * Every check_interval iterations the whole grid evaluates the residuals on the unscaled
//     problem (H y, G' lambda, G y as independent warp-per-row dots spread over the CTAs, seven
//     max-norms exchanged through L2 behind one grid barrier), and every CTA takes the identical
//     rho decision; a switch reloads the W slice and recomputes the bias rows
//     b = -[D_k; G D_k] g_s it owns.
//   * L2/HBM tier, structured layer: the lambda rows of W, [rho G, -diag(rho), I]
//     (layers.cpp:159-161), are streamed as their first n columns only and the publisher adds the
//     two diagonal terms; rows are partitioned by bytes (CTAs [0, G12) own R12 of the first n + m
//     rows, the others R3 lambda rows).  The ring takes all the shared memory the vectors leave, as
//     3 large stages whose chunk width follows the stage size (configure_launch).
//   * The unscaled y / z / lambda of a residual pass alias the idle copy of the iterate (scratch()).
//   * Nothing is launched per iteration; the result record is written straight into host-mapped
//     memory, so the host sees one launch and one stream synchronisation per call.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cqp_internal.h"
#include "cqp_device.cuh"

namespace cqp {
namespace {

// Loader warps: fetch the whole iterate (nc2 column pairs) from ring slot `q` into shared memory
// `xs`.  All loads of a batch are in flight together; only entries still holding the sentinel are
// re-polled.  `lt` is the thread's index among the `nfetch` fetching threads (the loader warps; in the
// L2/HBM tier also the compute warps, which would otherwise idle through the exchange).
template <int U>
__device__ __forceinline__ void fetch_iterate(const double* q, double* xs, int nc2, int lt, int nfetch, int* dbg,
                                              int iter) {
  double2* xs2 = reinterpret_cast<double2*>(xs);
  for (int base = lt; base < nc2; base += nfetch * U) {
    double2 v[U];
    unsigned pending = 0;  // bit u: entry u of this batch is not in shared memory yet
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c2 = base + u * nfetch;
      if (c2 < nc2) {
        v[u] = load_pair(q + 2 * c2);
        pending |= 1u << u;
      }
    }
    long long t0 = 0;
    unsigned spins = 0;
    while (pending) {
      // one pass over the batch: store what has landed, then re-issue ALL armed entries back to
      // back, so that a re-poll round costs one L2 round trip, not one per entry
      unsigned again = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if ((pending >> u) & 1u) {
          if (is_sentinel(v[u].x) || is_sentinel(v[u].y)) again |= 1u << u;
          else xs2[base + u * nfetch] = v[u];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if ((again >> u) & 1u) v[u] = load_pair(q + 2 * (base + u * nfetch));
      pending = again;
      if (pending && (++spins & 0x3FF) == 0) {
        if (t0 == 0) t0 = clock64();
        else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, 100 + base, iter);
      }
    }
  }
}

// Direct fetch (resident tier): compute thread `t` polls ring slot `q` for its own column pairs
// c2 = t + u * kComputeThreads of v_i, keeps them in registers (xv) and leaves a copy in shared memory
// (xs) for the residual passes.  All its loads are in flight together; only armed entries are re-polled.
template <int U>
__device__ __forceinline__ bool fetch_own(const double* q, double* xs, int nc2, int t, double2 (&xv)[U], int* dbg,
                                          int iter) {
  double2* xs2 = reinterpret_cast<double2*>(xs);
  unsigned pending = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int c2 = t + u * kComputeThreads;
    if (c2 < nc2) {
      xv[u] = load_pair(q + 2 * c2);
      pending |= 1u << u;
    }
  }
  long long t0 = 0;
  unsigned spins = 0;
  bool repolled = false;
  while (pending) {
    unsigned again = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if ((pending >> u) & 1u) {
        if (is_sentinel(xv[u].x) || is_sentinel(xv[u].y)) again |= 1u << u;
        else xs2[t + u * kComputeThreads] = xv[u];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((again >> u) & 1u) xv[u] = load_pair(q + 2 * (t + u * kComputeThreads));
    pending = again;
    if (pending) repolled = true;
    if (pending && (++spins & 0x3FF) == 0) {
      if (t0 == 0) t0 = clock64();
      else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, 100 + t, iter);
    }
  }
  return repolled;
}

__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned& epoch, unsigned nblocks, int* dbg) {
  __syncthreads();
  epoch += nblocks;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    unsigned seen, spins = 0;
    long long t0 = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
      if ((++spins & 0x3FF) == 0) {
        if (t0 == 0) t0 = clock64();
        else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, 5, (int)epoch);
      }
    } while (seen < epoch);
  }
  __syncthreads();
}

// The same barrier in two halves, so that work which does not depend on the other CTAs can run
// between the arrival and the wait.
__device__ __forceinline__ void grid_barrier_arrive(unsigned* counter, unsigned& epoch, unsigned nblocks) {
  __syncthreads();
  epoch += nblocks;
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
}

__device__ __forceinline__ void grid_barrier_wait(unsigned* counter, unsigned epoch, int* dbg) {
  if (threadIdx.x == 0) {
    unsigned seen, spins = 0;
    long long t0 = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
      if ((++spins & 0x3FF) == 0) {
        if (t0 == 0) t0 = clock64();
        else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(dbg, 5, (int)epoch);
      }
    } while (seen < epoch);
  }
  __syncthreads();
}

template <int RB>
struct Log2;
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };
template <> struct Log2<16> { static constexpr int v = 4; };

// Reduce RB per-lane partial sums across the warp with RB + (5 - log2 RB) - 1 shuffles of a
// double instead of 5*RB.  Afterwards every lane holds the warp total of row
// (lane >> (5 - log2 RB)).
template <int RB>
__device__ __forceinline__ double warp_butterfly(double (&acc)[RB], int lane) {
  int width = 16;
#pragma unroll
  for (int half = RB / 2; half >= 1; half >>= 1) {
    const bool upper = (lane & width) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? acc[i] : acc[i + half];
      const double keep = upper ? acc[i + half] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, width);
    }
    width >>= 1;
  }
#pragma unroll
  for (; width >= 1; width >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], width);
  return acc[0];
}

// acc[r] += M[r, c2-th column pair] . x pair, for the RB rows of one super-block.
template <int RB>
__device__ __forceinline__ void fma_rows(const double* __restrict__ M, int ld, int nvalid, int c2,
                                         const double2 xv, double (&acc)[RB]) {
  constexpr int CH = RB == 16 ? 4 : RB;  // rows loaded per batch (register pressure at RB = 16)
#pragma unroll
  for (int r0 = 0; r0 < RB; r0 += CH) {
    double2 w[CH];
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      w[r] = (r0 + r < nvalid) ? reinterpret_cast<const double2*>(M + (size_t)(r0 + r) * ld)[c2]
                               : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      acc[r0 + r] = fma(w[r].x, xv.x, acc[r0 + r]);
      acc[r0 + r] = fma(w[r].y, xv.y, acc[r0 + r]);
    }
  }
}

struct Smem {
  double* sW;    // R * Dpad resident slice (tier 0) / streaming ring (tier 1); p.wdoubles doubles
  double* xs;    // 2 * XS     iterate (cache space), double buffered by iteration parity; XS = xs_stride()
                 // The unscaled y / z / lambda of a residual pass (and the g_s scratch of load_layer)
                 // live in whichever of the two buffers does NOT hold the current iterate: see scratch().
  double* sred;  // kWarps * 16          (resident tier: 3 x 16 words: the penalty grid, its log10 and the bounds
                 //                        between neighbours, which the rho rule reads at every check)
  double* spart; // 2 * kComputeWarps * Rcap   per-warp partials of the hot loop, by parity
  double* sb;    // Rp  bias rows
  double* slo;   // Rp
  double* shi;   // Rp
  double* sval;  // 128 + Rp scratch
  unsigned long long* bars;  // full[2], xready[2], go, (pad), wfull[kMaxStages], wempty[kMaxStages]
};

__host__ __device__ inline int round_up(int x, int q) { return (x + q - 1) / q * q; }

// Doubles between the two shared-memory copies of the iterate: room for D entries, and for the
// three separately padded vectors [uy (npad); uz (mpad); ul (mpad)] that alias the idle copy.
__host__ __device__ inline int xs_stride(int Dpad, int npad, int mpad) {
  const int v = npad + 2 * mpad;
  return v > Dpad ? v : Dpad;
}

struct Scratch {
  double* uy;  // npad  unscaled y (also scratch for g_s)
  double* uz;  // mpad  unscaled z
  double* ul;  // mpad  unscaled lambda
};

// `wdoubles`: doubles reserved at the front for W: the resident slice R * Dpad (tier 0) or the
// streaming ring stages * kStageDoubles (tier 1).
__host__ __device__ inline size_t smem_doubles(int R, int rb, int Dpad, int npad, int mpad,
                                               size_t wdoubles, int nparts = kComputeWarps) {
  const int Rp = (R + 1) & ~1;
  const int Rcap = round_up(R, rb);
  return wdoubles + 2 * (size_t)xs_stride(Dpad, npad, mpad) + kWarps * 16 +
         2 * (size_t)nparts * Rcap + 4 * (size_t)Rp + 128 + 8 + 2 * kMaxStages;
}

template <int RB>
__device__ __forceinline__ Smem carve(unsigned char* raw, const RunParams& p) {
  Smem s;
  double* base = reinterpret_cast<double*>(raw);
  const int Rp = (p.R + 1) & ~1;
  const int Rcap = round_up(p.R, RB);
  s.sW = base;
  s.xs = base + p.wdoubles;
  s.sred = s.xs + 2 * xs_stride(p.Dpad, p.npad, p.mpad);
  s.spart = s.sred + kWarps * 16;
  s.sb = s.spart + 2 * p.nparts * Rcap;
  s.slo = s.sb + Rp;
  s.shi = s.slo + Rp;
  s.sval = s.shi + Rp;
  s.bars = reinterpret_cast<unsigned long long*>(s.sval + 128 + Rp);  // 8 + 2 kMaxStages words
  return s;
}

// The scratch vectors alias the copy of the iterate that is idle while `cur` (one of the two
// copies, or null before the first iterate is loaded) is the current one.  Idle means: iteration i
// has completed everywhere in this CTA (its readers of v_{i-1} are done) and the fetch of v_{i+1},
// which overwrites that copy, has not been released yet -- true during a residual pass, the layer
// switch that follows it, the prologue and the epilogue.
__device__ __forceinline__ Scratch scratch(const RunParams& p, const Smem& s, const double* cur) {
  const int XS = xs_stride(p.Dpad, p.npad, p.mpad);
  double* base = (cur == s.xs + XS) ? s.xs : s.xs + XS;
  Scratch q;
  q.uy = base;
  q.uz = base + p.npad;
  q.ul = q.uz + p.mpad;
  return q;
}

// Makes layer k current for this CTA: W slice -> shared memory (tier 0), bias rows for the
// rows it owns: b = -[D_k; G D_k] g_s, 0 on the lambda rows (layers.cpp:168-175).
// Uses s.uy as scratch for g_s = cost_scale * E o g (layers.cpp:181).
template <int RB>
__device__ void load_layer(const RunParams& p, const Smem& s, int k, int row0, int nrows, const double* cur,
                           bool copy_w = true) {
  const int t = threadIdx.x;
  const Scratch sc = scratch(p, s, cur);
  __syncthreads();
  if (p.w_smem && copy_w) {
    const double2* src =
        reinterpret_cast<const double2*>(p.W + ((size_t)k * p.D + row0) * p.Dpad);
    double2* dst = reinterpret_cast<double2*>(s.sW);
    const int count = nrows * (p.Dpad >> 1);
    for (int i = t; i < count; i += kThreads) dst[i] = __ldg(src + i);
  }
  for (int i = t; i < p.npad; i += kThreads)
    sc.uy[i] = (i < p.n) ? p.cost_scale * (p.E[i] * __ldcg(p.g + i)) : 0.0;  // (g, c, d change per server step: not through L1)
  __syncthreads();
  const int nm = p.n + p.m;
  const double* DG = p.Dk + (size_t)k * nm * p.npad;  // [D_k; G D_k], (n+m) x npad
  {  // warp per row, 8 loads per lane in flight (these GEMVs are one-shot: latency, not bandwidth)
    const int lane = t & 31, warp = t >> 5;
    for (int r = warp; r < nrows; r += kWarps) {
      const int row = row0 + r;
      double bias = 0.0;
      if (row < nm) bias = -warp_row_dot_mlp<8>(DG + (size_t)row * p.npad, sc.uy, p.npad, lane);
      else if (p.structured) bias = -p.rho_vec[(size_t)k * p.m + (row - nm)];  // W(row, row - m), see the publisher
      if (lane == 0) s.sb[r] = bias;
    }
  }
  __syncthreads();
}

// Residual pass on the unscaled problem (solver.cpp:67-70,119-134; epilogue :90-95 when
// `final`).  `xs` is the shared-memory copy of the iterate (filled by the loader warps).  On
// return every thread of every CTA holds the same seven norms in out[]:
//   0 ||Gy - z||  1 ||Hy + g + G'lam||  2 ||Hy||  3 ||G'lam||  4 ||Gy||  5 ||z||  6 ||g||
template <int RB>
__device__ void residual_pass(const RunParams& p, const Smem& s, const double* xs, bool final,
                              unsigned& epoch, int& pass, double (&out)[7]) {
  const int t = threadIdx.x;
  const int n = p.n, m = p.m;
  const Scratch sc = scratch(p, s, xs);
  CQP_STAMPR(p.dbg, pass, 0);  // entered (thread 0: the compute warps' last poll has landed)
  __syncthreads();
  CQP_STAMPR(p.dbg, pass, 1);  // every warp of the CTA is here
  // unscale (layers.hpp:57-59)
  for (int i = t; i < p.npad; i += kThreads) sc.uy[i] = (i < n) ? p.E[i] * xs[i] : 0.0;
  for (int i = t; i < p.mpad; i += kThreads) {
    double z = 0.0, l = 0.0;
    if (i < m) {
      z = xs[n + i] / p.F[i];
      if (final) {  // solver.cpp:94  z = clamp(z, p.c, p.d) in original units
        const double lo = __ldcg(p.c + i), hi = __ldcg(p.d + i);
        z = z < lo ? lo : z;
        z = z > hi ? hi : z;
      }
      l = (p.F[i] * xs[n + m + i]) / p.cost_scale;
    }
    sc.uz[i] = z;
    sc.ul[i] = l;
  }
  __syncthreads();
  CQP_STAMPR(p.dbg, pass, 2);  // unscaled

  double mx[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int G = p.G;
  const int lane = t & 31, warp = t >> 5;
  // This CTA owns rows [h0, h0 + cn) of H and G' and rows [g0, g0 + cm) of G: 2 cn + cm independent
  // row dots, one warp each (8 loads per lane in flight), all in parallel; results meet in shared
  // memory (s.sval) and thread r combines row r.
  const int pern = (n + G - 1) / G, perm = (m + G - 1) / G;
  const int h0 = blockIdx.x * pern, g0 = blockIdx.x * perm;
  const int cn = max(0, min(pern, n - h0)), cm = max(0, min(perm, m - g0));
  const int cap3 = 40;  // rows of one kind that fit s.sval (3 * 40 <= 128); larger shares loop
  for (int c0 = 0; c0 < max(cn, cm); c0 += cap3) {
    const int bn = max(0, min(cap3, cn - c0)), bm = max(0, min(cap3, cm - c0));
    for (int d = warp; d < 2 * bn + bm; d += kWarps) {
      double val;
      if (d < bn) val = warp_row_dot_mlp<8>(p.H + (size_t)(h0 + c0 + d) * p.npad, sc.uy, p.npad, lane);
      else if (d < 2 * bn) val = warp_row_dot_mlp<8>(p.Gt + (size_t)(h0 + c0 + d - bn) * p.mpad, sc.ul, p.mpad, lane);
      else val = warp_row_dot_mlp<8>(p.Gr + (size_t)(g0 + c0 + d - 2 * bn) * p.npad, sc.uy, p.npad, lane);
      if (lane == 0) s.sval[d] = val;
    }
    __syncthreads();
    if (t < bn) {
      const int row = h0 + c0 + t;
      const double hy = s.sval[t], gtl = s.sval[bn + t];
      const double gi = __ldcg(p.g + row);
      const double dual = (hy + gi) + gtl;  // (H y + g) + G' lambda
      mx[6] = nanmax(mx[6], fabs(gi));
      mx[1] = nanmax(mx[1], fabs(dual));
      mx[2] = nanmax(mx[2], fabs(hy));
      mx[3] = nanmax(mx[3], fabs(gtl));
    }
    if (t < bm) {
      const double gy = s.sval[2 * bn + t];
      const double z = sc.uz[g0 + c0 + t];
      mx[0] = nanmax(mx[0], fabs(gy - z));
      mx[4] = nanmax(mx[4], fabs(gy));
      mx[5] = nanmax(mx[5], fabs(z));
    }
    __syncthreads();
  }
  CQP_STAMPR(p.dbg, pass, 3);  // row dots done
  // the threads t < 40 hold values: warps 0 and 1 reduce them, then two lanes meet in shared memory
  if (warp < 2) {
#pragma unroll
    for (int k = 0; k < 7; ++k) {
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) mx[k] = nanmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], w));
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 7; ++k) s.sval[warp * 8 + k] = mx[k];
    }
  }
  __syncthreads();
  // The records are double-buffered by pass parity: a final pass may follow a check pass with no
  // grid barrier or iterate exchange in between, so a fast CTA writes its next record while a slow
  // one still reads this pass's (a third pass cannot start before every CTA left this one's barrier
  // AND the next one's).
  double* partial = p.partial + (size_t)(pass & 1) * 8 * (size_t)(G + 1);
  CQP_STAMPR(p.dbg, pass, 4);  // CTA maxima ready
  ++pass;
  if (t < 7) __stcg(partial + (size_t)blockIdx.x * 8 + t, nanmax(s.sval[t], s.sval[8 + t]));
  grid_barrier(p.barrier, epoch, G, p.dbg);
  CQP_STAMPR(p.dbg, pass - 1, 5);  // grid barrier passed
  // all-CTA max of the seven norms: thread b < G fetches CTA b's record (loads in flight
  // together), then a shuffle + shared-memory max (max is exact, so the order is irrelevant).
  // (One warp per norm, five records per lane, saves 0.2 us of the 7 us check in the resident tier -- and
  // costs the streamed instantiations, whose layer loop moves with any change of this function, 4 % per
  // iteration.  The per-warp maxima sit in the upper half of sred: its first 48 words hold the grid.)
  {
    double mine[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) mine[k] = (t < G) ? __ldcg(partial + (size_t)t * 8 + k) : 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) mine[k] = nanmax(mine[k], __shfl_xor_sync(0xffffffffu, mine[k], w));
    }
    const int lane_ = t & 31, warp_ = t >> 5;
    if (lane_ == 0) {
#pragma unroll
      for (int k = 0; k < 7; ++k) s.sred[64 + warp_ * 8 + k] = mine[k];
    }
    __syncthreads();
    if (t < 7) {
      double best = 0.0;
      for (int w = 0; w < kWarps; ++w) best = nanmax(best, s.sred[64 + w * 8 + t]);
      s.sval[t] = best;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 7; ++k) out[k] = s.sval[k];
  __syncthreads();
  CQP_STAMPR(p.dbg, pass - 1, 6);  // all-CTA maxima known
}

// All-SM grid, iterate exchanged through the L2 ring (cooperative launch).  Small problems whose
// ladder level fits one thread-block cluster's shared memory use cqp_cluster.cu instead.
// STREAM selects the L2/HBM tier's code (W through the cp.async.bulk ring) at compile time, so the
// shared-memory-resident tier keeps its registers.
// SERVER: the resident MPC control-step loop (cqp_mpc_server_start) is its own instantiation, so that
// the plain launches keep their code (wrapping the body in the request loop cost the streamed tier 17 %
// per iteration: 11.0 -> 12.9 us at D = 4080, same registers, worse schedule).
// FETCH: who brings v_i into the CTA.  0: the loader warps; 1: loaders + the compute warps (cofetch);
// 2 (resident tier only, "direct"): every compute thread polls the ring for ITS OWN column pairs of v_i
// and keeps them in registers -- a thread multiplies only those columns, so the iterate needs no
// shared-memory staging, no loader warps and no xready hand-off inside the loop (a copy still goes to
// shared memory for the residual passes).  WREG > 0: the thread also keeps its WREG column pairs of the
// CTA's RB rows of W_k in registers (reloaded at a rho switch), so a layer reads nothing from shared
// memory but the partial sums.  Same products, same summation order: the bits do not depend on FETCH / WREG.
template <int RB, bool STREAM, int FETCH = (STREAM ? 1 : 0), bool SERVER = false, int WREG = 0>
__global__ void __launch_bounds__(kThreads, 1) run_kernel(const RunParams p) {
  static_assert(!(STREAM && FETCH == 2), "direct fetch is for the shared-memory-resident tier");
  static_assert(WREG == 0 || FETCH == 2, "register-resident W needs the direct fetch");
  constexpr bool COFETCH = FETCH == 1;
  constexpr bool DIRECT = FETCH == 2;
  constexpr int XU = 2;  // direct fetch: column pairs per compute thread (nc2 <= XU * kComputeThreads)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem s = carve<RB>(smem_raw, p);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // warp roles: [0,16) compute, 16 publisher, [17,21) loaders
  const bool compute = warp < kComputeWarps;
  const bool publisher = warp == kComputeWarps;
  const int lt = t - (kComputeThreads + 32);  // loader thread index (in [0, kLoaderThreads) for loader warps)
  const bool loader = lt >= 0 && lt < kLoaderThreads;
  unsigned long long* full = s.bars;        // [2] compute -> publisher: partials of iteration i
  unsigned long long* xready = s.bars + 2;  // [2] loaders -> compute: v_i is in xs[i&1]
  unsigned long long* go = s.bars + 4;      //     publisher -> loaders: v_i rows published
  unsigned long long* wfull = s.bars + 8;                 // [NS] streamer -> compute: stage holds a W chunk
  unsigned long long* wempty = s.bars + 8 + kMaxStages;   // [NS] compute -> streamer: stage consumed
  // L2/HBM tier: W_k is streamed through a shared-memory ring by the publisher warp with
  // cp.async.bulk (mbarrier complete_tx), kStageRows rows x kStagePairs column pairs per stage; the
  // ring runs ahead of the compute warps, also across iterations (W does not depend on v).
  const int NS = STREAM ? p.stream_stages : 1;
  constexpr bool streaming = STREAM;
  auto init_barriers = [&](bool again) {  // thread 0; `again`: a later server step re-initialises them
    if (again) {
      mbar_inval(&full[0]); mbar_inval(&full[1]); mbar_inval(&xready[0]); mbar_inval(&xready[1]); mbar_inval(go);
      for (int k = 0; k < (STREAM ? NS : 0); ++k) { mbar_inval(&wfull[k]); mbar_inval(&wempty[k]); }
    }
    mbar_init(&full[0], kComputeWarps);
    mbar_init(&full[1], kComputeWarps);
    mbar_init(&xready[0], kLoaderWarps + (COFETCH ? kComputeWarps : 0));  // (unused by the direct fetch)
    mbar_init(&xready[1], kLoaderWarps + (COFETCH ? kComputeWarps : 0));
    mbar_init(go, 1);
    for (int k = 0; k < (STREAM ? NS : 0); ++k) {
      mbar_init(&wfull[k], 1);
      mbar_init(&wempty[k], kComputeWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy
  };
  if (t == 0) init_barriers(false);
  if constexpr (!STREAM) {  // (the streamed instantiation reads the grid from global memory: see the rho rule below)
    if (p.L <= 16 && t < p.L) {  // (visible to thread 0's first decision behind many CTA barriers)
      s.sred[t] = p.grid[t];
      s.sred[16 + t] = p.log_grid[t];
      s.sred[32 + t] = p.grid_bound ? p.grid_bound[t] : 0.0;
    }
  }
  const int n = p.n, m = p.m, D = p.D;
  const int XS = xs_stride(p.Dpad, p.npad, p.mpad);  // doubles between the two copies of the iterate
  const int nc2 = p.Dpad >> 1;
  const int nc2p = (nc2 + 7) & ~7;  // rows of the re-tiled copy are padded to 8 pairs = 128 B
  // rows this CTA owns; L2/HBM tier: column pairs it streams per row (wc2), pair offset of its slice
  // inside a level of Wt (wslice) with row pitch wpitch, rows per super-block (sbr)
  int row0 = blockIdx.x * p.R;
  int nrows = max(0, min(p.R, D - row0));
  int wc2 = nc2, wpitch = nc2p, sbr = STREAM ? p.sb_rows : kStageRows;
  int cwp = (STREAM && p.Wt) ? p.cw12 : kStagePairs;  // column pairs per ring stage
  size_t wslice = (size_t)row0 * nc2p;
  const bool structured = STREAM && p.structured;
  if (structured) {
    const int nm = n + m;
    if ((int)blockIdx.x < p.G12) {
      row0 = blockIdx.x * p.R12;
      nrows = max(0, min(p.R12, nm - row0));
      wslice = (size_t)row0 * nc2p;
    } else {
      const int r3 = ((int)blockIdx.x - p.G12) * p.R3;
      row0 = nm + r3;
      nrows = max(0, min(p.R3, m - r3));
      wc2 = (n + 1) >> 1;
      wpitch = (wc2 + 7) & ~7;
      wslice = (size_t)nm * nc2p + (size_t)r3 * wpitch;
      sbr = p.sb_rows3;
      cwp = p.cw3;
    }
  }
  const int Rcap = round_up(p.R, RB);
  const bool owns_pad = (p.Dpad != D) && (row0 + nrows == D);  // last CTA also drives the pad slot
  unsigned epoch = 0;
  int pass = 0;  // residual passes so far (parity selects the record buffer)

  int layer = p.state[0];
  CQP_STAMP0(p.dbg, 0);  // (-DCQP_TRACE: prologue / epilogue timeline of CTA 0, tools/trace_tier1.py)
  if (blockIdx.x == 0 && t == 0) *p.barrier_next = 0u;  // counter of the NEXT launch (ping-pong)

  // Resident MPC server (SERVER): the loop below is one control step per request { x0 from the
  // mailbox -> instantiate -> refresh_z -> total_iters layers -> final pass -> answer }; the W slice of
  // the resident tier stays in shared memory between steps.  A plain launch runs the body once.
  unsigned long long served = p.served;
  int resident_layer = -1;
  // (two spare words of the barrier block: the kernel may not own static shared memory, its dynamic
  // allocation is the full 227 KB)
  unsigned long long& cmd_s = s.bars[5];
  unsigned long long& want_full_s = s.bars[6];
  // The pieces of a step's prologue.  A plain launch runs them in the reference's order; the resident
  // server runs everything that does not depend on the request (refresh_z, v_0) BEFORE it waits for it.
  auto step_bounds = [&]() {  // c~ = [-inf; F o c; -inf], d~ = [+inf; F o d; +inf] (layers.cpp:182-186, 223-226)
    for (int r = t; r < nrows; r += kThreads) {
      const int row = row0 + r;
      double lo = -INFINITY, hi = INFINITY;
      if (row >= n && row < n + m) {
        lo = p.F[row - n] * __ldcg(p.c + row - n);
        hi = p.F[row - n] * __ldcg(p.d + row - n);
      }
      s.slo[r] = lo;
      s.shi[r] = hi;
    }
  };
  auto refresh_rows = [&]() {  // Solver::refresh_z (solver.cpp:197-200): this CTA's rows of z_s <- G_s y_s, in slot 0
    double* v = p.vq;
    const Scratch sc = scratch(p, s, nullptr);  // (no iterate in shared memory yet)
    for (int i = t; i < p.npad; i += kThreads) sc.uy[i] = (i < n) ? __ldcg(v + i) : 0.0;
    __syncthreads();
    const int per = (m + p.G - 1) / p.G;
    const int g0 = blockIdx.x * per;
    const int g1 = min(m, g0 + per);
    for (int row = g0 + warp; row < g1; row += kWarps) {
      const double zs = warp_row_dot_mlp<8>(p.Gs + (size_t)row * p.npad, sc.uy, p.npad, lane);
      if (lane == 0) __stcg(v + n + row, zs);
    }
  };
  auto load_v0 = [&]() {  // v_0 -> xs[0] (slot 0 holds the iterate between launches / steps)
    for (int i = t; i < XS; i += kThreads) {
      s.xs[i] = (i < D) ? __ldcg(p.vq + i) : 0.0;
      s.xs[XS + i] = 0.0;
    }
    __syncthreads();
  };
  for (;;) {
  unsigned long long req = 0;
  long long t_step = 0;
  if constexpr (SERVER) {
    // before the request: what only needs the previous step's result
    if (served != p.served) {
      grid_barrier(p.barrier, epoch, p.G, p.dbg);  // every CTA's rows of the last iterate are in slot 0
      if (t == 0) init_barriers(true);              // (every role left them behind the last pass)
    }
    refresh_rows();
    grid_barrier(p.barrier, epoch, p.G, p.dbg);    // every CTA's rows of z_s are in slot 0
    load_v0();
    if (warp == 0) {
      int want = 1;
      const unsigned long long r = (blockIdx.x == 0) ? server_fetch_request(p, served, lane, want)
                                                     : (lane == 0 ? server_wait_relay(p, served, want) : 0ull);
      if (lane == 0) { cmd_s = r; want_full_s = (unsigned long long)want; }
    }
    __syncthreads();
    req = cmd_s;
    if (req == kSrvExit) break;
    t_step = globaltimer_ns();
    // mpc::instantiate (mpc.cpp:260-270): this CTA's share of the rows of [g; c; d]
    const int rows = n + m, per = (rows + p.G - 1) / p.G;
    const int r0 = (int)blockIdx.x * per, r1 = min(rows, r0 + per);
    for (int row = r0 + warp; row < r1; row += kWarps)
      instantiate_row(row, lane, p.mpc_og, p.mpc_oc, p.mpc_cb, p.mpc_db, p.mpc_x0, n, p.mpc_nx, p.mpc_nxpad, p.g_w, p.c_w, p.d_w);
    __threadfence();
    grid_barrier(p.barrier, epoch, p.G, p.dbg);    // every CTA's rows of g, c, d are visible
    step_bounds();
    load_layer<RB>(p, s, layer, row0, nrows, nullptr, resident_layer != layer);  // (bias rows; scratch in the second copy)
    resident_layer = layer;
  } else {
    step_bounds();
    if (p.do_refresh) {
      refresh_rows();
      grid_barrier_arrive(p.barrier, epoch, p.G);  // (waited for below: the bias rows do not depend on z_s)
    }
    CQP_STAMP0(p.dbg, 1);  // bounds + this CTA's rows of refresh_z done
    load_layer<RB>(p, s, layer, row0, nrows, nullptr, resident_layer != layer);  // (scratch in the second copy, cleared below)
    resident_layer = layer;
    if (p.do_refresh) grid_barrier_wait(p.barrier, epoch, p.dbg);  // every CTA's rows of z_s are in slot 0
    CQP_STAMP0(p.dbg, 2);  // bias rows done, refresh_z complete
    load_v0();
  }

  int n_trace = 1, n_hist = 0;
  if (blockIdx.x == 0 && t == 0) {
    p.trace[0] = 0;
    p.trace[1] = layer;
  }

  CQP_STAMP0(p.dbg, 3);  // v_0 in shared memory: iterations start
  bool converged = false;
  int iters_done = 0;
  int until_check = p.check_interval;
  constexpr int shift = 5 - Log2<RB>::v;
  unsigned wstage = 0, wphase = 0;  // ring position of the next W chunk to consume (compute) / issue (streamer)
  const int npart = streaming ? 4 : kComputeWarps;  // per-row partials the publisher adds up
  constexpr bool cofetch = COFETCH;  // the compute warps fetch v_i together with the loaders
  const int nfetch = cofetch ? kComputeThreads + kLoaderThreads : kLoaderThreads;  // threads that fetch v_i
  // direct fetch: this thread's column pairs of the current iterate, and (WREG) of the CTA's rows of W_k
  unsigned* early_polls = reinterpret_cast<unsigned*>(&s.bars[7]);  // direct fetch: first polls that came back armed
  int gate = p.gate_cycles;                                          // ... and the publisher's gate (cycles)
  if (DIRECT && t == 0) *early_polls = 0u;
  double2 xv[XU];
  double2 wreg[WREG > 0 ? RB : 1][WREG > 0 ? WREG : 1];
  auto load_wreg = [&]() {  // (after load_layer: the slice of the active level is in shared memory)
    if constexpr (WREG > 0) {
#pragma unroll
      for (int r = 0; r < RB; ++r) {
#pragma unroll
        for (int u = 0; u < WREG; ++u) {
          const int c2 = t + u * kComputeThreads;
          wreg[r][u] = (compute && r < nrows && c2 < nc2)
                           ? reinterpret_cast<const double2*>(s.sW + (size_t)r * p.Dpad)[c2]
                           : make_double2(0.0, 0.0);
        }
      }
    }
  };
  if constexpr (DIRECT) {
    if (compute) {
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int c2 = t + u * kComputeThreads;
        xv[u] = c2 < nc2 ? reinterpret_cast<const double2*>(s.xs)[c2] : make_double2(0.0, 0.0);
      }
    }
    load_wreg();
  }
  for (int i = 1; i <= p.total_iters; ++i) {
    // ---- one fused layer: v <- clamp(W v + b, c~, d~)  (solver.cpp:59-63) ----
    const int b = i & 1;
    const int par = ((i - 1) >> 1) & 1;  // phase parity of the k-th use of a [2]-split barrier
    double* part = s.spart + (size_t)b * p.nparts * Rcap;
    if (DIRECT && compute) {
      if constexpr (DIRECT) {
        if (lane == 0 && warp == 0) { progress(p.dbg, 0, i * 10 + 1); CQP_STAMP(p.dbg, i, 1); }  // v_{i-1} in registers
        if (lane == 0 && warp == 15) CQP_STAMP(p.dbg, i, 10);
        double acc[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] = 0.0;
        if constexpr (WREG > 0) {
#pragma unroll
          for (int r = 0; r < RB; ++r) {
#pragma unroll
            for (int u = 0; u < WREG; ++u) {
              acc[r] = fma(wreg[r][u].x, xv[u].x, acc[r]);
              acc[r] = fma(wreg[r][u].y, xv[u].y, acc[r]);
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < XU; ++u) {
            const int c2 = t + u * kComputeThreads;
            if (c2 < nc2) fma_rows<RB>(s.sW, p.Dpad, nrows, c2, xv[u], acc);
          }
        }
        if (lane == 0 && warp == 0) CQP_STAMP(p.dbg, i, 3);
        const double total = warp_butterfly<RB>(acc, lane);
        if ((lane & ((1 << shift) - 1)) == 0) part[warp * Rcap + (lane >> shift)] = total;
        __syncwarp();
        if (lane == 0 && warp == 0) CQP_STAMP(p.dbg, i, 2);
        if (lane == 0 && warp == 15) CQP_STAMP(p.dbg, i, 11);
        if (lane == 0) mbar_arrive(&full[b]);
        if (lane == 0 && warp == 0) progress(p.dbg, 0, i * 10 + 3);
        // The wait for this CTA's own publish keeps the compute warps of a CTA within one iteration of each
        // other (a warp whose threads own no column pair has nothing to poll for: without the wait it runs
        // ahead and arrives on `full` twice in one phase -- seen as a hang).  Polls issued while the
        // publishes are in flight cannot complete and slow every CTA's publishes down (they hit the very
        // L2 lines the publishes go to): hence the pause (launch_run).
        mbar_wait(go, (i - 1) & 1, p.dbg, 9, i);
        if (p.poll_delay_ns > 0) __nanosleep(p.poll_delay_ns);
        // v_i: this thread's own column pairs, straight from the ring into registers (+ a copy in xs[b]
        // for the residual passes: xs[b] held v_{i-2}, which nobody reads inside the loop)
        const bool repolled = fetch_own<XU>(p.vq + (size_t)(i & 3) * p.ring_ld, s.xs + (size_t)b * XS, nc2, t, xv, p.dbg, i);
        // The vote reconverges the warp behind the polling loop -- without it the lanes whose pairs landed
        // first run the next layer's products on their own, and the layer time follows the arrival pattern
        // (same problem in another handle, i.e. at other addresses: 1.72 or 2.2 - 3.2 us per iteration,
        // tools/ab_instances.py) -- and feeds the publisher's gate: this warp's first poll came back armed.
        if (__any_sync(0xffffffffu, repolled) && lane == 0) atomicAdd(early_polls, 1u);
        if (lane == 0 && warp == 0) CQP_STAMP(p.dbg, i, 0);  // v_i landed (this warp's pairs)
      }
    } else if (compute) {
      if (lane == 0 && warp == 0) { progress(p.dbg, 0, i * 10 + 1); CQP_STAMP(p.dbg, i, 0); }
      if (i > 1) mbar_wait(&xready[b ^ 1], ((i - 2) >> 1) & 1, p.dbg, 1, i);
      if (lane == 0 && warp == 0) { progress(p.dbg, 0, i * 10 + 2); CQP_STAMP(p.dbg, i, 1); }  // v_{i-1} landed
      if (lane == 0 && warp == 15) CQP_STAMP(p.dbg, i, 10);
      const double2* x2 = reinterpret_cast<const double2*>(s.xs + (size_t)(b ^ 1) * XS);
      const double* Wrows = p.w_smem ? s.sW : (p.W + ((size_t)layer * D + row0) * p.Dpad);
      if (streaming) {
        // thread (pc = t & 127, rq = t >> 7): column pair pc of the chunk, rows 4 rq .. 4 rq + 3 of
        // the 16-row super-block; the 4 warps that share rq leave 4 partials per row
        const int pc = t & (kStagePairs - 1), rq = t >> 7;
        for (int rb0 = 0; rb0 < nrows; rb0 += sbr) {
          const int nv = min(sbr, nrows - rb0);
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (int c0 = 0; c0 < wc2; c0 += cwp) {
            const unsigned stage = wstage, ph = wphase;  // (stage, phase) advance without integer division
            if (++wstage == (unsigned)NS) { wstage = 0; wphase ^= 1u; }
            mbar_wait(&wfull[stage], (int)ph, p.dbg, 7, i);
#ifdef CQP_TRACE_CHUNKS
            if (t == 0 && blockIdx.x == 0 && i == CQP_TRACE_AT) {
              const int ci = (rb0 / sbr) * ((wc2 + kStagePairs - 1) / kStagePairs) + c0 / kStagePairs;
              if (ci < 48) reinterpret_cast<volatile long long*>(p.dbg + 64)[ci] = clock64();
            }
#endif
            const double2* st = reinterpret_cast<const double2*>(s.sW) + (size_t)stage * (p.stage_doubles / 2);
            const int cw = p.Wt ? min(cwp, wc2 - c0) : kStagePairs;  // stage row stride (pairs)
            const int cend = p.Wt ? cw : min(kStagePairs, wc2 - c0);
            for (int pp = pc; pp < cend; pp += kStagePairs) {  // (chunks wider than 128 pairs: several passes)
              const double2 xv = x2[c0 + pp];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                if (4 * rq + j < nv) {
                  const double2 w = st[(4 * rq + j) * cw + pp];
                  acc[j] = fma(w.x, xv.x, acc[j]);
                  acc[j] = fma(w.y, xv.y, acc[j]);
                }
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&wempty[stage]);
          }
          const double total = warp_butterfly<4>(acc, lane);  // lane 8 j holds row 4 rq + j
          const int row = rb0 + 4 * rq + (lane >> 3);
          if ((lane & 7) == 0 && row < nrows) part[(warp & 3) * Rcap + row] = total;
        }
      } else
      for (int rb0 = 0; rb0 < nrows; rb0 += RB) {
        const int nv = min(RB, nrows - rb0);
        double acc[RB];
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[r] = 0.0;
        for (int c2 = t; c2 < nc2; c2 += kComputeThreads)
          fma_rows<RB>(Wrows + (size_t)rb0 * p.Dpad, p.Dpad, nv, c2, x2[c2], acc);
        if (lane == 0 && warp == 0 && rb0 == 0) CQP_STAMP(p.dbg, i, 3);
        const double total = warp_butterfly<RB>(acc, lane);
        if ((lane & ((1 << shift) - 1)) == 0) part[warp * Rcap + rb0 + (lane >> shift)] = total;
      }
      __syncwarp();
      if (lane == 0 && warp == 0) CQP_STAMP(p.dbg, i, 2);
      if (lane == 0 && warp == 15) CQP_STAMP(p.dbg, i, 11);
      if (lane == 0) mbar_arrive(&full[b]);
      if (lane == 0 && warp == 0) progress(p.dbg, 0, i * 10 + 3);
      if (cofetch) {
        // L2/HBM tier: large iterate, idle compute warps: they fetch v_i together with the loaders
        // (xs[b] held v_{i-2}, which every warp finished reading before any warp entered iteration i).
        // Like the loaders they start polling only once this CTA has published its own rows: earlier
        // polls cannot succeed and would compete with the W prefetch for L2 bandwidth.
        mbar_wait(go, (i - 1) & 1, p.dbg, 9, i);
        if (p.poll_delay_ns > 0) __nanosleep(p.poll_delay_ns);
        fetch_iterate<4>(p.vq + (size_t)(i & 3) * p.ring_ld, s.xs + (size_t)b * XS, nc2, t, nfetch, p.dbg, i);
        __syncwarp();
        if (lane == 0) mbar_arrive(&xready[b]);
      }
    } else if (publisher) {
      if (lane == 0) { progress(p.dbg, 1, i * 10 + 1); CQP_STAMP(p.dbg, i, 4); }
      // L2/HBM tier: this warp is also the W streamer.  It issues the chunks of iteration i (paced
      // by the compute warps through wempty), publishes v_i, and then starts on iteration i + 1
      // at once, so the first NS chunks of the next iteration load during the iterate exchange.
      if (streaming) {
        for (int rb0 = 0; rb0 < nrows; rb0 += sbr) {
          const int nv = min(sbr, nrows - rb0);
          for (int c0 = 0; c0 < wc2; c0 += cwp) {
            const unsigned stage = wstage, ph = wphase;
            if (++wstage == (unsigned)NS) { wstage = 0; wphase ^= 1u; }
            mbar_wait(&wempty[stage], (int)(ph ^ 1u), p.dbg, 8, i);  // (a fresh barrier passes at once)
            const unsigned bytes = 16u * (unsigned)min(cwp, wc2 - c0);
            if (lane == 0) {
              asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(
                               smem_u32(&wfull[stage])),
                           "r"(bytes * (unsigned)nv)
                           : "memory");
            }
            __syncwarp();
#ifdef CQP_TRACE_CHUNKS
            if (lane == 0 && blockIdx.x == 0 && i == CQP_TRACE_AT) {
              const int ci = (rb0 / sbr) * ((wc2 + kStagePairs - 1) / kStagePairs) + c0 / kStagePairs;
              if (ci < 48) reinterpret_cast<volatile long long*>(p.dbg + 64)[48 + ci] = clock64();
            }
#endif
            if (p.Wt) {  // re-tiled W: the whole stage is one contiguous block
              if (lane == 0) {
                // (row pitches are multiples of 8 pairs = 128 B, so every block is 128 B aligned)
                const double* src = p.Wt + 2 * ((size_t)layer * p.wt_level_pairs + wslice + (size_t)rb0 * wpitch + (size_t)nv * c0);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(s.sW + (size_t)stage * p.stage_doubles)),
                    "l"(src), "r"(bytes * (unsigned)nv), "r"(smem_u32(&wfull[stage]))
                    : "memory");
              }
            } else if (lane < nv) {
              const double* src = p.W + ((size_t)layer * D + row0 + rb0 + lane) * p.Dpad + 2 * (size_t)c0;
              const unsigned dst = smem_u32(s.sW + (size_t)stage * p.stage_doubles + (size_t)lane * (2 * kStagePairs));
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                  "l"(src), "r"(bytes), "r"(smem_u32(&wfull[stage]))
                  : "memory");
            }
          }
        }
      }
      mbar_wait(&full[b], par, p.dbg, 2, i);
      if (lane == 0) { progress(p.dbg, 1, i * 10 + 2); CQP_STAMP(p.dbg, i, 5); }
      double* qout = p.vq + (size_t)(i & 3) * p.ring_ld;
      double* qclr = p.vq + (size_t)((i + 2) & 3) * p.ring_ld;
      const double* xprev = s.xs + (size_t)(b ^ 1) * XS;  // v_{i-1} (complete: the compute warps read it)
      // (one row per lane and trip: issuing three rows' loads together was measured 2-4 % SLOWER
      // per iteration at the robot-sized configs: the first rows are published later)
      for (int r = lane; r < nrows; r += 32) {
        double x = 0.0;
#pragma unroll
        for (int w = 0; w < npart; ++w) x += part[w * Rcap + r];
        // structured layer, lambda row j: + W(row, n + j) z_j + W(row, n + m + j) lambda_j = -rho_j z_j + lambda_j
        if (structured && row0 + r >= n + m) x += fma(s.sb[r], xprev[row0 + r - m], xprev[row0 + r]);
        else x += s.sb[r];
        const double lo = s.slo[r], hi = s.shi[r];
        x = x < lo ? lo : x;
        x = x > hi ? hi : x;
        if (x != x) x = __longlong_as_double(0x7FF8000000000000ll);  // never publish the sentinel
        if (p.fence_mode == 2) publish_release(qout + row0 + r, x);
        else publish(qout + row0 + r, x);
      }
      if (owns_pad && lane == 0) publish(qout + D, 0.0);
      __syncwarp();
      if (lane == 0) CQP_STAMP(p.dbg, i, 6);
      // re-arm this CTA's rows of the slot that will carry v_{i+2}; every reader of its old
      // content (v_{i-2}) finished before any v_{i-1} row was published, and all of v_{i-1} has
      // been consumed by this CTA.  The fence orders the re-arm before the next iteration's
      // publish (off the compute warps' critical path).  The re-arm stores are issued BEFORE the
      // fetching warps are released (B200, direct fetch, D = 900: 1.86 -> 1.75 us per iteration).
      const double sentinel = __longlong_as_double((long long)kSentinel);
      for (int r = lane; r < nrows; r += 32) publish(qclr + row0 + r, sentinel);
      if (owns_pad && lane == 0) publish(qclr + D, sentinel);
      if constexpr (DIRECT) {
        // Gate of the direct fetch.  A first poll that arrives before the last CTA's rows costs a second L2
        // round trip (everybody waits for the slowest CTA); one that arrives late costs only its lateness
        // (measured: a fixed gate of g cycles adds exactly g cycles per iteration).  How long after its own
        // publish a CTA should start polling depends on where it sits in the skew of the grid, so every CTA
        // steers its own gate: the compute warps count the first polls that came back armed, and the publisher
        // releases them a little later after an iteration that had some, a little earlier after one without
        // (B200, D = 600 ... 1020: 1.72 - 1.81 us per iteration, fixed 120 cycles: 1.77 - 1.86).
        const unsigned early = *reinterpret_cast<volatile unsigned*>(early_polls);
        __syncwarp();
        if (lane == 0) *reinterpret_cast<volatile unsigned*>(early_polls) = 0u;  // (the compute warps are parked on `go`)
        if (p.gate_adapt) gate = early ? min(gate + p.gate_up, p.gate_max) : max(gate - p.gate_down, 0);
        if (gate > 0) {
          const long long t0 = clock64();
          while (clock64() - t0 < gate) {}
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(go);
      if (p.fence_mode == 0) __threadfence();
      if (lane == 0) { progress(p.dbg, 1, i * 10 + 3); CQP_STAMP(p.dbg, i, 7); }
    } else if (loader && !DIRECT) {
      if (lt == 0) progress(p.dbg, 2, i * 10 + 1);
      mbar_wait(go, (i - 1) & 1, p.dbg, 3, i);
      if (p.poll_delay_ns > 0) __nanosleep(p.poll_delay_ns);  // (see launch_run)
      if (lt == 0) { progress(p.dbg, 2, i * 10 + 2); CQP_STAMP(p.dbg, i, 8); }
      if (cofetch)
        fetch_iterate<4>(p.vq + (size_t)(i & 3) * p.ring_ld, s.xs + (size_t)b * XS, nc2, kComputeThreads + lt, nfetch,
                         p.dbg, i);
      else
        fetch_iterate<8>(p.vq + (size_t)(i & 3) * p.ring_ld, s.xs + (size_t)b * XS, nc2, lt, nfetch, p.dbg, i);
      __syncwarp();
      if (lt == 0) CQP_STAMP(p.dbg, i, 9);
      if (lane == 0) mbar_arrive(&xready[b]);
      if (lt == 0) progress(p.dbg, 2, i * 10 + 3);
    }
    iters_done = i;
    if (--until_check != 0) continue;  // (a countdown: no integer division in the loop)
    until_check = p.check_interval;

    // ---- convergence check + penalty adaptation (solver.cpp:65-87) ----
    double nr[7];
    const double* xcur = s.xs + (size_t)(i & 1) * XS;
    residual_pass<RB>(p, s, xcur, false, epoch, pass, nr);
    const double r_prim = nr[0], r_dual = nr[1];
    if (blockIdx.x == 0 && t == 0 && n_hist < p.cap) {
      p.hist_i[2 * n_hist] = i;
      p.hist_i[2 * n_hist + 1] = layer;
      p.hist_r[2 * n_hist] = r_prim;
      p.hist_r[2 * n_hist + 1] = r_dual;
    }
    ++n_hist;
    if (p.adaptive) {
      int cand;
      if constexpr (STREAM) {
        // The streamed instantiations keep the rule as every thread's own computation from global memory: ANY
        // change here moves their layer loop's schedule (the single-thread version below cost the streamed
        // loop 5-9 % per iteration, and even the log10-free index 4 % in the resident server), and a check
        // is 1 of 25 iterations of 5-11 us there.
        const double rho_cur = p.grid[layer];
        double rho_nom = rho_cur;
        if (!(r_prim == 0.0 || r_dual == 0.0)) {
          const double g_norm = nr[6];
          double num = nr[2] < nr[3] ? nr[3] : nr[2];  // std::max({hy, gtl, ||g||, 1e-4})
          num = num < g_norm ? g_norm : num;
          num = num < 1e-4 ? 1e-4 : num;
          double den = nr[4] < nr[5] ? nr[5] : nr[4];  // std::max({gy, ||z||, 1e-4})
          den = den < 1e-4 ? 1e-4 : den;
          rho_nom = rho_cur * sqrt((r_prim * num) / (r_dual * den));
        }
        const int cand_near = nearest_grid_index(p.log_grid, p.L, rho_nom);
        const double a = rho_nom / rho_cur, b = rho_cur / rho_nom;
        const double ratio = a < b ? b : a;
        cand = ratio >= p.threshold ? cand_near : layer;
      } else {
        // the rule is evaluated by ONE thread per CTA (sqrt, two divisions and the scan of the grid in FP64:
        // all 640 threads doing it cost 1.8 us per check) and handed to the others through shared memory;
        // every CTA still takes the identical decision from identical data
        int* cand_s = reinterpret_cast<int*>(s.sval + 16);
        if (t == 0) {
          const bool grid_smem = p.L <= 16;
          const double* grid_v = grid_smem ? s.sred : p.grid;
          const double* grid_log = grid_smem ? s.sred + 16 : p.log_grid;
          const double* grid_bnd = p.grid_bound ? (grid_smem ? s.sred + 32 : p.grid_bound) : nullptr;
          const double rho_cur = grid_v[layer];
          double rho_nom = rho_cur;
          if (!(r_prim == 0.0 || r_dual == 0.0)) {
            const double g_norm = nr[6];
            double num = nr[2] < nr[3] ? nr[3] : nr[2];  // std::max({hy, gtl, ||g||, 1e-4})
            num = num < g_norm ? g_norm : num;
            num = num < 1e-4 ? 1e-4 : num;
            double den = nr[4] < nr[5] ? nr[5] : nr[4];  // std::max({gy, ||z||, 1e-4})
            den = den < 1e-4 ? 1e-4 : den;
            rho_nom = rho_cur * sqrt((r_prim * num) / (r_dual * den));
          }
          const int cand_near = nearest_grid_index_fast(grid_log, grid_bnd, p.L, rho_nom);
          const double a = rho_nom / rho_cur, b = rho_cur / rho_nom;
          const double ratio = a < b ? b : a;
          *cand_s = ratio >= p.threshold ? cand_near : layer;
        }
        __syncthreads();
        cand = *cand_s;
      }
      if (cand != layer) {
        layer = cand;
        if (blockIdx.x == 0 && t == 0 && n_trace < p.cap) {
          p.trace[2 * n_trace] = i;
          p.trace[2 * n_trace + 1] = cand;
        }
        ++n_trace;
        load_layer<RB>(p, s, layer, row0, nrows, xcur);
        resident_layer = layer;
        load_wreg();
      }
    }
    CQP_STAMPR(p.dbg, pass - 1, 7);  // decision taken (layer switch included)
    if (p.early_exit && r_prim <= p.eps_prim && r_dual <= p.eps_dual) {
      converged = true;
      break;
    }
  }

  // ---- epilogue (solver.cpp:90-99) ----
  if (t == 0) progress(p.dbg, 3, iters_done * 10 + 9);
  CQP_STAMP0(p.dbg, 4);  // iterations done
  double nr[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double* xfinal = s.xs + (size_t)(iters_done & 1) * XS;
  // Server step whose caller takes only u0 (cqp_mpc_step_x0 with out == NULL): the report is not
  // observable, so the final residual evaluation (solver.cpp:94-95) is skipped; the iterate and u0
  // are the same bits.  What remains of the pass is its grid barrier (every CTA has fetched v_k from the
  // ring before the ring is reset below) and the unscaled controls y[0:nu] for the extraction.
  const bool fast = SERVER && want_full_s == 0ull;
  if (fast) {
    __syncthreads();
    grid_barrier(p.barrier, epoch, p.G, p.dbg);
    if (blockIdx.x == 0) {
      const Scratch sc = scratch(p, s, xfinal);
      for (int i = t; i < p.mpc_nu; i += kThreads) sc.uy[i] = p.E[i] * xfinal[i];
      __syncthreads();
    }
  } else {
    residual_pass<RB>(p, s, xfinal, true, epoch, pass, nr);
  }
  CQP_STAMP0(p.dbg, 5);  // final residual pass done
  // Every CTA has read the final iterate (the pass ends behind a grid barrier): restore the
  // between-launch invariant  q[0] = iterate, q[1..3] = sentinel  for the rows this CTA owns.
  {
    const double sentinel = __longlong_as_double((long long)kSentinel);
    const int count = nrows + (owns_pad ? 1 : 0);
    for (int r = t; r < count; r += kThreads) {
      const int row = row0 + r;
      p.vq[row] = (row < D) ? xfinal[row] : 0.0;
      p.vq[(size_t)p.ring_ld + row] = sentinel;
      p.vq[2 * (size_t)p.ring_ld + row] = sentinel;
      p.vq[3 * (size_t)p.ring_ld + row] = sentinel;
    }
  }
  if (blockIdx.x == 0) {
    const Scratch sc = scratch(p, s, xfinal);  // unscaled solution left by the final residual pass
    mpc_extract_control(p, sc.uy, t);
    if (!SERVER || want_full_s) {
      for (int i = t; i < n; i += kThreads) p.out_y[i] = sc.uy[i];
      for (int i = t; i < m; i += kThreads) {
        p.out_z[i] = sc.uz[i];
        p.out_lam[i] = sc.ul[i];
      }
    }
    if (t == 0) {
      DevResultHead h;
      h.r_prim = nr[0];
      h.r_dual = nr[1];
      h.iterations = iters_done;
      h.status = (converged || (nr[0] <= p.eps_prim && nr[1] <= p.eps_dual)) ? CQP_SOLVED
                                                                             : CQP_MAX_ITERS;
      h.n_trace = n_trace;
      h.n_hist = n_hist;
      h.final_layer = layer;
      h.final_buf = 0;
      *p.head = h;
      p.state[0] = layer;
    }
  }
  if constexpr (!SERVER) break;
  // answer: the result record is host-mapped; every writer fences system-wide, then one thread
  // publishes the request number
  if (blockIdx.x == 0 && t == 0) p.mb[kMbStepNs] = (unsigned long long)(globaltimer_ns() - t_step);  // (up to the fence)
  if (blockIdx.x == 0) __threadfence_system();  // (only CTA 0 writes the record)
  __syncthreads();
  if (blockIdx.x == 0 && t == 0) p.mb[kMbResp] = req;
  served = req;
  }  // server loop
  if (SERVER && blockIdx.x == 0 && t == 0) {
    __threadfence_system();
    p.mb[kMbExited] = 1ull;
  }
  CQP_STAMP0(p.dbg, 6);
}

// ---- small helper kernels ---------------------------------------------------------------

__global__ void transpose_pad_kernel(const double* __restrict__ src, int rows, int cols,
                                     double* __restrict__ dst, int ld, int src_ld) {
  // src column-major rows x cols (leading dimension src_ld) -> dst row-major rows x ld (pad zeroed)
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx: column block, by: row block
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + threadIdx.x, c = bx + j;
    tile[j][threadIdx.x] = (r < rows && c < cols) ? src[(size_t)c * src_ld + r] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < ld) dst[(size_t)r * ld + c] = tile[threadIdx.x][j];
  }
}

__global__ void untranspose_kernel(const double* __restrict__ src, int rows, int cols, int ld,
                                   double* __restrict__ dst) {
  // src row-major rows x ld -> dst column-major rows x cols
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + j, c = bx + threadIdx.x;
    tile[j][threadIdx.x] = (r < rows && c < cols) ? src[(size_t)r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + threadIdx.x, c = bx + j;
    if (r < rows && c < cols) dst[(size_t)c * rows + r] = tile[threadIdx.x][j];
  }
}

// out[row] = alpha * M[row, :] . x(scaled on the fly) ; one warp per row.
// mode 0: x given; mode 1: x_i = cost_scale * E_i * g_i (g_s, for the bias read-back)
__global__ void rows_dot_kernel(const double* __restrict__ M, int rows, int cols, int ld,
                                const double* __restrict__ x, const double* __restrict__ E,
                                double cost_scale, int mode, double alpha,
                                double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double acc = 0.0;
  for (int c = lane; c < cols; c += 32) {
    const double xv = mode ? cost_scale * (E[c] * x[c]) : x[c];
    acc = fma(M[(size_t)warp * ld + c], xv, acc);
  }
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
  if (lane == 0) out[warp] = alpha * acc;
}

// warm_start (solver.cpp:144-156): y_s = y / E, lambda_s = cost_scale * (lambda / F); z_s is
// filled by the refresh kernel afterwards.
__global__ void warm_scale_kernel(const double* __restrict__ y, const double* __restrict__ lam,
                                  const double* __restrict__ E, const double* __restrict__ F,
                                  double cost_scale, int n, int m, double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = y[i] / E[i];
  if (i < m) v[n + m + i] = cost_scale * (lam[i] / F[i]);
}

__global__ void set_state_kernel(int* state, int layer) { state[0] = layer; }

// mpc::instantiate on the device (mpc.cpp:260-270): g = offset_g x0, shift = offset_c x0,
// c = c_base - shift, d = d_base - shift.  One warp per row of [offset_g; offset_c].
struct X0Arg {
  double x[kMaxInlineX0];  // x0 travels in the kernel's parameter block: no host->device copy per step
};

template <bool INLINE>
__global__ void instantiate_kernel(const double* __restrict__ og, const double* __restrict__ oc,
                                   const double* __restrict__ cb, const double* __restrict__ db,
                                   double* __restrict__ x0_dev, const X0Arg xa, int n, int m, int nx, int nxpad,
                                   double* __restrict__ g, double* __restrict__ c, double* __restrict__ d) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const double* x0 = INLINE ? xa.x : x0_dev;
  if (INLINE && blockIdx.x == 0)  // keep a device copy for the control extraction of the run kernel
    for (int j = threadIdx.x; j < nx; j += blockDim.x) x0_dev[j] = xa.x[j];
  if (row >= n + m) return;
  instantiate_row(row, lane, og, oc, cb, db, x0, n, nx, nxpad, g, c, d, !INLINE);
}

// Row-major W_k ([D][Dpad]) -> the streaming layout of the L2/HBM tier (RunParams::Wt): inside the
// row slice of every CTA, every super-block of sbr <= 16 rows (nv valid rows) stores its 128-pair column
// chunks one after the other, each as [nv][cw] pairs.  One thread per (row, column pair).
// Structured layer (G12 > 0): rows < nm are cut into slices of R12 rows with all nc2 pairs; the
// lambda rows follow in slices of R3 rows with only their first ceil(n / 2) pairs (the dense
// block rho G; columns >= n are dropped / zeroed: the publisher adds the two diagonal terms).
struct RetilePlan {
  int D, nc2, n, nm;
  int G12, R12, R3;    // G12 == 0: uniform slices of R12 rows
  int sbr12, sbr3;
  int cw12, cw3;       // chunk width (column pairs per ring stage) of the two slice kinds
};

__global__ void retile_kernel(const double2* __restrict__ src, double2* __restrict__ dst, const RetilePlan q) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)q.D * q.nc2) return;
  const int row = (int)(idx / q.nc2), c2 = (int)(idx - (size_t)row * q.nc2);
  const int nc2p = (q.nc2 + 7) & ~7;  // slices start on 128-byte boundaries (bulk copies are faster aligned)
  int lr, nrows, sbr, wc2 = q.nc2, pitch = nc2p, cwp = q.cw12;
  size_t slice;
  double2 val = src[idx];
  if (q.G12 > 0 && row >= q.nm) {
    wc2 = (q.n + 1) >> 1;
    if (c2 >= wc2) return;
    if (2 * c2 + 1 >= q.n) val.y = 0.0;  // odd n: the pair's second column belongs to block (3,2)
    pitch = (wc2 + 7) & ~7;
    const int r3 = row - q.nm, b = r3 / q.R3;
    lr = r3 - b * q.R3;
    nrows = min(q.R3, (q.D - q.nm) - b * q.R3);
    slice = (size_t)q.nm * nc2p + (size_t)(b * q.R3) * pitch;
    sbr = q.sbr3;
    cwp = q.cw3;
  } else {
    const int limit = q.G12 > 0 ? q.nm : q.D;
    const int b = row / q.R12;
    lr = row - b * q.R12;
    nrows = min(q.R12, limit - b * q.R12);
    slice = (size_t)(b * q.R12) * nc2p;
    sbr = q.sbr12;
  }
  const int sb = lr / sbr, r = lr - sb * sbr;
  const int nv = min(sbr, nrows - sb * sbr);
  const int c = c2 / cwp, pc = c2 - c * cwp;
  const int cw = min(cwp, wc2 - c * cwp);
  dst[slice + (size_t)(sb * sbr) * pitch + (size_t)nv * (c * cwp) + (size_t)r * cw + pc] = val;
}

template <int RB, bool STREAM, int FETCH, int WREG = 0>
int launch_run_rb2(cqp_handle* h, RunParams& p) {
  void* args[] = {&p};  // (shared-memory opt-in: set once per handle by set_run_attributes)
  const void* fn = p.server ? (const void*)run_kernel<RB, STREAM, FETCH, true, WREG> : (const void*)run_kernel<RB, STREAM, FETCH, false, WREG>;
  CQP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(h->G), dim3(kThreads), args, (size_t)h->smem_bytes, h->stream));
  return CQP_OK;
}

// Register-resident W (direct fetch): instantiated where RB rows x WREG column pairs (4 registers each)
// leave the kernel inside its 96-register budget.
template <int RB> constexpr int kMaxWreg = RB == 4 ? 2 : (RB == 8 ? 1 : 0);

template <int RB>
int launch_run_rb(cqp_handle* h, RunParams& p) {
  if (!p.w_smem && p.stream_stages > 0) return launch_run_rb2<RB, true, 1>(h, p);
  if (p.cofetch == 2) {
    if constexpr (kMaxWreg<RB> >= 2) if (p.wreg == 2) return launch_run_rb2<RB, false, 2, 2>(h, p);
    if constexpr (kMaxWreg<RB> >= 1) if (p.wreg == 1) return launch_run_rb2<RB, false, 2, 1>(h, p);
    return launch_run_rb2<RB, false, 2>(h, p);
  }
  return p.cofetch ? launch_run_rb2<RB, false, 1>(h, p) : launch_run_rb2<RB, false, 0>(h, p);
}

// Opt every instance of the grid kernel this handle can launch into the full 227 KB of dynamic
// shared memory -- once, at handle creation, not per launch (the attribute is per function and
// device, so it is set to the maximum: handles of different sizes share the functions).
template <int RB>
int set_run_attributes_rb() {
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  CQP_CUDA(cudaFuncSetAttribute(run_kernel<RB, false, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes));
  if constexpr (kMaxWreg<RB> >= 1) {
    CQP_CUDA((cudaFuncSetAttribute(run_kernel<RB, false, 2, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)));
    CQP_CUDA((cudaFuncSetAttribute(run_kernel<RB, false, 2, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)));
  }
  if constexpr (kMaxWreg<RB> >= 2) {
    CQP_CUDA((cudaFuncSetAttribute(run_kernel<RB, false, 2, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)));
    CQP_CUDA((cudaFuncSetAttribute(run_kernel<RB, false, 2, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemBytes)));
  }
  return CQP_OK;
}

int set_run_attributes(int rb) {
  switch (rb) {
    case 4: return set_run_attributes_rb<4>();
    case 8: return set_run_attributes_rb<8>();
    default: return set_run_attributes_rb<16>();
  }
}

int env_int(const char* name, int fallback) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : fallback;
}

}  // namespace

// Tuning / test knobs are read from the environment ONCE, when the handle is created; nothing on
// the per-launch path (a kHz MPC loop) touches the environment.
static void read_knobs(cqp_handle* h) {
  h->knob_poll_delay_ns = env_int("CQP_POLL_DELAY_NS", -1);  // -1: the tier's default
  // 0: fence after the re-arm (default); 2: release-store publish.  (The former mode 1, no fence at
  // all, broke the ring's ordering argument and is gone: it maps to 0.)
  h->knob_fence_mode = env_int("CQP_FENCE_MODE", 0) == 2 ? 2 : 0;
  h->knob_cofetch = env_int("CQP_COFETCH", 2);  // 0: loader warps only; 1: + compute warps; 2: direct fetch (resident tier)
  h->knob_wreg = env_int("CQP_WREG", 1);
  // direct fetch, the publisher's gate: "initial cycles, adapt (0/1), step up, step down, maximum"
  if (const char* e = std::getenv("CQP_GATE"))
    std::sscanf(e, "%d,%d,%d,%d,%d", &h->knob_gate[0], &h->knob_gate[1], &h->knob_gate[2], &h->knob_gate[3], &h->knob_gate[4]);
  h->knob_exact_log = env_int("CQP_EXACT_LOG", 0) != 0;  // A/B: always take log10 in the rho rule
  h->knob_sb_balance = env_int("CQP_SB_BALANCE", 1) != 0;
  h->knob_no_retile = std::getenv("CQP_NO_RETILE") != nullptr;
  h->knob_wide_chunks = env_int("CQP_WIDE_CHUNKS", 1) != 0;
}

int configure_launch(cqp_handle* h) {
  const int D = h->D;
  read_knobs(h);
  h->cluster = 0;
  // Small problems (one ladder level fits the shared memory of ONE thread-block cluster) run the
  // cluster kernel of cqp_cluster.cu: the iterate never leaves the SMs.  CQP_FORCE_TIER=0/1 pins
  // the all-SM grid kernel (tests, A/B measurements).
  const char* force_tier = std::getenv("CQP_FORCE_TIER");
  const bool force_grid = force_tier && (force_tier[0] == '0' || force_tier[0] == '1');
  if (!force_grid && configure_cluster(h) == CQP_OK && h->cluster) {
    // Where the cluster kernel would have to keep W_k in shared memory (more than 32 rows per CTA: D > 512)
    // the all-SM grid with the direct fetch is faster (B200, D = 540: 2.29 vs 1.57 us per iteration; D = 420,
    // register mode: 1.51 vs 1.88).  The test hooks that pin a cluster shape keep the cluster kernel.
    const bool pinned = std::getenv("CQP_CLUSTER_SIZE") || std::getenv("CQP_CLUSTER_MODE") ||
                        (force_tier && force_tier[0] == '2');
    if (h->npt > 0 || pinned || h->knob_cofetch != 2) return CQP_OK;
  }
  h->cluster = 0;
  h->structured = 0;
  h->nparts = kComputeWarps;
  int G = h->num_sms;
  int R = (D + G - 1) / G;
  if (R < 1) R = 1;
  G = (D + R - 1) / R;
  h->R = R;
  h->G = G;
  h->rb = R <= 4 ? 4 : (R <= 8 ? 8 : 16);
  h->wdoubles = R * h->Dpad;
  h->stream_stages = 0;
  size_t need = smem_doubles(R, h->rb, h->Dpad, h->npad, h->mpad, (size_t)h->wdoubles) * sizeof(double);
  h->w_smem = need <= (size_t)kMaxSmemBytes ? 1 : 0;
  if (force_tier && force_tier[0] == '1') h->w_smem = 0;  // test hook: stream W from L2/HBM
  // Resident tier, direct fetch (run_kernel, FETCH == 2): needs every row of the CTA in one row block and at
  // most two column pairs per compute thread.
  h->fetch = h->knob_cofetch ? 1 : 0;
  if (h->w_smem && h->knob_cofetch == 2 && R <= h->rb && (h->Dpad >> 1) <= 2 * kComputeThreads) h->fetch = 2;
  if (!h->w_smem) {
    // L2/HBM tier: give the rest of the shared memory to the W streaming ring
    const size_t base = smem_doubles(R, h->rb, h->Dpad, h->npad, h->mpad, 0) * sizeof(double);
    if (base > (size_t)kMaxSmemBytes) {
      set_error("problem too large for the persistent kernel's shared-memory vectors");
      return CQP_ERR_CAPACITY;
    }
    // Ring plan: everything the vectors leave free goes to the ring, cut into a FEW LARGE stages
    // (one cp.async.bulk each).  Measured on B200: the per-SM streaming rate grows with the bytes in
    // flight (quadruped-sized: 3 x 30 KB were latency-bound at 66 GB/s per SM) and with the copy
    // size (Atlas-sized, same bytes in flight: 4 x 28 KB 7.3 us per iteration, 2 x 64 KB 6.2 us).
    const bool no_retile = h->knob_no_retile;
    int want_stages = 3;
    if (const char* e = std::getenv("CQP_STREAM_STAGES")) want_stages = std::max(2, std::min(kMaxStages, std::atoi(e)));
    auto plan_ring = [&](size_t base_bytes, int& stages, int& stage_doubles) {
      stages = 0;
      stage_doubles = kStageDoubles;
      if (base_bytes >= (size_t)kMaxSmemBytes) return;
      const size_t avail = (size_t)kMaxSmemBytes - base_bytes;
      if (no_retile) {  // row-segment streaming: fixed 16 x 128-pair stages
        stages = std::min(kMaxStages, (int)(avail / (kStageDoubles * sizeof(double))));
        if (stages < 2) stages = 0;
        return;
      }
      for (int ns = want_stages; ns >= 2; --ns) {
        const size_t sb = (avail / ns) & ~(size_t)127;
        if (sb >= kStageDoubles * sizeof(double)) { stages = ns; stage_doubles = (int)(sb / sizeof(double)); return; }
      }
    };
    // handles that always stream keep 4 partial sums per row instead of 16
    int stages = 0;
    h->nparts = 4;
    size_t base_used = smem_doubles(R, h->rb, h->Dpad, h->npad, h->mpad, 0, 4) * sizeof(double);
    plan_ring(base_used, stages, h->stage_doubles);
    if (stages < 2) {  // no room for a ring: plain global loads, 16 partials
      h->nparts = kComputeWarps;
      base_used = base;
      stages = 0;
      h->stage_doubles = kStageDoubles;
    }
    h->stream_stages = stages;
    h->wdoubles = stages * h->stage_doubles;
    need = base_used + (size_t)h->wdoubles * sizeof(double);
    // Structured layer: the lambda rows are streamed as n columns instead of D, so they go to
    // fewer CTAs with more rows each: pick G12 + G3 <= G that minimises the largest per-CTA
    // byte count max(R12 D, R3 n).  CQP_SINGLE_DENSE=1 keeps the dense layer (A/B runs).
    const char* dense = std::getenv("CQP_SINGLE_DENSE");
    const int n = h->n, m = h->m, nm = n + m;
    if (stages >= 2 && !(dense && dense[0] == '1') && !h->knob_no_retile && m >= 1 && n >= 2 && G >= 2) {
      // a lambda row costs more than its bytes (many short rows: more ring stages per byte, more rows
      // for the single publisher warp), so its CTAs get a little less than an equal share of bytes
      double lambda_weight = 1.25;  // (B200: Atlas-sized 6.3 -> 5.3 us per iteration, quadruped-sized 11.2 -> 10.8; 1.1 .. 1.5 alike)
      if (const char* e = std::getenv("CQP_LAMBDA_WEIGHT")) lambda_weight = std::atof(e);
      long long best = -1;
      int bestR12 = 0, bestR3 = 0;
      for (int g12 = 1; g12 < G; ++g12) {
        const int r12 = (nm + g12 - 1) / g12, r3 = (m + (G - g12) - 1) / (G - g12);
        const long long cost = std::max((long long)r12 * D, (long long)(lambda_weight * r3 * n));
        if (best < 0 || cost < best) { best = cost; bestR12 = r12; bestR3 = r3; }
      }
      const int Rs = std::max(bestR12, bestR3);
      const size_t base_s = smem_doubles(Rs, 16, h->Dpad, h->npad, h->mpad, 0, 4) * sizeof(double);
      int stages_s = 0, stage_doubles_s = kStageDoubles;
      plan_ring(base_s, stages_s, stage_doubles_s);
      const bool force = std::getenv("CQP_FORCE_STRUCTURED") != nullptr;  // tests: also where it does not pay
      if (stages_s >= 2 && (best < (long long)(lambda_weight * R * D) || force)) {
        h->structured = 1;
        h->R12 = bestR12; h->R3 = bestR3;
        h->G12 = (nm + bestR12 - 1) / bestR12;
        h->G = h->G12 + (m + bestR3 - 1) / bestR3;
        h->R = Rs;
        h->rb = 16;
        h->stream_stages = stages_s;
        h->stage_doubles = stage_doubles_s;
        h->wdoubles = stages_s * h->stage_doubles;
        need = base_s + (size_t)h->wdoubles * sizeof(double);
      }
    }
  }
  h->smem_bytes = (int)need;
  return set_run_attributes(h->rb);
}

// Rows per super-block of the W stream: the R rows of a CTA are cut into ceil(R / 16) equal parts
// (R = 18 -> 9 + 9 rather than 16 + 2, so that no ring stage is nearly empty).
static int stream_sb_rows(const cqp_handle* h, int R) {
  if (!h->knob_sb_balance) return kStageRows;  // A/B knob (CQP_SB_BALANCE=0)
  const int nsb = (R + kStageRows - 1) / kStageRows;
  return (R + nsb - 1) / nsb;
}

// Column pairs per ring stage for super-blocks of up to `sbr` rows streaming `wc2` pairs per row: as
// wide as the 32 KB stage allows (multiple of 8 pairs = 128 B), then evened out over the chunks of
// a row so that no stage is nearly empty.  CQP_WIDE_CHUNKS=0 keeps 128-pair chunks (A/B runs).
static int stream_chunk_pairs(const cqp_handle* h, int sbr, int wc2, int stage_doubles) {
  if (!h->knob_wide_chunks) return kStagePairs;
  const int cwmax = ((stage_doubles / 2) / sbr) & ~7;
  const int nch = (wc2 + cwmax - 1) / cwmax;
  const int even = (((wc2 + nch - 1) / nch) + 7) & ~7;
  return std::max(kStagePairs, std::min(even, cwmax));
}

// double2 elements of one re-tiled ladder level (rows padded to 8 pairs = 128 bytes)
static size_t wt_level_pairs(const cqp_handle* h) {
  const int nc2p = ((h->Dpad >> 1) + 7) & ~7;
  if (!h->structured) return (size_t)h->D * nc2p;
  const int wp3 = (((h->n + 1) >> 1) + 7) & ~7;
  return (size_t)(h->n + h->m) * nc2p + (size_t)h->m * wp3;
}

// L2/HBM tier: build the streaming copy of the ladder (RunParams::Wt).  Called once W is complete
// (end of handle creation); launch_run re-checks so that a handle never streams a stale copy.
int prepare_streaming(cqp_handle* h) {
  if (h->cluster || h->w_smem || h->stream_stages <= 0 || h->Wt || h->knob_no_retile) return CQP_OK;
  const size_t per = (size_t)h->D * h->Dpad;
  const size_t per_t = 2 * wt_level_pairs(h);  // re-tiled level: rows padded to 128 bytes
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&h->Wt), sizeof(double) * per_t * h->L));
  CQP_CUDA(cudaMemsetAsync(h->Wt, 0, sizeof(double) * per_t * h->L, h->stream));
  const size_t pairs = per / 2;
  RetilePlan q{};
  q.D = h->D; q.nc2 = h->Dpad >> 1; q.n = h->n; q.nm = h->n + h->m;
  if (h->structured) {
    q.G12 = h->G12; q.R12 = h->R12; q.R3 = h->R3;
    q.sbr12 = stream_sb_rows(h, h->R12); q.sbr3 = stream_sb_rows(h, h->R3);
  } else {
    q.G12 = 0; q.R12 = h->R; q.R3 = 1; q.sbr12 = stream_sb_rows(h, h->R); q.sbr3 = 1;
  }
  q.cw12 = h->cw12 = stream_chunk_pairs(h, q.sbr12, q.nc2, h->stage_doubles);
  q.cw3 = h->cw3 = stream_chunk_pairs(h, q.sbr3, (h->n + 1) >> 1, h->stage_doubles);
  for (int k = 0; k < h->L; ++k) {
    retile_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, h->stream>>>(
        reinterpret_cast<const double2*>(h->W + per * k), reinterpret_cast<double2*>(h->Wt + per_t * k), q);
    CQP_CUDA(cudaGetLastError());
  }
  return CQP_OK;
}

int launch_run(cqp_handle* h, bool early_exit, int total_iters, bool do_refresh) {
  RunParams p{};
  p.n = h->n; p.m = h->m; p.D = h->D;
  p.npad = h->npad; p.mpad = h->mpad; p.Dpad = h->Dpad;
  p.L = h->L; p.R = h->R; p.G = h->G; p.w_smem = h->w_smem;
  p.W = h->W; p.Dk = h->Dk; p.H = h->H; p.Gr = h->Gr; p.Gt = h->Gt; p.Gs = h->Gs;
  p.E = h->E; p.F = h->F; p.cost_scale = h->cost_scale;
  p.grid = h->dgrid; p.log_grid = h->dlog_grid;
  p.grid_bound = (h->grid_bounds && !h->knob_exact_log) ? h->dlog_grid + h->L : nullptr;
  p.g = h->g; p.c = h->c; p.d = h->d;
  p.vq = h->vq; p.ring_ld = h->ring_ld; p.state = h->state; p.partial = h->partial;
  p.eps_prim = h->s.eps_prim; p.eps_dual = h->s.eps_dual; p.threshold = h->s.rho_switch_threshold;
  p.check_interval = h->s.check_interval; p.adaptive = h->s.adaptive_rho;
  p.early_exit = early_exit ? 1 : 0; p.total_iters = total_iters; p.do_refresh = do_refresh ? 1 : 0;
  p.cap = h->res_cap;
  unsigned char* base = static_cast<unsigned char*>(h->dres);
  p.head = reinterpret_cast<DevResultHead*>(base);
  size_t off = sizeof(DevResultHead);
  p.trace = reinterpret_cast<int*>(base + off); off += sizeof(int) * 2 * (size_t)h->res_cap;
  p.hist_i = reinterpret_cast<int*>(base + off); off += sizeof(int) * 2 * (size_t)h->res_cap;
  p.hist_r = reinterpret_cast<double*>(base + off); off += sizeof(double) * 2 * (size_t)h->res_cap;
  p.out_y = reinterpret_cast<double*>(base + off); off += sizeof(double) * (size_t)h->n;
  p.out_z = reinterpret_cast<double*>(base + off); off += sizeof(double) * (size_t)h->m;
  p.out_lam = reinterpret_cast<double*>(base + off); off += sizeof(double) * (size_t)h->m;
  p.out_u = reinterpret_cast<double*>(base + off);
  if (h->mpc_extract) {
    p.mpc_K = h->mpc_K; p.mpc_x0 = h->mpc_x0; p.mpc_ulo = h->mpc_ulo; p.mpc_uhi = h->mpc_uhi;
    p.mpc_nx = h->mpc_nx; p.mpc_nxpad = h->mpc_nxpad; p.mpc_nu = h->mpc_nu;
  }
  if (h->srv_running) {  // (set by server_launch around this call)
    p.server = 1;
    p.mb = h->mb_dev; p.served = h->srv_req; p.srv_seq = h->srv_seq; p.idle_ns = h->srv_idle_ns;
    p.mpc_og = h->mpc_og; p.mpc_oc = h->mpc_oc; p.mpc_cb = h->mpc_cb; p.mpc_db = h->mpc_db;
    p.mpc_x0_w = h->mpc_x0; p.g_w = h->g; p.c_w = h->c; p.d_w = h->d;
  }
  // The other CTAs publish within a few hundred ns of this one: a first poll issued right at `go`
  // mostly finds sentinels and costs a second L2 round trip, and the extra polling traffic slows the
  // publishes themselves.  A short pause before the first poll is a net win (B200, D = 900 / 1500:
  // 2.90 -> 2.60 / 4.11 -> 3.78 us per iteration at 100-200 ns; 400 ns is too long).
  const bool delay_set = h->knob_poll_delay_ns >= 0;
  p.poll_delay_ns = delay_set ? h->knob_poll_delay_ns : 150;
  p.fence_mode = h->knob_fence_mode;
  // grid-barrier counters ping-pong between launches: this launch counts on barrier[parity]
  // (zeroed by the previous launch, or at allocation) and zeroes the other one.  The parity only
  // advances once the launch has been accepted (see the end of this function): a failed launch
  // never ran, so it neither used its counter nor zeroed the other one.
  p.barrier = h->barrier + (h->launch_parity & 1);
  p.barrier_next = h->barrier + ((h->launch_parity + 1) & 1);
  p.dbg = h->dbg_dev;
  auto launched = [&](int rc) {
    if (rc == CQP_OK) h->launch_parity ^= 1;
    return rc;
  };
  if (h->cluster) return launched(launch_cluster(h, p));
  int rc_stream = prepare_streaming(h);  // (no-op unless the ladder was replaced)
  if (rc_stream) return rc_stream;
  p.Wt = (!h->w_smem) ? h->Wt : nullptr;
  p.wdoubles = h->wdoubles;
  p.stream_stages = h->stream_stages;
  p.sb_rows = stream_sb_rows(h, h->structured ? h->R12 : h->R);
  p.structured = (h->structured && p.Wt) ? 1 : 0;
  p.G12 = h->G12; p.R12 = h->R12; p.R3 = h->R3;
  p.sb_rows3 = h->structured ? stream_sb_rows(h, h->R3) : 1;
  p.cw12 = h->cw12; p.cw3 = h->cw3;  // (what prepare_streaming re-tiled Wt with)
  p.stage_doubles = p.Wt ? h->stage_doubles : kStageDoubles;
  // resident tier: the compute warps, idle during the exchange, fetch v_i along with the loader warps
  // (B200, 1000 iterations: D = 900 2576 -> 2468 us, D = 1500 3924 -> 3706 us); CQP_COFETCH=0 for A/B runs
  p.cofetch = h->w_smem ? h->fetch : 1;
  // direct fetch: the W slice lives in registers too where it fits (see run_kernel)
  p.wreg = 0;
  if (p.cofetch == 2 && h->knob_wreg != 0) {
    const int u = ((h->Dpad >> 1) + kComputeThreads - 1) / kComputeThreads;
    const int maxw = h->rb == 4 ? 2 : (h->rb == 8 ? 1 : 0);
    if (u <= maxw) p.wreg = u;
  }
  // with 608 fetching threads the first poll of the resident tier is best issued at once (B200, 1000
  // iterations: D = 900 2456 -> 2358 us, D = 1500 3701 -> 3667 us); the streamed tier keeps the pause
  // (Atlas-sized 5.34 vs 5.55 us per iteration: early polls compete with the W stream)
  if (p.w_smem && p.cofetch && !delay_set) p.poll_delay_ns = 0;
  // Direct fetch: no pause on the fetching side (__nanosleep is no instrument for this: it sleeps 44 / 113 /
  // 241 / 497 / 1005 ns for requests of <= 50 / 100 / 150-200 / 300-400 / 600-1000 ns, tools/nanosleep_bench.cu);
  // the publisher gates the first poll instead (run_kernel).
  if (p.w_smem && p.cofetch == 2 && !delay_set) p.poll_delay_ns = 0;
  p.gate_cycles = h->knob_gate[0]; p.gate_adapt = h->knob_gate[1]; p.gate_up = h->knob_gate[2];
  p.gate_down = h->knob_gate[3]; p.gate_max = h->knob_gate[4];

  p.nparts = h->nparts;
  p.wt_level_pairs = wt_level_pairs(h);
  p.rho_vec = h->rho_vec;
  // (A launch of very few iterations could stream W once instead of copying the slice into shared
  // memory first, at about the same cost -- but the streamed code adds a row's products up in another
  // order, so the bits of fixed_iters(k) would depend on how the iterations are split over launches and
  // the resident server would not reproduce a launch per step.  The order is a property of the handle.)
  switch (h->rb) {
    case 4: return launched(launch_run_rb<4>(h, p));
    case 8: return launched(launch_run_rb<8>(h, p));
    default: return launched(launch_run_rb<16>(h, p));
  }
}

int launch_refresh_z(cqp_handle* h) {
  double* v = h->vq;  // slot 0 holds the iterate between launches
  const int threads = 256, rows_per_block = threads / 32;
  rows_dot_kernel<<<(h->m + rows_per_block - 1) / rows_per_block, threads, 0, h->stream>>>(
      h->Gs, h->m, h->n, h->npad, v, nullptr, 1.0, 0, 1.0, v + h->n);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int launch_warm_start(cqp_handle* h, const double* dy, const double* dlam, int layer_index) {
  CQP_CUDA(cudaMemsetAsync(h->vq, 0, sizeof(double) * (size_t)h->Dpad, h->stream));
  const int cnt = h->n > h->m ? h->n : h->m;
  warm_scale_kernel<<<(cnt + 255) / 256, 256, 0, h->stream>>>(dy, dlam, h->E, h->F, h->cost_scale,
                                                             h->n, h->m, h->vq);
  CQP_CUDA(cudaGetLastError());
  set_state_kernel<<<1, 1, 0, h->stream>>>(h->state, layer_index);
  CQP_CUDA(cudaGetLastError());
  return launch_refresh_z(h);
}

int launch_instantiate(cqp_handle* h, const double* x0_host) {
  const int rows = h->n + h->m, threads = 256, rows_per_block = threads / 32;
  const int blocks = (rows + rows_per_block - 1) / rows_per_block;
  X0Arg xa;
  if (h->mpc_nx <= kMaxInlineX0) {
    std::memcpy(xa.x, x0_host, sizeof(double) * h->mpc_nx);
    instantiate_kernel<true><<<blocks, threads, 0, h->stream>>>(h->mpc_og, h->mpc_oc, h->mpc_cb, h->mpc_db, h->mpc_x0,
                                                               xa, h->n, h->m, h->mpc_nx, h->mpc_nxpad, h->g, h->c,
                                                               h->d);
  } else {
    std::memcpy(h->hx0, x0_host, sizeof(double) * h->mpc_nx);
    CQP_CUDA(cudaMemcpyAsync(h->mpc_x0, h->hx0, sizeof(double) * h->mpc_nx, cudaMemcpyHostToDevice, h->stream));
    instantiate_kernel<false><<<blocks, threads, 0, h->stream>>>(h->mpc_og, h->mpc_oc, h->mpc_cb, h->mpc_db,
                                                                h->mpc_x0, xa, h->n, h->m, h->mpc_nx, h->mpc_nxpad,
                                                                h->g, h->c, h->d);
  }
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int launch_set_state(cqp_handle* h, int layer) {
  set_state_kernel<<<1, 1, 0, h->stream>>>(h->state, layer);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int launch_transpose_pad(cudaStream_t st, const double* src, int rows, int cols, double* dst,
                         int ld, int src_ld) {
  dim3 grid((ld + 31) / 32, (rows + 31) / 32), block(32, 8);
  transpose_pad_kernel<<<grid, block, 0, st>>>(src, rows, cols, dst, ld, src_ld > 0 ? src_ld : rows);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int launch_untranspose(cudaStream_t st, const double* src, int rows, int cols, int ld,
                       double* dst) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  untranspose_kernel<<<grid, block, 0, st>>>(src, rows, cols, ld, dst);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int launch_bias(cqp_handle* h, int k, double* b_out) {
  const int nm = h->n + h->m;
  CQP_CUDA(cudaMemsetAsync(b_out, 0, sizeof(double) * (size_t)h->D, h->stream));
  const int threads = 256, rows_per_block = threads / 32;
  rows_dot_kernel<<<(nm + rows_per_block - 1) / rows_per_block, threads, 0, h->stream>>>(
      h->Dk + (size_t)k * nm * h->npad, nm, h->n, h->npad, h->g, h->E, h->cost_scale, 1, -1.0,
      b_out);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

}  // namespace cqp
