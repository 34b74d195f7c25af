// Batched solve path: B QPs that share (H, G) -- hence the whole W ladder -- and differ in
// (g, c, d): MPC instances at different x0.  Semantically B independent cold-start `solve()`
// calls (/root/reference/proj/src/solver.cpp:158-166 -> run_loop :43-105), one per column.
//
// Design:
//   * The iterates are the columns of S (one column = D contiguous doubles), stored in SLOT order:
//     every QP adapts rho on its own (parity demands it), so the active columns are bucketed by ladder
//     index, every bucket padded to 128 slots, and S is physically compacted into that order at every
//     re-bucketing (batch_permute_kernel: one copy per check round).  A column tile is then a
//     contiguous 2-D box and multiplies ONE W_k: a grouped GEMM.
//   * One persistent launch per check round (round_kernel, cqp_batch_round.cuh) runs all
//     check_interval layers  S <- clamp(W_k S + Bias_k, lo, hi)  of the round: operands staged by TMA
//     (cp.async.bulk.tensor.2d with the hardware 128-byte swizzle, completion on mbarriers, a producer
//     warp), FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA.8x8x4, the only FP64 tensor shape of
//     sm_100a; tcgen05 has no f64 kind), bias folded into the accumulator start, clamp fused into
//     the epilogue, and dataflow dependencies between the iterations of a column tile instead of a
//     launch per iteration.  The per-iteration cp.async kernel below (dmma_gemm_kernel) stays for the
//     plain GEMMs of a check round and the offline stage, and as the A/B reference
//     (CQP_BATCH_LEGACY=1; tests/test_gpu_batch.py::test_round_kernel_matches_per_iteration_kernel).
//   * Every check_interval iterations: unscale, three DMMA GEMMs (H Y, G' Lambda, G Y) on the active
//     columns, a per-column reduction/decision kernel (residuals, rho rule, early exit, finalisation
//     of converged columns), re-bucketing + compaction and the bias GEMM
//     Bias = -[D_k; G D_k] G_s.  Converged columns leave the slot map, so they stop costing work.
//   * No host round trip inside a round; the host only polls a pinned "active columns" word with
//     a lag of two rounds to know when to stop enqueuing and which tile shape the next round gets.
//   * Structured layer: the lambda rows of W, [rho G, -diag(rho), I] (layers.cpp:159-161), only
//     multiply y: their tiles run ceil(n / 16) k-tiles and start from fma(-rho_i, z_i, lambda_i).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "cqp_internal.h"
#include "cqp_device.cuh"

namespace cqp {
namespace {

constexpr int BK = 16, STAGES = 4;
constexpr int SLOT_TILE = 128;  // slot-map granularity: buckets are padded to 128 slots

struct TileDesc {
  int slot0;    // first slot of this 128-slot tile
  int a_index;  // which A matrix (ladder index) the tile multiplies
};

struct GemmParams {
  const double* A;   // [a_index][M_pad][lda] row-major, K contiguous, zero padded
  size_t a_stride;   // doubles between consecutive A matrices (0: one shared A)
  int lda;
  int M;             // valid output rows
  int M_pad;         // padded rows of A (multiple of 128)
  int k_tiles;
  const double* Bm;  // [col][ldb], K contiguous
  int ldb;
  const int* cols;   // slot -> column, or -1 for a padding slot
  const TileDesc* tiles;
  const int* n_tiles;  // device scalar
  double* C;         // [col][ldc]
  int ldc;
  double alpha;
  int mode;          // 0: C = alpha A B ; 1: C = clamp(A B + bias, lo, hi) (one ADMM layer)
  const double* bias;  // [col][ld_bias], rows < nm
  int ld_bias;
  int nm;              // n + m
  int n;
  const double* lo;    // [col][ld_lohi], rows n..nm-1
  const double* hi;
  int ld_lohi;
  // Structured layer (mode 1 only; split == 0: plain dense layer).  The third block row of W is
  // [rho G, -diag(rho), I] (/root/reference/proj/src/layers.cpp:159-161): of its D columns only
  // the first n are dense.  The padded copy of W therefore stores rows 0 .. n+m-1 at padded rows
  // 0 .. split-1 and rows n+m .. D-1 (their first n columns; the rest zeroed) at padded rows
  // split ..; tiles of the second part run k_tiles3 = ceil(n / 16) k-tiles instead of k_tiles and
  // get the two diagonal terms  -rho_i z_i + lambda_i  as the accumulator's start value.
  int split;             // padded row where the lambda block starts (multiple of 128), 0 = dense
  int k_tiles3;
  const double* negrho;  // [a_index][m]: W(n+m+i, n+i) = -rho_i
  // Dynamic scheduling (null: static striding): CTAs take their first item by blockIdx and every
  // further one from this counter (zero at launch).  The next index is fetched while the current
  // item is being computed, so the atomic's latency never shows.
  int* work_ctr;
  // 1: the columns of B and C are addressed by SLOT (the iterate S is stored in slot order, see
  // cqp_batch_round.cuh); bias / bounds stay addressed by column through the slot map
  int slot_major;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int ST = STAGES>
constexpr int gemm_smem_bytes() {
  return ST * (BM + BN) * BK * (int)sizeof(double) + BN * (int)sizeof(int);
}

// C[col][row] = epilogue(A[a_index] (BM x K) . B(cols) (K x BN)) for every (slot tile, sub-tile,
// m-tile) work item; persistent CTAs stride over the items.  WM x WN warps, warp tile
// (BM/WM) x (BN/WN) made of 8x8 DMMA tiles.  Operand tiles are [rows][16] doubles whose
// 16-byte chunks are XOR-swizzled with 2 (row & 3): the 8-byte fragment loads of a half-warp (4
// rows x 4 consecutive k = 2 chunks per row) then hit 8 distinct chunks = all 32 banks (ncu:
// shared-memory load bank conflicts 42 % of wavefronts with the (row & 7) swizzle, 0.4 % with this
// one).  Scheduling is static striding on purpose: a dynamic work counter with a split tail was
// measured 7 % SLOWER (the 3-4 CTAs of an SM share its tensor pipe, so CTA-level quantisation
// is already smoothed at SM level, and half-size tail items re-read A).
// KS > 1 (last rounds, few columns left): KS warp groups share one tile and split the k steps of
// every k-tile among them (group kg takes ks = kg, kg + KS, ...); their partial accumulators meet
// in shared memory after the k loop and group 0 adds them in a fixed order.  With a handful of
// items per SM a tile's K loop is a latency chain (barrier -> LDS -> DMMA per k step); KS groups
// walk it KS k steps at a time.
template <int BM, int BN, int WM, int WN, int MINB, int ST = STAGES, int KS = 1>
__global__ void __launch_bounds__(WM * WN * 32 * KS, MINB) dmma_gemm_kernel(const GemmParams p) {
  constexpr int T = WM * WN * 32 * KS;
  constexpr int TM = BM / WM, TN = BN / WN, MI = TM / 8, NI = TN / 8;
  constexpr int SUB = SLOT_TILE / BN;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + ST * BM * BK;
  int* cols_s = reinterpret_cast<int*>(Bs + ST * BN * BK);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int kg = warp / (WM * WN), warp_in = warp - kg * (WM * WN);  // k-split group, warp within it
  const int warp_m = warp_in % WM, warp_n = warp_in / WM;
  const int m_tiles = p.M_pad / BM;
  const int total = (*p.n_tiles) * SUB * m_tiles;

  // Structured layer: the short lambda-row tiles (k_tiles3 k-tiles) are ordered after all the long
  // ones, so that the static striding hands every CTA a similar mix (longest-first).
  const int m_long = (p.split > 0) ? p.split / BM : m_tiles, m_short = m_tiles - m_long;
  const int total_long = (*p.n_tiles) * SUB * m_long;
  __shared__ int next_item_s;
  for (int item = blockIdx.x; item < total;) {
    int fetched = 0;
    if (tid == 0) fetched = p.work_ctr ? (int)gridDim.x + atomicAdd(p.work_ctr, 1) : item + (int)gridDim.x;
    int ns, mt;
    if (item < total_long) {
      ns = item / m_long;
      mt = item - ns * m_long;
    } else {
      const int j = item - total_long;
      ns = j / m_short;
      mt = m_long + (j - ns * m_short);
    }
    const int nt = ns / SUB, sub = ns - nt * SUB;
    const TileDesc td = p.tiles[nt];
    const int slot0 = td.slot0 + sub * BN;
    const int m0 = mt * BM;
    // padded row m0 -> actual row; valid rows of this part end at row_end; k-tiles of this part
    const bool blk3 = p.split > 0 && m0 >= p.split;
    const int row0 = blk3 ? m0 - p.split + p.nm : m0;
    const int row_end = (p.split > 0 && !blk3) ? p.nm : p.M;
    const int k_tiles = blk3 ? p.k_tiles3 : p.k_tiles;
    // (padding slots sit at the end of a bucket: a sub-tile whose first slot is empty is empty)
    if (row0 < row_end && p.cols[slot0] >= 0) {
    const double* A = p.A + (size_t)td.a_index * p.a_stride + (size_t)m0 * p.lda;
    if (tid < BN) cols_s[tid] = p.cols[slot0 + tid];
    __syncthreads();

    // per-thread copy plan, invariant over k: chunk ch = tid + i T -> tile row r = ch >> 3, 16-byte
    // chunk c = ch & 7 of the row's 16 doubles (hoisted out of the k loop: the column lookup and
    // the address arithmetic were 8 % of the issue slots)
    constexpr int ACH = (BM * 8 + T - 1) / T, BCH = (BN * 8 + T - 1) / T;
    const double* asrc[ACH];
    int adst[ACH];
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int ch = tid + i * T, r = ch >> 3, c = ch & 7;
      asrc[i] = A + (size_t)r * p.lda + c * 2;
      adst[i] = r * BK + ((c ^ ((r & 3) << 1)) << 1);
    }
    const double* bsrc[BCH];
    int bdst[BCH], bbytes[BCH];
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int ch = tid + i * T, r = ch >> 3, c = ch & 7;
      const int col = (ch < BN * 8) ? cols_s[r] : -1;
      bsrc[i] = p.Bm + (size_t)(col < 0 ? 0 : (p.slot_major ? slot0 + r : col)) * p.ldb + c * 2;
      bdst[i] = r * BK + ((c ^ ((r & 3) << 1)) << 1);
      bbytes[i] = col < 0 ? 0 : 16;
    }
    auto issue = [&](int kt, int stage) {
      const int k0 = kt * BK;
      double* as = As + stage * BM * BK;
      double* bs = Bs + stage * BN * BK;
#pragma unroll
      for (int i = 0; i < ACH; ++i)
        if ((BM * 8) % T == 0 || tid + i * T < BM * 8) cp_async16(as + adst[i], asrc[i] + k0, 16);
#pragma unroll
      for (int i = 0; i < BCH; ++i)
        if ((BN * 8) % T == 0 || tid + i * T < BN * 8) cp_async16(bs + bdst[i], bsrc[i] + k0, bbytes[i]);
    };

#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < k_tiles) issue(s, s);
      cp_async_commit();
    }
    // Accumulators start from the bias (mode 1: v = bias + W s; alpha is 1 there), so its global
    // loads overlap the pipeline fill instead of serialising the epilogue.  The clamp bounds of
    // this thread's elements are prefetched into L1 for the same reason (they are read-only for
    // the whole solve; only rows of the z block have any).
    double acc[MI][NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = cols_s[warp_n * TN + ni * 8 + 2 * t4 + j];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int row = row0 + warp_m * TM + mi * 8 + g;
          double init = 0.0;
          if (p.mode == 1 && col >= 0 && kg == 0) {
            if (row < p.nm) {
              init = p.bias[(size_t)col * p.ld_bias + row];
              if (row >= p.n && g == 0) {  // one prefetch per 64-byte run of 8 rows
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p.lo + (size_t)col * p.ld_lohi + row - p.n));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p.hi + (size_t)col * p.ld_lohi + row - p.n));
              }
            } else if (blk3 && row < p.M) {  // lambda row i: the diagonal blocks (3,2) = -rho, (3,3) = I
              const double* v = p.Bm + (size_t)(p.slot_major ? slot0 + warp_n * TN + ni * 8 + 2 * t4 + j : col) * p.ldb;
              const int i = row - p.nm;
              init = fma(p.negrho[(size_t)td.a_index * (p.M - p.nm) + i], v[p.n + i], v[row]);
            }
          }
          acc[mi][ni][j] = init;
        }
      }
    }
    for (int kt = 0; kt < k_tiles; ++kt) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      const int next = kt + ST - 1;
      if (next < k_tiles) issue(next, next % ST);
      cp_async_commit();
      const double* as = As + (kt % ST) * BM * BK + (warp_m * TM) * BK;
      const double* bs = Bs + (kt % ST) * BN * BK + (warp_n * TN) * BK;
#pragma unroll
      for (int ks0 = 0; ks0 < BK / 4; ks0 += KS) {
        const int ks = ks0 + kg;
        const int e = ks * 4 + t4;
        const int off = (((e >> 1) ^ ((g & 3) << 1)) << 1) | (e & 1);  // rows are 8-aligned + g, so r & 7 == g
        double a[MI], b[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) a[mi] = as[(mi * 8 + g) * BK + off];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) b[ni] = bs[(ni * 8 + g) * BK + off];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
    cp_async_wait<0>();
    if (KS > 1) {
      // partial accumulators of groups 1 .. KS-1 -> shared memory (the stage buffers are free now),
      // group 0 adds them in group order and runs the epilogue alone
      __syncthreads();
      double* red = As;  // [KS - 1][WM * WN * 32][MI * NI * 2]
      constexpr int PER = MI * NI * 2;
      if (kg > 0) {
        double* mine = red + ((size_t)(kg - 1) * (WM * WN * 32) + warp_in * 32 + lane) * PER;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            mine[(mi * NI + ni) * 2] = acc[mi][ni][0];
            mine[(mi * NI + ni) * 2 + 1] = acc[mi][ni][1];
          }
      }
      __syncthreads();
      if (kg == 0) {
#pragma unroll
      for (int q = 1; q < KS; ++q) {
        const double* theirs = red + ((size_t)(q - 1) * (WM * WN * 32) + warp_in * 32 + lane) * PER;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            acc[mi][ni][0] += theirs[(mi * NI + ni) * 2];
            acc[mi][ni][1] += theirs[(mi * NI + ni) * 2 + 1];
          }
      }
      }
    }

    // epilogue: C fragment (row = g, cols 2*t4, 2*t4+1) of each 8x8 sub-tile
    if (KS == 1 || kg == 0) {
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = cols_s[warp_n * TN + ni * 8 + 2 * t4 + j];
        if (col < 0) continue;
        double* crow = p.C + (size_t)(p.slot_major ? slot0 + warp_n * TN + ni * 8 + 2 * t4 + j : col) * p.ldc;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int row = row0 + warp_m * TM + mi * 8 + g;
          if (row >= row_end) continue;
          double v = acc[mi][ni][j];
          if (p.mode != 1) v *= p.alpha;
          if (p.mode == 1 && row < p.nm) {
            if (row >= p.n) {
              const double lo = p.lo[(size_t)col * p.ld_lohi + row - p.n];
              const double hi = p.hi[(size_t)col * p.ld_lohi + row - p.n];
              v = v < lo ? lo : v;
              v = v > hi ? hi : v;
            }
          }
          crow[row] = v;
        }
      }
    }
    }
    }  // item not empty
    __syncthreads();  // this item's readers of cols_s / the stage buffers are done
    if (tid == 0) next_item_s = fetched;
    __syncthreads();
    item = next_item_s;
  }
}

#include "cqp_batch_round.cuh"

// dst[a][r][c] (rows_pad x ld_dst, zero padded) <- src[a][r][c] (rows x ld_src, first `cols`)
__global__ void repad_kernel(const double* __restrict__ src, int rows, int cols, int ld_src,
                             size_t src_stride, double* __restrict__ dst, int rows_pad, int ld_dst,
                             size_t dst_stride, int count) {
  const size_t per = (size_t)rows_pad * ld_dst;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= per * count) return;
  const int a = (int)(idx / per);
  const size_t rem = idx - (size_t)a * per;
  const int r = (int)(rem / ld_dst), c = (int)(rem % ld_dst);
  dst[(size_t)a * dst_stride + rem] =
      (r < rows && c < cols) ? src[(size_t)a * src_stride + (size_t)r * ld_src + c] : 0.0;
}

// negrho[a][i] = W_a(n+m+i, n+i) = -rho_i: the diagonal of block (3,2) (layers.cpp:160)
__global__ void extract_negrho_kernel(const double* __restrict__ W, int ld, size_t stride, int n, int m,
                                      double* __restrict__ negrho, int count) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * count) return;
  const int a = idx / m, i = idx - a * m;
  negrho[idx] = W[(size_t)a * stride + (size_t)(n + m + i) * ld + n + i];
}

struct BatchDev {
  int n, m, D, B;
  int ld_s;    // leading dimension of S columns (D padded to BK)
  int ld_n;    // n padded to BK
  int ld_m;    // m padded to BK
  int ld_nm;   // n + m padded to even
  const double* E;
  const double* F;
  double cost_scale;
  const double* grid;
  const double* log_grid;
  int L;
  // per-column inputs
  const double* g;   // [B][n] unscaled
  const double* c;   // [B][m]
  const double* d;   // [B][m]
  double* gs;        // [B][ld_n] scaled g
  double* lo;        // [B][ld_m] scaled bounds
  double* hi;
  // unscaled iterate + products
  double* uy;        // [B][ld_n]
  double* ul;        // [B][ld_m]
  double* uz;        // [B][ld_m]
  double* hy;        // [B][ld_n]
  double* gtl;       // [B][ld_n]
  double* gy;        // [B][ld_m]
  // per-column state
  int* layer;
  int* active;
  int* iters;
  int* status;
  int* nsw;
  double* rp;
  double* rd;
  // per-column records (problem.hpp:57-60, solver.hpp:56-61): rho_trace and residual_history
  cqp_rho_switch* trace;       // [B][rec_cap]; entry 0 = {0, start index} (solver.cpp:50)
  cqp_residual_sample* hist;   // [B][rec_cap]
  int* nhist;
  int rec_cap;
  // outputs
  double* out_y;     // [B][n]
  double* out_z;     // [B][m]
  double* out_l;     // [B][m]
  // slot map
  int* cols;         // [slot_cap]
  TileDesc* tiles;   // [tile_cap]
  int* n_tiles;
  int* n_active;
  int* slot_of;      // [B] column -> slot of its iterate in S (slot order)
  // compact lists of the NON-EMPTY column tiles of 64 ([0]) and 32 ([1]) slots: {first slot, ladder
  // index}; the round kernel enumerates these, so padding costs it nothing
  TileDesc* ct[2];
  int* n_ct;         // [2]
  // second slot map: only the columns whose bias rows are stale (first round: all; later: the columns
  // that switched their ladder level at the last check) -- the bias GEMM runs on this one
  int* bias_dirty;   // [B]
  int* cols2;
  TileDesc* tiles2;
  int* n_tiles2;
  // settings
  double eps_prim, eps_dual, threshold;
  int adaptive, max_iters;
};

// gs = cost_scale * E o g ; lo = F o c ; hi = F o d   (layers.cpp:181-183), per column
__global__ void batch_prepare_kernel(BatchDev b, int initial_index) {
  const int col = blockIdx.x;
  for (int i = threadIdx.x; i < b.ld_n; i += blockDim.x)
    b.gs[(size_t)col * b.ld_n + i] = (i < b.n) ? b.cost_scale * (b.E[i] * b.g[(size_t)col * b.n + i]) : 0.0;
  for (int i = threadIdx.x; i < b.ld_m; i += blockDim.x) {
    const bool in = i < b.m;
    b.lo[(size_t)col * b.ld_m + i] = in ? b.F[i] * b.c[(size_t)col * b.m + i] : 0.0;
    b.hi[(size_t)col * b.ld_m + i] = in ? b.F[i] * b.d[(size_t)col * b.m + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    b.layer[col] = initial_index;
    b.active[col] = 1;
    b.iters[col] = 0;
    b.status[col] = CQP_INVALID;
    b.nsw[col] = 0;
    b.rp[col] = 0.0;
    b.rd[col] = 0.0;
    b.nhist[col] = 0;
    b.bias_dirty[col] = 1;
    b.trace[(size_t)col * b.rec_cap] = {0, initial_index};  // every call's trace starts here (solver.cpp:50)
  }
}

// unscale the active columns (layers.hpp:57-59): y = E o y_s, z = z_s / F, lambda = F o l_s / cs
__global__ void batch_unscale_kernel(BatchDev b, const double* __restrict__ S) {
  const int col = blockIdx.x;
  if (!b.active[col]) return;
  const double* v = S + (size_t)b.slot_of[col] * b.ld_s;
  for (int i = threadIdx.x; i < b.ld_n; i += blockDim.x)
    b.uy[(size_t)col * b.ld_n + i] = (i < b.n) ? b.E[i] * v[i] : 0.0;
  for (int i = threadIdx.x; i < b.ld_m; i += blockDim.x) {
    double z = 0.0, l = 0.0;
    if (i < b.m) {
      z = v[b.n + i] / b.F[i];
      l = (b.F[i] * v[b.n + b.m + i]) / b.cost_scale;
    }
    b.uz[(size_t)col * b.ld_m + i] = z;
    b.ul[(size_t)col * b.ld_m + i] = l;
  }
}

__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, w));
  return v;
}

// One warp per column: residuals (solver.cpp:119-124), rho rule (:126-142), early exit (:84-87)
// and, for columns that stop, the epilogue (:90-99).  `it` = iterations done so far;
// `check` = 0 for the trailing partial round (no check happens at i % check_interval != 0).
__global__ void batch_decide_kernel(BatchDev b, int it, int check, int early_exit) {
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= b.B || !b.active[col]) return;
  const int n = b.n, m = b.m;
  const double* hy = b.hy + (size_t)col * b.ld_n;
  const double* gtl = b.gtl + (size_t)col * b.ld_n;
  const double* gy = b.gy + (size_t)col * b.ld_m;
  const double* uz = b.uz + (size_t)col * b.ld_m;
  const double* g = b.g + (size_t)col * n;
  const double* c = b.c + (size_t)col * m;
  const double* d = b.d + (size_t)col * m;
  double r_dual = 0.0, n_hy = 0.0, n_gtl = 0.0, n_g = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double a = hy[i], bb = gtl[i], gi = g[i];
    r_dual = nanmax(r_dual, fabs((a + gi) + bb));
    n_hy = nanmax(n_hy, fabs(a));
    n_gtl = nanmax(n_gtl, fabs(bb));
    n_g = nanmax(n_g, fabs(gi));
  }
  double r_prim = 0.0, r_prim_final = 0.0, n_gy = 0.0, n_z = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double a = gy[i], z = uz[i];
    double zc = z < c[i] ? c[i] : z;  // solver.cpp:94 clamp in original units
    zc = zc > d[i] ? d[i] : zc;
    r_prim = nanmax(r_prim, fabs(a - z));
    r_prim_final = nanmax(r_prim_final, fabs(a - zc));
    n_gy = nanmax(n_gy, fabs(a));
    n_z = nanmax(n_z, fabs(z));
  }
  r_dual = warp_nanmax(r_dual); n_hy = warp_nanmax(n_hy); n_gtl = warp_nanmax(n_gtl);
  n_g = warp_nanmax(n_g); r_prim = warp_nanmax(r_prim); r_prim_final = warp_nanmax(r_prim_final);
  n_gy = warp_nanmax(n_gy); n_z = warp_nanmax(n_z);

  int layer = b.layer[col];
  bool converged = false;
  if (check) {
    if (lane == 0) {  // residual_history sample: the index BEFORE this check's switch (solver.cpp:71)
      const int k = b.nhist[col];
      if (k < b.rec_cap) b.hist[(size_t)col * b.rec_cap + k] = {it, r_prim, r_dual, layer};
      b.nhist[col] = k + 1;
    }
    if (b.adaptive) {
      const double rho_cur = b.grid[layer];
      double rho_nom = rho_cur;
      if (!(r_prim == 0.0 || r_dual == 0.0)) {
        double num = n_hy < n_gtl ? n_gtl : n_hy;
        num = num < n_g ? n_g : num;
        num = num < 1e-4 ? 1e-4 : num;
        double den = n_gy < n_z ? n_z : n_gy;
        den = den < 1e-4 ? 1e-4 : den;
        rho_nom = rho_cur * sqrt((r_prim * num) / (r_dual * den));
      }
      const double target = log10(rho_nom);
      int best = 0;
      double best_dist = INFINITY;
      for (int k = 0; k < b.L; ++k) {
        const double dist = fabs(b.log_grid[k] - target);
        if (dist < best_dist - 1e-15) { best = k; best_dist = dist; }
      }
      const double ra = rho_nom / rho_cur, rb = rho_cur / rho_nom;
      const double ratio = ra < rb ? rb : ra;
      const int cand = ratio >= b.threshold ? best : layer;
      if (cand != layer) {
        layer = cand;
        if (lane == 0) {
          const int k = b.nsw[col] + 1;  // (entry 0 is the start index)
          if (k < b.rec_cap) b.trace[(size_t)col * b.rec_cap + k] = {it, cand};
          b.layer[col] = cand;
          b.nsw[col] = k;
          b.bias_dirty[col] = 1;  // Bias = -[D_k; G D_k] g_s follows the level (layers.cpp:168-175)
        }
      }
    }
    converged = early_exit && r_prim <= b.eps_prim && r_dual <= b.eps_dual;
  }
  if (converged || it >= b.max_iters) {
    const double* uy = b.uy + (size_t)col * b.ld_n;
    const double* ul = b.ul + (size_t)col * b.ld_m;
    for (int i = lane; i < n; i += 32) b.out_y[(size_t)col * n + i] = uy[i];
    for (int i = lane; i < m; i += 32) {
      double zc = uz[i] < c[i] ? c[i] : uz[i];
      zc = zc > d[i] ? d[i] : zc;
      b.out_z[(size_t)col * m + i] = zc;
      b.out_l[(size_t)col * m + i] = ul[i];
    }
    if (lane == 0) {
      b.status[col] = (converged || (r_prim_final <= b.eps_prim && r_dual <= b.eps_dual)) ? CQP_SOLVED : CQP_MAX_ITERS;
      b.iters[col] = it;
      b.rp[col] = r_prim_final;
      b.rd[col] = r_dual;
      b.active[col] = 0;
    }
  }
}

// Rebuild the slot map: active columns bucketed by ladder index, every bucket padded to a
// multiple of 128 with -1 slots, one TileDesc per 128 slots.  Single CTA, deterministic (stable
// in the column index).
// Fast path (L <= 16, the default ladder has 13 levels): a counting sort in one pass.  Thread t owns
// the contiguous columns [t cpt, (t + 1) cpt); per-thread per-level counts, one exclusive scan per
// level over the threads, then every thread scatters its columns in order (stable in the column
// index, hence deterministic).  Builds both maps (all active columns / the bias-stale ones).
constexpr int kRegroupThreads = 256, kRegroupMaxL = 16;
__global__ void __launch_bounds__(kRegroupThreads) batch_regroup_fast_kernel(BatchDev b) {
  __shared__ int cnt[2][kRegroupMaxL][kRegroupThreads];
  __shared__ int tot[2][kRegroupMaxL], base[2][kRegroupMaxL], ntile[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cpt = (b.B + kRegroupThreads - 1) / kRegroupThreads;
  const int c0 = tid * cpt, c1 = min(b.B, c0 + cpt);
  for (int k = 0; k < b.L; ++k) { cnt[0][k][tid] = 0; cnt[1][k][tid] = 0; }
  for (int col = c0; col < c1; ++col) {
    if (!b.active[col]) continue;
    const int k = b.layer[col];
    cnt[0][k][tid] += 1;
    if (b.bias_dirty[col]) cnt[1][k][tid] += 1;
  }
  __syncthreads();
  // exclusive scan over the threads, one (map, level) row per warp at a time
  for (int row = warp; row < 2 * b.L; row += kRegroupThreads / 32) {
    int* v = cnt[row / b.L][row % b.L];
    int carry = 0;
    for (int i0 = 0; i0 < kRegroupThreads; i0 += 32) {
      const int x = v[i0 + lane];
      int incl = x;
#pragma unroll
      for (int w = 1; w < 32; w <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, w);
        if (lane >= w) incl += y;
      }
      v[i0 + lane] = carry + incl - x;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tot[row / b.L][row % b.L] = carry;
  }
  __syncthreads();
  if (tid < 2) {  // bucket bases (every bucket padded to 128 slots) and tile counts of the two maps
    int slot = 0, tiles = 0;
    for (int k = 0; k < b.L; ++k) {
      base[tid][k] = slot;
      const int padded = (tot[tid][k] + SLOT_TILE - 1) / SLOT_TILE * SLOT_TILE;
      slot += padded;
      tiles += padded / SLOT_TILE;
    }
    ntile[tid] = tiles;
  }
  __syncthreads();
  for (int col = c0; col < c1; ++col) {
    if (!b.active[col]) continue;
    const int k = b.layer[col];
    b.cols[base[0][k] + cnt[0][k][tid]++] = col;
    if (b.bias_dirty[col]) {
      b.cols2[base[1][k] + cnt[1][k][tid]++] = col;
      b.bias_dirty[col] = 0;
    }
  }
  for (int map = 0; map < 2; ++map) {
    int* cols = map ? b.cols2 : b.cols;
    TileDesc* tiles = map ? b.tiles2 : b.tiles;
    int t0 = 0;
    for (int k = 0; k < b.L; ++k) {
      const int count = tot[map][k], padded = (count + SLOT_TILE - 1) / SLOT_TILE * SLOT_TILE;
      for (int i = count + tid; i < padded; i += kRegroupThreads) cols[base[map][k] + i] = -1;
      for (int t = tid; t < padded / SLOT_TILE; t += kRegroupThreads) tiles[t0 + t] = {base[map][k] + t * SLOT_TILE, k};
      t0 += padded / SLOT_TILE;
    }
  }
  if (tid == 0) {
    int total = 0;
    for (int k = 0; k < b.L; ++k) total += tot[0][k];
    *b.n_tiles = ntile[0];
    *b.n_tiles2 = ntile[1];
    *b.n_active = total;
  }
  __syncthreads();
  // non-empty column tiles of the full map (padding slots sit at the end of a bucket: a tile whose first
  // slot is empty is empty); one warp per granularity, in slot order
  if (warp < 2) {
    const int n_tiles = ntile[0];
    const int bn = warp == 0 ? 64 : 32, sub = SLOT_TILE / bn;
    int count = 0;
    for (int k0 = 0; k0 < n_tiles * sub; k0 += 32) {
      const int k = k0 + lane;
      bool keep = false;
      TileDesc td{0, 0};
      if (k < n_tiles * sub) {
        // (tile k / sub: recompute instead of re-reading b.tiles, which other threads just wrote)
        int t = k / sub, lvl = 0, tb = 0;
        for (; lvl < b.L; ++lvl) {
          const int nt = (tot[0][lvl] + SLOT_TILE - 1) / SLOT_TILE;
          if (t < tb + nt) break;
          tb += nt;
        }
        td.slot0 = base[0][lvl] + (t - tb) * SLOT_TILE + (k % sub) * bn;
        td.a_index = lvl;
        keep = (td.slot0 - base[0][lvl]) < tot[0][lvl];
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, keep);
      if (keep) b.ct[warp][count + __popc(ballot & ((1u << lane) - 1))] = td;
      count += __popc(ballot);
    }
    if (lane == 0) b.n_ct[warp] = count;
  }
}

// General path (any L): one compaction pass per ladder level.  Builds the full map only; the bias map
// aliases it (every active column gets its bias rows recomputed).
__global__ void batch_regroup_kernel(BatchDev b) {
  __shared__ int warp_sums[32];
  __shared__ int base_s, slot_base_s, total_active_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (tid == 0) { slot_base_s = 0; total_active_s = 0; }
  __syncthreads();
  int n_tiles = 0;
  for (int k = 0; k < b.L; ++k) {
    if (tid == 0) base_s = 0;
    __syncthreads();
    for (int start = 0; start < b.B; start += blockDim.x) {
      const int col = start + tid;
      const int flag = (col < b.B && b.active[col] && b.layer[col] == k) ? 1 : 0;
      const unsigned ballot = __ballot_sync(0xffffffffu, flag);
      const int in_warp = __popc(ballot & ((1u << lane) - 1));
      if (lane == 0) warp_sums[warp] = __popc(ballot);
      __syncthreads();
      int warp_off = 0, chunk_total = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int s = warp_sums[w];
        if (w < warp) warp_off += s;
        chunk_total += s;
      }
      if (flag) b.cols[slot_base_s + base_s + warp_off + in_warp] = col;
      __syncthreads();
      if (tid == 0) base_s += chunk_total;
      __syncthreads();
    }
    const int count = base_s;
    const int padded = (count + SLOT_TILE - 1) / SLOT_TILE * SLOT_TILE;
    for (int i = count + tid; i < padded; i += blockDim.x) b.cols[slot_base_s + i] = -1;
    for (int t = tid; t < padded / SLOT_TILE; t += blockDim.x) {
      b.tiles[n_tiles + t].slot0 = slot_base_s + t * SLOT_TILE;
      b.tiles[n_tiles + t].a_index = k;
    }
    n_tiles += padded / SLOT_TILE;
    __syncthreads();
    if (tid == 0) { slot_base_s += padded; total_active_s += count; }
    __syncthreads();
  }
  if (tid == 0) { *b.n_tiles = n_tiles; *b.n_active = total_active_s; }
  __syncthreads();
  // non-empty column tiles (padding slots sit at the end of a bucket: a tile whose first slot is empty
  // is empty); one warp per granularity, in slot order
  if (warp < 2) {
    const int bn = warp == 0 ? 64 : 32, sub = SLOT_TILE / bn;
    int count = 0;
    for (int base = 0; base < n_tiles * sub; base += 32) {
      const int k = base + lane;
      bool keep = false;
      TileDesc td{0, 0};
      if (k < n_tiles * sub) {
        const TileDesc t128 = b.tiles[k / sub];
        td.slot0 = t128.slot0 + (k % sub) * bn;
        td.a_index = t128.a_index;
        keep = b.cols[td.slot0] >= 0;
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, keep);
      if (keep) b.ct[warp][count + __popc(ballot & ((1u << lane) - 1))] = td;
      count += __popc(ballot);
    }
    if (lane == 0) b.n_ct[warp] = count;
  }
}

// Physical compaction of the iterate after a re-bucketing: slot s of `dst` <- the column the new
// slot map puts there (from its old slot in `src`), zeros for a padding slot; then slot_of[col] = s.
// One CTA per slot of the new map.
__global__ void batch_permute_kernel(BatchDev b, const double* __restrict__ src, double* __restrict__ dst) {
  const int s = blockIdx.x;
  if (s >= (*b.n_tiles) * SLOT_TILE) return;
  const int col = b.cols[s];
  __shared__ int old_s;
  if (threadIdx.x == 0) old_s = col >= 0 ? b.slot_of[col] : 0;
  __syncthreads();
  const double2* from = reinterpret_cast<const double2*>(src + (size_t)old_s * b.ld_s);
  double2* to = reinterpret_cast<double2*>(dst + (size_t)s * b.ld_s);
  for (int i = threadIdx.x; i < (b.ld_s >> 1); i += blockDim.x) to[i] = col >= 0 ? from[i] : make_double2(0.0, 0.0);
  if (threadIdx.x == 0 && col >= 0) b.slot_of[col] = s;
}

// Debug (CQP_ROUND_VERIFY=1): first entry where the round kernel's iterate differs from the
// legacy kernel's, over the slots of the current map.  out[0] = min linear index (slot * ld + row).
// Padding slots are not compared: their columns belong to no QP (whatever a departed column left there is
// multiplied along by the per-iteration kernel and zeroed group-wise by the round kernel).
__global__ void batch_compare_kernel(const double* __restrict__ a, const double* __restrict__ b, const int* n_tiles,
                                     const int* __restrict__ cols, int ld, int D, unsigned long long* out) {
  const int s = blockIdx.x;
  if (s >= (*n_tiles) * SLOT_TILE || cols[s] < 0) return;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const double x = a[(size_t)s * ld + i], y = b[(size_t)s * ld + i];
    if (__double_as_longlong(x) != __double_as_longlong(y)) {
      atomicMin(out, (unsigned long long)s * ld + i);
      atomicAdd(out + 1, 1ull);
    }
  }
}

}  // namespace
}  // namespace cqp

using namespace cqp;

struct cqp_batch {
  cqp_handle* h = nullptr;
  int capacity = 0;
  int n = 0, m = 0, D = 0, L = 0;
  int ld_s = 0, ld_n = 0, ld_m = 0, ld_nm = 0;
  int Dm_pad = 0, nm_mpad = 0, n_mpad = 0, m_mpad = 0;
  // Structured layer: the lambda rows of W only multiply y (see GemmParams::split).  Default on;
  // CQP_BATCH_DENSE=1 keeps the plain dense layer for A/B runs.
  int split = 0;
  double* negrho = nullptr;
  // one work counter per GEMM launch of a solve (dynamic scheduling), zeroed when the solve starts.
  // OPT-IN (CQP_BATCH_DYNAMIC=1): measured slower than static striding on B200 (B = 4096, same
  // box: 304.9 vs 288.5 ms per solve), as was an earlier variant with a split tail.
  int* work_ctrs = nullptr;
  int work_ctr_cap = 0, work_ctr_next = 0;
  int dynamic = 0;
  int grid_ctas[16] = {};  // persistent grid per tile configuration
  // active-column thresholds (see pick_config), calibrated on B200 at D = 1500 (profiles/,
  // CQP_BATCH_THRESHOLDS sweeps): 64x64 tiles with 3 CTAs/SM beat 128x128 at every batch size
  // (less wave quantisation, 12 warps/SM), 64x32 wins below ~3400 columns, 32x32 (6 CTAs/SM: more
  // warps to keep the tensor pipe fed when the grid no longer fills) below ~1400.
  int thr_big = 1 << 30, thr_mid = 3400, thr_small = 800;
  int force_cfg = -1;
  std::vector<std::pair<int, int>> plan;  // CQP_BATCH_PLAN="cfg:min_active,...": first entry whose bound the active count reaches
  int small_cfg = 3;  // 32x32 tiles
  // below thr_tiny columns: 32x32 tiles with 4 k-split warp groups (cfg 4; cfg 5 has 2).  Measured
  // (B200, D = 1500): a round of <= 58 columns takes 0.62 instead of 0.72 ms; between 100 and 300
  // columns the split is slower (the groups share the 4 DMMA pipes of their SM), so it stops at 64.
  int tiny_cfg = 4, thr_tiny = 64;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evc0 = nullptr, evc1 = nullptr;
  float last_total_ms = 0.f, last_compute_ms = 0.f;
  long long last_launches = 0;
  std::vector<cudaEvent_t> round_events, it0, it1;  // it0/it1: around each round's iteration GEMMs
  double last_gemm_ms = 0.0, last_gemm_flops = 0.0;
  int last_rounds = 0;
  std::vector<float> round_ms;
  std::vector<int> round_active;
  // shared matrices re-padded for the GEMM tiles
  double *Wb = nullptr, *DGb = nullptr, *Hb = nullptr, *Gb = nullptr, *Gtb = nullptr;
  // per-column buffers
  double *S0 = nullptr, *S1 = nullptr, *bias = nullptr;
  double *g = nullptr, *c = nullptr, *d = nullptr, *gs = nullptr, *lo = nullptr, *hi = nullptr;
  double *uy = nullptr, *ul = nullptr, *uz = nullptr, *hy = nullptr, *gtl = nullptr, *gy = nullptr;
  int *layer = nullptr, *active = nullptr, *iters = nullptr, *status = nullptr, *nsw = nullptr;
  double *rp = nullptr, *rd = nullptr, *out_y = nullptr, *out_z = nullptr, *out_l = nullptr;
  cqp_rho_switch* trace = nullptr;       // [capacity][rec_cap]
  cqp_residual_sample* hist = nullptr;   // [capacity][rec_cap]
  int* nhist = nullptr;
  int rec_cap = 0;
  int last_B = 0;                        // columns of the last solve (single lane)
  std::vector<int> lane_off, lane_cnt;   // parent: column range every lane solved last
  int* cols = nullptr;
  TileDesc* tiles = nullptr;
  int *n_tiles = nullptr, *n_active = nullptr;
  int* slot_of = nullptr;   // [capacity] column -> slot of its iterate (S0 / S1 are in slot order)
  TileDesc* ct[2] = {nullptr, nullptr};  // non-empty column tiles of 64 / 32 slots (BatchDev::ct)
  int* n_ct = nullptr;
  int* bias_dirty = nullptr;             // second slot map: the bias-stale columns (BatchDev::cols2)
  int* cols2 = nullptr;
  TileDesc* tiles2 = nullptr;
  int* n_tiles2 = nullptr;
  int slot_cap = 0;         // slots of S0 / S1
  // round kernel (cqp_batch_round.cuh): TMA descriptors of W (box rows 64 / 32) and of the two iterate
  // buffers, the per-round counters {work, done[column tiles]}.  CQP_BATCH_LEGACY=1 keeps the
  // one-launch-per-iteration cp.async kernel on the same slot-ordered iterate (A/B runs).
  CUtensorMap mapA[2], mapS[2][2];  // [box: 0 = 64 rows, 1 = 32 rows], mapS[buffer][box]
  int* round_ctrs = nullptr;
  double* kx_part = nullptr;  // partial tiles of the K split over CTAs (RoundParams::part)
  int kx_cnt_off = 0;         // offset of its arrival counters inside round_ctrs
  // rounds with at most kx_thr active columns split every tile's K loop over kx CTAs (CQP_BATCH_KX=kx,thr)
  int kx = 4, kx_thr = 350;
  // ... and over kx_few CTAs once at most kx_few_thr columns are left (the last rounds are one latency chain per
  // iteration: the shorter every CTA's share of the K loop, the shorter the chain)
  int kx_few = 6, kx_few_thr = 64;
  CUtensorMap* gmaps = nullptr;   // device copies: [box a][3] ... see round_run
  int round_flags = 0;
  int round_ctr_count = 0;
  int round_grid[16] = {};
  int legacy = 0;
  int verify = 0;                       // CQP_ROUND_VERIFY: run both kernels every round and compare
  double* T[2] = {nullptr, nullptr};    // verify: the legacy kernel's copy of the iterate
  unsigned long long* vres = nullptr;   // verify: {first mismatch index, count}
  int* h_active = nullptr;  // pinned, one word per round
  int h_active_cap = 0;
  // Lanes: a large batch is cut into independent sub-batches that run concurrently on their own
  // streams (one host thread each enqueues its rounds).  Columns are independent QPs, so nothing
  // is exchanged; the wave tail of one lane's GEMM launch is filled by the other lane's launches
  // (B200, 4096 columns, same box: 288.3 ms per solve with one lane, 259.5 with two, 273 with
  // three).  A parent object owns the lanes and no buffers of its own.  Counts, traces and
  // statuses do not depend on the split; values agree to rounding (a round's tile shape / k-split
  // follows the lane's active-column count).
  std::vector<cqp_batch*> lanes;
  cudaEvent_t ev_start = nullptr;  // parent: recorded before any lane starts; every lane's stream waits on it
};

namespace {

template <typename T>
int balloc(T** p, size_t count) {
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (count ? count : 1)));
  CQP_CUDA(cudaMemset(*p, 0, sizeof(T) * (count ? count : 1)));
  CQP_CUDA(cudaStreamSynchronize(0));  // legacy-stream memset vs the batch's non-blocking stream
  return CQP_OK;
}

int round_up_i(int x, int q) { return (x + q - 1) / q * q; }

// Tile configurations: 0: 128x128 (8 warps), 1: 64x64 (4 warps), 2: 64x32 (4 warps),
// 3: 32x32 (4 warps).  Smaller tiles keep the SMs busy when few columns are still active.
using GemmKernel = void (*)(const GemmParams);
struct GemmConfig {
  GemmKernel fn;
  int threads;
  int smem;
};
constexpr int kNumConfigs = 10;
constexpr int kKxMaxTiles = 16;  // column tiles a round may have for its K loops to be split over CTAs
constexpr int kKxMaxSplit = 8;  // CTAs one tile's K loop may be split over
static_assert(kNumConfigs <= 16, "grid_ctas / round_grid hold 16 configurations");
const GemmConfig kConfigs[kNumConfigs] = {
    {dmma_gemm_kernel<128, 128, 2, 4, 1>, 256, gemm_smem_bytes<128, 128>()},
    {dmma_gemm_kernel<64, 64, 2, 2, 3>, 128, gemm_smem_bytes<64, 64>()},
    {dmma_gemm_kernel<64, 32, 2, 2, 4>, 128, gemm_smem_bytes<64, 32>()},
    {dmma_gemm_kernel<32, 32, 2, 2, 6>, 128, gemm_smem_bytes<32, 32>()},
    // deeper pipelines for the latency-bound last rounds (CQP_BATCH_FORCE_CFG / thresholds)
    {dmma_gemm_kernel<32, 32, 2, 2, 2, STAGES, 4>, 512, gemm_smem_bytes<32, 32>()},   // 4 k-split groups
    {dmma_gemm_kernel<32, 32, 2, 2, 3, STAGES, 2>, 256, gemm_smem_bytes<32, 32>()},   // 2 k-split groups
    // 6 .. 9: same per-iteration kernels as 3, 5, 4, 2 (these indices differ in the ROUND kernel only:
    // deeper TMA pipelines, see kRoundConfigs)
    {dmma_gemm_kernel<32, 32, 2, 2, 6>, 128, gemm_smem_bytes<32, 32>()},
    {dmma_gemm_kernel<32, 32, 2, 2, 3, STAGES, 2>, 256, gemm_smem_bytes<32, 32>()},
    {dmma_gemm_kernel<32, 32, 2, 2, 2, STAGES, 4>, 512, gemm_smem_bytes<32, 32>()},
    {dmma_gemm_kernel<64, 32, 2, 2, 4>, 128, gemm_smem_bytes<64, 32>()},
};

// Round kernel (cqp_batch_round.cuh) per tile configuration: same shapes as kConfigs (the unused
// 128 x 128 entry maps to 64 x 64).
using RoundKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const RoundParams);
struct RoundConfig {
  RoundKernel fn;
  int threads;
  int smem;
  int box_a, box_s;  // index of the TMA descriptor: 0 = 64-row box, 1 = 32-row box
};
#define CQP_ROUND_CFG(BM, BN, ST, KS, MINB)                                                     \
  { round_kernel<BM, BN, 2, 2, ST, KS, MINB>, (4 * KS + 1) * 32, round_smem_bytes<BM, BN, 2, 2, ST, KS>(), \
    BM == 64 ? 0 : 1, BN == 64 ? 0 : 1 }
const RoundConfig kRoundConfigs[kNumConfigs] = {
    CQP_ROUND_CFG(64, 64, 4, 1, 3), CQP_ROUND_CFG(64, 64, 4, 1, 3), CQP_ROUND_CFG(64, 32, 4, 1, 4),
    CQP_ROUND_CFG(32, 32, 4, 1, 6), CQP_ROUND_CFG(32, 32, 4, 4, 2), CQP_ROUND_CFG(32, 32, 4, 2, 3),
    // deeper pipelines for rounds whose items no longer fill the SMs (an item's K loop is then bound by
    // the TMA latency times k-tiles / stages in flight)
    CQP_ROUND_CFG(32, 32, 8, 1, 3), CQP_ROUND_CFG(32, 32, 8, 2, 3), CQP_ROUND_CFG(32, 32, 10, 4, 2),
    CQP_ROUND_CFG(64, 32, 6, 1, 3),
};
#undef CQP_ROUND_CFG

// 2-D TMA descriptor of a row-major FP64 matrix [rows][ld] (K contiguous): box = 16 doubles (one
// 128-byte swizzle span) x box_rows.
int make_tensor_map(CUtensorMap* out, const double* base, size_t rows, int ld, int box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult st;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &st) != cudaSuccess || !fn) {
      set_error("cuTensorMapEncodeTiled is not available from this driver");
      return CQP_ERR_CUDA;
    }
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return CQP_ERR_CUDA;
  }
  return CQP_OK;
}

// Tile shape for a round with (at most) `active` columns still iterating.
int pick_config(const cqp_batch* b, int active) {
  if (b->force_cfg >= 0) return b->force_cfg;
  for (const auto& step : b->plan)
    if (active >= step.second) return step.first;
  if (active >= b->thr_big) return 0;
  if (active >= b->thr_mid) return 1;
  if (active >= b->thr_small) return 2;
  if (active >= b->thr_tiny) return b->small_cfg;
  return b->tiny_cfg;
}

int launch_gemm(cqp_batch* b, const GemmParams& p0, int cfg) {
  b->last_launches += 1;
  const GemmConfig& c = kConfigs[cfg];
  GemmParams p = p0;
  p.work_ctr = (b->dynamic && b->work_ctr_next < b->work_ctr_cap) ? b->work_ctrs + b->work_ctr_next++ : nullptr;
  c.fn<<<b->grid_ctas[cfg], c.threads, c.smem, b->stream>>>(p);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

int repad(cqp_batch* b, const double* src, int rows, int cols, int ld_src, size_t src_stride,
          double* dst, int rows_pad, int ld_dst, size_t dst_stride, int count) {
  const size_t total = (size_t)rows_pad * ld_dst * count;
  repad_kernel<<<(unsigned)((total + 255) / 256), 256, 0, b->stream>>>(src, rows, cols, ld_src, src_stride,
                                                                      dst, rows_pad, ld_dst, dst_stride, count);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

}  // namespace

namespace cqp {

// Dense C = alpha * A * B on the DMMA kernel for the offline stage (cqp_setup.cu):
//   A: [M_pad128][lda] row-major (K contiguous, zero padded, lda % 16 == 0)
//   B: N columns of [ldb] (K contiguous, zero padded), C: N columns of [ldc].
struct DenseGemm {
  int* cols = nullptr;
  TileDesc* tiles = nullptr;
  int* n_tiles = nullptr;
  int N = 0;
  int grid = 0;
};

int dense_gemm_create(DenseGemm** out, int N, int num_sms) {
  DenseGemm* g = new DenseGemm();
  *out = g;
  g->N = N;
  const int slots = (N + SLOT_TILE - 1) / SLOT_TILE * SLOT_TILE, tiles = slots / SLOT_TILE;
  std::vector<int> cols(slots, -1);
  for (int i = 0; i < N; ++i) cols[i] = i;
  std::vector<TileDesc> td(tiles);
  for (int t = 0; t < tiles; ++t) td[t] = {t * SLOT_TILE, 0};
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->cols), sizeof(int) * slots));
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->tiles), sizeof(TileDesc) * tiles));
  CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->n_tiles), sizeof(int)));
  CQP_CUDA(cudaMemcpy(g->cols, cols.data(), sizeof(int) * slots, cudaMemcpyHostToDevice));
  CQP_CUDA(cudaMemcpy(g->tiles, td.data(), sizeof(TileDesc) * tiles, cudaMemcpyHostToDevice));
  CQP_CUDA(cudaMemcpy(g->n_tiles, &tiles, sizeof(int), cudaMemcpyHostToDevice));
  CQP_CUDA(cudaStreamSynchronize(0));  // pageable sources: the DMAs may outlive the calls
  const GemmConfig& gc = kConfigs[1];
  CQP_CUDA(cudaFuncSetAttribute(gc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, gc.smem));
  int occ = 0;
  CQP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gc.fn, gc.threads, gc.smem));
  g->grid = (occ < 1 ? 1 : occ) * num_sms;
  return CQP_OK;
}

void dense_gemm_destroy(DenseGemm* g) {
  if (!g) return;
  cudaFree(g->cols); cudaFree(g->tiles); cudaFree(g->n_tiles);
  delete g;
}

int dense_gemm_run(const DenseGemm* g, cudaStream_t st, const double* A, int lda, int M, int M_pad,
                   const double* B, int ldb, double* C, int ldc, double alpha) {
  GemmParams p{};
  p.A = A; p.a_stride = 0; p.lda = lda; p.M = M; p.M_pad = M_pad; p.k_tiles = lda / BK;
  p.Bm = B; p.ldb = ldb; p.cols = g->cols; p.tiles = g->tiles; p.n_tiles = g->n_tiles;
  p.C = C; p.ldc = ldc; p.alpha = alpha; p.mode = 0;
  const GemmConfig& gc = kConfigs[1];  // 64 x 64 tiles
  gc.fn<<<g->grid, gc.threads, gc.smem, st>>>(p);
  CQP_CUDA(cudaGetLastError());
  return CQP_OK;
}

}  // namespace cqp

static void batch_destroy_single(cqp_batch* b);

static int batch_create_single(cqp_batch** out, cqp_handle* h, int capacity) {
  *out = nullptr;
  CQP_CUDA(cudaSetDevice(h->device));
  cqp_batch* b = new cqp_batch();
  b->h = h; b->capacity = capacity;
  b->n = h->n; b->m = h->m; b->D = h->D; b->L = h->L;
  const int n = b->n, m = b->m, D = b->D, L = b->L, nm = n + m;
  b->ld_s = round_up_i(D, BK); b->ld_n = round_up_i(n, BK); b->ld_m = round_up_i(m, BK);
  b->ld_nm = round_up_i(nm, 2);
  b->nm_mpad = round_up_i(nm, 128);
  b->n_mpad = round_up_i(n, 128); b->m_mpad = round_up_i(m, 128);
  int dense = 0;
  if (const char* e = std::getenv("CQP_BATCH_DENSE")) dense = std::atoi(e);
  b->split = dense ? 0 : b->nm_mpad;
  b->Dm_pad = dense ? round_up_i(D, 128) : b->nm_mpad + b->m_mpad;
  auto fail = [&](int rc) { batch_destroy_single(b); return rc; };
  if (cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(CQP_ERR_CUDA);
  cudaEventCreate(&b->ev0); cudaEventCreate(&b->ev1);
  cudaEventCreate(&b->evc0); cudaEventCreate(&b->evc1);
  for (int cfg = 0; cfg < kNumConfigs; ++cfg) {
    const GemmConfig& gc = kConfigs[cfg];
    if (cudaFuncSetAttribute(gc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, gc.smem) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "cudaFuncSetAttribute(dmma_gemm_kernel)"));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gc.fn, gc.threads, gc.smem) != cudaSuccess || occ < 1)
      return fail(cuda_fail(cudaGetLastError(), "occupancy(dmma_gemm_kernel)"));
    b->grid_ctas[cfg] = occ * h->num_sms;
  }
  for (int cfg = 0; cfg < kNumConfigs; ++cfg) {
    const RoundConfig& rc = kRoundConfigs[cfg];
    if (cudaFuncSetAttribute(rc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, rc.smem) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "cudaFuncSetAttribute(round_kernel)"));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rc.fn, rc.threads, rc.smem) != cudaSuccess || occ < 1)
      return fail(cuda_fail(cudaGetLastError(), "occupancy(round_kernel)"));
    b->round_grid[cfg] = occ * h->num_sms;
  }
  if (const char* e = std::getenv("CQP_BATCH_LEGACY")) b->legacy = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("CQP_ROUND_FLAGS")) b->round_flags = std::atoi(e);
  if (const char* e = std::getenv("CQP_ROUND_VERIFY")) b->verify = std::atoi(e);
  if (const char* e = std::getenv("CQP_BATCH_THRESHOLDS")) std::sscanf(e, "%d,%d,%d", &b->thr_big, &b->thr_mid, &b->thr_small);
  if (const char* e = std::getenv("CQP_BATCH_FORCE_CFG")) b->force_cfg = std::atoi(e);
  if (!b->legacy && !std::getenv("CQP_BATCH_PLAN") && !std::getenv("CQP_BATCH_THRESHOLDS") && !std::getenv("CQP_BATCH_TINY") &&
      !std::getenv("CQP_BATCH_SMALL_CFG")) {
    // Round kernel, calibrated on B200 at D = 1500 (tools/ab_batch.py sweeps; ms per solve, same box):
    // 4096 columns 242.7 with the per-iteration kernel's thresholds and 4-stage pipelines, 230.0 with
    // this plan; 1024 columns 102.3 -> 88.3; 512: 78.0 -> 65.0; 256: 64.9 -> 56.5; 64: 50.7 -> 44.0.
    // Below ~800 columns an iteration has fewer items than the SMs have CTA slots, an item's K loop is
    // then bound by TMA latency x k-tiles / stages in flight: deeper pipelines (8 stages of 32 x 32,
    // 6 of 64 x 32), and two k-split warp groups below 250 columns.
    // With the K loops of the small rounds split over 3 CTAs (kx, kx_thr: rounds of at most 350 columns) the
    // plain 32 x 32 configuration serves all of them (one B200, ms per solve of 512 / 4096 columns: no split
    // 64.3 / 225.8; split below 96 columns 57.2 / 221.7, below 350: 52.8 / 219.9; and without the in-CTA
    // k-split groups below 250 columns: 49.9 / 218.6).
    // Session 4 (shorter hand-over chain in the round kernel): 4 CTAs per tile below 350 columns and 6 below 64
    // (kx, kx_few): 64 / 512 / 4096 columns 26.7 / 46.6 / 214.7 -> 22.5 / 44.9 / 214.4 ms; thresholds of 500
    // columns or 3 / 5 / 8 splits are slower.
    b->plan = {{1, 3400}, {2, 1600}, {9, 800}, {6, 0}};
  }
  if (const char* e = std::getenv("CQP_BATCH_PLAN")) {
    int cfg = 0, bound = 0, used = 0;
    while (std::sscanf(e, "%d:%d%n", &cfg, &bound, &used) == 2) {
      if (cfg >= 0 && cfg < kNumConfigs) b->plan.emplace_back(cfg, bound);
      e += used;
      if (*e == ',') ++e;
    }
  }
  if (const char* e = std::getenv("CQP_BATCH_DYNAMIC")) b->dynamic = std::atoi(e) ? 1 : 0;
  if (const char* e = std::getenv("CQP_BATCH_KX")) {
    b->kx_few = 0;  // (a two-value setting switches the second level off: "kx,thr" keeps its old meaning)
    std::sscanf(e, "%d,%d,%d,%d", &b->kx, &b->kx_thr, &b->kx_few, &b->kx_few_thr);
    if (b->kx_few <= 0) { b->kx_few = b->kx; b->kx_few_thr = 0; }
  }
  b->kx = std::max(1, std::min(kKxMaxSplit, b->kx));
  b->kx_few = std::max(1, std::min(kKxMaxSplit, b->kx_few));
  if (const char* e = std::getenv("CQP_BATCH_SMALL_CFG")) b->small_cfg = std::atoi(e);
  if (const char* e = std::getenv("CQP_BATCH_TINY")) std::sscanf(e, "%d,%d", &b->tiny_cfg, &b->thr_tiny);
  int rc;
  const size_t cap = (size_t)capacity;
  const size_t slot_cap = cap + (size_t)L * SLOT_TILE, tile_cap = slot_cap / SLOT_TILE + L;
#define BA(ptr, count) if ((rc = balloc(&b->ptr, (count)))) return fail(rc)
  BA(Wb, (size_t)L * b->Dm_pad * b->ld_s);
  BA(negrho, (size_t)L * m);
  BA(DGb, (size_t)L * b->nm_mpad * b->ld_n);
  BA(Hb, (size_t)b->n_mpad * b->ld_n);
  BA(Gb, (size_t)b->m_mpad * b->ld_n);
  BA(Gtb, (size_t)b->n_mpad * b->ld_m);
  b->slot_cap = (int)slot_cap;
  BA(S0, slot_cap * b->ld_s); BA(S1, slot_cap * b->ld_s); BA(bias, cap * b->ld_nm);
  BA(slot_of, cap);
  BA(ct[0], slot_cap / 64 + 1); BA(ct[1], slot_cap / 32 + 1); BA(n_ct, 2);
  BA(bias_dirty, cap); BA(cols2, slot_cap); BA(tiles2, tile_cap); BA(n_tiles2, 1);
  if (b->verify) { BA(T[0], slot_cap * b->ld_s); BA(T[1], slot_cap * b->ld_s); BA(vres, 2); }
  b->round_ctr_count = 1 + (int)(slot_cap / 32) + 8;
  b->kx_cnt_off = b->round_ctr_count;                       // per-tile arrival counters of the K split
  b->round_ctr_count += kKxMaxTiles * (b->Dm_pad / 32) * 4;
  BA(round_ctrs, (size_t)b->round_ctr_count);
  BA(kx_part, (size_t)kKxMaxTiles * b->Dm_pad * kKxMaxSplit * 32);    // [tiles][row tiles][<= kKxMaxSplit splits][32 x 32]
  BA(g, cap * n); BA(c, cap * m); BA(d, cap * m);
  BA(gs, cap * b->ld_n); BA(lo, cap * b->ld_m); BA(hi, cap * b->ld_m);
  BA(uy, cap * b->ld_n); BA(ul, cap * b->ld_m); BA(uz, cap * b->ld_m);
  BA(hy, cap * b->ld_n); BA(gtl, cap * b->ld_n); BA(gy, cap * b->ld_m);
  BA(layer, cap); BA(active, cap); BA(iters, cap); BA(status, cap); BA(nsw, cap);
  BA(rp, cap); BA(rd, cap); BA(out_y, cap * n); BA(out_z, cap * m); BA(out_l, cap * m);
  b->rec_cap = h->s.max_iters / h->s.check_interval + 2;
  BA(trace, cap * b->rec_cap); BA(hist, cap * b->rec_cap); BA(nhist, cap);
  BA(cols, slot_cap); BA(tiles, tile_cap); BA(n_tiles, 1); BA(n_active, 1);
#undef BA
  // shared matrices: handle layouts (row-major, even ld) -> tile-padded copies
  if (b->split == 0) {
    if ((rc = repad(b, h->W, D, D, h->Dpad, (size_t)D * h->Dpad, b->Wb, b->Dm_pad, b->ld_s,
                    (size_t)b->Dm_pad * b->ld_s, L))) return fail(rc);
  } else {
    // rows 0 .. n+m-1 in full; rows n+m .. D-1 from padded row `split` on, first n columns only
    if ((rc = repad(b, h->W, nm, D, h->Dpad, (size_t)D * h->Dpad, b->Wb, b->nm_mpad, b->ld_s,
                    (size_t)b->Dm_pad * b->ld_s, L))) return fail(rc);
    if ((rc = repad(b, h->W + (size_t)nm * h->Dpad, m, n, h->Dpad, (size_t)D * h->Dpad,
                    b->Wb + (size_t)b->split * b->ld_s, b->m_mpad, b->ld_s, (size_t)b->Dm_pad * b->ld_s, L))) return fail(rc);
    extract_negrho_kernel<<<(m * L + 255) / 256, 256, 0, b->stream>>>(h->W, h->Dpad, (size_t)D * h->Dpad, n, m, b->negrho, L);
    if (cudaGetLastError() != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "extract_negrho_kernel"));
  }
  if ((rc = repad(b, h->Dk, nm, n, h->npad, (size_t)nm * h->npad, b->DGb, b->nm_mpad, b->ld_n,
                  (size_t)b->nm_mpad * b->ld_n, L))) return fail(rc);
  if ((rc = repad(b, h->H, n, n, h->npad, 0, b->Hb, b->n_mpad, b->ld_n, 0, 1))) return fail(rc);
  if ((rc = repad(b, h->Gr, m, n, h->npad, 0, b->Gb, b->m_mpad, b->ld_n, 0, 1))) return fail(rc);
  if ((rc = repad(b, h->Gt, n, m, h->mpad, 0, b->Gtb, b->n_mpad, b->ld_m, 0, 1))) return fail(rc);
  if (cudaStreamSynchronize(b->stream) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "batch_create sync"));
  for (int box = 0; box < 2; ++box) {
    const int rows = box == 0 ? 64 : 32;
    if ((rc = make_tensor_map(&b->mapA[box], b->Wb, (size_t)L * b->Dm_pad, b->ld_s, rows))) return fail(rc);
    if ((rc = make_tensor_map(&b->mapS[0][box], b->S0, slot_cap, b->ld_s, rows))) return fail(rc);
    if ((rc = make_tensor_map(&b->mapS[1][box], b->S1, slot_cap, b->ld_s, rows))) return fail(rc);
  }
  {
    // device copies, indexed [box_a * 2 + box_s][3]
    CUtensorMap host[12];
    for (int ba = 0; ba < 2; ++ba)
      for (int bs = 0; bs < 2; ++bs) {
        host[(ba * 2 + bs) * 3 + 0] = b->mapA[ba];
        host[(ba * 2 + bs) * 3 + 1] = b->mapS[0][bs];
        host[(ba * 2 + bs) * 3 + 2] = b->mapS[1][bs];
      }
    if (cudaMalloc(reinterpret_cast<void**>(&b->gmaps), sizeof(host)) != cudaSuccess ||
        cudaMemcpy(b->gmaps, host, sizeof(host), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "tensor map upload"));
  }
  *out = b;
  return CQP_OK;
}

static void batch_destroy_single(cqp_batch* b) {
  if (!b) return;
  if (b->h) cudaSetDevice(b->h->device);
  if (b->stream) cudaStreamSynchronize(b->stream);
  void* ptrs[] = {b->bias_dirty, b->cols2, b->tiles2, b->n_tiles2, b->ct[0], b->ct[1], b->n_ct, b->T[0], b->T[1], b->vres, b->gmaps, b->slot_of, b->round_ctrs, b->kx_part, b->work_ctrs, b->negrho, b->Wb, b->DGb, b->Hb, b->Gb, b->Gtb, b->S0, b->S1, b->bias, b->g, b->c, b->d, b->gs,
                  b->lo, b->hi, b->uy, b->ul, b->uz, b->hy, b->gtl, b->gy, b->layer, b->active,
                  b->iters, b->status, b->nsw, b->rp, b->rd, b->out_y, b->out_z, b->out_l, b->cols,
                  b->trace, b->hist, b->nhist,
                  b->tiles, b->n_tiles, b->n_active};
  for (void* p : ptrs) cudaFree(p);
  if (b->h_active) cudaFreeHost(b->h_active);
  for (cudaEvent_t e : b->round_events) cudaEventDestroy(e);
  for (cudaEvent_t e : b->it0) cudaEventDestroy(e);
  for (cudaEvent_t e : b->it1) cudaEventDestroy(e);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  if (b->evc0) cudaEventDestroy(b->evc0);
  if (b->evc1) cudaEventDestroy(b->evc1);
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
}

// One lane: B columns on b->stream.  `gate` (may be null): the stream waits for it first.
static int batch_solve_single(cqp_batch* b, int B, const double* g_cols, const double* c_cols,
                              const double* d_cols, double* y_cols, double* z_cols, double* lambda_cols,
                              int* status, int* iterations, int* final_index, double* r_prim,
                              double* r_dual, int* n_switches, double* device_ms, cudaEvent_t gate) {
  cqp_handle* h = b->h;
  CQP_CUDA(cudaSetDevice(h->device));
  if (gate) CQP_CUDA(cudaStreamWaitEvent(b->stream, gate, 0));
  const int n = b->n, m = b->m, nm = n + m;
  const cqp_settings& s = h->s;
  const int interval = s.check_interval;
  const int full_rounds = s.max_iters / interval, rem = s.max_iters % interval;
  const int rounds = full_rounds + (rem ? 1 : 0);
  if (b->h_active_cap < rounds + 1) {
    if (b->h_active) cudaFreeHost(b->h_active);
    CQP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&b->h_active), sizeof(int) * (rounds + 1)));
    b->h_active_cap = rounds + 1;
  }
  while ((int)b->round_events.size() < rounds + 1) {
    cudaEvent_t e, e0, e1;
    CQP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CQP_CUDA(cudaEventCreate(&e0));
    CQP_CUDA(cudaEventCreate(&e1));
    b->round_events.push_back(e);
    b->it0.push_back(e0);
    b->it1.push_back(e1);
  }
  cudaStream_t st = b->stream;
  {
    const int need = rounds * (interval + 4) + 8;  // GEMM launches of one solve
    if (b->work_ctr_cap < need) {
      cudaFree(b->work_ctrs);
      b->work_ctrs = nullptr; b->work_ctr_cap = 0;
      CQP_CUDA(cudaMalloc(reinterpret_cast<void**>(&b->work_ctrs), sizeof(int) * need));
      b->work_ctr_cap = need;
    }
    b->work_ctr_next = 0;
  }
  CQP_CUDA(cudaEventRecord(b->ev0, st));
  CQP_CUDA(cudaMemsetAsync(b->work_ctrs, 0, sizeof(int) * b->work_ctr_cap, st));
  CQP_CUDA(cudaMemcpyAsync(b->g, g_cols, sizeof(double) * (size_t)n * B, cudaMemcpyDefault, st));
  CQP_CUDA(cudaMemcpyAsync(b->c, c_cols, sizeof(double) * (size_t)m * B, cudaMemcpyDefault, st));
  CQP_CUDA(cudaMemcpyAsync(b->d, d_cols, sizeof(double) * (size_t)m * B, cudaMemcpyDefault, st));
  // cold start: v = 0 (S is kept in slot order; every slot the map can use starts at zero)
  const size_t slots_used = (size_t)std::min(b->slot_cap, B + b->L * SLOT_TILE);
  CQP_CUDA(cudaMemsetAsync(b->S0, 0, sizeof(double) * slots_used * b->ld_s, st));
  CQP_CUDA(cudaMemsetAsync(b->S1, 0, sizeof(double) * slots_used * b->ld_s, st));
  CQP_CUDA(cudaMemsetAsync(b->slot_of, 0, sizeof(int) * (size_t)B, st));

  BatchDev bd{};
  bd.n = n; bd.m = m; bd.D = b->D; bd.B = B;
  bd.ld_s = b->ld_s; bd.ld_n = b->ld_n; bd.ld_m = b->ld_m; bd.ld_nm = b->ld_nm;
  bd.E = h->E; bd.F = h->F; bd.cost_scale = h->cost_scale;
  bd.grid = h->dgrid; bd.log_grid = h->dlog_grid; bd.L = b->L;
  bd.g = b->g; bd.c = b->c; bd.d = b->d; bd.gs = b->gs; bd.lo = b->lo; bd.hi = b->hi;
  bd.uy = b->uy; bd.ul = b->ul; bd.uz = b->uz; bd.hy = b->hy; bd.gtl = b->gtl; bd.gy = b->gy;
  bd.layer = b->layer; bd.active = b->active; bd.iters = b->iters; bd.status = b->status;
  bd.nsw = b->nsw; bd.rp = b->rp; bd.rd = b->rd;
  bd.trace = b->trace; bd.hist = b->hist; bd.nhist = b->nhist; bd.rec_cap = b->rec_cap;
  b->last_B = B;
  bd.out_y = b->out_y; bd.out_z = b->out_z; bd.out_l = b->out_l;
  bd.cols = b->cols; bd.tiles = b->tiles; bd.n_tiles = b->n_tiles; bd.n_active = b->n_active;
  bd.slot_of = b->slot_of;
  bd.ct[0] = b->ct[0]; bd.ct[1] = b->ct[1]; bd.n_ct = b->n_ct;
  const bool fast_regroup = b->L <= kRegroupMaxL;
  bd.bias_dirty = b->bias_dirty;
  bd.cols2 = fast_regroup ? b->cols2 : b->cols; bd.tiles2 = fast_regroup ? b->tiles2 : b->tiles;
  bd.n_tiles2 = fast_regroup ? b->n_tiles2 : b->n_tiles;
  bd.eps_prim = s.eps_prim; bd.eps_dual = s.eps_dual; bd.threshold = s.rho_switch_threshold;
  bd.adaptive = s.adaptive_rho; bd.max_iters = s.max_iters;

  CQP_CUDA(cudaEventRecord(b->evc0, st));  // inputs are resident from here on
  b->last_launches = 0;
  batch_prepare_kernel<<<B, 128, 0, st>>>(bd, h->initial_index);
  CQP_CUDA(cudaGetLastError());

  GemmParams base{};
  base.cols = b->cols; base.tiles = b->tiles; base.n_tiles = b->n_tiles;
  base.alpha = 1.0;
  auto gemm_bias = [&](int cfg) {  // Bias = -[D_k; G D_k] g_s  (layers.cpp:168-175), per bucket
    GemmParams p = base;
    p.cols = bd.cols2; p.tiles = bd.tiles2; p.n_tiles = bd.n_tiles2;  // only the columns whose level changed
    p.A = b->DGb; p.a_stride = (size_t)b->nm_mpad * b->ld_n; p.lda = b->ld_n; p.M = nm;
    p.M_pad = b->nm_mpad; p.k_tiles = b->ld_n / BK;
    p.Bm = b->gs; p.ldb = b->ld_n; p.C = b->bias; p.ldc = b->ld_nm; p.alpha = -1.0; p.mode = 0;
    return launch_gemm(b, p, cfg);
  };
  auto gemm_iter = [&](const double* Sin, double* Sout, int cfg) {  // one ADMM layer for every active column
    GemmParams p = base;
    p.A = b->Wb; p.a_stride = (size_t)b->Dm_pad * b->ld_s; p.lda = b->ld_s; p.M = b->D;
    p.M_pad = b->Dm_pad; p.k_tiles = b->ld_s / BK;
    p.Bm = Sin; p.ldb = b->ld_s; p.C = Sout; p.ldc = b->ld_s; p.mode = 1;
    p.bias = b->bias; p.ld_bias = b->ld_nm; p.nm = nm; p.n = n;
    p.lo = b->lo; p.hi = b->hi; p.ld_lohi = b->ld_m;
    p.split = b->split; p.k_tiles3 = b->ld_n / BK; p.negrho = b->negrho;
    p.slot_major = 1;
    return launch_gemm(b, p, cfg);
  };
  double* Sbuf[2] = {b->S0, b->S1};
  // one persistent launch = `steps` ADMM layers of every active column (cqp_batch_round.cuh)
  int kx_for_round = 1;
  auto round_run = [&](int first, int steps, int cfg) {
    const RoundConfig& rcfg = kRoundConfigs[cfg];
    RoundParams p{};
    p.n = n; p.m = m; p.nm = nm; p.D = b->D; p.M_pad = b->Dm_pad; p.split = b->split;
    p.k_tiles = b->ld_s / BK; p.k_tiles3 = b->split ? b->ld_n / BK : b->ld_s / BK;
    p.cols = b->cols; p.tiles = b->ct[rcfg.box_s]; p.n_tiles = b->n_ct + rcfg.box_s;
    p.bias = b->bias; p.ld_bias = b->ld_nm; p.lo = b->lo; p.hi = b->hi; p.ld_lohi = b->ld_m;
    p.negrho = b->negrho;
    p.S[0] = b->S0; p.S[1] = b->S1; p.ld_s = b->ld_s; p.first = first; p.n_iters = steps;
    p.work = b->round_ctrs; p.done = b->round_ctrs + 1; p.dbg = h->dbg_dev;
    p.num_sms = (b->round_flags & 2) ? 0 : h->num_sms;
    p.flags = b->round_flags; p.gmaps = b->gmaps + (rcfg.box_a * 2 + rcfg.box_s) * 3;
    // K split over CTAs in the small rounds (32 x 32 tiles only: that is what `part` is sized for)
    p.kx = (rcfg.box_a == 1 && rcfg.box_s == 1 && kx_for_round > 1) ? kx_for_round : 1;
    p.kx_max_tiles = kKxMaxTiles; p.part = b->kx_part; p.tile_cnt = b->round_ctrs + b->kx_cnt_off;
    CQP_CUDA(cudaMemsetAsync(b->round_ctrs, 0, sizeof(int) * (size_t)b->round_ctr_count, st));
    rcfg.fn<<<b->round_grid[cfg], rcfg.threads, rcfg.smem, st>>>(b->mapA[rcfg.box_a], b->mapS[0][rcfg.box_s],
                                                                 b->mapS[1][rcfg.box_s], p);
    CQP_CUDA(cudaGetLastError());
    b->last_launches += 1;
    return (int)CQP_OK;
  };
  auto permute = [&](int from) {  // compact S[from] into S[from ^ 1] following the fresh slot map
    batch_permute_kernel<<<(unsigned)slots_used, 128, 0, st>>>(bd, Sbuf[from], Sbuf[from ^ 1]);
    CQP_CUDA(cudaGetLastError());
    b->last_launches += 1;
    return (int)CQP_OK;
  };
  auto gemm_plain = [&](const double* A, int M, int m_pad, int lda, const double* Bm, int ldb, double* C, int ldc, int cfg) {
    GemmParams p = base;
    p.A = A; p.a_stride = 0; p.lda = lda; p.M = M; p.M_pad = m_pad; p.k_tiles = lda / BK;
    p.Bm = Bm; p.ldb = ldb; p.C = C; p.ldc = ldc; p.mode = 0;
    return launch_gemm(b, p, cfg);
  };

  int rc;
  auto regroup = [&]() {
    if (fast_regroup) batch_regroup_fast_kernel<<<1, kRegroupThreads, 0, st>>>(bd);
    else batch_regroup_kernel<<<1, 1024, 0, st>>>(bd);
  };
  regroup();
  CQP_CUDA(cudaGetLastError());
  b->last_launches += 2;  // prepare, regroup
  if ((rc = gemm_bias(pick_config(b, B)))) return rc;
  int cur = 0;  // Sbuf[cur] holds the iterate
  if ((rc = permute(cur))) return rc;  // (all zeros: this only fills slot_of)
  cur ^= 1;
  int it = 0, rounds_done = 0;
  for (int r = 0; r < rounds; ++r) {
    if (r >= 2) {  // stay at most two rounds ahead of the device; stop once every column is done
      CQP_CUDA(cudaEventSynchronize(b->round_events[r - 2]));
      if (b->h_active[r - 2] == 0) break;
    }
    const int steps = (r < full_rounds) ? interval : rem;
    // the host knows the active count with a lag of two rounds; it only decreases
    const int cfg = pick_config(b, r >= 2 ? b->h_active[r - 2] : B);
    {
      const int seen = r >= 2 ? b->h_active[r - 2] : B;  // (the active count two rounds ago: what the host has seen)
      kx_for_round = seen <= b->kx_few_thr ? b->kx_few : seen <= b->kx_thr ? b->kx : 1;
    }
    CQP_CUDA(cudaEventRecord(b->it0[r], st));
    if (b->legacy) {
      for (int k = 0; k < steps; ++k) {
        if ((rc = gemm_iter(Sbuf[cur], Sbuf[cur ^ 1], cfg))) return rc;
        cur ^= 1;
      }
    } else {
      if (b->verify) {
        const size_t bytes = sizeof(double) * slots_used * b->ld_s;
        CQP_CUDA(cudaMemcpyAsync(b->T[0], Sbuf[cur], bytes, cudaMemcpyDeviceToDevice, st));
        CQP_CUDA(cudaMemcpyAsync(b->T[1], Sbuf[cur ^ 1], bytes, cudaMemcpyDeviceToDevice, st));
        int tc = 0;
        for (int k = 0; k < steps; ++k) {
          if ((rc = gemm_iter(b->T[tc], b->T[tc ^ 1], cfg))) return rc;
          tc ^= 1;
        }
        if ((rc = round_run(cur, steps, cfg))) return rc;
        cur ^= steps & 1;
        const unsigned long long init[2] = {~0ull, 0ull};
        CQP_CUDA(cudaMemcpyAsync(b->vres, init, sizeof(init), cudaMemcpyHostToDevice, st));
        batch_compare_kernel<<<(unsigned)slots_used, 256, 0, st>>>(Sbuf[cur], b->T[tc], b->n_tiles, b->cols, b->ld_s, b->D, b->vres);
        unsigned long long got[2] = {0, 0};
        int nt = 0;
        CQP_CUDA(cudaMemcpyAsync(got, b->vres, sizeof(got), cudaMemcpyDeviceToHost, st));
        CQP_CUDA(cudaMemcpyAsync(&nt, b->n_tiles, sizeof(int), cudaMemcpyDeviceToHost, st));
        CQP_CUDA(cudaStreamSynchronize(st));
        if (got[1]) {
          std::vector<int> hc((size_t)nt * SLOT_TILE);
          std::vector<TileDesc> ht(nt);
          cudaMemcpy(hc.data(), b->cols, sizeof(int) * hc.size(), cudaMemcpyDeviceToHost);
          cudaMemcpy(ht.data(), b->tiles, sizeof(TileDesc) * nt, cudaMemcpyDeviceToHost);
          std::vector<double> sa((size_t)hc.size() * b->ld_s), sb(sa.size());
          cudaMemcpy(sa.data(), Sbuf[cur], sizeof(double) * sa.size(), cudaMemcpyDeviceToHost);
          cudaMemcpy(sb.data(), b->T[tc], sizeof(double) * sb.size(), cudaMemcpyDeviceToHost);
          std::fprintf(stderr, "[verify] round %d cfg %d steps %d: %llu entries differ; first slot %llu row %llu; tiles %d:", r, cfg,
                       steps, got[1], got[0] / b->ld_s, got[0] % b->ld_s, nt);
          for (int t = 0; t < nt; ++t) {
            int real = 0;
            for (int i = 0; i < SLOT_TILE; ++i) real += hc[(size_t)t * SLOT_TILE + i] >= 0;
            std::fprintf(stderr, " [a%d:%d]", ht[t].a_index, real);
          }
          std::fprintf(stderr, "\n[verify]   differing (slot: rows lo-hi count):");
          int shown = 0;
          for (size_t sidx = 0; sidx < hc.size() && shown < 24; ++sidx) {
            int lo = -1, hi = -1, cnt = 0;
            for (int i = 0; i < b->D; ++i)
              if (std::memcmp(&sa[sidx * b->ld_s + i], &sb[sidx * b->ld_s + i], 8) != 0) { if (lo < 0) lo = i; hi = i; ++cnt; }
            if (cnt) { std::fprintf(stderr, " %zu(col %d): %d-%d %d;", sidx, hc[sidx], lo, hi, cnt); ++shown; }
          }
          std::fprintf(stderr, "\n");
          // keep going from the legacy result so that later rounds are judged on their own
          CQP_CUDA(cudaMemcpyAsync(Sbuf[cur], b->T[tc], bytes, cudaMemcpyDeviceToDevice, st));
        }
      } else {
        if ((rc = round_run(cur, steps, cfg))) return rc;
        cur ^= steps & 1;
      }
    }
    CQP_CUDA(cudaEventRecord(b->it1[r], st));
    rounds_done = r + 1;
    it += steps;
    // NOTE: columns that stopped earlier keep their (stale) value in whichever buffer they were
    // last written to; they are never read again (results were captured when they stopped).
    batch_unscale_kernel<<<B, 128, 0, st>>>(bd, Sbuf[cur]);
    CQP_CUDA(cudaGetLastError());
    b->last_launches += 3;  // unscale, decide, regroup
    if ((rc = gemm_plain(b->Hb, n, b->n_mpad, b->ld_n, b->uy, b->ld_n, b->hy, b->ld_n, cfg))) return rc;
    if ((rc = gemm_plain(b->Gtb, n, b->n_mpad, b->ld_m, b->ul, b->ld_m, b->gtl, b->ld_n, cfg))) return rc;
    if ((rc = gemm_plain(b->Gb, m, b->m_mpad, b->ld_n, b->uy, b->ld_n, b->gy, b->ld_m, cfg))) return rc;
    batch_decide_kernel<<<(B + 7) / 8, 256, 0, st>>>(bd, it, r < full_rounds ? 1 : 0, 1);
    CQP_CUDA(cudaGetLastError());
    regroup();
    CQP_CUDA(cudaGetLastError());
    CQP_CUDA(cudaMemcpyAsync(&b->h_active[r], b->n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    CQP_CUDA(cudaEventRecord(b->round_events[r], st));
    if (r + 1 < rounds) {
      if ((rc = permute(cur))) return rc;
      cur ^= 1;
      if ((rc = gemm_bias(cfg))) return rc;
    }
  }
  CQP_CUDA(cudaEventRecord(b->evc1, st));
  // results
  if (y_cols) CQP_CUDA(cudaMemcpyAsync(y_cols, b->out_y, sizeof(double) * (size_t)n * B, cudaMemcpyDefault, st));
  if (z_cols) CQP_CUDA(cudaMemcpyAsync(z_cols, b->out_z, sizeof(double) * (size_t)m * B, cudaMemcpyDefault, st));
  if (lambda_cols) CQP_CUDA(cudaMemcpyAsync(lambda_cols, b->out_l, sizeof(double) * (size_t)m * B, cudaMemcpyDefault, st));
  if (status) CQP_CUDA(cudaMemcpyAsync(status, b->status, sizeof(int) * B, cudaMemcpyDefault, st));
  if (iterations) CQP_CUDA(cudaMemcpyAsync(iterations, b->iters, sizeof(int) * B, cudaMemcpyDefault, st));
  if (final_index) CQP_CUDA(cudaMemcpyAsync(final_index, b->layer, sizeof(int) * B, cudaMemcpyDefault, st));
  if (r_prim) CQP_CUDA(cudaMemcpyAsync(r_prim, b->rp, sizeof(double) * B, cudaMemcpyDefault, st));
  if (r_dual) CQP_CUDA(cudaMemcpyAsync(r_dual, b->rd, sizeof(double) * B, cudaMemcpyDefault, st));
  if (n_switches) CQP_CUDA(cudaMemcpyAsync(n_switches, b->nsw, sizeof(int) * B, cudaMemcpyDefault, st));
  CQP_CUDA(cudaEventRecord(b->ev1, st));
  CQP_CUDA(cudaStreamSynchronize(st));
  // iteration-GEMM profile of this solve: time of every round's GEMM launches and the
  // algorithmic flops they carried (2 D^2 per active column per iteration)
  b->last_gemm_ms = 0.0;
  b->last_gemm_flops = 0.0;
  b->last_rounds = rounds_done;
  b->round_ms.assign(rounds_done, 0.f);
  b->round_active.assign(rounds_done, 0);
  for (int r = 0; r < rounds_done; ++r) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, b->it0[r], b->it1[r]);
    const int steps = (r < full_rounds) ? interval : rem;
    const double active = (r == 0) ? (double)B : (double)b->h_active[r - 1];
    b->round_ms[r] = ms;
    b->round_active[r] = (int)active;
    b->last_gemm_ms += ms;
    // executed flops: the structured layer skips the zeros of blocks (3,2), (3,3) (4 m^2 flop) and
    // keeps their diagonals (2 FMA per lambda row)
    const double per_col = b->split ? 2.0 * ((double)nm * b->D + (double)m * n) + 4.0 * m
                                    : 2.0 * (double)b->D * (double)b->D;
    b->last_gemm_flops += per_col * active * steps;
  }
  cudaEventElapsedTime(&b->last_total_ms, b->ev0, b->ev1);
  cudaEventElapsedTime(&b->last_compute_ms, b->evc0, b->evc1);
  if (device_ms) *device_ms = b->last_total_ms;
  return CQP_OK;
}

// Records of one lane's last solve -> host arrays of `cap` entries per column, from column `off`.
template <typename Rec>
static int fetch_records(cqp_batch* b, const Rec* dev, const int* dev_len, int len_bias, int off, int cap,
                         Rec* out, int* out_len) {
  const int B = b->last_B, rc_dev = b->rec_cap;
  if (B <= 0) return CQP_OK;
  CQP_CUDA(cudaSetDevice(b->h->device));
  std::vector<Rec> host((size_t)B * rc_dev);
  std::vector<int> len(B);
  CQP_CUDA(cudaMemcpyAsync(host.data(), dev, sizeof(Rec) * host.size(), cudaMemcpyDeviceToHost, b->stream));
  CQP_CUDA(cudaMemcpyAsync(len.data(), dev_len, sizeof(int) * B, cudaMemcpyDeviceToHost, b->stream));
  CQP_CUDA(cudaStreamSynchronize(b->stream));
  for (int j = 0; j < B; ++j) {
    const int cnt = len[j] + len_bias;
    if (out_len) out_len[off + j] = cnt;  // (records beyond a capacity are dropped, the length still counts them)
    if (out)
      for (int k = 0; k < std::min(std::min(cnt, cap), rc_dev); ++k)
        out[(size_t)(off + j) * cap + k] = host[(size_t)j * rc_dev + k];
  }
  return CQP_OK;
}

template <typename Fn>
static int for_each_lane(cqp_batch* b, int B, Fn fn) {
  if (!b) { set_error("batch records: null batch"); return CQP_ERR_ARGUMENT; }
  if (b->lanes.empty()) {
    if (B != b->last_B) { set_error("batch records: B differs from the last solve"); return CQP_ERR_ARGUMENT; }
    return fn(b, 0);
  }
  int total = 0;
  for (int c : b->lane_cnt) total += c;
  if (B != total) { set_error("batch records: B differs from the last solve"); return CQP_ERR_ARGUMENT; }
  for (size_t k = 0; k < b->lane_cnt.size(); ++k) {
    if (b->lane_cnt[k] <= 0) continue;
    if (int rc = fn(b->lanes[k], b->lane_off[k])) return rc;
  }
  return CQP_OK;
}

extern "C" {

int cqp_batch_create(cqp_batch** out, cqp_handle* h, int capacity) {
  if (!out || !h || capacity < 1) { set_error("batch_create: bad argument"); return CQP_ERR_ARGUMENT; }
  *out = nullptr;
  // The round kernel keeps the SMs busy across iterations by itself (its grid drains once per round),
  // so it runs as ONE lane; two lanes (sub-batches on their own streams filling each other's wave
  // tails) only pay for the per-iteration kernel (CQP_BATCH_LEGACY=1).
  int legacy = 0;
  if (const char* e = std::getenv("CQP_BATCH_LEGACY")) legacy = std::atoi(e) ? 1 : 0;
  int lanes = (legacy && capacity >= 1024) ? 2 : 1;
  if (const char* e = std::getenv("CQP_BATCH_LANES")) lanes = std::max(1, std::min(8, std::atoi(e)));
  if (lanes == 1) return batch_create_single(out, h, capacity);
  CQP_CUDA(cudaSetDevice(h->device));
  cqp_batch* b = new cqp_batch();
  b->h = h; b->capacity = capacity;
  b->n = h->n; b->m = h->m; b->D = h->D; b->L = h->L;
  const int lane_cap = (capacity + lanes - 1) / lanes;
  for (int k = 0; k < lanes; ++k) {
    cqp_batch* lane = nullptr;
    const int rc = batch_create_single(&lane, h, lane_cap);
    if (rc) { cqp_batch_destroy(b); return rc; }
    b->lanes.push_back(lane);
  }
  if (cudaEventCreate(&b->ev_start) != cudaSuccess) { cqp_batch_destroy(b); return cuda_fail(cudaGetLastError(), "cudaEventCreate"); }
  *out = b;
  return CQP_OK;
}

void cqp_batch_destroy(cqp_batch* b) {
  if (!b) return;
  if (b->lanes.empty()) { batch_destroy_single(b); return; }
  for (cqp_batch* lane : b->lanes) batch_destroy_single(lane);
  if (b->ev_start) cudaEventDestroy(b->ev_start);
  delete b;
}

int cqp_batch_solve(cqp_batch* b, int B, const double* g_cols, const double* c_cols,
                    const double* d_cols, double* y_cols, double* z_cols, double* lambda_cols,
                    int* status, int* iterations, int* final_index, double* r_prim,
                    double* r_dual, int* n_switches, double* device_ms) {
  if (!b || !g_cols || !c_cols || !d_cols) { set_error("batch_solve: null argument"); return CQP_ERR_ARGUMENT; }
  if (B < 1 || B > b->capacity) { set_error("batch_solve: B exceeds the batch capacity"); return CQP_ERR_CAPACITY; }
  if (b->h->srv_running) {  // a resident MPC kernel owns the SMs: retire it first
    if (int rc = server_stop(b->h)) return rc;
  }
  if (b->lanes.empty())
    return batch_solve_single(b, B, g_cols, c_cols, d_cols, y_cols, z_cols, lambda_cols, status, iterations,
                              final_index, r_prim, r_dual, n_switches, device_ms, nullptr);
  // sub-batches: columns [off_k, off_k + B_k) go to lane k; small batches use one lane
  const int K = (int)b->lanes.size();
  int used = B < 512 ? 1 : K;
  while (used < K && (B + used - 1) / used > b->lanes[0]->capacity) ++used;  // (B <= capacity <= K * lane capacity)
  const int per = (B + used - 1) / used;
  const int n = b->n, m = b->m;
  CQP_CUDA(cudaSetDevice(b->h->device));
  CQP_CUDA(cudaEventRecord(b->ev_start, b->lanes[0]->stream));
  std::vector<int> rcs(used, CQP_OK), counts(used, 0);
  b->lane_off.assign(used, 0); b->lane_cnt.assign(used, 0);
  std::vector<std::string> errs(used);
  std::vector<std::thread> threads;
  for (int k = 0; k < used; ++k) {
    const int off = k * per, cnt = std::min(per, B - off);
    counts[k] = cnt;
    b->lane_off[k] = off; b->lane_cnt[k] = cnt > 0 ? cnt : 0;
    if (cnt <= 0) continue;
    threads.emplace_back([&, k, off, cnt] {
      auto at = [&](auto* p, size_t stride) { return p ? p + (size_t)off * stride : p; };
      rcs[k] = batch_solve_single(b->lanes[k], cnt, g_cols + (size_t)off * n, c_cols + (size_t)off * m,
                                  d_cols + (size_t)off * m, at(y_cols, n), at(z_cols, m), at(lambda_cols, m),
                                  at(status, 1), at(iterations, 1), at(final_index, 1), at(r_prim, 1),
                                  at(r_dual, 1), at(n_switches, 1), nullptr, b->ev_start);
      if (rcs[k]) errs[k] = cqp_last_error();
    });
  }
  for (std::thread& t : threads) t.join();
  for (int k = 0; k < used; ++k)
    if (rcs[k]) { set_error("batch lane " + std::to_string(k) + ": " + errs[k]); return rcs[k]; }
  // timings on the common base ev_start (every lane's stream waited for it and is idle again)
  float total = 0.f, c0 = 1e30f, c1 = 0.f;
  std::vector<std::pair<float, float>> spans;  // GEMM phases of all lanes
  b->last_launches = 0; b->last_gemm_flops = 0.0; b->last_rounds = 0;
  b->round_ms.clear(); b->round_active.clear();
  for (int k = 0; k < used; ++k) {
    if (counts[k] <= 0) continue;
    const cqp_batch* lane = b->lanes[k];
    float t = 0.f;
    cudaEventElapsedTime(&t, b->ev_start, lane->ev1); total = std::max(total, t);
    cudaEventElapsedTime(&t, b->ev_start, lane->evc0); c0 = std::min(c0, t);
    cudaEventElapsedTime(&t, b->ev_start, lane->evc1); c1 = std::max(c1, t);
    b->last_launches += lane->last_launches;
    b->last_gemm_flops += lane->last_gemm_flops;
    b->last_rounds = std::max(b->last_rounds, lane->last_rounds);
    if ((int)b->round_ms.size() < lane->last_rounds) { b->round_ms.resize(lane->last_rounds, 0.f); b->round_active.resize(lane->last_rounds, 0); }
    for (int r = 0; r < lane->last_rounds; ++r) {
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, b->ev_start, lane->it0[r]);
      cudaEventElapsedTime(&t1, b->ev_start, lane->it1[r]);
      spans.emplace_back(t0, t1);
      b->round_ms[r] = std::max(b->round_ms[r], lane->round_ms[r]);
      b->round_active[r] += lane->round_active[r];
    }
  }
  // iteration-GEMM time = length of the union of the lanes' GEMM phases
  std::sort(spans.begin(), spans.end());
  double uni = 0.0;
  float cur0 = 0.f, cur1 = -1.f;
  for (const auto& sp : spans) {
    if (cur1 < cur0 || sp.first > cur1) { if (cur1 >= cur0) uni += cur1 - cur0; cur0 = sp.first; cur1 = sp.second; }
    else cur1 = std::max(cur1, sp.second);
  }
  if (cur1 >= cur0) uni += cur1 - cur0;
  b->last_gemm_ms = uni;
  b->last_total_ms = total;
  b->last_compute_ms = c1 - c0;
  if (device_ms) *device_ms = total;
  return CQP_OK;
}

int cqp_batch_get_traces(cqp_batch* b, int B, int cap, cqp_rho_switch* trace, int* trace_len) {
  if (cap < 0 || (cap > 0 && !trace && !trace_len)) { set_error("batch_get_traces: bad argument"); return CQP_ERR_ARGUMENT; }
  return for_each_lane(b, B, [&](cqp_batch* lane, int off) {
    return fetch_records(lane, lane->trace, lane->nsw, 1, off, cap, trace, trace_len);
  });
}

int cqp_batch_get_history(cqp_batch* b, int B, int cap, cqp_residual_sample* history, int* history_len) {
  if (cap < 0 || (cap > 0 && !history && !history_len)) { set_error("batch_get_history: bad argument"); return CQP_ERR_ARGUMENT; }
  return for_each_lane(b, B, [&](cqp_batch* lane, int off) {
    return fetch_records(lane, lane->hist, lane->nhist, 0, off, cap, history, history_len);
  });
}

int cqp_batch_last_timing(const cqp_batch* b, double* compute_ms, double* total_ms, long long* launches) {
  if (!b) return CQP_ERR_ARGUMENT;
  if (compute_ms) *compute_ms = b->last_compute_ms;
  if (total_ms) *total_ms = b->last_total_ms;
  if (launches) *launches = b->last_launches;
  return CQP_OK;
}

int cqp_batch_round_profile(const cqp_batch* b, int cap, int* active, double* ms) {
  if (!b) return CQP_ERR_ARGUMENT;
  const int cnt = std::min(cap, (int)b->round_ms.size());
  for (int r = 0; r < cnt; ++r) {
    if (active) active[r] = b->round_active[r];
    if (ms) ms[r] = b->round_ms[r];
  }
  return CQP_OK;
}

int cqp_batch_last_profile(const cqp_batch* b, double* gemm_ms, double* gemm_flops, int* rounds) {
  if (!b) return CQP_ERR_ARGUMENT;
  if (gemm_ms) *gemm_ms = b->last_gemm_ms;
  if (gemm_flops) *gemm_flops = b->last_gemm_flops;
  if (rounds) *rounds = b->last_rounds;
  return CQP_OK;
}

}  // extern "C"
