// Batched path, iteration kernel: ONE persistent launch runs a whole check round (check_interval
// ADMM layers, /root/reference/proj/src/solver.cpp:59-63 per column) of the batch.
//
// Included by cqp_batch.cu (inside namespace cqp { namespace { ... } }) after TileDesc / SLOT_TILE.
//
//   * Operands are staged by TMA: cp.async.bulk.tensor.2d (SASS UTMALDG) moves a BM x 16 tile of
//     W_k and a BN x 16 tile of S into shared memory with the hardware 128-byte swizzle and
//     completes on an mbarrier (complete_tx); a dedicated producer warp issues the copies, the
//     consumer warps only wait on `full[stage]`, run DMMA.8x8x4 (mma.sync m8n8k4 f64: the FP64
//     tensor shape of sm_100a; tcgen05 has no f64 kind) and release the stage through `empty[stage]`.
//     No cp.async bookkeeping, no CTA-wide barrier in the K loop, and the producer runs ahead into
//     the next work item, so there is no pipeline-fill bubble between tiles.
//   * S is stored in SLOT order (physically compacted at every re-bucketing, batch_permute_kernel):
//     the 128 columns of a slot tile are contiguous, which is what makes them one 2-D TMA box.
//   * Fragment rows are permuted, g -> 2 (g & 3) | (g >> 2): the four rows a half-warp reads in one
//     8-byte LDS then sit at row-in-8 = {0, 2, 4, 6} (or {1, 3, 5, 7}), and the XOR of the 128-byte
//     swizzle (16-byte chunk ^ row-in-8) sends the two chunks {2 ks, 2 ks + 1} of those rows to eight
//     distinct chunks = all 32 banks.  (With the identity mapping rows 0 and 1 collide.)  The C
//     fragment is mapped back through the same permutation in the epilogue.
//   * Dataflow across iterations: work item = (iteration, column tile, row tile), taken from one
//     atomic counter in that order.  Item (i, c, *) reads column tile c of iteration i - 1, so the
//     producer waits until done[c] has counted every row tile of iteration i - 1 (each consumer
//     warp adds 1 after its stores, release at gpu scope; the producer's acquire + fence.proxy.async
//     orders the generic-proxy stores before its async-proxy reads).  Columns of different tiles
//     never wait for each other, so launches no longer end in a wave tail 25 times per round: the
//     grid drains once, at the end of the round.  Items are handed out in index order, so the owner
//     of the lowest unfinished item is always resident and never blocked: no deadlock whatever part
//     of the grid the device keeps resident (two lanes can run their kernels concurrently).
//   * The chain of one iteration is kept short (it is what a small round costs): the producer hands the
//     tile descriptor and the tile's slot map to the consumers through the shared-memory item ring, a
//     warp's completion is ONE release red behind a warp meeting (cumulative over every lane's stores;
//     no __threadfence per thread), the K split's arrival counter one acq_rel atom, and groups of 8
//     padding slots get no fragment loads and no DMMAs (32 x 32 tiles).
//   * KS > 1 (last rounds, a handful of columns): KS warp groups split the k steps of every k-tile
//     and meet in shared memory; a tile's K loop is a latency chain, KS groups walk it KS steps at a
//     time.
#pragma once

#include <cuda.h>
#include <type_traits>

struct RoundParams {
  int n, m, nm, D;
  int M_pad;        // padded rows of one ladder level in Wb
  int split;        // padded row where the lambda block starts (0: dense layer)
  int k_tiles, k_tiles3;
  const int* cols;  // slot -> column (-1: padding slot)
  const TileDesc* tiles;  // the NON-EMPTY column tiles of BN slots: {first slot, ladder index} (BatchDev::ct)
  const int* n_tiles;
  const double* bias; int ld_bias;
  const double* lo; const double* hi; int ld_lohi;
  const double* negrho;  // [L][m]
  double* S[2];     // iterate in slot order, [slot][ld_s]
  int ld_s;
  int first;        // S[first] holds the iterate when the round starts
  int n_iters;
  int* work;        // item counter (zero at launch)
  int* done;        // [column tiles of BN slots] consumer-warp completions of this round (zero at launch)
  int* dbg;
  int num_sms;                // CTAs beyond ceil(items per iteration / num_sms) * num_sms retire at once (see the kernel)
  // Small rounds: the K loop of every (column tile, row tile) is split over `kx` work items (= CTAs on
  // different SMs); the splits leave their partial accumulators in `part`, and the LAST one to arrive (a
  // counter per tile and consumer warp in `tile_cnt`, zero at launch) adds them up in split order, so the sum
  // does not depend on who arrives when.  Used while the round has at most kx_max_tiles column tiles.
  int kx, kx_max_tiles;
  double* part;               // [kx_max_tiles * m_tiles][kx][BM * BN]
  int* tile_cnt;              // [kx_max_tiles * m_tiles][consumer warps of group 0]
  int flags;                  // debug switches (CQP_ROUND_FLAGS): 1 = TMA descriptors read from global memory, 2 = padding groups are not skipped
  const CUtensorMap* gmaps;   // [3] copies of the descriptors in global memory: A, S0, S1
};

__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acq_rel_gpu_add(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void named_barrier(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int kRoundQ = 4;  // depth of the producer -> consumer item ring
// ring entry: {item, first slot, ladder index, -, slot map of the tile's BN slots}
__host__ __device__ constexpr int round_ring_ints(int BN) { return 4 + BN; }

template <int BM, int BN, int WM, int WN, int ST, int KS>
constexpr int round_smem_bytes() {
  constexpr int MI = BM / WM / 8, NI = BN / WN / 8;
  return 1024 /* alignment slack: the 128-byte swizzle wants 1024-byte aligned tiles */ + ST * (BM + BN) * 128 +
         (KS > 1 ? (KS - 1) * WM * WN * 32 * MI * NI * 2 * 8 : 0) + 8 * (2 * ST + 2 * kRoundQ) + 4 * round_ring_ints(BN) * kRoundQ + 16;
}

template <int BM, int BN, int WM, int WN, int ST, int KS, int MINB>
__global__ void __launch_bounds__((WM * WN * KS + 1) * 32, MINB)
round_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapS0,
             const __grid_constant__ CUtensorMap mapS1, const RoundParams p) {
  constexpr int NW = WM * WN;    // warps of one k-split group
  constexpr int NCW = NW * KS;   // consumer warps; warp NCW is the producer
  constexpr int TM = BM / WM, TN = BN / WN, MI = TM / 8, NI = TN / 8;
  constexpr int A_BYTES = BM * 128, STAGE_BYTES = (BM + BN) * 128;
  constexpr int PER = MI * NI * 2;
  extern __shared__ unsigned char round_smem_raw[];
  // (pointer arithmetic on the shared array, not an integer round trip: the compiler keeps the
  // shared address space and emits LDS, not generic loads)
  unsigned char* base = round_smem_raw + ((1024u - (smem_u32(round_smem_raw) & 1023u)) & 1023u);
  double* red = reinterpret_cast<double*>(base + ST * STAGE_BYTES);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(red + (KS > 1 ? (KS - 1) * NW * 32 * PER : 0));
  unsigned long long* empty = full + ST;
  unsigned long long* sfull = empty + ST;
  unsigned long long* sempty = sfull + kRoundQ;
  int* item_s = reinterpret_cast<int*>(sempty + kRoundQ);
  constexpr int RING = round_ring_ints(BN);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m_tiles = p.M_pad / BM;
  const int n_ct = __ldcg(p.n_tiles);
  const int KX = (p.kx > 1 && n_ct <= p.kx_max_tiles) ? p.kx : 1;  // (the same value in every CTA)
  const int per_tile_col = m_tiles * KX;
  const int per_iter = n_ct * per_tile_col;
  const int total = per_iter * p.n_iters;
  // row tiles that hold rows at all (the others are padding between the two parts of the structured
  // layer and are skipped: they must not count as completions either, or the skipped tiles of LATER
  // iterations, which nothing holds back, would release an iteration early)
  int m_real = 0;
  for (int mt = 0; mt < m_tiles; ++mt) {
    const int m0 = mt * BM;
    const bool blk3 = p.split > 0 && m0 >= p.split;
    m_real += (blk3 ? m0 - p.split + p.nm : m0) < ((p.split > 0 && !blk3) ? p.nm : p.D) ? 1 : 0;
  }
  // Small rounds: no more CTAs than one iteration has items, rounded up to whole CTAs-per-SM layers.
  // Surplus CTAs would only hold items of later iterations, and the items that ARE runnable would land
  // on whatever CTAs happen to be free: several on one SM while other SMs idle (an item is bound by
  // its SM's DMMA pipe: 12 us for a 32 x 32 tile at D = 1500).  With one layer per SM the runnable
  // items spread evenly, as the block scheduler spreads a fresh launch.
  if (p.num_sms > 0 && (int)blockIdx.x >= ((per_iter + p.num_sms - 1) / p.num_sms) * p.num_sms && blockIdx.x >= (unsigned)p.num_sms) return;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCW); }
    for (int q = 0; q < kRoundQ; ++q) { mbar_init(&sfull[q], 1); mbar_init(&sempty[q], NCW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int q = 0, qph = 0;
  unsigned stage = 0, sph = 0;

  if (warp == NCW) {
    // ===== producer: item fetch, dependency wait, TMA issue =====
    if (lane != 0) return;
    for (;;) {
      const int item = atomicAdd(p.work, 1);
      // the consumers learn about the item only once its inputs are complete: they read S too (the
      // diagonal terms of the lambda rows)
      TileDesc td;
      td.slot0 = 0; td.a_index = 0;
      // (the tile descriptor and the tile's slot map ride along: the consumers' bias loads then do not
      // wait behind two more dependent round trips to L2; the producer fetches them while it waits for
      // the item's inputs anyway)
      bool have_slot = false;
      auto take_slot = [&]() {
        if (!have_slot) mbar_wait(&sempty[q], qph ^ 1, p.dbg, 20, item);
        have_slot = true;
      };
      auto hand_over = [&](int value) {
        take_slot();
        int* ring = item_s + q * RING;
        ring[0] = value;
        ring[1] = td.slot0;
        ring[2] = td.a_index;
        mbar_arrive(&sfull[q]);
        have_slot = false;
        if (++q == kRoundQ) { q = 0; qph ^= 1; }
      };
      if (item >= total) { hand_over(-1); break; }
      const int it = item / per_iter, r = item - it * per_iter;
      const int ns = r / per_tile_col, r2 = r - ns * per_tile_col;
      const int mt = r2 / KX, kx = r2 - mt * KX;
      td.slot0 = __ldcg(&p.tiles[ns].slot0);
      td.a_index = __ldcg(&p.tiles[ns].a_index);
      const int slot0 = td.slot0;
      const int m0 = mt * BM;
      const bool blk3 = p.split > 0 && m0 >= p.split;
      const int row0 = blk3 ? m0 - p.split + p.nm : m0;
      const int row_end = (p.split > 0 && !blk3) ? p.nm : p.D;
      if (row0 >= row_end) { hand_over(item); continue; }  // row tile of padding only: the consumers skip it too
      {
        take_slot();
        int4* ring_cols = reinterpret_cast<int4*>(item_s + q * RING + 4);
        const int4* src = reinterpret_cast<const int4*>(p.cols + slot0);
#pragma unroll
        for (int i = 0; i < BN / 4; ++i) ring_cols[i] = __ldcg(src + i);
      }
      if (it > 0) {
        const int need = it * m_real * NW;
        long long t0 = 0;
        unsigned spins = 0;
        while (ld_acquire_gpu(p.done + ns) < need) {
          if ((++spins & 0x3FF) == 0) {
            if (t0 == 0) t0 = clock64();
            else if (clock64() - t0 > kSpinLimitCycles) watchdog_fire(p.dbg, 21, item);
          }
        }
        fence_proxy_async();  // the generic-proxy stores just acquired, before the async-proxy reads below
      }
      hand_over(item);
      const CUtensorMap* mapS = ((p.first ^ it) & 1) ? &mapS1 : &mapS0;
      const CUtensorMap* mapAp = &mapA;
      if (p.flags & 1) { mapAp = p.gmaps; mapS = p.gmaps + 1 + ((p.first ^ it) & 1); }
      const int a_row = td.a_index * p.M_pad + m0;
      const int k_tiles = blk3 ? p.k_tiles3 : p.k_tiles;
      const int kt_per = (k_tiles + KX - 1) / KX;
      const int kt0 = kx * kt_per, kt1 = min(k_tiles, kt0 + kt_per);  // this split's k-tiles
      for (int kt = kt0; kt < kt1; ++kt) {
        mbar_wait(&empty[stage], (int)(sph ^ 1u), p.dbg, 22, item);
        mbar_expect_tx(&full[stage], STAGE_BYTES);
        const unsigned dst = smem_u32(base + stage * STAGE_BYTES);
        tma_load_2d(dst, mapAp, kt * 16, a_row, smem_u32(&full[stage]));
        tma_load_2d(dst + A_BYTES, mapS, kt * 16, slot0, smem_u32(&full[stage]));
        if (++stage == (unsigned)ST) { stage = 0; sph ^= 1u; }
      }
    }
    return;
  }

  // ===== consumers =====
  const int g = lane >> 2, t4 = lane & 3;
  const int kg = warp / NW, warp_in = warp - kg * NW;
  const int warp_m = warp_in % WM, warp_n = warp_in / WM;
  const int pg = ((g & 3) << 1) | (g >> 2);  // tile row-in-8 of fragment row g (see the header)
  // tile column-in-8 of the C fragment's columns 2 t4, 2 t4 + 1
  const int pc0 = (((2 * t4) & 3) << 1) | ((2 * t4) >> 2), pc1 = (((2 * t4 + 1) & 3) << 1) | ((2 * t4 + 1) >> 2);
  for (;;) {
    mbar_wait(&sfull[q], qph, p.dbg, 23, 0);
    const int* ring = item_s + q * RING;
    const int item = ring[0];
    TileDesc td;
    td.slot0 = ring[1];
    td.a_index = ring[2];
    int colv[NI][2];  // this thread's columns (slot map of the tile, from the ring)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      colv[ni][0] = ring[4 + warp_n * TN + ni * 8 + pc0];
      colv[ni][1] = ring[4 + warp_n * TN + ni * 8 + pc1];
    }
    __syncwarp();
    if (item < 0) break;  // (the branch needs the loaded value: the slot is released only after the reads returned)
    // (the values read above feed address arithmetic below, so the loads have returned before the release)
    __syncwarp();
    if (lane == 0) mbar_arrive(&sempty[q]);
    if (++q == kRoundQ) { q = 0; qph ^= 1; }
    const int it = item / per_iter, r = item - it * per_iter;
    const int ns = r / per_tile_col, r2 = r - ns * per_tile_col;
    const int mt = r2 / KX, kx = r2 - mt * KX;
    const int slot0 = td.slot0;
    const int m0 = mt * BM;
    const bool blk3 = p.split > 0 && m0 >= p.split;
    const int row0 = blk3 ? m0 - p.split + p.nm : m0;
    const int row_end = (p.split > 0 && !blk3) ? p.nm : p.D;
    bool finalize = true;  // this warp writes the tile (always, unless the K loop is split over CTAs)
    if (row0 < row_end) {
      const int k_tiles_all = blk3 ? p.k_tiles3 : p.k_tiles;
      const int kt_per = (k_tiles_all + KX - 1) / KX;
      const int kt0 = kx * kt_per;
      const int k_tiles = max(0, min(k_tiles_all, kt0 + kt_per) - kt0);  // this split's k-tiles
      const double* Sin = p.S[(p.first ^ it) & 1];
      double* Sout = p.S[(p.first ^ it ^ 1) & 1];
      // Accumulators start from the bias (rows < n + m) or from the two diagonal terms of a lambda row,
      // -rho_i z_i + lambda_i (blocks (3,2), (3,3) of W, layers.cpp:159-161); the loads overlap the
      // first stages.  S is read with ld.cg: these addresses are rewritten every other iteration.
      double acc[MI][NI][2];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int cs = slot0 + warp_n * TN + ni * 8 + (j ? pc1 : pc0);
          const int col = colv[ni][j];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            const int row = row0 + warp_m * TM + mi * 8 + pg;
            double init = 0.0;
            if (col >= 0 && kg == 0 && kx == 0) {
              if (row < p.nm) {
                init = __ldcg(p.bias + (size_t)col * p.ld_bias + row);
              } else if (blk3 && row < p.D) {
                const double* v = Sin + (size_t)cs * p.ld_s;
                const int i = row - p.nm;
                init = fma(p.negrho[(size_t)td.a_index * p.m + i], __ldcg(v + p.n + i), __ldcg(v + row));
              }
            }
            acc[mi][ni][j] = init;
          }
        }
      }
      // Stage release discipline: a stage goes back to the TMA producer only once the DMMAs that consume
      // its fragment loads have been ISSUED (an issued DMMA has its operands, so the loads have
      // returned).  Program order alone does not give that: ptxas moves the arrive up, right behind
      // the last (still in flight) LDS and ahead of the DMMAs (seen in SASS; the refill then raced with
      // that load: wrong ni = last fragment).  So the arrive for k-tile kt sits behind the full-wait
      // loop of k-tile kt + 1, and the last one behind the epilogue's fence / the reduction barrier.
      // Partially filled column tiles (the last tile of every ladder level; in the late rounds every tile):
      // a group of 8 slots that holds padding only gets no fragment loads and no DMMAs.  Its accumulators
      // stay at their initial 0, which is what W 0 adds up to, and the columns that are there see the same
      // products in the same order: bit-identical, and the SM's DMMA pipe (what bounds an item) is busy for
      // the occupied groups only.  The stage waits and releases are kept, so the pipeline protocol is the same.
      // (The 32 x 32 configurations only: they serve the rounds below 800 columns, where the partial tiles
      // are a visible share; the large tiles keep their schedule.)
      constexpr bool SKIP = (BM == 32 && BN == 32);
      unsigned act = (1u << NI) - 1u;
      if (SKIP && !(p.flags & 2)) {  // (CQP_ROUND_FLAGS=2: A/B switch, no skipping)
        act = 0;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
          act |= __any_sync(0xffffffffu, colv[ni][0] >= 0 || colv[ni][1] >= 0) ? (1u << ni) : 0u;
      }
      int held = -1;
      auto k_loop = [&](auto guard) {
        constexpr bool GUARD = decltype(guard)::value;
        for (int kt = 0; kt < k_tiles; ++kt) {
          mbar_wait(&full[stage], (int)sph, p.dbg, 24, item);
          if (held >= 0 && lane == 0) mbar_arrive(&empty[held]);
          if (!GUARD || act != 0) {
            const double* as = reinterpret_cast<const double*>(base + stage * STAGE_BYTES) + (warp_m * TM + pg) * 16;
            const double* bs = reinterpret_cast<const double*>(base + stage * STAGE_BYTES + A_BYTES) + (warp_n * TN + pg) * 16;
            double a[MI], b[NI];
#pragma unroll
            for (int ks0 = 0; ks0 < 4; ks0 += KS) {
              const int ks = ks0 + kg;
              const int e = ks * 4 + t4;
              const int off = (((e >> 1) ^ pg) << 1) | (e & 1);
#pragma unroll
              for (int mi = 0; mi < MI; ++mi) a[mi] = as[mi * 128 + off];
#pragma unroll
              for (int ni = 0; ni < NI; ++ni)
                if (!GUARD || ((act >> ni) & 1u)) b[ni] = bs[ni * 128 + off];
#pragma unroll
              for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
                  if (!GUARD || ((act >> ni) & 1u)) dmma884(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
            }
          }
          held = (int)stage;
          if (++stage == (unsigned)ST) { stage = 0; sph ^= 1u; }
        }
      };
      if (!SKIP || act == (1u << NI) - 1u) k_loop(std::false_type{});
      else k_loop(std::true_type{});
      if (KS > 1) {
        // partial accumulators of groups 1 .. KS-1 meet in `red`; group 0 adds them in group order
        named_barrier(1, NCW * 32);  // the previous item's readers of `red` are done
        if (kg > 0) {
          double* mine = red + ((size_t)(kg - 1) * (NW * 32) + warp_in * 32 + lane) * PER;
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              mine[(mi * NI + ni) * 2] = acc[mi][ni][0];
              mine[(mi * NI + ni) * 2 + 1] = acc[mi][ni][1];
            }
        }
        named_barrier(1, NCW * 32);
        if (kg == 0) {
#pragma unroll
          for (int qq = 1; qq < KS; ++qq) {
            const double* theirs = red + ((size_t)(qq - 1) * (NW * 32) + warp_in * 32 + lane) * PER;
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
      if (KX > 1 && kg == 0) {
        // K split over CTAs: leave this split's partial tile in global memory; the last split to arrive
        // (per consumer warp) adds all of them up in split order and goes on to the epilogue
        const size_t tile = (size_t)ns * m_tiles + mt;
        double* mine = p.part + ((tile * KX + kx) * NW + warp_in) * (32 * PER) + lane;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            __stcg(mine + ((mi * NI + ni) * 2) * 32, acc[mi][ni][0]);
            __stcg(mine + ((mi * NI + ni) * 2 + 1) * 32, acc[mi][ni][1]);
          }
        // the warp meets, lane 0 counts the arrival with an acq_rel atom (release: cumulative over every lane's
        // partial stores; acquire: the last arriver's re-reads below, behind the second meeting, see all splits)
        __syncwarp();
        int old = 0;
        if (lane == 0) old = atom_acq_rel_gpu_add(p.tile_cnt + tile * NW + warp_in, 1);
        old = __shfl_sync(0xffffffffu, old, 0);
        finalize = ((old + 1) % KX) == 0;  // (KX arrivals per iteration; iterations of a column tile do not overlap)
        if (finalize) {
          __syncwarp();
          for (int q2 = 0; q2 < KX; ++q2) {
            const double* theirs = p.part + ((tile * KX + q2) * NW + warp_in) * (32 * PER) + lane;
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) {
                const double v0 = __ldcg(theirs + ((mi * NI + ni) * 2) * 32);
                const double v1 = __ldcg(theirs + ((mi * NI + ni) * 2 + 1) * 32);
                acc[mi][ni][0] = q2 == 0 ? v0 : acc[mi][ni][0] + v0;
                acc[mi][ni][1] = q2 == 0 ? v1 : acc[mi][ni][1] + v1;
              }
          }
        }
      }
      if (kg == 0 && finalize) {
        // epilogue: clamp the z rows (solver.cpp:62), store in slot order.  Padding slots hold zeros
        // and stay zero (no bias, W 0 = 0).
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int cs = slot0 + warp_n * TN + ni * 8 + (j ? pc1 : pc0);
            const int col = colv[ni][j];
            double* crow = Sout + (size_t)cs * p.ld_s;
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              const int row = row0 + warp_m * TM + mi * 8 + pg;
              if (row >= row_end) continue;
              double v = acc[mi][ni][j];
              if (col >= 0 && row >= p.n && row < p.nm) {
                const double lo = __ldcg(p.lo + (size_t)col * p.ld_lohi + row - p.n);
                const double hi = __ldcg(p.hi + (size_t)col * p.ld_lohi + row - p.n);
                v = v < lo ? lo : v;
                v = v > hi ? hi : v;
              }
              crow[row] = v;
            }
          }
        }
        // The stores become visible device-wide through the release of the warp's completion count below
        // (the warp meets first, so lane 0's release is cumulative over every lane's stores: the usual
        // "all store, barrier, one thread releases" pattern; a __threadfence per thread here and another one
        // in front of the red cost 0.5 us per iteration each in the small rounds).  The proxy fence orders
        // them for the async proxy: other CTAs read them with TMA.
        fence_proxy_async();
      }
      // the item's last stage (see the release discipline above): behind the fence (group 0) or behind the
      // reduction barrier, whose shared-memory stores carry the accumulators (groups > 0)
      if (held >= 0 && lane == 0) mbar_arrive(&empty[held]);
    }
    // one completion per consumer warp of group 0: the producer of the next iteration waits for
    // m_real * NW of them per column tile
    if (kg == 0 && row0 < row_end && finalize) {
      __syncwarp();
      if (lane == 0) red_release_gpu_add(p.done + ns, 1);
    }
  }
}
