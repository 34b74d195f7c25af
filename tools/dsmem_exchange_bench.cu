// Micro-benchmark (GPU box): cost of the per-iteration all-to-all of the iterate inside ONE
// thread-block cluster, for the exchange patterns considered for cqp_cluster.cu.  Every CTA owns R
// values per iteration and must deliver them to all C CTAs; an iteration may start once all C*R
// values have arrived (mbarrier tx count).  No arithmetic: this is the exchange floor.
//   mode 0: st.async 8 B per (row, peer)                      [C*R packets + complete_tx per CTA]
//   mode 1: st.async.v2 16 B per (row pair, peer)
//   mode 2: rows -> local staging, named barrier, ONE cp.async.bulk per peer (R*8 bytes)
//   mode 3: like 1, plus 20 dependent DFMAs + 4-level butterfly per row (compute stand-in)
//   mode 4: plain st.shared::cluster 8 B, data-as-flag: 4-slot ring, consumers poll their LOCAL copy
//           for non-sentinel values, the owner re-arms slot (i+2)&3 remotely + fence.acq_rel.cluster
//   mode 5: mode 4 plus the compute stand-in
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o dsmem_bench tools/dsmem_exchange_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void arm(unsigned long long* bar, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(unsigned long long* bar, int parity) {
  unsigned ok;
  long long t0 = clock64();
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (!ok && clock64() - t0 > 2000000000ll) __trap();  // ~1 s: a protocol bug must not hang the box
  } while (!ok);
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(int R, int iters, int active_rows_per_warp, long long* out, double* sink) {
  extern __shared__ __align__(16) unsigned char raw[];
  const int C = gridDim.x;
  const int D = C * R;
  double* xs = reinterpret_cast<double*>(raw);                       // [2][D]
  double* stage = xs + 4 * D;                                         // [2][R]   (xs: up to 4 slots)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(stage + 2 * R);  // xready[2]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (t == 0) {
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    arm(&bars[0], 8u * D);
    arm(&bars[1], 8u * D);
  }
  for (int i = t; i < 4 * D; i += 512) xs[i] = (MODE >= 4 && i >= D) ? __longlong_as_double(-1ll) : 1.0;
  __syncthreads();
  csync();
  const int RW = active_rows_per_warp;          // rows per warp (2 or 4), even
  const int nwarps = (R + RW - 1) / RW;         // active warps
  const bool active = warp < nwarps;
  const int r0 = warp * RW;
  const unsigned xs_a = smem_u32(xs), bar_a = smem_u32(&bars[0]);
  long long t0 = 0;
  double acc = 0.0;
  for (int i = 1; i <= iters; ++i) {
    const int b = i & 1;
    if (i == 101 && t == 0) t0 = clock64();
    if (MODE >= 4) {
      if (!active) continue;
      // poll v_{i-1} in the local slot (i-1)&3: lane covers pairs lane, lane + 32, ...
      const double* src = xs + ((i - 1) & 3) * D;
      double v = 0.0;
      long long w0 = clock64();
      for (int c2 = lane; c2 < D / 2; c2 += 32) {
        double a, bb;
        do {
          asm volatile("ld.relaxed.cluster.shared::cta.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(bb) : "r"(smem_u32(src + 2 * c2)) : "memory");
          if (clock64() - w0 > 2000000000ll) __trap();
        } while (__double_as_longlong(a) == -1ll || __double_as_longlong(bb) == -1ll);
        v += a + bb;
      }
      if (MODE == 5) {
        double a0 = v, a1 = v;
#pragma unroll
        for (int k = 0; k < 10; ++k) { a0 = fma(a0, 0.999, v); a1 = fma(a1, 0.998, v); }
        v = a0 + a1;
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
        v *= 1e-3;
      }
      v = v * 1e-9 + 1.0;
      acc += v;
      const unsigned peer = lane & (C - 1);
      const int step = 32 / C;
      for (int r = lane / C; r < RW && r0 + r < R; r += step) {
        const unsigned off = 8u * (rank * R + r0 + r);
        asm volatile("st.relaxed.cluster.shared::cluster.f64 [%0], %1;" ::"r"(mapa(xs_a + 8u * ((i & 3) * D) + off, peer)), "d"(v) : "memory");
      }
      for (int r = lane / C; r < RW && r0 + r < R; r += step) {
        const unsigned off = 8u * (rank * R + r0 + r);
        asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(mapa(xs_a + 8u * (((i + 2) & 3) * D) + off, peer)), "l"(-1ll) : "memory");
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      continue;
    }
    if (i > 1 && active) {
      wait(&bars[b ^ 1], ((i - 2) >> 1) & 1);
      if (t == 0) arm(&bars[b ^ 1], 8u * D);
    }
    if (!active) continue;
    double v = xs[(b ^ 1) * D + ((lane + i) % D)];
    if (MODE == 3) {
      double a0 = v, a1 = v;
#pragma unroll
      for (int k = 0; k < 10; ++k) { a0 = fma(a0, 0.999, v); a1 = fma(a1, 0.998, v); }
      v = a0 + a1;
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
      v *= 1e-3;
    }
    acc += v;
    if (MODE == 0) {
      // lane -> (peer = lane & 15, row slot = lane >> 4), rows r0 + slot, r0 + slot + 2, ...
      const unsigned peer = lane & (C - 1);
      const int step = 32 / C;
      for (int r = lane / C; r < RW && r0 + r < R; r += step) {
        const unsigned dst = mapa(xs_a + 8u * (b * D + rank * R + r0 + r), peer);
        const unsigned bd = mapa(bar_a + 8u * b, peer);
        asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(dst), "l"(__double_as_longlong(v)), "r"(bd) : "memory");
      }
    } else if (MODE == 1 || MODE == 3) {
      // lane -> (peer = lane & 15, pair slot = lane >> 4): 16-byte pushes of row pairs
      const unsigned peer = lane & (C - 1);
      const int step = 32 / C;
      for (int pr = lane / C; 2 * pr < RW && r0 + 2 * pr < R; pr += step) {
        const unsigned dst = mapa(xs_a + 8u * (b * D + rank * R + r0 + 2 * pr), peer);
        const unsigned bd = mapa(bar_a + 8u * b, peer);
        asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(dst), "l"(__double_as_longlong(v)), "l"(__double_as_longlong(v + 1.0)), "r"(bd) : "memory");
      }
    } else if (MODE == 2) {
      if (lane < RW && r0 + lane < R) stage[b * R + r0 + lane] = v;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(nwarps * 32) : "memory");
      if (warp == 0 && lane < C) {
        const unsigned dst = mapa(xs_a + 8u * (b * D + rank * R), (unsigned)lane);
        const unsigned bd = mapa(bar_a + 8u * b, (unsigned)lane);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "r"(smem_u32(stage + b * R)), "r"(8u * R), "r"(bd) : "memory");
      }
    }
  }
  if (active && MODE < 4) wait(&bars[iters & 1], ((iters - 1) >> 1) & 1);
  if (t == 0 && rank == 0) out[0] = clock64() - t0;
  if (acc == 123.456) sink[0] = acc;
  __syncthreads();
  csync();
}

template <int MODE>
void run(int C, int R, int RW, const char* name) {
  long long* out;
  double* sink;
  cudaMallocManaged(&out, 8);
  cudaMalloc(&sink, 8);
  const int iters = 2100;
  const size_t smem = sizeof(double) * (4 * C * R + 2 * R) + 64;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  printf("%-28s C=%2d R=%2d rows/warp=%d : ", name, C, R, RW);
  fflush(stdout);
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, bench<MODE>, R, iters, RW, out, sink);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s\n", cudaGetErrorString(e));
      fflush(stdout);
      exit(1);
    }
  }
  printf("%7.1f cycles/iteration\n", (double)out[0] / (iters - 100));
  fflush(stdout);
  cudaFree(out);
  cudaFree(sink);
}

int main() {
  for (int C : {16, 8}) {
    for (int R : {20, 40}) {
      for (int RW : {2, 4}) {
        if ((R + RW - 1) / RW > 16) continue;
        run<0>(C, R, RW, "st.async 8B");
        run<1>(C, R, RW, "st.async.v2 16B");
        run<2>(C, R, RW, "stage + cp.async.bulk");
        run<3>(C, R, RW, "v2 + fma/butterfly stand-in");
        run<4>(C, R, RW, "plain st + local poll");
        run<5>(C, R, RW, "plain st + poll + stand-in");
      }
    }
  }
  return 0;
}
