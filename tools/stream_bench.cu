// Micro-benchmark (GPU box): how fast can 148 persistent CTAs stream a D x D FP64 matrix (row
// slices of R rows per CTA) from HBM through a shared-memory ring with cp.async.bulk?
//   mode 0: stage = 16 rows x 2 KB segments (row-major W, 16 bulk copies per 32 KB stage)
//   mode 1: stage = ONE contiguous 32 KB bulk copy (W re-tiled per CTA in HBM)
//   mode 2: stage = 4 rows x 8 KB segments
// Consumers (16 warps) read every byte of the stage from shared memory (LDS.128 + 2 DFMA).
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kStageBytes = 32768;
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  long long t0 = clock64();
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (!ok && clock64() - t0 > 4000000000ll) __trap();
  } while (!ok);
}

template <int MODE>
__global__ void __launch_bounds__(544, 1) stream(const double* __restrict__ W, size_t row_doubles, int rows_per_cta,
                                                 int NS, int reps, double* sink) {
  extern __shared__ __align__(128) unsigned char raw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(raw);
  unsigned long long* empty = full + 8;
  double* ring = reinterpret_cast<double*>(raw + 128);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) {
    for (int k = 0; k < NS; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[k])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(smem_u32(&empty[k])) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t slice_bytes = (size_t)rows_per_cta * row_doubles * 8;
  const int chunks = (int)(slice_bytes / kStageBytes);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(W) + (size_t)blockIdx.x * slice_bytes;
  unsigned cnt = 0;
  double acc = 0.0;
  long long prof[4] = {0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    if (warp == 16) {  // producer
      for (int c = 0; c < chunks; ++c, ++cnt) {
        const unsigned stage = cnt % NS, ph = (cnt / NS) & 1;
        const long long c0 = clock64();
        mbar_wait(&empty[stage], ph ^ 1);
        const long long c1 = clock64();
        if (lane == 0)
          asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(smem_u32(&full[stage])), "r"(kStageBytes) : "memory");
        __syncwarp();
        const long long c2 = clock64();
        const unsigned dst0 = smem_u32(ring) + stage * kStageBytes;
        if (MODE == 1) {
          if (lane == 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst0), "l"(base + (size_t)c * kStageBytes), "r"(kStageBytes), "r"(smem_u32(&full[stage])) : "memory");
          const long long c3 = clock64();
          if (lane == 0 && blockIdx.x == 0 && sink) { prof[0] += c1 - c0; prof[1] += c2 - c1; prof[2] += c3 - c2; prof[3] += 1; }
        } else {
          // row-major slice: rows of row_doubles*8 bytes; a stage covers NR rows x SEG bytes
          constexpr int NR = MODE == 0 ? 16 : 4, SEG = kStageBytes / NR;
          const size_t row_bytes = row_doubles * 8;
          const int segs_per_row = (int)(row_bytes / SEG);
          const int rb = c / segs_per_row, sc = c - rb * segs_per_row;  // row block, segment column
          if (lane < NR)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst0 + lane * SEG), "l"(base + ((size_t)rb * NR + lane) * row_bytes + (size_t)sc * SEG), "r"(SEG), "r"(smem_u32(&full[stage])) : "memory");
        }
      }
    } else {
      for (int c = 0; c < chunks; ++c, ++cnt) {
        const unsigned stage = cnt % NS, ph = (cnt / NS) & 1;
        mbar_wait(&full[stage], ph);
        const double2* st = reinterpret_cast<const double2*>(ring + (size_t)stage * (kStageBytes / 8));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double2 w = st[j * 512 + t];
          acc = fma(w.x, 1.0000001, acc);
          acc = fma(w.y, 0.9999999, acc);
        }
        __syncwarp();
        if (lane == 0) asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_u32(&empty[stage])) : "memory");
      }
    }
  }
  if (acc == 1.2345) sink[0] = acc;
  if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 16 * 32 && prof[3] > 0)
    printf("    producer per chunk: wait(empty) %lld, expect_tx %lld, bulk issue %lld cycles (%lld chunks)\n",
           prof[0] / prof[3], prof[1] / prof[3], prof[2] / prof[3], prof[3]);
}

template <int MODE>
void run(const double* W, int D, int R, int G, int NS, const char* name, double* sink) {
  const size_t smem = 128 + (size_t)NS * kStageBytes;
  cudaFuncSetAttribute(stream<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 20;
  stream<MODE><<<G, 544, smem>>>(W, (size_t)D, R, NS, 2, sink);
  cudaEventRecord(e0);
  stream<MODE><<<G, 544, smem>>>(W, (size_t)D, R, NS, reps, sink);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)G * R * D * 8 * reps;
  printf("%-34s D=%d R=%d G=%d stages=%d : %7.1f GB/s  (%s)\n", name, D, R, G, NS, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
  fflush(stdout);
}

int main() {
  const int D = 4096, G = 148, R = 28;  // 148 x 28 rows x 32 KB = 136 MB per sweep (> L2)
  double* W; double* sink;
  cudaMalloc(&W, (size_t)G * R * D * 8);
  cudaMemset(W, 0, (size_t)G * R * D * 8);
  cudaMalloc(&sink, 8);
  for (int NS : {2, 4, 6}) {
    run<0>(W, D, R, G, NS, "16 rows x 2 KB per stage", sink);
    run<2>(W, D, R, G, NS, "4 rows x 8 KB per stage", sink);
    run<1>(W, D, R, G, NS, "one contiguous 32 KB per stage", sink);
  }
  // L2-resident case: 54 MB (Atlas-sized level)
  const int R2 = 11;
  for (int NS : {4, 6}) {
    run<0>(W, D, R2, G, NS, "L2-resident, 16 rows x 2 KB", sink);
    run<1>(W, D, R2, G, NS, "L2-resident, contiguous 32 KB", sink);
  }
  return 0;
}
