// Scratch (GPU box): how long does __nanosleep(d) really sleep?  One warp per CTA, 148 CTAs, 200 samples.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int d, long long* out) {
  long long best = 1ll << 60, worst = 0, sum = 0;
  for (int i = 0; i < 200; ++i) {
    long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    __nanosleep(d);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    long long dt = t1 - t0;
    best = dt < best ? dt : best; worst = dt > worst ? dt : worst; sum += dt;
  }
  if (threadIdx.x == 0) { out[blockIdx.x * 3] = best; out[blockIdx.x * 3 + 1] = worst; out[blockIdx.x * 3 + 2] = sum / 200; }
}
__global__ void kc(int d, long long* out) {  // same with clock64
  long long best = 1ll << 60, worst = 0, sum = 0;
  for (int i = 0; i < 200; ++i) {
    long long t0 = clock64();
    __nanosleep(d);
    long long dt = clock64() - t0;
    best = dt < best ? dt : best; worst = dt > worst ? dt : worst; sum += dt;
  }
  if (threadIdx.x == 0) { out[blockIdx.x * 3] = best; out[blockIdx.x * 3 + 1] = worst; out[blockIdx.x * 3 + 2] = sum / 200; }
}
int main() {
  long long* o; cudaMallocManaged(&o, 148 * 3 * sizeof(long long));
  for (int d : {0, 20, 50, 100, 150, 200, 300, 400, 600, 1000}) {
    kc<<<148, 32>>>(d, o); cudaDeviceSynchronize();
    long long b = 1ll << 60, w = 0, s = 0;
    for (int i = 0; i < 148; ++i) { b = o[3*i] < b ? o[3*i] : b; w = o[3*i+1] > w ? o[3*i+1] : w; s += o[3*i+2]; }
    printf("nanosleep(%4d): clock64 cycles min %lld max %lld mean %lld  (= %.0f / %.0f / %.0f ns at 1.965 GHz)\n", d, b, w, s / 148, b / 1.965, w / 1.965, s / 148 / 1.965);
  }
  k<<<148, 32>>>(200, o); cudaDeviceSynchronize();
  printf("globaltimer resolution check: nanosleep(200) min %lld max %lld mean %lld ns\n", o[0], o[1], o[2]);
  return 0;
}
