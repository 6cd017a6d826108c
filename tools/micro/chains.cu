// Random dependent 8 B reads over 2 GiB: throughput vs independent chains per thread
// and threads per SM (how much memory-level parallelism the list walk needs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int C>
__global__ void rd(const uint2* __restrict__ a, uint32_t mask, uint32_t iters, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = hsh(t * C + c);
  for (uint32_t i = 0; i < iters; ++i) {
    uint2 v[C];
#pragma unroll
    for (int c = 0; c < C; ++c) asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v[c].x), "=r"(v[c].y) : "l"(a + (x[c] & mask)));
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = hsh(x[c] + v[c].y);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) acc += x[c];
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  const size_t n = 1ull << 28;
  uint2* a; uint32_t* o;
  cudaMalloc(&a, n * 8); cudaMalloc(&o, 4); cudaMemset(a, 1, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int C, int blocks, int threads) {
    uint32_t iters = (uint32_t)(((size_t)1 << 27) / ((size_t)blocks * threads * C));
    kern<<<blocks, threads>>>(a, (uint32_t)(n - 1), iters, o);
    cudaEventRecord(e0); kern<<<blocks, threads>>>(a, (uint32_t)(n - 1), iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double acc = (double)blocks * threads * C * iters;
    printf("chains/thread %d  threads %7d  %7.3f ms  %6.2f G acc/s  %5.2f TB/s@128B\n", C, blocks * threads, ms, acc / ms / 1e6, acc * 128 / ms / 1e9);
  };
  for (int bps : {2, 4, 8}) {
    run(rd<1>, 1, 148 * bps, 256); run(rd<2>, 2, 148 * bps, 256); run(rd<4>, 4, 148 * bps, 256); run(rd<8>, 8, 148 * bps, 256);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
