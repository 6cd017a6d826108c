// Unstable in-warp slot assignment by shared-memory atomics (warp-private counters,
// random 8-bit digits) vs the stable 8-ballot peer mask.  Warp-ranks per second.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int MODE>
__global__ void k(uint32_t iters, uint32_t* out) {
  __shared__ uint32_t cnt[8][256];
  uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, acc = 0;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t x = hsh(threadIdx.x + blockIdx.x * 977);
  for (uint32_t i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t d = x >> 24;
    if (MODE == 0) acc += atomicAdd(&cnt[w][d], 1u);
    else {
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b)
        asm volatile("{ .reg .pred p; .reg .b32 t, bb, s;\n and.b32 t, %1, %2;\n setp.ne.u32 p, t, 0;\n"
                     " vote.sync.ballot.b32 bb, p, 0xffffffff;\n selp.b32 s, 0, 0xffffffff, p;\n"
                     " lop3.b32 %0, %0, bb, s, 0x60; }" : "+r"(peers) : "r"(d), "r"(1u << b));
      acc += __popc(peers & ((1u << lane) - 1));
    }
  }
  if (acc == 0x7777777) out[0] = acc;
}
int main() {
  uint32_t* o; cudaMalloc(&o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint32_t iters = 4096; const int blocks = 148 * 4, threads = 256;
  for (int mode = 0; mode < 2; ++mode) {
    auto f = mode == 0 ? k<0> : k<1>;
    f<<<blocks, threads>>>(iters, o);
    cudaEventRecord(e0); f<<<blocks, threads>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-8s %7.3f ms  %6.1f G warp-ranks/s\n", mode ? "ballot8" : "atoms", ms, (double)blocks * threads / 32 * iters / ms / 1e6);
  }
}
