// Do conflicting lanes of one shared-memory atomicAdd instruction receive old values in
// ascending lane order?  Counts violations over many random trials.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void k(uint32_t iters, uint32_t nbins, unsigned long long* bad, unsigned long long* checks) {
  __shared__ uint32_t cnt[8][256];
  uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t x = hsh(threadIdx.x * 7919 + blockIdx.x * 977);
  unsigned long long nb = 0, nc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x = hsh(x + i);
    uint32_t d = x % nbins;
    uint32_t old = atomicAdd(&cnt[w][d], 1u);
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t lower = peers & ((1u << lane) - 1);
    // stable order <=> old == (value before the instruction) + popc(lower)
    uint32_t leader = __ffs(peers) - 1;
    uint32_t base = __shfl_sync(0xffffffffu, old, leader);  // leader's old is the minimum if ordered
    nb += (old != base + __popc(lower));
    nc += 1;
  }
  atomicAdd(bad, nb); atomicAdd(checks, nc);
}
int main() {
  unsigned long long *b, *c; cudaMalloc(&b, 8); cudaMalloc(&c, 8);
  for (uint32_t nbins : {2u, 4u, 16u, 256u}) {
    cudaMemset(b, 0, 8); cudaMemset(c, 0, 8);
    k<<<148 * 4, 256>>>(2000, nbins, b, c);
    unsigned long long hb, hc; cudaMemcpy(&hb, b, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("bins %3u: %llu of %llu lane results out of lane order\n", nbins, hb, hc);
  }
}
