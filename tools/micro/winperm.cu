// Microbenchmark: the relink's apply without shared-memory windows.  2^28 (v, succ) pairs,
// grouped by window of 2^wl ids (as an MSD partition level would leave them), applied by
// plain random 4 B global stores.  Unlike winstore.cu the targets are a PERMUTATION inside
// each window (every out_next word is written exactly once, as in the real relink), so a
// line that stays in L2 until all its words are written can leave as full sectors with no
// fill read.  Time per window size; run under ncu for the DRAM bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void mkpairs(uint2* pairs, uint32_t n, uint32_t wlog2) {
  const uint32_t mask = (1u << wlog2) - 1;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t win = p >> wlog2;
    const uint32_t off = ((p & mask) * 0x9E3779B1u + 0x5bd1e995u) & mask;  // bijection on the window
    pairs[p] = make_uint2((win << wlog2) | off, p);
  }
}
__global__ void apply(const uint2* __restrict__ pairs, uint32_t n, uint32_t* out) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint2 x = __ldcs(pairs + p);
    out[x.x] = x.y;
  }
}
// tile-ordered: CTA i takes pair tiles i, i + grid, ... (4096 pairs per tile), so the
// active targets at any time lie in the windows of ~grid consecutive tiles
__global__ void apply_tiles(const uint2* __restrict__ pairs, uint32_t n, uint32_t* out) {
  for (uint32_t t0 = blockIdx.x * 4096u; t0 < n; t0 += gridDim.x * 4096u)
    for (uint32_t j = threadIdx.x; j < 4096u && t0 + j < n; j += blockDim.x) {
      const uint2 x = __ldcs(pairs + t0 + j);
      out[x.x] = x.y;
    }
}
int main() {
  const uint32_t n = 1u << 28;
  uint2* pairs; uint32_t* out;
  cudaMalloc(&pairs, (size_t)n * 8); cudaMalloc(&out, (size_t)n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (uint32_t wl : {14u, 18u, 20u, 21u, 22u, 23u, 24u, 28u}) {
    mkpairs<<<1184, 256>>>(pairs, n, wl);
    for (int k = 0; k < 2; ++k) {
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (k == 0) apply<<<148 * 8, 256>>>(pairs, n, out); else apply_tiles<<<148 * 4, 512>>>(pairs, n, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      printf("window %8u KB  %s  %7.3f ms  (%.2f TB/s of 12 B/pair)\n", (4u << wl) >> 10, k ? "tiles " : "stride",
             best, 12.0 * n / best / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
