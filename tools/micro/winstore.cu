// Microbenchmark: random 4 B stores confined to consecutive windows of W bytes (like the
// binned relink): how large may a window be before L2 evicts partial sectors to HBM?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// pairs[p] = (target index, value); targets of pair block b all lie in window b
__global__ void mkpairs(uint2* pairs, uint32_t n, uint32_t wlog2) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    uint32_t win = p >> wlog2, off = hsh(p) & ((1u << wlog2) - 1);  // not a permutation; fine
    pairs[p] = make_uint2((win << wlog2) | off, p);
  }
}
template <int POL>
__global__ void apply(const uint2* __restrict__ pairs, uint32_t n, uint32_t* out) {
  uint64_t pol;
  if (POL == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    uint2 x = __ldcs(pairs + p);
    if (POL == 0) out[x.x] = x.y;
    else asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(out + x.x), "r"(x.y), "l"(pol) : "memory");
  }
}
int main() {
  const uint32_t n = 1u << 28;
  uint2* pairs; uint32_t* out;
  cudaMalloc(&pairs, (size_t)n * 8); cudaMalloc(&out, (size_t)n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (uint32_t wl : {14u, 16u, 18u, 20u, 22u, 24u}) {
    mkpairs<<<1184, 256>>>(pairs, n, wl);
    for (int pol = 0; pol < 2; ++pol) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (pol == 0) apply<0><<<1184, 256>>>(pairs, n, out); else apply<1><<<1184, 256>>>(pairs, n, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("window %6u KB  policy %s  %7.3f ms\n", (4u << wl) >> 10, pol ? "evict_last" : "default  ", ms);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
