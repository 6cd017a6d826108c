// Microbenchmark: random 8 B reads / 4 B writes over a large array; which load/store
// flavour and L2 fetch-granularity limit give the fewest DRAM sectors per access.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int MODE>
__global__ void rd(const uint2* __restrict__ a, uint32_t mask, uint32_t iters, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0, x = hsh(t);
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t idx = (x ^ acc) & mask;  // dependent chain like a list walk
    uint2 v;
    if (MODE == 0) v = a[idx];
    else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a + idx));
    else if (MODE == 2) asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a + idx));
    else if (MODE == 3) asm volatile("ld.global.cv.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a + idx));
    else if (MODE == 4) { uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("ld.global.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a + idx), "l"(pol)); }
    acc += v.x + hsh(i + x);
    x = hsh(x + v.y);
  }
  if (acc == 0x12345) out[0] = acc;
}

__global__ void wr(uint32_t* __restrict__ a, uint32_t mask, uint32_t iters) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x = hsh(t * 2654435761u);
  for (uint32_t i = 0; i < iters; ++i) { x = hsh(x + i); a[x & mask] = x; }
}

int main(int argc, char** argv) {
  int lim = argc > 1 ? atoi(argv[1]) : 0;
  if (lim) { cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lim); size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity); printf("set limit %d -> %s, now %zu\n", lim, cudaGetErrorString(e), v); }
  else { size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity); printf("default limit %zu\n", v); }
  const size_t n = 1ull << 28;  // 2 GiB of uint2
  uint2* a; uint32_t* o;
  cudaMalloc(&a, n * 8); cudaMalloc(&o, 4); cudaMemset(a, 1, n * 8);
  const int blocks = 148 * 8, threads = 256; const uint32_t iters = 512;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double accesses = (double)blocks * threads * iters;
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(a, (uint32_t)(n - 1), iters, o);
    cudaEventRecord(e0); kern<<<blocks, threads>>>(a, (uint32_t)(n - 1), iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.3f ms  %6.2f G acc/s\n", name, ms, accesses / ms / 1e6);
  };
  run(rd<0>, "ld.global");
  run(rd<1>, "ld.global.nc.L1::no_allocate");
  run(rd<2>, "ld.global.cg");
  run(rd<3>, "ld.global.cv");
  run(rd<4>, "ld.L2::evict_first");
  {
    uint32_t* w = (uint32_t*)a; const size_t nw = 1ull << 28;
    wr<<<blocks, threads>>>(w, (uint32_t)(nw - 1), iters);
    cudaEventRecord(e0); wr<<<blocks, threads>>>(w, (uint32_t)(nw - 1), iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.3f ms  %6.2f G acc/s\n", "random 4B store (1 GiB)", ms, accesses / ms / 1e6);
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
