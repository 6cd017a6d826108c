// Microbenchmark: apply (v, succ) pairs binned by v >> B into distributed shared memory.
// One thread-block cluster of C CTAs owns one bin of C * W ids (W ids of u32 window per
// CTA); every CTA reads 1/C of the bin's pairs and stores each succ into the owning
// CTA's window with st.shared::cluster, then each CTA writes its window out coalesced.
// Question: is this a 12 B/node relink (read 8 B pair, write 4 B) at HBM speed?
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// pairs of bin b: a random permutation of the bin's ids (x -> (x * odd + c) mod 2^bl)
__global__ void mkpairs(uint2* pairs, uint32_t n, uint32_t bl) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t bin = p >> bl, m = (1u << bl) - 1;
    const uint32_t off = ((p & m) * 0x9E3779B1u + hsh(bin)) & m;
    pairs[p] = make_uint2((bin << bl) | off, p);
  }
}

template <int C>
__global__ void __launch_bounds__(1024) apply(const uint2* __restrict__ pairs, uint32_t n, uint32_t* __restrict__ out,
                                              uint32_t wl) {
  extern __shared__ __align__(16) uint32_t win[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  const uint32_t W = 1u << wl;
  const uint32_t bin = blockIdx.x / C;
  const uint32_t b0 = bin * C * W;
  const uint32_t cnt = C * W;
  const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(win);
  cl.sync();
  for (uint32_t i = rank * blockDim.x + threadIdx.x; i < cnt; i += C * blockDim.x) {
    const uint2 x = __ldcs(pairs + b0 + i);
    const uint32_t o = x.x - b0;
    const uint32_t dst = o >> wl, lo = o & (W - 1);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(wbase + lo * 4), "r"(dst));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(x.y) : "memory");
  }
  cl.sync();
  uint4* d = reinterpret_cast<uint4*>(out + b0 + rank * W);
  for (uint32_t i = threadIdx.x; i < W / 4; i += blockDim.x) __stcs(d + i, reinterpret_cast<const uint4*>(win)[i]);
}

// baseline: single CTA window (C = 1) without cluster
__global__ void __launch_bounds__(1024) apply1(const uint2* __restrict__ pairs, uint32_t n, uint32_t* __restrict__ out,
                                               uint32_t wl) {
  extern __shared__ __align__(16) uint32_t win[];
  const uint32_t W = 1u << wl, b0 = blockIdx.x * W;
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
    const uint2 x = __ldcs(pairs + b0 + i);
    win[x.x - b0] = x.y;
  }
  __syncthreads();
  uint4* d = reinterpret_cast<uint4*>(out + b0);
  for (uint32_t i = threadIdx.x; i < W / 4; i += blockDim.x) __stcs(d + i, reinterpret_cast<const uint4*>(win)[i]);
}

template <int C>
float run(const uint2* pairs, uint32_t n, uint32_t* out, uint32_t wl, int threads) {
  const size_t smem = 4u << wl;
  cudaFuncSetAttribute(apply<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C > 8) cudaFuncSetAttribute(apply<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n >> wl);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, apply<C>, pairs, n, out, wl);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    if (e != cudaSuccess) { printf("launch C=%d: %s\n", C, cudaGetErrorString(e)); return -1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const uint32_t n = 1u << 28;
  uint2* pairs; uint32_t* out;
  cudaMalloc(&pairs, (size_t)n * 8); cudaMalloc(&out, (size_t)n * 4);
  for (uint32_t wl : {14u, 15u}) {
    for (int threads : {512, 1024}) {
      // single-CTA windows
      mkpairs<<<1184, 256>>>(pairs, n, wl);
      cudaFuncSetAttribute(apply1, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << wl);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); apply1<<<n >> wl, threads, 4u << wl>>>(pairs, n, out, wl); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("C=1  W=%6u ids thr=%4d  %7.3f ms  %6.0f GB/s (12 B/node)\n", 1u << wl, threads, best, 12.0 * n / best / 1e6);
      // clusters
      for (int C : {2, 4, 8, 16}) {
        const uint32_t bl = wl + (C == 2 ? 1 : C == 4 ? 2 : C == 8 ? 3 : 4);
        mkpairs<<<1184, 256>>>(pairs, n, bl);
        float ms = C == 2 ? run<2>(pairs, n, out, wl, threads) : C == 4 ? run<4>(pairs, n, out, wl, threads)
                 : C == 8 ? run<8>(pairs, n, out, wl, threads) : run<16>(pairs, n, out, wl, threads);
        printf("C=%-2d W=%6u ids thr=%4d  %7.3f ms  %6.0f GB/s (12 B/node)\n", C, 1u << wl, threads, ms, 12.0 * n / ms / 1e6);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
