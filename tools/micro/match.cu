// Throughput of warp peer-mask computation for 8-bit digits: match.any vs 8 ballots,
// as a function of how many distinct digit values a warp holds.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint32_t distinct, uint32_t iters, uint32_t* out) {
  uint32_t lane = threadIdx.x & 31, acc = 0;
  uint32_t d = (lane * 7 + blockIdx.x) % distinct;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t dd = (d + i) & 255;
    uint32_t peers;
    if (MODE == 0) peers = __match_any_sync(0xffffffffu, dd);
    else if (MODE == 2) {
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        asm("{ .reg .pred p; .reg .b32 t, bb, s;\n"
            "  and.b32 t, %1, %2;\n"
            "  setp.ne.u32 p, t, 0;\n"
            "  vote.sync.ballot.b32 bb, p, 0xffffffff;\n"
            "  selp.b32 s, 0, 0xffffffff, p;\n"
            "  lop3.b32 %0, %0, bb, s, 0x60; }" : "+r"(peers) : "r"(dd), "r"(1u << b));
      }
    } else {
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) { uint32_t bb = __ballot_sync(0xffffffffu, (dd >> b) & 1u); peers &= ((dd >> b) & 1u) ? bb : ~bb; }
    }
    acc += __popc(peers & ((1u << lane) - 1));
  }
  if (acc == 0x7777777) out[0] = acc;
}
int main() {
  uint32_t* o; cudaMalloc(&o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const uint32_t iters = 4096; const int blocks = 148 * 8, threads = 256;
  for (uint32_t dist : {1u, 2u, 4u, 8u, 16u, 32u}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      f<<<blocks, threads>>>(dist, iters, o);
      cudaEventRecord(e0); f<<<blocks, threads>>>(dist, iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_ops = (double)blocks * threads / 32 * iters;
      printf("distinct %2u  %-8s %7.3f ms  %6.1f G warp-ranks/s\n", dist, mode == 2 ? "ptx8" : mode ? "ballot8" : "match", ms, warp_ops / ms / 1e6);
    }
  }
}
