// common.cuh -- shared device/host helpers of the CUDA path (libpbit.so).
// Nothing here is shared with oracle/ (the two sides share no code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define PBIT_NULL32 0xFFFFFFFFu

// Device-side bounds checks (compute-sanitizer is closed on this GPU pool): a build with
// -DPBIT_BOUNDS_CHECK=1 traps on any index outside its buffer at the places where the
// kernels compute addresses from data (slot offsets, scatter targets, window offsets, peer
// ranks); the GPU test suite runs against that build too (tools/build_variants.py bounds=
// -DPBIT_BOUNDS_CHECK=1, PBIT_LIB_PATH).  Compiled out otherwise.
#ifndef PBIT_BOUNDS_CHECK
#define PBIT_BOUNDS_CHECK 0
#endif
#if PBIT_BOUNDS_CHECK
#define PBIT_ASSERT(cond)                                                                      \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("pbit bounds check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,    \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                     \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define PBIT_ASSERT(cond) do { } while (0)
#endif

namespace pbit {

// ----------------------------------------------------------------------------- errors
// Device-side error word (OR of bits); any bit set => PBIT_ERR_INVALID_LIST.
enum : int {
  E_BAD_INDEX = 1,   // a next[] entry >= n that is not NULL
  E_DYN_FULL = 2,    // more split segments than any valid list can need (cycle without ruler)
  E_CHAIN = 4,       // the ruler chain from the head is cyclic or does not hold exactly n nodes
};

// ----------------------------------------------------------------------------- records
// Node record packed by k_pack so that one random 32 B sector read in the walk
// serves both the key and the successor (the paper's AoS `struct Node{next,data}`,
// P:14-17).  Keys of <= 32 bits are widened to u32.
template <int KB> struct Rec { using T = uint2; };      // {key, next}
template <> struct Rec<8> { using T = uint4; };         // {key lo, key hi, next, 0}

template <int KB> struct KeyOf { using T = uint32_t; };
template <> struct KeyOf<8> { using T = unsigned long long; };

// ----------------------------------------------------------------------------- rulers
// Ruling-set selection.  Node ids are cut into blocks of s = 2^s_log2 consecutive ids;
// block r holds exactly one ruler, at offset hash(r) mod span inside the block.  The
// ruler index of a ruler node is therefore v >> s_log2: no table, no compaction.  The
// head becomes ruler R (an extra one) unless it is a ruler already.
__host__ __device__ __forceinline__ uint32_t ruler_hash(uint32_t x) {
  x ^= 0x6A09E667u;
  x ^= x >> 16; x *= 0x21F0AAADu;
  x ^= x >> 15; x *= 0x735A2D97u;
  x ^= x >> 15;
  return x;
}

struct RulerSel {
  uint32_t n;        // nodes
  uint32_t s_log2;   // spacing exponent
  uint32_t R;        // number of id blocks = ceil(n / s)

  __host__ __device__ __forceinline__ uint32_t offset_in_block(uint32_t r) const {
    uint32_t base = r << s_log2;
    uint32_t span = n - base;
    uint32_t s = 1u << s_log2;
    uint32_t h = ruler_hash(r);
    return span >= s ? (h & (s - 1)) : (h % span);
  }
  __host__ __device__ __forceinline__ uint32_t node_of(uint32_t r) const {
    return (r << s_log2) + offset_in_block(r);
  }
  __host__ __device__ __forceinline__ bool is_ruler(uint32_t v) const {
    uint32_t r = v >> s_log2;
    return (v & ((1u << s_log2) - 1)) == offset_in_block(r);
  }
};

// ----------------------------------------------------------------------------- division
// x / d for a divisor fixed per launch (Granlund-Montgomery; d = 1 by a branch): the
// multi-GPU walk divides every node id by the rank slice S to find the rank that owns it.
struct FastDiv {
  uint32_t d = 1, m = 0, s = 1;
  __host__ static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d < 1 ? 1 : d;
    if (f.d == 1) return f;
    uint32_t sh = 0;
    while ((1ull << sh) < f.d) ++sh;  // ceil(log2 d)
    f.s = sh;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << sh) - f.d)) / f.d) + 1);
    return f;
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t x) const {
#ifdef __CUDA_ARCH__
    const uint32_t t = __umulhi(x, m);
#else
    const uint32_t t = (uint32_t)(((unsigned long long)x * m) >> 32);
#endif
    return d == 1 ? x : (t + ((x - t) >> 1)) >> (s - 1);
  }
};

// ----------------------------------------------------------------------------- plan
// Device-side pass plan written by k_plan: the non-trivial digits, low to high.
// A digit whose histogram has one bin holding all n keys cannot reorder anything
// and its pass is skipped (the top digits of keys < 2^16).
struct Plan {
  uint32_t npasses;
  uint32_t digit[64];
  uint32_t skewed[2];  // bit d: some value of digit d holds more than n/16 of the keys
};

// ----------------------------------------------------------------------------- loads
__device__ __forceinline__ uint2 ld_stream_u2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long r;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Lanes of the warp whose digit equals this lane's digit, restricted to `vmask`:
// RB ballots, one per digit bit, each folded in as peers &= (bit ? B : ~B).  Written in
// PTX because the compiler's version spends ~6 instructions per bit (SHF, LOP3, ISETP,
// SEL, VOTE, LOP3); this is 4 (LOP3.P, VOTE, SEL, LOP3) -- 1.87x the throughput on
// B200 (tools/micro/match.cu; match.any is slower once a warp holds > 12 digit values).
template <int RB>
__device__ __forceinline__ uint32_t warp_peers(uint32_t d, uint32_t vmask) {
  uint32_t peers = vmask;
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    asm volatile("{ .reg .pred p; .reg .b32 t, bb, s;\n"
        "  and.b32 t, %1, %2;\n"
        "  setp.ne.u32 p, t, 0;\n"
        "  vote.sync.ballot.b32 bb, p, 0xffffffff;\n"
        "  selp.b32 s, 0, 0xffffffff, p;\n"
        "  lop3.b32 %0, %0, bb, s, 0x60; }"
        : "+r"(peers) : "r"(d), "r"(1u << b));
  }
  return peers;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ----------------------------------------------------------------------------- histograms
// One count into a per-CTA shared-memory histogram, from every lane of a warp at once (the
// whole warp must call it; `valid` masks lanes without an item).  SURVEY §8(a) a2:
//   0  one shared atomic per lane;
//   1  __match_any_sync groups the lanes holding the same bin; the lowest lane of each
//      group adds the group's size (one atomic per distinct bin in the warp);
//   2  __ballot_sync of the lanes sharing lane 0's bin: lane 0 adds them all, the others
//      add 1 each (one extra ballot; pays off when one value dominates the warp).
// Measured on B200: mode 0 wins for every histogram here (pack of C3: 0.78
// ms, vs 6.65 ms with match.any and 2.19 ms with the ballot), so it is the default.
#ifndef PBIT_HIST_MODE
#define PBIT_HIST_MODE 0
#endif
template <int MODE = PBIT_HIST_MODE>
__device__ __forceinline__ void hist_add(uint32_t* __restrict__ h, uint32_t bin, bool valid) {
  if constexpr (MODE == 0) {
    if (valid) atomicAdd(h + bin, 1u);
  } else if constexpr (MODE == 1) {
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? bin : 0xFFFFFFFFu);
    if (valid && (peers & lanemask_lt()) == 0u) atomicAdd(h + bin, (uint32_t)__popc(peers));
  } else {
    const uint32_t b0 = __shfl_sync(0xffffffffu, bin, 0);
    const uint32_t eq = __ballot_sync(0xffffffffu, valid && bin == b0);
    if ((threadIdx.x & 31u) == 0u) {
      if (eq) atomicAdd(h + b0, (uint32_t)__popc(eq));
    } else if (valid && !((eq >> (threadIdx.x & 31u)) & 1u)) {
      atomicAdd(h + bin, 1u);
    }
  }
}

}  // namespace pbit
