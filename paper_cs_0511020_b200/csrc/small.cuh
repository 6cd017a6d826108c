// small.cuh -- one-launch sort of a small list: n <= SMALL_N.
//
// The general path spends most of a C1-sized call (2^16 nodes) on ~12 kernel launches and
// a mid-call host read of the pass plan.  Here ONE thread-block cluster (SMALL_CTAS CTAs,
// one per SM) does every step, synchronised by cluster barriers, on L2-resident scratch:
//   1. list ranking by pointer jumping (Wyllie): dist[v] = nodes from v to the end of the
//      list; the list is valid iff every pointer reaches NULL and dist[head] == n
//      (reading Q10) -- then v sits at list position n - dist[v];
//   2. (key, id) scattered to list order (the key-order map of N1 applied);
//   3. stable LSD counting-sort passes: CTA c owns a contiguous range of positions, ranks
//      its items in input order (rank_items), and takes its offsets from the per-(CTA,
//      digit) counts of the whole cluster; a digit with one full bin is skipped;
//   4. relink: out_next (and out_prev, N2) from the sorted ids.
// Same unique result as the general path, checked by the same parity tests.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace pbit {

#ifndef PBIT_SMALL_CTAS
#define PBIT_SMALL_CTAS 16
#endif
constexpr int SMALL_CTAS = PBIT_SMALL_CTAS;  // 16: a non-portable cluster size (set at launch)
constexpr int SMALL_THREADS = 1024;
constexpr uint32_t SMALL_N = 65536;  // <= SMALL_CTAS * SMALL_THREADS * SMALL_IPT
constexpr int SMALL_IPT = (int)(SMALL_N / (SMALL_CTAS * SMALL_THREADS));  // items per thread per pass
constexpr int SMALL_WARPS = SMALL_THREADS / 32;

struct SmallArgs {
  const void* keys;      // user keys (KB bytes each), node-indexed
  const uint32_t* next;  // user successors
  uint32_t head, n;
  uint32_t* out_next;
  uint32_t* out_prev;    // nullable
  uint32_t* d_head;
  uint32_t* passes;      // digits actually sorted (trivial ones skipped)
  int* err;
  KeyMap km;
  // scratch (n entries each, double-buffered)
  uint2* dn[2];          // {dist, nx}: one 8 B gather per pointer-jumping step
  void* lkey[2];         // list-order sort keys (u32, or u64 for 8-byte keys)
  uint32_t* lid[2];      // list-order node ids
  uint32_t* hist;        // [SMALL_CTAS][256] per pass
};

__device__ __forceinline__ void small_sync() {
  __threadfence();  // global scratch written before the barrier is visible after it
  cooperative_groups::this_cluster().sync();
}

template <int KB, int RADIX_BITS>
__global__ void __cluster_dims__(SMALL_CTAS, 1, 1) __launch_bounds__(SMALL_THREADS, 1)
k_small_sort(const __grid_constant__ SmallArgs a) {
  using KeyT = typename KeyOf<KB>::T;
  using KT = std::conditional_t<KB == 1, uint8_t, std::conditional_t<KB == 2, uint16_t,
             std::conditional_t<KB == 4, uint32_t, unsigned long long>>>;
  constexpr int RADIX = 1 << RADIX_BITS;
  constexpr int D = (KB * 8 + RADIX_BITS - 1) / RADIX_BITS;
  __shared__ WCnt wcnt[SMALL_WARPS][RADIX];
  __shared__ uint32_t s_base[RADIX], s_scan[SMALL_WARPS];
  __shared__ int s_trivial;
  __shared__ uint32_t s_scratch[32];  // rank_items' per-lane words for atomics that add nothing
  __shared__ int s_err;  // this CTA's error bits; combined over the cluster via DSMEM
  __shared__ int s_bad;

  const uint32_t n = a.n;
  const uint32_t c = cooperative_groups::this_cluster().block_rank();
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t gt = c * SMALL_THREADS + t, GT = SMALL_CTAS * SMALL_THREADS;

  if (t == 0) s_err = 0;
  __syncthreads();
  // ---- 1. ranking: dist = 1, nx = next; then rounds of dist += dist[nx], nx = nx[nx]
  for (uint32_t v = gt; v < n; v += GT) {
    const uint32_t x = a.next[v];
    if (x != PBIT_NULL32 && x >= n) atomicOr(&s_err, E_BAD_INDEX);
    a.dn[0][v] = make_uint2(1u, x >= n ? PBIT_NULL32 : x);
  }
  small_sync();
  int cur = 0;
  for (uint32_t span = 1; span < 2 * n; span <<= 1) {  // ceil(log2 n) + 1 rounds
    const uint2* src = a.dn[cur];
    // a thread's SMALL_IPT nodes at once: two dependent L2 round trips per round
    uint2 e[SMALL_IPT], f[SMALL_IPT];
#pragma unroll
    for (int i = 0; i < SMALL_IPT; ++i) {
      const uint32_t v = gt + i * GT;
      e[i] = v < n ? src[v] : make_uint2(0u, PBIT_NULL32);
    }
#pragma unroll
    for (int i = 0; i < SMALL_IPT; ++i) f[i] = e[i].y != PBIT_NULL32 ? src[e[i].y] : make_uint2(0u, PBIT_NULL32);
#pragma unroll
    for (int i = 0; i < SMALL_IPT; ++i) {
      const uint32_t v = gt + i * GT;
      if (v < n) a.dn[cur ^ 1][v] = make_uint2(e[i].x + f[i].x, f[i].y);
    }
    cur ^= 1;
    small_sync();
  }
  // valid iff every pointer reached NULL and the head's chain holds all n nodes
  for (uint32_t v = gt; v < n; v += GT)
    if (a.dn[cur][v].y != PBIT_NULL32) atomicOr(&s_err, E_CHAIN);
  if (gt == 0 && a.dn[cur][a.head].x != n) atomicOr(&s_err, E_CHAIN);
  small_sync();
  {  // every CTA ORs the cluster's error bits (DSMEM reads after the barrier), so the
     // decision is uniform; the error word needs no memset before the launch
    auto cl = cooperative_groups::this_cluster();
    int e = 0;
    if (t < SMALL_CTAS) e = *cl.map_shared_rank(&s_err, t);
    e = __reduce_or_sync(0xffffffffu, w == 0 ? e : 0);
    if (t == 0) s_bad = e;
    __syncthreads();
    const int bad = s_bad;
    if (c == 0 && t == 0) *a.err = bad;
    if (bad) {
      cl.sync();  // no CTA exits while another may still read its s_err
      return;
    }
  }

  // ---- 2. list order: position of v = n - dist[v]
  for (uint32_t v = gt; v < n; v += GT) {
    const uint32_t p = n - a.dn[cur][v].x;
    unsigned long long k = reinterpret_cast<const KT*>(a.keys)[v];
    if (!a.km.identity()) k = a.km(k, KB * 8);
    reinterpret_cast<KeyT*>(a.lkey[0])[p] = (KeyT)k;
    a.lid[0][p] = v;
  }
  small_sync();

  // ---- 3. stable LSD passes; CTA c owns positions [lo, hi)
  const uint32_t lo = (uint32_t)(((unsigned long long)n * c) / SMALL_CTAS);
  const uint32_t hi = (uint32_t)(((unsigned long long)n * (c + 1)) / SMALL_CTAS);
  const uint32_t cnt = hi - lo;
  const uint32_t wofs = w * (32 * SMALL_IPT);
  int src = 0;
  uint32_t passes = 0;
  for (int dg = 0; dg < D; ++dg) {
    const KeyT* kin = reinterpret_cast<const KeyT*>(a.lkey[src]);
    for (uint32_t i = t; i < SMALL_WARPS * RADIX * sizeof(WCnt) / 4; i += SMALL_THREADS)
      reinterpret_cast<uint32_t*>(&wcnt[0][0])[i] = 0;
    if (t == 0) s_trivial = 0;
    __syncthreads();
    KeyT key[SMALL_IPT];
    uint32_t rd[SMALL_IPT];
#pragma unroll
    for (int i = 0; i < SMALL_IPT; ++i) {
      const uint32_t j = wofs + i * 32 + lane;
      key[i] = j < cnt ? kin[lo + j] : (KeyT)0;
    }
    rank_items<KeyT, RADIX_BITS, SMALL_IPT, RANK_ATOMIC, false>(key, rd, dg * RADIX_BITS, wcnt[w], wofs, lane, cnt,
                                                                false, (uint32_t)__cvta_generic_to_shared(s_scratch));
    __syncthreads();
    if (t < RADIX) {  // exclusive prefix over the warps (in place); the CTA's digit counts
      uint32_t tot = 0;
      for (int ww = 0; ww < SMALL_WARPS; ++ww) {
        const uint32_t x = wcnt[ww][t];
        wcnt[ww][t] = (WCnt)tot;
        tot += x;
      }
      a.hist[c * 256 + t] = tot;
    }
    small_sync();
    // base of (this CTA, digit t) = all keys of smaller digits + this digit's keys in
    // lower CTAs (= earlier positions)
    uint32_t col = 0, below = 0;
    if (t < RADIX) {
      for (uint32_t q = 0; q < SMALL_CTAS; ++q) {
        const uint32_t h = a.hist[q * 256 + t];
        col += h;
        below += q < c ? h : 0u;
      }
      if (col == n) s_trivial = 1;  // one digit value everywhere: nothing to reorder
    }
    {
      uint32_t x = col;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) s_scan[w] = x;
      __syncthreads();
      uint32_t add = 0;
      for (uint32_t q = 0; q < w; ++q) add += s_scan[q];
      if (t < RADIX) s_base[t] = x - col + add + below;
    }
    __syncthreads();
    const bool trivial = s_trivial != 0;
    small_sync();  // every CTA has read this pass's counts (the next pass rewrites them)
    if (trivial) continue;
    KeyT* kout = reinterpret_cast<KeyT*>(a.lkey[src ^ 1]);
    const uint32_t* iin = a.lid[src];
    uint32_t* iout = a.lid[src ^ 1];
#pragma unroll
    for (int i = 0; i < SMALL_IPT; ++i) {
      const uint32_t j = wofs + i * 32 + lane;
      if (j < cnt) {
        const uint32_t d = rd[i] >> 16;
        const uint32_t pos = s_base[d] + wcnt[w][d] + (rd[i] & 0xFFFFu);
        kout[pos] = key[i];
        iout[pos] = iin[lo + j];
      }
    }
    src ^= 1;
    ++passes;
    small_sync();
  }

  // ---- 4. relink (the paper's merge) and the doubly-linked repair (N2)
  const uint32_t* ids = a.lid[src];
  for (uint32_t p = gt; p < n; p += GT) {
    a.out_next[ids[p]] = p + 1 < n ? ids[p + 1] : PBIT_NULL32;
    if (a.out_prev) a.out_prev[ids[p]] = p > 0 ? ids[p - 1] : PBIT_NULL32;
  }
  if (gt == 0) {
    *a.d_head = ids[0];
    *a.passes = passes;
  }
}

}  // namespace pbit
