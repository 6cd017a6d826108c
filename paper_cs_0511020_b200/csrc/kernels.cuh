// kernels.cuh -- the sm_100a kernels of the Pbit hot path.
//
//   k_pack      a1/a2  AoS (key,next) records + histograms of every digit (one sweep)
//   k_walk      a1     ruling-set walk: every segment written in list order to its slot
//   k_rank_*    a1     ruler-list ranking by pointer jumping; validates the chain
//   k_gather    a1     segments -> list-order (key, id) arrays
//   k_plan      a3     exclusive scans of the digit histograms -> bucket bases, pass plan
//   k_onesweep  a3/a4  one stable LSD pass: warp-ballot ranking, decoupled lookback,
//                      smem-staged scatter with 128-bit stores
//   k_relink    a5     out_next from the sorted ids (the paper's merge)
//
// Paper anchors: the split loop is the stable scatter; the end-marker
// recursion is the ascending order of the bucket bases; merge is relink.
#pragma once
#include "common.cuh"

namespace pbit {

constexpr int PACK_THREADS = 256;
constexpr int WALK_THREADS = 256;
constexpr int SWEEP_THREADS = 256;
constexpr int SWEEP_WARPS = SWEEP_THREADS / 32;

// ============================================================================ a1/a2: pack
// Reads key[v], next[v] (streaming, coalesced), writes the AoS record kn[v], and counts
// every digit of every key into a per-CTA smem histogram (flushed once per CTA).
template <int KB>
__global__ void __launch_bounds__(PACK_THREADS)
k_pack(const void* __restrict__ keys, const uint32_t* __restrict__ next, uint32_t n,
       typename Rec<KB>::T* __restrict__ kn, uint32_t* __restrict__ hist, int K, int D,
       int* __restrict__ err) {
  extern __shared__ uint32_t s_hist[];
  const int radix = 1 << K;
  const int nb = D * radix;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const uint32_t mask = radix - 1;
  int bad = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint32_t nx = __ldcs(next + v);
    bad |= (nx != PBIT_NULL32) & (nx >= n);
    if constexpr (KB == 8) {
      unsigned long long k = __ldcs(reinterpret_cast<const unsigned long long*>(keys) + v);
      kn[v] = make_uint4((uint32_t)k, (uint32_t)(k >> 32), nx, 0u);
      for (int d = 0; d < D; ++d) atomicAdd(&s_hist[d * radix + (int)((k >> (d * K)) & mask)], 1u);
    } else {
      uint32_t k;
      if constexpr (KB == 1) k = reinterpret_cast<const uint8_t*>(keys)[v];
      else if constexpr (KB == 2) k = reinterpret_cast<const uint16_t*>(keys)[v];
      else k = __ldcs(reinterpret_cast<const uint32_t*>(keys) + v);
      kn[v] = make_uint2(k, nx);
      for (int d = 0; d < D; ++d) atomicAdd(&s_hist[d * radix + (int)((k >> (d * K)) & mask)], 1u);
    }
  }
  if (bad) atomicOr(err, E_BAD_INDEX);
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// ============================================================================ a1: walk
// One thread walks one segment at a time: from its ruler node along next[] until the
// next ruler (or NULL), writing (key, id) of each visited node into the segment's slot
// in list order -- the same sequential traversal as the paper's split loop L=L->next
// (P:353), which is what makes the result stable.  A segment longer than `cap` is cut:
// the walker opens a dynamic ruler (slot R_static + k) at the current node and goes on.
// Rulers are handed out per CTA from a contiguous range through a smem counter.
template <int KB>
__global__ void __launch_bounds__(WALK_THREADS)
k_walk(const typename Rec<KB>::T* __restrict__ kn, RulerSel sel, uint32_t R_static, uint32_t head,
       typename Rec<KB>::T* __restrict__ slots, uint32_t cap, uint32_t* __restrict__ seg_len,
       uint32_t* __restrict__ seg_succ, uint32_t* __restrict__ dyn_count, uint32_t dyn_cap,
       uint32_t per_cta, int* __restrict__ err) {
  using RT = typename Rec<KB>::T;
  __shared__ uint32_t s_next;
  if (threadIdx.x == 0) s_next = 0;
  __syncthreads();
  const uint32_t n = sel.n;
  const uint32_t lo = blockIdx.x * per_cta;
  const uint32_t hi = min(lo + per_cta, R_static);
  for (;;) {
    const uint32_t r = lo + atomicAdd(&s_next, 1u);
    if (r >= hi) break;
    uint32_t u = r < sel.R ? sel.node_of(r) : head;
    uint32_t cur = r, j = 0;
    RT* out = slots + (size_t)cur * cap;
    for (;;) {
      RT x;
      if constexpr (KB == 8) x = ld_stream_u4(kn + u); else x = ld_stream_u2(kn + u);
      uint32_t v;
      if constexpr (KB == 8) { v = x.z; x.z = u; } else { v = x.y; x.y = u; }
      out[j] = x;  // (key, id)
      ++j;
      if (v == PBIT_NULL32) { seg_len[cur] = j; seg_succ[cur] = PBIT_NULL32; break; }
      if (v >= n) { atomicOr(err, E_BAD_INDEX); seg_len[cur] = j; seg_succ[cur] = PBIT_NULL32; break; }
      if (sel.is_ruler(v)) { seg_len[cur] = j; seg_succ[cur] = v >> sel.s_log2; break; }
      if (j == cap) {
        const uint32_t k = atomicAdd(dyn_count, 1u);
        if (k >= dyn_cap) { atomicOr(err, E_DYN_FULL); seg_len[cur] = j; seg_succ[cur] = PBIT_NULL32; break; }
        const uint32_t r2 = R_static + k;
        seg_len[cur] = cap; seg_succ[cur] = r2;
        cur = r2; j = 0; out = slots + (size_t)cur * cap;
      }
      u = v;
    }
  }
}

// ============================================================================ a1: rank
// Pointer jumping (Wyllie) over the ruler list: dist[r] = nodes from the first node of
// segment r to the end of the list.  After ceil(log2 R)+1 rounds every succ is NULL
// unless the ruler graph has a cycle.
__global__ void k_rank_init(const uint32_t* __restrict__ seg_len, const uint32_t* __restrict__ seg_succ,
                            uint32_t R_static, const uint32_t* __restrict__ dyn_count, uint32_t dyn_cap,
                            unsigned long long* __restrict__ dist, uint32_t* __restrict__ succ,
                            const int* __restrict__ err) {
  if (*err) return;
  const uint32_t R = R_static + min(*dyn_count, dyn_cap);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    dist[r] = seg_len[r];
    succ[r] = seg_succ[r];
  }
}

__global__ void k_rank_jump(const unsigned long long* __restrict__ d_in, const uint32_t* __restrict__ s_in,
                            unsigned long long* __restrict__ d_out, uint32_t* __restrict__ s_out,
                            uint32_t R_static, const uint32_t* __restrict__ dyn_count, uint32_t dyn_cap,
                            const int* __restrict__ err) {
  if (*err) return;
  const uint32_t R = R_static + min(*dyn_count, dyn_cap);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const uint32_t s = s_in[r];
    unsigned long long d = d_in[r];
    uint32_t s2 = s;
    if (s != PBIT_NULL32) { d += d_in[s]; s2 = s_in[s]; }
    d_out[r] = d;
    s_out[r] = s2;
  }
}

// Validation (reading Q10): the chain from the head ruler must end (succ NULL) and hold
// exactly n nodes; then every node lies on it.
__global__ void k_rank_check(const unsigned long long* __restrict__ dist, const uint32_t* __restrict__ succ,
                             uint32_t head_ruler, uint32_t n, int* __restrict__ err) {
  if (*err) return;
  if (succ[head_ruler] != PBIT_NULL32 || dist[head_ruler] != (unsigned long long)n) atomicOr(err, E_CHAIN);
}

// ============================================================================ a1: gather
// Segment r occupies list positions [n - dist[r], n - dist[r] + len[r]).  One warp per
// segment copies its slot into the list-order arrays (coalesced both ways).
template <int KB>
__global__ void k_gather(const typename Rec<KB>::T* __restrict__ slots, uint32_t cap,
                         const uint32_t* __restrict__ seg_len, const unsigned long long* __restrict__ dist,
                         uint32_t R_static, const uint32_t* __restrict__ dyn_count, uint32_t dyn_cap, uint32_t n,
                         typename KeyOf<KB>::T* __restrict__ keys_lo, uint32_t* __restrict__ ids_lo,
                         const int* __restrict__ err) {
  if (*err) return;
  const uint32_t R = R_static + min(*dyn_count, dyn_cap);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = warp; r < R; r += nwarps) {
    const uint32_t len = seg_len[r];
    const uint32_t off = n - (uint32_t)dist[r];
    const typename Rec<KB>::T* src = slots + (size_t)r * cap;
    for (uint32_t j = lane; j < len; j += 32) {
      if constexpr (KB == 8) {
        uint4 x = src[j];
        keys_lo[off + j] = ((unsigned long long)x.y << 32) | x.x;
        ids_lo[off + j] = x.z;
      } else {
        uint2 x = src[j];
        keys_lo[off + j] = x.x;
        ids_lo[off + j] = x.y;
      }
    }
  }
}

// ============================================================================ a3: plan
// Exclusive scan of each digit's histogram (bucket bases, ascending = the ascending
// end-marker order of P:379-380) and the list of non-trivial digits.  One CTA.
__global__ void __launch_bounds__(256)
k_plan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ bases, Plan* __restrict__ plan,
       int D, int K, uint32_t n, const int* __restrict__ err) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_np;
  const int radix = 1 << K;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_np = 0;
  __syncthreads();
  for (int d = 0; d < D; ++d) {
    // radix <= 256 == blockDim
    const uint32_t c = t < radix ? hist[d * radix + t] : 0u;
    const int trivial = __syncthreads_or(c == n);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    uint32_t add = 0;
    for (int i = 0; i < w; ++i) add += s_warp[i];
    if (t < radix) bases[d * radix + t] = x - c + add;
    if (t == 0 && !trivial) plan->digit[s_np++] = d;
    __syncthreads();
  }
  if (t == 0) plan->npasses = (*err) ? 0u : s_np;
}

// ============================================================================ a3/a4: onesweep
// One stable counting-sort pass on digit plan->digit[slot] (Merrill & Garland style
// single-pass scan with decoupled lookback).  Tile = 256 threads x IPT items, taken in
// launch order from an atomic ticket so every predecessor tile is running or done.
//
// Status word per (tile, digit): count[31:0] | flag[33:32] (1 aggregate, 2 inclusive)
// | epoch[63:34]; the status array is zeroed once per call and each pass slot uses its
// own epoch, so stale words from earlier passes never match.
template <typename KeyT, int RADIX_BITS, int IPT>
__global__ void __launch_bounds__(SWEEP_THREADS)
k_onesweep(const Plan* __restrict__ plan, int slot, KeyT* keys0, uint32_t* ids0, KeyT* keys1, uint32_t* ids1,
           const uint32_t* __restrict__ bases, unsigned long long* status, uint32_t* tile_ctr, uint32_t n,
           const int* __restrict__ err) {
  constexpr int RADIX = 1 << RADIX_BITS;
  constexpr int TILE = SWEEP_THREADS * IPT;
  constexpr int WARP_ITEMS = 32 * IPT;
  static_assert(RADIX <= SWEEP_THREADS, "one thread per digit value");

  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wcnt[SWEEP_WARPS][RADIX];
  __shared__ uint32_t s_dstart[RADIX];
  __shared__ uint32_t s_goff[RADIX];
  __shared__ uint32_t s_scan[SWEEP_WARPS];
  __shared__ __align__(16) KeyT s_keys[TILE];
  __shared__ __align__(16) uint32_t s_ids[TILE];

  if (*err) return;
  const uint32_t npasses = plan->npasses;
  if ((uint32_t)slot >= npasses) return;
  const int digit_idx = plan->digit[slot];
  const int shift = digit_idx * RADIX_BITS;
  const bool last = (uint32_t)slot + 1 == npasses;
  const KeyT* __restrict__ kin = (slot & 1) ? keys1 : keys0;
  const uint32_t* __restrict__ iin = (slot & 1) ? ids1 : ids0;
  KeyT* __restrict__ kout = (slot & 1) ? keys0 : keys1;
  uint32_t* __restrict__ iout = (slot & 1) ? ids0 : ids1;
  const unsigned long long epoch = (unsigned long long)(slot + 1);

  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < SWEEP_WARPS * RADIX; i += SWEEP_THREADS) (&s_wcnt[0][0])[i] = 0;
  if (t == 0) s_tile = atomicAdd(tile_ctr + slot, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t tile_base = tile * (uint32_t)TILE;
  const uint32_t tile_count = min((uint32_t)TILE, n - tile_base);

  // ---- load (warp-striped: each load instruction covers 32 consecutive elements)
  KeyT key[IPT];
  uint32_t id[IPT];
  uint32_t rank[IPT];
  const uint32_t wbase = tile_base + w * WARP_ITEMS;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t p = wbase + i * 32 + lane;
    if (p < n) { key[i] = kin[p]; id[i] = iin[p]; }
    else { key[i] = 0; id[i] = 0; }
  }

  // ---- stable in-warp ranking: items in input order, equal digits grouped by ballots
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t p = wbase + i * 32 + lane;
    const bool valid = p < n;
    const uint32_t d = (uint32_t)(key[i] >> shift) & (RADIX - 1);
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < RADIX_BITS; ++b) {
      const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bb : ~bb;
    }
    const int leader = 31 - __clz(peers | 1u);
    uint32_t before = 0;
    if (valid && lane == leader) before = atomicAdd(&s_wcnt[w][d], (uint32_t)__popc(peers));
    before = __shfl_sync(0xffffffffu, before, leader);
    rank[i] = before + __popc(peers & lanemask_lt());
  }
  __syncthreads();

  // ---- per digit: exclusive over warps, tile total, publish aggregate, scan over digits
  uint32_t total = 0;
  if (t < RADIX) {
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) {
      const uint32_t c = s_wcnt[ww][t];
      s_wcnt[ww][t] = total;
      total += c;
    }
    if (tile > 0 && total)  // zero aggregates are implied by the epoch-matched zero word below
      st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (1ull << 32) | total);
    else if (tile > 0)
      st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (1ull << 32));
  }
  {
    uint32_t x = total;  // threads >= RADIX contribute 0
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_scan[w] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) add += (ww < w) ? s_scan[ww] : 0u;
    if (t < RADIX) s_dstart[t] = x - total + add;
  }
  __syncthreads();

  // ---- stage the tile in smem in (digit, input order) order
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t p = wbase + i * 32 + lane;
    if (p < n) {
      const uint32_t d = (uint32_t)(key[i] >> shift) & (RADIX - 1);
      const uint32_t lp = s_dstart[d] + s_wcnt[w][d] + rank[i];
      s_keys[lp] = key[i];
      s_ids[lp] = id[i];
    }
  }

  // ---- decoupled lookback, one thread per digit value
  if (t < RADIX) {
    unsigned long long excl = 0;
    if (tile == 0) {
      st_relaxed_u64(status + t, (epoch << 34) | (2ull << 32) | total);
    } else {
      int64_t pr = (int64_t)tile - 1;
      for (;;) {
        const unsigned long long wv = ld_relaxed_u64(status + (size_t)pr * RADIX + t);
        if ((wv >> 34) != epoch) continue;  // predecessor has not published yet
        excl += (uint32_t)wv;
        if (((wv >> 32) & 3ull) == 2ull) break;
        --pr;
      }
      st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (2ull << 32) | (excl + total));
    }
    s_goff[t] = bases[digit_idx * RADIX + t] + (uint32_t)excl - s_dstart[t];
  }
  __syncthreads();

  // ---- write out: runs of equal digits land contiguously; 4 consecutive staged items
  // per thread, one 128-bit store when they share a digit and the target is aligned.
  const int nq = (int)((tile_count + 3) >> 2);
  for (int q = t; q < nq; q += SWEEP_THREADS) {
    const uint32_t j0 = (uint32_t)q * 4;
    if (j0 + 3 < tile_count) {
      const uint32_t d0 = (uint32_t)(s_keys[j0] >> shift) & (RADIX - 1);
      const uint32_t d3 = (uint32_t)(s_keys[j0 + 3] >> shift) & (RADIX - 1);
      const uint32_t g0 = s_goff[d0] + j0;
      if (d0 == d3 && (g0 & 3u) == 0) {  // staged order is digit-sorted, so d0==d3 => all equal
        const uint4 iv = *reinterpret_cast<const uint4*>(&s_ids[j0]);
        *reinterpret_cast<uint4*>(iout + g0) = iv;
        if (!last) {
          if constexpr (sizeof(KeyT) == 4) {
            *reinterpret_cast<uint4*>(kout + g0) = *reinterpret_cast<const uint4*>(&s_keys[j0]);
          } else {
            *reinterpret_cast<uint4*>(kout + g0) = *reinterpret_cast<const uint4*>(&s_keys[j0]);
            *reinterpret_cast<uint4*>(kout + g0 + 2) = *reinterpret_cast<const uint4*>(&s_keys[j0 + 2]);
          }
        }
        continue;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t j = j0 + e;
      if (j < tile_count) {
        const KeyT k = s_keys[j];
        const uint32_t d = (uint32_t)(k >> shift) & (RADIX - 1);
        const uint32_t g = s_goff[d] + j;
        iout[g] = s_ids[j];
        if (!last) kout[g] = k;
      }
    }
  }
}

// ============================================================================ a5: relink
// out_next[ids[p]] = ids[p+1], out_next[ids[n-1]] = NULL, head = ids[0]: the paper's
// end-splice merge of sorted fragments, one write per node.
__global__ void k_relink(const Plan* __restrict__ plan, const uint32_t* __restrict__ ids0,
                         const uint32_t* __restrict__ ids1, uint32_t n, uint32_t* __restrict__ out_next,
                         uint32_t* __restrict__ d_head, const int* __restrict__ err) {
  if (*err) return;
  const uint32_t* __restrict__ ids = (plan->npasses & 1) ? ids1 : ids0;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t v = ids[p];
    const uint32_t s = (p + 1 < n) ? ids[p + 1] : PBIT_NULL32;
    out_next[v] = s;
    if (p == 0) *d_head = v;
  }
}

}  // namespace pbit
