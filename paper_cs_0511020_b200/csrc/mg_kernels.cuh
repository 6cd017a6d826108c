// mg_kernels.cuh -- kernels used only by the multi-GPU path (pbit_sort_list_mg).
// The single-GPU kernels (kernels.cuh) do the rest.  Rank r of G owns node ids
// [r*S, r*S + n_local) and, after the top-digit exchange, the sorted positions
// [r*S, r*S + S) of the output.
#pragma once
#include "kernels.cuh"

namespace pbit {

// Count-only ruling-set walk over this rank's rulers: blocks [b_lo, b_hi) of the global
// id space (a rank's id slice is a whole number of blocks) plus, on the rank owning the
// head, the head's extra ruler `head_ruler_idx`.  Every rank holds the full kn replica,
// so segments may leave the rank's slice.  No slots: the list-order records are written
// later by k_emit_walk straight to their final positions.  A walk longer than n steps is
// a cycle without a ruler (invalid list).
template <int KB>
__global__ void __launch_bounds__(WALK_THREADS)
k_walk_count(const typename Rec<KB>::T* __restrict__ kn, RulerSel sel, uint32_t b_lo, uint32_t b_hi,
             uint32_t head_ruler_idx, uint32_t head, uint2* __restrict__ seg, uint32_t per_cta,
             int* __restrict__ err) {
  using RT = typename Rec<KB>::T;
  __shared__ uint32_t s_next;
  if (threadIdx.x == 0) s_next = 0;
  __syncthreads();
  const uint32_t n = sel.n;
  const uint32_t total = (b_hi - b_lo) + (head_ruler_idx != PBIT_NULL32 ? 1u : 0u);
  const uint32_t lo = blockIdx.x * per_cta;
  const uint32_t hi = min(lo + per_cta, total);
  for (;;) {
    const uint32_t i = lo + atomicAdd(&s_next, 1u);
    if (i >= hi) break;
    const bool is_head = i == b_hi - b_lo;
    const uint32_t r = is_head ? head_ruler_idx : b_lo + i;
    if (!is_head && r >= sel.R) { seg[r] = make_uint2(0, PBIT_NULL32); continue; }
    uint32_t u = is_head ? head : sel.node_of(r);
    uint32_t len = 0, succ = PBIT_NULL32;
    for (;;) {
      RT x;
      if constexpr (KB == 8) x = ld_stream_u4(kn + u); else x = ld_stream_u2(kn + u);
      uint32_t v;
      if constexpr (KB == 8) v = x.z; else v = x.y;
      ++len;
      if (v == PBIT_NULL32) break;
      if (v >= n) { atomicOr(err, E_BAD_INDEX); break; }
      if (sel.is_ruler(v)) { succ = v >> sel.s_log2; break; }
      if (len > n) { atomicOr(err, E_CHAIN); break; }
      u = v;
    }
    seg[r] = make_uint2(len, succ);
  }
}

// Emit the list-order records of positions [P0, P1): each thread re-walks one segment
// that overlaps the range (segments in list order from part_first) and writes its nodes'
// (key, id) at their final positions.
template <int KB>
__global__ void __launch_bounds__(256)
k_emit_walk(const typename Rec<KB>::T* __restrict__ kn, RulerSel sel, uint32_t head,
            const uint2* __restrict__ seg, const uint32_t* __restrict__ seg_ord, const uint32_t* __restrict__ seg_pos,
            const uint32_t* __restrict__ part_first, int rank, const uint32_t* __restrict__ nseg, uint32_t P0,
            uint32_t P1, typename KeyOf<KB>::T* __restrict__ keys_c, uint32_t* __restrict__ ids_c,
            const int* __restrict__ err) {
  using RT = typename Rec<KB>::T;
  if (*err || P0 >= P1) return;
  const uint32_t k0 = part_first[rank], ns = *nseg;
  for (uint32_t k = k0 + blockIdx.x * blockDim.x + threadIdx.x; k < ns; k += gridDim.x * blockDim.x) {
    const uint32_t pos = seg_pos[k];
    if (pos >= P1) break;  // segments are in list order
    const uint32_t r = seg_ord[k];
    const uint32_t len = seg[r].x;
    if (pos + len <= P0) continue;
    uint32_t u = r < sel.R ? sel.node_of(r) : head;
    for (uint32_t j = 0; j < len; ++j) {
      const uint32_t p = pos + j;
      if (p >= P1) break;
      RT x;
      if constexpr (KB == 8) x = ld_stream_u4(kn + u); else x = ld_stream_u2(kn + u);
      if (p >= P0) {
        if constexpr (KB == 8) {
          keys_c[p - P0] = ((unsigned long long)x.y << 32) | x.x;
          ids_c[p - P0] = u;
          u = x.z;
        } else {
          keys_c[p - P0] = x.x;
          ids_c[p - P0] = u;
          u = x.y;
        }
      } else {
        if constexpr (KB == 8) u = x.z; else u = x.y;
      }
    }
  }
}

// Histograms of every digit of m keys (a chunk in list order).
template <typename KeyT>
__global__ void __launch_bounds__(256)
k_chunk_hist(const KeyT* __restrict__ keys, uint32_t m, int K, int D, uint32_t* __restrict__ hist,
             const int* __restrict__ err) {
  extern __shared__ uint32_t s_hist[];
  if (*err) return;
  const int radix = 1 << K;
  for (int i = threadIdx.x; i < D * radix; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
    const KeyT k = keys[p];
    for (int d = 0; d < D; ++d) atomicAdd(&s_hist[d * radix + (int)((k >> (d * K)) & (radix - 1))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < D * radix; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// A one-pass plan (the top-digit partition pass) and exclusive bases of one digit.
static __global__ void k_single_plan(const uint32_t* __restrict__ hist, int digit, int K, Plan* __restrict__ plan,
                              uint32_t* __restrict__ bases, const int* __restrict__ err) {
  if (threadIdx.x != 0) return;
  const int radix = 1 << K;
  uint32_t acc = 0;
  for (int b = 0; b < radix; ++b) {
    bases[digit * radix + b] = acc;
    acc += hist[digit * radix + b];
  }
  plan->npasses = (*err) ? 0u : 1u;
  plan->digit[0] = digit;
}

// For each query key q: how many of the m sorted keys are below q (le = 0) or up to q
// (le = 1) -- a binary search per thread (the splitter refinement of pbit_sort_list_mg).
template <typename KeyT>
__global__ void k_count_below(const KeyT* __restrict__ keys, uint32_t m, const unsigned long long* __restrict__ q,
                              uint32_t nq, int le, uint32_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += gridDim.x * blockDim.x) {
    const unsigned long long v = q[i];
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo) >> 1);
      const unsigned long long k = (unsigned long long)keys[mid];
      if (le ? k <= v : k < v) lo = mid + 1; else hi = mid;
    }
    out[i] = lo;
  }
}

// (v, w) pairs of this rank's sorted positions, counted (pass 0) or scattered (pass 1) by
// the owner rank of v: owner = v / S.  dir +1: w = the successor (`edge` = the next rank's
// first id, or NULL, after the last position); dir -1: w = the predecessor (`edge` = the
// previous rank's last id, or NULL, before the first position) -- out_prev (N2).
static __global__ void __launch_bounds__(256)
k_pairs_owner(const Plan* __restrict__ plan, const uint32_t* __restrict__ ids0, const uint32_t* __restrict__ ids1,
              uint32_t m, uint32_t edge, int dir, uint32_t S, int G, uint32_t* __restrict__ counts,
              const uint32_t* __restrict__ offsets, uint32_t* __restrict__ fill, uint2* __restrict__ send, int scatter,
              const int* __restrict__ err) {
  __shared__ uint32_t s_cnt[64];
  __shared__ uint32_t s_base[64];
  if (*err) return;
  const uint32_t* __restrict__ ids = (plan->npasses & 1) ? ids1 : ids0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) s_cnt[g] = 0;
  __syncthreads();
  const uint32_t per = (m + gridDim.x - 1) / gridDim.x;
  const uint32_t p0 = blockIdx.x * per, p1 = min(m, p0 + per);
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) atomicAdd(&s_cnt[ids[p] / S], 1u);
  __syncthreads();
  if (!scatter) {
    for (int g = threadIdx.x; g < G; g += blockDim.x)
      if (s_cnt[g]) atomicAdd(&counts[g], s_cnt[g]);
    return;
  }
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    s_base[g] = s_cnt[g] ? offsets[g] + atomicAdd(&fill[g], s_cnt[g]) : 0u;
    s_cnt[g] = 0;
  }
  __syncthreads();
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const uint32_t v = ids[p];
    const uint32_t w = dir > 0 ? (p + 1 < m ? ids[p + 1] : edge) : (p > 0 ? ids[p - 1] : edge);
    const uint32_t o = v / S;
    const uint32_t at = s_base[o] + atomicAdd(&s_cnt[o], 1u);
    send[at] = make_uint2(v, w);
  }
}

// The first and the last sorted id of this rank (NULL when it holds no position), for
// the stitch: out[0] = first, out[1] = last.
static __global__ void k_first_last_id(const Plan* __restrict__ plan, const uint32_t* __restrict__ ids0,
                                       const uint32_t* __restrict__ ids1, uint32_t m, uint32_t* __restrict__ out) {
  const uint32_t* ids = (plan->npasses & 1) ? ids1 : ids0;
  out[0] = m ? ids[0] : PBIT_NULL32;
  out[1] = m ? ids[m - 1] : PBIT_NULL32;
}


}  // namespace pbit
