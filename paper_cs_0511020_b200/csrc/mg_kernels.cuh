// mg_kernels.cuh -- kernels used only by the multi-GPU path (pbit_sort_list_mg).
// The single-GPU kernels (kernels.cuh) do the rest.  Rank r of G owns node ids
// [r*S, r*S + n_local) and, after the key-range exchange, the sorted positions
// [r*S, r*S + S) of the output.
#pragma once
#include "kernels.cuh"

namespace pbit {

// ============================================================================ rulers
// Which rank walked ruler r and where its records are in that rank's slots (the walk's
// WalkMap of every rank, mg.cu): static rulers r < Gs belong to rank r / bpr (slot
// r - q*bpr); the head's extra ruler Gs to the rank owning the head (slot bpr); rank q's
// dynamic rulers are Gs + 1 + q*dcap + k (slot bpr + 1 + k).  One rank: slot(r) = r.
struct MgRulers {
  FastDiv bpr, dcap;
  uint32_t Gs, head_owner, cap;
  __device__ __forceinline__ void locate(uint32_t r, uint32_t& q, uint32_t& slot) const {
    if (r < Gs) {
      q = bpr.div(r);
      slot = r - q * bpr.d;
    } else if (r == Gs) {
      q = head_owner;
      slot = bpr.d;
    } else {
      const uint32_t k = r - Gs - 1;
      q = dcap.div(k);
      slot = bpr.d + 1 + (k - q * dcap.d);
    }
  }
};

// ============================================================================ NCCL transport
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

// ============================================================================ peer transport (N4)
// The list-order chunk of positions [P0, P1) straight from the walkers' segment slots,
// which every rank maps (peer loads over NVLink; the local rank's own slots directly).
// Each warp copies GATHER_SEGS consecutive segments of the list at once.
struct PeerSlots {
  const void* slots[64];
};

template <int KB>
__global__ void __launch_bounds__(256)
k_mg_gather(const __grid_constant__ PeerSlots ps, MgRulers mr, uint32_t cap, const uint2* __restrict__ seg,
            const uint32_t* __restrict__ seg_ord, const uint32_t* __restrict__ seg_pos,
            const uint32_t* __restrict__ part_first, int rank, const uint32_t* __restrict__ nseg, uint32_t P0,
            uint32_t P1, typename KeyOf<KB>::T* __restrict__ keys_c, uint32_t* __restrict__ ids_c,
            const int* __restrict__ err) {
  using RT = typename Rec<KB>::T;
  if (*err || P0 >= P1) return;
  const uint32_t k0 = part_first[rank], ns = *nseg;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t kb = k0 + warp * GATHER_SEGS; kb < ns; kb += nwarps * GATHER_SEGS) {
    if (seg_pos[kb] >= P1) break;  // segments are in list order
    const RT* src[GATHER_SEGS];
    uint32_t lo[GATHER_SEGS], hi[GATHER_SEGS], pos[GATHER_SEGS];
    uint32_t mx = 0;
#pragma unroll
    for (int q = 0; q < GATHER_SEGS; ++q) {
      const uint32_t k = kb + q;
      lo[q] = hi[q] = pos[q] = 0;
      src[q] = nullptr;
      if (k < ns) {
        const uint32_t r = seg_ord[k], p = seg_pos[k], len = seg[r].x;
        uint32_t owner, slot;
        mr.locate(r, owner, slot);
        PBIT_ASSERT(owner < 64 && len <= mr.cap);
        src[q] = reinterpret_cast<const RT*>(ps.slots[owner]) + (size_t)slot * cap;
        pos[q] = p;
        lo[q] = max(p, P0) - p;             // overlap with [P0, P1), relative to the segment
        hi[q] = min(p + len, P1);
        hi[q] = hi[q] > p ? hi[q] - p : 0u;
        if (hi[q] < lo[q]) hi[q] = lo[q];
        mx = max(mx, hi[q] - lo[q]);
      }
    }
    for (uint32_t j = lane; j < mx; j += 32) {
      RT x[GATHER_SEGS];
#pragma unroll
      for (int q = 0; q < GATHER_SEGS; ++q)
        if (lo[q] + j < hi[q]) x[q] = src[q][lo[q] + j];
#pragma unroll
      for (int q = 0; q < GATHER_SEGS; ++q) {
        const uint32_t e = lo[q] + j;
        if (e < hi[q]) {
          const uint32_t at = pos[q] + e - P0;
          if constexpr (KB == 8) {
            keys_c[at] = ((unsigned long long)x[q].y << 32) | x[q].x;
            ids_c[at] = x[q].z;
          } else {
            keys_c[at] = x[q].x;
            ids_c[at] = x[q].y;
          }
        }
      }
    }
  }
}

// ============================================================================ histograms
// Histograms of every digit of m keys (a chunk in list order, or the received keys),
// warp-aggregated by hist_add (common.cuh); per-CTA counters are flushed to the global
// histogram once.
template <typename KeyT>
__global__ void __launch_bounds__(256)
k_chunk_hist(const KeyT* __restrict__ keys, uint32_t m, int K, int D, uint32_t* __restrict__ hist,
             const int* __restrict__ err) {
  extern __shared__ uint32_t s_hist[];
  if (*err) return;
  const int radix = 1 << K;
  for (int i = threadIdx.x; i < D * radix; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t p0 = blockIdx.x * blockDim.x; p0 < m; p0 += stride) {  // warp-uniform trip count
    const uint32_t p = p0 + threadIdx.x;
    const bool valid = p < m;
    const KeyT k = valid ? keys[p] : KeyT(0);
    for (int d = 0; d < D; ++d) hist_add(s_hist + d * radix, (uint32_t)(k >> (d * K)) & (uint32_t)(radix - 1), valid);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < D * radix; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// ============================================================================ splitters
// Exact splitters of the global (key, list position) order: split s sits
// at global rank x_s = min(n, (s+1)*S).  Radix refinement of k*_s = the key at sorted
// index x_s, 8 bits per round from the top, entirely on the device: per round every rank
// histograms the next 8-bit digit of its keys that match each splitter's prefix
// (k_split_count), the histograms are summed over the ranks (ncclAllReduce), and
// k_split_select appends to each prefix the largest digit c with
// below_s + #{keys with prefix_s and digit < c} <= x_s.  No host round trip.

// prefix[s] is non-decreasing in s, so a key matches the prefixes of a contiguous range of
// splitters; it is counted once, in the histogram of the first of them.
template <typename KeyT>
__global__ void __launch_bounds__(256)
k_split_count(const KeyT* __restrict__ keys, uint32_t m, uint32_t NS, const unsigned long long* __restrict__ prefix,
              int shift, uint32_t* __restrict__ hist, const int* __restrict__ err) {
  extern __shared__ uint32_t s_hist[];  // [NS][256]
  __shared__ unsigned long long s_pre[64];
  if (*err) return;
  for (uint32_t i = threadIdx.x; i < NS * 256; i += blockDim.x) s_hist[i] = 0;
  if (threadIdx.x < NS) s_pre[threadIdx.x] = prefix[threadIdx.x];
  __syncthreads();
  const int hi_shift = shift + 8;  // bits above the digit of this round
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
    const unsigned long long k = (unsigned long long)keys[p];
    const unsigned long long top = hi_shift >= 64 ? 0ull : (k >> hi_shift);
    uint32_t lo = 0, hi = NS;  // first s with prefix[s] >= top
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pre[mid] < top) lo = mid + 1; else hi = mid;
    }
    if (lo < NS && s_pre[lo] == top) atomicAdd(&s_hist[lo * 256 + (uint32_t)((k >> shift) & 255u)], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < NS * 256; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

static __global__ void k_split_select(uint32_t* __restrict__ hist, uint32_t NS, unsigned long long n,
                                      unsigned long long S, unsigned long long* __restrict__ prefix,
                                      unsigned long long* __restrict__ below) {
  __shared__ unsigned long long s_pre[64];
  const uint32_t s = threadIdx.x;
  if (s < NS) s_pre[s] = prefix[s];
  __syncthreads();
  if (s < NS) {
    uint32_t f = s;  // the splitter whose histogram holds the keys of this prefix
    while (f > 0 && s_pre[f - 1] == s_pre[s]) --f;
    const unsigned long long x = min(n, (unsigned long long)(s + 1) * S);
    const uint32_t* h = hist + f * 256;
    unsigned long long cum = 0, take = 0;
    uint32_t pick = 0;
    for (uint32_t c = 0; c < 256; ++c) {
      if (below[s] + cum <= x) { pick = c; take = cum; }
      cum += h[c];
    }
    below[s] += take;
    prefix[s] = (s_pre[s] << 8) | pick;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < NS * 256; i += blockDim.x) hist[i] = 0;  // for the next round
}

// Local bucket counts of the chunk (SplitTable buckets: 2*NS + 1 of them), warp-aggregated
// by hist_add.  kstar is read from the split table's staging area.
template <typename KeyT>
__global__ void __launch_bounds__(256)
k_split_buckets(const KeyT* __restrict__ keys, uint32_t m, const SplitTable* __restrict__ spt,
                uint32_t* __restrict__ cnt, const int* __restrict__ err) {
  __shared__ SplitTable sp;
  __shared__ uint32_t s_cnt[128];
  if (*err) return;
  for (uint32_t i = threadIdx.x; i < sizeof(SplitTable) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(&sp)[i] = reinterpret_cast<const uint32_t*>(spt)[i];
  if (threadIdx.x < 128) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t p0 = blockIdx.x * blockDim.x; p0 < m; p0 += stride) {
    const uint32_t p = p0 + threadIdx.x;
    const bool valid = p < m;
    const uint32_t b = valid ? split_bucket(sp, (unsigned long long)keys[p]) : 0u;
    hist_add(s_cnt, b, valid);
  }
  __syncthreads();
  if (threadIdx.x < 2 * sp.NS + 1 && s_cnt[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], s_cnt[threadIdx.x]);
}

// The exchange plan on the device, from every rank's bucket counts (cntall[q][b], all-
// gathered): per split s, lt_q = keys of rank q below k*_s, eq_q = keys equal to it; of
// the t_s = x_s - sum_q lt_q ties that go left, ranks take theirs in rank order (= list-
// position order: rank q's chunk holds the list positions before rank q+1's).  Same rule as
// the host planner pbit_mg_exchange_plan (mg.cu).  Writes, for rank r: the pass bases of
// its buckets, left[d] (first element of its bucket order going to rank d), dst_off[d]
// (where it lands in d's receive arrays), and recv[q] = {offset, count} of what r receives
// from q (the NCCL transport's receive plan).
static __global__ void k_split_plan(const uint32_t* __restrict__ cntall, uint32_t G, uint32_t r,
                                    unsigned long long n, unsigned long long S, SplitTable* __restrict__ spt,
                                    uint32_t* __restrict__ bases, uint32_t* __restrict__ recv) {
  if (threadIdx.x != 0) return;
  const uint32_t NS = spt->NS, NB = 2 * NS + 1;
  uint32_t left[64][65];  // left[q][d]: elements of rank q's bucket order going to ranks < d
  for (uint32_t q = 0; q < G; ++q) {
    uint32_t tot = 0;
    for (uint32_t b = 0; b < NB; ++b) tot += cntall[q * NB + b];
    left[q][0] = 0;
    left[q][G] = tot;
  }
  for (uint32_t s = 0; s < NS; ++s) {
    // the bucket holding the keys equal to k*_s: 2 j0 + 1, j0 = first split with that key
    uint32_t j0 = s;
    while (j0 > 0 && spt->kstar[j0 - 1] == spt->kstar[s]) --j0;
    unsigned long long L = 0;
    uint32_t lt[64], eq[64];
    for (uint32_t q = 0; q < G; ++q) {
      uint32_t a = 0;
      for (uint32_t b = 0; b <= 2 * j0; ++b) a += cntall[q * NB + b];
      lt[q] = a;
      eq[q] = cntall[q * NB + 2 * j0 + 1];
      L += a;
    }
    const unsigned long long x = min(n, (unsigned long long)(s + 1) * S);
    unsigned long long t = x > L ? x - L : 0ull;
    for (uint32_t q = 0; q < G; ++q) {
      const unsigned long long take = min((unsigned long long)eq[q], t);
      t -= take;
      left[q][s + 1] = lt[q] + (uint32_t)take;
    }
  }
  // bases of rank r's buckets (exclusive scan of its counts)
  uint32_t acc = 0;
  for (uint32_t b = 0; b < NB; ++b) { bases[b] = acc; acc += cntall[r * NB + b]; }
  for (uint32_t d = 0; d <= G; ++d) spt->left[d] = left[r][d];
  spt->G = G;
  for (uint32_t d = 0; d < G; ++d) {
    uint32_t roff = 0;  // what ranks q < r send to d lands first
    for (uint32_t q = 0; q < r; ++q) roff += left[q][d + 1] - left[q][d];
    spt->dst_off[d] = roff - left[r][d];  // mod 2^32
  }
  uint32_t racc = 0;
  for (uint32_t q = 0; q < G; ++q) {
    const uint32_t c = left[q][r + 1] - left[q][r];
    recv[2 * q] = racc;
    recv[2 * q + 1] = c;
    racc += c;
  }
}

// ============================================================================ stitch + relink routing
// The first and the last sorted id of this rank (NULL when it holds no position), for
// the stitch: out[0] = first, out[1] = last.
static __global__ void k_first_last_id(const uint32_t* __restrict__ ids, uint32_t m, uint32_t* __restrict__ out) {
  out[0] = m ? ids[0] : PBIT_NULL32;
  out[1] = m ? ids[m - 1] : PBIT_NULL32;
}

// edges[0] = the successor of this rank's last position (the next non-empty rank's first
// id, or NULL), edges[1] = the predecessor of its first position (the previous non-empty
// rank's last id, or NULL); edges[2] = rank 0's first id = the sorted list's head.
static __global__ void k_edges(const uint32_t* __restrict__ fl, uint32_t G, uint32_t r, uint32_t* __restrict__ edges) {
  uint32_t nx = PBIT_NULL32, pv = PBIT_NULL32;
  for (uint32_t d = r + 1; d < G; ++d)
    if (fl[2 * d] != PBIT_NULL32) { nx = fl[2 * d]; break; }
  for (int d = (int)r - 1; d >= 0; --d)
    if (fl[2 * d + 1] != PBIT_NULL32) { pv = fl[2 * d + 1]; break; }
  edges[0] = nx;
  edges[1] = pv;
  edges[2] = fl[0];
}

// Relink records of this rank's sorted positions, routed to the owner of v (owner = v / S):
// (v, succ) -- and with out_prev (v, succ, pred) -- with the stitch edges past either end.
// Phase 0 counts per owner; phase 1 scatters: a CTA claims its run in every owner's region
// with one atomic per owner (`fill`), and the lanes of a warp with the same owner (found by
// __match_any_sync) take consecutive places with one shared atomic.  dst[d] + base[d] is
// where this rank's records for owner d start: a peer's receive buffer (N4) or this rank's
// send buffer (NCCL transport).
struct PairDst {
  void* dst[64];
};

template <int W>
__global__ void __launch_bounds__(256)
k_pairs_owner(const uint32_t* __restrict__ ids, uint32_t m, const uint32_t* __restrict__ edges, FastDiv S, uint32_t G,
              uint32_t* __restrict__ counts, const uint32_t* __restrict__ base, uint32_t* __restrict__ fill,
              const __grid_constant__ PairDst pd, int scatter, const int* __restrict__ err) {
  using R = typename RelinkRec<W>::T;
  __shared__ uint32_t s_cnt[64];
  __shared__ uint32_t s_base[64];
  if (*err) return;
  if (threadIdx.x < 64) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t per = (m + gridDim.x - 1) / gridDim.x;
  const uint32_t p0 = blockIdx.x * per, p1 = min(m, p0 + per);
  const uint32_t lane = threadIdx.x & 31;
  // every warp runs the same number of trips (the shuffles need whole warps)
  auto owner_rank = [&](uint32_t p, bool valid, uint32_t& o, uint32_t& peers) {
    o = valid ? S.div(ids[p]) : 0xFFFFFFFFu;
    peers = __match_any_sync(0xffffffffu, o);
  };
  for (uint32_t q0 = p0; q0 < p1; q0 += blockDim.x) {
    const uint32_t p = q0 + threadIdx.x;
    const bool valid = p < p1;
    uint32_t o, peers;
    owner_rank(p, valid, o, peers);
    if (valid && (peers & lanemask_lt()) == 0u) atomicAdd(&s_cnt[o], (uint32_t)__popc(peers));
  }
  __syncthreads();
  if (!scatter) {
    if (threadIdx.x < G && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]);
    return;
  }
  if (threadIdx.x < G) {
    s_base[threadIdx.x] = s_cnt[threadIdx.x] ? base[threadIdx.x] + atomicAdd(&fill[threadIdx.x], s_cnt[threadIdx.x]) : 0u;
    s_cnt[threadIdx.x] = 0;
  }
  __syncthreads();
  const uint32_t e_next = edges[0], e_prev = edges[1];
  for (uint32_t q0 = p0; q0 < p1; q0 += blockDim.x) {
    const uint32_t p = q0 + threadIdx.x;
    const bool valid = p < p1;
    uint32_t o, peers;
    owner_rank(p, valid, o, peers);
    const int leader = __ffs(peers) - 1;
    uint32_t at = 0;
    if (valid && lane == (uint32_t)leader) at = atomicAdd(&s_cnt[o], (uint32_t)__popc(peers));
    at = __shfl_sync(0xffffffffu, at, leader < 0 ? 0 : leader) + __popc(peers & lanemask_lt());
    if (valid) {
      R rec;
      rec.x = ids[p];
      rec.y = p + 1 < m ? ids[p + 1] : e_next;
      if constexpr (W == 3) rec.z = p > 0 ? ids[p - 1] : e_prev;
      PBIT_ASSERT(o < G);
      reinterpret_cast<R*>(pd.dst[o])[s_base[o] + at] = rec;
    }
  }
  __threadfence_system();  // peer stores (the owner's window): visible before the barrier collective
}

// The routing plan of the relink records from the all-gathered counts (cntall[q][d] =
// records rank q sends to owner d): base[d] = where rank r's records start in d's receive
// buffer (peer transport) and, for the NCCL transport, sbase[d] = where they start in r's
// send buffer, plus recv[q] = {offset, count} of what r receives from q.
static __global__ void k_pairs_plan(const uint32_t* __restrict__ cntall, uint32_t G, uint32_t r,
                                    uint32_t* __restrict__ base, uint32_t* __restrict__ sbase,
                                    uint32_t* __restrict__ recv) {
  if (threadIdx.x != 0) return;
  uint32_t sacc = 0, racc = 0;
  for (uint32_t d = 0; d < G; ++d) {
    uint32_t b = 0;
    for (uint32_t q = 0; q < r; ++q) b += cntall[q * G + d];
    base[d] = b;
    sbase[d] = sacc;
    sacc += cntall[r * G + d];
    recv[2 * d] = racc;
    recv[2 * d + 1] = cntall[d * G + r];
    racc += cntall[d * G + r];
  }
}

}  // namespace pbit
