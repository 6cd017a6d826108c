// kernels.cuh -- the sm_100a kernels of the Pbit hot path.
//
//   k_pack      a1/a2  AoS (key,next) records + histograms of every digit (one sweep);
//                      applies the key-order map (signed / float / descending, N1)
//   k_walk      a1     ruling-set walk: every segment written in list order to its slot
//   k_rank_*    a1     ruler-list ranking (second ruling set + pointer jumping);
//                      validates the chain
//   k_gather    a1     segments -> list-order (key, id) arrays (only when no pass runs;
//                      otherwise pass 0 gathers its tiles itself)
//   k_plan      a3     exclusive scans of the digit histograms -> bucket bases, pass plan
//   k_onesweep  a3/a4  one stable LSD pass: TMA tile loads, in-warp ranking (lane-ordered
//                      shared atomics, or ballots), decoupled lookback, smem-staged
//                      coalesced scatter; SRC_SPLIT: the multi-GPU key-range partition,
//                      stored straight into the destination ranks' arrays
//   k_materialize N3   the sorted node ids / keys (pbit_opts.out_order / out_keys)
//   k_relink_*  a5     out_next (and out_prev, N2) from the sorted ids (the paper's merge,
//                      P:273-280): (v, succ[, pred]) records binned by v in MSD partition
//                      levels, applied in shared-memory windows
//   k_array_*   N3     pbit_sort_array's prep (key map + histograms) and finish
//
// Paper anchors: the split loop is the stable scatter; the end-marker
// recursion is the ascending order of the bucket bases; merge is relink.
#pragma once
#include "common.cuh"

#include <cooperative_groups.h>
#include <type_traits>

namespace pbit {

// Programmatic dependent launch (launch_pdl in launch.cuh): a kernel of the pipeline may be
// launched while its predecessor is still finishing; it waits here for the predecessor's
// completion and memory before touching anything, then lets its own successor launch.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int PACK_THREADS = 256;
constexpr int WALK_THREADS = 256;
#ifndef PBIT_WALK_FLUSH
#define PBIT_WALK_FLUSH 128
#endif
#ifndef PBIT_WALK_FLUSH64
#define PBIT_WALK_FLUSH64 256
#endif
// walk record stores per group: 16 records either way (8 B records for keys <= 32 bits,
// 16 B for 64-bit keys; measured: u32 256 B groups 14.4 ms vs 7.37, u64 128 B 4.51 ms vs
// 256 B 4.22 ms on C4)
constexpr int WALK_FLUSH_BYTES = PBIT_WALK_FLUSH;
constexpr int WALK_FLUSH_BYTES64 = PBIT_WALK_FLUSH64;
#ifndef PBIT_SWEEP_THREADS
#define PBIT_SWEEP_THREADS 512
#endif
constexpr int SWEEP_THREADS = PBIT_SWEEP_THREADS;  // 16 warps x 16 items: 8192-item tiles halve the lookback traffic
constexpr int SWEEP_WARPS = SWEEP_THREADS / 32;
#ifndef PBIT_SWEEP_IPT
#define PBIT_SWEEP_IPT 16
#endif
#ifndef PBIT_WCNT32
#define PBIT_WCNT32 0
#endif
constexpr int SWEEP_IPT32 = PBIT_SWEEP_IPT;                       // items per thread, keys <= 32 bits
#ifndef PBIT_SWEEP_IPT64
#define PBIT_SWEEP_IPT64 (PBIT_SWEEP_IPT == 16 ? 12 : PBIT_SWEEP_IPT * 3 / 4 + 1)
#endif
constexpr int SWEEP_IPT64 = PBIT_SWEEP_IPT64;  // 64-bit keys
// write-out of the stable passes: 128-bit stores over 16 B-aligned groups of every digit
// run (1), or one 4 B store per element, consecutive threads on consecutive elements (0)
// decoupled lookback: ns to sleep when the nearest predecessor has published nothing new
// (0 = poll again at once)
#ifndef PBIT_LB_SLEEP
#define PBIT_LB_SLEEP 0
#endif
// in-warp ranking: branch on the warp-uniform "all lanes share one digit" test (1) or
// select the addend per lane and skip zero addends (0)
#ifndef PBIT_RANK_UNIBRANCH
#define PBIT_RANK_UNIBRANCH 1
#endif
#ifndef PBIT_VEC_STORE
#define PBIT_VEC_STORE 0
#endif
// in-warp ranking: the "all lanes share one digit" test by match.all (1) or by a shuffle of
// lane 0's digit and a vote (0)
#ifndef PBIT_RANK_MATCHALL
#define PBIT_RANK_MATCHALL 1
#endif
// in-warp ranking without a branch around the atomic: lanes with nothing to add hit their
// own scratch word (1)
#ifndef PBIT_RANK_PRED
#define PBIT_RANK_PRED 1
#endif
// pass kernel: the per-digit scan keeps the warps' exclusive prefixes in registers (1)
// instead of writing them to the warp counters and re-reading them (0)
#ifndef PBIT_SCAN_REG
#define PBIT_SCAN_REG 1
#endif
// pass 0 gather: lanes copy their own even-aligned segments by TMA in parallel (1) instead
// of the whole warp taking every segment in turn (0)
#ifndef PBIT_GATHER_LANEBULK
#define PBIT_GATHER_LANEBULK 1
#endif
// relink partition: the next tile's bin claims issued before the current tile's write-out (1)
#ifndef PBIT_PART_PIPE
#define PBIT_PART_PIPE 0
#endif
#ifndef PBIT_PP_DBG
#define PBIT_PP_DBG 0  // bisection knobs of the pipelined loop: 1 proxy fence, 2 claims after the write-out, 4 serial
#endif
// pass kernel: tiles ahead of its own whose keys and ids a CTA prefetches into L2
// (cp.async.bulk.prefetch.L2), about one resident wave (0 = none)
#ifndef PBIT_SWEEP_PREFETCH
#define PBIT_SWEEP_PREFETCH 74
#endif
// first pass (gather from the walk's slots): prefetch the segment table entries of the tile
// PBIT_SWEEP_PREFETCH ahead into L2 (1) or not (0)
#ifndef PBIT_GATHER_META_PREFETCH
#define PBIT_GATHER_META_PREFETCH 1
#endif
// per-warp digit counters of the pass ranking: u32 (one word per digit: no two digits
// share a word, so ATOMS lanes collide only on equal digits) or u16 pairs (half the smem)
using WCnt = std::conditional_t<PBIT_WCNT32 != 0, uint32_t, uint16_t>;

// ============================================================================ key order
// Order-preserving map of a key's bits to the unsigned integer the passes sort by
// (NEXT row N1).  Applied once, in the pack: every later kernel sees sort keys only,
// and nothing maps them back (the output is the relinked list, not the keys).
//   signed   flip the sign bit: two's complement order = unsigned order
//   float    sign bit set: flip all bits; else set the sign bit -- sign-magnitude order
//            of the bit patterns, the order of the paper's sign split + mantissa-then-
//            characteristic passes (reading Q18)
//   descending  complement the result: a stable ascending sort of ~k is the stable
//            descending sort of k (equal keys keep input order)
struct KeyMap {
  int kind;        // PBIT_KEY_UNSIGNED / SIGNED / FLOAT
  int descending;
  __host__ __device__ __forceinline__ unsigned long long operator()(unsigned long long k, int bits) const {
    const unsigned long long all = bits == 64 ? ~0ull : ((1ull << bits) - 1);
    const unsigned long long sign = 1ull << (bits - 1);
    if (kind == 1) k ^= sign;
    else if (kind == 2) k = (k & sign) ? (~k & all) : (k | sign);
    if (descending) k = ~k & all;
    return k;
  }
  __host__ __device__ __forceinline__ bool identity() const { return kind == 0 && !descending; }
  // the key bits back from a sort key (pbit_sort_array's out_keys)
  __host__ __device__ __forceinline__ unsigned long long inverse(unsigned long long k, int bits) const {
    const unsigned long long all = bits == 64 ? ~0ull : ((1ull << bits) - 1);
    const unsigned long long sign = 1ull << (bits - 1);
    if (descending) k = ~k & all;
    if (kind == 1) k ^= sign;
    else if (kind == 2) k = (k & sign) ? (k & ~sign) : (~k & all);
    return k;
  }
};

// ============================================================================ a1/a2: pack
// Reads key[v], next[v] (streaming, coalesced), writes the AoS record kn[v], and counts
// every digit of every key into a per-CTA smem histogram (flushed once per CTA).
// Four independent nodes per thread and iteration: 4x the loads in flight of one node
// per thread, every access still lane-contiguous.
//
// The counting is one shared atomic per digit (hist_add mode 0).  Warp-aggregated
// counting (PBIT_HIST_MODE 1: __match_any_sync groups, one atomic per distinct digit; 2:
// lane 0's digit by __ballot_sync) was measured on B200 and loses: C3 pack 0.78 ms plain,
// 6.65 ms match.any, 2.19 ms ballot; C5 4.0 / 17.5 / 8.1 ms.  The modes need
// the whole warp in every trip, so they take the warp-uniform loop below.
template <int KB>
__device__ __forceinline__ void pack_one(unsigned long long k, uint32_t nx, uint32_t v, bool ok, uint32_t n_ids,
                                         typename Rec<KB>::T* __restrict__ kn, uint32_t* s_hist, int radix,
                                         uint32_t mask, int K, int D, const KeyMap& km, int& bad) {
  if (ok) {
    bad |= (nx != PBIT_NULL32) & (nx >= n_ids);
    if (!km.identity()) k = km(k, KB * 8);
    if constexpr (KB == 8) kn[v] = make_uint4((uint32_t)k, (uint32_t)(k >> 32), nx, 0u);
    else kn[v] = make_uint2((uint32_t)k, nx);
  }
  for (int d = 0; d < D; ++d) hist_add(s_hist + d * radix, (uint32_t)(k >> (d * K)) & mask, ok);
}

template <int KB>
__global__ void __launch_bounds__(PACK_THREADS)
k_pack(const void* __restrict__ keys, const uint32_t* __restrict__ next, uint32_t n, uint32_t n_ids,
       typename Rec<KB>::T* __restrict__ kn, uint32_t* __restrict__ hist, int K, int D,
       int* __restrict__ err, KeyMap km) {
  pdl_enter();
  using KT = std::conditional_t<KB == 1, uint8_t, std::conditional_t<KB == 2, uint16_t,
             std::conditional_t<KB == 4, uint32_t, unsigned long long>>>;
  constexpr int U = 4;  // independent nodes per thread and iteration (all loads issued first)
  extern __shared__ uint32_t s_hist[];
  const int radix = 1 << K;
  const int nb = D * radix;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const uint32_t mask = radix - 1;
  int bad = 0;
  const KT* __restrict__ kp = reinterpret_cast<const KT*>(keys);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if constexpr (PBIT_HIST_MODE == 0) {
    uint32_t v = tid;
    for (; (unsigned long long)v + (U - 1) * (unsigned long long)stride < n; v += U * stride) {
      KT k[U];
      uint32_t nx[U];
#pragma unroll
      for (int e = 0; e < U; ++e) {
        k[e] = __ldcs(kp + v + e * stride);
        nx[e] = __ldcs(next + v + e * stride);
      }
#pragma unroll
      for (int e = 0; e < U; ++e)
        pack_one<KB>((unsigned long long)k[e], nx[e], v + e * stride, true, n_ids, kn, s_hist, radix, mask, K, D,
                     km, bad);
    }
    for (; v < n; v += stride)
      pack_one<KB>((unsigned long long)kp[v], __ldcs(next + v), v, true, n_ids, kn, s_hist, radix, mask, K, D, km,
                   bad);
  } else {
    const uint32_t lane = threadIdx.x & 31u;
    for (unsigned long long v0 = tid - lane; v0 < n; v0 += (unsigned long long)U * stride) {  // warp-uniform
      KT k[U];
      uint32_t nx[U];
      bool ok[U];
#pragma unroll
      for (int e = 0; e < U; ++e) {
        const unsigned long long v = v0 + lane + (unsigned long long)e * stride;
        ok[e] = v < n;
        k[e] = ok[e] ? __ldcs(kp + v) : KT(0);
        nx[e] = ok[e] ? __ldcs(next + v) : 0u;
      }
#pragma unroll
      for (int e = 0; e < U; ++e)
        pack_one<KB>((unsigned long long)k[e], nx[e], (uint32_t)(v0 + lane + (unsigned long long)e * stride), ok[e],
                     n_ids, kn, s_hist, radix, mask, K, D, km, bad);
    }
  }
  if (bad) atomicOr(err, E_BAD_INDEX);
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// ============================================================================ a1: walk
// Which rulers one walk launch handles and where their records go.  Ruler indices are
// global (they index the segment table); slots are local to the launching GPU.
//   static rulers  r in [r_lo, r_lo + n_static)   start at sel.node_of(r), slot r - r_lo
//   the head       r = head_idx (unless NULL)      starts at the head,      slot head_slot
//   dynamic        r = dyn_base + k                opened by a cut segment, slot dyn_slot0 + k
// Single GPU: r_lo = 0 and slot(r) = r (head_idx = head_slot = R, dyn_base = dyn_slot0 =
// R_static).
struct WalkMap {
  uint32_t r_lo, n_static, head_idx, head_slot, dyn_base, dyn_slot0;
  __host__ __device__ __forceinline__ uint32_t count() const { return n_static + (head_idx != PBIT_NULL32 ? 1u : 0u); }
};

// Where the walk reads kn[u]: one array (single GPU, or the multi-GPU replica), or the
// owners' slices through peer pointers (multi-GPU, NEXT row N4: rank q owns ids
// [q*S, q*S + S) and its slice is mapped into every rank's address space).
template <typename RT>
struct KnSrc {
  const RT* kn;            // !PEER: node-indexed records
  const RT* peer[64];      // PEER: rank q's slice (local index u - q*S)
  FastDiv S;               // PEER: the rank slice
};

template <typename RT, bool PEER>
__device__ __forceinline__ RT load_kn(const KnSrc<RT>& src, const RT* const* s_peer, uint32_t u) {
  const RT* p;
  if constexpr (PEER) {
    const uint32_t q = src.S.div(u);
    p = s_peer[q] + (u - q * src.S.d);
  } else {
    p = src.kn + u;
  }
  if constexpr (sizeof(RT) == 16) return ld_stream_u4(reinterpret_cast<const uint4*>(p));
  else return ld_stream_u2(reinterpret_cast<const uint2*>(p));
}

// One thread walks one segment at a time: from its ruler node along next[] until the
// next ruler (or NULL), writing (key, id) of each visited node into the segment's slot
// in list order -- the same sequential traversal as the paper's split loop L=L->next
// (P:353), which is what makes the result stable.  A segment longer than `cap` is cut:
// the walker opens a dynamic ruler (WalkMap) at the current node and goes on.
// Rulers are handed out per CTA from a contiguous range through a smem counter.
template <int KB, bool PEER = false>
__global__ void __launch_bounds__(WALK_THREADS)
k_walk(const __grid_constant__ KnSrc<typename Rec<KB>::T> src, RulerSel sel, WalkMap wm, uint32_t head,
       typename Rec<KB>::T* __restrict__ slots, uint32_t cap, uint2* __restrict__ seg,
       uint32_t* __restrict__ dyn_count, uint32_t dyn_cap, uint32_t per_cta, int* __restrict__ err,
       int no_writes) {  // no_writes: timing experiments only
  pdl_enter();
  using RT = typename Rec<KB>::T;
  // Records are staged in registers and stored in groups of WALK_FLUSH_BYTES, always as
  // whole 32 B sectors: a partial-sector store costs an HBM read-modify-write on B200.
  constexpr int B = (KB == 8 ? WALK_FLUSH_BYTES64 : WALK_FLUSH_BYTES) / (int)sizeof(RT);
  __shared__ uint32_t s_next;
  __shared__ const RT* s_peer[PEER ? 64 : 1];
  if (threadIdx.x == 0) s_next = 0;
  if constexpr (PEER)
    if (threadIdx.x < 64) s_peer[threadIdx.x] = src.peer[threadIdx.x];
  __syncthreads();
  const uint32_t n = sel.n;
  const uint32_t total = wm.count();
  const uint32_t lo = blockIdx.x * per_cta;
  const uint32_t hi = min(lo + per_cta, total);
  RT buf[B];
  for (;;) {
    const uint32_t i = lo + atomicAdd(&s_next, 1u);
    if (i >= hi) break;
    const bool is_head = i == wm.n_static;
    uint32_t u = is_head ? head : sel.node_of(wm.r_lo + i);
    uint32_t cur = is_head ? wm.head_idx : wm.r_lo + i, j = 0;  // j: records of segment `cur` already stored
    RT* out = slots + (size_t)(is_head ? wm.head_slot : i) * cap;
    for (;;) {
      // one group of up to B steps, unrolled so that buf[] is indexed statically
      uint32_t m = 0, succ = PBIT_NULL32;
      bool end = false;
#pragma unroll
      for (int q = 0; q < B; ++q) {
        if (!end) {
          RT x = load_kn<RT, PEER>(src, s_peer, u);
          uint32_t v;
          if constexpr (KB == 8) { v = x.z; x.z = u; } else { v = x.y; x.y = u; }
          buf[q] = x;
          m = q + 1;
          if (v == PBIT_NULL32) end = true;
          else if (v >= n) { atomicOr(err, E_BAD_INDEX); end = true; }
          else if (sel.is_ruler(v)) { succ = v >> sel.s_log2; end = true; }
          u = v;
        }
      }
      PBIT_ASSERT(j + m <= cap);
      if (!no_writes) {
        uint4* o = reinterpret_cast<uint4*>(out + j);
        const uint4* bb = reinterpret_cast<const uint4*>(buf);
        if (m == (uint32_t)B) {
#pragma unroll
          for (int q = 0; q < B * (int)sizeof(RT) / 16; ++q) o[q] = bb[q];
        } else {  // segment end: whole 32 B sectors (the slot has room: cap % B == 0)
          const uint32_t nsec = (m * (uint32_t)sizeof(RT) + 31u) / 32u;
#pragma unroll
          for (int q = 0; q < B * (int)sizeof(RT) / 32; ++q)
            if ((uint32_t)q < nsec) { o[2 * q] = bb[2 * q]; o[2 * q + 1] = bb[2 * q + 1]; }
        }
      }
      j += m;
      if (end) {
        seg[cur] = make_uint2(j, succ);
        break;
      }
      if (j == cap) {  // cap is a multiple of B
        const uint32_t k = atomicAdd(dyn_count, 1u);
        if (k >= dyn_cap) { atomicOr(err, E_DYN_FULL); seg[cur] = make_uint2(j, PBIT_NULL32); break; }
        const uint32_t r2 = wm.dyn_base + k;
        seg[cur] = make_uint2(cap, r2);
        cur = r2; j = 0; out = slots + (size_t)(wm.dyn_slot0 + k) * cap;
      }
    }
  }
}

// ============================================================================ a1: rank
// The segments form the ruler list (seg[r] = {nodes in segment r, next ruler}).  It is
// ranked by a second ruling set: sub-rulers (one per block of 2^s2 ruler ids, by hash,
// plus the head's ruler) sum their sub-segments (walk A, L2-resident reads), the short
// sub-ruler list is ranked by pointer jumping (Wyllie), and walk B hands every ruler its
// distance to the end of the list: dist[r] = nodes from the first node of segment r to
// the end.  Segment r then occupies list positions [n - dist[r], n - dist[r] + len[r]).
static __global__ void k_rank_walk_a(const uint2* __restrict__ seg, RulerSel sub, uint32_t R_static,
                              const uint32_t* __restrict__ dyn_count, uint32_t dyn_cap, uint32_t head_ruler,
                              uint32_t nsub, unsigned long long* __restrict__ sdist, uint32_t* __restrict__ scnt,
                              uint32_t* __restrict__ ssucc, int* __restrict__ err) {
  pdl_enter();
  if (*err) return;
  const uint32_t R = R_static + min(*dyn_count, dyn_cap);
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nsub; q += gridDim.x * blockDim.x) {
    const uint32_t rq = q < sub.R ? sub.node_of(q) : head_ruler;
    if (rq >= R || seg[rq].x == 0) { sdist[q] = 0; scnt[q] = 0; ssucc[q] = PBIT_NULL32; continue; }  // unused entry
    unsigned long long acc = 0;
    uint32_t r = rq, steps = 0, succ = PBIT_NULL32;
    for (;;) {
      const uint2 x = seg[r];
      acc += x.x;
      if (x.y == PBIT_NULL32) break;
      if (sub.is_ruler(x.y)) { succ = x.y >> sub.s_log2; break; }
      if (++steps > R) { atomicOr(err, E_CHAIN); break; }  // ruler cycle without a sub-ruler
      r = x.y;
    }
    sdist[q] = acc;
    scnt[q] = steps + 1;  // rulers in this sub-segment
    ssucc[q] = succ;
  }
}

static __global__ void k_rank_jump(const unsigned long long* __restrict__ d_in, const uint32_t* __restrict__ c_in,
                            const uint32_t* __restrict__ s_in, unsigned long long* __restrict__ d_out,
                            uint32_t* __restrict__ c_out, uint32_t* __restrict__ s_out, uint32_t m,
                            const int* __restrict__ err) {
  pdl_enter();
  if (*err) return;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const uint32_t s = s_in[r];
    unsigned long long d = d_in[r];
    uint32_t c = c_in[r];
    uint32_t s2 = s;
    if (s != PBIT_NULL32) { d += d_in[s]; c += c_in[s]; s2 = s_in[s]; }
    d_out[r] = d;
    c_out[r] = c;
    s_out[r] = s2;
  }
}

// All pointer-jumping rounds in ONE cooperative launch (grid-wide barrier between rounds)
// instead of one launch per round: the rounds are ~8 us each, mostly launch latency even
// with programmatic dependent launch.  The blocks of this one launch wait on each other
// at the barrier (cooperative launch: all of them are resident).  Ends with the check of
// k_rank_check; the result is in buffer (rounds & 1).
static __global__ void __launch_bounds__(256)
k_rank_jump_grid(unsigned long long* __restrict__ d0, uint32_t* __restrict__ c0, uint32_t* __restrict__ s0,
                 unsigned long long* __restrict__ d1, uint32_t* __restrict__ c1, uint32_t* __restrict__ s1, uint32_t m,
                 int rounds, uint32_t head_sub, uint32_t n, int* __restrict__ err) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  if (*err) return;  // written by earlier kernels only: the same value in every block
  for (int r = 0; r < rounds; ++r) {
    const bool odd = r & 1;
    const unsigned long long* d_in = odd ? d1 : d0;
    const uint32_t* c_in = odd ? c1 : c0;
    const uint32_t* s_in = odd ? s1 : s0;
    unsigned long long* d_out = odd ? d0 : d1;
    uint32_t* c_out = odd ? c0 : c1;
    uint32_t* s_out = odd ? s0 : s1;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
      const uint32_t sx = s_in[i];
      unsigned long long d = d_in[i];
      uint32_t c = c_in[i], s2 = sx;
      if (sx != PBIT_NULL32) { d += d_in[sx]; c += c_in[sx]; s2 = s_in[sx]; }
      d_out[i] = d;
      c_out[i] = c;
      s_out[i] = s2;
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const bool odd = rounds & 1;
    const uint32_t* s = odd ? s1 : s0;
    const unsigned long long* d = odd ? d1 : d0;
    if (s[head_sub] != PBIT_NULL32 || d[head_sub] != (unsigned long long)n) atomicOr(err, E_CHAIN);
  }
}

// Small ruler lists (nsub <= RANK_SMALL): all pointer-jumping rounds in one CTA with the
// arrays in shared memory (one launch instead of log2(nsub) + 1), then the check of
// k_rank_check; results back in place (d, c, s).
constexpr int RANK_SMALL = 6144;  // 2 x 6144 x 16 B = 192 KB of shared memory
static __global__ void __launch_bounds__(1024)
k_rank_jump_block(unsigned long long* __restrict__ d, uint32_t* __restrict__ c, uint32_t* __restrict__ s, uint32_t m,
                  int rounds, uint32_t head_sub, uint32_t n, int* __restrict__ err) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char sraw[];
  unsigned long long* sd = reinterpret_cast<unsigned long long*>(sraw);  // [2][RANK_SMALL]
  uint32_t* sc = reinterpret_cast<uint32_t*>(sd + 2 * RANK_SMALL);      // [2][RANK_SMALL]
  uint32_t* ss = sc + 2 * RANK_SMALL;                                   // [2][RANK_SMALL]
  if (*err) return;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) { sd[i] = d[i]; sc[i] = c[i]; ss[i] = s[i]; }
  __syncthreads();
  int cur = 0;
  for (int r = 0; r < rounds; ++r) {
    const uint32_t a = cur * RANK_SMALL, b = (cur ^ 1) * RANK_SMALL;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t nx = ss[a + i];
      unsigned long long dd = sd[a + i];
      uint32_t cc = sc[a + i], n2 = nx;
      if (nx != PBIT_NULL32) { dd += sd[a + nx]; cc += sc[a + nx]; n2 = ss[a + nx]; }
      sd[b + i] = dd; sc[b + i] = cc; ss[b + i] = n2;
    }
    cur ^= 1;
    __syncthreads();
  }
  const uint32_t a = cur * RANK_SMALL;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) { d[i] = sd[a + i]; c[i] = sc[a + i]; s[i] = ss[a + i]; }
  if (threadIdx.x == 0 && (ss[a + head_sub] != PBIT_NULL32 || sd[a + head_sub] != (unsigned long long)n))
    atomicOr(err, E_CHAIN);
}

// Validation (reading Q10): the chain from the head must end (succ NULL) and hold exactly
// n nodes; then every node lies on it.
static __global__ void k_rank_check(const unsigned long long* __restrict__ dist, const uint32_t* __restrict__ succ,
                             uint32_t head_sub, uint32_t n, int* __restrict__ err) {
  pdl_enter();
  if (*err) return;
  if (succ[head_sub] != PBIT_NULL32 || dist[head_sub] != (unsigned long long)n) atomicOr(err, E_CHAIN);
}

// Walk B also numbers the segments in list order: seg_ord[k] = the k-th segment of the
// list, so later kernels visit segments in list order (adjacent output runs are then
// written close together in time and their shared boundary sectors merge in L2).
static __global__ void k_rank_walk_b(const uint2* __restrict__ seg, RulerSel sub, uint32_t R_static,
                              const uint32_t* __restrict__ dyn_count, uint32_t dyn_cap, uint32_t head_ruler,
                              uint32_t nsub, uint32_t head_sub, const unsigned long long* __restrict__ sdist,
                              const uint32_t* __restrict__ scnt, uint32_t* __restrict__ dist,
                              uint32_t* __restrict__ seg_ord, uint32_t* __restrict__ seg_pos,
                              uint32_t* __restrict__ tile_first, uint32_t tile, uint32_t n,
                              uint32_t* __restrict__ nseg_out, const int* __restrict__ err) {
  pdl_enter();
  if (*err) return;
  const uint32_t R = R_static + min(*dyn_count, dyn_cap);
  const uint32_t total = scnt[head_sub];  // segments on the chain (= R for a valid list)
  if (blockIdx.x == 0 && threadIdx.x == 0) *nseg_out = total;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nsub; q += gridDim.x * blockDim.x) {
    const uint32_t rq = q < sub.R ? sub.node_of(q) : head_ruler;
    if (rq >= R || seg[rq].x == 0) continue;
    uint32_t D = (uint32_t)sdist[q];
    uint32_t k = total - scnt[q];
    uint32_t r = rq;
    for (;;) {
      dist[r] = D;
      const uint2 x = seg[r];
      const uint32_t pos = n - D;  // list position of the segment's first node
      seg_pos[k] = pos;
      // every tile (or, in the multi-GPU path, rank chunk) whose first position lies in
      // this segment starts at it (single GPU: segments are shorter than a tile, so at
      // most one; multi-GPU segments are not cut and may span several chunks)
      for (uint32_t tb = (pos + tile - 1) / tile; (unsigned long long)tb * tile < (unsigned long long)pos + x.x; ++tb)
        tile_first[tb] = k;
      seg_ord[k++] = r;
      D -= x.x;
      if (x.y == PBIT_NULL32 || sub.is_ruler(x.y)) break;
      r = x.y;
    }
  }
}

// ============================================================================ a1: gather
// Segment r occupies list positions [n - dist[r], n - dist[r] + len[r]).  Each warp
// copies GATHER_SEGS consecutive segments of the list at once (their loads in flight
// together) from the slots to the list-order arrays; both sides are contiguous runs.
constexpr int GATHER_SEGS = 4;
template <int KB>
__global__ void __launch_bounds__(256)
k_gather(const typename Rec<KB>::T* __restrict__ slots, uint32_t cap,
         const uint2* __restrict__ seg, const uint32_t* __restrict__ dist,
         const uint32_t* __restrict__ seg_ord, const uint32_t* __restrict__ nseg, uint32_t n,
         typename KeyOf<KB>::T* __restrict__ keys_lo, uint32_t* __restrict__ ids_lo,
         const Plan* __restrict__ plan, const int* __restrict__ err) {
  pdl_enter();
  using RT = typename Rec<KB>::T;
  if (*err) return;
  if (plan->npasses != 0) return;  // the first pass gathers the segments itself
  const uint32_t R = *nseg;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r0 = warp * GATHER_SEGS; r0 < R; r0 += nwarps * GATHER_SEGS) {
    uint32_t len[GATHER_SEGS], off[GATHER_SEGS], rr[GATHER_SEGS];
#pragma unroll
    for (int q = 0; q < GATHER_SEGS; ++q) {
      const uint32_t k = r0 + q;
      rr[q] = k < R ? seg_ord[k] : 0u;
      len[q] = k < R ? seg[rr[q]].x : 0u;
      off[q] = k < R ? n - dist[rr[q]] : 0u;
    }
    uint32_t mx = 0;
#pragma unroll
    for (int q = 0; q < GATHER_SEGS; ++q) mx = max(mx, len[q]);
    for (uint32_t j = lane; j < mx; j += 32) {
      RT x[GATHER_SEGS];
#pragma unroll
      for (int q = 0; q < GATHER_SEGS; ++q)
        if (j < len[q]) x[q] = __ldcs(slots + (size_t)rr[q] * cap + j);
#pragma unroll
      for (int q = 0; q < GATHER_SEGS; ++q) {
        if (j < len[q]) {
          if constexpr (KB == 8) {
            keys_lo[off[q] + j] = ((unsigned long long)x[q].y << 32) | x[q].x;
            ids_lo[off[q] + j] = x[q].z;
          } else {
            keys_lo[off[q] + j] = x[q].x;
            ids_lo[off[q] + j] = x[q].y;
          }
        }
      }
    }
  }
}

// ============================================================================ a3: plan
// Exclusive scan of each digit's histogram (bucket bases, ascending = the ascending
// end-marker order of P:379-380) and the list of non-trivial digits.  One CTA.
static __global__ void __launch_bounds__(256)
k_plan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ bases, Plan* __restrict__ plan,
       int D, int K, uint32_t n, const int* __restrict__ err) {
  pdl_enter();
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_np;
  const int radix = 1 << K;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) { s_np = 0; plan->skewed[0] = plan->skewed[1] = 0u; }
  __syncthreads();
  for (int d = 0; d < D; ++d) {
    // radix <= 256 == blockDim
    const uint32_t c = t < radix ? hist[d * radix + t] : 0u;
    const int trivial = __syncthreads_or(c == n);
    const int skewed = __syncthreads_or(c > n / 16u);
    if (t == 0 && skewed) plan->skewed[d >> 5] |= 1u << (d & 31);
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
// One stable counting-sort pass on digit a.digit (single-pass scan with decoupled
// lookback, Merrill & Garland).  Tile = SWEEP_THREADS (512) threads x IPT items, taken
// in launch order from an atomic ticket so every predecessor tile is running or done.
//
//  1. TMA bulk copy (cp.async.bulk + mbarrier) of the tile's keys and ids into smem
//     (pass 0 of the list sort: gathered from the walk's segment slots, gather_tile).
//  2. Stable in-warp ranking (rank_items): a warp ranks 32 consecutive items at a time,
//     in input order, on its private u16 digit counters -- one lane-ordered shared
//     atomic per item (RANK_ATOMIC; lanes sharing lane 0's digit take one atomic on
//     skewed middle passes), or peer masks from ballots / match.any with the group
//     leader bumping the counter (RANK_BALLOT / RANK_MATCH).
//  3. Per-digit warp offsets + tile totals; the aggregate is published at once.
//  4. Stage the tile in smem in (digit, input order) order.
//  5. Decoupled lookback, one thread per digit value.
//  6. Coalesced write-out: consecutive threads store consecutive staged elements, which
//     land contiguously inside each digit run.
//
// Status word per (tile, digit): count[31:0] | flag[33:32] (1 aggregate, 2 inclusive)
// | epoch[63:34]; the status array is zeroed once per call and each pass slot has its
// own epoch, so stale words from earlier passes never match.
template <typename KeyT, int RADIX_BITS, int IPT>
struct SweepSmem {
  static constexpr int RADIX = 1 << RADIX_BITS;
  static constexpr int TILE = SWEEP_THREADS * IPT;
  KeyT k[TILE + 32];       // input keys, later the staged output keys (+ a word per lane
                           // for the staging stores of items past the last tile's end)
  uint32_t iin[TILE];      // input ids
  uint32_t iout[TILE + 32];  // staged output ids (+ the same scratch words)
  WCnt wcnt[SWEEP_WARPS][RADIX];
  uint32_t dstart[RADIX];
  uint32_t goff[RADIX];
  uint32_t gpre[RADIX + 1];  // 128-bit write-out: exclusive scan of each digit run's 16 B groups
  uint32_t scan[SWEEP_WARPS];
  uint32_t scratch[32];    // the ranking's per-lane words for atomics that add nothing
  uint32_t tile;
  int bad;
  unsigned long long mbar;
};

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, unsigned long long* mbar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(gsrc), "r"(bytes), "r"(m) : "memory");
}

// Load-time check of the lane order of conflicting shared-memory atomics (RANK_ATOMIC).
// Every lane adds 1 to a warp-private counter chosen by a hashed digit; the result must
// equal (value before the instruction) + (number of lower lanes with the same digit).
static __global__ void k_selftest_atomic_order(uint32_t iters, uint32_t* bad) {
  __shared__ WCnt cnt[SWEEP_WARPS][256];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < SWEEP_WARPS * 256; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t x = ruler_hash(threadIdx.x * 7919u + blockIdx.x * 977u), nb = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x = ruler_hash(x + i);
    const uint32_t nbins = 2u << (i & 7);  // 2 .. 256 digit values
    const uint32_t d = x & (nbins - 1);
    uint32_t old;
    if constexpr (sizeof(WCnt) == 4) {
      old = atomicAdd(reinterpret_cast<uint32_t*>(&cnt[w][d]), 1u);
    } else {
      const uint32_t sh = (d & 1u) << 4;
      old = (atomicAdd(reinterpret_cast<uint32_t*>(&cnt[w][0]) + (d >> 1), 1u << sh) >> sh) & 0xFFFFu;
    }
    const uint32_t peers = warp_peers<8>(d, 0xffffffffu);
    const int leader = __ffs(peers) - 1;
    const uint32_t base = __shfl_sync(0xffffffffu, old, leader);
    nb += old != base + __popc(peers & lanemask_lt());
    if ((i & 63) == 63) {  // keep the counters from overflowing
      __syncwarp();
      for (int j = lane; j < 256; j += 32) cnt[w][j] = 0;
      __syncwarp();
    }
  }
  if (nb) atomicAdd(bad, nb);
}

struct SplitTable;  // the multi-GPU key-range partition (below)

// What one launch of k_onesweep sorts: one key pass (digit `digit`, input buffer `src`).
struct SweepArgs {
  const void* kin[2];
  const uint32_t* vin[2];
  void* kout[2];
  uint32_t* vout[2];
  const uint32_t* bases;  // [digit][RADIX] bucket bases
  unsigned long long* status;
  uint32_t* tile_ctr;
  const int* err;
  uint32_t n;
  int slot;  // ticket counter + epoch, unique per launch in a call
  int debug_no_lookback;  // timing experiments only (wrong output)
  // host-resolved pass parameters (the host reads the plan after one sync, so no CTA
  // starts with dependent loads of the plan or the error word)
  int digit;      // digit index
  int last;       // the last pass of the sort (write ids only)
  int src;        // input buffer index
  int combine;    // ranking: lanes sharing lane 0's digit take one atomic (skewed digits)
  // first key pass (GATHER): the tile is read from the walk's segment slots, in list order
  const void* slots;
  uint32_t cap;
  const uint2* seg;               // {len, succ} per segment
  const uint32_t* seg_ord;        // k-th segment of the list
  const uint32_t* seg_pos;        // list position of the k-th segment's first node
  const uint32_t* tile_first;     // ordinal of the segment holding each tile's first position
  const uint32_t* nseg;
  const SplitTable* split;        // SRC_SPLIT: the multi-GPU partition (device memory)
};

// In-warp stable ranking modes (RANK template parameter of k_onesweep).
enum : int { RANK_BALLOT = 0, RANK_MATCH = 1, RANK_ATOMIC = 2 };

// Stable rank of each of a warp's IPT x 32 items among the warp's items of the same digit
// (items in input order), accumulated in the warp's private u16 counters wcnt[w][*].
// rd[i] = rank | digit << 16.  FULL: every item is valid (all tiles but the last).
template <typename KeyT, int RADIX_BITS, int IPT, int RANK, bool FULL>
__device__ __forceinline__ void rank_items(const KeyT (&key)[IPT], uint32_t (&rd)[IPT], int shift,
                                           WCnt* __restrict__ wrow, uint32_t wofs, uint32_t lane,
                                           uint32_t tile_count, bool combine, uint32_t scratch) {
  constexpr int RADIX = 1 << RADIX_BITS;
  if (RANK == RANK_ATOMIC && combine) {
    // Skewed digits after the first pass: the input is sorted by the lower digits, so a
    // heavy key fills long input stretches that a few other keys interrupt.  The lanes
    // sharing lane 0's digit (eq) take ONE atomic, issued by lane 0 (the lowest lane, so
    // the lane order of the remaining conflicting atomics is unchanged); the other lanes
    // add 1 each as usual.
#if PBIT_RANK_PRED
    if constexpr (sizeof(WCnt) == 2) {
      // branch-free: a lane with nothing to add (in lane 0's group but not lane 0, or past
      // the tile's end) adds 0 to its own scratch word instead of skipping the atomic, so
      // every lane issues one ATOMS with no divergent branch around it; the lane mask is
      // hoisted and in_eq comes from the compare itself
      const uint32_t lt = lanemask_lt();
      const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(wrow);
      const uint32_t mine = scratch + lane * 4u;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const bool valid = FULL || (wofs + i * 32 + lane < tile_count);
        const uint32_t d = (uint32_t)(key[i] >> shift) & (RADIX - 1);
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
        const bool in_eq = valid && d == d0;
        const uint32_t eq = __ballot_sync(0xffffffffu, in_eq);  // valid lanes: a prefix
        const uint32_t add = lane == 0 ? (uint32_t)__popc(eq) : (valid && !in_eq ? 1u : 0u);
        const uint32_t sh = (d & 1u) << 4;
        const uint32_t addr = add ? wbase + ((d >> 1) << 2) : mine;
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(add << sh) : "memory");
        uint32_t r = (old >> sh) & 0xFFFFu;
        const uint32_t r0 = __shfl_sync(0xffffffffu, r, 0);
        r = in_eq ? r0 + (uint32_t)__popc(eq & lt) : r;
        rd[i] = r | (d << 16);
      }
      return;
    } else
#endif
    {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const bool valid = FULL || (wofs + i * 32 + lane < tile_count);
      const uint32_t d = (uint32_t)(key[i] >> shift) & (RADIX - 1);
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
      const uint32_t eq = __ballot_sync(0xffffffffu, valid && d == d0);  // valid lanes: a prefix
      const bool in_eq = (eq >> lane) & 1u;
      const uint32_t add = lane == 0 ? (uint32_t)__popc(eq) : (valid && !in_eq ? 1u : 0u);
      uint32_t r = 0;
      if constexpr (sizeof(WCnt) == 4) {
        if (add) r = atomicAdd(reinterpret_cast<uint32_t*>(wrow + d), add);
      } else {
        const uint32_t sh = (d & 1u) << 4;
        uint32_t* wc = reinterpret_cast<uint32_t*>(wrow) + (d >> 1);
        if (add) r = (atomicAdd(wc, add << sh) >> sh) & 0xFFFFu;
      }
      const uint32_t r0 = __shfl_sync(0xffffffffu, r, 0);
      r = in_eq ? r0 + (uint32_t)__popc(eq & lanemask_lt()) : r;
      rd[i] = r | (d << 16);
    }
    return;
    }
  }
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const bool valid = FULL || (wofs + i * 32 + lane < tile_count);
    const uint32_t d = (uint32_t)(key[i] >> shift) & (RADIX - 1);
    if constexpr (RANK == RANK_ATOMIC) {
      // One shared atomic per item on the warp's private counters.
      // Conflicting lanes of one ATOMS are served in ascending lane order on sm_100a --
      // measured, not documented: checked at load time by k_selftest_atomic_order
      // (pbit.cu), which falls back to RANK_BALLOT if it ever fails.  A warp whose items
      // share one digit (equal-key runs) lets lane 0 add 32 instead of serialising.
#if PBIT_RANK_MATCHALL
      // one match.all instead of shfl + compare + vote (an invalid lane never matches)
      int all_eq = 0;
      __match_all_sync(0xffffffffu, valid ? d : 0x10000u + lane, &all_eq);
      const bool uni = all_eq != 0;
#else
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
      const bool uni = __all_sync(0xffffffffu, d == d0 && valid);
#endif
      uint32_t r = 0;
#if PBIT_RANK_PRED
      if constexpr (sizeof(WCnt) == 2) {
        // branch-free (see the combining path): lanes 1-31 of an all-equal warp and lanes
        // past the tile's end add 0 to their own scratch word
        const uint32_t sh = (d & 1u) << 4;
        const uint32_t add = uni ? (lane == 0 ? 32u : 0u) : (valid ? 1u : 0u);
        const uint32_t addr = add ? (uint32_t)__cvta_generic_to_shared(wrow) + ((d >> 1) << 2) : scratch + lane * 4u;
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(add << sh) : "memory");
        r = (old >> sh) & 0xFFFFu;
        const uint32_t r0 = __shfl_sync(0xffffffffu, r, 0);
        r = uni ? r0 + lane : r;
        rd[i] = r | (d << 16);
        continue;
      }
#endif
#if PBIT_RANK_UNIBRANCH
      // `uni` is warp-uniform: branch on it, so that a full tile's common case (every lane
      // adds 1) issues its atomic without a per-lane predicate or reconvergence barrier
      if (uni) {
        if (lane == 0) {
          if constexpr (sizeof(WCnt) == 4) {
            r = atomicAdd(reinterpret_cast<uint32_t*>(wrow + d), 32u);
          } else {
            const uint32_t sh = (d & 1u) << 4;
            r = (atomicAdd(reinterpret_cast<uint32_t*>(wrow) + (d >> 1), 32u << sh) >> sh) & 0xFFFFu;
          }
        }
        r = __shfl_sync(0xffffffffu, r, 0) + lane;
      } else if (FULL || valid) {
        if constexpr (sizeof(WCnt) == 4) {
          r = atomicAdd(reinterpret_cast<uint32_t*>(wrow + d), 1u);
        } else {
          const uint32_t sh = (d & 1u) << 4;
          r = (atomicAdd(reinterpret_cast<uint32_t*>(wrow) + (d >> 1), 1u << sh) >> sh) & 0xFFFFu;
        }
      }
#else
      const uint32_t add = uni ? (lane == 0 ? 32u : 0u) : (valid ? 1u : 0u);
      if constexpr (sizeof(WCnt) == 4) {
        if (add) r = atomicAdd(reinterpret_cast<uint32_t*>(wrow + d), add);
      } else {  // two u16 counters per word
        const uint32_t sh = (d & 1u) << 4;
        uint32_t* wc = reinterpret_cast<uint32_t*>(wrow) + (d >> 1);
        if (add) r = (atomicAdd(wc, add << sh) >> sh) & 0xFFFFu;
      }
      const uint32_t r0 = __shfl_sync(0xffffffffu, r, 0);
      r = uni ? r0 + lane : r;
#endif
      rd[i] = r | (d << 16);
    } else {
      const uint32_t vmask = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
      uint32_t peers;
      if constexpr (RANK == RANK_MATCH) peers = __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu) & vmask;
      else peers = warp_peers<RADIX_BITS>(d, vmask);
      const int leader = 31 - __clz(peers | 1u);
      uint32_t before = 0;
      if (valid && lane == (uint32_t)leader) {
        before = wrow[d];
        wrow[d] = (WCnt)(before + __popc(peers));
      }
      before = __shfl_sync(0xffffffffu, before, leader);
      rd[i] = (before + __popc(peers & lanemask_lt())) | (d << 16);
    }
  }
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc) : "memory");
}

#ifndef PBIT_GATHER_UNROLL
#define PBIT_GATHER_UNROLL 1
#endif
constexpr int GATHER_UNROLL = PBIT_GATHER_UNROLL;  // copy loop per segment: ~2 trips of 32 records

// Fill the tile [P, P + count) of the list order straight from the walk's segment slots
// (replaces a separate gather pass over n x 16 B).  Each warp fetches the metadata of 32
// segments at once (one lane each), then copies the overlapping part of each with
// cp.async (no registers, all copies in flight together).
#ifndef PBIT_GATHER_BULK
#define PBIT_GATHER_BULK 1
#endif
template <typename KeyT, int TILE>
__device__ __forceinline__ void gather_tile(const SweepArgs& a, uint32_t tile, uint32_t P, uint32_t count,
                                            KeyT* sk, uint32_t* sv, uint32_t w, uint32_t lane,
                                            unsigned long long* mbar) {
  constexpr bool WIDE = sizeof(KeyT) == 8;
  const uint32_t E = P + count;
  const uint32_t nseg = *a.nseg;
  const uint32_t cap = a.cap;  // kernel parameters in registers: the loops below reload them otherwise
  const unsigned char* __restrict__ slots = reinterpret_cast<const unsigned char*>(a.slots);
  // warp w takes segments first + w + SWEEP_WARPS * i: all warps share the copying
  for (uint32_t kb = a.tile_first[tile] + w;; kb += SWEEP_WARPS * 32) {
    const uint32_t k = kb + lane * SWEEP_WARPS;
    uint32_t pos = E, r = 0, len = 0;
    if (k < nseg) {
      pos = a.seg_pos[k];
      // segments in ordinal order tile the list: the k-th one ends where the next starts,
      // so its length comes from the (sequential, cached) position table instead of a
      // random load of its segment-table entry (one dependent round trip less)
      if (pos < E) {
        r = a.seg_ord[k];
        len = (k + 1 < nseg ? a.seg_pos[k + 1] : a.n) - pos;
      }
    }
    uint32_t todo = __ballot_sync(0xffffffffu, pos < E);
    if (!todo) break;
#if PBIT_GATHER_LANEBULK
    if constexpr (!WIDE && PBIT_GATHER_BULK) {
      // every lane whose segment starts at an even list position copies it itself: one
      // TMA bulk copy of the aligned middle plus <= 2 edge records, no warp-serial step;
      // the warp-cooperative loop below takes only the odd-aligned (and short) segments
      const uint32_t lo = max(P, pos), hi = min(E, pos + len);
      const bool mine = pos < E && (pos & 1u) == 0u && hi >= lo + 4u;
      if (mine) {
        const uint32_t a0 = (lo + 1u) & ~1u, a1 = hi & ~1u;
        PBIT_ASSERT(hi - P <= (uint32_t)TILE && len <= cap);
        const uint2* src = reinterpret_cast<const uint2*>(slots) + (size_t)r * cap;
        uint2* dst = reinterpret_cast<uint2*>(sk);
        const uint32_t bytes = (a1 - a0) * 8u;
        const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
        bulk_g2s(dst + (a0 - P), src + (a0 - pos), bytes, mbar);
        if (lo < a0) cp_async8(dst + (lo - P), src + (lo - pos));
        if (a1 < hi) cp_async8(dst + (a1 - P), src + (a1 - pos));
      }
      todo &= ~__ballot_sync(0xffffffffu, mine);
    }
#endif
    while (todo) {
      const int q = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t sp = __shfl_sync(0xffffffffu, pos, q);
      const uint32_t sr = __shfl_sync(0xffffffffu, r, q);
      const uint32_t sl = __shfl_sync(0xffffffffu, len, q);
      const uint32_t lo = max(P, sp), hi = min(E, sp + sl);
      PBIT_ASSERT(hi <= lo || (hi - P <= (uint32_t)TILE && sl <= cap));
      if constexpr (!WIDE && PBIT_GATHER_BULK) {
        // a segment starting at an even list position has its records at the same 16 B
        // alignment in the slot and in the tile (slots and tiles start 16 B-aligned): one
        // TMA bulk copy for its even-aligned middle, cp.async for the <= 2 edge records
        if ((sp & 1u) == 0u && hi - lo >= 4u) {
          const uint32_t a0 = (lo + 1u) & ~1u, a1 = hi & ~1u;
          const uint2* src = reinterpret_cast<const uint2*>(slots) + (size_t)sr * cap;
          uint2* dst = reinterpret_cast<uint2*>(sk);
          if (lane == 0) {
            const uint32_t bytes = (a1 - a0) * 8u;
            const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
            bulk_g2s(dst + (a0 - P), src + (a0 - sp), bytes, mbar);
          }
          if (lane == 1 && lo < a0) cp_async8(dst + (lo - P), src + (lo - sp));
          if (lane == 2 && a1 < hi) cp_async8(dst + (a1 - P), src + (a1 - sp));
          continue;
        }
      }
#pragma unroll (GATHER_UNROLL)
      for (uint32_t x = lo + lane; x < hi; x += 32) {
        if constexpr (WIDE) {
          const uint4* rec = reinterpret_cast<const uint4*>(slots) + (size_t)sr * cap + (x - sp);
          cp_async8(sk + (x - P), &rec->x);
          cp_async4(sv + (x - P), &rec->z);
        } else {  // one 8 B copy of the whole record into the AoS tile (k_onesweep AOS)
          const uint2* rec = reinterpret_cast<const uint2*>(slots) + (size_t)sr * cap + (x - sp);
          cp_async8(reinterpret_cast<uint2*>(sk) + (x - P), rec);
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if constexpr (!WIDE && PBIT_GATHER_BULK) {
    __syncthreads();  // every expect_tx is registered before the barrier's one arrival
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(m) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(m) : "memory");
  }
}

// Where the first pass's tile comes from (k_onesweep SRC): TMA of keys and ids; the
// walk's segment slots (list sort, pass 0); TMA of keys with ids = positions (array sort).
// SRC_SPLIT (multi-GPU): TMA of keys and ids, the digit is the key's bucket among the
// splitters, and the write-out sends each element to its destination rank (SplitTable).
enum : int { SRC_TMA = 0, SRC_GATHER = 1, SRC_IOTA = 2, SRC_SPLIT = 3 };

// The key-range partition of the multi-GPU sort (pbit_sort_list_mg, SRC_SPLIT), written
// on the device by k_split_plan.  Bucket of key k: j = #{s : kstar[s] < k}, then
// 2j + (j < NS && kstar[j] == k): buckets in key order, the keys equal to a splitter key in
// their own bucket.  The pass sorts a rank's list-order chunk stably by bucket; element g
// of that order goes to rank d = #{s in 1..G-1 : left[s] <= g}, at index g + dst_off[d] of
// that rank's receive arrays (dst_k[d], dst_i[d]: a peer's window -- N4 -- or, with the
// NCCL transport, this rank's send buffer with dst_off = 0).
struct SplitTable {
  uint32_t G, NS;
  unsigned long long kstar[64];
  uint32_t left[65];
  uint32_t dst_off[64];
  void* dst_k[64];
  uint32_t* dst_i[64];
};

__device__ __forceinline__ uint32_t split_bucket(const SplitTable& sp, unsigned long long k) {
  uint32_t lo = 0, hi = sp.NS;  // lower_bound: first s with kstar[s] >= k
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sp.kstar[mid] < k) lo = mid + 1; else hi = mid;
  }
  return 2u * lo + ((lo < sp.NS && sp.kstar[lo] == k) ? 1u : 0u);
}

__device__ __forceinline__ uint32_t split_dest(const SplitTable& sp, uint32_t g) {
  uint32_t lo = 1, hi = sp.G;  // ranks d >= 1 whose first element left[d] <= g
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sp.left[mid] <= g) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

template <typename KeyT, int RADIX_BITS, int IPT, int RANK, int SRC = SRC_TMA>
__global__ void __launch_bounds__(SWEEP_THREADS, 1024 / SWEEP_THREADS)
k_onesweep(const __grid_constant__ SweepArgs a) {
  pdl_enter();
  using S = SweepSmem<KeyT, RADIX_BITS, IPT>;
  constexpr int RADIX = S::RADIX;
  constexpr int TILE = S::TILE;
  constexpr int WARP_ITEMS = 32 * IPT;
  static_assert(RADIX <= SWEEP_THREADS, "one thread per digit value");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const uint32_t n = a.n;
  const int slot = a.slot;
  const int src = a.src;
  const int shift = a.digit * RADIX_BITS;
  const bool last = a.last != 0;
  const uint32_t* __restrict__ bases = a.bases + a.digit * RADIX;
  const KeyT* __restrict__ kin = reinterpret_cast<const KeyT*>(a.kin[src]);
  const uint32_t* __restrict__ iin = a.vin[src];
  const int dst = src ^ 1;
  KeyT* __restrict__ kout = reinterpret_cast<KeyT*>(a.kout[dst]);
  uint32_t* __restrict__ iout = a.vout[dst];
  const unsigned long long epoch = (unsigned long long)(slot + 1);
  unsigned long long* status = a.status;
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;

  SplitTable& sp = *reinterpret_cast<SplitTable*>(smem_raw + sizeof(S));  // SRC_SPLIT only
  if constexpr (SRC == SRC_SPLIT) {
    for (uint32_t i = threadIdx.x; i < sizeof(SplitTable) / 4; i += SWEEP_THREADS)
      reinterpret_cast<uint32_t*>(&sp)[i] = reinterpret_cast<const uint32_t*>(a.split)[i];
  }
  if (t == 0) {
    sm.bad = *a.err;  // an invalid list (found after the pass was queued): no pass runs
    sm.tile = atomicAdd(a.tile_ctr + slot, 1u);
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(m));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (sm.bad) return;  // uniform: every CTA read the same word (set before the pass)
  const uint32_t tile = sm.tile;
  const uint32_t tile_base = tile * (uint32_t)TILE;
  const uint32_t tile_count = min((uint32_t)TILE, n - tile_base);
  const bool full_tile = tile_count == (uint32_t)TILE;

  // ---- TMA bulk loads of the tile (sizes rounded up to 16 B; buffers padded to 256 B);
  // the first key pass gathers the tile from the segment slots instead
  constexpr bool GATHER = SRC == SRC_GATHER;
#if PBIT_GATHER_META_PREFETCH
  // first pass: warm L2 with the segment table entries (list positions and slots, both in
  // list-ordinal order) of the tile PBIT_SWEEP_PREFETCH tickets ahead
  if (GATHER && t == 0) {
    const uint32_t pt = tile + (uint32_t)PBIT_SWEEP_PREFETCH;
    if ((size_t)(pt + 1) * TILE < n) {
      const uint32_t k0 = a.tile_first[pt] & ~3u, k1 = (a.tile_first[pt + 1] + 4u) & ~3u;
      const uint32_t bytes = min(k1 - k0, 4096u) * 4u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.seg_pos + k0), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.seg_ord + k0), "r"(bytes) : "memory");
    }
  }
#endif
  if (GATHER) gather_tile<KeyT, TILE>(a, tile, tile_base, tile_count, sm.k, sm.iin, w, lane, &sm.mbar);
  if (!GATHER && t == 0) {
    const uint32_t kb = (tile_count * (uint32_t)sizeof(KeyT) + 15u) & ~15u;
    const uint32_t ib = SRC == SRC_IOTA ? 0u : (tile_count * 4u + 15u) & ~15u;
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(m), "r"(kb + ib) : "memory");
    bulk_g2s(sm.k, kin + tile_base, kb, &sm.mbar);
    if (SRC != SRC_IOTA) bulk_g2s(sm.iin, iin + tile_base, ib, &sm.mbar);
#if PBIT_SWEEP_PREFETCH
    // warm L2 with the tile a CTA launched about one resident wave later will take (tickets
    // are handed out in launch order), so its TMA load hits L2 instead of waiting on HBM
    const uint32_t pt = tile + (uint32_t)PBIT_SWEEP_PREFETCH;
    if ((size_t)pt * TILE < n) {
      const uint32_t pc = min((uint32_t)TILE, n - pt * (uint32_t)TILE);
      const uint32_t pkb = (pc * (uint32_t)sizeof(KeyT) + 15u) & ~15u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kin + (size_t)pt * TILE), "r"(pkb) : "memory");
      if (SRC != SRC_IOTA) {
        const uint32_t pib = (pc * 4u + 15u) & ~15u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(iin + (size_t)pt * TILE), "r"(pib) : "memory");
      }
    }
#endif
  }
  if (SRC == SRC_IOTA)
    for (uint32_t j = t; j < tile_count; j += SWEEP_THREADS) sm.iin[j] = tile_base + j;
  for (uint32_t i = t; i < SWEEP_WARPS * RADIX * sizeof(WCnt) / 4; i += SWEEP_THREADS)
    reinterpret_cast<uint32_t*>(&sm.wcnt[0][0])[i] = 0;
  if (!GATHER) {
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(m) : "memory");
    }
  }
  __syncthreads();

  // ---- stable in-warp ranking.  AOS (pass 0 with keys <= 32 bits): the gather copied
  // whole (key, id) records into the k and iin buffers viewed as one uint2 array
  constexpr bool AOS = GATHER && sizeof(KeyT) == 4;
  const uint2* __restrict__ srec = reinterpret_cast<const uint2*>(sm.k);
  const uint32_t wofs = w * WARP_ITEMS;
  KeyT key[IPT];
  uint32_t rd[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) key[i] = AOS ? (KeyT)srec[wofs + i * 32 + lane].x : sm.k[wofs + i * 32 + lane];
  const bool combine = a.combine != 0;
  if constexpr (SRC == SRC_SPLIT) {  // digit = the key's splitter bucket
    uint32_t dg[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) dg[i] = split_bucket(sp, (unsigned long long)key[i]);
    if (full_tile) rank_items<uint32_t, RADIX_BITS, IPT, RANK, true>(dg, rd, 0, sm.wcnt[w], wofs, lane, tile_count, combine,
                                                         (uint32_t)__cvta_generic_to_shared(sm.scratch));
    else rank_items<uint32_t, RADIX_BITS, IPT, RANK, false>(dg, rd, 0, sm.wcnt[w], wofs, lane, tile_count, combine,
                                                         (uint32_t)__cvta_generic_to_shared(sm.scratch));
  } else {
    if (full_tile) rank_items<KeyT, RADIX_BITS, IPT, RANK, true>(key, rd, shift, sm.wcnt[w], wofs, lane, tile_count, combine,
                                                     (uint32_t)__cvta_generic_to_shared(sm.scratch));
    else rank_items<KeyT, RADIX_BITS, IPT, RANK, false>(key, rd, shift, sm.wcnt[w], wofs, lane, tile_count, combine,
                                                     (uint32_t)__cvta_generic_to_shared(sm.scratch));
  }
  __syncthreads();

  // ---- per digit (thread t = digit t): exclusive over warps, tile total, aggregate
  uint32_t total = 0;
#if PBIT_SCAN_REG
  // the warps' exclusive prefixes stay in registers (two u16 per word) until the tile's
  // digit start is known: one read and one write of each warp counter instead of two each
  constexpr int NPW = (SWEEP_WARPS + 1) / 2;
  uint32_t wpre[NPW];
#pragma unroll
  for (int q = 0; q < NPW; ++q) wpre[q] = 0;
  if (t < RADIX) {
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) {
      const uint32_t c = sm.wcnt[ww][t];
      wpre[ww >> 1] |= total << ((ww & 1) * 16);
      total += c;
    }
    if (tile > 0) st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (1ull << 32) | total);
  }
#else
  if (t < RADIX) {
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) {
      const uint32_t c = sm.wcnt[ww][t];
      sm.wcnt[ww][t] = (WCnt)total;
      total += c;
    }
    if (tile > 0) st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (1ull << 32) | total);
  }
#endif
  {
    uint32_t x = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) sm.scan[w] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) add += (ww < (int)w) ? sm.scan[ww] : 0u;
    if (t < RADIX) {
      const uint32_t ds = x - total + add;
      sm.dstart[t] = ds;
#if PBIT_SCAN_REG
#pragma unroll
      for (int ww = 0; ww < SWEEP_WARPS; ++ww) sm.wcnt[ww][t] = (WCnt)(((wpre[ww >> 1] >> ((ww & 1) * 16)) & 0xFFFFu) + ds);
#else
#pragma unroll
      for (int ww = 0; ww < SWEEP_WARPS; ++ww) sm.wcnt[ww][t] = (WCnt)(sm.wcnt[ww][t] + ds);
#endif
    }
  }
  __syncthreads();

  // ---- stage in (digit, input order) order: keys from registers into sm.k (every warp
  // read its keys before the barriers above), values from sm.iin into sm.iout
  // (non-AOS passes: an item past the last tile's end is staged into its lane's scratch
  // slot, index TILE + lane, instead of being skipped -- no branch per item; the AOS first
  // pass keeps the branch, measured faster there)
  if constexpr (AOS) {
    // ids first (they live in the records the keys will overwrite), then the keys
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t j = wofs + i * 32 + lane;
      if (full_tile || j < tile_count) {
        const uint32_t d = rd[i] >> 16;
        const uint32_t lp = sm.wcnt[w][d] + (rd[i] & 0xFFFFu);
        sm.iout[lp] = srec[j].y;
        rd[i] = lp | (d << 16);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t j = wofs + i * 32 + lane;
      if (full_tile || j < tile_count) sm.k[rd[i] & 0xFFFFu] = last ? (KeyT)(rd[i] >> 16) : key[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t j = wofs + i * 32 + lane;
      const uint32_t d = rd[i] >> 16;
      const uint32_t lp = (full_tile || j < tile_count) ? sm.wcnt[w][d] + (rd[i] & 0xFFFFu) : (uint32_t)TILE + lane;
      sm.iout[lp] = sm.iin[j];
      sm.k[lp] = last ? (KeyT)d : key[i];  // the last key pass needs only digits
    }
  }
  // ---- decoupled lookback, one thread per digit value, LB_WIN predecessors per step
  uint32_t ngrp = 0;  // 16 B-aligned groups of 4 output slots the digit's run touches
  if (t < RADIX) {
    constexpr int LB_WIN = 4;
    unsigned long long excl = 0;
    if (tile == 0 || a.debug_no_lookback) {
      st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (2ull << 32) | total);
    } else {
      int64_t hi = (int64_t)tile - 1;  // nearest predecessor not yet accounted for
      for (;;) {
        unsigned long long wv[LB_WIN];
#pragma unroll
        for (int q = 0; q < LB_WIN; ++q)
          wv[q] = hi - q >= 0 ? ld_relaxed_u64(status + (size_t)(hi - q) * RADIX + t) : 0ull;
        bool done = false;
        int q = 0;
#pragma unroll
        for (; q < LB_WIN; ++q) {
          if (hi - q < 0 || (wv[q] >> 34) != epoch) break;  // not published: resume here
          excl += (uint32_t)wv[q];
          if (((wv[q] >> 32) & 3ull) == 2ull) { done = true; break; }
        }
        if (done) break;
        hi -= q;
#if PBIT_LB_SLEEP
        // nothing new from the nearest predecessor yet: back off instead of re-polling at
        // once, leaving the issue slots to the other CTA's warps on this SM
        if (q == 0) __nanosleep(PBIT_LB_SLEEP);
#endif
      }
      st_relaxed_u64(status + (size_t)tile * RADIX + t, (epoch << 34) | (2ull << 32) | (excl + total));
    }
    sm.goff[t] = bases[t] + (uint32_t)excl - sm.dstart[t];
    const uint32_t gs = bases[t] + (uint32_t)excl;  // the run's first global slot
    ngrp = total ? ((gs + total + 3u) >> 2) - (gs >> 2) : 0u;
  }
  __syncthreads();
  constexpr bool VEC = PBIT_VEC_STORE && SRC != SRC_SPLIT;
  if constexpr (VEC) {  // exclusive scan of the group counts over the digits
    uint32_t x = ngrp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) sm.scan[w] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int ww = 0; ww < SWEEP_WARPS; ++ww) add += (ww < (int)w) ? sm.scan[ww] : 0u;
    if (t < RADIX) sm.gpre[t] = x - ngrp + add;
    if (t == RADIX - 1) sm.gpre[RADIX] = x + add;
    __syncthreads();
  }

  // ---- coalesced write-out: consecutive threads store consecutive staged elements,
  // which land contiguously inside each digit run
  if constexpr (SRC == SRC_SPLIT) {
    // element g of the bucket order goes to its destination rank's receive arrays
    for (uint32_t j = t; j < tile_count; j += SWEEP_THREADS) {
      const KeyT k = sm.k[j];
      const uint32_t g = sm.goff[split_bucket(sp, (unsigned long long)k)] + j;
      const uint32_t d = split_dest(sp, g);
      const uint32_t at = g + sp.dst_off[d];
      PBIT_ASSERT(g < n && d < sp.G);
      reinterpret_cast<KeyT*>(sp.dst_k[d])[at] = k;
      sp.dst_i[d][at] = sm.iout[j];
    }
    // the stores may go to other GPUs' memory (peer transport): make them visible at
    // system scope before this kernel completes and the ranks' barrier collective runs
    __threadfence_system();
  } else if (VEC && ((((uintptr_t)iout | (last ? 0 : (uintptr_t)kout)) & 15u) == 0)) {
    // 128-bit stores: every digit run is cut at 16 B boundaries of the OUTPUT arrays into
    // groups of 4 slots; thread q takes group q (its digit by binary search over the group
    // prefix); a whole group leaves as one 16 B store of ids (and one or two of keys), the
    // <= 2 partial groups at the ends of a run as scalar stores
    const uint32_t ngroups = sm.gpre[RADIX];
    for (uint32_t q = t; q < ngroups; q += SWEEP_THREADS) {
      uint32_t lo = 0, hi = RADIX;  // the last digit d with gpre[d] <= q
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm.gpre[mid] <= q) lo = mid; else hi = mid;
      }
      const uint32_t d = lo;
      const uint32_t go = sm.goff[d];
      const uint32_t j_lo = sm.dstart[d];
      const uint32_t j_hi = d + 1 < (uint32_t)RADIX ? sm.dstart[d + 1] : tile_count;
      const uint32_t A = (((go + j_lo) >> 2) + (q - sm.gpre[d])) << 2;  // first slot of the group
      const int j0 = (int)(A - go);  // its staged index (negative before the run's first slot)
      if (j0 >= (int)j_lo && j0 + 4 <= (int)j_hi) {
        *reinterpret_cast<uint4*>(iout + A) = make_uint4(sm.iout[j0], sm.iout[j0 + 1], sm.iout[j0 + 2], sm.iout[j0 + 3]);
        if (!last) {
          if constexpr (sizeof(KeyT) == 8) {
            *reinterpret_cast<ulonglong2*>(kout + A) = make_ulonglong2(sm.k[j0], sm.k[j0 + 1]);
            *reinterpret_cast<ulonglong2*>(kout + A + 2) = make_ulonglong2(sm.k[j0 + 2], sm.k[j0 + 3]);
          } else {
            *reinterpret_cast<uint4*>(kout + A) = make_uint4(sm.k[j0], sm.k[j0 + 1], sm.k[j0 + 2], sm.k[j0 + 3]);
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = j0 + e;
          if (j >= (int)j_lo && j < (int)j_hi) {
            iout[A + e] = sm.iout[j];
            if (!last) kout[A + e] = sm.k[j];
          }
        }
      }
    }
  } else if (!last) {
#pragma unroll 4
    for (uint32_t j = t; j < tile_count; j += SWEEP_THREADS) {
      const KeyT k = sm.k[j];
      const uint32_t g = sm.goff[(uint32_t)(k >> shift) & (RADIX - 1)] + j;
      PBIT_ASSERT(g < n);
      kout[g] = k;
      iout[g] = sm.iout[j];
    }
  } else {
#pragma unroll 4
    for (uint32_t j = t; j < tile_count; j += SWEEP_THREADS) {
      const uint32_t g = sm.goff[(uint32_t)sm.k[j]] + j;
      PBIT_ASSERT(g < n);
      iout[g] = sm.iout[j];
    }
  }
}

// ============================================================================ N3: array sort
// pbit_sort_array -- the "table" of the paper's tables-vs-lists comparison:
// the same stable passes over an array, with no ranking and no relink.
// k_array_prep: user keys (any width) -> sort keys (KeyMap applied, widened to the pass
// key type) + histograms of every digit (per-CTA smem).
template <int KB>
__global__ void __launch_bounds__(PACK_THREADS)
k_array_prep(const void* __restrict__ keys, uint32_t n, typename KeyOf<KB>::T* __restrict__ kout,
             uint32_t* __restrict__ hist, int K, int D, KeyMap km) {
  using KT = std::conditional_t<KB == 1, uint8_t, std::conditional_t<KB == 2, uint16_t,
             std::conditional_t<KB == 4, uint32_t, unsigned long long>>>;
  extern __shared__ uint32_t s_hist[];
  const int radix = 1 << K;
  const int nb = D * radix;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const uint32_t mask = radix - 1;
  const KT* __restrict__ kp = reinterpret_cast<const KT*>(keys);
  const uint32_t lane = threadIdx.x & 31u;
  for (unsigned long long v0 = blockIdx.x * blockDim.x + threadIdx.x - lane; v0 < n;
       v0 += (unsigned long long)gridDim.x * blockDim.x) {  // warp-uniform trips (hist_add)
    const unsigned long long v = v0 + lane;
    const bool ok = v < n;
    unsigned long long k = ok ? (unsigned long long)__ldcs(kp + v) : 0ull;
    if (!km.identity()) k = km(k, KB * 8);
    if (ok) kout[v] = (typename KeyOf<KB>::T)k;
    for (int d = 0; d < D; ++d) hist_add(s_hist + d * radix, (uint32_t)(k >> (d * K)) & mask, ok);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// out_keys[i] = the original bits of the i-th sorted key (inverse KeyMap, narrowed);
// iota: out_index[i] = i (no pass ran: the input order is the sorted order).
template <int KB>
__global__ void __launch_bounds__(256)
k_array_finish(const typename KeyOf<KB>::T* __restrict__ ksorted, uint32_t n, void* __restrict__ out_keys,
               uint32_t* __restrict__ out_index, KeyMap km) {
  using KT = std::conditional_t<KB == 1, uint8_t, std::conditional_t<KB == 2, uint16_t,
             std::conditional_t<KB == 4, uint32_t, unsigned long long>>>;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (out_keys) {
      unsigned long long k = ksorted[v];
      if (!km.identity()) k = km.inverse(k, KB * 8);
      reinterpret_cast<KT*>(out_keys)[v] = (KT)k;
    }
    if (out_index) out_index[v] = v;
  }
}

// ============================================================================ N3: records
// Materialise the sorted order (pbit_opts.out_order / out_keys): the final ids, and the
// final sort keys mapped back to the input bit patterns.  Skipped for an invalid list.
template <int KB>
__global__ void __launch_bounds__(256)
k_materialize(const uint32_t* __restrict__ ids, const typename KeyOf<KB>::T* __restrict__ ksorted, uint32_t n,
              uint32_t* __restrict__ out_order, void* __restrict__ out_keys, KeyMap km, const int* __restrict__ err) {
  using KT = std::conditional_t<KB == 1, uint8_t, std::conditional_t<KB == 2, uint16_t,
             std::conditional_t<KB == 4, uint32_t, unsigned long long>>>;
  pdl_enter();
  if (*err) return;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (out_order) out_order[v] = ids[v];
    if (out_keys) {
      unsigned long long k = ksorted[v];
      if (!km.identity()) k = km.inverse(k, KB * 8);
      reinterpret_cast<KT*>(out_keys)[v] = (KT)k;
    }
  }
}

// ============================================================================ a5: relink
// out_next[ids[p]] = ids[p+1], out_next[ids[n-1]] = NULL, head = ids[0]: the paper's
// end-splice merge of sorted fragments, one write per node; with out_prev (N2,
// the doubly-linked repair of P:1179-1181) also out_prev[ids[p]] = ids[p-1] in the SAME
// pass chain: records carry (v, succ, pred) instead of (v, succ).
//
// On B200 a random 4 B store costs a 32 B HBM read + write even when the stores are
// confined to a 64 KB window (measured: tools/micro/winstore.cu), and distributed shared
// memory windows are 2-4x slower than one CTA's (tools/micro/dsmem.cu), so no kernel here
// issues scattered stores to HBM.  The records are grouped by fine bin
// v >> RELINK_FINE_SHIFT with MSD partition levels of <= 8 bits (k_relink_part), then each
// fine bin is applied in a 64 KB shared-memory window per output and written out coalesced.
//
// The ids are a permutation of [0, n), so every bin's size is known in closed form (bin
// b of a level with shift s holds exactly the ids [b << s, (b+1) << s)): no histogram,
// no scan.  Order inside a bin does not matter (each v occurs once), so a tile claims its
// space in a bin with one global atomicAdd per (tile, bin) -- no lookback.
constexpr int RELINK_FINE_SHIFT = 14;  // 16384 ids = 64 KB smem window
constexpr int PART_THREADS = 512;

struct u32x3 { uint32_t x, y, z; };  // (v, succ, pred): 12 B relink record
template <int W> struct RelinkRec { using T = uint2; };   // (v, succ)
template <> struct RelinkRec<3> { using T = u32x3; };

// W words per record: 4096-record tiles of pairs (2 CTAs/SM), 2048 of triples (the
// tiles divide every parent bin, >= 2^22 ids)
template <int W> struct PartCfg {
  static constexpr int IPT = W == 2 ? 8 : 4;
  static constexpr int TILE = PART_THREADS * IPT;
};
constexpr int PART_TILE = PartCfg<2>::TILE;

// The MSD levels for n ids: level l partitions by v's bits [shift_l, shift_l + bits_l);
// level 0 takes the top bits, the last level has shift RELINK_FINE_SHIFT.
struct RelinkLevels {
  int L = 0;
  int shift[4] = {0, 0, 0, 0};
  int bits[4] = {0, 0, 0, 0};
  __host__ explicit RelinkLevels(uint32_t n) {
    int top = 0;
    while (top < 32 && (1ull << top) < (unsigned long long)n) ++top;
    const int total = top - RELINK_FINE_SHIFT;
    if (total <= 0) return;
    L = (total + 7) / 8;
    int sh = RELINK_FINE_SHIFT + 8 * (L - 1);
    for (int l = 0; l < L; ++l) {
      bits[l] = l == 0 ? total - 8 * (L - 1) : 8;
      shift[l] = sh;
      sh -= 8;
    }
  }
  // cursor words of level l: one per bin of that level over all ids
  __host__ static size_t cursors(uint32_t n, int shift) { return ((size_t)n >> shift) + 1; }
};

// One partition level.  FROM_IDS (level 0 of the single-GPU sort): the input is the
// sorted id array and the record of position p is (ids[p], ids[p+1][, ids[p-1]]) (NULL
// past either end).  Otherwise the input is records; v_off is subtracted from v on load
// (the multi-GPU path receives global ids).  A tile lies inside one bin of the previous
// level (tiles divide the bins), so its local bin index is (v >> shift) & (2^bits - 1) and
// its global bin index is (tile's parent bin) << bits | local.
//
// Persistent CTAs walk the tiles round-robin; the next tile's TMA bulk load is issued
// before the current tile is ranked, so HBM reads stay in flight while the CTA ranks,
// claims and stores.
template <int W>
struct PartSmem {
  using R = typename RelinkRec<W>::T;
  static constexpr int TILE = PartCfg<W>::TILE;
  R in[2][TILE];  // double-buffered tile loads (FROM_IDS: u32 ids + 4 look-behind + 4 look-ahead)
  R stage[TILE];  // the tile in bin order
  uint32_t cnt[256], start[256], gofs[256], warp[PART_THREADS / 32];
#if PBIT_PART_PIPE
  uint32_t cnt2[2][256], start2[2][256];  // per-slot counts / starts of the pipelined loop
#endif
  unsigned long long mbar[2];
};

template <bool FROM_IDS, int W>
__global__ void __launch_bounds__(PART_THREADS, 2)
k_relink_part(const uint32_t* __restrict__ ids, const typename RelinkRec<W>::T* __restrict__ pin,
              typename RelinkRec<W>::T* __restrict__ pout, uint32_t n, uint32_t v_off, int shift, int bits,
              uint32_t* __restrict__ cursor, const int* __restrict__ err, uint32_t lo = 0) {
  // records [lo, n) of the input (lo: a whole bin of the previous level; 0 for FROM_IDS)
  using R = typename RelinkRec<W>::T;
  constexpr int TILE = PartCfg<W>::TILE;
  constexpr int IPT = PartCfg<W>::IPT;
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PartSmem<W>& sm = *reinterpret_cast<PartSmem<W>*>(smem_raw);
  if (*err) return;
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t nb = 1u << bits, mask = nb - 1;
  const uint32_t ntiles = (n - lo + TILE - 1) / TILE;
  auto issue = [&](uint32_t tile, int buf) {  // thread 0: TMA bulk load of one tile
    const uint32_t base = lo + tile * (uint32_t)TILE;
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar[buf]);
    uint32_t bytes;
    const void* src;
    if constexpr (FROM_IDS) {  // the tile's ids plus 4 look-ahead (and 4 look-behind for W = 3)
      const uint32_t lo = (W == 3 && base >= 4u) ? base - 4u : base;
      const uint32_t c = min(base + (uint32_t)TILE + 4u, n) - lo;
      bytes = ((c + 3u) & ~3u) * 4u;
      src = ids + lo;
    } else {
      const uint32_t c = min((uint32_t)TILE, n - base);
      bytes = ((c * (uint32_t)sizeof(R)) + 15u) & ~15u;  // buffers are padded by 16 B
      src = pin + base;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
    bulk_g2s(&sm.in[buf][0], src, bytes, &sm.mbar[buf]);
  };
  if (t == 0) {
    for (int b = 0; b < 2; ++b) {
      const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar[b]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(m));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
#if PBIT_PART_PIPE
    if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
#endif
  }
  __syncthreads();
#if PBIT_PART_PIPE
  // Software-pipelined: the global bin claims of the CTA's next tile are issued before the
  // current tile is written out and consumed one tile later, so their L2 round trip is off
  // the tile's critical path.  Every bin's records stay one dense run per tile (the record
  // order inside a bin is free: the apply scatters by v).
  {
    R x[IPT];
    uint32_t r[IPT];
    auto wait_tile = [&](uint32_t q) {
      const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar[q & 1u]);
      const uint32_t par = (q >> 1) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(m), "r"(par) : "memory");
    };
    // items of the CTA's q-th tile into registers, ranked on the slot's bin counters
    auto load_rank = [&](uint32_t q, uint32_t tile) {
      const uint32_t base = lo + tile * (uint32_t)TILE;
      const uint32_t cnt = min((uint32_t)TILE, n - base);
      const uint32_t* in_ids = reinterpret_cast<const uint32_t*>(&sm.in[q & 1u][0]);
      const uint32_t off = (FROM_IDS && W == 3 && base >= 4u) ? 4u : 0u;
      uint32_t* c = sm.cnt2[q & 1u];
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t j = i * PART_THREADS + t;
        if (j < cnt) {
          if constexpr (FROM_IDS) {
            x[i].x = in_ids[off + j];
            x[i].y = base + j + 1 < n ? in_ids[off + j + 1] : PBIT_NULL32;
            if constexpr (W == 3) x[i].z = base + j > 0 ? in_ids[off + j - 1] : PBIT_NULL32;
          } else {
            x[i] = sm.in[q & 1u][j];
            x[i].x -= v_off;
          }
          r[i] = atomicAdd(&c[(x[i].x >> shift) & mask], 1u);
        }
      }
    };
    // exclusive scan of a tile's bin counts (start2[slot]) and its claims (returned, t < nb)
    auto scan_claim = [&](uint32_t q, uint32_t tile, uint32_t& claim, uint32_t& my_start) {
      const uint32_t base = lo + tile * (uint32_t)TILE;
      const uint32_t parent = FROM_IDS ? 0u : base >> (shift + bits);
      const uint32_t c = t < nb ? sm.cnt2[q & 1u][t] : 0u;
      uint32_t y = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= (uint32_t)o) y += z;
      }
      if (lane == 31) sm.warp[w] = y;
      __syncthreads();
      uint32_t add = 0;
      for (uint32_t qq = 0; qq < w; ++qq) add += sm.warp[qq];
      claim = 0;
      my_start = 0;
      if (t < nb) {
        my_start = y - c + add;
        sm.start2[q & 1u][t] = my_start;
        if (c) claim = atomicAdd(cursor + ((parent << bits) | t), c);
      }
    };
    uint32_t tile = blockIdx.x;
    if (tile < ntiles) {
      if (t < 256) { sm.cnt2[0][t] = 0; sm.cnt2[1][t] = 0; }
      wait_tile(0);
      __syncthreads();
      load_rank(0, tile);
      __syncthreads();
      if (t == 0 && tile + 2u * gridDim.x < ntiles) issue(tile + 2u * gridDim.x, 0);  // buffer 0 is consumed
      uint32_t claim_cur, start_cur;
      scan_claim(0, tile, claim_cur, start_cur);
      __syncthreads();
      for (uint32_t q = 0;; ++q) {
        const uint32_t s = q & 1u;
        const uint32_t base = lo + tile * (uint32_t)TILE;
        const uint32_t cnt = min((uint32_t)TILE, n - base);
        const uint32_t parent = FROM_IDS ? 0u : base >> (shift + bits);
        // stage tile q in bin order
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t j = i * PART_THREADS + t;
          if (j < cnt) sm.stage[sm.start2[s][(x[i].x >> shift) & mask] + r[i]] = x[i];
        }
        if (t < 256) sm.cnt2[s][t] = 0;  // tile q's counts were read by its scan (barriers since)
        if (t < nb) sm.gofs[t] = (((parent << bits) | t) << shift) + claim_cur - start_cur;
        const uint32_t next = tile + gridDim.x;
        const bool has_next = next < ntiles;  // CTA-uniform
        __syncthreads();  // stage and gofs of tile q visible; slot s counters zeroed
        uint32_t claim_nx = 0, start_nx = 0;
        auto prep_next = [&](int part) {  // part 1: load + rank + refill, part 2: scan + claims
          if (!has_next) return;
          if (part & 1) {
            wait_tile(q + 1);
            load_rank(q + 1, next);
            __syncthreads();
#if PBIT_PP_DBG & 1
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
#endif
            if (t == 0 && next + 2u * gridDim.x < ntiles) issue(next + 2u * gridDim.x, (q + 1) & 1u);
          }
          if (part & 2) scan_claim(q + 1, next, claim_nx, start_nx);  // consumed one tile later
        };
#if PBIT_PP_DBG & 4
        (void)0;
#elif PBIT_PP_DBG & 2
        prep_next(1);
#else
        prep_next(3);
#endif
        // coalesced write-out of tile q
#pragma unroll 4
        for (uint32_t j = t; j < cnt; j += PART_THREADS) {
          const R p = sm.stage[j];
          const uint32_t b = (p.x >> shift) & mask;
          PBIT_ASSERT(sm.gofs[b] + j < n);
          if constexpr (W == 2) __stcs(pout + (sm.gofs[b] + j), p);
          else pout[sm.gofs[b] + j] = p;
        }
#if PBIT_PP_DBG & 4
        __syncthreads();
        prep_next(3);
#elif PBIT_PP_DBG & 2
        __syncthreads();
        prep_next(2);
#endif
        __syncthreads();  // stage and gofs are rewritten for tile q + 1
        if (!has_next) break;
        claim_cur = claim_nx;
        start_cur = start_nx;
        tile = next;
      }
    }
    return;
  }
#endif
  uint32_t it = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    if (t == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, buf ^ 1);
    if (t < 256) sm.cnt[t] = 0;
    {
      const uint32_t m = (uint32_t)__cvta_generic_to_shared(&sm.mbar[buf]);
      const uint32_t par = (it >> 1) & 1u;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(m), "r"(par) : "memory");
    }
    __syncthreads();
    const uint32_t base = lo + tile * (uint32_t)TILE;
    const uint32_t cnt = min((uint32_t)TILE, n - base);
    R x[IPT];
    uint32_t r[IPT];
    const uint32_t* in_ids = reinterpret_cast<const uint32_t*>(&sm.in[buf][0]);
    const uint32_t off = (FROM_IDS && W == 3 && base >= 4u) ? 4u : 0u;  // look-behind shift
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t j = i * PART_THREADS + t;
      if (j < cnt) {
        if constexpr (FROM_IDS) {
          x[i].x = in_ids[off + j];
          x[i].y = base + j + 1 < n ? in_ids[off + j + 1] : PBIT_NULL32;
          if constexpr (W == 3) x[i].z = base + j > 0 ? in_ids[off + j - 1] : PBIT_NULL32;
        } else {
          x[i] = sm.in[buf][j];
          x[i].x -= v_off;
        }
        r[i] = atomicAdd(&sm.cnt[(x[i].x >> shift) & mask], 1u);
      }
    }
    __syncthreads();
    // exclusive scan of the tile's bin counts; claim the tile's space in every bin
    const uint32_t parent = FROM_IDS ? 0u : base >> (shift + bits);
    uint32_t claim = 0, my_start = 0;
    {
      const uint32_t c = t < nb ? sm.cnt[t] : 0u;
      uint32_t y = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= (uint32_t)o) y += z;
      }
      if (lane == 31) sm.warp[w] = y;
      __syncthreads();
      uint32_t add = 0;
      for (uint32_t q = 0; q < w; ++q) add += sm.warp[q];
      if (t < nb) {
        my_start = y - c + add;
        sm.start[t] = my_start;
        if (c) claim = atomicAdd(cursor + ((parent << bits) | t), c);  // round trip overlaps the staging
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t j = i * PART_THREADS + t;
      if (j < cnt) sm.stage[sm.start[(x[i].x >> shift) & mask] + r[i]] = x[i];
    }
    // gofs[b] = where the bin's claimed run starts minus where it starts in the stage
    // (mod 2^32), so a staged record j goes to gofs[b] + j: one table lookup per record
    if (t < nb) sm.gofs[t] = (((parent << bits) | t) << shift) + claim - my_start;
    __syncthreads();
    // coalesced write-out: consecutive threads store consecutive staged records, which
    // land contiguously inside each bin's run
#pragma unroll 4
    for (uint32_t j = t; j < cnt; j += PART_THREADS) {
      const R p = sm.stage[j];
      const uint32_t b = (p.x >> shift) & mask;
      PBIT_ASSERT(sm.gofs[b] + j < n);
      if constexpr (W == 2) __stcs(pout + (sm.gofs[b] + j), p);
      else pout[sm.gofs[b] + j] = p;
    }
    __syncthreads();  // stage, start and gofs are rewritten by the next tile
  }
}

static __global__ void k_relink_head(const uint32_t* __restrict__ ids, uint32_t* __restrict__ d_head,
                                     const int* __restrict__ err) {
  pdl_enter();
  if (*err) return;
  *d_head = ids[0];
}

// Last step: one CTA per fine bin: scatter into a 64 KB smem window per output, write it
// out coalesced.  FROM_IDS: n <= 2^14, one window, the records come straight from the
// sorted ids.  W = 3 also fills out_prev.
template <bool FROM_IDS, int W>
__global__ void __launch_bounds__(512)
k_relink_apply(const uint32_t* __restrict__ ids, const typename RelinkRec<W>::T* __restrict__ recs, uint32_t n,
               uint32_t v_off, uint32_t* __restrict__ out_next, uint32_t* __restrict__ out_prev,
               const int* __restrict__ err, uint32_t bin0 = 0) {
  using R = typename RelinkRec<W>::T;
  pdl_enter();
  extern __shared__ __align__(16) uint32_t s_win[];  // [W - 1][2^RELINK_FINE_SHIFT]
  uint32_t* s_prev = s_win + (1u << RELINK_FINE_SHIFT);
  if (*err) return;
  const uint32_t f0 = (bin0 + blockIdx.x) << RELINK_FINE_SHIFT;  // launches may cover a range of bins
  const uint32_t cnt = min((uint32_t)(1u << RELINK_FINE_SHIFT), n - f0);
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    if constexpr (FROM_IDS) {
      s_win[ids[i]] = i + 1 < n ? ids[i + 1] : PBIT_NULL32;
      if constexpr (W == 3) s_prev[ids[i]] = i > 0 ? ids[i - 1] : PBIT_NULL32;
    } else {
      R p;
      if constexpr (W == 2) p = __ldcs(recs + f0 + i); else p = recs[f0 + i];
      const uint32_t v = p.x - v_off - f0;
      PBIT_ASSERT(v < (1u << RELINK_FINE_SHIFT));
      s_win[v] = p.y;
      if constexpr (W == 3) s_prev[v] = p.z;
    }
  }
  __syncthreads();
  for (int o = 0; o < W - 1; ++o) {
    uint32_t* dst = (o == 0 ? out_next : out_prev) + f0;
    const uint32_t* src = o == 0 ? s_win : s_prev;
    if ((cnt & 3u) == 0 && ((uintptr_t)dst & 15u) == 0) {
      for (uint32_t i = threadIdx.x; i < cnt / 4; i += blockDim.x)
        __stcs(reinterpret_cast<uint4*>(dst) + i, reinterpret_cast<const uint4*>(src)[i]);
    } else {
      for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = src[i];
    }
  }
}

}  // namespace pbit
