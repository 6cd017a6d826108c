// launch.cuh -- host-side launch helpers shared by pbit.cu and mg.cu.
#pragma once
#include <cuda_runtime.h>

#include <stdlib.h>

#include <algorithm>
#include <utility>
#include <atomic>
#include <mutex>

#include "kernels.cuh"
#include "pbit_internal.h"

namespace pbit {

// cudaFuncSetAttribute is per device: run `set` once per (call site, device) -- under a
// lock, and marked done only after it ran, so a concurrent caller on another stream never
// launches before the attributes are in place.
template <typename F>
static inline void once_per_device(std::atomic<unsigned long long>& done, F&& set) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  set();
  done.fetch_or(bit, std::memory_order_release);
}

// One k_onesweep launch (sets the dynamic-smem attribute once per instantiation).
template <typename KeyT, int RB, int IPT, int RANK, int SRC>
static void launch_one_m(const SweepArgs& a, cudaStream_t st) {
  using S = SweepSmem<KeyT, RB, IPT>;
  constexpr size_t smem = sizeof(S) + (SRC == SRC_SPLIT ? sizeof(SplitTable) : 0);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_onesweep<KeyT, RB, IPT, RANK, SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  });
  const uint32_t ntiles = (a.n + S::TILE - 1) / S::TILE;
  launch_pdl(k_onesweep<KeyT, RB, IPT, RANK, SRC>, ntiles, SWEEP_THREADS, smem, st, a);
}

template <typename KeyT, int RB, int IPT, int SRC = SRC_TMA>
static void launch_one(const SweepArgs& a, cudaStream_t st, int mode) {
  if (mode == RANK_ATOMIC) launch_one_m<KeyT, RB, IPT, RANK_ATOMIC, SRC>(a, st);
  else if (mode == RANK_MATCH) launch_one_m<KeyT, RB, IPT, RANK_MATCH, SRC>(a, st);
  else launch_one_m<KeyT, RB, IPT, RANK_BALLOT, SRC>(a, st);
}

// The key passes of a host-side plan: pass i sorts digit plan.digit[i] (slot i, its own
// ticket counter and lookback epoch), reading buffer i & 1.  first_src: where pass 0's
// tiles come from (SRC_*).  final_ids: if set, the last pass writes its ids there.
template <int KB, int RB>
static void launch_key_passes(SweepArgs a, const Plan& plan, bool keep_keys, cudaStream_t st, cudaEvent_t* ev,
                              int ev_base, int first_src, uint32_t* final_ids = nullptr) {
  using KeyT = typename KeyOf<KB>::T;
  constexpr int IPT = (KB == 8) ? SWEEP_IPT64 : SWEEP_IPT32;
  // PBIT_COMBINE (experiments, tests): 0 never combine, 2 on every pass
  const char* ce = getenv("PBIT_COMBINE");
  const int combine_env = ce ? atoi(ce) : 1;
  for (uint32_t s = 0; s < plan.npasses; ++s) {
    a.slot = (int)s;
    a.digit = (int)plan.digit[s];
    a.src = (int)(s & 1);
    a.last = (s + 1 == plan.npasses) && !keep_keys;
    // lane-0 combining in the ranking: on a skewed digit whose input is sorted by the
    // lower digits (not the first pass) and not yet grouped by key (not the last)
    const bool skewed = (plan.skewed[a.digit >> 5] >> (a.digit & 31)) & 1u;
    a.combine = combine_env == 2 || (combine_env == 1 && skewed && s > 0 && s + 1 < plan.npasses);
    if (final_ids && s + 1 == plan.npasses) a.vout[a.src ^ 1] = final_ids;
    const int src = s == 0 ? first_src : SRC_TMA;
    if (src == SRC_GATHER) launch_one<KeyT, RB, IPT, SRC_GATHER>(a, st, rank_mode());
    else if (src == SRC_IOTA) launch_one<KeyT, RB, IPT, SRC_IOTA>(a, st, rank_mode());
    else launch_one<KeyT, RB, IPT, SRC_TMA>(a, st, rank_mode());
    if (ev) cudaEventRecord(ev[ev_base + s], st);
  }
}

template <int KB>
static void launch_key_passes_k(int K, const SweepArgs& a, const Plan& plan, bool keep_keys, cudaStream_t st,
                                cudaEvent_t* ev, int ev_base, int first_src, uint32_t* final_ids = nullptr) {
  switch (K) {
#define PBIT_K(RB) case RB: launch_key_passes<KB, RB>(a, plan, keep_keys, st, ev, ev_base, first_src, final_ids); break;
    PBIT_K(1) PBIT_K(2) PBIT_K(3) PBIT_K(4) PBIT_K(5) PBIT_K(6) PBIT_K(7) PBIT_K(8)
#undef PBIT_K
  }
}

// Launch with programmatic dependent launch allowed: the kernel (which starts with
// pdl_enter()) may be scheduled while its predecessor on the stream is still draining,
// hiding the launch gap between dependent kernels.  PBIT_PDL=0 builds the plain launch.
#ifndef PBIT_PDL
#define PBIT_PDL 1
#endif
template <typename... KArgs, typename... Args>
static inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = PBIT_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Grid of a grid-stride kernel: at most one full wave (every CTA resident at once).  A
// grid of sms x 8 CTAs for a kernel that fits 6 per SM runs a second, one-third-full wave
// after the first, with every CTA holding an equal share of the work.
template <typename Kern>
static inline int full_wave(Kern kernel, int threads, size_t smem, int sms, uint64_t want_blocks) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
#ifdef PBIT_FIXED_GRID  // A/B experiments: the old fixed grid
  occ = 8;
#endif
  const uint64_t cap = (uint64_t)sms * (uint64_t)std::max(occ, 1);
  return (int)std::max<uint64_t>(1, std::min(want_blocks, cap));
}

// Cursor words launch_relink needs (zeroed by the caller before the call).
static inline size_t relink_cursor_words(uint32_t n) {
  RelinkLevels lv(n);
  size_t c = 0;
  for (int l = 0; l < lv.L; ++l) c += RelinkLevels::cursors(n, lv.shift[l]);
  return c + 1;
}

// a5 relink of n local ids: out_next[v] = succ (and out_prev[v] = pred when out_prev is
// set: records of three words).  Source: the sorted ids (`ids`, records formed on the fly)
// or records (`recs`, v - v_off = local id; pairs if out_prev is NULL, else triples).
// rbuf[2]: n records each (+16 B of padding); when the source is records it must not be
// rbuf[0] (level 0 writes rbuf[0]).  Returns the number of kernels launched.
// Host-buffer calls (pbit_sort_list with host pointers): the apply kernel runs in `chunks`
// launches over consecutive ranges of fine bins, and each range of out_next (out_prev) is
// copied to the host on `copy` as soon as its launch is done, overlapping the D2H with the
// rest of the apply.
struct RelinkD2H {
  int chunks = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t* ev = nullptr;  // chunks events
  uint32_t* h_next = nullptr;
  uint32_t* h_prev = nullptr;
};

template <int W>
static uint32_t launch_relink_w(const uint32_t* ids, const void* recs, uint32_t v_off, uint32_t n, void* rbuf0,
                                void* rbuf1, uint32_t* cursors, uint32_t* out_next, uint32_t* out_prev,
                                const int* err, cudaStream_t st, int sms, const RelinkD2H* d2h = nullptr) {
  using R = typename RelinkRec<W>::T;
  constexpr size_t WIN = (size_t)(W - 1) * (4u << RELINK_FINE_SHIFT);
  static std::atomic<unsigned long long> attr{0};
  static int part_occ = 1;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_relink_apply<true, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WIN);
    cudaFuncSetAttribute(k_relink_apply<false, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WIN);
    cudaFuncSetAttribute(k_relink_part<true, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PartSmem<W>));
    cudaFuncSetAttribute(k_relink_part<false, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PartSmem<W>));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_relink_part<false, W>, PART_THREADS,
                                                      sizeof(PartSmem<W>)) != cudaSuccess) {
      cudaGetLastError();
      occ = 1;
    }
    part_occ = std::max(occ, 1);
  });
  if (n == 0) return 0;
  RelinkLevels lv(n);
  const uint32_t nfine = (n + (1u << RELINK_FINE_SHIFT) - 1) >> RELINK_FINE_SHIFT;
  if (lv.L == 0) {
    if (ids) k_relink_apply<true, W><<<1, 512, WIN, st>>>(ids, nullptr, n, 0, out_next, out_prev, err);
    else k_relink_apply<false, W><<<1, 512, WIN, st>>>(nullptr, (const R*)recs, n, v_off, out_next, out_prev, err);
    return 1;
  }
  constexpr uint32_t TILE = PartCfg<W>::TILE;
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t grid = std::min<uint32_t>(ntiles, (uint32_t)(sms * part_occ));
  const size_t psm = sizeof(PartSmem<W>);
  const R* in = (const R*)recs;
  R* buf[2] = {(R*)rbuf0, (R*)rbuf1};
  if (d2h && d2h->chunks > 1 && lv.L == 2 && ids) {
    // host buffers, two levels: level 0 on everything, then per group of level-0 bins its
    // level-1 partition, its apply and the copy of its ids' results -- the copies start
    // after the first group instead of after the whole level 1
    k_relink_part<true, W><<<grid, PART_THREADS, psm, st>>>(ids, nullptr, buf[0], n, 0, lv.shift[0], lv.bits[0],
                                                            cursors, err);
    uint32_t* cur1 = cursors + RelinkLevels::cursors(n, lv.shift[0]);
    const uint32_t nb0 = ((n - 1) >> lv.shift[0]) + 1;
    const uint32_t per = (nb0 + d2h->chunks - 1) / d2h->chunks;
    uint32_t launched = 1;
    for (int c = 0; c < d2h->chunks; ++c) {
      const uint32_t b0 = c * per, b1 = std::min(nb0, b0 + per);
      if (b0 >= b1) break;
      const uint32_t lo = b0 << lv.shift[0];
      const uint32_t hi = (uint32_t)std::min<uint64_t>(n, (uint64_t)b1 << lv.shift[0]);
      const uint32_t g1 = std::min<uint32_t>((hi - lo + TILE - 1) / TILE, (uint32_t)(sms * part_occ));
      k_relink_part<false, W><<<g1, PART_THREADS, psm, st>>>(nullptr, buf[0], buf[1], hi, 0u, lv.shift[1],
                                                             lv.bits[1], cur1, err, lo);
      const uint32_t f0 = lo >> RELINK_FINE_SHIFT, f1 = (hi + (1u << RELINK_FINE_SHIFT) - 1) >> RELINK_FINE_SHIFT;
      k_relink_apply<false, W><<<f1 - f0, 512, WIN, st>>>(nullptr, buf[1], n, 0, out_next, out_prev, err, f0);
      launched += 2;
      cudaEventRecord(d2h->ev[c], st);
      cudaStreamWaitEvent(d2h->copy, d2h->ev[c], 0);
      cudaMemcpyAsync(d2h->h_next + lo, out_next + lo, (size_t)(hi - lo) * 4, cudaMemcpyDeviceToHost, d2h->copy);
      if (W == 3) cudaMemcpyAsync(d2h->h_prev + lo, out_prev + lo, (size_t)(hi - lo) * 4, cudaMemcpyDeviceToHost, d2h->copy);
    }
    return launched;
  }
  for (int l = 0; l < lv.L; ++l) {
    R* out = buf[l & 1];
    if (l == 0 && ids)
      k_relink_part<true, W><<<grid, PART_THREADS, psm, st>>>(ids, nullptr, out, n, 0, lv.shift[l], lv.bits[l],
                                                              cursors, err);
    else
      k_relink_part<false, W><<<grid, PART_THREADS, psm, st>>>(nullptr, in, out, n, l == 0 ? v_off : 0u,
                                                               lv.shift[l], lv.bits[l], cursors, err);
    cursors += RelinkLevels::cursors(n, lv.shift[l]);
    in = out;
  }
  // the relink kernels are launched plainly: with PDL the waiting apply CTAs would take
  // SM room from the persistent partition kernel (C3 relink +0.04 ms, measured)
  if (!d2h || d2h->chunks <= 1) {
    k_relink_apply<false, W><<<nfine, 512, WIN, st>>>(nullptr, in, n, 0, out_next, out_prev, err);
    return (uint32_t)lv.L + 1;
  }
  const uint32_t per = (nfine + d2h->chunks - 1) / d2h->chunks;
  uint32_t launched = (uint32_t)lv.L;
  for (int c = 0; c < d2h->chunks; ++c) {
    const uint32_t b0 = c * per, b1 = std::min(nfine, b0 + per);
    if (b0 >= b1) break;
    k_relink_apply<false, W><<<b1 - b0, 512, WIN, st>>>(nullptr, in, n, 0, out_next, out_prev, err, b0);
    ++launched;
    cudaEventRecord(d2h->ev[c], st);
    cudaStreamWaitEvent(d2h->copy, d2h->ev[c], 0);
    const size_t v0 = (size_t)b0 << RELINK_FINE_SHIFT, v1 = std::min((size_t)n, (size_t)b1 << RELINK_FINE_SHIFT);
    cudaMemcpyAsync(d2h->h_next + v0, out_next + v0, (v1 - v0) * 4, cudaMemcpyDeviceToHost, d2h->copy);
    if (W == 3) cudaMemcpyAsync(d2h->h_prev + v0, out_prev + v0, (v1 - v0) * 4, cudaMemcpyDeviceToHost, d2h->copy);
  }
  return launched;
}

static inline uint32_t launch_relink(const uint32_t* ids, const void* recs, uint32_t v_off, uint32_t n, void* rbuf0,
                                     void* rbuf1, uint32_t* cursors, uint32_t* out_next, uint32_t* out_prev,
                                     const int* err, cudaStream_t st, int sms, const RelinkD2H* d2h = nullptr) {
  return out_prev
             ? launch_relink_w<3>(ids, recs, v_off, n, rbuf0, rbuf1, cursors, out_next, out_prev, err, st, sms, d2h)
             : launch_relink_w<2>(ids, recs, v_off, n, rbuf0, rbuf1, cursors, out_next, nullptr, err, st, sms, d2h);
}

}  // namespace pbit
