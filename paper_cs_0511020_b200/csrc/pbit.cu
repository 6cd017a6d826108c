// pbit.cu -- host orchestrator + C-ABI entry of the single-GPU Pbit list sort.
//
// pbit_sort_list (include/pbit.h) runs, on the caller's stream:
//   k_pack -> k_plan [its pass plan is copied to the host and read while the walk runs]
//   -> k_walk -> k_rank_walk_a, k_rank_jump^r (or k_rank_jump_block), k_rank_walk_b
//   -> k_onesweep per non-trivial digit (the first gathers from the walk's slots;
//      k_gather only when no pass runs) -> k_relink_part per level -> k_relink_apply
// then one small D2H of {head, error, passes} and a stream sync.  Host buffers: the copies
// run on a second stream in chunks, overlapped with the pack and the apply (HostIO).
// pbit_sort_array (the "table" of P:1118-1177) runs k_array_prep -> k_plan -> the passes.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "../../include/pbit.h"
#include "kernels.cuh"
#include "pbit_internal.h"
#include "launch.cuh"
#include "small.cuh"

namespace pbit {

// Text of the last CUDA/NCCL failure seen by this host thread (pbit_last_error()).
static thread_local char g_last_err[256] = "";

// The small host-visible results of a call (the pass plan mid-call; head, error word and
// pass count at the end) land in pinned memory: into a pageable destination each small
// cudaMemcpyAsync is a staged copy that blocks the host.  One box per host thread (calls
// are synchronous, so a thread has at most one call in flight).
struct HostBox {
  Plan plan;
  int err;
  uint32_t head, npasses;
  uint32_t small[4];  // run_small: {err, head, passes}
};
static HostBox* host_box() {
  struct Holder {
    HostBox* pinned = nullptr;
    HostBox pageable{};
    bool tried = false;
    ~Holder() { if (pinned) cudaFreeHost(pinned); }
  };
  static thread_local Holder h;
#ifndef PBIT_PAGEABLE_RESULTS
  if (!h.tried) {
    h.tried = true;
    if (cudaHostAlloc((void**)&h.pinned, sizeof(HostBox), cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      h.pinned = nullptr;
    }
  }
#endif
  return h.pinned ? h.pinned : &h.pageable;
}
void set_last_error(const char* what, const char* detail) {
  snprintf(g_last_err, sizeof g_last_err, "%s: %s", what, detail ? detail : "");
}

// ----------------------------------------------------------------------------- device info
// Per device: SM count, and the library's own stream-ordered memory pool for workspace.
// The pool's release threshold is 0 by default (PBIT_POOL_KEEP_GB=x keeps x GB mapped
// between calls); the device's default pool, which other code may use, is left alone.
// pbit_workspace_trim() hands cached workspace back.
struct DevInfo {
  int sms = 0;
  cudaMemPool_t pool = nullptr;
};
static std::mutex g_dev_mu;
static DevInfo g_dev[64];

int device_info(int dev, int* sms) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (dev < 0 || dev >= 64) return PBIT_ERR_CUDA;
  DevInfo& d = g_dev[dev];
  if (!d.sms) {
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return PBIT_ERR_CUDA;
  }
  if (!d.pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return PBIT_ERR_CUDA;
    }
    // default 0: workspace goes back to the device when a call ends (the paper's sort
    // needs O(1) memory; this one O(n) only while it runs).  PBIT_POOL_KEEP_GB=x
    // keeps up to x GB mapped between calls (repeated calls then skip the re-mapping)
    const char* e = getenv("PBIT_POOL_KEEP_GB");
    uint64_t keep = e ? (uint64_t)(atof(e) * 1e9) : 0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    d.pool = pool;
  }
  *sms = d.sms;
  return PBIT_OK;
}

cudaError_t ws_alloc(void** ptr, size_t bytes, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (device_info(dev, &sms) != PBIT_OK) return cudaErrorMemoryAllocation;
  e = cudaMallocFromPoolAsync(ptr, bytes, g_dev[dev].pool, st);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

// ----------------------------------------------------------------------------- planning
void make_plan(uint64_t n, int key_bits, int K, SortPlan* p) {
  p->n = (uint32_t)n;
  p->key_bits = key_bits;
  p->K = K;
  p->D = (key_bits + K - 1) / K;
  // ruler spacing 2^s_log2 nodes per segment, by list size (measured): the
  // walk wants enough segments per resident walker that the longest chains do not set
  // its time (shorter segments on mid-size lists), ranking and pass 0's gather want fewer,
  // longer segments (longer ones on the largest lists, where the ruler list's ranking
  // leaves the L2)
  static const int env_s = [] { const char* e = getenv("PBIT_RULER_LOG2"); return e ? atoi(e) : -1; }();
  int s_log2 = n >= (1ull << 30) ? 7 : n >= (1ull << 26) ? 6 : n >= (1ull << 24) ? 5 : n >= (1ull << 22) ? 4 : 5;
  if (env_s > 0) s_log2 = env_s;
  while (s_log2 > 2 && (n >> s_log2) < (1u << 13)) --s_log2;
  p->s_log2 = s_log2;
#ifndef PBIT_CAP_SHIFT
#define PBIT_CAP_SHIFT 2
#endif
  p->cap = (1u << PBIT_CAP_SHIFT) << s_log2;
  p->R = (uint32_t)((n + (1ull << s_log2) - 1) >> s_log2);
  // one sub-ruler per 8 rulers on ruler lists below 2^20 (their sub-segment walks are the
  // latency-bound part), per 16 above (where the pointer jumping over the sub-rulers is);
  // measured, DESIGN.md §7
  static const int env_sub = [] { const char* e = getenv("PBIT_SUB_LOG2"); return e ? atoi(e) : -1; }();
  p->sub_log2 = env_sub > 0 ? env_sub : (p->R < (1u << 20) ? 3 : 4);
  p->dyn_cap = (uint32_t)(n / p->cap + 1);
}

static int debug_env(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}

// the pointer jumping of the ranking as one launch per round chained by programmatic
// dependent launch (default), or all rounds in one cooperative launch (PBIT_RANK_GRID=1:
// measured slower -- the grid barrier costs more than a PDL-chained launch)
static bool rank_grid_enabled() {
  static const bool v = [] { const char* e = getenv("PBIT_RANK_GRID"); return e && atoi(e) == 1; }();
  return v;
}

// PBIT_SMALL=0 sends small lists through the general path too (experiments, tests)
static bool small_path_disabled() {
  static const bool v = [] { const char* e = getenv("PBIT_SMALL"); return e && atoi(e) == 0; }();
  return v;
}

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

#ifndef PBIT_EARLY_PLAN
#define PBIT_EARLY_PLAN 1
#endif

// ----------------------------------------------------------------------------- dispatch
// In-warp ranking mode for the stable key passes, per device: RANK_ATOMIC unless that
// device's self-test fails (or PBIT_RANK=ballot|match|atomic overrides, for experiments).
// The lane order of conflicting shared atomics is measured, not documented, so it is
// checked on every device before its first sort (pbit_rank_mode() reports the verdict).
static std::atomic<int> g_rank_mode[64];
static std::once_flag g_rank_init;

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); dev = 0; }
  return dev & 63;
}

int rank_mode() { return g_rank_mode[current_device()].load(std::memory_order_relaxed); }

void init_rank_mode(cudaStream_t st) {
  std::call_once(g_rank_init, [] { for (auto& m : g_rank_mode) m.store(-1); });
  std::atomic<int>& slot = g_rank_mode[current_device()];
  if (slot.load() >= 0) return;
  int mode = RANK_ATOMIC;
  if (const char* e = getenv("PBIT_RANK")) {
    mode = !strcmp(e, "ballot") ? RANK_BALLOT : !strcmp(e, "match") ? RANK_MATCH : RANK_ATOMIC;
  } else {
    uint32_t* d_bad = nullptr;
    uint32_t bad = 1;
    if (ws_alloc((void**)&d_bad, 4, st) == cudaSuccess) {
      cudaMemsetAsync(d_bad, 0, 4, st);
      k_selftest_atomic_order<<<64, 256, 0, st>>>(4096, d_bad);
      cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st);
      cudaFreeAsync(d_bad, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) bad = 1;
    }
    cudaGetLastError();
    if (bad) mode = RANK_BALLOT;
  }
  slot.store(mode);
}

size_t sweep_tile(int key_bits) { return (size_t)SWEEP_THREADS * (key_bits == 64 ? SWEEP_IPT64 : SWEEP_IPT32); }

// Workspace layout (all 256-byte aligned).
struct Ws {
  void* kn; void* slots; uint2* seg; uint32_t* dist;
  unsigned long long* sdist[2]; uint32_t* scnt[2]; uint32_t* ssucc[2]; uint32_t* seg_ord; uint32_t* seg_pos;
  uint32_t* tile_first;
  void* keys[2]; uint32_t* ids[2]; unsigned long long* status; uint2* pairs[2];
  // control block (zeroed per call)
  uint32_t* hist; uint32_t* bases; Plan* plan; int* err; uint32_t* dyn_count; uint32_t* tile_ctr; uint32_t* d_head;
  uint32_t* cursors; uint32_t* nseg;
  size_t ctl_bytes; void* ctl; size_t status_bytes;
};

static size_t carve(const SortPlan& p, char* base, Ws* w) {
  const size_t n = p.n;
  const int kb = p.key_bits / 8;
  const size_t rec = kb == 8 ? 16 : 8;
  const size_t kbytes = kb == 8 ? 8 : 4;
  const size_t Rmax = (size_t)p.R + 1 + p.dyn_cap;
  const int radix = 1 << p.K;
  const size_t tile = sweep_tile(p.key_bits);
  const size_t ntiles = (n + tile - 1) / tile;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* q = base ? base + off : nullptr; off += align_up(bytes); return (void*)q; };
  w->kn = take(n * rec);
  // the slots also hold the two relink record buffers (dead slots by then): n records of
  // up to 12 B (v, succ, pred) each, plus the 16 B of padding the tile loads may read
  const size_t rbuf = align_up(n * 12 + 16);
  w->slots = take(std::max(Rmax * p.cap * rec, 2 * rbuf));
  for (int i = 0; i < 2; ++i) w->pairs[i] = base ? (uint2*)((char*)w->slots + i * rbuf) : nullptr;
  w->seg = (uint2*)take(Rmax * 8);
  w->dist = (uint32_t*)take(Rmax * 4);
  const size_t nsub = (Rmax >> p.sub_log2) + 2;
  for (int i = 0; i < 2; ++i) {
    w->sdist[i] = (unsigned long long*)take(nsub * 8);
    w->scnt[i] = (uint32_t*)take(nsub * 4);
    w->ssucc[i] = (uint32_t*)take(nsub * 4);
  }
  w->seg_ord = (uint32_t*)take(Rmax * 4);
  w->seg_pos = (uint32_t*)take(Rmax * 4);
  w->tile_first = (uint32_t*)take((ntiles + 1) * 4);
  for (int i = 0; i < 2; ++i) { w->keys[i] = take(n * kbytes); w->ids[i] = (uint32_t*)take(n * 4); }
  w->status_bytes = ntiles * (radix > 256 ? radix : 256) * 8;  // relink passes use 256
  w->status = (unsigned long long*)take(w->status_bytes);
  const size_t ctl0 = off;
  w->hist = (uint32_t*)take((size_t)p.D * radix * 4);
  w->bases = (uint32_t*)take((size_t)p.D * radix * 4);
  w->plan = (Plan*)take(sizeof(Plan));
  w->err = (int*)take(4);
  w->dyn_count = (uint32_t*)take(4);
  w->tile_ctr = (uint32_t*)take(80 * 4);
  w->d_head = (uint32_t*)take(4);
  w->cursors = (uint32_t*)take(relink_cursor_words(p.n) * 4);
  w->nseg = (uint32_t*)take(4);
  w->ctl = base ? base + ctl0 : nullptr;
  w->ctl_bytes = off - ctl0;
  return off;
}

// ----------------------------------------------------------------------------- host buffers
// pbit_sort_list on host buffers: the keys and successors go to the device in HOSTIO_CHUNKS
// copies on a second stream, each chunk packed as soon as it has landed, and out_next
// (out_prev) comes back in as many copies, each as soon as the relink's apply kernel has
// written its range of ids -- the copies overlap the pack and the apply instead of
// bracketing the whole call.
constexpr int HOSTIO_CHUNKS = 8;
struct HostIO {
  const void* h_keys;
  const uint32_t* h_next;
  uint32_t* h_out;
  uint32_t* h_prev;
  cudaStream_t copy;
  cudaEvent_t* ev;  // HOSTIO_CHUNKS events
  bool results_copied = false;  // set once the relink has queued the result copies
};
static void hostio_resources(cudaStream_t* copy, cudaEvent_t** ev) {
  // one copy stream and its events per (host thread, device), released when the thread ends
  struct Res {
    cudaStream_t cs[64] = {};
    cudaEvent_t evs[64][HOSTIO_CHUNKS] = {};
    ~Res() {
      for (int d = 0; d < 64; ++d) {
        if (!cs[d]) continue;
        cudaStreamDestroy(cs[d]);
        for (int i = 0; i < HOSTIO_CHUNKS; ++i) cudaEventDestroy(evs[d][i]);
      }
    }
  };
  static thread_local Res r;
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (!r.cs[dev]) {
    cudaStreamCreateWithFlags(&r.cs[dev], cudaStreamNonBlocking);
    for (int i = 0; i < HOSTIO_CHUNKS; ++i) cudaEventCreateWithFlags(&r.evs[dev][i], cudaEventDisableTiming);
  }
  *copy = r.cs[dev];
  *ev = r.evs[dev];
}

// ----------------------------------------------------------------------------- the device path
template <int KB>
static int run_device(const void* keys, const uint32_t* next, uint32_t head, const SortPlan& p, uint32_t* out_next,
                      uint32_t* out_prev, uint32_t* out_head, cudaStream_t st, int sms, float* phase_ms,
                      uint32_t* passes_run, uint32_t* launches_out, HostIO* hio = nullptr,
                      uint32_t* out_order = nullptr, void* out_keys = nullptr) {
  using RT = typename Rec<KB>::T;
  Ws w;
  const size_t bytes = carve(p, nullptr, &w);
  char* base = nullptr;
  if (ws_alloc((void**)&base, bytes, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  carve(p, base, &w);

  // phase events come from a per-thread pool (created once), so timed calls carry no
  // event creation on the host between kernels
  static thread_local cudaEvent_t ev_pool[64][PBIT_NUM_PHASES + 1];
  static thread_local bool ev_ready[64] = {};
  const bool timing = phase_ms != nullptr;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  cudaEvent_t* ev = ev_pool[cur_dev & 63];
  if (timing) {
    if (!ev_ready[cur_dev & 63]) {
      for (int i = 0; i <= PBIT_NUM_PHASES; ++i) cudaEventCreate(&ev[i]);
      ev_ready[cur_dev & 63] = true;
    }
    cudaEventRecord(ev[PBIT_NUM_PHASES], st);  // start
  }
  const uint32_t n = p.n;
  const int radix = 1 << p.K;
  uint32_t launches = 0;
  init_rank_mode(st);

  cudaMemsetAsync(w.ctl, 0, w.ctl_bytes, st);
  cudaMemsetAsync(w.status, 0, w.status_bytes, st);

  // a1/a2: pack + histograms
  {
    NvtxRange nv("pbit.pack");
    const size_t smem = (size_t)p.D * radix * 4;
    const int blocks = full_wave(k_pack<KB>, PACK_THREADS, smem, sms, (n + PACK_THREADS - 1) / PACK_THREADS);
    const KeyMap km{p.key_kind, p.descending};
    if (!hio) {
      launch_pdl(k_pack<KB>, blocks, PACK_THREADS, smem, st, keys, next, n, n, (RT*)w.kn, w.hist, p.K, p.D, w.err, km);
      ++launches;
    } else {  // copy chunk c on the copy stream, pack it on st once it has landed
      cudaEventRecord(hio->ev[0], st);  // the staging buffers were allocated on st
      cudaStreamWaitEvent(hio->copy, hio->ev[0], 0);
      const uint32_t per = (uint32_t)((((uint64_t)n + HOSTIO_CHUNKS - 1) / HOSTIO_CHUNKS + 255) & ~255ull);
      for (int c = 0; c < HOSTIO_CHUNKS; ++c) {
        const uint32_t v0 = c * per;
        if (v0 >= n) break;
        const uint32_t cnt = std::min(per, n - v0);
        cudaMemcpyAsync((char*)keys + (size_t)v0 * KB, (const char*)hio->h_keys + (size_t)v0 * KB, (size_t)cnt * KB,
                        cudaMemcpyHostToDevice, hio->copy);
        cudaMemcpyAsync((uint32_t*)next + v0, hio->h_next + v0, (size_t)cnt * 4, cudaMemcpyHostToDevice, hio->copy);
        cudaEventRecord(hio->ev[c], hio->copy);
        cudaStreamWaitEvent(st, hio->ev[c], 0);
        const int cb = full_wave(k_pack<KB>, PACK_THREADS, smem, sms, (cnt + PACK_THREADS - 1) / PACK_THREADS);
        k_pack<KB><<<cb, PACK_THREADS, smem, st>>>((const char*)keys + (size_t)v0 * KB, next + v0, cnt, n,
                                                    (RT*)w.kn + v0, w.hist, p.K, p.D, w.err, km);
        ++launches;
      }
    }
  }
#if PBIT_EARLY_PLAN
  // a3, early: the bucket bases and the pass plan depend only on the histograms, complete
  // after the pack.  The plan is copied to the host now and read while the walk runs, so
  // the passes are queued behind the ranking with no host round trip in between; every
  // later kernel checks the device error word itself (an invalid list found by the walk
  // or the ranking stops them, and out_next stays untouched).
  launch_pdl(k_plan, 1, 256, 0, st, w.hist, w.bases, w.plan, p.D, p.K, n, w.err);
  ++launches;
  HostBox* hb = host_box();
  cudaMemcpyAsync(&hb->plan, w.plan, sizeof(Plan), cudaMemcpyDeviceToHost, st);
  static thread_local cudaEvent_t plan_ev[64] = {};
  cudaEvent_t& pev = plan_ev[cur_dev & 63];
  if (!pev) cudaEventCreateWithFlags(&pev, cudaEventDisableTiming);
  cudaEventRecord(pev, st);
#endif
  if (timing) cudaEventRecord(ev[PBIT_PHASE_PACK], st);

  // a1: walk
  RulerSel sel{n, (uint32_t)p.s_log2, p.R};
  nvtxRangePushA("pbit.walk");
  const bool head_is_ruler = sel.is_ruler(head);
  const uint32_t R_static = p.R + (head_is_ruler ? 0u : 1u);
  const uint32_t head_ruler = head_is_ruler ? (head >> p.s_log2) : p.R;
  {
    static const int walk_occ = [] {  // resident walk CTAs per SM (one arch per process)
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_walk<KB, false>, WALK_THREADS, 0);
      occ = std::max(occ, 1);
      if (int cap_occ = debug_env("PBIT_WALK_OCC")) occ = std::min(occ, cap_occ);  // experiments
      return occ;
    }();
    int blocks = sms * walk_occ;  // one wave: the rulers are split statically over the CTAs
    const uint32_t min_per = 4;
    if ((uint32_t)blocks * min_per > R_static) blocks = std::max(1u, (R_static + min_per - 1) / min_per);
    const uint32_t per_cta = (R_static + blocks - 1) / blocks;
    KnSrc<RT> src{};
    src.kn = (const RT*)w.kn;
    const WalkMap wm{0u, p.R, head_is_ruler ? PBIT_NULL32 : p.R, p.R, R_static, R_static};  // slot(r) = r
    launch_pdl(k_walk<KB, false>, blocks, WALK_THREADS, 0, st, src, sel, wm, head, (RT*)w.slots, p.cap,
               w.seg, w.dyn_count, p.dyn_cap, per_cta, w.err, debug_env("PBIT_DEBUG_WALK_NOWRITE"));
    ++launches;
  }
  if (timing) cudaEventRecord(ev[PBIT_PHASE_WALK], st);
  nvtxRangePop();

  // a1: ruler ranking (second ruling set + pointer jumping over the sub-rulers)
  {
    NvtxRange nv("pbit.rank");
    const uint32_t Rmax = R_static + p.dyn_cap;
    const int SUB_LOG2 = p.sub_log2;
    RulerSel sub{Rmax, (uint32_t)SUB_LOG2, (Rmax + (1u << SUB_LOG2) - 1) >> SUB_LOG2};
    const bool hs = sub.is_ruler(head_ruler);
    const uint32_t nsub = sub.R + (hs ? 0u : 1u);
    const uint32_t head_sub = hs ? (head_ruler >> SUB_LOG2) : sub.R;
    const int sblocks = full_wave(k_rank_walk_a, 256, 0, sms, (nsub + 255) / 256);
    launch_pdl(k_rank_walk_a, sblocks, 256, 0, st, w.seg, sub, R_static, w.dyn_count, p.dyn_cap, head_ruler, nsub,
               w.sdist[0], w.scnt[0], w.ssucc[0], w.err);
    int rounds = 1;
    while ((1ull << rounds) < nsub) ++rounds;
    rounds += 1;
    int cur = 0;
    if (nsub <= (uint32_t)RANK_SMALL) {  // every round in one CTA (small lists: launch latency)
      static std::atomic<unsigned long long> attr{0};
      once_per_device(attr, [] {
        cudaFuncSetAttribute(k_rank_jump_block, cudaFuncAttributeMaxDynamicSharedMemorySize, RANK_SMALL * 32);
      });
      launch_pdl(k_rank_jump_block, 1, 1024, RANK_SMALL * 32, st, w.sdist[0], w.scnt[0], w.ssucc[0], nsub, rounds,
                 head_sub, n, w.err);
      launches += 1;
    } else if (rank_grid_enabled()) {  // every round in one cooperative launch
      static std::atomic<unsigned long long> attr{0};
      static int occ = 1;
      once_per_device(attr, [] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_rank_jump_grid, 256, 0) != cudaSuccess) {
          cudaGetLastError();
          o = 1;
        }
        occ = std::max(o, 1);
      });
      const int gblocks = std::max(1, std::min(sblocks, sms * occ));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = gblocks;
      cfg.blockDim = 256;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_rank_jump_grid, w.sdist[0], w.scnt[0], w.ssucc[0], w.sdist[1], w.scnt[1],
                         w.ssucc[1], nsub, rounds, head_sub, n, w.err);
      cur = rounds & 1;
      launches += 1;
    } else {
      for (int i = 0; i < rounds; ++i) {
        launch_pdl(k_rank_jump, sblocks, 256, 0, st, w.sdist[cur], w.scnt[cur], w.ssucc[cur], w.sdist[cur ^ 1],
                   w.scnt[cur ^ 1], w.ssucc[cur ^ 1], nsub, w.err);
        cur ^= 1;
      }
      launch_pdl(k_rank_check, 1, 1, 0, st, w.sdist[cur], w.ssucc[cur], head_sub, n, w.err);
      launches += rounds + 1;
    }
    launch_pdl(k_rank_walk_b, sblocks, 256, 0, st, w.seg, sub, R_static, w.dyn_count, p.dyn_cap, head_ruler, nsub,
               head_sub, w.sdist[cur], w.scnt[cur], w.dist, w.seg_ord, w.seg_pos, w.tile_first,
               (uint32_t)sweep_tile(p.key_bits), n, w.nseg, w.err);
    launches += 2;
    if (timing) cudaEventRecord(ev[PBIT_PHASE_RANK], st);
    if (hio) {  // the error word is final once the ranking has validated the list
      cudaMemcpyAsync(&hb->err, w.err, 4, cudaMemcpyDeviceToHost, st);
      cudaEventRecord(hio->ev[HOSTIO_CHUNKS - 1], st);
    }
  }
  // the host reads the pass plan once, so every pass gets its digit and parity as kernel
  // parameters and trivial digits are not launched
#if PBIT_EARLY_PLAN
  const bool ok = cudaEventSynchronize(pev) == cudaSuccess;  // long complete: the walk ran since
  const Plan hplan = hb->plan;
#else
  launch_pdl(k_plan, 1, 256, 0, st, w.hist, w.bases, w.plan, p.D, p.K, n, w.err);
  ++launches;
  HostBox* hb = host_box();
  cudaMemcpyAsync(&hb->plan, w.plan, sizeof(Plan), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hb->err, w.err, 4, cudaMemcpyDeviceToHost, st);
  int herr = cudaStreamSynchronize(st) != cudaSuccess ? -1 : hb->err;
  const Plan hplan = hb->plan;
  const bool ok = herr == 0;
#endif
  if (ok && hplan.npasses == 0) {  // a1: gather to list order -- only when no pass can fuse it
    const uint32_t Rmax = R_static + p.dyn_cap;
    const int gblocks = full_wave(k_gather<KB>, 256, 0, sms, (Rmax + 8 * GATHER_SEGS - 1) / (8 * GATHER_SEGS));
    k_gather<KB><<<gblocks, 256, 0, st>>>((const RT*)w.slots, p.cap, w.seg, w.dist, w.seg_ord, w.nseg, n,
                                          (typename KeyOf<KB>::T*)w.keys[0], w.ids[0], w.plan, w.err);
    ++launches;
  }
  if (timing) cudaEventRecord(ev[PBIT_PHASE_GATHER], st);

  // a3/a4: passes
  nvtxRangePushA("pbit.passes");
  SweepArgs sa{};
  sa.kin[0] = w.keys[0]; sa.kin[1] = w.keys[1]; sa.vin[0] = w.ids[0]; sa.vin[1] = w.ids[1];
  sa.kout[0] = w.keys[0]; sa.kout[1] = w.keys[1]; sa.vout[0] = w.ids[0]; sa.vout[1] = w.ids[1];
  sa.bases = w.bases; sa.status = w.status; sa.tile_ctr = w.tile_ctr; sa.err = w.err; sa.n = n;
  sa.slots = w.slots; sa.cap = p.cap; sa.seg = w.seg; sa.seg_ord = w.seg_ord; sa.seg_pos = w.seg_pos;
  sa.tile_first = w.tile_first; sa.nseg = w.nseg;
  { const char* e = getenv("PBIT_DEBUG_NO_LOOKBACK"); sa.debug_no_lookback = e ? atoi(e) : 0; }
  if (ok) {
    // out_keys (N3 records): the last pass keeps the keys too
    launch_key_passes_k<KB>(p.K, sa, hplan, out_keys != nullptr, st, timing ? ev : nullptr, PBIT_PHASE_PASS0,
                            SRC_GATHER);
    launches += hplan.npasses;
  }
  if (timing)
    for (int s2 = ok ? (int)hplan.npasses : 0; s2 < p.D; ++s2) cudaEventRecord(ev[PBIT_PHASE_PASS0 + s2], st);

  nvtxRangePop();
  // a5: relink: (v, succ) pairs grouped by v's fine bin (MSD partition levels), then
  // each 2^14-id bin applied in a shared-memory window
  // host buffers: the results are copied to the caller's arrays while the apply runs, so an
  // invalid list must be known before the relink is queued (out_next is never touched
  // then); the host waits for the ranking here while the passes run
  const bool valid_for_copy = !hio || (cudaEventSynchronize(hio->ev[HOSTIO_CHUNKS - 1]) == cudaSuccess && hb->err == 0);
  if (ok && valid_for_copy && !sa.debug_no_lookback) {
    NvtxRange nv("pbit.relink");
    const uint32_t* fin = w.ids[hplan.npasses & 1u];  // buffer holding the final ids
    launch_pdl(k_relink_head, 1, 1, 0, st, fin, w.d_head, w.err);
    ++launches;
    if (out_order || out_keys) {  // N3: the sorted records (skipped for an invalid list)
      const int mb = full_wave(k_materialize<KB>, 256, 0, sms, (n + 255) / 256);
      const KeyMap km{p.key_kind, p.descending};
      launch_pdl(k_materialize<KB>, mb, 256, 0, st, fin, (const typename KeyOf<KB>::T*)w.keys[hplan.npasses & 1u], n,
                 out_order, out_keys, km, w.err);
      ++launches;
    }
    // N2: with out_prev the records are (v, succ, pred): both outputs in one chain
    RelinkD2H d2h;
    if (hio && RelinkLevels(n).L > 0) {
      d2h.chunks = HOSTIO_CHUNKS;
      d2h.copy = hio->copy;
      d2h.ev = hio->ev;
      d2h.h_next = hio->h_out;
      d2h.h_prev = hio->h_prev;
      hio->results_copied = true;
    }
    launches += launch_relink(fin, nullptr, 0, n, w.pairs[0], w.pairs[1], w.cursors, out_next, out_prev, w.err, st,
                              sms, hio ? &d2h : nullptr);
    if (hio && hio->results_copied) {  // the workspace and the staging buffers outlive the copies
      cudaEventRecord(hio->ev[0], hio->copy);
      cudaStreamWaitEvent(st, hio->ev[0], 0);
    }
  }
  if (timing) cudaEventRecord(ev[PBIT_PHASE_RELINK], st);

  // results: {head, err, npasses}
  HostBox& res = *hb;
  cudaError_t e1 = cudaMemcpyAsync(&res.head, w.d_head, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaMemcpyAsync(&res.err, w.err, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e3 = cudaMemcpyAsync(&res.npasses, &w.plan->npasses, 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(base, st);
  cudaError_t es = cudaStreamSynchronize(st);
  cudaError_t el = cudaGetLastError();
  int rc = PBIT_OK;
  if (e1 || e2 || e3 || es || el) {
    rc = PBIT_ERR_CUDA;
    const cudaError_t e = es ? es : el ? el : e1 ? e1 : e2 ? e2 : e3;
    set_last_error("pbit_sort_list", cudaGetErrorString(e));
  }
  if (timing) {
    if (rc == PBIT_OK) {
      for (int i = 0; i < PBIT_NUM_PHASES; ++i) phase_ms[i] = 0.f;
      cudaEvent_t prev = ev[PBIT_NUM_PHASES];
      auto el_ms = [&](cudaEvent_t a, cudaEvent_t b) { float ms = 0; cudaEventElapsedTime(&ms, a, b); return ms; };
      phase_ms[PBIT_PHASE_PACK] = el_ms(prev, ev[PBIT_PHASE_PACK]);
      phase_ms[PBIT_PHASE_WALK] = el_ms(ev[PBIT_PHASE_PACK], ev[PBIT_PHASE_WALK]);
      phase_ms[PBIT_PHASE_RANK] = el_ms(ev[PBIT_PHASE_WALK], ev[PBIT_PHASE_RANK]);
      phase_ms[PBIT_PHASE_GATHER] = el_ms(ev[PBIT_PHASE_RANK], ev[PBIT_PHASE_GATHER]);
      cudaEvent_t a = ev[PBIT_PHASE_GATHER];
      for (int s = 0; s < p.D; ++s) { phase_ms[PBIT_PHASE_PASS0 + s] = el_ms(a, ev[PBIT_PHASE_PASS0 + s]); a = ev[PBIT_PHASE_PASS0 + s]; }
      phase_ms[PBIT_PHASE_RELINK] = el_ms(a, ev[PBIT_PHASE_RELINK]);
    }
  }
  if (rc) return rc;
  if (res.err) return PBIT_ERR_INVALID_LIST;
  *out_head = res.head;
  if (passes_run) *passes_run = res.npasses;
  if (launches_out) *launches_out = launches;
  return PBIT_OK;
}

bool key_kind_ok(int key_kind, int key_bits) {
  if (key_kind == PBIT_KEY_UNSIGNED || key_kind == PBIT_KEY_SIGNED) return true;
  return key_kind == PBIT_KEY_FLOAT && key_bits >= 16;  // IEEE binary16/32/64
}

// Small lists (n <= SMALL_N): the whole sort in one cluster launch (small.cuh).  Digit
// widths 4 (the paper's) and 8; phase_ms reports the kernel under PBIT_PHASE_WALK.
template <int KB>
static int run_small(const void* keys, const uint32_t* next, uint32_t head, uint32_t n, int K, KeyMap km,
                     uint32_t* out_next, uint32_t* out_prev, uint32_t* out_head, cudaStream_t st, float* phase_ms,
                     uint32_t* passes_run, uint32_t* launches_out) {
  using KeyT = typename KeyOf<KB>::T;
  const size_t a4 = align_up((size_t)n * 4), ak = align_up((size_t)n * sizeof(KeyT));
  const size_t bytes = 6 * a4 + 2 * ak + align_up(SMALL_CTAS * 256 * 4) + 256;  // dn: 2 x 2 x a4
  char* base = nullptr;
  if (ws_alloc((void**)&base, bytes, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  SmallArgs sa{};
  sa.keys = keys; sa.next = next; sa.head = head; sa.n = n; sa.out_next = out_next; sa.out_prev = out_prev;
  sa.km = km;
  char* q = base;
  for (int i = 0; i < 2; ++i) { sa.dn[i] = (uint2*)q; q += 2 * a4; }
  for (int i = 0; i < 2; ++i) { sa.lid[i] = (uint32_t*)q; q += a4; sa.lkey[i] = q; q += ak; }
  sa.hist = (uint32_t*)q; q += align_up(SMALL_CTAS * 256 * 4);
  sa.err = (int*)q; sa.d_head = (uint32_t*)(q + 4); sa.passes = (uint32_t*)(q + 8);
  static thread_local cudaEvent_t ev[2];
  static thread_local bool ev_ready = false;
  if (phase_ms && !ev_ready) { cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]); ev_ready = true; }
  if (phase_ms) cudaEventRecord(ev[0], st);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    if (SMALL_CTAS > 8) {
      cudaFuncSetAttribute(k_small_sort<KB, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_small_sort<KB, 8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
  });
  if (K == 4) k_small_sort<KB, 4><<<SMALL_CTAS, SMALL_THREADS, 0, st>>>(sa);
  else k_small_sort<KB, 8><<<SMALL_CTAS, SMALL_THREADS, 0, st>>>(sa);
  if (phase_ms) cudaEventRecord(ev[1], st);
  uint32_t* res_words = host_box()->small;
  cudaMemcpyAsync(res_words, q, 12, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(base, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  const cudaError_t el = cudaGetLastError();
  if (es || el) {
    set_last_error("pbit_sort_list (small)", cudaGetErrorString(es ? es : el));
    return PBIT_ERR_CUDA;
  }
  if (res_words[0]) return PBIT_ERR_INVALID_LIST;
  if (phase_ms) {
    for (int i = 0; i < PBIT_NUM_PHASES; ++i) phase_ms[i] = 0.f;
    cudaEventElapsedTime(&phase_ms[PBIT_PHASE_WALK], ev[0], ev[1]);
  }
  *out_head = res_words[1];
  if (passes_run) *passes_run = res_words[2];
  if (launches_out) *launches_out = 1;
  return PBIT_OK;
}

int sort_device(const void* keys, const uint32_t* next, uint32_t head, uint64_t n, int key_bits, int K,
                int key_kind, int descending, uint32_t* out_head, uint32_t* out_next, uint32_t* out_prev,
                cudaStream_t st, float* phase_ms, uint32_t* passes_run, uint32_t* launches, HostIO* hio,
                uint32_t* out_order, void* out_keys) {
  NvtxRange nv("pbit_sort_list");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PBIT_ERR_CUDA;
  int sms = 0;
  if (int rc = device_info(dev, &sms)) return rc;
  init_rank_mode(st);
  if (n <= SMALL_N && (K == 4 || K == 8) && rank_mode() == RANK_ATOMIC && !small_path_disabled() && !hio &&
      !out_order && !out_keys) {
    const KeyMap km{key_kind, descending ? 1 : 0};
    const uint32_t n32 = (uint32_t)n;
    switch (key_bits) {
      case 8: return run_small<1>(keys, next, head, n32, K, km, out_next, out_prev, out_head, st, phase_ms, passes_run, launches);
      case 16: return run_small<2>(keys, next, head, n32, K, km, out_next, out_prev, out_head, st, phase_ms, passes_run, launches);
      case 32: return run_small<4>(keys, next, head, n32, K, km, out_next, out_prev, out_head, st, phase_ms, passes_run, launches);
      default: return run_small<8>(keys, next, head, n32, K, km, out_next, out_prev, out_head, st, phase_ms, passes_run, launches);
    }
  }
  SortPlan p;
  make_plan(n, key_bits, K, &p);
  p.key_kind = key_kind;
  p.descending = descending ? 1 : 0;
  switch (key_bits) {
    case 8: return run_device<1>(keys, next, head, p, out_next, out_prev, out_head, st, sms, phase_ms, passes_run, launches, hio,
                                 out_order, out_keys);
    case 16: return run_device<2>(keys, next, head, p, out_next, out_prev, out_head, st, sms, phase_ms, passes_run, launches, hio,
                                 out_order, out_keys);
    case 32: return run_device<4>(keys, next, head, p, out_next, out_prev, out_head, st, sms, phase_ms, passes_run, launches, hio,
                                 out_order, out_keys);
    default: return run_device<8>(keys, next, head, p, out_next, out_prev, out_head, st, sms, phase_ms, passes_run, launches, hio,
                                 out_order, out_keys);
  }
}

// ----------------------------------------------------------------------------- N3: arrays
// pbit_sort_array on device pointers: prep (key map + histograms) -> plan -> passes (the
// first generates the ids) -> the last pass writes out_index; out_keys by k_array_finish.
template <int KB>
static int run_array(const void* keys, uint32_t n, int key_bits, int K, KeyMap km, uint32_t* out_index,
                     void* out_keys, cudaStream_t st, int sms, float* phase_ms, uint32_t* passes_run,
                     uint32_t* launches_out) {
  using KeyT = typename KeyOf<KB>::T;
  const int radix = 1 << K, D = (key_bits + K - 1) / K;
  const size_t tile = sweep_tile(key_bits), ntiles = (n + tile - 1) / tile;
  const size_t kb = align_up((size_t)n * sizeof(KeyT) + 16), ib = align_up((size_t)n * 4 + 16);
  const size_t status_bytes = ntiles * (radix > 256 ? radix : 256) * 8;
  const size_t ctl_bytes = align_up((size_t)D * radix * 4) * 2 + align_up(sizeof(Plan)) + 256 + align_up(80 * 4);
  char* base = nullptr;
  if (ws_alloc((void**)&base, 2 * kb + 2 * ib + align_up(status_bytes) + ctl_bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return PBIT_ERR_OOM;
  }
  KeyT* kbuf[2] = {(KeyT*)base, (KeyT*)(base + kb)};
  uint32_t* ibuf[2] = {(uint32_t*)(base + 2 * kb), (uint32_t*)(base + 2 * kb + ib)};
  unsigned long long* status = (unsigned long long*)(base + 2 * kb + 2 * ib);
  char* ctl = base + 2 * kb + 2 * ib + align_up(status_bytes);
  uint32_t* hist = (uint32_t*)ctl;
  uint32_t* bases = (uint32_t*)(ctl + align_up((size_t)D * radix * 4));
  Plan* plan = (Plan*)(ctl + 2 * align_up((size_t)D * radix * 4));
  int* err = (int*)((char*)plan + align_up(sizeof(Plan)));
  uint32_t* tile_ctr = (uint32_t*)((char*)err + 256);

  static thread_local cudaEvent_t ev_pool[64][PBIT_NUM_PHASES + 1];
  static thread_local bool ev_ready[64] = {};
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  cudaEvent_t* ev = ev_pool[cur_dev & 63];
  const bool timing = phase_ms != nullptr;
  if (timing) {
    if (!ev_ready[cur_dev & 63]) {
      for (int i = 0; i <= PBIT_NUM_PHASES; ++i) cudaEventCreate(&ev[i]);
      ev_ready[cur_dev & 63] = true;
    }
    cudaEventRecord(ev[PBIT_NUM_PHASES], st);
  }
  uint32_t launches = 0;
  init_rank_mode(st);
  cudaMemsetAsync(ctl, 0, ctl_bytes, st);
  cudaMemsetAsync(status, 0, status_bytes, st);
  {
    const int blocks = full_wave(k_array_prep<KB>, PACK_THREADS, (size_t)D * radix * 4, sms,
                                 (n + PACK_THREADS - 1) / PACK_THREADS);
    k_array_prep<KB><<<blocks, PACK_THREADS, (size_t)D * radix * 4, st>>>(keys, n, kbuf[0], hist, K, D, km);
    k_plan<<<1, 256, 0, st>>>(hist, bases, plan, D, K, n, err);
    launches += 2;
  }
  if (timing) cudaEventRecord(ev[PBIT_PHASE_PACK], st);
  HostBox* hb = host_box();
  cudaMemcpyAsync(&hb->plan, plan, sizeof(Plan), cudaMemcpyDeviceToHost, st);
  const bool synced = cudaStreamSynchronize(st) == cudaSuccess;
  const Plan hplan = hb->plan;
  const int fblocks = full_wave(k_array_finish<KB>, 256, 0, sms, (n + 255) / 256);
  if (synced) {
    if (hplan.npasses == 0) {  // one digit value everywhere: the input order is sorted
      k_array_finish<KB><<<fblocks, 256, 0, st>>>(kbuf[0], n, out_keys, out_index, km);
      ++launches;
    } else {
      SweepArgs sa{};
      sa.kin[0] = kbuf[0]; sa.kin[1] = kbuf[1]; sa.vin[0] = ibuf[0]; sa.vin[1] = ibuf[1];
      sa.kout[0] = kbuf[0]; sa.kout[1] = kbuf[1]; sa.vout[0] = ibuf[0]; sa.vout[1] = ibuf[1];
      sa.bases = bases; sa.status = status; sa.tile_ctr = tile_ctr; sa.err = err; sa.n = n;
      launch_key_passes_k<KB>(K, sa, hplan, out_keys != nullptr, st, timing ? ev : nullptr, PBIT_PHASE_PASS0,
                              SRC_IOTA, out_index);
      launches += hplan.npasses;
      if (out_keys) {
        k_array_finish<KB><<<fblocks, 256, 0, st>>>(kbuf[hplan.npasses & 1u], n, out_keys, nullptr, km);
        ++launches;
      }
    }
  }
  if (timing) cudaEventRecord(ev[PBIT_PHASE_RELINK], st);
  cudaFreeAsync(base, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  const cudaError_t el = cudaGetLastError();
  if (!synced || es || el) {
    set_last_error("pbit_sort_array", cudaGetErrorString(es ? es : el));
    return PBIT_ERR_CUDA;
  }
  if (timing) {
    for (int i = 0; i < PBIT_NUM_PHASES; ++i) phase_ms[i] = 0.f;
    auto el_ms = [&](cudaEvent_t a, cudaEvent_t b) { float ms = 0; cudaEventElapsedTime(&ms, a, b); return ms; };
    phase_ms[PBIT_PHASE_PACK] = el_ms(ev[PBIT_NUM_PHASES], ev[PBIT_PHASE_PACK]);
    cudaEvent_t a = ev[PBIT_PHASE_PACK];
    for (uint32_t q = 0; q < hplan.npasses; ++q) {
      phase_ms[PBIT_PHASE_PASS0 + q] = el_ms(a, ev[PBIT_PHASE_PASS0 + q]);
      a = ev[PBIT_PHASE_PASS0 + q];
    }
    phase_ms[PBIT_PHASE_RELINK] = el_ms(a, ev[PBIT_PHASE_RELINK]);
  }
  if (passes_run) *passes_run = hplan.npasses;
  if (launches_out) *launches_out = launches;
  return PBIT_OK;
}

// pointer kind: 1 device (current device), 0 host (registered or pageable), -1 other device / error
int pointer_kind(const void* ptr, int dev) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) { cudaGetLastError(); return 0; }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return a.device == dev ? 1 : -1;
  return 0;
}

}  // namespace pbit

using namespace pbit;

extern "C" {

uint32_t pbit_version(void) { return (0u << 16) | (1u << 8) | 0u; }

const char* pbit_last_error(void) { return g_last_err; }

const char* pbit_status_string(int s) {
  switch (s) {
    case PBIT_OK: return "ok";
    case PBIT_ERR_INVALID_ARG: return "invalid argument";
    case PBIT_ERR_INVALID_LIST: return "invalid list";
    case PBIT_ERR_OOM: return "out of device memory";
    case PBIT_ERR_CUDA: return "CUDA error";
    case PBIT_ERR_NCCL: return "NCCL error";
    case PBIT_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

int pbit_rank_mode(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
  int sms = 0;
  if (device_info(dev, &sms) != PBIT_OK) return -1;
  init_rank_mode((cudaStream_t)0);
  return rank_mode();
}

int pbit_workspace_trim(uint64_t keep_bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) { cudaGetLastError(); return PBIT_ERR_CUDA; }
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    pool = g_dev[dev].pool;
  }
  if (!pool) return PBIT_OK;  // no call on this device yet: nothing cached
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(pool, keep_bytes) != cudaSuccess) {
    cudaGetLastError();
    return PBIT_ERR_CUDA;
  }
  return PBIT_OK;
}

int pbit_sort_list(const void* keys, const uint32_t* next, uint32_t head, uint64_t n, int key_bits,
                   uint32_t* out_head, uint32_t* out_next, const pbit_opts* opts) {
  if (!out_head) return PBIT_ERR_INVALID_ARG;
  if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return PBIT_ERR_INVALID_ARG;
  const int K = pass_bits(opts && opts->digit_bits ? opts->digit_bits : 8);
  if (!K) return PBIT_ERR_INVALID_ARG;
  if (n > 0xFFFFFFFEull) return PBIT_ERR_INVALID_ARG;
  const int key_kind = opts ? opts->key_kind : PBIT_KEY_UNSIGNED;
  const int descending = opts ? opts->descending : 0;
  if (!key_kind_ok(key_kind, key_bits)) return PBIT_ERR_INVALID_ARG;
  uint32_t* out_prev = opts ? opts->out_prev : nullptr;
  if (out_prev && out_prev == out_next) return PBIT_ERR_INVALID_ARG;
  uint32_t* out_order = opts ? opts->out_order : nullptr;
  void* out_keys = opts ? opts->out_keys : nullptr;
  cudaStream_t st = opts ? (cudaStream_t)opts->stream : (cudaStream_t)0;
  float* phase_ms = opts ? opts->phase_ms : nullptr;
  uint32_t* passes_run = opts ? opts->passes_run : nullptr;
  uint32_t* launches = opts ? opts->launches : nullptr;
  if (passes_run) *passes_run = 0;
  if (launches) *launches = 0;
  if (n == 0) {
    if (head != PBIT_NULL) return PBIT_ERR_INVALID_LIST;
    *out_head = PBIT_NULL;
    return PBIT_OK;
  }
  if (!keys || !next || !out_next) return PBIT_ERR_INVALID_ARG;
  if ((uint64_t)head >= n) return PBIT_ERR_INVALID_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_CUDA; }
  const int kk = pointer_kind(keys, dev), kn = pointer_kind(next, dev), ko = pointer_kind(out_next, dev);
  const int kp = out_prev ? pointer_kind(out_prev, dev) : ko;
  const int kr = out_order ? pointer_kind(out_order, dev) : ko;
  const int ky = out_keys ? pointer_kind(out_keys, dev) : ko;
  if (kk < 0 || kn < 0 || ko < 0 || kp < 0 || kr < 0 || ky < 0) return PBIT_ERR_INVALID_ARG;
  if (kk == 1 && kn == 1 && ko == 1 && kp == 1 && kr == 1 && ky == 1)
    return sort_device(keys, next, head, n, key_bits, K, key_kind, descending, out_head, out_next, out_prev, st,
                       phase_ms, passes_run, launches, nullptr, out_order, out_keys);
  if (kk != 0 || kn != 0 || ko != 0 || kp != 0 || kr != 0 || ky != 0) return PBIT_ERR_INVALID_ARG;  // mixed

  // host buffers: stage through device memory inside the call
  const size_t kbytes = n * (size_t)(key_bits / 8), nbytes = n * 4;
  char* d = nullptr;
  const size_t a = align_up(kbytes), b = align_up(nbytes);
  if (ws_alloc((void**)&d, 2 * a + 4 * b, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  uint32_t* d_prev = out_prev ? (uint32_t*)(d + a + 2 * b) : nullptr;
  uint32_t* d_order = out_order ? (uint32_t*)(d + a + 3 * b) : nullptr;
  void* d_keys = out_keys ? (void*)(d + a + 4 * b) : nullptr;
  int rc = PBIT_OK;
  const bool small = n <= SMALL_N;  // the single-cluster path: plain copies around one launch
  HostIO hio{keys, next, out_next, out_prev, nullptr, nullptr};
  if (!small) {
    int sms = 0;
    if (device_info(dev, &sms)) rc = PBIT_ERR_CUDA;
    hostio_resources(&hio.copy, &hio.ev);
  } else if (cudaMemcpyAsync(d, keys, kbytes, cudaMemcpyHostToDevice, st) ||
             cudaMemcpyAsync(d + a, next, nbytes, cudaMemcpyHostToDevice, st)) {
    rc = PBIT_ERR_CUDA;
  }
  if (!rc) rc = sort_device(d, (const uint32_t*)(d + a), head, n, key_bits, K, key_kind, descending, out_head,
                            (uint32_t*)(d + a + b), d_prev, st, phase_ms, passes_run, launches, small ? nullptr : &hio,
                            d_order, d_keys);
  if (!rc && !hio.results_copied) {
    if (cudaMemcpyAsync(out_next, d + a + b, nbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
    if (!rc && out_prev && cudaMemcpyAsync(out_prev, d_prev, nbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
  }
  // the sorted records (a valid list only: rc is PBIT_OK here)
  if (!rc && out_order && cudaMemcpyAsync(out_order, d_order, nbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
  if (!rc && out_keys && cudaMemcpyAsync(out_keys, d_keys, kbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
  cudaFreeAsync(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !rc) rc = PBIT_ERR_CUDA;
  cudaGetLastError();
  return rc;
}

int pbit_sort_array(const void* keys, uint64_t n, int key_bits, uint32_t* out_index, void* out_keys,
                    const pbit_opts* opts) {
  if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return PBIT_ERR_INVALID_ARG;
  const int K = pass_bits(opts && opts->digit_bits ? opts->digit_bits : 8);
  if (!K) return PBIT_ERR_INVALID_ARG;
  if (n > 0xFFFFFFFEull) return PBIT_ERR_INVALID_ARG;
  const KeyMap km{opts ? opts->key_kind : PBIT_KEY_UNSIGNED, opts && opts->descending ? 1 : 0};
  if (!key_kind_ok(km.kind, key_bits)) return PBIT_ERR_INVALID_ARG;
  if (!out_index && !out_keys) return PBIT_ERR_INVALID_ARG;
  cudaStream_t st = opts ? (cudaStream_t)opts->stream : (cudaStream_t)0;
  float* phase_ms = opts ? opts->phase_ms : nullptr;
  uint32_t* passes_run = opts ? opts->passes_run : nullptr;
  uint32_t* launches = opts ? opts->launches : nullptr;
  if (passes_run) *passes_run = 0;
  if (launches) *launches = 0;
  if (n == 0) return PBIT_OK;
  if (!keys) return PBIT_ERR_INVALID_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_CUDA; }
  int sms = 0;
  if (int rc = device_info(dev, &sms)) return rc;
  const int kk = pointer_kind(keys, dev);
  const int ki = out_index ? pointer_kind(out_index, dev) : kk;
  const int ko = out_keys ? pointer_kind(out_keys, dev) : kk;
  if (kk < 0 || ki < 0 || ko < 0 || kk != ki || kk != ko) return PBIT_ERR_INVALID_ARG;
  const uint32_t n32 = (uint32_t)n;
  auto run = [&](const void* k, uint32_t* oi, void* ok) {
    switch (key_bits) {
      case 8: return run_array<1>(k, n32, 8, K, km, oi, ok, st, sms, phase_ms, passes_run, launches);
      case 16: return run_array<2>(k, n32, 16, K, km, oi, ok, st, sms, phase_ms, passes_run, launches);
      case 32: return run_array<4>(k, n32, 32, K, km, oi, ok, st, sms, phase_ms, passes_run, launches);
      default: return run_array<8>(k, n32, 64, K, km, oi, ok, st, sms, phase_ms, passes_run, launches);
    }
  };
  if (kk == 1) return run(keys, out_index, out_keys);
  // host buffers: stage through device memory inside the call
  const size_t kbytes = n * (size_t)(key_bits / 8), nbytes = n * 4;
  char* d = nullptr;
  const size_t a = align_up(kbytes), b = align_up(nbytes);
  if (ws_alloc((void**)&d, 2 * a + b, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  int rc = cudaMemcpyAsync(d, keys, kbytes, cudaMemcpyHostToDevice, st) ? PBIT_ERR_CUDA : PBIT_OK;
  if (!rc) rc = run(d, out_index ? (uint32_t*)(d + 2 * a) : nullptr, out_keys ? d + a : nullptr);
  if (!rc && out_index && cudaMemcpyAsync(out_index, d + 2 * a, nbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
  if (!rc && out_keys && cudaMemcpyAsync(out_keys, d + a, kbytes, cudaMemcpyDeviceToHost, st)) rc = PBIT_ERR_CUDA;
  cudaFreeAsync(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !rc) rc = PBIT_ERR_CUDA;
  cudaGetLastError();
  return rc;
}

}  // extern "C"
