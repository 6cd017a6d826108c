// mg.cu -- pbit_sort_list_mg: one list sorted by G ranks (one process per GPU) over an
// NCCL communicator, plus the NCCL communicator helpers.
//
// Rank r owns node ids [r*S, r*S + n_local), S = 64 * ceil(ceil(n/G) / 64), and after the
// key-range exchange holds sorted positions [r*S, r*S + S) of the output.
// Two transports move the data between the ranks:
//
//   PEER (NEXT row N4, the default where every rank can map every other rank's memory --
//   NVLink / NVSwitch peers, CUDA IPC): no replica.  Each rank packs its slice into a
//   window of device memory that every rank maps; the walk reads kn[v] from v's owner
//   with peer loads; the list-order chunk is gathered from the walkers' segment slots;
//   the key-range partition pass stores every element straight into its destination
//   rank's receive arrays (the scatter fused with the all-to-all); the relink records are
//   stored straight into their owner's receive buffer.  NCCL carries only small
//   collectives (histograms, segment tables, counts) that also order the phases.
//   NCCL (the bit-identity reference): a kn replica by ncclAllGather, a count walk and an
//   emit walk over it, and ncclSend/ncclRecv for both exchanges.
//
// Steps (both transports):
//   0  the ranks agree on their arguments (one all-reduce; pbit.h)
//   1  pack the own slice (+ every digit's histogram)           ncclAllReduce(histograms)
//   2  ruling-set walk of the own rulers                         ncclAllGather(segment table)
//   3  rank the ruler list (every rank, redundantly; validates the list)
//   4  the list-order chunk of positions [r*S, r*S + S)
//   5  exact splitters of the global (key, list position) order, 8 bits per round on the
//      device (ncclAllReduce of candidate histograms); bucket counts and the exchange plan
//      on the device (ncclAllGather)
//   6  one stable partition pass by splitter bucket -> the destination ranks
//   7  stable local sort of the received runs (source-rank order = list-position order for
//      equal keys, so the stable passes restore the global stable order)
//   8  stitch (ncclAllGather of first / last ids) and route (v, succ[, pred]) to the owner
//      of v; the owner applies them with the single-GPU binned relink.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/pbit.h"
#include "launch.cuh"
#include "mg_kernels.cuh"
#include "pbit_internal.h"

static_assert(sizeof(ncclUniqueId) == PBIT_MG_UNIQUE_ID_BYTES, "NCCL unique id size");

// The ruling set of the multi-GPU walk: the single-GPU spacing for n nodes (make_plan), at
// most 64 so that every rank's id slice (pbit_mg_slice: a multiple of 64) is a whole number
// of ruler blocks (make_plan picks 128 from 2^30 nodes).  Exported for tests.
extern "C" int pbit_mg_ruler_blocks(uint64_t n, int nranks, uint32_t* spacing, uint32_t* blocks_per_rank) {
  if (!spacing || !blocks_per_rank || nranks < 1 || n > 0xFFFFFFFEull) return PBIT_ERR_INVALID_ARG;
  pbit::SortPlan p;
  pbit::make_plan(n, 32, 8, &p);
  const int s_log2 = p.s_log2 > 6 ? 6 : p.s_log2;
  const uint64_t S = pbit_mg_slice(n, nranks), s = 1ull << s_log2;
  if (S % s || (uint64_t)nranks * (S / s) * s < n || (uint64_t)nranks * S > 0xFFFFFFFFull) return PBIT_ERR_UNSUPPORTED;
  *spacing = (uint32_t)s;
  *blocks_per_rank = (uint32_t)(S / s);
  return PBIT_OK;
}

namespace pbit {

namespace {

struct Bump {
  char* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (count * sizeof(T) + 16 + 255) & ~(size_t)255;  // +16 B: tile loads may read past the end
    return p;
  }
};

#define NCCLCHK(x)                                          \
  do {                                                      \
    ncclResult_t r_ = (x);                                  \
    if (r_ != ncclSuccess) {                                \
      set_last_error(#x, ncclGetErrorString(r_));           \
      rc = PBIT_ERR_NCCL;                                   \
      goto done;                                            \
    }                                                       \
  } while (0)

#define CUDACHK(x)                                          \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) {                                \
      set_last_error(#x, cudaGetErrorString(e_));           \
      rc = PBIT_ERR_CUDA;                                   \
      goto done;                                            \
    }                                                       \
  } while (0)

// Failure detection: wait for the stream while polling the communicator's
// asynchronous error, with a timeout (PBIT_MG_TIMEOUT_S, default 300 s), instead of a
// blocking synchronize that would hang forever if a peer died.  On an NCCL error or the
// timeout the call returns PBIT_ERR_NCCL; the caller then aborts the communicator
// (pbit_mg_comm_abort), which also releases the stream.
static int mg_wait(cudaStream_t st, ncclComm_t comm) {
  static const double timeout_s = [] { const char* e = getenv("PBIT_MG_TIMEOUT_S"); return e ? atof(e) : 300.0; }();
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return PBIT_OK;
    if (q != cudaErrorNotReady) {
      set_last_error("pbit_sort_list_mg", cudaGetErrorString(q));
      return PBIT_ERR_CUDA;
    }
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(comm, &ar) != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
      set_last_error("pbit_sort_list_mg: NCCL asynchronous error", ncclGetErrorString(ar));
      return PBIT_ERR_NCCL;
    }
    if ((spin & 255u) == 255u &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      set_last_error("pbit_sort_list_mg", "timed out waiting for the collectives (PBIT_MG_TIMEOUT_S)");
      return PBIT_ERR_NCCL;
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

#define MGWAIT()                     \
  do {                               \
    const int rc_ = mg_wait(st, comm); \
    if (rc_) {                       \
      rc = rc_;                      \
      goto done;                     \
    }                                \
  } while (0)

// An ncclGroupStart ... ncclGroupEnd bracket whose end runs on every exit path (an error
// inside the group still closes it).
struct NcclGroup {
  bool open = false;
  ncclResult_t start() { const ncclResult_t r = ncclGroupStart(); open = r == ncclSuccess; return r; }
  ncclResult_t end() { open = false; return ncclGroupEnd(); }
  ~NcclGroup() { if (open) ncclGroupEnd(); }
};

// Small host-visible results land in pinned memory (a pageable destination would make
// each cudaMemcpyAsync wait for the stream): one box per host thread, one call at a time.
struct MgBox {
  Plan plan;
  int err;
  uint32_t res[4];
};
MgBox* mg_box() {
  struct Holder {
    MgBox* pinned = nullptr;
    MgBox pageable{};
    bool tried = false;
    ~Holder() { if (pinned) cudaFreeHost(pinned); }
  };
  static thread_local Holder h;
  if (!h.tried) {
    h.tried = true;
    if (cudaHostAlloc((void**)&h.pinned, sizeof(MgBox), cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      h.pinned = nullptr;
    }
  }
  return h.pinned ? h.pinned : &h.pageable;
}

// ----------------------------------------------------------------------------- peer window (N4)
// One window of device memory per communicator and rank (cudaMalloc, so it can be shared by
// CUDA IPC), mapped by every rank: peers read its kn slice and segment slots and write its
// receive arrays.  Cached between calls, re-created (collectively) when a call needs more;
// released by pbit_mg_comm_destroy / _abort.  Ranks in the same process (the multi-rank
// test harness) use each other's pointers directly.
struct PeerWin {
  int G = 0;
  char* local = nullptr;
  size_t bytes = 0;
  char* peer[64] = {};
  bool mapped[64] = {};
};
std::mutex g_win_mu;
std::map<void*, PeerWin> g_wins;
std::map<void*, int> g_last_transport;  // the transport of each communicator's last call

void win_release(PeerWin& w) {
  for (int q = 0; q < 64; ++q) {
    if (w.mapped[q] && w.peer[q]) cudaIpcCloseMemHandle(w.peer[q]);
    w.peer[q] = nullptr;
    w.mapped[q] = false;
  }
  if (w.local) cudaFree(w.local);
  cudaGetLastError();
  w.local = nullptr;
  w.bytes = 0;
  w.G = 0;
}

struct IpcRec {
  cudaIpcMemHandle_t h;
  uint64_t ptr, pid, host;
  int32_t ok, pad;
};

uint64_t host_key() {
  char name[256] = {};
  gethostname(name, sizeof name - 1);
  uint64_t h = 1469598103934665603ull;
  for (const char* c = name; *c; ++c) h = (h ^ (uint8_t)*c) * 1099511628211ull;
  return h;
}

// Every rank returns the same verdict: PBIT_OK with the window mapped everywhere, or
// PBIT_ERR_UNSUPPORTED (some rank could not allocate, export or map) -- the caller then
// takes the NCCL transport.
int peer_window(ncclComm_t comm, int G, int r, size_t need, cudaStream_t st, PeerWin** out) {
  PeerWin* wp;
  {  // the map lock covers the lookup only: the collectives below must not hold it (ranks
     // of one process -- the test harness -- would wait for each other in them)
    std::lock_guard<std::mutex> lk(g_win_mu);
    wp = &g_wins[(void*)comm];  // std::map references stay valid; one thread per communicator
  }
  PeerWin& w = *wp;
  *out = &w;
  if (w.local && w.G == G && w.bytes >= need) return PBIT_OK;  // the same on every rank (same calls)
  win_release(w);
  int ok = 1;
  IpcRec me{};
  if (cudaMalloc((void**)&w.local, need) != cudaSuccess) { cudaGetLastError(); w.local = nullptr; ok = 0; }
  if (ok && cudaIpcGetMemHandle(&me.h, w.local) != cudaSuccess) { cudaGetLastError(); ok = 0; }
  me.ptr = (uint64_t)(uintptr_t)w.local;
  me.pid = (uint64_t)getpid();
  me.host = host_key();
  me.ok = ok;
  std::vector<IpcRec> all(G);
  char* d = nullptr;
  int rc = PBIT_OK;
  if (ws_alloc((void**)&d, sizeof(IpcRec) * (G + 1) + 64, st) != cudaSuccess) {
    cudaGetLastError();
    win_release(w);
    return PBIT_ERR_OOM;
  }
  int* d_ok = (int*)(d + sizeof(IpcRec) * (G + 1));
  int* h_ok = &mg_box()->err;
  if (cudaMemcpyAsync(d + sizeof(IpcRec) * G, &me, sizeof me, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      ncclAllGather(d + sizeof(IpcRec) * G, d, sizeof(IpcRec), ncclUint8, comm, st) != ncclSuccess ||
      cudaMemcpyAsync(all.data(), d, sizeof(IpcRec) * G, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = PBIT_ERR_NCCL;
  if (!rc) rc = mg_wait(st, comm);
  if (!rc) {
    for (int q = 0; q < G && ok; ++q) {
      if (q == r) { w.peer[q] = w.local; continue; }
      if (!all[q].ok) { ok = 0; break; }
      if (all[q].pid == me.pid && all[q].host == me.host) {  // same process: the pointer is valid here
        w.peer[q] = (char*)(uintptr_t)all[q].ptr;
      } else if (cudaIpcOpenMemHandle((void**)&w.peer[q], all[q].h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
        w.mapped[q] = true;
      } else {
        cudaGetLastError();
        w.peer[q] = nullptr;
        ok = 0;
      }
    }
    // every rank must have mapped every window: agree (min) before anyone relies on it
    *h_ok = 0;
    if (cudaMemcpyAsync(d_ok, &ok, sizeof ok, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        ncclAllReduce(d_ok, d_ok + 1, 1, ncclInt32, ncclMin, comm, st) != ncclSuccess ||
        cudaMemcpyAsync(h_ok, d_ok + 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = PBIT_ERR_NCCL;
    if (!rc) rc = mg_wait(st, comm);
  }
  cudaFreeAsync(d, st);
  if (rc) { win_release(w); return rc; }
  if (!*h_ok) { win_release(w); return PBIT_ERR_UNSUPPORTED; }
  w.G = G;
  w.bytes = need;
  return PBIT_OK;
}

enum Transport { T_PEER = 0, T_NCCL = 1, T_HYBRID = 2 };

// PBIT_MG_TRANSPORT=peer|hybrid|nccl (default: peer where the ranks can map each other).
// hybrid = the peer transport with a kn replica (ncclAllGather) walked locally instead of
// remote node reads -- for fabrics where small random peer reads are slow.
int transport_request() {
  const char* e = getenv("PBIT_MG_TRANSPORT");  // read per call (tests switch it)
  if (e && !strcmp(e, "nccl")) return T_NCCL;
  if (e && !strcmp(e, "hybrid")) return T_HYBRID;
  return T_PEER;
}

// pbit_sort_list_mg's own status for "the per-rank dynamic ruler table overflowed" (a list
// whose rulers leave some rank far more nodes to walk than it owns): the call is redone
// with the NCCL transport, whose walk does not cut segments.
constexpr int RC_DYN_OVERFLOW = 100;

template <int KB>
int run_mg(const void* keys_local, const uint32_t* next_local, uint32_t head, uint32_t n, uint32_t S,
           uint32_t n_local, int K, KeyMap km, uint32_t* out_head, uint32_t* out_next_local,
           uint32_t* out_prev_local, bool with_prev, ncclComm_t comm, int G, int r, cudaStream_t st,
           int transport, uint32_t* launches_out, uint32_t* out_order_local = nullptr, void* out_keys_local = nullptr) {
  using RT = typename Rec<KB>::T;
  using KeyT = typename KeyOf<KB>::T;
  constexpr int REC_WORDS = sizeof(RT) / 4;
  const ncclDataType_t key_t = KB == 8 ? ncclUint64 : ncclUint32;
  const bool peer = transport != T_NCCL;       // windows, slot walk, peer stores
  const bool replica = transport != T_PEER;    // a kn replica by ncclAllGather (NCCL, hybrid)
  uint32_t launches = 0;
  int rc = PBIT_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (int e = device_info(dev, &sms)) return e;
  init_rank_mode(st);

  SortPlan p;
  make_plan(n, KB * 8, K, &p);
  uint32_t s = 0, bpr = 0;
  if (pbit_mg_ruler_blocks(n, G, &s, &bpr) != PBIT_OK) {
    set_last_error("pbit_sort_list_mg", "ruler blocks do not tile the rank slices");
    return PBIT_ERR_UNSUPPORTED;
  }
  p.s_log2 = __builtin_ctz(s);
  p.R = (uint32_t)(((uint64_t)n + s - 1) >> p.s_log2);
  p.cap = 4u << p.s_log2;
  const int radix = 1 << K;
  const uint32_t Gs = (uint32_t)G * bpr;           // static rulers (+1: the head's extra ruler)
  const uint32_t cap = p.cap;
  const uint32_t dcap = peer ? S / cap + 1 : 0u;   // dynamic rulers per rank (cut segments)
  const uint32_t Rmax = Gs + 1 + (uint32_t)G * dcap;
  RulerSel sel{n, (uint32_t)p.s_log2, p.R};
  const bool head_is_ruler = sel.is_ruler(head);
  const uint32_t head_ruler = head_is_ruler ? (head >> p.s_log2) : Gs;
  const uint32_t head_owner = head / S;
  const bool own_head = head_owner == (uint32_t)r;
  const uint32_t P0 = std::min<uint64_t>(n, (uint64_t)r * S), P1 = std::min<uint64_t>(n, (uint64_t)(r + 1) * S);
  const uint32_t m = P1 - P0;                      // sorted positions held by this rank
  const uint32_t lo = r * S;
  RulerSel sub{Rmax, 4u, (Rmax + 15) >> 4};
  const bool hs = sub.is_ruler(head_ruler);
  const uint32_t nsub = sub.R + (hs ? 0u : 1u);
  const uint32_t head_sub = hs ? (head_ruler >> 4) : sub.R;
  const size_t tile = sweep_tile(KB * 8);
  const size_t ntiles = (S + tile - 1) / tile;
  const int D = p.D;
  const uint32_t NS = (uint32_t)G - 1;             // splitters
  const uint32_t NB = 2 * NS + 1;                  // splitter buckets
  const int W = with_prev ? 3 : 2;                 // relink record words
  const uint32_t n_static = p.R > r * bpr ? std::min(bpr, p.R - r * bpr) : 0u;
  // one rank with the peer transport: its slots ARE the list (slot(r) = r, as on a single
  // GPU), so the first local pass gathers its tiles from them and the relink reads the
  // sorted ids directly -- nothing is exchanged
  const bool solo = peer && G == 1;
  const uint32_t nslots = bpr + 1 + dcap;

  // ---- the window (peer transport): [kn slice][segment slots][recv keys][recv ids]; the
  // relink records a rank receives land in its slot area (dead by then)
  const size_t a_kn = ((size_t)S * sizeof(RT) + 255) & ~(size_t)255;
  const size_t a_slots = std::max(((size_t)nslots * cap * sizeof(RT) + 255) & ~(size_t)255,
                                  ((size_t)S * 12 + 16 + 255) & ~(size_t)255);
  const size_t a_rk = ((size_t)S * sizeof(KeyT) + 16 + 255) & ~(size_t)255;
  const size_t a_ri = ((size_t)S * 4 + 16 + 255) & ~(size_t)255;
  PeerWin* win = nullptr;
  if (peer) {
    if (int e = peer_window(comm, G, r, a_kn + a_slots + a_rk + a_ri, st, &win)) return e;
  }
  auto wk = [&](int q, size_t off) -> char* { return win->peer[q] + off; };

  // ---- workspace (the library's pool)
  Bump b;
  RT* kn_rep = nullptr; uint2* seg = nullptr; uint32_t *dist = nullptr, *seg_ord = nullptr, *seg_pos = nullptr;
  unsigned long long* sdist[2] = {}; uint32_t* scnt[2] = {}; uint32_t* ssucc[2] = {};
  KeyT *keys_c = nullptr, *kb1 = nullptr, *recv_k = nullptr, *send_k = nullptr;
  uint32_t *ids_c = nullptr, *ib1 = nullptr, *recv_i = nullptr, *send_i = nullptr;
  unsigned long long* status = nullptr;
  void *rbuf0 = nullptr, *rbuf1 = nullptr, *psend = nullptr, *precvb = nullptr;
  RT* slots_own = nullptr;
  // control block (zeroed per call)
  uint32_t *hist_l = nullptr, *hist_g = nullptr, *bases_g = nullptr, *hist_r = nullptr, *bases_r = nullptr,
           *part_first = nullptr, *tile_ctr = nullptr, *nseg = nullptr, *zero = nullptr, *dyn_count = nullptr,
           *shist = nullptr, *bcnt = nullptr, *cntall_b = nullptr, *sbases = nullptr, *srecv = nullptr,
           *fl = nullptr, *fl_all = nullptr, *edges = nullptr, *pcnt = nullptr, *pcntall = nullptr,
           *pbase = nullptr, *psbase = nullptr, *precv = nullptr, *pfill = nullptr, *cursors = nullptr,
           *barrier_w = nullptr;
  unsigned long long* below = nullptr;
  Plan *plan_g = nullptr, *plan_r = nullptr;
  SplitTable* split = nullptr;
  int* err = nullptr;
  size_t ctl_off = 0, ctl_end = 0;
  auto carve = [&]() {
    if (replica) kn_rep = b.take<RT>((size_t)G * S);
    seg = b.take<uint2>(Rmax);
    dist = b.take<uint32_t>(Rmax);
    seg_ord = b.take<uint32_t>(Rmax);
    seg_pos = b.take<uint32_t>(Rmax);
    for (int i = 0; i < 2; ++i) {
      sdist[i] = b.take<unsigned long long>(nsub + 1);
      scnt[i] = b.take<uint32_t>(nsub + 1);
      ssucc[i] = b.take<uint32_t>(nsub + 1);
    }
    keys_c = b.take<KeyT>(S);
    ids_c = b.take<uint32_t>(S);
    kb1 = b.take<KeyT>(S);
    ib1 = b.take<uint32_t>(S);
    if (!peer) {
      recv_k = b.take<KeyT>(S);
      recv_i = b.take<uint32_t>(S);
      send_k = b.take<KeyT>(S);
      send_i = b.take<uint32_t>(S);
      psend = b.take<uint32_t>((size_t)S * W);
      precvb = b.take<uint32_t>((size_t)S * W);
    }
    status = b.take<unsigned long long>(ntiles * 256);
    rbuf0 = b.take<uint32_t>((size_t)S * W);
    rbuf1 = b.take<uint32_t>((size_t)S * W);
    ctl_off = b.off;
    hist_l = b.take<uint32_t>((size_t)D * radix);
    hist_g = b.take<uint32_t>((size_t)D * radix);
    bases_g = b.take<uint32_t>((size_t)D * radix);
    hist_r = b.take<uint32_t>((size_t)D * radix);
    bases_r = b.take<uint32_t>((size_t)D * radix);
    part_first = b.take<uint32_t>(solo ? ntiles + 2 : (size_t)G + 2);  // solo: per pass tile
    tile_ctr = b.take<uint32_t>(80);
    nseg = b.take<uint32_t>(1);
    zero = b.take<uint32_t>(1);
    dyn_count = b.take<uint32_t>(1);
    shist = b.take<uint32_t>(64 * 256);
    below = b.take<unsigned long long>(64);
    bcnt = b.take<uint32_t>(128);
    cntall_b = b.take<uint32_t>((size_t)G * 128);
    sbases = b.take<uint32_t>(128);
    srecv = b.take<uint32_t>(2 * 64);
    fl = b.take<uint32_t>(2);
    fl_all = b.take<uint32_t>(2 * 64);
    edges = b.take<uint32_t>(4);
    pcnt = b.take<uint32_t>(64);
    pcntall = b.take<uint32_t>(64 * 64);
    pbase = b.take<uint32_t>(64);
    psbase = b.take<uint32_t>(64);
    precv = b.take<uint32_t>(2 * 64);
    pfill = b.take<uint32_t>(64);
    cursors = b.take<uint32_t>(relink_cursor_words(S));
    barrier_w = b.take<uint32_t>(2);
    plan_g = b.take<Plan>(1);
    plan_r = b.take<Plan>(1);
    split = b.take<SplitTable>(1);
    err = b.take<int>(1);
    ctl_end = b.off;
  };
  carve();
  const size_t bytes = b.off;
  char* base = nullptr;
  if (ws_alloc((void**)&base, bytes, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  b = Bump{base, 0};
  carve();
  if (peer) {
    slots_own = (RT*)(win->local + a_kn);
    recv_k = (KeyT*)(win->local + a_kn + a_slots);
    recv_i = (uint32_t*)(win->local + a_kn + a_slots + a_rk);
  }

  // host-side state (declared before the first goto)
  // NVTX ranges (SURVEY §5 tracing): the call, and each protocol step inside it; the stack
  // is unwound at `done` whatever step a failure left
  int nvtx_depth = 1;
  nvtxRangePushA("pbit_sort_list_mg");
  auto nvtx_step = [&](const char* name) {
    if (nvtx_depth > 1) { nvtxRangePop(); --nvtx_depth; }
    nvtxRangePushA(name);
    ++nvtx_depth;
  };
  MgBox* hb = mg_box();
  const Plan& h_plan = hb->plan;
  uint32_t h_left[66] = {}, h_srecv[128] = {}, h_prow[64] = {}, h_psbase[64] = {}, h_precv[128] = {};
  std::vector<uint32_t> h_pall((size_t)G * G);
  SplitTable h_split{};
  cudaEvent_t plan_ev = nullptr;
  const KeyT* rk = nullptr;
  const uint32_t* ri = nullptr;
  const uint32_t* fin = nullptr;
  const KeyT* fin_k = nullptr;
  {
    CUDACHK(cudaMemsetAsync(base + ctl_off, 0, ctl_end - ctl_off, st));
    CUDACHK(cudaMemsetAsync(seg, 0, sizeof(uint2) * Rmax, st));
    CUDACHK(cudaMemsetAsync(status, 0, ntiles * 256 * 8, st));

    // ---- 1. pack the own slice; histograms of every digit of every key
    nvtx_step("pbit.mg.pack");
    {
      RT* kn_own = replica ? kn_rep + lo : (RT*)win->local;
      if (n_local) {
        const int blocks = full_wave(k_pack<KB>, PACK_THREADS, (size_t)D * radix * 4, sms,
                                     (n_local + PACK_THREADS - 1) / PACK_THREADS);
        ++launches;
        k_pack<KB><<<blocks, PACK_THREADS, (size_t)D * radix * 4, st>>>(keys_local, next_local, n_local, n, kn_own,
                                                                         hist_l, K, D, err, km);
      }
      if (replica) NCCLCHK(ncclAllGather(kn_rep + lo, kn_rep, (size_t)S * REC_WORDS, ncclUint32, comm, st));
      NCCLCHK(ncclAllReduce(hist_l, hist_g, (size_t)D * radix, ncclUint32, ncclSum, comm, st));
      // the global pass plan (a digit trivial globally is trivial on every rank): read by
      // the host while the walk, the ranking and the exchange run
      ++launches;
      k_plan<<<1, 256, 0, st>>>(hist_g, bases_g, plan_g, D, K, n, err);
      CUDACHK(cudaMemcpyAsync(&hb->plan, plan_g, sizeof(Plan), cudaMemcpyDeviceToHost, st));
      CUDACHK(cudaEventCreateWithFlags(&plan_ev, cudaEventDisableTiming));
      CUDACHK(cudaEventRecord(plan_ev, st));
    }

    // ---- 2. walk the own rulers; share the segment table
    nvtx_step("pbit.mg.walk");
    if (peer) {
      KnSrc<RT> src{};
      for (int q = 0; q < G; ++q) src.peer[q] = (const RT*)wk(q, 0);
      src.S = FastDiv::make(S);
      src.kn = kn_rep;  // hybrid: the replica, read locally
      const WalkMap wm{r * bpr, n_static, own_head && !head_is_ruler ? Gs : PBIT_NULL32, bpr,
                       Gs + 1 + (uint32_t)r * dcap, bpr + 1};
      const uint32_t total = wm.count();
      if (total) {
        static const int occ = [] {
          int o = 0;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_walk<KB, true>, WALK_THREADS, 0);
          return std::max(o, 1);
        }();
        int blocks = sms * occ;
        if ((uint32_t)blocks * 4 > total) blocks = std::max(1u, (total + 3) / 4);
        const uint32_t per = (total + blocks - 1) / blocks;
        ++launches;
        if (replica)
          k_walk<KB, false><<<blocks, WALK_THREADS, 0, st>>>(src, sel, wm, head, slots_own, cap, seg, dyn_count, dcap,
                                                             per, err, 0);
        else
          k_walk<KB, true><<<blocks, WALK_THREADS, 0, st>>>(src, sel, wm, head, slots_own, cap, seg, dyn_count, dcap,
                                                            per, err, 0);
      }
    } else {
      const uint32_t b_lo = r * bpr, b_hi = (r + 1) * bpr;
      const uint32_t total = bpr + (own_head && !head_is_ruler ? 1u : 0u);
      int blocks = sms * (2048 / WALK_THREADS);
      if ((uint32_t)blocks * 4 > total) blocks = std::max(1u, (total + 3) / 4);
      const uint32_t per = (total + blocks - 1) / blocks;
      ++launches;
      k_walk_count<KB><<<blocks, WALK_THREADS, 0, st>>>(kn_rep, sel, b_lo, b_hi,
                                                        own_head && !head_is_ruler ? Gs : PBIT_NULL32, head, seg, per,
                                                        err);
    }
    NCCLCHK(ncclAllGather(seg + (size_t)r * bpr, seg, (size_t)bpr * 2, ncclUint32, comm, st));
    if (dcap) NCCLCHK(ncclAllGather(seg + Gs + 1 + (size_t)r * dcap, seg + Gs + 1, (size_t)dcap * 2, ncclUint32, comm, st));
    NCCLCHK(ncclAllReduce(seg + Gs, seg + Gs, 2, ncclUint32, ncclMax, comm, st));
    NCCLCHK(ncclAllReduce(err, err, 1, ncclInt32, ncclMax, comm, st));

    // ---- 3. rank the ruler list (identical on every rank)
    nvtx_step("pbit.mg.rank");
    {
      const int sblocks = full_wave(k_rank_walk_a, 256, 0, sms, (nsub + 255) / 256);
      ++launches;
      k_rank_walk_a<<<sblocks, 256, 0, st>>>(seg, sub, Rmax, zero, 0, head_ruler, nsub, sdist[0], scnt[0], ssucc[0],
                                             err);
      int rounds = 1;
      while ((1ull << rounds) < nsub) ++rounds;
      rounds += 1;
      int cur = 0;
      for (int i = 0; i < rounds; ++i) {
        ++launches;
        k_rank_jump<<<sblocks, 256, 0, st>>>(sdist[cur], scnt[cur], ssucc[cur], sdist[cur ^ 1], scnt[cur ^ 1],
                                             ssucc[cur ^ 1], nsub, err);
        cur ^= 1;
      }
      ++launches;
      k_rank_check<<<1, 1, 0, st>>>(sdist[cur], ssucc[cur], head_sub, n, err);
      ++launches;
      k_rank_walk_b<<<sblocks, 256, 0, st>>>(seg, sub, Rmax, zero, 0, head_ruler, nsub, head_sub, sdist[cur],
                                             scnt[cur], dist, seg_ord, seg_pos, part_first,
                                             solo ? (uint32_t)tile : S, n, nseg, err);
    }

    // ---- 4. the list-order chunk of positions [P0, P1)
    nvtx_step("pbit.mg.chunk");
    if (cudaEventSynchronize(plan_ev) != cudaSuccess) { rc = PBIT_ERR_CUDA; goto done; }
    if (m && (!solo || h_plan.npasses == 0)) {
      const int blocks = std::max(1, std::min((int)((m / 64 + 2 + 255) / 256), sms * 8));
      ++launches;
      if (peer) {
        PeerSlots ps{};
        for (int q = 0; q < G; ++q) ps.slots[q] = wk(q, a_kn);
        MgRulers mr{FastDiv::make(bpr), FastDiv::make(std::max(dcap, 1u)), Gs, head_owner, cap};
        k_mg_gather<KB><<<blocks, 256, 0, st>>>(ps, mr, cap, seg, seg_ord, seg_pos, part_first, r, nseg, P0, P1,
                                                keys_c, ids_c, err);
      } else {
        k_emit_walk<KB><<<blocks, 256, 0, st>>>(kn_rep, sel, head, seg, seg_ord, seg_pos, part_first, r, nseg, P0, P1,
                                                keys_c, ids_c, err);
      }
    }

    if (G > 1) {
      // ---- 5. splitters, bucket counts, exchange plan -- all on the device
      nvtx_step("pbit.mg.splitters");
      h_split.G = (uint32_t)G;
      h_split.NS = NS;
      for (int d = 0; d < G; ++d) {
        h_split.dst_k[d] = peer ? (void*)wk(d, a_kn + a_slots) : (void*)send_k;
        h_split.dst_i[d] = peer ? (uint32_t*)wk(d, a_kn + a_slots + a_rk) : send_i;
      }
      CUDACHK(cudaMemcpyAsync(split, &h_split, sizeof h_split, cudaMemcpyHostToDevice, st));
      const int rounds = KB;  // 8 bits per round
      const int cblocks = std::max(1, std::min((int)((m + 255) / 256), sms * 2));
      static std::atomic<unsigned long long> attr{0};
      once_per_device(attr, [] {
        cudaFuncSetAttribute(k_split_count<KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 256 * 4);
      });
      for (int i = rounds - 1; i >= 0; --i) {
        if (m) {
          ++launches;
          k_split_count<KeyT><<<cblocks, 256, NS * 256 * 4, st>>>(keys_c, m, NS, split->kstar, 8 * i, shist, err);
        }
        NCCLCHK(ncclAllReduce(shist, shist, (size_t)NS * 256, ncclUint32, ncclSum, comm, st));
        ++launches;
        k_split_select<<<1, 64, 0, st>>>(shist, NS, n, S, split->kstar, below);
      }
      if (m) {
        ++launches;
        k_split_buckets<KeyT><<<cblocks, 256, 0, st>>>(keys_c, m, split, bcnt, err);
      }
      NCCLCHK(ncclAllGather(bcnt, cntall_b, NB, ncclUint32, comm, st));
      ++launches;
      k_split_plan<<<1, 32, 0, st>>>(cntall_b, (uint32_t)G, (uint32_t)r, n, S, split, sbases, srecv);
      if (!peer) {  // the NCCL transport scatters into the local send buffer in bucket order
        CUDACHK(cudaMemsetAsync(split->dst_off, 0, sizeof(uint32_t) * 64, st));
        CUDACHK(cudaMemcpyAsync(h_left, split->left, sizeof(uint32_t) * (G + 1), cudaMemcpyDeviceToHost, st));
        CUDACHK(cudaMemcpyAsync(h_srecv, srecv, sizeof(uint32_t) * 2 * G, cudaMemcpyDeviceToHost, st));
      }

      // ---- 6. one stable partition pass by splitter bucket, scattered to the destinations
      nvtx_step("pbit.mg.exchange");
      if (m) {
        SweepArgs sa{};
        sa.kin[0] = keys_c; sa.vin[0] = ids_c;
        sa.bases = sbases; sa.status = status; sa.tile_ctr = tile_ctr; sa.err = err; sa.n = m;
        sa.slot = 79;  // its own ticket counter and lookback epoch (the sort passes use 0..)
        sa.digit = 0; sa.src = 0; sa.last = 0; sa.split = split;
        constexpr int IPT = (KB == 8) ? SWEEP_IPT64 : SWEEP_IPT32;
        ++launches;
        launch_one<KeyT, 7, IPT, SRC_SPLIT>(sa, st, rank_mode());
      }
      if (peer) {
        // every rank's partition has landed before anyone reads its receive arrays
        NCCLCHK(ncclAllReduce(barrier_w, barrier_w + 1, 1, ncclUint32, ncclSum, comm, st));
      } else {
        MGWAIT();  // the host needs the send / receive ranges
        NcclGroup grp;
        NCCLCHK(grp.start());
        for (int d = 0; d < G; ++d) {
          const uint32_t sc = h_left[d + 1] - h_left[d], rcn = h_srecv[2 * d + 1];
          if (sc) {
            NCCLCHK(ncclSend(send_k + h_left[d], sc, key_t, d, comm, st));
            NCCLCHK(ncclSend(send_i + h_left[d], sc, ncclUint32, d, comm, st));
          }
          if (rcn) {
            NCCLCHK(ncclRecv(recv_k + h_srecv[2 * d], rcn, key_t, d, comm, st));
            NCCLCHK(ncclRecv(recv_i + h_srecv[2 * d], rcn, ncclUint32, d, comm, st));
          }
        }
        NCCLCHK(grp.end());
      }
      rk = recv_k;
      ri = recv_i;
    } else {
      rk = keys_c;  // one rank: the chunk is the whole list
      ri = ids_c;
    }

    // ---- 7. stable local sort of the received runs (the global plan's digits; the bases
    // from the local histogram -- one rank: the global one, and the first pass gathers
    // from the slots)
    nvtx_step("pbit.mg.local_sort");
    {
      uint32_t* ri_w = const_cast<uint32_t*>(ri);
      KeyT* rk_w = const_cast<KeyT*>(rk);
      fin = ri;
      fin_k = rk;
      const Plan hp = h_plan;
      if (m && hp.npasses) {
        if (!solo) {
          ++launches;
          k_chunk_hist<KeyT><<<std::max(1, std::min((int)((m + 255) / 256), sms * 4)), 256, (size_t)D * radix * 4,
                               st>>>(rk, m, K, D, hist_r, err);
          ++launches;
          k_plan<<<1, 256, 0, st>>>(hist_r, bases_r, plan_r, D, K, m, err);
        }
        SweepArgs la{};
        la.kin[0] = rk_w; la.kin[1] = kb1; la.vin[0] = ri_w; la.vin[1] = ib1;
        la.kout[0] = rk_w; la.kout[1] = kb1; la.vout[0] = ri_w; la.vout[1] = ib1;
        la.bases = solo ? bases_g : bases_r; la.status = status; la.tile_ctr = tile_ctr; la.err = err; la.n = m;
        if (solo) {
          la.slots = slots_own; la.cap = cap; la.seg = seg; la.seg_ord = seg_ord; la.seg_pos = seg_pos;
          la.tile_first = part_first; la.nseg = nseg;
        }
        // the last pass keeps the keys when the sorted keys are asked for (N3 records)
        launch_key_passes_k<KB>(K, la, hp, out_keys_local != nullptr, st, nullptr, 0, solo ? SRC_GATHER : SRC_TMA);
        launches += hp.npasses;
        fin = (hp.npasses & 1u) ? ib1 : ri;
        fin_k = (hp.npasses & 1u) ? kb1 : rk;
      }
    }

    // N3 records: this rank's sorted positions [P0, P1) -- ids and keys (skipped for an
    // invalid list, like every later kernel)
    if (m && (out_order_local || out_keys_local)) {
      ++launches;
      k_materialize<KB><<<std::max(1, std::min((int)((m + 255) / 256), sms * 8)), 256, 0, st>>>(
          fin, fin_k, m, out_order_local, out_keys_local, km, err);
    }

    // ---- 8. stitch and relink: every rank's first and last sorted id (all-gather), then
    // (v, successor[, predecessor]) routed to the owner of v
    nvtx_step("pbit.mg.relink");
    ++launches;
    k_first_last_id<<<1, 1, 0, st>>>(fin, m, fl);
    NCCLCHK(ncclAllGather(fl, fl_all, 2, ncclUint32, comm, st));
    ++launches;
    k_edges<<<1, 1, 0, st>>>(fl_all, (uint32_t)G, (uint32_t)r, edges);
    if (solo) {  // every record is this rank's own: relink straight from the sorted ids
      launches += launch_relink(fin, nullptr, 0, n, rbuf0, rbuf1, cursors, out_next_local,
                                with_prev ? out_prev_local : nullptr, err, st, sms);
    } else {
      const int pblocks = std::max(1, std::min((int)((m + 4095) / 4096), sms * 4));
      const FastDiv fS = FastDiv::make(S);
      PairDst pd{};
      if (m) {
        ++launches;
        if (W == 3) k_pairs_owner<3><<<pblocks, 256, 0, st>>>(fin, m, edges, fS, G, pcnt, nullptr, nullptr, pd, 0, err);
        else k_pairs_owner<2><<<pblocks, 256, 0, st>>>(fin, m, edges, fS, G, pcnt, nullptr, nullptr, pd, 0, err);
      }
      NCCLCHK(ncclAllGather(pcnt, pcntall, G, ncclUint32, comm, st));
      ++launches;
      k_pairs_plan<<<1, 32, 0, st>>>(pcntall, (uint32_t)G, (uint32_t)r, pbase, psbase, precv);
      void* recvrec = peer ? (void*)(win->local + a_kn) : precvb;
      for (int d = 0; d < G; ++d) pd.dst[d] = peer ? (void*)wk(d, a_kn) : psend;
      if (m) {
        ++launches;
        if (W == 3)
          k_pairs_owner<3><<<pblocks, 256, 0, st>>>(fin, m, edges, fS, G, nullptr, peer ? pbase : psbase, pfill, pd, 1, err);
        else
          k_pairs_owner<2><<<pblocks, 256, 0, st>>>(fin, m, edges, fS, G, nullptr, peer ? pbase : psbase, pfill, pd, 1, err);
      }
      if (peer) {
        NCCLCHK(ncclAllReduce(barrier_w, barrier_w + 1, 1, ncclUint32, ncclSum, comm, st));
      } else {
        CUDACHK(cudaMemcpyAsync(h_pall.data(), pcntall, 4ull * G * G, cudaMemcpyDeviceToHost, st));
        CUDACHK(cudaMemcpyAsync(h_prow, pcntall + (size_t)r * G, 4ull * G, cudaMemcpyDeviceToHost, st));
        CUDACHK(cudaMemcpyAsync(h_psbase, psbase, 4ull * G, cudaMemcpyDeviceToHost, st));
        CUDACHK(cudaMemcpyAsync(h_precv, precv, 8ull * G, cudaMemcpyDeviceToHost, st));
        CUDACHK(cudaMemcpyAsync(&hb->err, err, 4, cudaMemcpyDeviceToHost, st));
        MGWAIT();
        // an invalid list stopped every kernel after the ranking (the error word is the same
        // on every rank: all-reduced after the walk, then the same redundant ranking)
        if (hb->err & E_DYN_FULL) { rc = RC_DYN_OVERFLOW; goto done; }
        if (hb->err) { rc = PBIT_ERR_INVALID_LIST; goto done; }
        // every rank checks EVERY rank's receive total against its node count, from the same
        // all-gathered matrix, so all take the same branch (none is left in the exchange)
        for (int d = 0; d < G; ++d) {
          uint64_t racc = 0;
          for (int q = 0; q < G; ++q) racc += h_pall[(size_t)q * G + d];
          const uint64_t lo_d = std::min<uint64_t>(n, (uint64_t)d * S), hi_d = std::min<uint64_t>(n, (uint64_t)(d + 1) * S);
          if (racc != hi_d - lo_d) { set_last_error("pbit_sort_list_mg", "relink routing mismatch"); rc = PBIT_ERR_CUDA; goto done; }
        }
        NcclGroup grp;
        NCCLCHK(grp.start());
        for (int d = 0; d < G; ++d) {
          if (h_prow[d])
            NCCLCHK(ncclSend((uint32_t*)psend + (size_t)W * h_psbase[d], (size_t)W * h_prow[d], ncclUint32, d, comm, st));
          if (h_precv[2 * d + 1])
            NCCLCHK(ncclRecv((uint32_t*)precvb + (size_t)W * h_precv[2 * d], (size_t)W * h_precv[2 * d + 1], ncclUint32,
                             d, comm, st));
        }
        NCCLCHK(grp.end());
      }
      // the received records (global v): out[v - lo] = succ (and pred) for every own id v
      if (n_local)
        launches += launch_relink(nullptr, recvrec, lo, n_local, rbuf0, rbuf1, cursors, out_next_local,
                                  with_prev ? out_prev_local : nullptr, err, st, sms);
    }
    CUDACHK(cudaMemcpyAsync(&hb->err, err, 4, cudaMemcpyDeviceToHost, st));
    CUDACHK(cudaMemcpyAsync(hb->res, edges, 12, cudaMemcpyDeviceToHost, st));
    MGWAIT();
    CUDACHK(cudaGetLastError());
    if (hb->err & E_DYN_FULL) { rc = RC_DYN_OVERFLOW; goto done; }  // every rank sees it (all-reduced)
    if (hb->err) { rc = PBIT_ERR_INVALID_LIST; goto done; }
    *out_head = hb->res[2];  // rank 0 always holds sorted position 0 (n > 0)
    if (launches_out) *launches_out = launches;
  }
done:
  while (nvtx_depth-- > 0) nvtxRangePop();
  if (plan_ev) cudaEventDestroy(plan_ev);
  cudaFreeAsync(base, st);
  if (rc != PBIT_ERR_NCCL) cudaStreamSynchronize(st);  // a stuck collective is released by the caller's abort
  return rc;
}

}  // namespace

}  // namespace pbit

using namespace pbit;

extern "C" {

int pbit_mg_get_unique_id(void* id_out) {
  if (!id_out) return PBIT_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PBIT_ERR_NCCL;
  memcpy(id_out, &id, sizeof id);
  return PBIT_OK;
}

int pbit_mg_comm_init(void** comm_out, int nranks, const void* id, int rank) {
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return PBIT_ERR_INVALID_ARG;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t c;
  if (ncclCommInitRank(&c, nranks, uid, rank) != ncclSuccess) return PBIT_ERR_NCCL;
  *comm_out = (void*)c;
  return PBIT_OK;
}

static void release_window(void* comm) {
  std::lock_guard<std::mutex> lk(g_win_mu);
  g_last_transport.erase(comm);
  auto it = g_wins.find(comm);
  if (it != g_wins.end()) {
    win_release(it->second);
    g_wins.erase(it);
  }
}

int pbit_mg_comm_abort(void* comm) {
  if (!comm) return PBIT_ERR_INVALID_ARG;
  const int rc = ncclCommAbort((ncclComm_t)comm) == ncclSuccess ? PBIT_OK : PBIT_ERR_NCCL;
  release_window(comm);
  return rc;
}

int pbit_mg_comm_destroy(void* comm) {
  if (!comm) return PBIT_ERR_INVALID_ARG;
  release_window(comm);
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? PBIT_OK : PBIT_ERR_NCCL;
}

// Host-side plan of the exchange (step 5), exported so the multi-rank logic can be tested
// without GPUs (k_split_plan is its device twin).  Every rank's chunk is sorted stably by
// splitter bucket; splitter s sits at global rank x_s = min(n, (s+1)*S) of the final order
// and has key k*_s.  lt[q*(G-1)+s] / le[q*(G-1)+s] = keys of rank q below / up to k*_s.
// Elements below k*_s go left of the split; of the t_s = x_s - sum_q lt ties that also go
// left, ranks take theirs in rank order (= list-position order).  Rank r sends to d the
// contiguous range [left_r(d-1), left_r(d)) of its bucket order and receives, in
// source-rank order, from every q the range [left_q(r-1), left_q(r)).
void pbit_mg_exchange_plan(int G, int r, uint64_t n, uint64_t S, const uint64_t* lt, const uint64_t* le,
                           uint64_t* send_off, uint64_t* send_count, uint64_t* recv_off, uint64_t* recv_count) {
  const int NS = G - 1;
  std::vector<uint64_t> left((size_t)G * (G + 1), 0);  // left[q][s+1]: rank q's elements left of split s
  for (int q = 0; q < G; ++q) {
    const uint64_t lo = std::min<uint64_t>(n, (uint64_t)q * S), hi = std::min<uint64_t>(n, (uint64_t)(q + 1) * S);
    left[(size_t)q * (G + 1) + 0] = 0;
    left[(size_t)q * (G + 1) + G] = hi - lo;  // the chunk size
  }
  for (int sp = 0; sp < NS; ++sp) {
    const uint64_t x = std::min<uint64_t>(n, (uint64_t)(sp + 1) * S);
    uint64_t L = 0;
    for (int q = 0; q < G; ++q) L += lt[(size_t)q * NS + sp];
    uint64_t t = x > L ? x - L : 0;
    for (int q = 0; q < G; ++q) {
      const uint64_t a = lt[(size_t)q * NS + sp], eq = le[(size_t)q * NS + sp] - a;
      const uint64_t take = std::min(eq, t);
      t -= take;
      left[(size_t)q * (G + 1) + sp + 1] = a + take;
    }
  }
  uint64_t racc = 0;
  for (int d = 0; d < G; ++d) {
    send_off[d] = left[(size_t)r * (G + 1) + d];
    send_count[d] = left[(size_t)r * (G + 1) + d + 1] - send_off[d];
    recv_off[d] = racc;
    recv_count[d] = left[(size_t)d * (G + 1) + r + 1] - left[(size_t)d * (G + 1) + r];
    racc += recv_count[d];
  }
}

uint64_t pbit_mg_slice(uint64_t n_global, int nranks) {
  if (nranks < 1) return 0;
  const uint64_t per = (n_global + nranks - 1) / nranks;
  return (per + 63) / 64 * 64;
}

// Every rank's verdict on its arguments, and the arguments every rank must share, agreed
// by one small all-reduce before any data moves: a bad argument on one rank then fails the
// call on every rank, instead of leaving the others waiting in the first collective.
// shared[0..ns): must be equal on all ranks (compared as max and ~max(~x) = min);
// flags[0..nf): returned as the maximum over the ranks.  Returns the largest status any
// rank reported, or INVALID_ARG if the shared values differ.
static int mg_agree(int rc_local, const uint64_t* shared, int ns, uint64_t* flags, int nf, ncclComm_t comm,
                    cudaStream_t st) {
  std::vector<uint64_t> h(1 + 2 * (size_t)ns + nf);
  h[0] = (uint64_t)rc_local;
  for (int i = 0; i < ns; ++i) { h[1 + i] = shared[i]; h[1 + ns + i] = ~shared[i]; }
  for (int i = 0; i < nf; ++i) h[1 + 2 * ns + i] = flags[i];
  uint64_t* d = nullptr;
  const size_t bytes = 8 * h.size();
  if (ws_alloc((void**)&d, bytes, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  int rc = PBIT_OK;
  if (cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = PBIT_ERR_CUDA;
  if (!rc && ncclAllReduce(d, d, h.size(), ncclUint64, ncclMax, comm, st) != ncclSuccess) rc = PBIT_ERR_NCCL;
  if (!rc && cudaMemcpyAsync(h.data(), d, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) rc = PBIT_ERR_CUDA;
  if (!rc) rc = mg_wait(st, comm);
  cudaFreeAsync(d, st);
  if (rc) return rc;
  for (int i = 0; i < nf; ++i) flags[i] = h[1 + 2 * ns + i];
  for (int i = 0; i < ns; ++i)
    if (h[1 + i] != ~h[1 + ns + i]) {
      set_last_error("pbit_sort_list_mg", "the ranks passed different shared arguments");
      return std::max<int>((int)h[0], PBIT_ERR_INVALID_ARG);
    }
  return (int)h[0];
}

int pbit_sort_list_mg(const void* keys_local, const uint32_t* next_local, uint32_t head, uint64_t n_global,
                      uint64_t node_lo, uint64_t n_local, int key_bits, uint32_t* out_head,
                      uint32_t* out_next_local, void* nccl_comm, const pbit_opts* opts) {
  if (!nccl_comm || !out_head) return PBIT_ERR_INVALID_ARG;  // no communicator to agree over
  ncclComm_t comm = (ncclComm_t)nccl_comm;
  int G = 0, r = 0;
  if (ncclCommCount(comm, &G) != ncclSuccess) return PBIT_ERR_NCCL;
  if (ncclCommUserRank(comm, &r) != ncclSuccess) return PBIT_ERR_NCCL;
  cudaStream_t st = opts ? (cudaStream_t)opts->stream : (cudaStream_t)0;
  const int K = pass_bits(opts && opts->digit_bits ? opts->digit_bits : 8);
  uint32_t* out_prev_local = opts ? opts->out_prev : nullptr;
  const KeyMap km{opts ? opts->key_kind : PBIT_KEY_UNSIGNED, opts && opts->descending ? 1 : 0};
  const uint64_t S = pbit_mg_slice(n_global, G);
  // this rank's own checks (status codes as in pbit.h)
  const int rc_local = [&]() -> int {
    if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return PBIT_ERR_INVALID_ARG;
    if (!K) return PBIT_ERR_INVALID_ARG;
    if (n_global > 0xFFFFFFFEull) return PBIT_ERR_INVALID_ARG;
    if (out_prev_local && out_prev_local == out_next_local) return PBIT_ERR_INVALID_ARG;
    if (!key_kind_ok(km.kind, key_bits)) return PBIT_ERR_INVALID_ARG;
    if (G > 64) return PBIT_ERR_UNSUPPORTED;
    const uint64_t want_lo = (uint64_t)r * S;
    const uint64_t want_n = n_global > want_lo ? std::min<uint64_t>(S, n_global - want_lo) : 0;
    if (node_lo != want_lo || n_local != want_n) return PBIT_ERR_UNSUPPORTED;
    if ((uint64_t)G * S > 0xFFFFFFFFull) return PBIT_ERR_UNSUPPORTED;
    if (n_global && (uint64_t)head >= n_global) return PBIT_ERR_INVALID_ARG;
    if (n_local && (!keys_local || !next_local || !out_next_local)) return PBIT_ERR_INVALID_ARG;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_CUDA; }
    if (n_local && (pointer_kind(keys_local, dev) != 1 || pointer_kind(next_local, dev) != 1 ||
                    pointer_kind(out_next_local, dev) != 1 ||
                    (out_prev_local && pointer_kind(out_prev_local, dev) != 1) ||
                    (opts && opts->out_order && pointer_kind(opts->out_order, dev) != 1) ||
                    (opts && opts->out_keys && pointer_kind(opts->out_keys, dev) != 1)))
      return PBIT_ERR_INVALID_ARG;
    return PBIT_OK;
  }();
  // shared by all ranks: the list, the key format, the digit width, the transport.
  // out_prev: the ranks that own nodes must all pass it or none (flags: some rank with /
  // without it)
  const uint64_t shared[7] = {n_global, head, (uint64_t)key_bits, (uint64_t)K, (uint64_t)km.kind,
                              (uint64_t)km.descending, (uint64_t)transport_request()};
  uint32_t* out_order_local = opts ? opts->out_order : nullptr;
  void* out_keys_local = opts ? opts->out_keys : nullptr;
  uint64_t flags[6] = {n_local && out_prev_local ? 1ull : 0ull, n_local && !out_prev_local ? 1ull : 0ull,
                       n_local && out_order_local ? 1ull : 0ull, n_local && !out_order_local ? 1ull : 0ull,
                       n_local && out_keys_local ? 1ull : 0ull, n_local && !out_keys_local ? 1ull : 0ull};
  int rc = mg_agree(rc_local, shared, 7, flags, 6, comm, st);
  if (rc) return rc;
  if ((flags[0] && flags[1]) || (flags[2] && flags[3]) || (flags[4] && flags[5])) {
    set_last_error("pbit_sort_list_mg", "out_prev / out_order / out_keys passed on some ranks but not on others");
    return PBIT_ERR_INVALID_ARG;
  }
  const bool with_prev = flags[0] != 0;
  if (n_global == 0) {
    if (head != PBIT_NULL) return PBIT_ERR_INVALID_LIST;
    *out_head = PBIT_NULL;
    return PBIT_OK;
  }
  int transport = transport_request();
  for (;;) {
#define PBIT_RUN_MG(KB)                                                                                          \
    run_mg<KB>(keys_local, next_local, head, (uint32_t)n_global, (uint32_t)S, (uint32_t)n_local, K, km, out_head, \
               out_next_local, out_prev_local, with_prev, comm, G, r, st, transport, opts ? opts->launches : nullptr, \
               out_order_local, out_keys_local)
    switch (key_bits) {
      case 8: rc = PBIT_RUN_MG(1); break;
      case 16: rc = PBIT_RUN_MG(2); break;
      case 32: rc = PBIT_RUN_MG(4); break;
      default: rc = PBIT_RUN_MG(8); break;
    }
#undef PBIT_RUN_MG
    // the peer transport is unavailable (some rank cannot map the others' memory), or its
    // per-rank dynamic ruler table overflowed: every rank saw the same verdict -> NCCL
    if (transport != T_NCCL && (rc == PBIT_ERR_UNSUPPORTED || rc == RC_DYN_OVERFLOW)) {
      transport = T_NCCL;
      continue;
    }
    {
      std::lock_guard<std::mutex> lk(g_win_mu);
      g_last_transport[(void*)comm] = transport;
    }
    return rc;
  }
}

int pbit_mg_transport(void* comm) {
  if (!comm) return -1;
  std::lock_guard<std::mutex> lk(g_win_mu);
  auto it = g_last_transport.find(comm);
  return it == g_last_transport.end() ? -1 : it->second;
}

}  // extern "C"
