// mg.cu -- pbit_sort_list_mg: one list sorted by G ranks (one process per GPU) over an
// NCCL communicator, plus the NCCL communicator helpers.
//
// Rank r owns node ids [r*S, r*S + n_local), S = 64 * ceil(ceil(n/G) / 64), and after the
// exchange holds sorted positions [r*S, r*S + S) of the output.  SURVEY §8(e):
//   1  pack own slice -> kn replica         ncclAllGather(kn), ncclAllReduce(digit histograms)
//   2  count-walk own rulers                 ncclAllGather(segment table), ncclAllReduce(error)
//   3  rank the ruler list (every rank, redundantly; validates the list)
//   4  emit-walk the segments covering own positions [r*S, r*S+S) -> list-order chunk
//   0  the ranks agree on their arguments (one all-reduce; pbit.h)
//   5  stable local sort of the chunk by the full key; exact splitters of the global
//      (key, list position) order at ranks (s+1)*S by radix refinement (ncclAllReduce
//      of candidate counts per digit); the host planner splits ties in rank order;
//      the sorted ranges are exchanged                                   ncclSend/Recv
//   6  full local sort of the received runs (stable LSD, all non-trivial digits)
//   7  stitch (ncclAllGather of first ids) and route (v, succ) to the owner of v
//                                           ncclSend/Recv; local windowed relink
// Received streams are concatenated in source-rank order: elements with equal keys from
// lower ranks have smaller list positions, so the stable local sort of step 6 restores
// the global stable order exactly.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <vector>

#include "../../include/pbit.h"
#include "launch.cuh"
#include "mg_kernels.cuh"
#include "pbit_internal.h"

static_assert(sizeof(ncclUniqueId) == PBIT_MG_UNIQUE_ID_BYTES, "NCCL unique id size");

namespace pbit {

namespace {

struct Bump {
  char* base = nullptr;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (count * sizeof(T) + 255) & ~(size_t)255;
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

template <int KB>
int run_mg(const void* keys_local, const uint32_t* next_local, uint32_t head, uint32_t n, uint32_t S,
           uint32_t n_local, int K, KeyMap km, uint32_t* out_head, uint32_t* out_next_local,
           uint32_t* out_prev_local, bool with_prev, ncclComm_t comm, int G, int r, cudaStream_t st,
           uint32_t* launches_out) {
  using RT = typename Rec<KB>::T;
  uint32_t launches = 0;
  using KeyT = typename KeyOf<KB>::T;
  constexpr int REC_WORDS = sizeof(RT) / 4;
  const ncclDataType_t key_t = KB == 8 ? ncclUint64 : ncclUint32;
  int rc = PBIT_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (int e = device_info(dev, &sms)) return e;
  init_rank_mode(st);

  SortPlan p;
  make_plan(n, KB * 8, K, &p);
  // a rank's id slice must be a whole number of ruler blocks: S is a multiple of 64
  // (pbit_mg_slice), so the spacing is at most 64 here (make_plan picks 128 from 2^30)
  if (p.s_log2 > 6) {
    p.s_log2 = 6;
    p.R = (uint32_t)(((uint64_t)n + 63) >> 6);
  }
  const int radix = 1 << K;
  const uint32_t s = 1u << p.s_log2;
  const uint32_t bpr = S / s;                      // ruler blocks per rank
  if ((uint64_t)G * bpr * s < (uint64_t)n || S % s) {
    set_last_error("pbit_sort_list_mg", "ruler blocks do not tile the rank slices");
    return PBIT_ERR_UNSUPPORTED;
  }
  const uint32_t Gs = (uint32_t)G * bpr;           // segment-table entries (+1: head ruler)
  RulerSel sel{n, (uint32_t)p.s_log2, p.R};
  const bool head_is_ruler = sel.is_ruler(head);
  const uint32_t head_ruler = head_is_ruler ? (head >> p.s_log2) : Gs;
  const bool own_head = head / S == (uint32_t)r;
  const uint32_t P0 = std::min<uint64_t>(n, (uint64_t)r * S), P1 = std::min<uint64_t>(n, (uint64_t)(r + 1) * S);
  const uint32_t m = P1 - P0;                      // sorted positions held by this rank
  const uint32_t lo = r * S;
  const uint32_t Rmax = Gs + 1;
  RulerSel sub{Rmax, 4u, (Rmax + 15) >> 4};
  const bool hs = sub.is_ruler(head_ruler);
  const uint32_t nsub = sub.R + (hs ? 0u : 1u);
  const uint32_t head_sub = hs ? (head_ruler >> 4) : sub.R;
  const size_t tile = sweep_tile(KB * 8);
  const size_t ntiles = (S + tile - 1) / tile;
  const int D = p.D;

  // ---- workspace
  Bump b;
  RT* kn = nullptr; uint2* seg = nullptr; uint32_t *dist = nullptr, *seg_ord = nullptr, *seg_pos = nullptr;
  uint32_t* part_first = nullptr; unsigned long long* sdist[2] = {}; uint32_t* scnt[2] = {}; uint32_t* ssucc[2] = {};
  KeyT* kbuf[2] = {}; uint32_t* ibuf[2] = {}; unsigned long long* status = nullptr;
  uint2 *send_p = nullptr, *pr[2] = {};
  uint32_t *hist_l = nullptr, *hist_g = nullptr, *hist_a = nullptr, *hist_b = nullptr, *bases_p = nullptr,
           *bases_l = nullptr, *cursors = nullptr, *cntmat = nullptr, *firsts = nullptr, *cnt = nullptr,
           *offs = nullptr, *fill = nullptr, *cntall = nullptr, *tile_ctr = nullptr, *nseg = nullptr,
           *zero = nullptr, *tile_first_unused = nullptr, *mg_c = nullptr, *mg_call = nullptr;
  unsigned long long* mg_q = nullptr;
  Plan *plan_g = nullptr, *plan_p = nullptr, *plan_l = nullptr;
  int* err = nullptr;
  size_t ctl_off = 0, ctl_end = 0;
  std::vector<uint32_t> h_counts, h_cntall;
  Plan h_plan{};
  int h_err = 0;
  uint32_t h_firsts[130];  // first and last sorted id of every rank
  auto carve = [&]() {
    kn = b.take<RT>((size_t)G * S);
    seg = b.take<uint2>(Rmax);
    dist = b.take<uint32_t>(Rmax);
    seg_ord = b.take<uint32_t>(Rmax);
    seg_pos = b.take<uint32_t>(Rmax);
    tile_first_unused = b.take<uint32_t>(1);
    for (int i = 0; i < 2; ++i) {
      sdist[i] = b.take<unsigned long long>(nsub + 1);
      scnt[i] = b.take<uint32_t>(nsub + 1);
      ssucc[i] = b.take<uint32_t>(nsub + 1);
      kbuf[i] = b.take<KeyT>(S);
      ibuf[i] = b.take<uint32_t>(S);
      pr[i] = b.take<uint2>(S);
    }
    status = b.take<unsigned long long>(ntiles * 256);
    send_p = b.take<uint2>(S);
    ctl_off = b.off;
    part_first = b.take<uint32_t>(G + 2);  // zeroed with the control block
    hist_l = b.take<uint32_t>((size_t)D * radix);
    hist_g = b.take<uint32_t>((size_t)D * radix);
    hist_a = b.take<uint32_t>((size_t)D * radix);
    hist_b = b.take<uint32_t>((size_t)D * radix);
    bases_p = b.take<uint32_t>((size_t)D * radix);
    bases_l = b.take<uint32_t>((size_t)D * radix);
    cursors = b.take<uint32_t>(relink_cursor_words(S));
    cntmat = b.take<uint32_t>((size_t)G * radix);
    firsts = b.take<uint32_t>(2 * G + 2);
    cnt = b.take<uint32_t>(G);
    offs = b.take<uint32_t>(G);
    fill = b.take<uint32_t>(G);
    cntall = b.take<uint32_t>((size_t)G * G);
    tile_ctr = b.take<uint32_t>(80);
    nseg = b.take<uint32_t>(1);
    zero = b.take<uint32_t>(1);
    plan_g = b.take<Plan>(1);
    plan_p = b.take<Plan>(1);
    plan_l = b.take<Plan>(1);
    err = b.take<int>(1);
    ctl_end = b.off;
    mg_q = b.take<unsigned long long>((size_t)64 * 256);
    mg_c = b.take<uint32_t>((size_t)64 * 256);
    mg_call = b.take<uint32_t>((size_t)2 * 64 * 64);
  };
  carve();
  const size_t bytes = b.off;
  char* base = nullptr;
  if (ws_alloc((void**)&base, bytes, st) != cudaSuccess) { cudaGetLastError(); return PBIT_ERR_OOM; }
  b = Bump{base, 0};
  carve();

  {
    CUDACHK(cudaMemsetAsync(base + ctl_off, 0, ctl_end - ctl_off, st));
    CUDACHK(cudaMemsetAsync(seg, 0, sizeof(uint2) * Rmax, st));
    CUDACHK(cudaMemsetAsync(status, 0, ntiles * 256 * 8, st));

    // ---- 1. pack the own slice into its place of the replica; local histograms
    if (n_local) {
      const int blocks = full_wave(k_pack<KB>, PACK_THREADS, (size_t)D * radix * 4, sms,
                                   (n_local + PACK_THREADS - 1) / PACK_THREADS);
      ++launches;
      k_pack<KB><<<blocks, PACK_THREADS, (size_t)D * radix * 4, st>>>(keys_local, next_local, n_local, n,
                                                                       kn + lo, hist_l, K, D, err, km);
    }
    NCCLCHK(ncclAllGather(kn + lo, kn, (size_t)S * REC_WORDS, ncclUint32, comm, st));
    NCCLCHK(ncclAllReduce(hist_l, hist_g, (size_t)D * radix, ncclUint32, ncclSum, comm, st));

    // ---- 2. count-walk the own rulers, share the segment table
    {
      const uint32_t b_lo = r * bpr, b_hi = (r + 1) * bpr;
      const uint32_t total = bpr + (own_head && !head_is_ruler ? 1u : 0u);
      int blocks = sms * (2048 / WALK_THREADS);
      if ((uint32_t)blocks * 4 > total) blocks = std::max(1u, (total + 3) / 4);
      const uint32_t per = (total + blocks - 1) / blocks;
      ++launches;
      k_walk_count<KB><<<blocks, WALK_THREADS, 0, st>>>(kn, sel, b_lo, b_hi,
                                                        own_head && !head_is_ruler ? Gs : PBIT_NULL32, head, seg, per,
                                                        err);
    }
    NCCLCHK(ncclAllGather(seg + (size_t)r * bpr, seg, (size_t)bpr * 2, ncclUint32, comm, st));
    NCCLCHK(ncclAllReduce(seg + Gs, seg + Gs, 2, ncclUint32, ncclMax, comm, st));
    NCCLCHK(ncclAllReduce(err, err, 1, ncclInt32, ncclMax, comm, st));

    // ---- 3. rank the ruler list (identical on every rank)
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
                                             scnt[cur], dist, seg_ord, seg_pos, part_first, S, n, nseg, err);
    }
    ++launches;
    k_plan<<<1, 256, 0, st>>>(hist_g, bases_l, plan_g, D, K, n, err);
    CUDACHK(cudaMemcpyAsync(&h_plan, plan_g, sizeof(Plan), cudaMemcpyDeviceToHost, st));
    CUDACHK(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
    MGWAIT();
    if (h_err) { rc = PBIT_ERR_INVALID_LIST; goto done; }

    // ---- 4. emit the list-order chunk of positions [P0, P1)
    if (m) {
      const int blocks = std::max(1, std::min((int)((Gs / G + 2 + 255) / 256), sms * 8));
      ++launches;
      k_emit_walk<KB><<<blocks, 256, 0, st>>>(kn, sel, head, seg, seg_ord, seg_pos, part_first, r, nseg, P0, P1,
                                              kbuf[0], ibuf[0], err);
    }

    const Plan* final_plan = plan_l;  // parity of the final ids: fin[npasses & 1]
    uint32_t* fin[2] = {ibuf[0], ibuf[1]};
    if (h_plan.npasses == 0) {
      // every digit trivial: all keys equal, the list order is the sorted order
      CUDACHK(cudaMemsetAsync(plan_l, 0, sizeof(Plan), st));
    } else {
      // ---- 5a. stable local sort of the chunk (kbuf[0], ibuf[0]) by the full key
      SweepArgs pa{};
      pa.kin[0] = kbuf[0]; pa.kin[1] = kbuf[1]; pa.vin[0] = ibuf[0]; pa.vin[1] = ibuf[1];
      pa.kout[0] = kbuf[0]; pa.kout[1] = kbuf[1]; pa.vout[0] = ibuf[0]; pa.vout[1] = ibuf[1];
      pa.bases = bases_p; pa.status = status; pa.tile_ctr = tile_ctr; pa.err = err; pa.n = m;
      // keep_keys below: the sorted keys are needed for the splitters and the exchange
      if (m) {
        ++launches;
        k_chunk_hist<KeyT><<<std::max(1, std::min((int)((m + 255) / 256), sms * 4)), 256, (size_t)D * radix * 4, st>>>(
            kbuf[0], m, K, D, hist_a, err);
      }
      ++launches;
      k_plan<<<1, 256, 0, st>>>(hist_a, bases_p, plan_p, D, K, m, err);
      Plan h_pp{};
      CUDACHK(cudaMemcpyAsync(&h_pp, plan_p, sizeof(Plan), cudaMemcpyDeviceToHost, st));
      MGWAIT();
      if (m) { launch_key_passes_k<KB>(K, pa, h_pp, true, st, nullptr, 0, SRC_TMA); launches += h_pp.npasses; }
      const int pa_par = (int)(h_pp.npasses & 1u);  // sorted chunk in kbuf/ibuf[pa_par]
      const KeyT* sk = kbuf[pa_par];

      // ---- 5b. exact splitters of the final (key, list position) order: split s sits at
      // global rank x_s = (s+1)*S.  Radix refinement from the top digit: per round, the
      // global count of keys below each candidate (prefix, c) -- lower bounds in every
      // rank's sorted chunk, summed by ncclAllReduce -- fixes one more digit of k*_s.
      const int NS = G - 1;
      std::vector<unsigned long long> prefix(std::max(NS, 1), 0ull), h_q;
      std::vector<uint32_t> h_cnt;
      for (int i = D - 1; i >= 0 && NS > 0; --i) {
        const int wbits = i == D - 1 ? KB * 8 - K * (D - 1) : K;
        const int nc = 1 << wbits;
        h_q.assign((size_t)NS * nc, 0ull);
        for (int sp = 0; sp < NS; ++sp)
          for (int c = 0; c < nc; ++c) h_q[(size_t)sp * nc + c] = ((prefix[sp] << wbits) | (unsigned long long)c) << (K * i);
        CUDACHK(cudaMemcpyAsync(mg_q, h_q.data(), 8ull * NS * nc, cudaMemcpyHostToDevice, st));
        ++launches;
        k_count_below<KeyT><<<(NS * nc + 255) / 256, 256, 0, st>>>(sk, m, mg_q, NS * nc, 0, mg_c);
        NCCLCHK(ncclAllReduce(mg_c, mg_c, (size_t)NS * nc, ncclUint32, ncclSum, comm, st));
        h_cnt.resize((size_t)NS * nc);
        CUDACHK(cudaMemcpyAsync(h_cnt.data(), mg_c, 4ull * NS * nc, cudaMemcpyDeviceToHost, st));
        MGWAIT();
        for (int sp = 0; sp < NS; ++sp) {
          const uint64_t x = std::min<uint64_t>(n, (uint64_t)(sp + 1) * S);
          int pick = 0;  // the largest candidate with (global count below it) <= x
          for (int c = 0; c < nc; ++c)
            if (h_cnt[(size_t)sp * nc + c] <= x) pick = c;
          prefix[sp] = (prefix[sp] << wbits) | (unsigned long long)pick;
        }
      }
      // ---- 5c. per-rank counts below / up to each splitter key; the exchange plan
      std::vector<uint64_t> soff(G), scount(G), roff(G), rcount(G);
      {
        std::vector<uint64_t> h_lt((size_t)G * std::max(NS, 1)), h_le((size_t)G * std::max(NS, 1));
        if (NS > 0) {
          CUDACHK(cudaMemcpyAsync(mg_q, prefix.data(), 8ull * NS, cudaMemcpyHostToDevice, st));
          ++launches;
          k_count_below<KeyT><<<1, 64, 0, st>>>(sk, m, mg_q, NS, 0, mg_c);
          ++launches;
          k_count_below<KeyT><<<1, 64, 0, st>>>(sk, m, mg_q, NS, 1, mg_c + NS);
          NCCLCHK(ncclAllGather(mg_c, mg_call, (size_t)2 * NS, ncclUint32, comm, st));
          h_cnt.resize((size_t)2 * NS * G);
          CUDACHK(cudaMemcpyAsync(h_cnt.data(), mg_call, 8ull * NS * G, cudaMemcpyDeviceToHost, st));
          MGWAIT();
          for (int q = 0; q < G; ++q)
            for (int sp = 0; sp < NS; ++sp) {
              h_lt[(size_t)q * NS + sp] = h_cnt[(size_t)q * 2 * NS + sp];
              h_le[(size_t)q * NS + sp] = h_cnt[(size_t)q * 2 * NS + NS + sp];
            }
        }
        pbit_mg_exchange_plan(G, r, n, S, h_lt.data(), h_le.data(), soff.data(), scount.data(), roff.data(),
                              rcount.data());
      }
      uint64_t racc = 0;
      for (int d = 0; d < G; ++d) racc += rcount[d];
      if (racc != m) { set_last_error("pbit_sort_list_mg", "exchange size mismatch"); rc = PBIT_ERR_CUDA; goto done; }
      // ---- 5d. exchange sorted ranges; receive in source-rank order into the other buffer
      const int pb = pa_par ^ 1;
      NCCLCHK(ncclGroupStart());
      for (int d = 0; d < G; ++d) {
        if (scount[d]) {
          NCCLCHK(ncclSend(kbuf[pa_par] + soff[d], scount[d], key_t, d, comm, st));
          NCCLCHK(ncclSend(ibuf[pa_par] + soff[d], scount[d], ncclUint32, d, comm, st));
        }
        if (rcount[d]) {
          NCCLCHK(ncclRecv(kbuf[pb] + roff[d], rcount[d], key_t, d, comm, st));
          NCCLCHK(ncclRecv(ibuf[pb] + roff[d], rcount[d], ncclUint32, d, comm, st));
        }
      }
      NCCLCHK(ncclGroupEnd());

      // ---- 6. stable sort of the received runs (source order = list-position order for
      // equal keys), buffers swapped so the passes start from buffer pb
      CUDACHK(cudaMemsetAsync(status, 0, ntiles * 256 * 8, st));
      CUDACHK(cudaMemsetAsync(tile_ctr, 0, 80 * 4, st));
      CUDACHK(cudaMemsetAsync(hist_b, 0, 4ull * D * radix, st));
      if (m) {
        ++launches;
        k_chunk_hist<KeyT><<<std::max(1, std::min((int)((m + 255) / 256), sms * 4)), 256, (size_t)D * radix * 4, st>>>(
            kbuf[pb], m, K, D, hist_b, err);
      }
      ++launches;
      k_plan<<<1, 256, 0, st>>>(hist_b, bases_l, plan_l, D, K, m, err);
      Plan h_pl{};
      CUDACHK(cudaMemcpyAsync(&h_pl, plan_l, sizeof(Plan), cudaMemcpyDeviceToHost, st));
      MGWAIT();
      SweepArgs la = pa;
      la.kin[0] = kbuf[pb]; la.kin[1] = kbuf[pb ^ 1]; la.vin[0] = ibuf[pb]; la.vin[1] = ibuf[pb ^ 1];
      la.kout[0] = kbuf[pb]; la.kout[1] = kbuf[pb ^ 1]; la.vout[0] = ibuf[pb]; la.vout[1] = ibuf[pb ^ 1];
      la.bases = bases_l;
      if (m) { launch_key_passes_k<KB>(K, la, h_pl, false, st, nullptr, 0, SRC_TMA); launches += h_pl.npasses; }
      fin[0] = ibuf[pb];
      fin[1] = ibuf[pb ^ 1];
    }

    // ---- 7. stitch and relink: every rank's first and last sorted id (all-gather), then
    // (v, successor) -- and, for out_prev, (v, predecessor) -- routed to the owner of v
    ++launches;
    k_first_last_id<<<1, 1, 0, st>>>(final_plan, fin[0], fin[1], m, firsts + 2 * G);
    NCCLCHK(ncclAllGather(firsts + 2 * G, firsts, 2, ncclUint32, comm, st));
    CUDACHK(cudaMemcpyAsync(h_firsts, firsts, 8ull * G, cudaMemcpyDeviceToHost, st));
    MGWAIT();
    for (int dir = 1; dir >= -1; dir -= 2) {
      // with_prev is the same on every rank (agreed before the first collective): a rank
      // without own nodes still routes its share of the (v, pred) pairs
      if (dir < 0 && !with_prev) continue;
      uint32_t* out_local = dir > 0 ? out_next_local : out_prev_local;
      uint32_t edge = PBIT_NULL32;  // next rank's first id / previous rank's last id
      if (dir > 0) {
        for (int d = r + 1; d < G; ++d)
          if (h_firsts[2 * d] != PBIT_NULL32) { edge = h_firsts[2 * d]; break; }
      } else {
        for (int d = r - 1; d >= 0; --d)
          if (h_firsts[2 * d + 1] != PBIT_NULL32) { edge = h_firsts[2 * d + 1]; break; }
      }
      CUDACHK(cudaMemsetAsync(cnt, 0, 4ull * G, st));
      CUDACHK(cudaMemsetAsync(fill, 0, 4ull * G, st));
      const int pblocks = std::max(1, std::min((int)((m + 4095) / 4096), sms * 4));
      if (m) {
        ++launches;
        k_pairs_owner<<<pblocks, 256, 0, st>>>(final_plan, fin[0], fin[1], m, edge, dir, S, G, cnt, nullptr,
                                               nullptr, nullptr, 0, err);
      }
      NCCLCHK(ncclAllGather(cnt, cntall, G, ncclUint32, comm, st));
      h_cntall.resize((size_t)G * G);
      CUDACHK(cudaMemcpyAsync(h_cntall.data(), cntall, 4ull * G * G, cudaMemcpyDeviceToHost, st));
      MGWAIT();
      std::vector<uint32_t> h_offs(G);
      uint32_t acc = 0;
      for (int d = 0; d < G; ++d) { h_offs[d] = acc; acc += h_cntall[(size_t)r * G + d]; }
      CUDACHK(cudaMemcpyAsync(offs, h_offs.data(), 4ull * G, cudaMemcpyHostToDevice, st));
      if (m) {
        ++launches;
        k_pairs_owner<<<pblocks, 256, 0, st>>>(final_plan, fin[0], fin[1], m, edge, dir, S, G, nullptr, offs, fill,
                                               send_p, 1, err);
      }
      uint32_t racc = 0;
      NCCLCHK(ncclGroupStart());
      for (int d = 0; d < G; ++d) {
        const uint32_t sc = h_cntall[(size_t)r * G + d], rcn = h_cntall[(size_t)d * G + r];
        if (sc) NCCLCHK(ncclSend(send_p + h_offs[d], 2ull * sc, ncclUint32, d, comm, st));
        if (rcn) NCCLCHK(ncclRecv(pr[1] + racc, 2ull * rcn, ncclUint32, d, comm, st));
        racc += rcn;
      }
      NCCLCHK(ncclGroupEnd());
      if (racc != n_local) { set_last_error("pbit_sort_list_mg", "relink routing mismatch"); rc = PBIT_ERR_CUDA; goto done; }
      // the received pairs (global v): out[v - lo] = w for every own id v, in any order
      if (n_local) {
        CUDACHK(cudaMemsetAsync(cursors, 0, relink_cursor_words(S) * 4, st));
        launches += launch_relink(nullptr, pr[1], lo, n_local, pr[0], pr[1], cursors, out_local, err, st, sms);
      }
    }
    CUDACHK(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
    MGWAIT();
    CUDACHK(cudaGetLastError());
    if (h_err) { rc = PBIT_ERR_INVALID_LIST; goto done; }
    *out_head = h_firsts[0];  // rank 0 always holds sorted position 0 (n > 0)
    if (launches_out) *launches_out = launches;
  }
done:
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

int pbit_mg_comm_abort(void* comm) {
  if (!comm) return PBIT_ERR_INVALID_ARG;
  return ncclCommAbort((ncclComm_t)comm) == ncclSuccess ? PBIT_OK : PBIT_ERR_NCCL;
}

int pbit_mg_comm_destroy(void* comm) {
  if (!comm) return PBIT_ERR_INVALID_ARG;
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? PBIT_OK : PBIT_ERR_NCCL;
}

// Host-side plan of the exchange (step 5), exported so the multi-rank logic can be tested
// without GPUs.  Every rank's chunk is sorted by (key, list position); splitter s sits at
// global rank x_s = min(n, (s+1)*S) of the final order and has key k*_s.
// lt[q*(G-1)+s] / le[q*(G-1)+s] = keys of rank q below / up to k*_s.  Elements below k*_s
// go left of the split; of the t_s = x_s - sum_q lt ties that also go left, ranks take
// theirs in rank order (= list-position order).  Rank r sends to d the contiguous range
// [left_r(d-1), left_r(d)) of its sorted chunk and receives, in source-rank order, from
// every q the range [left_q(r-1), left_q(r)).
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
                    (out_prev_local && pointer_kind(out_prev_local, dev) != 1)))
      return PBIT_ERR_INVALID_ARG;
    return PBIT_OK;
  }();
  // shared by all ranks: the list, the key format, the digit width.  out_prev: the ranks
  // that own nodes must all pass it or none (flags: some rank with / without it)
  const uint64_t shared[6] = {n_global, head, (uint64_t)key_bits, (uint64_t)K, (uint64_t)km.kind,
                              (uint64_t)km.descending};
  uint64_t flags[2] = {n_local && out_prev_local ? 1ull : 0ull, n_local && !out_prev_local ? 1ull : 0ull};
  int rc = mg_agree(rc_local, shared, 6, flags, 2, comm, st);
  if (rc) return rc;
  if (flags[0] && flags[1]) {
    set_last_error("pbit_sort_list_mg", "out_prev passed on some ranks but not on others");
    return PBIT_ERR_INVALID_ARG;
  }
  const bool with_prev = flags[0] != 0;
  if (n_global == 0) {
    if (head != PBIT_NULL) return PBIT_ERR_INVALID_LIST;
    *out_head = PBIT_NULL;
    return PBIT_OK;
  }
#define PBIT_RUN_MG(KB)                                                                                          \
  run_mg<KB>(keys_local, next_local, head, (uint32_t)n_global, (uint32_t)S, (uint32_t)n_local, K, km, out_head,   \
             out_next_local, out_prev_local, with_prev, comm, G, r, st, opts ? opts->launches : nullptr)
  switch (key_bits) {
    case 8: return PBIT_RUN_MG(1);
    case 16: return PBIT_RUN_MG(2);
    case 32: return PBIT_RUN_MG(4);
    default: return PBIT_RUN_MG(8);
  }
#undef PBIT_RUN_MG
}

}  // extern "C"
