/*
 * include/pbit.h -- C-ABI of the B200-native Pbit list sort (libpbit.so).
 *
 * Pbit (arXiv cs/0511020) sorts a singly-linked list stably by its keys: it splits
 * the list into Omega = 2^K sub-lists by successive K-bit patterns of the key,
 * most significant first, recurses, and concatenates the sorted fragments
 * ("Split the list in relation to the bit pattern ... merge sorted fragments of
 * the list"; listing P:346-361, ascending loops P:379-380).  On the
 * GPU the same unique result is reached by list ranking + stable LSD radix passes
 * + relink.  The paper's `Node *Pbit(Node *L, unsigned M, Node *P)`
 * returns the new head and relinks `next` in situ.
 *
 * Representation.  A node is an index v in [0, n).  `next[v]` (u32) is the
 * paper's `L->next` and PBIT_NULL is its NULL (P:8).  `keys` holds the
 * paper's `L->data`: an unsigned key of key_bits = M bits (P:63-64,
 * `size = sizeof(data)<<3`), little-endian, node-indexed, element size
 * key_bits/8 bytes.
 *
 * Result.  With v_0 = head, v_{i+1} = next[v_i], the output is the list order
 * sorted ascending and STABLY by unsigned key (equal keys keep input-list order,
 * P:4):  *out_head = w_0, out_next[w_i] = w_{i+1}, out_next[w_{n-1}] =
 * PBIT_NULL.  This result is unique, so every digit width K gives bit-identical
 * output.  pbit_opts.key_kind / .descending select signed or floating-point keys
 * and the descending order, also stable.
 *
 * Ownership.  The caller owns every array.  The library takes stream-ordered workspace
 * from its own memory pool on the current device (cudaMallocFromPoolAsync on the call's
 * stream) and frees it before returning; by default the pool then hands the memory back
 * to the device (release threshold 0; PBIT_POOL_KEEP_GB=x keeps up to x GB mapped between
 * calls, see pbit_workspace_trim).  It never keeps pointers to caller arrays.
 *
 * Synchronisation.  Every call is synchronous: it returns after the work on
 * opts->stream has finished (out_head and the status are host values).  Calls on
 * distinct streams or devices may run concurrently from different host threads.
 *
 * Errors.  Functions return a pbit_status and never throw or abort.
 *   PBIT_ERR_INVALID_ARG  null pointer; key_bits not in {8,16,32,64}; digit_bits out
 *                         of range; key_kind not 0/1/2 or float keys of 8 bits;
 *                         head >= n (n > 0); n > 2^32-2 (PBIT_NULL is not a node id);
 *                         pointers that mix host and device memory.
 *   PBIT_ERR_INVALID_LIST the input is not one NULL-terminated chain of exactly n
 *                         nodes starting at head (cycle, short chain, index >= n,
 *                         a node reached twice).  out_next is NOT modified (the check
 *                         completes before the relink kernel writes).
 *   PBIT_ERR_OOM          workspace allocation failed (the paper's push overflow
 *                         path).
 *   PBIT_ERR_CUDA / _NCCL a propagated runtime error.
 */
#ifndef PBIT_H_
#define PBIT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBIT_NULL 0xFFFFFFFFu /* the list terminator, the paper's NULL (P:8) */

typedef enum {
    PBIT_OK = 0,
    PBIT_ERR_INVALID_ARG = 1,
    PBIT_ERR_INVALID_LIST = 2,
    PBIT_ERR_OOM = 3,
    PBIT_ERR_CUDA = 4,
    PBIT_ERR_NCCL = 5,
    PBIT_ERR_UNSUPPORTED = 6
} pbit_status;

/* Phases whose device time is reported in pbit_opts.phase_ms (CUDA events on the
 * call's stream).  PBIT_PHASE_PASS0 + i is the i-th scheduled radix pass slot. */
enum {
    PBIT_PHASE_PACK = 0,      /* AoS (key,next) pack + all-digit histograms       */
    PBIT_PHASE_WALK = 1,      /* ruling-set walk: segments in list order           */
    PBIT_PHASE_RANK = 2,      /* ruler-list ranking (segment offsets, validation)  */
    PBIT_PHASE_GATHER = 3,    /* segments -> list-order (key, id) arrays + plan    */
    PBIT_PHASE_RELINK = 4,    /* out_next from the sorted ids                      */
    PBIT_PHASE_PASS0 = 5,     /* radix pass slots follow: PASS0 .. PASS0+63        */
    PBIT_NUM_PHASES = 5 + 64
};

typedef struct {
    int digit_bits;  /* K, the bit-pattern length.  0 = auto (8).  1..16
                        (SPEC's range); K need not divide key_bits (the top pattern
                        is narrower).  The paper's default is K = 4.
                        Every K gives the same bytes.  K <= 8 runs K-bit passes; a
                        wider pattern is sorted as stable 8-bit sub-passes,
                        so K = 9..16 runs the passes of K = 8.                       */
    void *stream;    /* cudaStream_t for every launch; NULL = legacy default stream */
    int validate;    /* ignored: validation always runs (it is fused into the ranking
                        and costs one scalar check), whatever this field holds       */
    float *phase_ms; /* optional host array of PBIT_NUM_PHASES floats: device ms per
                        phase, filled after the call (adds CUDA events); else NULL  */
    uint32_t *passes_run; /* optional host out: number of radix passes executed (the
                        non-trivial digits; trivial ones are skipped)               */
    uint32_t *launches; /* optional host out: kernels this call launched            */
    int key_kind;    /* how the key bits are ordered (NEXT row N1):
                        PBIT_KEY_UNSIGNED (0, default) unsigned integers;
                        PBIT_KEY_SIGNED   (1) two's complement integers, the dispatcher
                                          of P:444-466 (stable: DESIGN.md reading Q13);
                        PBIT_KEY_FLOAT    (2) IEEE 754 binary16/32/64 by key_bits (16,
                                          32, 64; 8 is INVALID_ARG), ordered as the
                                          paper's mantissa-then-characteristic passes
                                          with a sign split give (reading
                                          Q18): -NaN < -inf < .. < -0.0 < +0.0 < .. <
                                          +inf < +NaN (IEEE totalOrder).            */
    int descending;  /* 0 ascending, 1 descending; stable in
                        both directions: equal keys keep input-list order.          */
    uint32_t *out_prev; /* optional (NEXT row N2, doubly-linked lists): n predecessor
                        ids of the sorted list, out_prev[w_{i+1}] = w_i and
                        out_prev[w_0] = PBIT_NULL -- the paper's "reverse connection"
                        repair.  Same memory kind as out_next, must not
                        alias it; pbit_sort_list_mg: this rank's n_local predecessors
                        (device).  NULL = singly-linked.                           */
    uint32_t *out_order; /* optional (NEXT row N3, record materialisation): the n node ids
                        in sorted order, out_order[i] = w_i (the walk of the sorted list
                        from *out_head).  Same memory kind as out_next.
                        pbit_sort_list_mg: this rank's sorted positions (below).    */
    void *out_keys;  /* optional: the n keys in sorted order, out_keys[i] = keys[w_i]
                        (the input bit patterns, key_bits/8 bytes each).  Same memory
                        kind as out_next.  With a payload array,
                        payload[out_order[i]] materialises the sorted records.
                        Neither is written when the list is invalid.                */
} pbit_opts;

enum { PBIT_KEY_UNSIGNED = 0, PBIT_KEY_SIGNED = 1, PBIT_KEY_FLOAT = 2 };

/*
 * pbit_sort_list -- stable ascending sort of one singly-linked list.
 *
 *   keys      [in]  n keys, key_bits/8 bytes each, node-indexed (u8/u16/u32/u64).
 *   next      [in]  n successor ids (u32), PBIT_NULL terminates.
 *   head      [in]  first node id (PBIT_NULL iff n == 0).
 *   n         [in]  number of nodes, 0 <= n <= 2^32-2.
 *   key_bits  [in]  M in {8, 16, 32, 64}.
 *   out_head  [out] HOST pointer: head of the sorted list.
 *   out_next  [out] n successor ids of the sorted list.  May alias `next`
 *                   (in-place relink, as the paper's in situ sort).
 *   opts      [in]  may be NULL (defaults).
 *
 * keys/next/out_next are either all CUDA device pointers on the current device
 * (the fast path: nothing is copied) or all host pointers (pinned or pageable;
 * the library stages them through device memory inside the call).
 */
int pbit_sort_list(const void *keys, const uint32_t *next, uint32_t head, uint64_t n,
                   int key_bits, uint32_t *out_head, uint32_t *out_next, const pbit_opts *opts);

/*
 * pbit_sort_array -- the "table" of the paper's tables-versus-lists comparison (section
 * 12; NEXT row N3): a stable sort of an ARRAY of n keys by the same radix
 * passes, with no list ranking and no relink.
 *
 *   keys      [in]  n keys, key_bits/8 bytes each (ordered per opts->key_kind /
 *                   opts->descending, as pbit_sort_list).
 *   n         [in]  0 <= n <= 2^32-2.
 *   key_bits  [in]  M in {8, 16, 32, 64}.
 *   out_index [out] optional: n u32, out_index[i] = position in `keys` of the i-th key
 *                   of the sorted order (equal keys keep their array order).
 *   out_keys  [out] optional: n keys, the sorted keys (the input bit patterns).
 *   opts      [in]  may be NULL; out_prev is ignored.
 * At least one output is required.  keys / out_index / out_keys are all device pointers
 * on the current device or all host pointers (staged).  Errors as pbit_sort_list
 * (no INVALID_LIST).
 */
int pbit_sort_array(const void *keys, uint64_t n, int key_bits, uint32_t *out_index, void *out_keys,
                    const pbit_opts *opts);

/*
 * pbit_sort_list_mg -- the same sort of ONE list whose nodes are sharded over the
 * G ranks of an NCCL communicator (one process per GPU).
 *
 *   keys_local     [in]  device, n_local keys of nodes [node_lo, node_lo+n_local).
 *   next_local     [in]  device, their successors as GLOBAL ids (PBIT_NULL ends).
 *   head           [in]  global id of the first node, identical on every rank.
 *   n_global       [in]  total nodes over all ranks.
 *   node_lo,n_local[in]  this rank's slice of node ids: node_lo = rank * S and
 *                        n_local = min(S, n_global - node_lo) with S = pbit_mg_slice(n_global,
 *                        G) (ceil(n_global / G) rounded up to 64); else PBIT_ERR_UNSUPPORTED.
 *   key_bits       [in]  as above.
 *   out_head       [out] host: head of the sorted list (same on every rank).
 *   out_next_local [out] device, n_local global successor ids for this rank's nodes.
 *   nccl_comm      [in]  ncclComm_t (see pbit_mg_comm_init) spanning the G ranks.
 *   opts           [in]  as above (stream used for every kernel and collective).
 * Collective: every rank must call it with the same head, n_global, key_bits, K,
 * key_kind and descending, and the ranks that own nodes all with or all without
 * opts->out_prev.  The ranks first agree on their arguments (one small all-reduce): if any
 * rank's arguments are invalid, or the shared ones differ, EVERY rank returns the error
 * (the largest status code any rank saw) before data moves.  A NULL nccl_comm or
 * out_head returns PBIT_ERR_INVALID_ARG on that rank alone (the others then time out in
 * the agreement with PBIT_ERR_NCCL after PBIT_MG_TIMEOUT_S).
 * Rank r returns the successors of its own nodes; the sorted positions it computed
 * internally are [r*S, r*S + S) (key-range sharding: exact splitters of the global
 * (key, list position) order, so the shards are equal in size even under heavy duplicates).
 * opts->out_order / out_keys (device, n_local entries each): this rank's share of the
 * sorted records -- the node ids and keys at the sorted positions [r*S, r*S + n_local)
 * (the same count as its node slice); the ranks that own nodes pass them all or none.
 *
 * Transport (PBIT_MG_TRANSPORT, read at every call; pbit_mg_transport reports the one
 * used): "peer" (default) -- every rank maps the others' device memory through CUDA IPC:
 * the walk reads remote nodes with peer loads, the key-range partition and the relink
 * routing store straight into the destination rank's memory, NCCL carries only small
 * collectives; "hybrid" -- the same with a kn replica (ncclAllGather) walked locally;
 * "nccl" -- replica + ncclSend/ncclRecv.  Every transport gives the same bytes.  If a rank
 * cannot map the others, the ranks agree on it and the call runs on "nccl".  The peer
 * windows (cudaMalloc; ~56 B per node of the slice for 32-bit keys, mostly segment slots) are kept per
 * communicator and freed by pbit_mg_comm_destroy / pbit_mg_comm_abort.
 */
int pbit_sort_list_mg(const void *keys_local, const uint32_t *next_local, uint32_t head,
                      uint64_t n_global, uint64_t node_lo, uint64_t n_local, int key_bits,
                      uint32_t *out_head, uint32_t *out_next_local, void *nccl_comm,
                      const pbit_opts *opts);

/* NCCL communicator helpers for callers that do not link NCCL themselves.  The
 * unique id (PBIT_MG_UNIQUE_ID_BYTES opaque bytes) is created on rank 0 and shared
 * by the caller (e.g. torch.distributed.broadcast_object_list). */
#define PBIT_MG_UNIQUE_ID_BYTES 128
int pbit_mg_get_unique_id(void *id_out /* PBIT_MG_UNIQUE_ID_BYTES host bytes */);
int pbit_mg_comm_init(void **comm_out, int nranks, const void *id, int rank);
int pbit_mg_comm_destroy(void *comm);
/* After pbit_sort_list_mg returned PBIT_ERR_NCCL (an asynchronous NCCL error, or no
 * progress for PBIT_MG_TIMEOUT_S seconds, default 300): abort the communicator, which also
 * ends its pending collectives on the call's stream.  The communicator is then unusable. */
int pbit_mg_comm_abort(void *comm);

/* The transport pbit_sort_list_mg used on this communicator in its last call: 0 = peer
 * (N4: every rank maps the others' windows through CUDA IPC; the walk reads remote nodes
 * with peer loads and the exchanges are stores into the destination's memory), 2 = hybrid
 * (PBIT_MG_TRANSPORT=hybrid: the peer transport with a kn replica by ncclAllGather walked
 * locally), 1 = NCCL (kn replica + ncclSend/ncclRecv; PBIT_MG_TRANSPORT=nccl forces it; also
 * the fallback when
 * a rank cannot map the others, or when the peer transport's per-rank table of cut
 * segments overflows).  -1 for a NULL communicator or one without a call yet. */
int pbit_mg_transport(void *comm);

/* The ruling set pbit_sort_list_mg uses for n nodes on nranks ranks: the ruler spacing (a
 * power of two <= 64, which divides every rank's id slice) and the ruler blocks per rank;
 * nranks * blocks * spacing >= n.  PBIT_ERR_UNSUPPORTED if the slices cannot be tiled (n
 * beyond 32-bit ids).  Host only; exported for tests. */
int pbit_mg_ruler_blocks(uint64_t n, int nranks, uint32_t *spacing, uint32_t *blocks_per_rank);

/* Node ids per rank for pbit_sort_list_mg: ceil(n_global / nranks) rounded up to 64. */
uint64_t pbit_mg_slice(uint64_t n_global, int nranks);

/* Host-side plan of the key-range exchange inside pbit_sort_list_mg (no device work;
 * exported for tests).  Each rank's chunk (sorted positions [q*slice, (q+1)*slice) of the
 * list order) is sorted by (key, list position); splitter s sits at global rank
 * min(n, (s+1)*slice) of the final order with key k*_s.  lt / le: nranks x (nranks-1)
 * counts, lt[q*(nranks-1)+s] = keys of rank q below k*_s, le[...] = keys up to k*_s.
 * Outputs (nranks each): the range of its sorted chunk rank `rank` sends to every rank,
 * and where (offset, count) it receives each source's range, in source-rank order. */
void pbit_mg_exchange_plan(int nranks, int rank, uint64_t n, uint64_t slice, const uint64_t *lt,
                           const uint64_t *le, uint64_t *send_off, uint64_t *send_count,
                           uint64_t *recv_off, uint64_t *recv_count);

/* Workspace.  Every call takes its workspace (about 60 B per node for 32-bit keys) from
 * the library's own stream-ordered memory pool on the current device and returns it at
 * the end of the call; the pool releases it to the device when the call's stream
 * synchronizes (release threshold 0) unless PBIT_POOL_KEEP_GB=x asks it to keep up to x GB
 * mapped between calls (repeated calls then skip the re-mapping).
 * pbit_workspace_trim synchronizes the current device and releases cached workspace
 * above keep_bytes (0 = all of it).  Returns PBIT_OK or PBIT_ERR_CUDA. */
int pbit_workspace_trim(uint64_t keep_bytes);

/* In-warp ranking of the radix passes on the current device, decided by a self-test of
 * the lane order of conflicting shared-memory atomics that runs once per device before
 * its first sort (the order is measured on sm_100a, not documented): 2 = lane-ordered
 * atomics (the default), 0 = ballot peer masks (the fallback if the test ever fails),
 * 1 = match.any; PBIT_RANK overrides.  -1 on a CUDA error. */
int pbit_rank_mode(void);

/* Text of the last CUDA or NCCL error seen by the calling host thread ("" if none). */
const char *pbit_last_error(void);

/* Human-readable name of a status code (static string). */
const char *pbit_status_string(int status);

/* Library version, (major << 16) | (minor << 8) | patch. */
uint32_t pbit_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PBIT_H_ */
