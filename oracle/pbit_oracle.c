/*
 * oracle/pbit_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of Pbit exactly as the paper
 * (arXiv cs/0511020, /root/reference/PAPER.md, cited "P:<line>") defines it, on
 * node arrays instead of pointers.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_cs_0511020_b200/csrc); neither includes nor links the other.
 *
 * Representation (reading Q9 in DESIGN.md): a node is an index v in [0, n);
 * the paper's `L->next` is next[v] (u32) and its NULL (P:8) is 0xFFFFFFFF;
 * the paper's `L->data` is key[v], an unsigned M-bit integer (M = 8/16/32/64).
 *
 * Every function cites the passage it follows.  Pinned by tests/test_oracle.py
 * against: the worked example (tests/golden/), bits(123,3)=15
 * (P:179-182), brute force over all link orders for n <= 6 (a stable sort of
 * the list-order sequence), seeded random lists vs numpy's stable argsort, the
 * counter identities relinks = n*M/K and merge visits = n,
 * the depth/live-table bound M/K with the memory formula T,
 * direction duality and the reverse-stability of odd M/K (Q1).
 * Nothing here is "parity unpinned".
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_NULL 0xFFFFFFFFu

enum { ORACLE_OK = 0, ORACLE_ERR_ARG = 1, ORACLE_ERR_LIST = 2, ORACLE_ERR_OOM = 3 };

/* Operation counters (SPEC metrics module).  Filled when non-NULL. */
typedef struct {
    uint64_t relinks;        /* +1 per node pushed into tab[] by the split loop   */
    uint64_t merge_visits;   /* +1 per node walked inside merge, exactly as the listing P:310-320 */
    uint32_t max_depth;      /* deepest active Pbit call (levels), <= M/K                        */
    uint32_t max_live_tabs;  /* most root tables tab[Omega] alive at once, <= M/K        */
    uint64_t bucket_scans;   /* tab slots visited by the loops of listing lines 8-9  */
} oracle_counters;

typedef struct {
    const uint8_t *key;      /* node-indexed keys, key_bytes each, little-endian host order   */
    int key_bytes;
    uint32_t *next;          /* the list being relinked in place                      */
    unsigned K;              /* pattern length                                      */
    uint32_t omega;          /* Omega = 2^K                                            */
    int descending;          /* 0: ascending loops P:379-380; 1: descending loops P:371-372    */
    unsigned fshift;         /* the sorted field: (key >> fshift) & fmask (0 / all ones for a  */
    uint64_t fmask;          /*   whole integer key; the mantissa or characteristic)  */
    uint32_t *tabs;          /* (M/K) root tables of Omega slots, one per recursion level     */
    uint32_t depth, live;
    oracle_counters c;
} ctx_t;

/* The key of node v as an unsigned integer (the paper's L->data), restricted to
 * the field being sorted (the whole key unless a float field is sorted). */
static uint64_t key_of(const ctx_t *x, uint32_t v) {
    const uint8_t *p = x->key + (size_t)v * (size_t)x->key_bytes;
    uint64_t k;
    switch (x->key_bytes) {
    case 1: k = p[0]; break;
    case 2: { uint16_t t; memcpy(&t, p, 2); k = t; break; }
    case 4: { uint32_t t; memcpy(&t, p, 4); k = t; break; }
    default: { uint64_t t; memcpy(&t, p, 8); k = t; break; }
    }
    return (k >> x->fshift) & x->fmask;
}

/* bits(number, M) = (number div 2^M) mod Omega, written in C as
 * (number >> M) & (Omega - 1). */
uint64_t oracle_bits(uint64_t number, unsigned M, unsigned K) {
    uint64_t omega = (uint64_t)1 << K;
    return (number >> M) & (omega - 1);
}

/* merge(A, B): splice list B behind the tail of list A; return the head.
 * Instrumented exactly as P:310-320: count the first node, then each advance. */
static uint32_t merge(ctx_t *x, uint32_t A, uint32_t B) {
    if (A == ORACLE_NULL) return B;               /* line 2: if(A==0) return B;     */
    x->c.merge_visits++;                          /* count++; first node (maybe only) */
    uint32_t temp = A;                            /* line 3                          */
    while (x->next[temp] != ORACLE_NULL) {        /* line 4: while(temp->next)       */
        temp = x->next[temp];
        x->c.merge_visits++;                      /* count++; n-node of list         */
    }
    x->next[temp] = B;                            /* line 5: temp->next = B          */
    return A;                                     /* line 6                          */
}

/* Pbit(L, M, P) -- the listing of P:346-361 with the loop direction of P:371-372
 * (descending) or P:379-380 (ascending).  `level` indexes the root table that the
 * listing declares as a local (`Node *tab[Omega]={NULL};`). */
static uint32_t Pbit(ctx_t *x, uint32_t L, unsigned M, uint32_t P, uint32_t level) {
    if (L != ORACLE_NULL) {                                       /* 2: if(L){          */
        M -= x->K;                                                /* 3: M-=K;           */
        uint32_t *tab = x->tabs + (size_t)level * x->omega;       /* 4: tab[Omega]={NULL} */
        for (uint32_t b = 0; b < x->omega; ++b) tab[b] = ORACLE_NULL;
        x->depth++; x->live++;
        if (x->depth > x->c.max_depth) x->c.max_depth = x->depth;
        if (x->live > x->c.max_live_tabs) x->c.max_live_tabs = x->live;

        /* 5: for(Node *i,**in; i=L; i->next=*in,*in=i){
         * 6:     in = tab + ((L->data>>M) & (Omega-1));
         * 7:     L = L->next; }
         * i.e. a push-front of every node into tab[digit]. */
        for (uint32_t i; (i = L) != ORACLE_NULL; ) {
            uint32_t *in = tab + oracle_bits(key_of(x, L), M, x->K); /* line 6 */
            L = x->next[L];                                          /* line 7 */
            x->next[i] = *in; *in = i;                               /* for-increment */
            x->c.relinks++;
        }

        if (M) {                                                  /* 8 */
            if (x->descending)
                for (uint32_t b = 0; b < x->omega; ++b) { x->c.bucket_scans++; P = Pbit(x, tab[b], M, P, level + 1); }
            else
                for (int64_t b = (int64_t)x->omega - 1; b >= 0; --b) { x->c.bucket_scans++; P = Pbit(x, tab[b], M, P, level + 1); }
        } else {                                                  /* 9 */
            if (x->descending)
                for (uint32_t b = 0; b < x->omega; ++b) { x->c.bucket_scans++; P = merge(x, tab[b], P); }
            else
                for (int64_t b = (int64_t)x->omega - 1; b >= 0; --b) { x->c.bucket_scans++; P = merge(x, tab[b], P); }
        }
        x->depth--; x->live--;
    }
    return P;                                                     /* 10: return P; */
}

/* The paper assumes a well-formed list (P:8: the last pointer shows NULL).  The
 * oracle rejects anything else before mutating (reading Q10): starting at head it
 * must reach NULL after exactly n nodes, every index < n.  Reaching NULL after
 * exactly n steps implies the n visited nodes are distinct (a repeat never ends). */
int oracle_validate_list(const uint32_t *next, uint32_t head, uint64_t n) {
    if (n == 0) return head == ORACLE_NULL ? ORACLE_OK : ORACLE_ERR_LIST;
    uint64_t steps = 0;
    uint32_t v = head;
    while (v != ORACLE_NULL) {
        if ((uint64_t)v >= n || steps >= n) return ORACLE_ERR_LIST;
        ++steps;
        v = next[v];
    }
    return steps == n ? ORACLE_OK : ORACLE_ERR_LIST;
}

/* The list order: order[i] = v_i with v_0 = head, v_{i+1} = next[v_i] -- the traversal
 * `L = L->next` of the split loop down to the NULL of the last node (P:8).  Used
 * by the checkers to read a sorted list (e.g. the payload sequence of C4, reading Q11).
 * The list must be valid (oracle_validate_list), else ORACLE_ERR_LIST. */
int oracle_list_order(const uint32_t *next, uint32_t head, uint64_t n, uint32_t *order) {
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;
    uint32_t v = head;
    for (uint64_t i = 0; i < n; ++i) { order[i] = v; v = next[v]; }
    return ORACLE_OK;
}

/* Sort the list (head, next[]) of n nodes by its M = key_bits unsigned keys with
 * pattern length K; the result goes to (*out_head, out_next[]).  out_next may
 * alias next.  Unsigned entry of the dispatcher P:444-466 (lines 14-15):
 * size = sizeof(data)<<3, then Pbit_ascending / Pbit_decreasing. */
int oracle_pbit_sort(const void *keys, int key_bits, const uint32_t *next, uint32_t head,
                     uint64_t n, unsigned K, int descending,
                     uint32_t *out_head, uint32_t *out_next, oracle_counters *counters) {
    if (!out_head || (n && (!keys || !next || !out_next))) return ORACLE_ERR_ARG;
    if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return ORACLE_ERR_ARG;
    if (K < 1 || K > 16 || (key_bits % K) != 0) return ORACLE_ERR_ARG;   /* reading Q7 */
    if (n > 0xFFFFFFFFull) return ORACLE_ERR_ARG;
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;

    ctx_t x;
    memset(&x, 0, sizeof x);
    x.key = (const uint8_t *)keys;
    x.key_bytes = key_bits / 8;
    x.K = K;
    x.omega = 1u << K;
    x.descending = descending;
    x.fshift = 0;
    x.fmask = ~(uint64_t)0;
    unsigned levels = (unsigned)key_bits / K;
    x.tabs = (uint32_t *)malloc((size_t)levels * x.omega * sizeof(uint32_t));
    if (!x.tabs) return ORACLE_ERR_OOM;
    if (out_next != next && n) memcpy(out_next, next, (size_t)n * sizeof(uint32_t));
    x.next = out_next;

    *out_head = Pbit(&x, head, (unsigned)key_bits, ORACLE_NULL, 0);

    free(x.tabs);
    if (counters) *counters = x.c;
    return ORACLE_OK;
}

/* ---------------------------------------------------------------- subtree-parallel baseline
 * The same sort on several host threads (an optional CPU baseline on nproc
 * threads whose output must be bit-identical).  The first two levels of the recursion run
 * exactly as Pbit runs them -- the split loop of P:351-353 at M-K, then at M-2K on every
 * bucket -- which leaves Omega^2 independent sublists, in list order (b1, b2) ascending
 * (the ascending loops of P:379-380 put bucket 0 first).  Each sublist's own recursion
 * Pbit(L, M-2K, NULL) runs on one of the threads: Pbit(L, M, P) is Pbit(L, M, NULL)
 * followed by P (the end marker is only ever spliced behind the last node), so
 * linking every sorted sublist's tail to the next one's head reproduces the serial result
 * node for node.  Ascending unsigned keys only (the cpu_baseline's sort). */
typedef struct {
    const ctx_t *proto;      /* keys, K, omega, next */
    unsigned M2;             /* bits left below the first two levels */
    const uint32_t *tab1;    /* the level-1 buckets */
    uint32_t *lists;         /* Omega^2 sublist heads (level-2 buckets) */
    uint32_t *heads, *tails; /* per sublist: sorted head and tail */
    int phase;               /* 0: split the level-1 buckets; 1: sort the sublists */
    uint32_t njobs;
    uint32_t next_job;       /* shared job counter */
    pthread_mutex_t mu;
    int oom;
} par_t;

static void *par_worker(void *arg) {
    par_t *w = (par_t *)arg;
    ctx_t x = *w->proto;
    memset(&x.c, 0, sizeof x.c);
    x.depth = x.live = 0;
    unsigned levels = w->M2 / x.K + 1;
    x.tabs = (uint32_t *)malloc((size_t)levels * x.omega * sizeof(uint32_t));
    for (;;) {
        pthread_mutex_lock(&w->mu);
        uint32_t j = w->next_job++;
        if (!x.tabs) w->oom = 1;
        pthread_mutex_unlock(&w->mu);
        if (j >= w->njobs || !x.tabs) break;
        if (w->phase == 0) {  /* level 2: the split loop on level-1 bucket j, M2 = M - 2K */
            uint32_t *tab2 = w->lists + (size_t)j * x.omega;
            for (uint32_t b = 0; b < x.omega; ++b) tab2[b] = ORACLE_NULL;
            for (uint32_t i, L = w->tab1[j]; (i = L) != ORACLE_NULL; ) {
                uint32_t *in = tab2 + oracle_bits(key_of(&x, L), w->M2, x.K);
                L = x.next[L];
                x.next[i] = *in; *in = i;
            }
            continue;
        }
        uint32_t L = w->lists[j];
        uint32_t h = (w->M2 && L != ORACLE_NULL) ? Pbit(&x, L, w->M2, ORACLE_NULL, 0) : L;
        uint32_t t = h;
        if (t != ORACLE_NULL)
            while (x.next[t] != ORACLE_NULL) t = x.next[t];
        w->heads[j] = h;
        w->tails[j] = t;
    }
    free(x.tabs);
    return NULL;
}

static int par_run(par_t *w, pthread_t *th, int nthreads) {
    w->next_job = 0;
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, par_worker, w) == 0) ++started;
    if (!started) par_worker(w);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    return w->oom ? ORACLE_ERR_OOM : ORACLE_OK;
}

int oracle_pbit_sort_par(const void *keys, int key_bits, const uint32_t *next, uint32_t head, uint64_t n,
                         unsigned K, int nthreads, uint32_t *out_head, uint32_t *out_next) {
    if (!out_head || (n && (!keys || !next || !out_next))) return ORACLE_ERR_ARG;
    if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return ORACLE_ERR_ARG;
    if (K < 1 || K > 8 || (key_bits % K) != 0 || (unsigned)key_bits < 2 * K) return ORACLE_ERR_ARG;
    if (n > 0xFFFFFFFFull) return ORACLE_ERR_ARG;
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    ctx_t x;
    memset(&x, 0, sizeof x);
    x.key = (const uint8_t *)keys;
    x.key_bytes = key_bits / 8;
    x.K = K;
    x.omega = 1u << K;
    x.fmask = ~(uint64_t)0;
    if (out_next != next && n) memcpy(out_next, next, (size_t)n * sizeof(uint32_t));
    x.next = out_next;
    const uint32_t om = x.omega, nj = om * om;
    uint32_t *tab1 = (uint32_t *)malloc(sizeof(uint32_t) * om);
    uint32_t *lists = (uint32_t *)malloc(sizeof(uint32_t) * nj);
    uint32_t *heads = (uint32_t *)malloc(sizeof(uint32_t) * nj);
    uint32_t *tails = (uint32_t *)malloc(sizeof(uint32_t) * nj);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    if (!tab1 || !lists || !heads || !tails || !th) { rc = ORACLE_ERR_OOM; goto out; }
    {
        /* level 1: the split loop on the whole list, M1 = M - K */
        const unsigned M1 = (unsigned)key_bits - K, M2 = M1 - K;
        for (uint32_t b = 0; b < om; ++b) tab1[b] = ORACLE_NULL;
        for (uint32_t i, L = head; (i = L) != ORACLE_NULL; ) {
            uint32_t *in = tab1 + oracle_bits(key_of(&x, L), M1, K);
            L = x.next[L];
            x.next[i] = *in; *in = i;
        }
        /* level 2 (the same split on every level-1 bucket, M2 = M - 2K), then the
         * independent sublists, both on the threads */
        par_t w;
        memset(&w, 0, sizeof w);
        w.proto = &x; w.M2 = M2; w.tab1 = tab1; w.lists = lists; w.heads = heads; w.tails = tails;
        pthread_mutex_init(&w.mu, NULL);
        w.phase = 0; w.njobs = om;
        rc = par_run(&w, th, nthreads);
        if (!rc) { w.phase = 1; w.njobs = nj; rc = par_run(&w, th, nthreads); }
        pthread_mutex_destroy(&w.mu);
        if (rc) goto out;
        /* concatenate in list order: every sorted sublist's tail -> the next one's head */
        uint32_t first = ORACLE_NULL, prev_tail = ORACLE_NULL;
        for (uint32_t j = 0; j < nj; ++j) {
            if (heads[j] == ORACLE_NULL) continue;
            if (prev_tail == ORACLE_NULL) first = heads[j]; else x.next[prev_tail] = heads[j];
            prev_tail = tails[j];
        }
        *out_head = first;
    }
out:
    free(tab1); free(lists); free(heads); free(tails); free(th);
    return rc;
}

/* ---------------------------------------------------------------- key kinds
 * kind 0: unsigned (above).  kind 1: signed two's complement integers, the dispatcher of
 * P:444-466.  kind 2: IEEE 754 floats (binary16/32/64 by key_bits).
 *
 * Reading Q13: the dispatcher's sign split pushes nodes to the
 * FRONT of L_negative / L_unsigned, which reverses equal keys once more than the even
 * number of Pbit levels restores, so the literal listing is reverse-stable.  The oracle
 * splits by appending at the tails instead (SPEC S:201 makes the same decision); the
 * split itself is otherwise the listing's (temp->data < 0 <=> sign bit set).
 *
 * Reading Q18: floats.  The paper sorts "in relation to mantissa first, and then once
 * more in relation to its characteristic. Such sorting is correct because Pbit is
 * stable" with the IEEE layouts of P:1196-1199, and says nothing about the
 * sign.  The oracle splits by the sign bit as the integer dispatcher does, sorts the
 * non-negative list by mantissa then by characteristic (ascending), and the negative
 * list by mantissa then characteristic in the descending direction (larger magnitude =
 * smaller number), negatives first.  Each field is padded to a multiple of 2K bits so
 * that M/K is even (reading Q1).  The resulting order is sign-magnitude order of the
 * bit patterns: -0.0 before +0.0, NaNs outside the infinities (IEEE 754 totalOrder). */

/* Append every node of the list (head, next) to the tail of one of two lists by the sign
 * bit of its key; returns the two heads (order inside each list = input order). */
static void split_sign(ctx_t *x, uint32_t head, int sign_bit, uint32_t *neg, uint32_t *nonneg) {
    uint32_t nh = ORACLE_NULL, nt = ORACLE_NULL, ph = ORACLE_NULL, pt = ORACLE_NULL;
    unsigned fs = x->fshift; uint64_t fm = x->fmask;
    x->fshift = 0; x->fmask = ~(uint64_t)0;
    for (uint32_t temp; (temp = head) != ORACLE_NULL; ) {
        head = x->next[head];
        x->next[temp] = ORACLE_NULL;
        if ((key_of(x, temp) >> sign_bit) & 1u) {                    /* temp->data < 0 */
            if (nt == ORACLE_NULL) nh = temp; else x->next[nt] = temp;
            nt = temp;
        } else {
            if (pt == ORACLE_NULL) ph = temp; else x->next[pt] = temp;
            pt = temp;
        }
    }
    x->fshift = fs; x->fmask = fm;
    *neg = nh; *nonneg = ph;
}

/* Pbit over one field of the keys: sorts the list L by (key >> shift) & (2^width - 1),
 * padded to M = a multiple of 2K bits, in the given direction, in front of end marker P. */
static uint32_t pbit_field(ctx_t *x, uint32_t L, unsigned shift, unsigned width, int desc, uint32_t P) {
    unsigned M = (width + 2 * x->K - 1) / (2 * x->K) * (2 * x->K);
    x->fshift = shift;
    x->fmask = width >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << width) - 1);
    x->descending = desc;
    return Pbit(x, L, M, P, 0);
}

int oracle_pbit_sort_kind(const void *keys, int key_bits, const uint32_t *next, uint32_t head,
                          uint64_t n, unsigned K, int kind, int descending,
                          uint32_t *out_head, uint32_t *out_next, oracle_counters *counters) {
    if (kind == 0)
        return oracle_pbit_sort(keys, key_bits, next, head, n, K, descending, out_head, out_next, counters);
    if (!out_head || (n && (!keys || !next || !out_next))) return ORACLE_ERR_ARG;
    if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return ORACLE_ERR_ARG;
    if (K < 1 || K > 16 || kind < 0 || kind > 2) return ORACLE_ERR_ARG;
    if (kind == 1 && (key_bits % K) != 0) return ORACLE_ERR_ARG;        /* reading Q7 */
    if (kind == 2 && key_bits == 8) return ORACLE_ERR_ARG;              /* no 8-bit IEEE format */
    if (n > 0xFFFFFFFFull) return ORACLE_ERR_ARG;
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;

    ctx_t x;
    memset(&x, 0, sizeof x);
    x.key = (const uint8_t *)keys;
    x.key_bytes = key_bits / 8;
    x.K = K;
    x.omega = 1u << K;
    x.fmask = ~(uint64_t)0;
    unsigned levels = ((unsigned)key_bits + 2 * K - 1) / K + 2;
    x.tabs = (uint32_t *)malloc((size_t)levels * x.omega * sizeof(uint32_t));
    if (!x.tabs) return ORACLE_ERR_OOM;
    if (out_next != next && n) memcpy(out_next, next, (size_t)n * sizeof(uint32_t));
    x.next = out_next;
    const int sign_bit = key_bits - 1;
    uint32_t neg, nonneg;
    split_sign(&x, head, sign_bit, &neg, &nonneg);                     /* P:450-455 (tail append) */
    const unsigned size = (unsigned)key_bits;
    if (kind == 1) {
        if (descending)   /* Pbit_decreasing(L_unsigned, size, Pbit_decreasing(L_negative, size)) */
            *out_head = pbit_field(&x, nonneg, 0, size, 1, pbit_field(&x, neg, 0, size, 1, ORACLE_NULL));
        else              /* Pbit_ascending(L_negative, size, Pbit_ascending(L_unsigned, size)) */
            *out_head = pbit_field(&x, neg, 0, size, 0, pbit_field(&x, nonneg, 0, size, 0, ORACLE_NULL));
    } else {
        /* IEEE 754 layouts: mantissa m bits, characteristic c bits */
        const unsigned m = key_bits == 16 ? 10 : key_bits == 32 ? 23 : 52;
        const unsigned c = key_bits == 16 ? 5 : key_bits == 32 ? 8 : 11;
        /* "sort the number in relation to mantissa first, and then once more in relation
         * to its characteristic"; the sign list order: see reading Q18 above */
        const int d_nonneg = descending ? 1 : 0, d_neg = descending ? 0 : 1;
        uint32_t a = pbit_field(&x, nonneg, 0, m, d_nonneg, ORACLE_NULL);
        uint32_t b = pbit_field(&x, neg, 0, m, d_neg, ORACLE_NULL);
        if (descending) {   /* non-negatives (largest first), then negatives */
            uint32_t tail = pbit_field(&x, b, m, c, d_neg, ORACLE_NULL);
            *out_head = pbit_field(&x, a, m, c, d_nonneg, tail);
        } else {            /* negatives (most negative first), then non-negatives */
            uint32_t tail = pbit_field(&x, a, m, c, d_nonneg, ORACLE_NULL);
            *out_head = pbit_field(&x, b, m, c, d_neg, tail);
        }
    }
    free(x.tabs);
    if (counters) *counters = x.c;
    return ORACLE_OK;
}

/* The "reverse connection" repair of a doubly-linked list after Pbit:
 * "going through its elements it should set up pointer `back' in such a way as to show
 * the element right behind".  back[head] = NULL.  The list must be valid (Q10). */
int oracle_repair_back(const uint32_t *next, uint32_t head, uint64_t n, uint32_t *back) {
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;
    uint32_t behind = ORACLE_NULL;
    for (uint32_t v = head; v != ORACLE_NULL; v = next[v]) {
        back[v] = behind;
        behind = v;
    }
    return ORACLE_OK;
}

/* First split only (P:351-353 at the top level, M -= K once): fills tab[Omega] with
 * the bucket heads and relinks next[] in place.  Exposed so tests can pin the
 * worked example's first-level groups. */
int oracle_split_once(const void *keys, int key_bits, uint32_t *next, uint32_t head,
                      uint64_t n, unsigned K, uint32_t *tab) {
    if (key_bits != 8 && key_bits != 16 && key_bits != 32 && key_bits != 64) return ORACLE_ERR_ARG;
    if (K < 1 || K > 16 || (key_bits % K) != 0) return ORACLE_ERR_ARG;
    int rc = oracle_validate_list(next, head, n);
    if (rc) return rc;
    ctx_t x;
    memset(&x, 0, sizeof x);
    x.key = (const uint8_t *)keys; x.key_bytes = key_bits / 8; x.K = K; x.omega = 1u << K;
    x.fmask = ~(uint64_t)0;
    x.next = next;
    unsigned M = (unsigned)key_bits - K;
    for (uint32_t b = 0; b < x.omega; ++b) tab[b] = ORACLE_NULL;
    uint32_t L = head;
    for (uint32_t i; (i = L) != ORACLE_NULL; ) {
        uint32_t *in = tab + oracle_bits(key_of(&x, L), M, K);
        L = next[L];
        next[i] = *in; *in = i;
    }
    return ORACLE_OK;
}

/* The paper's memory formula T = (Omega*4 + 3*4) * M/K + 2*4 bytes. */
uint64_t oracle_memory_bound_T(unsigned M, unsigned K) {
    uint64_t omega = (uint64_t)1 << K;
    return (omega * 4 + 3 * 4) * (M / K) + 2 * 4;
}
