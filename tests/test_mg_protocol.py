"""The multi-GPU protocol of pbit_sort_list_mg, simulated with world_size 2 and 3 over
torch.distributed gloo on CPU (no GPU here; NCCL cannot put two ranks on one GPU).

Each rank follows the steps of paper_cs_0511020_b200/csrc/mg.cu with numpy standing in
for the device kernels, and the product's own host-side exchange planner
(`pbit_mg_exchange_plan`, `pbit_mg_slice` from libpbit.so) deciding what moves where:
  1 own id slice -> replica (all_gather)         4 chunk of own list positions
  5 exact splitters (8-bit radix refinement rounds over all_reduced histograms), one
    stable partition by splitter bucket, per-rank counts (all_gather), the planner,
    point-to-point exchange, receive buffers concatenated in source-rank order
  6 stable local sort                              7 stitch (all_gather of first and last ids),
    (v, succ) and (v, pred) routed to the owner of v, applied to the owner's out_next /
    out_prev slices.
The assembled out_next must equal the paper-literal oracle bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NULL = 0xFFFFFFFF


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(arrays_out, counts_out, counts_in, rank, G, dtype):
    """Point-to-point all-to-allv: arrays_out[d] goes to rank d; returns the received
    arrays from every source in source-rank order."""
    reqs, bufs = [], []
    for d in range(G):
        if d == rank:
            continue
        if counts_out[d]:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arrays_out[d])), dst=d))
    for q in range(G):
        if q == rank:
            bufs.append(np.ascontiguousarray(arrays_out[rank]))
            continue
        t = torch.empty(int(counts_in[q]), dtype=dtype)
        if counts_in[q]:
            reqs.append(dist.irecv(t, src=q))
        bufs.append(t)
    for rq in reqs:
        rq.wait()
    return [b if isinstance(b, np.ndarray) else b.numpy() for b in bufs]


def _rank_main(rank, G, port, n, key_bits, seed, keys_kind, links, K, out_q):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=G)
    import paper_cs_0511020_b200 as pbit
    import workloads
    try:
        li = workloads.make_list(n, key_bits, seed, keys=keys_kind, links=links)
        keys_all = workloads.keys_numpy(li)
        next_all = workloads.next_numpy(li)
        S = pbit.mg_slice(n, G)
        lo = min(n, rank * S)
        hi = min(n, lo + S)
        keys_local, next_local = keys_all[lo:hi].copy(), next_all[lo:hi].copy()
        kdt = keys_local.dtype
        # ---- 1. replica of (key, next) by all_gather of padded slices
        pad = np.zeros(S, kdt)
        pad[: hi - lo] = keys_local
        padn = np.full(S, NULL, np.uint32)
        padn[: hi - lo] = next_local
        # keys travel as int64 bit patterns (gloo has no 8/16-bit or unsigned types)
        def to64(a):
            return a.view(np.int64) if kdt == np.uint64 else a.astype(np.int64)

        def from64(a):
            return a.view(np.uint64) if kdt == np.uint64 else a.astype(kdt)
        tk = [torch.empty(S, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(tk, torch.from_numpy(to64(pad)))
        tn = [torch.empty(S, dtype=torch.int32) for _ in range(G)]
        dist.all_gather(tn, torch.from_numpy(padn.view(np.int32)))
        key_rep = from64(np.concatenate([t.numpy() for t in tk]))[:n]
        next_rep = np.concatenate([t.numpy().view(np.uint32) for t in tn])[:n]
        # ---- 2-4. list order (the device ranks it with the ruling set) and own chunk
        order = np.empty(n, np.int64)
        v = li.head
        for p_ in range(n):
            order[p_] = v
            v = int(next_rep[v])
        assert v == NULL
        ids = order[lo:hi].astype(np.uint32)
        ck = key_rep[ids]
        # ---- 5. top non-trivial digit from the global histograms
        M = key_bits
        D = (M + K - 1) // K
        radix = 1 << K
        mask = np.uint64(radix - 1)
        hist_local = np.stack([np.bincount(((keys_local.astype(np.uint64) >> np.uint64(d * K)) & mask).astype(np.int64),
                                           minlength=radix) for d in range(D)]).astype(np.int64)
        th = torch.from_numpy(hist_local)
        dist.all_reduce(th)
        hist = th.numpy()
        nontrivial = [d for d in range(D) if hist[d].max() != n]
        if nontrivial:
            ck64 = ck.astype(np.uint64)
            # 5a. splitters by radix refinement, 8 bits per round from the top: histograms of
            # the next digit among the keys matching each splitter's prefix, summed over the
            # ranks (all_reduce); each prefix takes the largest digit c with
            # below + #(prefix, digit < c) <= x_s (k_split_count / k_split_select)
            NS = G - 1
            prefix = [0] * NS
            below = [0] * NS
            for i in range(key_bits // 8 - 1, -1, -1):
                top = ck64 >> np.uint64(8 * i + 8) if 8 * i + 8 < 64 else np.zeros_like(ck64)
                dig = ((ck64 >> np.uint64(8 * i)) & np.uint64(255)).astype(np.int64)
                h = np.stack([np.bincount(dig[top == np.uint64(prefix[sp])], minlength=256) for sp in range(NS)]) \
                    if NS else np.zeros((0, 256), np.int64)
                th = torch.from_numpy(h.astype(np.int64))
                dist.all_reduce(th)
                h = th.numpy()
                for sp in range(NS):
                    x = min(n, (sp + 1) * S)
                    cum = np.concatenate([[0], np.cumsum(h[sp])])[:256]
                    pick = max(c for c in range(256) if below[sp] + cum[c] <= x)
                    below[sp] += int(cum[pick])
                    prefix[sp] = (prefix[sp] << 8) | pick
            # 5b. ONE stable partition by splitter bucket (2j + [key == k*_j]): key ranges in
            # order, list order inside each bucket (the SRC_SPLIT pass)
            kst = np.array(prefix, dtype=np.uint64)
            jj = np.searchsorted(kst, ck64, side="left")
            eq = (jj < NS) & (kst[np.minimum(jj, max(NS - 1, 0))] == ck64) if NS else np.zeros(len(ck64), bool)
            perm = np.argsort(2 * jj + eq, kind="stable")
            ck, ids = ck[perm], ids[perm]
            # 5c. per-rank counts below / up to each splitter; the product's planner
            mine = np.concatenate([(ck64[:, None] < kst[None, :]).sum(0),
                                   (ck64[:, None] <= kst[None, :]).sum(0)]).astype(np.int64) \
                if NS else np.zeros(0, np.int64)
            allm = [torch.empty(2 * NS, dtype=torch.int64) for _ in range(G)]
            dist.all_gather(allm, torch.from_numpy(mine))
            lt = np.stack([t_.numpy()[:NS] for t_ in allm])
            le = np.stack([t_.numpy()[NS:] for t_ in allm])
            soff, scnt, roff, rcnt = pbit.mg_exchange_plan(G, rank, n, S, lt, le)   # the product's planner
            assert int(rcnt.sum()) == hi - lo
            kk = [to64(ck[soff[d]: soff[d] + scnt[d]]) for d in range(G)]
            ii = [ids[soff[d]: soff[d] + scnt[d]].view(np.int32) for d in range(G)]
            rk = _exchange(kk, scnt, rcnt, rank, G, torch.int64)
            ri = _exchange(ii, scnt, rcnt, rank, G, torch.int32)
            ck = from64(np.concatenate(rk))
            ids = np.concatenate([x.view(np.uint32) for x in ri])
            # 6. stable sort of the received runs (source order = position order for ties)
            perm = np.argsort(ck, kind="stable")
            ck, ids = ck[perm], ids[perm]
        # ---- 7. stitch (all_gather of every rank's first and last sorted id) and route
        # (v, succ) -- and (v, pred) for out_prev -- to the owner of v
        fl = torch.tensor([int(ids[0]) if len(ids) else NULL, int(ids[-1]) if len(ids) else NULL],
                          dtype=torch.int64)
        fls = [torch.empty(2, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(fls, fl)
        firsts = [int(f[0]) for f in fls]
        lasts = [int(f[1]) for f in fls]
        nxt = next((firsts[d] for d in range(rank + 1, G) if firsts[d] != NULL), NULL)
        prv = next((lasts[d] for d in range(rank - 1, -1, -1) if lasts[d] != NULL), NULL)
        succ = np.empty(len(ids), np.uint32)
        pred = np.empty(len(ids), np.uint32)
        if len(ids):
            succ[:-1] = ids[1:]
            succ[-1] = nxt
            pred[1:] = ids[:-1]
            pred[0] = prv
        owner = (ids // S).astype(np.int64) if len(ids) else np.zeros(0, np.int64)
        cnt_out = np.bincount(owner, minlength=G)
        tc = torch.from_numpy(cnt_out.astype(np.int64))
        allc = [torch.empty(G, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(allc, tc)
        cnt_in = np.array([int(allc[q][rank]) for q in range(G)])
        vv = [ids[owner == d].view(np.int32) for d in range(G)]
        rv = np.concatenate([x.view(np.uint32) for x in _exchange(vv, cnt_out, cnt_in, rank, G, torch.int32)])
        assert len(rv) == hi - lo
        full = []
        for w_ in (succ, pred):
            ss = [w_[owner == d].view(np.int32) for d in range(G)]
            rs = np.concatenate([x.view(np.uint32) for x in _exchange(ss, cnt_out, cnt_in, rank, G, torch.int32)])
            out_local = np.full(S, NULL, np.uint32)
            out_local[rv - lo] = rs
            outs = [torch.empty(S, dtype=torch.int32) for _ in range(G)]
            dist.all_gather(outs, torch.from_numpy(out_local.view(np.int32)))
            full.append(np.concatenate([o.numpy().view(np.uint32) for o in outs])[:n])
        if rank == 0:
            out_q.put(("ok", firsts[0], (full[0], full[1])))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        out_q.put(("error", traceback.format_exc(), None))
        raise
    finally:
        dist.destroy_process_group()


def _run(G, n, key_bits, seed, keys_kind="uniform", links="random", K=8):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, G, port, n, key_bits, seed, keys_kind, links, K, q))
             for r in range(G)]
    for p_ in procs:
        p_.start()
    status, head, out_next = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=120)
    assert status == "ok", head
    return head, out_next


@pytest.mark.parametrize("G,n,key_bits,keys_kind,links,K", [
    (2, 5000, 32, "uniform", "random", 8),
    (2, 4099, 32, "zipf", "random", 8),
    (3, 7001, 16, "uniform", "push", 4),
    (3, 3000, 64, "runs4096", "random", 8),
    (2, 2500, 32, "uniform", "random", 8),
    (2, 1000, 32, "equal", "random", 8),
    (3, 130, 8, "uniform", "identity", 4),
    (4, 6007, 32, "zipf", "random", 8),
    (4, 2048, 16, "equal", "push", 8),
])
def test_mg_protocol_matches_oracle(G, n, key_bits, keys_kind, links, K):
    import oracle
    import workloads
    head, (out_next, out_prev) = _run(G, n, key_bits, seed=n + G, keys_kind=keys_kind, links=links, K=K)
    li = workloads.make_list(n, key_bits, n + G, keys=keys_kind, links=links)
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, key_bits, 4)
    assert head == oh
    assert np.array_equal(out_next, on)
    assert np.array_equal(out_prev, oracle.repair_back(on, oh))  # N2 across ranks


def test_exchange_plan_is_position_exact():
    """Every rank receives exactly its slice of the final order, what rank r sends to d is
    what d expects from r, send ranges are contiguous, and ties on a splitter key are
    taken in rank (= list position) order."""
    import paper_cs_0511020_b200 as pbit
    rng = np.random.default_rng(0)
    for G in (2, 3, 5, 8):
        n = int(rng.integers(G * 50, G * 400))
        S = pbit.mg_slice(n, G)
        sizes = [max(0, min(n, (q + 1) * S) - min(n, q * S)) for q in range(G)]
        keys = [np.sort(rng.integers(0, 20, size=sz)) for sz in sizes]   # heavy ties
        allk = np.concatenate(keys)
        order = np.argsort(allk, kind="stable")                           # final order
        lt = np.zeros((G, G - 1), np.int64)
        le = np.zeros((G, G - 1), np.int64)
        for sp in range(G - 1):
            x = min(n, (sp + 1) * S)
            kstar = allk[order[x]] if x < n else allk.max() + 1
            for q in range(G):
                lt[q, sp] = np.searchsorted(keys[q], kstar, "left")
                le[q, sp] = np.searchsorted(keys[q], kstar, "right")
        plans = [pbit.mg_exchange_plan(G, r, n, S, lt, le) for r in range(G)]
        owner = np.repeat(np.arange(G), sizes)
        for r in range(G):
            soff, scnt, roff, rcnt = plans[r]
            assert int(rcnt.sum()) == sizes[r]
            assert int(scnt.sum()) == sizes[r]
            for d in range(G):
                assert scnt[d] == plans[d][3][r]
                if d + 1 < G:
                    assert soff[d] + scnt[d] == soff[d + 1]
            # rank r's received elements are exactly final positions [r*S, r*S + size_r)
            got = sorted(int(plans[q][0][r]) + j + int(sum(sizes[:q])) for q in range(G)
                         for j in range(int(plans[q][1][r])))
            want = sorted(int(i) for i in order[r * S: r * S + sizes[r]])
            assert got == want
