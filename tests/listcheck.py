"""Checkers used by the tests: the plain definition of the result and the invariants.

Plain definition: with v_0 = head, v_{i+1} = next[v_i],
sort the list-order sequence stably by unsigned key to w_0..w_{n-1}; then
out_head = w_0, out_next[w_i] = w_{i+1}, out_next[w_{n-1}] = NULL.  The stable
result is unique, so every correct sort returns exactly these arrays.
"""
from __future__ import annotations

import numpy as np

NULL = 0xFFFFFFFF


def walk(next_, head, limit=None):
    """List order of (head, next) as a python list (bounded walk)."""
    nx = np.asarray(next_, dtype=np.uint32)
    limit = len(nx) + 1 if limit is None else limit
    out, v = [], int(head)
    while v != NULL:
        out.append(v)
        if len(out) > limit:
            raise AssertionError("walk exceeded bound (cycle?)")
        v = int(nx[v])
    return out


def expected_by_definition_small(keys, next_, head):
    """Brute force with python's stable sorted() -- tiny inputs only."""
    seq = walk(next_, head)
    w = sorted(seq, key=lambda v: int(keys[v]))  # sorted() is stable
    return _links(w, len(next_))


def expected_by_definition(keys, order, descending=False):
    """Vectorised plain definition given the input list order (position -> node):
    a stable argsort (numpy kind='stable') of the list-order key sequence."""
    order = np.asarray(order, dtype=np.int64)
    k = np.asarray(keys)[order]
    if descending:
        # stable descending: reverse a stable ascending sort of the reversed sequence
        idx = np.argsort(k[::-1], kind="stable")[::-1]
        w = order[::-1][idx]
    else:
        w = order[np.argsort(k, kind="stable")]
    return _links(w, len(order))


def _links(w, n):
    out = np.full(n, NULL, dtype=np.uint32)
    w = np.asarray(w, dtype=np.int64)
    if n == 0:
        return NULL, out
    out[w[:-1]] = w[1:].astype(np.uint32)
    return int(w[0]), out


def check_sorted_list_properties(keys, order, out_head, out_next):
    """Properties that hold at any size and together force the unique stable answer:
    every edge v -> out_next[v] strictly increases (key, input rank); out_next has
    exactly one NULL; successors are distinct; out_head has no predecessor.  Strict
    increase forbids cycles, so the edges form one path over all n nodes, sorted and
    stable.  Vectorised (numpy); no walk needed."""
    order = np.asarray(order, dtype=np.int64)
    n = len(order)
    on = np.asarray(out_next, dtype=np.uint32)
    if n == 0:
        assert out_head == NULL
        return
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    keys = np.asarray(keys)
    is_null = on == NULL
    assert int(is_null.sum()) == 1, "exactly one NULL terminator"
    v = np.nonzero(~is_null)[0]
    s = on[~is_null].astype(np.int64)
    assert (s < n).all(), "successor out of range"
    cnt = np.bincount(s, minlength=n)
    assert (cnt <= 1).all(), "a node has two predecessors"
    assert 0 <= out_head < n and cnt[out_head] == 0, "head has a predecessor"
    kv, ks = keys[v], keys[s]
    ok = (kv < ks) | ((kv == ks) & (rank[v] < rank[s]))
    assert ok.all(), f"{int((~ok).sum())} edges break (key, input-rank) order"


# ----------------------------------------------------------------------------- torch (any device)
def unsigned_order_key(keys, key_bits):
    """int64 tensor whose signed order equals the unsigned order of the keys."""
    import torch
    k = keys.to(torch.int64)
    if key_bits == 8:
        return k & 0xFF
    if key_bits == 16:
        return k & 0xFFFF
    if key_bits == 32:
        return k & 0xFFFFFFFF
    return k ^ (-(1 << 63))


def order_key(keys, key_bits, kind="unsigned", descending=False):
    """int64 tensor whose signed order is the requested order of the key bits:
    unsigned; signed two's complement; IEEE 754 totalOrder for floats (sign-magnitude:
    -NaN < -inf < .. < -0.0 < +0.0 < .. < +inf < +NaN, reading Q18);
    descending reverses it (bitwise not: no overflow)."""
    import torch
    u = unsigned_order_key(keys, key_bits)
    if kind == "unsigned":
        k = u
    else:
        b = keys.to(torch.int64)
        if key_bits < 64:
            b = b & ((1 << key_bits) - 1)
            sign = 1 << (key_bits - 1)
            if kind == "signed":
                k = (b ^ sign) - sign
            else:
                mag = b & (sign - 1)
                k = torch.where((b & sign) != 0, -mag - 1, mag)
        else:
            if kind == "signed":
                k = b
            else:
                mag = b & ((1 << 63) - 1)
                k = torch.where(b < 0, -mag - 1, mag)
    return ~k if descending else k


def check_properties_torch(keys, key_bits, order, out_head, out_next, kind="unsigned", descending=False):
    """Same proof as check_sorted_list_properties, with torch ops on the tensors'
    device (used for the full-size configs, up to 2^30 nodes)."""
    import torch
    n = int(order.shape[0])
    if n == 0:
        assert out_head == NULL
        return
    dev = out_next.device
    on = out_next.to(torch.int64) & 0xFFFFFFFF
    is_null = on == NULL
    assert int(is_null.sum()) == 1, "exactly one NULL terminator"
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order.to(dev)] = torch.arange(n, device=dev)
    v = torch.nonzero(~is_null).squeeze(1)
    s = on[v]
    del is_null, on
    assert bool((s < n).all()), "successor out of range"
    cnt = torch.bincount(s, minlength=n)
    assert int(cnt.max()) <= 1, "a node has two predecessors"
    assert 0 <= out_head < n and int(cnt[out_head]) == 0, "head has a predecessor"
    del cnt
    k = order_key(keys.to(dev), key_bits, kind, descending)
    kv, ks = k[v], k[s]
    ok = (kv < ks) | ((kv == ks) & (rank[v] < rank[s]))
    bad = int((~ok).sum())
    assert bad == 0, f"{bad} edges break (key, input-rank) order"


def sampled_successors_torch(keys, key_bits, order, samples, kind="unsigned", descending=False):
    """The plain definition evaluated one output at a time: the successor of node v is
    the node with the smallest (key, input rank) above (key[v], rank[v])."""
    import torch
    n = int(order.shape[0])
    dev = keys.device
    rank = torch.empty(n, dtype=torch.int64, device=dev)
    rank[order.to(dev)] = torch.arange(n, device=dev)
    k = order_key(keys, key_bits, kind, descending)
    out = []
    for v in samples:
        kv, rv = k[v], rank[v]
        above = (k > kv) | ((k == kv) & (rank > rv))
        if not bool(above.any()):
            out.append(NULL)
            continue
        kk = torch.where(above, k, torch.full_like(k, torch.iinfo(torch.int64).max))
        kmin = kk.min()
        cand = above & (k == kmin)
        rr = torch.where(cand, rank, torch.full_like(rank, torch.iinfo(torch.int64).max))
        out.append(int(order.to(dev)[rr.min()]))
    return out
