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
