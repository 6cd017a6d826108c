"""Pins of the CPU oracle (oracle/pbit_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.  CPU only."""
from __future__ import annotations

import itertools
import os

import numpy as np
import pytest

import oracle
import workloads
from tests.listcheck import (NULL, check_sorted_list_properties, expected_by_definition,
                             expected_by_definition_small, walk)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_example.txt")


def _golden():
    d = {}
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split(None, 1)
        d[k] = v
    return d


def _chain(keys):
    n = len(keys)
    nxt = np.array(list(range(1, n)) + [NULL], np.uint32) if n else np.zeros(0, np.uint32)
    return nxt, (0 if n else NULL)


# ---------------------------------------------------------------- worked example P:84-98
def test_worked_example_output():
    g = _golden()
    keys = np.array([int(x) for x in g["input"].split()], np.uint8)
    nxt, head = _chain(keys)
    h, out = oracle.pbit_sort(keys, nxt, head, int(g["key_bits"]), int(g["K"]))
    seq = walk(out, h)
    assert [int(keys[v]) for v in seq] == [int(x) for x in g["output"].split()]
    # stability: the 3 at input position 1 precedes the 3 at input position 6
    val, pos = g["equal_key_positions"].split(":")
    assert [v for v in seq if keys[v] == int(val)] == [int(p) for p in pos.split(",")]


def test_worked_example_first_level_groups():
    g = _golden()
    keys = np.array([int(x) for x in g["input"].split()], np.uint8)
    nxt, head = _chain(keys)
    tab, relinked = oracle.split_once(keys, nxt, head, 8, 4)
    want = {int(b): sorted(int(x) for x in ks.split(",")) for b, ks in
            (t.split(":") for t in g["level1"].split())}
    got = {b: sorted(int(keys[v]) for v in walk(relinked, tab[b])) for b in range(16) if tab[b] != NULL}
    assert got == want
    # push-front leaves each bucket in reverse input order
    assert walk(relinked, tab[0]) == [6, 3, 1]


def test_bits_paper_example():
    # 123 / 8 = 15.375 -> 01111011 >> 3 = 00001111 = 15 (mod 16 keeps 15)
    assert oracle.bits(123, 3, 4) == 15
    assert oracle.bits(209, 4, 4) == 13 and oracle.bits(214, 4, 4) == 13  # P:91 group {209,214}
    assert oracle.bits(0xABCDEF12, 28, 4) == 0xA
    assert oracle.bits(0xFFFFFFFFFFFFFFFF, 56, 8) == 0xFF


def test_memory_formula_paper_values():
    # P:129-131 T(8)=160, T(32)=616; P:981-982 K=8: 4152
    assert oracle.memory_bound_T(8, 4) == 160
    assert oracle.memory_bound_T(32, 4) == 616
    assert oracle.memory_bound_T(32, 8) == 4152


# ---------------------------------------------------------------- brute force
ALPHABETS = {
    8: [0x00, 0x0F, 0x10, 0xFF, 0x7F, 0x80],
    16: [0x0000, 0x00FF, 0xFF00, 0xFFFF, 0x0F0F],
    32: [0, 1, 0x10, 0xFFFFFFFF, 0x80000000, 0x0000FFFF],
    64: [0, 0xFFFFFFFFFFFFFFFF, 0x8000000000000000, 0x00000000FFFFFFFF, 0x10],
}


@pytest.mark.parametrize("key_bits", [8, 16, 32, 64])
def test_brute_force_all_link_orders(key_bits):
    """Every link order of n <= 6 nodes, keys from an adversarial alphabet (extreme
    digits, duplicates) vs python's stable sorted() of the list-order sequence."""
    rng = np.random.default_rng(key_bits)
    alpha = ALPHABETS[key_bits]
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32, 64: np.uint64}[key_bits]
    for n in range(0, 7):
        keys = np.array([alpha[i] for i in rng.integers(0, len(alpha), n)], dt)
        perms = list(itertools.permutations(range(n)))
        if len(perms) > 240:
            perms = [perms[i] for i in rng.choice(len(perms), 240, replace=False)]
        for perm in perms:
            nxt = np.full(n, NULL, np.uint32)
            for a, b in zip(perm[:-1], perm[1:]):
                nxt[a] = b
            head = perm[0] if n else NULL
            h, out = oracle.pbit_sort(keys, nxt, head, key_bits, 4)
            eh, eout = expected_by_definition_small(keys, nxt, head)
            assert h == eh and np.array_equal(out, eout), (n, perm, keys)


@pytest.mark.parametrize("key_bits,keys_kind,links", [
    (8, "uniform", "random"), (16, "uniform", "random"), (32, "uniform", "random"),
    (32, "zipf", "random"), (64, "uniform", "random"), (64, "runs4096", "random"),
    (32, "equal", "random"), (32, "max", "identity"), (32, "sorted", "push"),
    (32, "reverse", "random"), (8, "uniform", "push"), (16, "uniform", "identity"),
])
@pytest.mark.parametrize("n", [1, 2, 3, 10, 100, 2048, 4099, 70001])
def test_seeded_random_lists_vs_stable_argsort(key_bits, keys_kind, links, n):
    li = workloads.make_list(n, key_bits, seed=n * 7 + key_bits, keys=keys_kind, links=links)
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    assert oracle.validate_list(nxt, li.head)
    h, out, cnt = oracle.pbit_sort(keys, nxt, li.head, key_bits, 4, with_counters=True)
    eh, eout = expected_by_definition(keys, li.order.numpy())
    assert h == eh and np.array_equal(out, eout)
    check_sorted_list_properties(keys, li.order.numpy(), h, out)
    # P:73 / P:328-330: n*M/K relinks and exactly n merge visits
    assert cnt["relinks"] == n * key_bits // 4
    assert cnt["merge_visits"] == n


# ---------------------------------------------------------------- counter identities
@pytest.mark.parametrize("key_bits,K", [(8, 4), (32, 4), (32, 8), (64, 4), (32, 16), (16, 2)])
def test_counter_identities_and_depth(key_bits, K):
    n = 5000
    li = workloads.make_list(n, key_bits, seed=5, keys="uniform")
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    _, _, c = oracle.pbit_sort(keys, nxt, li.head, key_bits, K, with_counters=True)
    assert c["relinks"] == n * (key_bits // K)          # split term of f(n)
    assert c["merge_visits"] == n                       # "Always count equal n"
    assert c["max_depth"] == key_bits // K              # M/K levels
    assert c["max_live_tabs"] <= key_bits // K          # at most M/K root tables
    omega = 1 << K
    assert c["max_live_tabs"] * omega * 4 <= oracle.memory_bound_T(key_bits, K)


def test_counters_empty_and_single():
    _, _, c = oracle.pbit_sort(np.zeros(0, np.uint32), np.zeros(0, np.uint32), NULL, 32, 4, with_counters=True)
    assert c["relinks"] == 0 and c["merge_visits"] == 0
    h, out, c = oracle.pbit_sort(np.array([7], np.uint32), np.array([NULL], np.uint32), 0, 32, 4,
                                 with_counters=True)
    assert h == 0 and out[0] == NULL and c["relinks"] == 8 and c["merge_visits"] == 1


# ---------------------------------------------------------------- direction + parity readings
def test_descending_duality_distinct_keys():
    """P:371-374 (loops 0..Omega-1) sort descending; with distinct keys it is the
    exact reverse of ascending (SPEC direction duality)."""
    n = 3000
    li = workloads.make_list(n, 32, seed=9, keys="uniform")
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    assert len(np.unique(keys)) == n
    ha, oa = oracle.pbit_sort(keys, nxt, li.head, 32, 4)
    hd, od = oracle.pbit_sort(keys, nxt, li.head, 32, 4, descending=True)
    assert walk(od, hd) == walk(oa, ha)[::-1]


def test_descending_stable_with_duplicates():
    n = 4000
    li = workloads.make_list(n, 16, seed=11, keys="uniform", key_range=50)
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    hd, od = oracle.pbit_sort(keys, nxt, li.head, 16, 4, descending=True)
    eh, eo = expected_by_definition(keys, li.order.numpy(), descending=True)
    assert hd == eh and np.array_equal(od, eo)


def test_odd_levels_are_reverse_stable():
    """Reading Q1: the push-front split reverses equal digits once per level, so the
    literal listing is stable only when M/K is even.  M=8, K=8 (one level) must
    reverse the order of equal keys -- documents why the oracle uses K=4."""
    keys = np.array([5, 5, 1, 5], np.uint8)
    nxt, head = _chain(keys)
    h, out = oracle.pbit_sort(keys, nxt, head, 8, 8)
    assert walk(out, h) == [2, 3, 1, 0]
    h, out = oracle.pbit_sort(keys, nxt, head, 8, 4)   # M/K = 2: stable
    assert walk(out, h) == [2, 0, 1, 3]


# ---------------------------------------------------------------- invalid lists
def test_invalid_lists_rejected():
    keys = np.arange(4, dtype=np.uint32)
    bad = {
        "cycle_through_head": (np.array([1, 2, 3, 0], np.uint32), 0),
        "cycle_off_path": (np.array([1, NULL, 3, 2], np.uint32), 0),
        "short": (np.array([1, 2, NULL, NULL], np.uint32), 0),
        "index_ge_n": (np.array([1, 9, 3, NULL], np.uint32), 0),
        "head_ge_n": (np.array([1, 2, 3, NULL], np.uint32), 4),
        "empty_head_not_null": (np.zeros(0, np.uint32), 0),
    }
    for name, (nxt, head) in bad.items():
        k = keys[: len(nxt)] if len(nxt) else np.zeros(1, np.uint32)
        with pytest.raises(oracle.OracleError) as e:
            oracle.pbit_sort(k, nxt, head, 32, 4)
        assert e.value.code == 2, name


def test_invalid_args_rejected():
    keys = np.arange(4, dtype=np.uint32)
    nxt = np.array([1, 2, 3, NULL], np.uint32)
    for kb, K in [(24, 4), (32, 3), (32, 0), (8, 16)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.pbit_sort(keys, nxt, 0, kb, K)
        assert e.value.code == 1


def test_in_place_alias():
    """out_next may alias next: the paper relinks in situ."""
    li = workloads.make_list(1000, 32, seed=3, keys="uniform", key_range=17)
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li).copy()
    h, out = oracle.pbit_sort(keys, nxt, li.head, 32, 4, out=nxt)
    eh, eo = expected_by_definition(keys, li.order.numpy())
    assert h == eh and np.array_equal(nxt, eo) and np.shares_memory(out, nxt)


# ---------------------------------------------------------------- key kinds (NEXT row N1)
KINDS_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "key_kinds.txt")


def _kinds_golden():
    d = {}
    for line in open(KINDS_GOLDEN):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split(None, 1)
            d[k] = v
    return d


def test_worked_example_descending():
    g = _kinds_golden()
    keys = np.array([int(x) for x in g["desc_input"].split()], np.uint8)
    nxt, head = _chain(keys)
    h, out = oracle.pbit_sort(keys, nxt, head, 8, 4, descending=True)
    seq = walk(out, h)
    assert [int(keys[v]) for v in seq] == [int(x) for x in g["desc_output"].split()]
    val, pos = g["desc_equal_key_positions"].split(":")
    assert [v for v in seq if keys[v] == int(val)] == [int(p) for p in pos.split(",")]


def test_signed_example():
    g = _kinds_golden()
    keys = np.array([int(x) for x in g["signed_input"].split()], np.int32)
    nxt, head = _chain(keys)
    h, out = oracle.pbit_sort(keys, nxt, head, 32, 4, kind="signed")
    assert [int(keys[v]) for v in walk(out, h)] == [int(x) for x in g["signed_output"].split()]


def test_float_example():
    g = _kinds_golden()
    keys = np.array([float(x) for x in g["float_input"].split()], np.float32)
    nxt, head = _chain(keys)
    h, out = oracle.pbit_sort(keys, nxt, head, 32, 4, kind="float")
    assert [float(keys[v]) for v in walk(out, h)] == [float(x) for x in g["float_output"].split()]


SIGNED_ALPHABETS = {8: [-128, -1, 0, 1, 127, -16], 16: [-32768, -256, -1, 0, 255, 32767],
                    32: [-2**31, -1, 0, 1, 2**31 - 1, -65536], 64: [-2**63, -1, 0, 2**63 - 1, -2**32]}
INT_DT = {8: np.int8, 16: np.int16, 32: np.int32, 64: np.int64}
FLOAT_DT = {16: np.float16, 32: np.float32, 64: np.float64}


def _float_key(x):
    """Order of the plain definition for floats without NaN: numeric, -0.0 before +0.0."""
    return (float(x), 0 if np.signbit(x) else 1)


@pytest.mark.parametrize("key_bits", [8, 16, 32, 64])
@pytest.mark.parametrize("descending", [False, True])
def test_signed_brute_force_all_link_orders(key_bits, descending):
    """Every link order of n <= 5 over an adversarial signed alphabet vs python's stable
    sorted() of the list-order sequence by the signed value (reverse=True keeps equal keys
    in input order)."""
    alpha = SIGNED_ALPHABETS[key_bits]
    rng = np.random.default_rng(key_bits)
    for n in range(0, 6):
        keys = np.array(rng.choice(alpha, size=n), dtype=INT_DT[key_bits])
        for perm in itertools.permutations(range(n)):
            nxt = np.full(n, NULL, np.uint32)
            for a, b in zip(perm, perm[1:]):
                nxt[a] = b
            head = perm[0] if n else NULL
            h, out = oracle.pbit_sort(keys, nxt, head, key_bits, 4, descending=descending, kind="signed")
            want = sorted(list(perm), key=lambda v: int(keys[v]), reverse=descending)
            assert walk(out, h) == want


@pytest.mark.parametrize("key_bits", [16, 32, 64])
@pytest.mark.parametrize("descending", [False, True])
def test_float_brute_force_all_link_orders(key_bits, descending):
    alpha = [-np.inf, -2.5, -1.0, -0.0, 0.0, 1.5, 2.5, np.inf, 6e-5, -6e-5]
    rng = np.random.default_rng(100 + key_bits)
    for n in range(0, 6):
        keys = np.array(rng.choice(alpha, size=n), dtype=FLOAT_DT[key_bits])
        for perm in itertools.permutations(range(n)):
            nxt = np.full(n, NULL, np.uint32)
            for a, b in zip(perm, perm[1:]):
                nxt[a] = b
            head = perm[0] if n else NULL
            h, out = oracle.pbit_sort(keys, nxt, head, key_bits, 4, descending=descending, kind="float")
            want = sorted(list(perm), key=lambda v: _float_key(keys[v]), reverse=descending)
            assert walk(out, h) == want


@pytest.mark.parametrize("key_bits", [16, 32, 64])
def test_float_random_vs_numpy_stable(key_bits):
    """Seeded random lists (no NaN, no -0.0) vs numpy's stable argsort of the values."""
    rng = np.random.default_rng(7 + key_bits)
    for n in [1, 2, 17, 1000, 4099]:
        vals = rng.normal(0, 100, n) * rng.choice([1e-3, 1, 1e3], n)
        vals = np.round(np.clip(vals, -6e4, 6e4), 1).astype(FLOAT_DT[key_bits])  # duplicates; f16 range
        vals[vals == 0] = 0.0
        order = rng.permutation(n)
        nxt = np.full(n, NULL, np.uint32)
        nxt[order[:-1]] = order[1:]
        for desc in (False, True):
            h, out = oracle.pbit_sort(vals, nxt, int(order[0]), key_bits, 4, descending=desc, kind="float")
            wh, wn = expected_by_definition(vals.astype(np.float64), order, descending=desc)
            assert h == wh and np.array_equal(out, wn)


def test_float_nan_and_signed_zero_total_order():
    """Reading Q18: sign-magnitude order of the bit patterns (IEEE 754 totalOrder):
    -NaN < -inf < ... < -0.0 < +0.0 < ... < +inf < +NaN, NaNs by payload."""
    bits = np.array([0x7FC00001, 0x3F800000, 0xFFC00001, 0xFF800000, 0x7FC00002, 0x00000000, 0x80000000,
                     0x7F800000], np.uint32)
    # the same values listed in totalOrder (derived from IEEE 754-2008 section 5.10)
    want_bits = [0xFFC00001, 0xFF800000, 0x80000000, 0x00000000, 0x3F800000, 0x7F800000, 0x7FC00001, 0x7FC00002]
    nxt, head = _chain(bits)
    h, out = oracle.pbit_sort(bits, nxt, head, 32, 4, kind="float")
    assert [int(bits[v]) for v in walk(out, h)] == want_bits
    h, out = oracle.pbit_sort(bits, nxt, head, 32, 4, kind="float", descending=True)
    assert [int(bits[v]) for v in walk(out, h)] == want_bits[::-1]


@pytest.mark.parametrize("key_bits", [8, 32, 64])
def test_signed_random_vs_numpy_stable(key_bits):
    rng = np.random.default_rng(11 + key_bits)
    info = np.iinfo(INT_DT[key_bits])
    for n in [1, 3, 100, 4099]:
        vals = rng.integers(info.min, info.max, n, dtype=INT_DT[key_bits], endpoint=True)
        vals[rng.random(n) < 0.3] = vals[0]  # duplicates
        order = rng.permutation(n)
        nxt = np.full(n, NULL, np.uint32)
        nxt[order[:-1]] = order[1:]
        for desc in (False, True):
            h, out = oracle.pbit_sort(vals, nxt, int(order[0]), key_bits, 4, descending=desc, kind="signed")
            wh, wn = expected_by_definition(vals, order, descending=desc)
            assert h == wh and np.array_equal(out, wn)


def test_kind_counter_identities():
    """relinks = n * (sum of the levels of every Pbit call a node goes through), merge
    visits = n per call: signed = one call of M/K levels, float = a
    mantissa call and a characteristic call (fields padded to a multiple of 2K bits)."""
    rng = np.random.default_rng(3)
    n = 777
    order = rng.permutation(n)
    nxt = np.full(n, NULL, np.uint32)
    nxt[order[:-1]] = order[1:]
    si = rng.integers(-1000, 1000, n).astype(np.int32)
    _, _, c = oracle.pbit_sort(si, nxt, int(order[0]), 32, 4, kind="signed", with_counters=True)
    assert c["relinks"] == n * 32 // 4 and c["merge_visits"] == n
    fl = rng.normal(0, 1, n).astype(np.float32)
    _, _, c = oracle.pbit_sort(fl, nxt, int(order[0]), 32, 4, kind="float", with_counters=True)
    assert c["relinks"] == n * (24 // 4 + 8 // 4) and c["merge_visits"] == 2 * n
    f64 = rng.normal(0, 1, n)
    _, _, c = oracle.pbit_sort(f64, nxt, int(order[0]), 64, 4, kind="float", with_counters=True)
    assert c["relinks"] == n * (56 // 4 + 16 // 4) and c["merge_visits"] == 2 * n


def test_literal_signed_split_is_reverse_stable():
    """Reading Q13 demonstrated: pushing to the FRONT of the sign lists (the listing,
    P:450-455) and then sorting with the paper's even number of levels returns equal keys
    in reverse input order -- which is why the oracle appends at the tails."""
    keys = np.array([5, -2, 5, -2, 5], np.int32)
    nxt, head = _chain(keys)
    # push-front split by hand, then the oracle's unsigned ascending Pbit on each list
    neg = [v for v in walk(nxt, head) if keys[v] < 0][::-1]
    pos = [v for v in walk(nxt, head) if keys[v] >= 0][::-1]
    seq = []
    for part in (neg, pos):
        sub_keys = keys[part].view(np.uint32)  # the sub-list as its own node array, in list order
        sub_next, sub_head = _chain(sub_keys)
        h, out = oracle.pbit_sort(sub_keys, sub_next, sub_head, 32, 4)
        seq += [part[i] for i in walk(out, h)]
    assert seq == [3, 1, 4, 2, 0]  # equal keys reversed: not stable
    h, out = oracle.pbit_sort(keys, nxt, head, 32, 4, kind="signed")
    assert walk(out, h) == [1, 3, 0, 2, 4]  # the oracle's reading: stable


# ---------------------------------------------------------------- doubly-linked repair (NEXT row N2)
def test_repair_back_examples():
    """repair([a->b->c]) -> back(c)=b, back(b)=a, back(a)=NULL; a single
    node gets NULL; the empty list stays empty."""
    nxt = np.array([2, NULL, 1], np.uint32)  # a=0 -> c=2 -> b=1
    back = oracle.repair_back(nxt, 0)
    assert back[2] == 0 and back[1] == 2 and back[0] == NULL
    assert list(oracle.repair_back(np.array([NULL], np.uint32), 0)) == [NULL]
    assert oracle.repair_back(np.zeros(0, np.uint32), NULL).size == 0
    with pytest.raises(oracle.OracleError):
        oracle.repair_back(np.array([1, 0], np.uint32), 0)  # cycle


def test_repair_back_after_sort_is_the_reverse_chain():
    """After a sort, back[] must satisfy back[next[x]] = x for every node x with a
    successor and back[head] = NULL: the plain definition w_{i+1} -> w_i."""
    rng = np.random.default_rng(9)
    n = 5003
    keys = rng.integers(0, 50, n).astype(np.uint32)
    order = rng.permutation(n)
    nxt = np.full(n, NULL, np.uint32)
    nxt[order[:-1]] = order[1:]
    h, out = oracle.pbit_sort(keys, nxt, int(order[0]), 32, 4)
    back = oracle.repair_back(out, h)
    w = walk(out, h)
    assert back[w[0]] == NULL
    assert all(back[b] == a for a, b in zip(w, w[1:]))


def test_order_key_checker_matches_python_sort():
    """The full-size checker's order key (tests/listcheck.order_key) against python's
    sort of the values -- pins the checker used for N1 at full size."""
    import torch
    from tests.listcheck import order_key
    rng = np.random.default_rng(12)
    for bits, dt in ((16, np.float16), (32, np.float32), (64, np.float64)):
        vals = np.concatenate([rng.normal(0, 10, 200), [0.0, -0.0, np.inf, -np.inf]]).astype(dt)
        t = torch.from_numpy(vals.view({16: np.int16, 32: np.int32, 64: np.int64}[bits]).copy())
        k = order_key(t, bits, "float").numpy()
        want = sorted(range(len(vals)), key=lambda i: (float(vals[i]), 0 if np.signbit(vals[i]) else 1))
        assert list(np.argsort(k, kind="stable")) == want
        kd = order_key(t, bits, "float", descending=True).numpy()
        assert list(np.argsort(kd, kind="stable")) == sorted(range(len(vals)), key=lambda i: (
            -float(vals[i]), 0 if not np.signbit(vals[i]) else 1))
    for bits, dt in ((8, np.int8), (32, np.int32), (64, np.int64)):
        info = np.iinfo(dt)
        vals = rng.integers(info.min, info.max, 300, dtype=dt, endpoint=True)
        t = torch.from_numpy(vals.copy())
        assert list(np.argsort(order_key(t, bits, "signed").numpy(), kind="stable")) == \
            sorted(range(len(vals)), key=lambda i: int(vals[i]))


@pytest.mark.parametrize("links", ["random", "identity", "push"])
def test_list_order_is_the_generators_order(links):
    # pinned to workloads' own construction of the list (next[order[p]] = order[p+1])
    li = workloads.make_list(5003, 32, seed=11, links=links)
    got = oracle.list_order(workloads.next_numpy(li), li.head)
    assert np.array_equal(got.astype(np.int64), li.order.numpy())


def test_list_order_rejects_invalid():
    with pytest.raises(oracle.OracleError):
        oracle.list_order(np.array([1, 0], np.uint32), 0)   # cycle
    assert oracle.list_order(np.zeros(0, np.uint32), oracle.ORACLE_NULL).shape == (0,)


@pytest.mark.parametrize("n,key_bits,keys,links,K,threads", [
    (0, 32, "uniform", "random", 4, 2), (1, 8, "uniform", "random", 4, 3), (2, 16, "equal", "push", 8, 2),
    (5000, 8, "uniform", "random", 4, 4), (50001, 32, "zipf", "random", 4, 8), (70001, 64, "runs4096", "random", 8, 3),
    (30000, 16, "equal", "push", 4, 5), (100003, 32, "uniform", "identity", 8, 1), (65537, 32, "sorted", "random", 2, 4)])
def test_subtree_parallel_oracle_is_bit_identical(n, key_bits, keys, links, K, threads):
    """SURVEY §8(d)'s optional subtree-parallel CPU baseline: the first two levels of the
    recursion as Pbit runs them, the rest on threads, the sorted sublists linked in list
    order -- the serial oracle's bytes (Pbit(L, M, P) = Pbit(L, M, NULL) followed by P)."""
    li = workloads.make_list(n, key_bits, seed=n + K, keys=keys, links=links)
    k, nx = workloads.keys_numpy(li), workloads.next_numpy(li)
    a = oracle.pbit_sort(k, nx, li.head, key_bits, K)
    b = oracle.pbit_sort_par(k, nx, li.head, key_bits, K, threads)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
