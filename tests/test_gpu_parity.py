"""Parity of the CUDA path (through the C-ABI) with the paper-literal oracle.

Bit-exact: the stable result is unique, so (out_head, out_next[]) must equal the
oracle's bytes for every digit width K.  Full BASELINE.json sizes (2^28-2^30) are
checked with properties that together force the unique answer
(tests/listcheck.check_properties_torch) plus sampled outputs evaluated one by one.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import workloads
from tests.listcheck import NULL, check_properties_torch, sampled_successors_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pbit(cuda_ok):
    import paper_cs_0511020_b200 as p
    return p


def _gpu_sort(pbit, li, K=0, **kw):
    h, out = pbit.sort_list(li.keys, li.next, li.head, key_bits=li.key_bits, digit_bits=K, **kw)
    torch.cuda.synchronize()
    return h, out.cpu().numpy().view(np.uint32)


def _oracle(li, K=4):
    return oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, li.key_bits, K)


def _assert_same(got, want, what=""):
    gh, go = got
    oh, oo = want
    assert gh == oh, f"{what}: head {gh} != {oh}"
    if not np.array_equal(go, oo):
        bad = np.nonzero(go != oo)[0]
        raise AssertionError(f"{what}: {len(bad)} of {len(oo)} next[] entries differ, first at {bad[:5]}")


# ---------------------------------------------------------------- BASELINE configs C1, C2 vs oracle
def test_c1_bit_exact_paper_K4(pbit):
    li = workloads.make_config("C1", device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=4), _oracle(li), "C1 K=4")


@pytest.mark.parametrize("K", [1, 2, 3, 5, 6, 7, 8])
def test_c1_every_digit_width_identical(pbit, K):
    li = workloads.make_config("C1", device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=K), _oracle(li), f"C1 K={K}")


def test_c2_bit_exact(pbit):
    li = workloads.make_config("C2", device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=8), _oracle(li), "C2 K=8")


# ---------------------------------------------------------------- ragged sizes, key widths, shapes
CASES = [
    (1, 32, "uniform", "random"), (2, 32, "uniform", "random"), (3, 8, "uniform", "push"),
    (31, 16, "uniform", "random"), (4095, 32, "zipf", "random"), (4097, 64, "uniform", "random"),
    (65537, 32, "uniform", "random"), (65537, 8, "uniform", "identity"), (100003, 16, "uniform", "push"),
    (100003, 32, "equal", "random"), (100003, 32, "max", "random"), (100003, 64, "equal", "identity"),
    (100003, 32, "sorted", "random"), (100003, 32, "reverse", "random"), (250001, 64, "runs4096", "random"),
    (1000003, 32, "zipf", "random"), (1000003, 64, "uniform", "push"), (1 << 20, 32, "uniform", "identity"),
    # the plan's size classes: 16-node segments and 8-ruler sub-segments (2^22..2^24),
    # 32-node segments (2^24..2^26)
    ((1 << 22) + 19, 32, "zipf", "random"), ((1 << 23) + 5, 64, "uniform", "random"),
    ((1 << 24) + 1, 16, "uniform", "random"),
]


@pytest.mark.parametrize("n,key_bits,keys,links", CASES)
def test_ragged_shapes_vs_oracle(pbit, n, key_bits, keys, links):
    li = workloads.make_list(n, key_bits, seed=n ^ key_bits, keys=keys, links=links, device="cuda")
    _assert_same(_gpu_sort(pbit, li), _oracle(li), f"{li.name}")


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 6, 7, 8])
def test_digit_width_sweep_zipf(pbit, K):
    li = workloads.make_list(300007, 32, seed=77, keys="zipf", device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=K), _oracle(li), f"K={K}")


@pytest.mark.parametrize("K", [9, 11, 12, 16])
def test_wide_patterns_vs_oracle_K16(pbit, K):
    """K = 9..16 (SPEC S:127's range): 8-bit sub-passes per pattern (reading Q7); the bytes
    are the oracle's, which sorts with 16-bit patterns literally (tab[65536])."""
    li = workloads.make_list(300007, 32, seed=79, keys="zipf", device="cuda")
    h, out, ph = pbit.sort_list(li.keys, li.next, li.head, digit_bits=K, timing=True)
    torch.cuda.synchronize()
    assert ph["passes_run"] <= 4
    _assert_same((h, out.cpu().numpy().view(np.uint32)), _oracle(li, K=16), f"K={K}")
    idx, _ = pbit.sort_array(li.keys, key_bits=32, digit_bits=K)
    kn = li.keys.cpu().numpy().view(np.uint32)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), np.argsort(kn, kind="stable").astype(np.uint32))


@pytest.mark.parametrize("n,key_bits,keys,K", [(300007, 32, "uniform", 8), (300007, 32, "zipf", 4),
                                                 (100003, 64, "runs4096", 8), (8191, 16, "equal", 3)])
def test_lane0_combining_on_every_pass(pbit, monkeypatch, n, key_bits, keys, K):
    """The ranking's lane-0 combining (normally only on skewed middle passes) forced on
    every pass, first and last included, on inputs of every shape."""
    monkeypatch.setenv("PBIT_COMBINE", "2")
    li = workloads.make_list(n, key_bits, seed=n + K, keys=keys, device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=K), _oracle(li), f"combine {li.name} K={K}")
    idx, _ = pbit.sort_array(li.keys, key_bits=key_bits, digit_bits=K)
    kn = workloads.keys_numpy(li)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), np.argsort(kn, kind="stable").astype(np.uint32))


@pytest.mark.parametrize("K", [3, 5, 8])
def test_digit_width_sweep_u64_narrow_top_digit(pbit, K):
    li = workloads.make_list(70001, 64, seed=78, keys="uniform", device="cuda")
    _assert_same(_gpu_sort(pbit, li, K=K), _oracle(li), f"u64 K={K}")


def test_small_key_range_skips_trivial_digits(pbit):
    li = workloads.make_list(500000, 32, seed=5, keys="uniform", key_range=1 << 16, device="cuda")
    h, out, ph = pbit.sort_list(li.keys, li.next, li.head, digit_bits=8, timing=True)
    torch.cuda.synchronize()
    assert ph["passes_run"] == 2
    _assert_same((h, out.cpu().numpy().view(np.uint32)), _oracle(li), "C5-shaped")


def test_largest_n_fails_cleanly_with_oom(pbit):
    """n = 2^32 - 2, the largest the ABI accepts (u32 ids, PBIT_NULL reserved): the
    workspace (~60 B/node) exceeds the 180 GB HBM, so the call must return PBIT_ERR_OOM
    before any kernel runs, with no size arithmetic overflowing on the way."""
    n = (1 << 32) - 2
    keys = torch.empty(n, dtype=torch.uint8, device="cuda")
    nx = torch.empty(n, dtype=torch.int32, device="cuda")
    with pytest.raises(pbit.PbitError) as e:
        pbit.sort_list(keys, nx, 0, key_bits=8, out_next=nx)  # in place: no third array
    assert e.value.code == 3
    del keys, nx
    torch.cuda.empty_cache()


def test_workspace_released_after_each_call_by_default(pbit):
    """Default: the workspace goes back to the device when the call ends (release
    threshold 0, pbit.h); the device's free memory after a call is what it was before."""
    li = workloads.make_list(1 << 22, 32, seed=12, keys="uniform", device="cuda")
    want = _oracle(li)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    got = _gpu_sort(pbit, li)   # allocates its output tensor (16 MB) from torch's cache
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)   # ~250 MB of workspace returned
    _assert_same(got, want, "default pool")
    pbit.workspace_trim(0)
    _assert_same(_gpu_sort(pbit, li), want, "after trim")


KEEP_SNIPPET = """
import torch, workloads, paper_cs_0511020_b200 as pbit
li = workloads.make_list(1 << 22, 32, seed=12, keys="uniform", device="cuda")
out = torch.empty_like(li.next)
torch.cuda.synchronize(); f0 = torch.cuda.mem_get_info()[0]
pbit.sort_list(li.keys, li.next, li.head, out_next=out); torch.cuda.synchronize()
f1 = torch.cuda.mem_get_info()[0]
pbit.workspace_trim(0); f2 = torch.cuda.mem_get_info()[0]
print(f0, f1, f2)
assert f1 <= f0 - (100 << 20), "PBIT_POOL_KEEP_GB: workspace should stay mapped"
assert f2 >= f0 - (64 << 20), "pbit_workspace_trim(0) should release it"
"""


def test_workspace_kept_with_pool_keep_gb_and_trimmed(pbit):
    """PBIT_POOL_KEEP_GB (opt-in) keeps the workspace mapped between calls;
    pbit_workspace_trim hands it back (subprocess: the pool reads the variable once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PBIT_POOL_KEEP_GB="8", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", KEEP_SNIPPET], capture_output=True, text=True, env=env, cwd=root,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_all_equal_keys_runs_no_pass(pbit):
    li = workloads.make_list(77777, 32, seed=6, keys="equal", device="cuda")
    h, out, ph = pbit.sort_list(li.keys, li.next, li.head, timing=True)
    torch.cuda.synchronize()
    assert ph["passes_run"] == 0
    _assert_same((h, out.cpu().numpy().view(np.uint32)), _oracle(li), "all equal")


# ---------------------------------------------------------------- API edge cases
def test_empty_and_singletons(pbit):
    h, out = pbit.sort_list(torch.zeros(0, dtype=torch.int32, device="cuda"),
                            torch.zeros(0, dtype=torch.int32, device="cuda"), NULL)
    assert h == NULL and out.numel() == 0
    k = torch.tensor([5], dtype=torch.int32, device="cuda")
    nx = torch.tensor([-1], dtype=torch.int32, device="cuda")
    h, out = pbit.sort_list(k, nx, 0)
    assert h == 0 and int(out[0]) == -1
    k = torch.tensor([9, 2], dtype=torch.int32, device="cuda")
    nx = torch.tensor([1, -1], dtype=torch.int32, device="cuda")
    h, out = pbit.sort_list(k, nx, 0)
    assert h == 1 and out.tolist() == [-1, 0]


def test_worked_example_on_gpu(pbit):
    keys = torch.tensor([21, 3, 209, 14, 156, 47, 3, 214], dtype=torch.uint8, device="cuda")
    nx = torch.tensor([1, 2, 3, 4, 5, 6, 7, -1], dtype=torch.int32, device="cuda")
    h, out = pbit.sort_list(keys, nx, 0, digit_bits=4)
    seq, v = [], h
    o = out.cpu().numpy().view(np.uint32)
    while v != NULL:
        seq.append(v)
        v = int(o[v])
    assert [int(keys[i]) for i in seq] == [3, 3, 14, 21, 47, 156, 209, 214]
    assert seq[:2] == [1, 6]  # stable: list position 1 before 6 (P:4)


def test_in_place_alias(pbit):
    li = workloads.make_list(123457, 32, seed=8, keys="zipf", device="cuda")
    want = _oracle(li)
    nx = li.next.clone()
    h, out = pbit.sort_list(li.keys, nx, li.head, out_next=nx)
    torch.cuda.synchronize()
    assert out.data_ptr() == nx.data_ptr()
    _assert_same((h, nx.cpu().numpy().view(np.uint32)), want, "in place")


def test_host_buffers(pbit):
    li = workloads.make_list(200003, 64, seed=9, keys="runs4096")
    k = workloads.keys_numpy(li)
    nx = workloads.next_numpy(li)
    h, out = pbit.sort_list(k, nx, li.head, key_bits=64)
    _assert_same((h, out), _oracle(li), "host buffers")
    kp = li.keys.pin_memory()
    npin = li.next.pin_memory()
    h2, out2 = pbit.sort_list(kp, npin, li.head)
    _assert_same((h2, out2.numpy().view(np.uint32)), _oracle(li), "pinned host buffers")


def test_side_stream_and_determinism(pbit):
    li = workloads.make_list(400009, 32, seed=10, keys="zipf", device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = pbit.sort_list(li.keys, li.next, li.head, stream=s)
    b = pbit.sort_list(li.keys, li.next, li.head)
    torch.cuda.synchronize()
    assert a[0] == b[0] and torch.equal(a[1], b[1])


# ---------------------------------------------------------------- invalid lists
def _bad_lists(n=50000):
    base = torch.arange(1, n + 1, dtype=torch.int32)
    base[-1] = -1
    cyc_head = base.clone(); cyc_head[-1] = 0                       # tail -> head
    cyc_off = base.clone(); cyc_off[n // 2] = -1; cyc_off[-1] = n // 2 + 1  # second half is a cycle
    short = base.clone(); short[n - 10] = -1                          # 10 nodes unreachable
    bad_idx = base.clone(); bad_idx[777] = n + 5                      # index >= n
    two_pred = base.clone(); two_pred[n - 2] = 5                      # node 5 reached twice
    small_cycle = base.clone(); small_cycle[1000] = 999               # 999 <-> 1000 loop
    return {"cycle_through_head": cyc_head, "cycle_off_path": cyc_off, "short": short,
            "index_ge_n": bad_idx, "two_predecessors": two_pred, "small_cycle": small_cycle}


# (n, K): the single-cluster small-list path (n <= 2^16, K 4/8) and the general path
@pytest.mark.parametrize("n,K", [(50000, 8), (50000, 3), (100003, 8)])
@pytest.mark.parametrize("name", list(_bad_lists().keys()))
def test_invalid_list_rejected_and_out_untouched(pbit, name, n, K):
    nx = _bad_lists(n)[name].cuda()
    keys = workloads.uniform_u32(nx.shape[0], 1, 1).to(torch.int32).cuda()
    out = torch.full_like(nx, 0x1234)
    with pytest.raises(pbit.PbitError) as e:
        pbit.sort_list(keys, nx, 0, out_next=out, digit_bits=K)
    assert e.value.code == 2
    torch.cuda.synchronize()
    assert bool((out == 0x1234).all()), "out_next modified on INVALID_LIST"
    with pytest.raises(oracle.OracleError):
        oracle.pbit_sort(keys.cpu().numpy().view(np.uint32), nx.cpu().numpy().view(np.uint32), 0, 32, 4)


@pytest.mark.parametrize("name", ["cycle_through_head", "short", "index_ge_n", "two_predecessors"])
def test_invalid_list_host_buffers_untouched(pbit, name):
    """Host buffers (the e2e path copies results back while the relink runs): an invalid
    list must leave the caller's host out_next untouched."""
    n = 200003
    nx = _bad_lists(n)[name].numpy().view(np.uint32)
    keys = workloads.uniform_u32(nx.shape[0], 1, 1).numpy().astype(np.uint32)
    out = np.full(nx.shape[0], 0x1234, np.uint32)
    with pytest.raises(pbit.PbitError) as e:
        pbit.sort_list(keys, nx, 0, out_next=out)
    assert e.value.code == 2
    assert (out == 0x1234).all(), "host out_next modified on INVALID_LIST"


def test_invalid_args(pbit):
    k = torch.zeros(4, dtype=torch.int32, device="cuda")
    nx = torch.tensor([1, 2, 3, -1], dtype=torch.int32, device="cuda")
    with pytest.raises(pbit.PbitError) as e:
        pbit.sort_list(k, nx, 4)
    assert e.value.code == 1
    with pytest.raises(pbit.PbitError) as e:  # mixed host/device
        pbit.sort_list(k.cpu(), nx, 0)
    assert e.value.code == 1


# ---------------------------------------------------------------- full BASELINE sizes (properties)
@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_full_size_configs(pbit, cfg):
    c = workloads.CONFIGS[cfg]
    li = workloads.make_config(cfg, device="cuda")
    h, out = pbit.sort_list(li.keys, li.next, li.head, digit_bits=c["digit_bits"])
    torch.cuda.synchronize()
    check_properties_torch(li.keys, li.key_bits, li.order, h, out)
    g = torch.Generator().manual_seed(1)
    samples = torch.randint(0, li.n, (6,), generator=g).tolist() + [h]
    want = sampled_successors_torch(li.keys, li.key_bits, li.order, samples)
    got = [int(out[v]) & 0xFFFFFFFF for v in samples]
    assert got == want
    del li, out
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- key kinds (NEXT row N1)
# The same seeded bit patterns read as signed integers or IEEE floats (uniform 32/64-bit
# patterns include NaNs, infinities, subnormals and both zeros), ascending and descending,
# against the oracle's paper-derived procedures.
KIND_CASES = [
    (1, 32, "uniform", "random", "signed", False), (2, 8, "uniform", "random", "signed", True),
    (4099, 8, "uniform", "push", "signed", False), (65537, 16, "uniform", "random", "signed", True),
    (100003, 32, "uniform", "random", "signed", False), (100003, 32, "zipf", "random", "signed", True),
    (70001, 64, "uniform", "identity", "signed", True), (70001, 64, "runs4096", "random", "signed", False),
    (100003, 32, "max", "random", "signed", True), (33333, 16, "uniform", "random", "float", False),
    (100003, 32, "uniform", "random", "float", False), (100003, 32, "uniform", "random", "float", True),
    (70001, 64, "uniform", "random", "float", False), (70001, 64, "uniform", "push", "float", True),
    (65537, 16, "equal", "random", "float", True), (100003, 32, "uniform", "random", "unsigned", True),
    (70001, 8, "uniform", "random", "unsigned", True), (250001, 64, "runs4096", "random", "unsigned", True),
    (1000003, 32, "zipf", "random", "float", True),
]


@pytest.mark.parametrize("n,key_bits,keys,links,kind,desc", KIND_CASES)
def test_key_kinds_vs_oracle(pbit, n, key_bits, keys, links, kind, desc):
    li = workloads.make_list(n, key_bits, seed=(n * 3) ^ key_bits, keys=keys, links=links, device="cuda")
    got = _gpu_sort(pbit, li, key_kind=kind, descending=desc)
    want = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, li.key_bits, 4,
                            descending=desc, kind=kind)
    _assert_same(got, want, f"{li.name} {kind} desc={desc}")


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 6, 7, 8])
def test_key_kinds_every_digit_width(pbit, K):
    li = workloads.make_list(65537, 32, seed=91, keys="uniform", device="cuda")
    want = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4,
                            descending=True, kind="float")
    _assert_same(_gpu_sort(pbit, li, K=K, key_kind="float", descending=True), want, f"float desc K={K}")


def test_float_special_values(pbit):
    """±0, ±inf, NaNs with payloads, subnormals, repeated: the IEEE totalOrder reading (Q18)."""
    special = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7FC00001,
                        0x00000001, 0x80000001, 0x3F800000, 0xBF800000, 0x7F7FFFFF, 0xFF7FFFFF], np.uint32)
    rng = np.random.default_rng(5)
    n = 50001
    bits = special[rng.integers(0, len(special), n)]
    order = rng.permutation(n)
    nxt = np.full(n, NULL, np.uint32)
    nxt[order[:-1]] = order[1:]
    kd = torch.from_numpy(bits.view(np.int32)).cuda()
    nd = torch.from_numpy(nxt.view(np.int32)).cuda()
    for desc in (False, True):
        h, out = pbit.sort_list(kd, nd, int(order[0]), key_bits=32, key_kind="float", descending=desc)
        torch.cuda.synchronize()
        want = oracle.pbit_sort(bits, nxt, int(order[0]), 32, 4, descending=desc, kind="float")
        _assert_same((h, out.cpu().numpy().view(np.uint32)), want, f"float specials desc={desc}")


def test_key_kind_invalid_args(pbit):
    k = torch.zeros(4, dtype=torch.uint8, device="cuda")
    nx = torch.tensor([1, 2, 3, -1], dtype=torch.int32, device="cuda")
    with pytest.raises(pbit.PbitError) as e:  # no 8-bit IEEE format
        pbit.sort_list(k, nx, 0, key_kind="float")
    assert e.value.code == 1


# ---------------------------------------------------------------- doubly-linked lists (NEXT row N2)
@pytest.mark.parametrize("n,key_bits,keys,links", [
    (1, 32, "uniform", "random"), (2, 8, "uniform", "random"), (3, 16, "equal", "push"),
    (16384, 32, "uniform", "random"), (16385, 32, "zipf", "random"), (70001, 64, "uniform", "random"),
    (1000003, 32, "zipf", "random"), (1 << 20, 16, "uniform", "identity")])
def test_doubly_linked_out_prev(pbit, n, key_bits, keys, links):
    """out_prev = the paper's reverse-connection repair of the sorted list,
    computed by the oracle from its own sorted out_next."""
    li = workloads.make_list(n, key_bits, seed=n + 5, keys=keys, links=links, device="cuda")
    prev = torch.empty_like(li.next)
    h, out = pbit.sort_list(li.keys, li.next, li.head, key_bits=key_bits, out_prev=prev)
    torch.cuda.synchronize()
    oh, on = _oracle(li)
    _assert_same((h, out.cpu().numpy().view(np.uint32)), (oh, on), f"{li.name} next")
    want_prev = oracle.repair_back(on, oh)
    assert np.array_equal(prev.cpu().numpy().view(np.uint32), want_prev)


def test_doubly_linked_host_buffers_and_args(pbit):
    li = workloads.make_list(40001, 32, seed=8, keys="uniform", device="cpu")
    prev = np.empty(li.n, np.uint32)
    out = np.empty(li.n, np.uint32)
    h, _ = pbit.sort_list(li.keys, li.next, li.head, out_next=out, out_prev=prev, descending=True,
                          key_kind="signed")
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4,
                              descending=True, kind="signed")
    assert h == oh and np.array_equal(out, on)
    assert np.array_equal(prev, oracle.repair_back(on, oh))
    k = li.keys.cuda()
    nx = li.next.cuda()
    o = torch.empty_like(nx)
    with pytest.raises(pbit.PbitError) as e:  # out_prev aliasing out_next
        pbit.sort_list(k, nx, li.head, out_next=o, out_prev=o)
    assert e.value.code == 1


# ---------------------------------------------------------------- arrays (NEXT row N3)
def _array_oracle(keys_np, key_bits, kind="unsigned", desc=False):
    """The oracle's Pbit on the array read as a list in array order (next[i] = i+1):
    the sorted list order is the stable sorted order of the array."""
    n = len(keys_np)
    nxt = np.arange(1, n + 1, dtype=np.uint32)
    if n:
        nxt[-1] = NULL
    h, out = oracle.pbit_sort(keys_np, nxt, 0 if n else NULL, key_bits, 4, descending=desc, kind=kind)
    from tests.listcheck import walk
    return np.array(walk(out, h), np.uint32)


@pytest.mark.parametrize("n,key_bits,keys,kind,desc", [
    (1, 32, "uniform", "unsigned", False), (7, 8, "uniform", "unsigned", True), (4097, 16, "uniform", "signed", False),
    (100003, 32, "zipf", "unsigned", False), (100003, 32, "uniform", "float", True),
    (70001, 64, "uniform", "signed", True), (70001, 64, "runs4096", "unsigned", False),
    (65537, 32, "equal", "unsigned", False), (1000003, 32, "uniform", "unsigned", False)])
def test_array_sort_vs_oracle(pbit, n, key_bits, keys, kind, desc):
    li = workloads.make_list(n, key_bits, seed=n ^ 77, keys=keys, device="cuda")
    idx, sk = pbit.sort_array(li.keys, key_bits=key_bits, want_keys=True, key_kind=kind, descending=desc)
    torch.cuda.synchronize()
    kn = workloads.keys_numpy(li)
    want = _array_oracle(kn, key_bits, kind, desc)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), want)
    assert np.array_equal(sk.cpu().numpy().view(kn.dtype), kn[want])


@pytest.mark.parametrize("K", [1, 3, 4, 8])
def test_array_digit_widths_and_host_buffers(pbit, K):
    li = workloads.make_list(50001, 32, seed=3, keys="zipf", device="cpu")
    kn = workloads.keys_numpy(li)
    want = _array_oracle(kn, 32)
    idx, _ = pbit.sort_array(kn, key_bits=32, digit_bits=K)  # numpy host buffers (staged)
    assert np.array_equal(np.asarray(idx).view(np.uint32), want)


# ---------------------------------------------------------------- N1-N3 at full BASELINE sizes (properties)
@pytest.mark.parametrize("cfg,kind,desc", [("C3", "float", False), ("C4", "signed", True), ("C3", "unsigned", True)])
def test_full_size_key_kinds(pbit, cfg, kind, desc):
    c = workloads.CONFIGS[cfg]
    li = workloads.make_config(cfg, device="cuda")
    h, out = pbit.sort_list(li.keys, li.next, li.head, digit_bits=c["digit_bits"], key_kind=kind, descending=desc)
    torch.cuda.synchronize()
    check_properties_torch(li.keys, li.key_bits, li.order, h, out, kind=kind, descending=desc)
    g = torch.Generator().manual_seed(2)
    samples = torch.randint(0, li.n, (4,), generator=g).tolist() + [h]
    want = sampled_successors_torch(li.keys, li.key_bits, li.order, samples, kind=kind, descending=desc)
    assert [int(out[v]) & 0xFFFFFFFF for v in samples] == want
    del li, out
    torch.cuda.empty_cache()


def test_full_size_doubly_linked_c3(pbit):
    li = workloads.make_config("C3", device="cuda")
    prev = torch.empty_like(li.next)
    h, out = pbit.sort_list(li.keys, li.next, li.head, out_prev=prev)
    torch.cuda.synchronize()
    check_properties_torch(li.keys, li.key_bits, li.order, h, out)
    on = out.to(torch.int64) & 0xFFFFFFFF
    pv = prev.to(torch.int64) & 0xFFFFFFFF
    has = on != NULL
    v = torch.nonzero(has).squeeze(1)
    assert bool((pv[on[v]] == v).all()), "prev[next[v]] != v"
    assert int(pv[h]) == NULL and int((pv == NULL).sum()) == 1
    del li, out, prev
    torch.cuda.empty_cache()


def test_full_size_array_c3(pbit):
    li = workloads.make_config("C3", device="cuda")
    idx, sk = pbit.sort_array(li.keys, want_keys=True)
    torch.cuda.synchronize()
    ix = idx.to(torch.int64) & 0xFFFFFFFF
    n = li.n
    assert int(torch.bincount(ix, minlength=n).max()) == 1, "index is not a permutation"
    from tests.listcheck import order_key
    k = order_key(li.keys, 32)[ix]
    ok = (k[:-1] < k[1:]) | ((k[:-1] == k[1:]) & (ix[:-1] < ix[1:]))
    assert bool(ok.all()), "array order not sorted/stable"
    assert torch.equal(sk, li.keys[ix]), "sorted keys differ from keys[index]"
    del li, idx, sk
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- extreme digit plans
@pytest.mark.parametrize("key_bits,K", [(64, 1), (64, 7), (32, 1), (16, 3), (8, 1), (64, 2)])
def test_extreme_digit_plans(pbit, key_bits, K):
    """Up to 64 passes (u64 keys, K = 1: the most the plan holds), narrow top digits."""
    li = workloads.make_list(5003, key_bits, seed=key_bits * 10 + K, keys="uniform", device="cuda")
    h, out, ph = pbit.sort_list(li.keys, li.next, li.head, digit_bits=K, timing=True)
    torch.cuda.synchronize()
    assert ph["passes_run"] == (key_bits + K - 1) // K
    _assert_same((h, out.cpu().numpy().view(np.uint32)), _oracle(li), f"u{key_bits} K={K}")
    idx, _ = pbit.sort_array(li.keys, key_bits=key_bits, digit_bits=K)
    torch.cuda.synchronize()
    kn = workloads.keys_numpy(li)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), np.argsort(kn, kind="stable").astype(np.uint32))


def test_head_positions_and_tiny_lists(pbit):
    """Every head position of small lists, n around the tile and window sizes."""
    for n in (2, 3, 17, 4095, 4096, 4097, 8191, 8192, 8193, 16383, 16384, 16385):
        li = workloads.make_list(n, 32, seed=n, keys="zipf", links="random", device="cuda")
        _assert_same(_gpu_sort(pbit, li), _oracle(li), f"n={n}")


def test_small_path_in_place_host_and_stream(pbit):
    """The single-cluster small-list path: in-place relink, host buffers, a side stream,
    out_prev -- against the oracle."""
    li = workloads.make_list(40009, 32, seed=21, keys="zipf", device="cuda")
    want = _oracle(li)
    nx = li.next.clone()
    h, out = pbit.sort_list(li.keys, nx, li.head, out_next=nx)  # in place
    torch.cuda.synchronize()
    _assert_same((h, out.cpu().numpy().view(np.uint32)), want, "small in-place")
    kh, nh = li.keys.cpu().numpy(), li.next.cpu().numpy()
    oh = np.empty(li.n, np.uint32)
    ph = np.empty(li.n, np.uint32)
    h2, _ = pbit.sort_list(kh, nh, li.head, out_next=oh, out_prev=ph)  # host buffers
    _assert_same((h2, oh), want, "small host")
    assert np.array_equal(ph, oracle.repair_back(want[1], want[0]))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h3, o3 = pbit.sort_list(li.keys, li.next, li.head, stream=s)
    s.synchronize()
    _assert_same((h3, o3.cpu().numpy().view(np.uint32)), want, "small side stream")


def test_concurrent_host_threads_on_own_streams(pbit):
    """pbit.h: thread-safe across distinct streams -- 4 host threads (ctypes releases the
    GIL), each sorting its own list on its own stream, small and general paths mixed."""
    import threading
    lists = [workloads.make_list(n, 32, seed=40 + i, keys="zipf", device="cuda")
             for i, n in enumerate((30011, 150001, 60013, 250007))]
    want = [_oracle(li) for li in lists]
    got = [None] * len(lists)
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            li = lists[i]
            with torch.cuda.stream(s):  # outputs allocated on (and used by) this stream
                for _ in range(3):
                    h, out = pbit.sort_list(li.keys, li.next, li.head)
            s.synchronize()
            got[i] = (h, out.cpu().numpy().view(np.uint32))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(lists))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for i in range(len(lists)):
        _assert_same(got[i], want[i], f"thread {i}")


def test_concurrent_host_buffer_calls(pbit):
    """The pipelined e2e of bench.py: host (pinned) buffers sorted from 3 host threads at
    once, each with its own stream -- every thread's chunked copies run on its own copy
    stream while another thread's sort runs; each result equals the oracle's."""
    import threading
    lists = [workloads.make_list(n, 32, seed=70 + i, keys=k)
             for i, (n, k) in enumerate((((1 << 20) + 3, "zipf"), (300007, "uniform"), ((1 << 21) - 5, "runs4096")))]
    want = [_oracle(li) for li in lists]
    got = [None] * len(lists)
    errors = []

    def work(i):
        try:
            li = lists[i]
            kh, nh = li.keys.pin_memory(), li.next.pin_memory()
            oh = torch.empty_like(nh).pin_memory()
            s = torch.cuda.Stream()
            for _ in range(3):
                h, _ = pbit.sort_list(kh, nh, li.head, out_next=oh, stream=s)
            got[i] = (h, oh.numpy().view(np.uint32).copy())
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(lists))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for i in range(len(lists)):
        _assert_same(got[i], want[i], f"host-buffer thread {i}")


# ---------------------------------------------------------------- N3: sorted records (out_order, out_keys)
@pytest.mark.parametrize("n,key_bits,keys,links,kind,desc", [
    (1, 32, "uniform", "random", "unsigned", False), (1000, 8, "uniform", "random", "unsigned", False),
    (65537, 16, "uniform", "push", "signed", True), (100003, 32, "zipf", "random", "unsigned", False),
    (250001, 64, "runs4096", "random", "float", False), (300007, 32, "equal", "random", "unsigned", False)])
def test_sorted_records_materialised(pbit, n, key_bits, keys, links, kind, desc):
    """out_order[i] = the i-th node of the oracle's sorted list, out_keys[i] = its key (input
    bits); device and host buffers; the payload follows through out_order (reading Q11)."""
    li = workloads.make_list(n, key_bits, seed=n * 7 + key_bits, keys=keys, links=links, device="cuda")
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, key_bits, 4,
                              descending=desc, kind=kind)
    order = oracle.list_order(on, oh)
    order_d = torch.empty(n, dtype=torch.int32, device="cuda")
    keys_d = torch.empty_like(li.keys)
    h, out = pbit.sort_list(li.keys, li.next, li.head, key_bits=key_bits, key_kind=kind, descending=desc,
                            out_order=order_d, out_keys=keys_d)
    torch.cuda.synchronize()
    assert h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on)
    assert np.array_equal(order_d.cpu().numpy().view(np.uint32), order)
    assert np.array_equal(workloads.keys_numpy(li)[order], keys_d.cpu().numpy().view(workloads.keys_numpy(li).dtype))
    if li.payload is not None:  # sorted records (key, payload) through out_order
        assert np.array_equal(li.payload[order_d.long()].cpu().numpy(), li.payload.cpu().numpy()[order])
    # host buffers
    kh, nh = workloads.keys_numpy(li), workloads.next_numpy(li)
    oh2, ko2 = np.empty(n, np.uint32), np.empty_like(kh)
    h2, out2 = pbit.sort_list(kh, nh, li.head, key_bits=key_bits, key_kind=kind, descending=desc,
                              out_order=oh2, out_keys=ko2)
    assert h2 == oh and np.array_equal(out2, on) and np.array_equal(oh2, order) and np.array_equal(ko2, kh[order])


def test_sorted_records_untouched_on_invalid_list(pbit):
    n = 100003
    nx = _bad_lists(n)["cycle_through_head"].cuda()
    keys = workloads.uniform_u32(n, 1, 1).to(torch.int32).cuda()
    order = torch.full((n,), 5, dtype=torch.int32, device="cuda")
    ko = torch.full((n,), 9, dtype=torch.int32, device="cuda")
    with pytest.raises(pbit.PbitError) as e:
        pbit.sort_list(keys, nx, 0, out_order=order, out_keys=ko)
    assert e.value.code == 2
    torch.cuda.synchronize()
    assert bool((order == 5).all()) and bool((ko == 9).all())


def test_plain_c_example_prints_the_papers_worked_example(pbit, tmp_path):
    """examples/sort_list.c: the C-ABI from a plain C program on host arrays, the worked
    example of P:84-98 (3 3 14 21 47 156 209 214)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "sort_list"
    libdir = os.path.dirname(os.path.abspath(pbit.LIB_PATH))
    subprocess.run(["cc", "-std=c99", "-I", os.path.join(root, "include"), os.path.join(root, "examples", "sort_list.c"),
                    os.path.abspath(pbit.LIB_PATH), f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["3", "3", "14", "21", "47", "156", "209", "214"]


RANK_SNIPPET = """
import numpy as np, torch, oracle, workloads, paper_cs_0511020_b200 as pbit
assert pbit.rank_mode() == {mode}, pbit.rank_mode()
for n, kb, keys, links, K in [(100003, 32, "zipf", "random", 8), (65537, 8, "uniform", "push", 4),
                               (250001, 64, "runs4096", "random", 8), (1000003, 32, "uniform", "random", 0),
                               (77777, 16, "equal", "identity", 5), (4097, 32, "sorted", "random", 3)]:
    li = workloads.make_list(n, kb, seed=n, keys=keys, links=links, device="cuda")
    h, out = pbit.sort_list(li.keys, li.next, li.head, key_bits=kb, digit_bits=K)
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, kb, 4)
    assert h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on), (n, kb, keys, K)
    idx, _ = pbit.sort_array(li.keys, key_bits=kb, digit_bits=K)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), np.argsort(workloads.keys_numpy(li), kind="stable"))
print("ok")
"""


@pytest.mark.parametrize("mode,code", [("ballot", 0), ("match", 1)])
def test_fallback_rankings_vs_oracle(pbit, mode, code):
    """The in-warp rankings other than the lane-ordered atomics: the ballot peer masks run
    if a device's atomic-order self-test ever fails (pbit_rank_mode), match.any on request;
    both must give the oracle's bytes (subprocess: the mode is decided once per device)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PBIT_RANK=mode, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", RANK_SNIPPET.format(mode=code)], capture_output=True, text=True,
                       env=env, cwd=root, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
