"""pbit_sort_list_mg through the C-ABI on the one GPU available: a 1-rank NCCL
communicator, with both transports -- peer (N4; one rank: the single-GPU pipeline inside
the multi-GPU call) and NCCL (pack + all-gather, count walk, segment-table exchange,
ranking, emit walk, local sort, stitch, owner routing, relink) -- compared bit-exactly
with the oracle.  G > 1: the real
kernels at G = 2-8 in tests/test_gpu_mg_threads.py (stand-in transport, one GPU), and the
protocol on CPU in tests/test_mg_protocol.py (gloo, world_size 2-4)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["peer", "hybrid", "nccl"])
def mg(cuda_ok, request):
    import os
    import paper_cs_0511020_b200 as p
    old = os.environ.get("PBIT_MG_TRANSPORT")
    os.environ["PBIT_MG_TRANSPORT"] = request.param   # read by the library on every call
    uid = p.mg_unique_id()
    comm = p.mg_comm_init(1, uid, 0)
    yield p, comm
    assert p.mg_transport(comm) == request.param
    p.mg_comm_destroy(comm)
    if old is None:
        os.environ.pop("PBIT_MG_TRANSPORT", None)
    else:
        os.environ["PBIT_MG_TRANSPORT"] = old


CASES = [
    (1, 32, "uniform", "random"), (2, 32, "uniform", "random"), (77, 8, "uniform", "push"),
    (4097, 32, "zipf", "random"), (100003, 64, "runs4096", "random"), (65536, 8, "uniform", "random"),
    (200001, 16, "uniform", "identity"), (300007, 32, "equal", "random"), (1 << 20, 32, "uniform", "random"),
]


@pytest.mark.parametrize("n,key_bits,keys,links", CASES)
def test_mg_single_rank_vs_oracle(mg, n, key_bits, keys, links):
    p, comm = mg
    li = workloads.make_list(n, key_bits, seed=n + 31, keys=keys, links=links, device="cuda")
    assert p.mg_slice(n, 1) >= n
    h, out = p.sort_list_mg(li.keys, li.next, li.head, n, 0, comm, key_bits=key_bits)
    torch.cuda.synchronize()
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, key_bits, 4)
    assert h == oh
    assert np.array_equal(out.cpu().numpy().view(np.uint32), on)


@pytest.mark.parametrize("K", [4, 8, 12])
def test_mg_digit_widths(mg, K):
    p, comm = mg
    li = workloads.make_list(250001, 32, seed=5, keys="zipf", device="cuda")
    h, out = p.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, digit_bits=K)
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4)
    assert h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on)


def test_mg_invalid_list(mg):
    p, comm = mg
    n = 10000
    nx = torch.arange(1, n + 1, dtype=torch.int32)
    nx[-1] = 0  # cycle through the head
    keys = torch.arange(n, dtype=torch.int32)
    out = torch.full((n,), 7, dtype=torch.int32, device="cuda")
    with pytest.raises(p.PbitError) as e:
        p.sort_list_mg(keys.cuda(), nx.cuda(), 0, n, 0, comm, out_next_local=out)
    assert e.value.code == 2
    assert bool((out == 7).all())


def test_mg_bad_slice_rejected(mg):
    p, comm = mg
    k = torch.zeros(100, dtype=torch.int32, device="cuda")
    nx = torch.arange(1, 101, dtype=torch.int32, device="cuda")
    nx[-1] = -1
    with pytest.raises(p.PbitError) as e:
        p.sort_list_mg(k[:50], nx[:50], 0, 100, 0, comm)  # a 1-rank comm must own all 100 nodes
    assert e.value.code == 6


@pytest.mark.parametrize("kind,desc", [("signed", False), ("float", True), ("unsigned", True)])
def test_mg_key_kinds(mg, kind, desc):
    p, comm = mg
    li = workloads.make_list(123457, 32, seed=17, keys="uniform", device="cuda")
    h, out = p.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, key_kind=kind, descending=desc)
    torch.cuda.synchronize()
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4,
                              descending=desc, kind=kind)
    assert h == oh
    assert np.array_equal(out.cpu().numpy().view(np.uint32), on)


@pytest.mark.parametrize("n,key_bits,keys", [(1, 32, "uniform"), (1000, 32, "zipf"), (200001, 64, "uniform")])
def test_mg_out_prev(mg, n, key_bits, keys):
    """N2 through the multi-GPU protocol (1 rank): out_prev = the oracle's repair walk."""
    p, comm = mg
    li = workloads.make_list(n, key_bits, seed=n + 9, keys=keys, device="cuda")
    prev = torch.empty_like(li.next)
    h, out = p.sort_list_mg(li.keys, li.next, li.head, n, 0, comm, out_prev_local=prev)
    torch.cuda.synchronize()
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, key_bits, 4)
    assert h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on)
    assert np.array_equal(prev.cpu().numpy().view(np.uint32), oracle.repair_back(on, oh))


def test_mg_sorted_records(mg):
    """N3 records through the multi-GPU call: out_order / out_keys of the rank's sorted
    positions (one rank: all of them) = the oracle's sorted list and its keys."""
    p, comm = mg
    li = workloads.make_list(200003, 32, seed=41, keys="zipf", device="cuda")
    order = torch.empty(li.n, dtype=torch.int32, device="cuda")
    skeys = torch.empty_like(li.keys)
    h, out = p.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, out_order_local=order, out_keys_local=skeys)
    torch.cuda.synchronize()
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4)
    want = oracle.list_order(on, oh)
    assert h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on)
    assert np.array_equal(order.cpu().numpy().view(np.uint32), want)
    assert np.array_equal(skeys.cpu().numpy().view(np.uint32), workloads.keys_numpy(li)[want])
