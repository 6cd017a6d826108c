"""The seeded generators: determinism, valid lists, and the distribution shapes the
configs promise (DESIGN.md input recipe).  CPU only."""
import numpy as np
import pytest
import torch

import workloads
from tests.listcheck import walk


@pytest.mark.parametrize("n", [0, 1, 2, 5, 1000, 4097, 1 << 16])
def test_permutation_is_bijective_and_deterministic(n):
    p = workloads.permutation(n, seed=42)
    assert torch.equal(torch.sort(p).values, torch.arange(n))
    assert torch.equal(p, workloads.permutation(n, seed=42))
    if n > 100:
        assert not torch.equal(p, workloads.permutation(n, seed=43))


@pytest.mark.parametrize("links", ["random", "identity", "push"])
def test_links_form_one_list_in_order(links):
    li = workloads.make_list(3001, 32, seed=1, links=links)
    assert walk(workloads.next_numpy(li), li.head) == li.order.tolist()


def test_random_links_are_scattered():
    li = workloads.make_list(1 << 20, 32, seed=1)
    o = li.order
    gap = (o[1:] - o[:-1]).abs()
    assert float((gap < 1024).float().mean()) < 0.01   # successors are not near in memory


def test_zipf_top_key_fraction():
    # Zipf(1.1) over 2^20 ranks: P(rank 1) = 1 / H_{2^20,1.1} ~= 0.124
    li = workloads.make_list(1 << 20, 32, seed=3, keys="zipf")
    k = workloads.keys_numpy(li)
    _, counts = np.unique(k, return_counts=True)
    top = counts.max() / len(k)
    assert 0.115 < top < 0.133


def test_key_ranges():
    li = workloads.make_config("C1")
    assert li.n == 1 << 16 and li.keys.dtype == torch.uint8
    k = workloads.keys_numpy(workloads.make_list(50000, 32, 2, key_range=1 << 16))
    assert k.max() < 1 << 16 and k.min() >= 0 and len(np.unique(k)) > 30000
    k64 = workloads.keys_numpy(workloads.make_list(50000, 64, 2))
    assert (k64 >> np.uint64(63)).sum() > 10000     # high bit used


def test_runs4096_reading_q12():
    li = workloads.make_list(4096 * 4, 64, seed=4, keys="runs4096")
    k = workloads.keys_numpy(li)[li.order.numpy()]     # keys along the list
    assert (np.diff(k[:4096].astype(np.float64)) >= 0).all()         # P-run ascending
    assert not (np.diff(k[4096:8192].astype(np.float64)) >= 0).all()  # R-run random
    assert li.payload is not None and li.payload.shape[0] == li.n


def test_u64_kinds_use_every_bit():
    # the u64 sorted / runs keys had bit 32 forced to 0
    for kind in ("runs4096", "sorted", "reverse", "uniform"):
        k = workloads.keys_numpy(workloads.make_list(1 << 14, 64, 5, keys=kind))
        for bit in (0, 31, 32, 33, 63):
            frac = float(((k >> np.uint64(bit)) & np.uint64(1)).mean())
            assert 0.4 < frac < 0.6, (kind, bit, frac)


def test_u64_runs_sorted_by_full_key():
    li = workloads.make_list(4096 * 3, 64, seed=8, keys="runs4096")
    k = workloads.keys_numpy(li)[li.order.numpy()]
    assert np.all(k[1:4096] >= k[:4095]) and np.all(k[8193:12288] >= k[8192:12287])


@pytest.mark.parametrize("kind,bits", [("runs4096", 64), ("zipf", 32), ("uniform", 8)])
def test_chunking_does_not_change_values(kind, bits, monkeypatch):
    ref = workloads.make_list(50001 if kind != "runs4096" else 4096 * 13 + 5, bits, 9, keys=kind)
    monkeypatch.setattr(workloads, "CHUNK", 4096 * 3)
    got = workloads.make_list(ref.n, bits, 9, keys=kind)
    assert torch.equal(ref.keys, got.keys) and torch.equal(ref.next, got.next) and ref.head == got.head
    if ref.payload is not None:
        assert torch.equal(ref.payload, got.payload)
