"""Bit-exact parity with the ORACLE at the full BASELINE.json sizes (north-star gate).

tests/golden/config_<name>.json holds, per config, the paper-literal oracle's result
(out_head, sha256 of out_next; for keys with a payload the sha256 of the payload sequence
along the sorted list, reading Q11), computed on the host by tools/make_goldens.py, which
imports only oracle/ and workloads.py (P:346-361 with the ascending loops P:379-380; the
stable result is unique, P:4, so every digit width must reproduce it).  Here the same
seeded list is generated on the device, its input hash is checked against the golden
(generator identity), and the CUDA path's output hash must equal the oracle's.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EXTRA = {  # tools/make_goldens.py EXTRA (kept in sync by test_golden_files_complete)
    "X26": dict(keys="zipf", links="random"),
    "X26u64": dict(keys="runs4096", links="random"),
}


def _goldens():
    out = {}
    for p in sorted(glob.glob(os.path.join(GOLDEN, "config_*.json"))):
        with open(p) as f:
            g = json.load(f)
        out[g["name"]] = g
    return out


GOLD = _goldens()


def _make(name, g, device):
    name = g.get("config", name)  # key-kind goldens ("C3_float") sort a config's list
    if name in workloads.CONFIGS:
        return workloads.make_config(name, device=device)
    e = EXTRA[name]
    return workloads.make_list(g["n"], g["key_bits"], g["seed"], keys=e["keys"], links=e["links"], device=device)


def _input_sha(li):
    h = hashlib.sha256()
    h.update(memoryview(np.ascontiguousarray(workloads.keys_numpy(li))).cast("B"))
    h.update(memoryview(np.ascontiguousarray(workloads.next_numpy(li))).cast("B"))
    h.update(np.array([li.head & 0xFFFFFFFF], np.uint32).tobytes())
    return h.hexdigest()


def test_golden_files_complete():
    """Every BASELINE config and the extra large cases have an oracle golden (CPU test)."""
    for name in ["C1", "C2", "C3", "C4", "C5", "X26", "X26u64", "ctx"]:
        assert name in GOLD, f"missing tests/golden/config_{name}.json (run tools/make_goldens.py {name})"
        g = GOLD[name]
        assert g["oracle_K"] == 4 and len(g["out_next_sha256"]) == 64
    assert "payload_seq_sha256" in GOLD["C4"]
    for name in ["C3_float", "C3_unsigned_desc", "C4_signed_desc"]:  # N1 at full size
        assert name in GOLD and GOLD[name]["config"] == name.split("_")[0]


def test_golden_c1_matches_oracle_here():
    """The golden of C1 reproduces with the oracle on this host (the script is honest)."""
    li = workloads.make_config("C1")
    assert _input_sha(li) == GOLD["C1"]["input_sha256"]
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 8, 4)
    assert oh == GOLD["C1"]["out_head"] and hashlib.sha256(on.tobytes()).hexdigest() == GOLD["C1"]["out_next_sha256"]


# every config at its BASELINE digit width; the extra cases also at the paper's K = 4 and
# at a width that does not divide the key (K = 11 as 8-bit sub-passes, reading Q7)
CASES = [(c, None) for c in ["C1", "C2", "C3", "C4", "C5", "X26", "X26u64", "ctx"]] + [
    ("X26", 4), ("X26", 6), ("X26u64", 11), ("C3", 4), ("C4", 4), ("C5", 4), ("C2", 3),
    ("ctx", 8), ("ctx", 16),  # the paper's own workload at its K = 4 (default), 8 and 16
    # key kinds and the descending order at full size (N1: P:371-372)
    ("C3_float", None), ("C3_unsigned_desc", None), ("C4_signed_desc", None)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,K", CASES)
def test_full_size_bit_exact_vs_oracle_golden(cuda_ok, name, K):
    import paper_cs_0511020_b200 as pbit
    g = GOLD[name]
    li = _make(name, g, "cuda")
    assert li.n == g["n"]
    assert _input_sha(li) == g["input_sha256"], "device generator differs from the host generator"
    cfg = g.get("config", name)
    K = K or (workloads.CONFIGS[cfg]["digit_bits"] if cfg in workloads.CONFIGS else 8)
    payload = li.payload
    h, out = pbit.sort_list(li.keys, li.next, li.head, key_bits=li.key_bits, digit_bits=K,
                            key_kind=g.get("kind", "unsigned"), descending=g.get("descending", False))
    torch.cuda.synchronize()
    on = out.cpu().numpy().view(np.uint32)
    del li, out
    torch.cuda.empty_cache()
    assert h == g["out_head"], f"{name} K={K}: head {h} != oracle {g['out_head']}"
    assert hashlib.sha256(on.tobytes()).hexdigest() == g["out_next_sha256"], f"{name} K={K}: out_next differs"
    if "payload_seq_sha256" in g:  # the payload follows its node (reading Q11)
        order = oracle.list_order(on, h)
        seq = payload.cpu().numpy()[order]
        assert hashlib.sha256(seq.tobytes()).hexdigest() == g["payload_seq_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["peer", "hybrid", "nccl"])
def test_mg_one_rank_full_size_c3_vs_oracle_golden(cuda_ok, transport, monkeypatch):
    """pbit_sort_list_mg on a real 1-rank NCCL communicator, every transport, on the full
    C3 list: the oracle's bytes."""
    import paper_cs_0511020_b200 as pbit
    monkeypatch.setenv("PBIT_MG_TRANSPORT", transport)   # read by the library on every call
    g = GOLD["C3"]
    li = _make("C3", g, "cuda")
    comm = pbit.mg_comm_init(1, pbit.mg_unique_id(), 0)
    try:
        h, out = pbit.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, digit_bits=8)
        torch.cuda.synchronize()
        assert pbit.mg_transport(comm) == transport
    finally:
        pbit.mg_comm_destroy(comm)
    on = out.cpu().numpy().view(np.uint32)
    del li, out
    torch.cuda.empty_cache()
    assert h == g["out_head"] and hashlib.sha256(on.tobytes()).hexdigest() == g["out_next_sha256"]
