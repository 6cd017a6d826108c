"""TEST INFRASTRUCTURE: pbit_sort_list_mg with G ranks, as G host threads on ONE GPU.

The library is the product's own objects linked with tests/fake_nccl/fake_nccl.cpp in
place of NCCL (NCCL refuses two ranks on one device), so every step of mg.cu -- its
kernels, its host planning, the exchanges -- runs for real at G > 1; only the transport
is emulated (device-to-device copies between the ranks' buffers, host barriers).  Each
case assembles the ranks' out_next (and out_prev) slices and compares them bit for bit
with the paper-literal oracle.  Prints one line per case; exit status 1 on any mismatch.

    python tests/fake_nccl/run_mg_threads.py            # the default case list
"""
from __future__ import annotations

import os
import sys
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import build_fake  # noqa: E402

os.environ["PBIT_LIB_PATH"] = build_fake.build()

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0511020_b200 as p  # noqa: E402
import workloads  # noqa: E402

assert p.LIB_PATH == os.environ["PBIT_LIB_PATH"], "the fake-NCCL library must be the one loaded"

# (G, n, key_bits, keys, links, K, kind, descending, with_prev)
CASES = [
    (2, 100003, 32, "uniform", "random", 0, "unsigned", False, True),
    (2, 4097, 32, "zipf", "random", 8, "unsigned", False, False),
    (3, 250001, 32, "zipf", "random", 0, "unsigned", False, True),
    (3, 77, 8, "uniform", "push", 4, "unsigned", False, False),       # a rank with no nodes
    (4, 130, 32, "zipf", "random", 0, "unsigned", False, True),       # two, with out_prev
    (4, 200001, 64, "runs4096", "random", 0, "unsigned", False, True),
    (4, 300007, 32, "equal", "random", 0, "unsigned", False, False),  # one key value
    (2, 123457, 32, "uniform", "random", 0, "float", True, False),
    (3, 123457, 16, "uniform", "identity", 5, "signed", False, True),
    (8, 1 << 20, 32, "uniform", "random", 0, "unsigned", False, True),
    (5, 65536, 8, "uniform", "random", 4, "unsigned", False, False),
    (6, 1000, 32, "zipf", "push", 0, "unsigned", False, True),          # ruler blocks > rulers
    (4, (1 << 22) + 37, 32, "zipf", "random", 0, "unsigned", False, False),
    (7, 777777, 64, "uniform", "random", 11, "signed", True, True),
]


def run_case(G, n, key_bits, keys, links, K, kind, desc, with_prev, seed):
    li = workloads.make_list(n, key_bits, seed=seed, keys=keys, links=links, device="cuda")
    S = p.mg_slice(n, G)
    uid = p.mg_unique_id()
    res, errs = [None] * G, [None] * G

    def rank(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            lo, hi = min(n, r * S), min(n, (r + 1) * S)
            with torch.cuda.stream(st):
                comm = p.mg_comm_init(G, uid, r)
                prev = torch.empty(hi - lo, dtype=torch.int32, device="cuda") if with_prev else None
                # the sorted records of this rank's positions (N3)
                order = torch.empty(hi - lo, dtype=torch.int32, device="cuda")
                skeys = torch.empty_like(li.keys[lo:hi])
                # node_lo = r * S even for a rank whose slice is empty (pbit.h)
                h, out = p.sort_list_mg(li.keys[lo:hi], li.next[lo:hi], li.head, n, r * S, comm, key_bits=key_bits,
                                        digit_bits=K, key_kind=kind, descending=desc, stream=st,
                                        out_prev_local=prev, out_order_local=order, out_keys_local=skeys)
                st.synchronize()
                res[r] = (h, out.cpu().numpy().view(np.uint32).copy(),
                          prev.cpu().numpy().view(np.uint32).copy() if with_prev else None, p.mg_transport(comm),
                          order.cpu().numpy().view(np.uint32).copy(), skeys.cpu().numpy().copy())
                p.mg_comm_destroy(comm)
        except Exception as e:  # noqa: BLE001  (reported by the main thread)
            errs[r] = e

    ts = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    import time
    t0 = time.time()
    while any(t.is_alive() for t in ts):
        time.sleep(0.05)
        # a rank that failed leaves the others waiting in a collective (as NCCL would)
        if any(errs) and time.time() - t0 > 5 or time.time() - t0 > 120:
            return False, (f"rank errors {[(r, repr(e)) for r, e in enumerate(errs) if e]}, "
                           f"ranks still inside the call: {[r for r, t in enumerate(ts) if t.is_alive()]}"), True
    if any(errs):
        return False, f"rank errors: {[repr(e) for e in errs if e]}", False
    heads = {r_[0] for r_ in res}
    used = {r_[3] for r_ in res}
    want_t = os.environ.get("PBIT_MG_TRANSPORT", "peer")
    if used != {want_t}:
        return False, f"transport {used} != {want_t}", False
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, key_bits, 4,
                              descending=desc, kind=kind)
    got = np.concatenate([r_[1] for r_ in res]) if n else np.zeros(0, np.uint32)
    if heads != {oh}:
        return False, f"heads {heads} != {oh}", False
    if not np.array_equal(got, on):
        bad = int(np.flatnonzero(got != on)[0])
        return False, f"out_next differs first at node {bad}: {got[bad]} != {on[bad]}", False
    if with_prev:
        gp = np.concatenate([r_[2] for r_ in res])
        if not np.array_equal(gp, oracle.repair_back(on, oh)):
            return False, "out_prev differs from the oracle's repair walk", False
    if n:
        want_order = oracle.list_order(on, oh)
        got_order = np.concatenate([r_[4] for r_ in res])
        if not np.array_equal(got_order, want_order):
            return False, "out_order differs from the oracle's sorted list", False
        kn_ = workloads.keys_numpy(li)
        got_keys = np.concatenate([r_[5] for r_ in res]).view(kn_.dtype)
        if not np.array_equal(got_keys, kn_[want_order]):
            return False, "out_keys differ from the keys along the oracle's sorted list", False
    return True, f"ok ({want_t})", False


def run_mismatch(G=3):
    """Rank 1 passes a different digit width: every rank must return INVALID_ARG from the
    argument agreement (none may be left waiting in a collective)."""
    n = 10007
    li = workloads.make_list(n, 32, seed=3, keys="uniform", device="cuda")
    S = p.mg_slice(n, G)
    uid = p.mg_unique_id()
    codes = [None] * G

    def rank(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        lo, hi = min(n, r * S), min(n, (r + 1) * S)
        with torch.cuda.stream(st):
            comm = p.mg_comm_init(G, uid, r)
            try:
                p.sort_list_mg(li.keys[lo:hi], li.next[lo:hi], li.head, n, r * S, comm, stream=st,
                               digit_bits=4 if r == 1 else 8)
                codes[r] = 0
            except p.PbitError as e:
                codes[r] = e.code
            p.mg_comm_destroy(comm)

    ts = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    ok = not any(t.is_alive() for t in ts) and codes == [1] * G
    print(f"G={G} mismatched digit_bits on rank 1: codes {codes}: {'ok' if ok else 'FAILED'}", flush=True)
    return ok


def run_invalid(G=3):
    """A cycle through the head: every rank must return INVALID_LIST (the error word is
    all-reduced, so no rank is left in an exchange) and leave its out_next untouched."""
    n = 30011
    nx_all = torch.arange(1, n + 1, dtype=torch.int32, device="cuda")
    nx_all[-1] = 0
    keys_all = torch.arange(n, dtype=torch.int32, device="cuda")
    S = p.mg_slice(n, G)
    uid = p.mg_unique_id()
    codes, kept = [None] * G, [None] * G

    def rank(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        lo, hi = min(n, r * S), min(n, (r + 1) * S)
        with torch.cuda.stream(st):
            comm = p.mg_comm_init(G, uid, r)
            out = torch.full((hi - lo,), 7, dtype=torch.int32, device="cuda")
            try:
                p.sort_list_mg(keys_all[lo:hi], nx_all[lo:hi], 0, n, r * S, comm, stream=st, out_next_local=out)
                codes[r] = 0
            except p.PbitError as e:
                codes[r] = e.code
            st.synchronize()
            kept[r] = bool((out == 7).all())
            p.mg_comm_destroy(comm)

    ts = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    ok = not any(t.is_alive() for t in ts) and codes == [2] * G and all(kept)
    print(f"G={G} invalid list (cycle): codes {codes}, out_next untouched {kept}: {'ok' if ok else 'FAILED'}",
          flush=True)
    return ok


def _is_ruler(v, n, s_log2):
    """The ruling-set selection of the product (common.cuh RulerSel), restated to BUILD an
    adversarial input (not to check an output)."""
    M = 0xFFFFFFFF
    r = v >> s_log2
    x = r ^ 0x6A09E667
    x ^= x >> 16
    x = (x * 0x21F0AAAD) & M
    x ^= x >> 15
    x = (x * 0x735A2D97) & M
    x ^= x >> 15
    s = 1 << s_log2
    span = n - (r << s_log2)
    off = (x & (s - 1)) if span >= s else x % span
    return (v & (s - 1)) == off


def run_dyn_overflow(G=2, n=120011):
    """A list whose rank-0 rulers head two segments covering almost every other node: rank
    0 must cut far more segments than its dynamic-ruler table holds (peer transport), the
    ranks see the overflow in the all-reduced error word and redo the call on the NCCL
    transport -- still bit-exact."""
    spacing, _ = p.mg_ruler_blocks(n, G)
    s_log2 = spacing.bit_length() - 1
    S = p.mg_slice(n, G)
    rul = np.array([_is_ruler(v, n, s_log2) for v in range(n)])
    ids = np.arange(n)
    A = ids[(ids < S) & rul]
    B = ids[(ids >= S) & rul]
    C0 = ids[(ids < S) & ~rul]
    C1 = ids[(ids >= S) & ~rul]
    order = np.concatenate([A[:1], C1, A[1:], C0, B]).astype(np.int64)
    assert len(order) == n and len(np.unique(order)) == n
    nxt = np.full(n, 0xFFFFFFFF, np.uint32)
    nxt[order[:-1]] = order[1:]
    keys = (np.arange(n, dtype=np.uint64) * 2654435761 % 1000).astype(np.uint32)
    kd = torch.from_numpy(keys.view(np.int32)).cuda()
    nd = torch.from_numpy(nxt.view(np.int32)).cuda()
    head = int(order[0])
    uid = p.mg_unique_id()
    res, errs = [None] * G, [None] * G

    def rank(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            lo, hi = min(n, r * S), min(n, (r + 1) * S)
            with torch.cuda.stream(st):
                comm = p.mg_comm_init(G, uid, r)
                h, out = p.sort_list_mg(kd[lo:hi], nd[lo:hi], head, n, r * S, comm, key_bits=32, stream=st)
                st.synchronize()
                res[r] = (h, out.cpu().numpy().view(np.uint32).copy(), p.mg_transport(comm))
                p.mg_comm_destroy(comm)
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    oh, on = oracle.pbit_sort(keys, nxt, head, 32, 4)
    ok = (not any(t.is_alive() for t in ts) and not any(errs) and {x[0] for x in res} == {oh}
          and np.array_equal(np.concatenate([x[1] for x in res]), on) and {x[2] for x in res} == {"nccl"})
    print(f"G={G} dynamic-ruler overflow on the peer transport: {'ok (fell back to nccl)' if ok else 'FAILED'} "
          f"{[repr(e) for e in errs if e]} {[x[2] for x in res if x]}", flush=True)
    return ok


def main(argv):
    cases = CASES
    if argv:  # e.g. "3,250001,32,zipf,random,0,unsigned,0,1"
        f = argv[0].split(",")
        cases = [(int(f[0]), int(f[1]), int(f[2]), f[3], f[4], int(f[5]), f[6], bool(int(f[7])), bool(int(f[8])))]
    fails = 0
    for i, c in enumerate(cases):
        ok, msg, stuck = run_case(*c, seed=1000 + i)
        print(f"G={c[0]} n={c[1]} u{c[2]} {c[3]}/{c[4]} K={c[5]} {c[6]}{' desc' if c[7] else ''}"
              f"{' +prev' if c[8] else ''}: {msg}", flush=True)
        fails += not ok
        if stuck:  # threads blocked in the fake transport cannot be joined: stop here
            print(f"{i + 1 - fails}/{len(cases)} cases bit-exact (stopped)", flush=True)
            os._exit(1)
    print(f"{len(cases) - fails}/{len(cases)} cases bit-exact", flush=True)
    if not argv and not run_mismatch():
        fails += 1
    if not argv and not run_invalid():
        fails += 1
    if not argv and os.environ.get("PBIT_MG_TRANSPORT", "peer") in ("peer", "hybrid") and not run_dyn_overflow():
        fails += 1
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
