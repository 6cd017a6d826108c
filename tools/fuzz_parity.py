"""Randomised parity sweep (GPU): many seeded random shapes through the C-ABI, each
compared bit-exactly with the oracle -- list sort (out_next, and out_prev on some), the
array sort, every key kind and direction, digit widths 1..16, sizes 1 .. ~3M covering the
single-cluster path and every size class of the general path.

    python tools/fuzz_parity.py [seconds] [seed] [max_n]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0511020_b200 as p  # noqa: E402
import workloads  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
max_n = int(sys.argv[3]) if len(sys.argv) > 3 else 3_000_000
KEYS = ["uniform", "zipf", "equal", "max", "sorted", "reverse", "runs4096"]
LINKS = ["random", "identity", "push"]
t0, cases, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    n = int(rng.choice([1, 2, 3, 31, 257, 4095, 65536, 65537]) if rng.random() < 0.3
            else int(np.exp(rng.uniform(np.log(2), np.log(max_n)))))
    kb = int(rng.choice([8, 16, 32, 64]))
    keys = str(rng.choice(KEYS))
    links = str(rng.choice(LINKS))
    K = int(rng.choice([0, 0, 1, 3, 4, 5, 8, 11, 16]))
    kind = str(rng.choice(["unsigned", "signed", "float"])) if kb >= 16 else str(rng.choice(["unsigned", "signed"]))
    desc = bool(rng.random() < 0.3)
    prev = bool(rng.random() < 0.3)
    seed = int(rng.integers(1 << 30))
    li = workloads.make_list(n, kb, seed=seed, keys=keys, links=links, device="cuda")
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, kb, 4,
                              descending=desc, kind=kind)
    pv = torch.empty_like(li.next) if prev else None
    h, out = p.sort_list(li.keys, li.next, li.head, key_bits=kb, digit_bits=K, key_kind=kind, descending=desc,
                         out_prev=pv)
    torch.cuda.synchronize()
    ok = h == oh and np.array_equal(out.cpu().numpy().view(np.uint32), on)
    if ok and prev:
        ok = np.array_equal(pv.cpu().numpy().view(np.uint32), oracle.repair_back(on, oh))
    if ok and n <= 1_000_000 and rng.random() < 0.3:  # the same keys as an array
        idx, _ = p.sort_array(li.keys, key_bits=kb, digit_bits=K, key_kind=kind, descending=desc)
        # the oracle's list sort of the array read as a list (next[i] = i + 1)
        nx = np.arange(1, n + 1, dtype=np.uint32)
        nx[-1] = 0xFFFFFFFF
        ah, an = oracle.pbit_sort(workloads.keys_numpy(li), nx, 0, kb, 4, descending=desc, kind=kind)
        want = np.empty(n, np.uint32)
        v = ah
        for i in range(n):
            want[i] = v
            v = an[v]
        ok = np.array_equal(idx.cpu().numpy().view(np.uint32), want)
    cases += 1
    if not ok:
        fails += 1
        print(f"FAIL n={n} u{kb} {keys}/{links} K={K} {kind}{' desc' if desc else ''}{' prev' if prev else ''} "
              f"seed={seed}", flush=True)
print(f"{cases - fails}/{cases} random cases bit-exact in {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
