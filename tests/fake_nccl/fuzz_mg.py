"""TEST INFRASTRUCTURE: randomised multi-rank sweep of pbit_sort_list_mg (G = 2..8 host
threads on one GPU, stand-in NCCL transport), every case bit-exact against the oracle.

    python tests/fake_nccl/fuzz_mg.py [seconds] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import run_mg_threads as R  # noqa: E402  (loads the stand-in-transport library first)

import numpy as np  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 180.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
t0, cases, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    G = int(rng.integers(2, 9))
    n = int(np.exp(rng.uniform(np.log(2), np.log(1_500_000))))
    kb = int(rng.choice([8, 16, 32, 64]))
    keys = str(rng.choice(["uniform", "zipf", "equal", "sorted", "reverse", "runs4096"]))
    links = str(rng.choice(["random", "identity", "push"]))
    K = int(rng.choice([0, 3, 4, 8, 12]))
    kind = str(rng.choice(["unsigned", "signed", "float"])) if kb >= 16 else "unsigned"
    desc = bool(rng.random() < 0.3)
    prev = bool(rng.random() < 0.4)
    ok, msg, stuck = R.run_case(G, n, kb, keys, links, K, kind, desc, prev, seed=int(rng.integers(1 << 30)))
    cases += 1
    if not ok:
        fails += 1
        print(f"FAIL G={G} n={n} u{kb} {keys}/{links} K={K} {kind} desc={desc} prev={prev}: {msg}", flush=True)
        if stuck:
            os._exit(1)
print(f"{cases - fails}/{cases} random multi-rank cases bit-exact in {time.time() - t0:.0f} s", flush=True)
sys.exit(1 if fails else 0)
