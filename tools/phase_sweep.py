"""Per-phase device ms of pbit_sort_list on a config (CUDA events inside the library)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0511020_b200 as pbit  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--digit-bits", type=int, default=0)
ap.add_argument("--tag", default="")
a = ap.parse_args()
c = workloads.CONFIGS[a.config]
li = workloads.make_config(a.config, device="cuda", n=a.n)
out = torch.empty_like(li.next)
K = a.digit_bits or c["digit_bits"]
for _ in range(2):
    pbit.sort_list(li.keys, li.next, li.head, digit_bits=K, out_next=out)
acc = {}
for _ in range(a.reps):
    _, _, ph = pbit.sort_list(li.keys, li.next, li.head, digit_bits=K, out_next=out, timing=True)
    for k, v in ph.items():
        acc[k] = acc.get(k, 0) + v / a.reps
tot = sum(v for k, v in acc.items() if k not in ("passes_run", "launches"))
print(json.dumps({"tag": a.tag, "config": a.config, "K": K, "total_ms": round(tot, 3),
                  **{k: round(v, 3) for k, v in acc.items()}}))
