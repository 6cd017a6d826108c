"""Run pbit_sort_list `--reps` times on a config (the command profiled by ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0511020_b200 as pbit  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--digit-bits", type=int, default=0)
a = ap.parse_args()
c = workloads.CONFIGS[a.config]
li = workloads.make_config(a.config, device="cuda", n=a.n)
out = torch.empty_like(li.next)
torch.cuda.synchronize()
for _ in range(a.reps):
    h, _ = pbit.sort_list(li.keys, li.next, li.head, digit_bits=a.digit_bits or c["digit_bits"], out_next=out)
torch.cuda.synchronize()
print("ok head", h)
