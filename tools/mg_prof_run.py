"""One pbit_sort_list_mg call on a 1-rank communicator (the command ncu profiles for the
multi-GPU protocol's per-kernel costs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0511020_b200 as pbit  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
li = workloads.make_config(cfg, device="cuda")
comm = pbit.mg_comm_init(1, pbit.mg_unique_id(), 0)
out = torch.empty_like(li.next)
pbit.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, out_next_local=out)
torch.cuda.synchronize()
pbit.mg_comm_destroy(comm)
print("ok")
