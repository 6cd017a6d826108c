"""Time pbit_sort_list_mg on a 1-rank communicator vs pbit_sort_list (same list): the
protocol's own cost on one GPU (no NVLink traffic)."""
import os
import sys

os.environ.setdefault("PBIT_POOL_KEEP_GB", "96")  # as bench.py: workspace kept mapped between calls
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0511020_b200 as pbit  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
li = workloads.make_config(cfg, device="cuda")
comm = pbit.mg_comm_init(1, pbit.mg_unique_id(), 0)
out = torch.empty_like(li.next)
st = torch.cuda.current_stream()
for name, fn in (("single", lambda: pbit.sort_list(li.keys, li.next, li.head, out_next=out)),
                 ("mg G=1", lambda: pbit.sort_list_mg(li.keys, li.next, li.head, li.n, 0, comm, out_next_local=out))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{cfg} {name}: {e0.elapsed_time(e1) / 5:.3f} ms"
          + (f" (transport {pbit.mg_transport(comm)})" if name.startswith("mg") else ""))
pbit.mg_comm_destroy(comm)
