"""Small sorts through every kernel family, for compute-sanitizer (one tool per gpurun call):
the general list path (pack, walk, ranking, passes, relink with out_prev), the single-cluster
small path, the array sort, host buffers, and the multi-GPU call on a 1-rank communicator
(both transports).  Inputs are generated on the host (no torch kernels to sanitise)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0511020_b200 as pbit  # noqa: E402
import workloads  # noqa: E402


def check(li, h, out):
    oh, on = oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, li.key_bits, 4)
    got = out.cpu().numpy().view(np.uint32) if isinstance(out, torch.Tensor) else out
    assert h == oh and np.array_equal(got, on), li.name


torch.cuda.set_device(0)
li = workloads.make_list(100003, 32, seed=7, keys="zipf")
prev = torch.empty(li.n, dtype=torch.int32, device="cuda")
h, out = pbit.sort_list(li.keys.cuda(), li.next.cuda(), li.head, out_prev=prev)
check(li, h, out)
li = workloads.make_config("C1")
h, out = pbit.sort_list(li.keys.cuda(), li.next.cuda(), li.head, digit_bits=4)
check(li, h, out)
li = workloads.make_list(70001, 64, seed=9, keys="runs4096")
h, out = pbit.sort_list(workloads.keys_numpy(li), workloads.next_numpy(li), li.head)   # host buffers
check(li, h, out)
idx, _ = pbit.sort_array(li.keys.cuda(), key_bits=64)
assert np.array_equal(idx.cpu().numpy(), np.argsort(workloads.keys_numpy(li), kind="stable"))
for t in ("peer", "nccl"):
    os.environ["PBIT_MG_TRANSPORT"] = t
    comm = pbit.mg_comm_init(1, pbit.mg_unique_id(), 0)
    li = workloads.make_list(50021, 32, seed=3, keys="uniform")
    h, out = pbit.sort_list_mg(li.keys.cuda(), li.next.cuda(), li.head, li.n, 0, comm)
    check(li, h, out)
    pbit.mg_comm_destroy(comm)
print("sanitize_small ok")
