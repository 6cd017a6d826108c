"""Host-side cost of one small call (C1): wall time per pbit_sort_list through the Python
binding vs through ctypes directly (preallocated output, no timing events), against the
kernel's device time."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0511020_b200 as p  # noqa: E402
import workloads  # noqa: E402

li = workloads.make_config("C1", device="cuda")
out = torch.empty_like(li.next)
for _ in range(20):
    p.sort_list(li.keys, li.next, li.head, digit_bits=4, out_next=out)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    p.sort_list(li.keys, li.next, li.head, digit_bits=4, out_next=out)
t1 = time.perf_counter()
oh = ctypes.c_uint32(0)
o = p._opts(4, torch.cuda.current_stream().cuda_stream, None, None)
kp, np_, op = li.keys.data_ptr(), li.next.data_ptr(), out.data_ptr()
f = p.lib.pbit_sort_list
t2 = time.perf_counter()
for _ in range(N):
    f(kp, np_, li.head, li.n, 8, ctypes.byref(oh), op, ctypes.byref(o))
t3 = time.perf_counter()
_, _, ph = p.sort_list(li.keys, li.next, li.head, digit_bits=4, out_next=out, timing=True)
print(f"python binding {1e6 * (t1 - t0) / N:.1f} us/call, raw ctypes {1e6 * (t3 - t2) / N:.1f} us/call, "
      f"kernel {1e3 * ph['walk']:.1f} us")
