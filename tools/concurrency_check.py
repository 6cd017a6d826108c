import sys, threading, numpy as np, torch
sys.path.insert(0, '.')
import paper_cs_0511020_b200 as pbit, workloads, oracle
lists = [workloads.make_list(n, 32, seed=40 + i, keys="zipf", device="cuda") for i, n in enumerate((30011, 150001, 60013, 250007))]
want = [oracle.pbit_sort(workloads.keys_numpy(li), workloads.next_numpy(li), li.head, 32, 4) for li in lists]
outs = [torch.empty_like(li.next) for li in lists]
errs = []
def work(i):
    try:
        s = torch.cuda.Stream(); li = lists[i]
        for _ in range(3):
            h, _ = pbit.sort_list(li.keys, li.next, li.head, out_next=outs[i], stream=s)
        s.synchronize()
        assert h == want[i][0] and np.array_equal(outs[i].cpu().numpy().view(np.uint32), want[i][1]), i
    except Exception as e:
        errs.append(repr(e))
ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
[t.start() for t in ts]; [t.join() for t in ts]
print("errors:", errs)
