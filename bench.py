#!/usr/bin/env python
"""bench.py -- sorted list nodes/s on B200 (BASELINE.json metric), one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A step is one pbit_sort_list call (the whole hot path) on the
configured synthetic list, inputs resident in HBM.  Default workload: C3 (n = 2^28
u32 Zipf(1.1) keys, random-permutation links) -- the 1-GPU config the north star gates
on.  Inputs (2 GiB) are larger than L2 (126 MB), so no explicit flush is needed.

N > 1 (torchrun): ONE list of the config's size is sorted by all ranks together through
pbit_sort_list_mg (node ids sharded by rank, key-range exchange over NCCL; strong
scaling); value = n / max-over-ranks device time.

--impl reference: the CPU oracle (the paper's algorithm, oracle/) timed on the host on
bounded samples of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# The library returns its workspace to the device after every call by default (pbit.h);
# a caller that sorts repeatedly keeps it mapped with PBIT_POOL_KEEP_GB (opt-in, stated
# in the JSON line's config).  Set before libpbit.so creates its pool.
os.environ.setdefault("PBIT_POOL_KEEP_GB", "96")

METRIC = "sorted list nodes/sec at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "nodes/s"

# Algorithmic bytes per node of each kernel phase: every
# array element the phase must read or write, counted once at element size.
#   kb = key bytes as stored in the pass buffers (4 for u8/u16/u32, 8 for u64)
def phase_bytes_per_node(key_bits: int):
    kin = key_bits // 8
    kb = 8 if key_bits == 64 else 4
    rec = 16 if key_bits == 64 else 8
    return {
        "pack": kin + 4 + rec,          # read key, next; write AoS record
        "walk": rec + (kb + 4),         # read record (random), write (key,id) to its slot
        "rank": 0,                      # per-ruler, ~n/64 entries: not per node
        "gather": (kb + 4) * 2,         # read slot, write list-order key + id
        "pass": (kb + 4) * 2,           # read key+id, write key+id
        "pass_last": (kb + 4) + 4,      # read key+id, write id
        "relink": 4 + 4,                # read sorted ids, write out_next (random)
    }


# Measured ceiling of dependent random 8 B reads on this B200 (G lines/s; each read moves a
# 128 B line): tools/micro/randread.cu, DESIGN.md §6.
WALK_LINE_CEILING_G = 39.5


def method_bytes_per_node(key_bits: int):
    """The one-read-one-write lower bound of the method: read key and next, write
    out_next."""
    return key_bits // 8 + 4 + 4


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bench_config(cfg: str, n: int, K: int, ws: int = 1) -> dict:
    """The `config` object of the JSON line: identical for our arm and the reference arm."""
    import workloads
    c = workloads.CONFIGS[cfg]
    kb = c["key_bits"]
    return {"workload": cfg, "desc": c["desc"], "n_per_gpu": n, "key_bits": kb, "digit_bits": K,
            "parallelism": "single GPU" if ws == 1 else f"one list, node ids sharded over {ws} ranks, "
                                                         "key-range exchange (NCCL)",
            "l2": "inputs larger than L2 (no flush needed)" if n * (kb // 8 + 4) > 126e6 else "inputs smaller than L2",
            "workspace_pool_keep_gb": float(os.environ.get("PBIT_POOL_KEEP_GB", "0"))}


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def full_size_oracle(cfg: str):
    """The oracle's time on the FULL config, from the golden it produced
    (tests/golden/config_<cfg>.json, tools/make_goldens.py; another host: context only)."""
    p = os.path.join(ROOT, "tests", "golden", f"config_{cfg}.json")
    try:
        with open(p) as f:
            g = json.load(f)
        return {"n": g["n"], "seconds": g["oracle_s"], "nodes_per_s": round(g["n"] / g["oracle_s"], 1),
                "cpu": g.get("cpu"), "source": os.path.relpath(p, ROOT)}
    except Exception:
        return None


def cpu_baseline(cfg: str, sample_n: int, reps: int = 1):
    """The oracle as it stands (paper-literal Pbit, K=4, one thread) on a bounded
    sample of the workload, on this host's cores."""
    import oracle
    import workloads
    c = workloads.CONFIGS[cfg]
    li = workloads.make_config(cfg, n=sample_n)
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    oracle.build()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.pbit_sort(keys, nxt, li.head, c["key_bits"], 4)
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    # SURVEY §8(d)'s optional variant: the recursion below the first two levels on every
    # host core (bit-identical to the serial oracle, tests/test_oracle.py)
    nthr = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.pbit_sort_par(keys, nxt, li.head, c["key_bits"], 4, nthr)
    tp = time.perf_counter() - t0
    return {"value": sample_n / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "cpu": cpu_model(), "host_threads": os.cpu_count(),
            "subtree_parallel": {"value": sample_n / tp, "unit": UNIT, "cores": nthr, "seconds": round(tp, 2)},
            "sample": f"{cfg}-shaped list, n={sample_n} of the config's {c['n']} (seed {c['seed']}), "
                      f"paper-literal Pbit K=4, mean of {reps} run(s), {t:.2f} s each, single thread",
            "full_size": full_size_oracle(cfg)}


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    import workloads
    c = workloads.CONFIGS[args.config]
    sample_n = min(c["n"], args.ref_sample)
    import oracle
    li = workloads.make_config(args.config, n=sample_n)
    keys, nxt = workloads.keys_numpy(li), workloads.next_numpy(li)
    oracle.build()
    for _ in range(args.warmup):
        oracle.pbit_sort(keys, nxt, li.head, c["key_bits"], 4)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.pbit_sort(keys, nxt, li.head, c["key_bits"], 4)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    value = sample_n / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32" if c["key_bits"] <= 32 else "u64",
            "data": "synthetic",
            "config": dict(bench_config(args.config, sample_n, args.digit_bits or c["digit_bits"], args.gpus),
                           sample_of_n=c["n"] if args.n is None else args.n,
                           parallelism="one host thread (the oracle, K=4)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu": cpu_model(),
                             "host_threads": os.cpu_count(),
                             "sample": f"each step: a bounded sample of the workload, a {args.config}-shaped list "
                                       f"of n={sample_n} (the config has {c['n']}) sorted by the paper-literal "
                                       f"Pbit (K=4) on one core; {args.steps} timed steps",
                             "full_size": full_size_oracle(args.config)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def load_traffic(cfg: str):
    """ncu dram bytes per launch for the config's kernels, from the committed profile
    summary (profiles/traffic_<cfg>.json written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


def nvlink_model(n: int, G: int, key_bits: int, transport: str) -> dict:
    """Bytes each rank moves over NVLink per pbit_sort_list_mg call (a model):
    the walk's remote node reads (one 32 B sector per remote step, (G-1)/G of the n/G steps a
    rank walks), the segment-table all-gather, the chunk gather from the walkers' slots, the
    key-range scatter and the relink routing ((G-1)/G of each rank's n/G records); the NCCL
    transport replaces the remote reads by an all-gather of the whole (key, next) array."""
    f = (G - 1) / G
    per = n / G
    kb = 8 if key_bits == 64 else 4
    rec = 16 if key_bits == 64 else 8
    seg_table = f * (n / 64 + n / 256) * 8
    parts = {"segment_table": seg_table, "key_range_exchange": f * per * (kb + 4), "relink_routing": f * per * 8}
    if transport == "peer":
        parts["walk_remote_reads"] = f * per * 32
        parts["chunk_gather"] = f * per * (kb + 4)
    else:
        parts["kn_allgather"] = f * n * rec
        parts["segment_table"] = f * (n / 64) * 8
    total = sum(parts.values())
    return {"transport": transport, "bytes_per_rank": round(total), "parts": {k: round(v) for k, v in parts.items()},
            "ms_at_770_gbs": round(total / 770e9 * 1e3, 3)}


def run_mg(args):
    """N > 1: one list sorted by every rank together (pbit_sort_list_mg)."""
    import torch
    import torch.distributed as dist

    import paper_cs_0511020_b200 as pbit
    import workloads

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [pbit.mg_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = pbit.mg_comm_init(ws, obj[0], rank)
    c = workloads.CONFIGS[args.config]
    K = args.digit_bits or c["digit_bits"]
    n = c["n"] if args.n is None else args.n
    li = workloads.make_config(args.config, device="cuda", n=n)
    S = pbit.mg_slice(n, ws)
    lo, hi = min(n, rank * S), min(n, rank * S + S)
    node_lo = rank * S  # pbit.h: node_lo = rank * S, also for a rank whose slice is empty
    keys, nxt, head, kb = li.keys[lo:hi].clone(), li.next[lo:hi].clone(), li.head, li.key_bits
    del li
    torch.cuda.empty_cache()
    out = torch.empty_like(nxt)
    st = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        pbit.sort_list_mg(keys, nxt, head, n, node_lo, comm, digit_bits=K, out_next_local=out)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            pbit.sort_list_mg(keys, nxt, head, n, node_lo, comm, digit_bits=K, out_next_local=out)
        e1.record(st)
        torch.cuda.synchronize()
    dist.barrier()
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    # end to end: host slice in, host out_next slice back, every step
    kh, nh = keys.cpu().pin_memory(), nxt.cpu().pin_memory()
    oh = torch.empty_like(nh).pin_memory()
    dist.barrier()
    e_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        kd, nd = kh.to("cuda", non_blocking=True), nh.to("cuda", non_blocking=True)
        pbit.sort_list_mg(kd, nd, head, n, node_lo, comm, digit_bits=K, out_next_local=out)
        oh.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
    e2e_t = torch.tensor([(time.perf_counter() - t0) / e_steps], device="cuda")
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    cpu = cpu_baseline(args.config, min(n, args.cpu_sample)) if rank == 0 and not args.no_cpu_baseline else None
    if rank == 0:
        peak, peak_src = load_peaks()
        mb = method_bytes_per_node(kb)
        per_rank_gbs = mb * (n / ws) / (ms / 1e3) / 1e9
        line = {"metric": METRIC, "value": n / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32" if kb <= 32 else "u64", "data": "synthetic",
                "config": bench_config(args.config, n, K, ws),
                "roofline": {"bound": "hbm", "achieved": round(per_rank_gbs, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(per_rank_gbs / peak, 4), "traffic": None,
                             "kernel": "pbit_sort_list_mg (whole call, method bytes per rank)",
                             "peak_source": peak_src},
                "cpu_baseline": cpu,
                "e2e": {"value": n / float(e2e_t.item()), "unit": UNIT,
                        "h2d_bytes_per_step": (hi - lo) * (kb // 8 + 4), "d2h_bytes_per_step": (hi - lo) * 4},
                "gpu_launches": pbit.last_mg_launches * args.steps, "clocks": clk.summary(),
                "nvlink_model": nvlink_model(n, ws, kb, pbit.mg_transport(comm))}
        print(json.dumps(line), flush=True)
    pbit.mg_comm_destroy(comm)
    dist.destroy_process_group()


def e2e_pipelined(pbit, kh, nh, oh, head, K, n, jobs, ws, threads=2):
    """Sorting a stream of lists from host memory: `threads` host threads, each with its own
    stream and pinned input/output buffers, call the same synchronous host-buffer C-ABI call
    `jobs` times each (calls on distinct streams may run concurrently, pbit.h).  One job's
    H2D overlaps another's device work and D2H (PCIe is full duplex), so the throughput is
    set by the host->device link, not by the sum of copies and compute.  Every job's output
    is checked against the single synchronous call's."""
    import threading

    import torch

    bufs = []
    for _ in range(threads):
        bufs.append((kh.clone().pin_memory(), nh.clone().pin_memory(), torch.empty_like(oh).pin_memory(),
                     torch.cuda.Stream()))
    gate = threading.Barrier(threads + 1)
    errs = []

    def work(i, reps):
        k_, n_, o_, s_ = bufs[i]
        try:
            for r in range(reps + 1):
                if r == 1:
                    gate.wait()  # first call (workspace, copy stream) outside the timed region
                h, _ = pbit.sort_list(k_, n_, head, out_next=o_, digit_bits=K, stream=s_)
                if h != head_ref[0]:
                    errs.append(f"thread {i}: head {h}")
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))
            gate.abort()

    head_ref = [pbit.sort_list(kh, nh, head, out_next=oh, digit_bits=K)[0]]
    ts = [threading.Thread(target=work, args=(i, jobs)) for i in range(threads)]
    for t in ts:
        t.start()
    try:
        gate.wait()
    except threading.BrokenBarrierError:
        pass
    t0 = time.perf_counter()
    for t in ts:
        t.join()
    el = time.perf_counter() - t0
    ok = not errs and all(torch.equal(b[2], oh) for b in bufs)
    return {"value": n * ws * threads * jobs / el if ok else None, "unit": UNIT, "host_threads": threads,
            "jobs": threads * jobs, "seconds": round(el, 4), "outputs_match": ok, "errors": errs[:3],
            "what": "the same host-buffer pbit_sort_list call from several host threads (own stream and "
                    "pinned buffers each): a stream of sort jobs, one job's H2D overlapping another's "
                    "sort and D2H; every output compared with the synchronous call's"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_cs_0511020_b200 as pbit
    import workloads

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    c = workloads.CONFIGS[args.config]
    K = args.digit_bits or c["digit_bits"]
    n = c["n"] if args.n is None else args.n
    li = workloads.make_config(args.config, device="cuda", n=n, seed=c["seed"] + 1000 * rank)
    keys, nxt, head, kb = li.keys, li.next, li.head, li.key_bits
    out = torch.empty_like(nxt)
    st = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        pbit.sort_list(keys, nxt, head, digit_bits=K, out_next=out)
    torch.cuda.synchronize()

    # ---- timed region: K calls, device events on the launching stream.  The library also
    # records CUDA events between its kernels on that stream (timing=True, pooled events),
    # which gives each kernel's live device time inside the same timed calls.
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases = {}
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        e0.record(st)
        for i in range(args.steps):
            step_ev[i].record(st)
            h, _, ph = pbit.sort_list(keys, nxt, head, digit_bits=K, out_next=out, timing=True)
            for k_, v in ph.items():
                phases[k_] = phases.get(k_, 0.0) + v
        step_ev[args.steps].record(st)
        e1.record(st)
        torch.cuda.synchronize()
    step_ms = sorted(step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps))
    ms_median = step_ms[len(step_ms) // 2] if len(step_ms) % 2 else 0.5 * (step_ms[len(step_ms) // 2 - 1] + step_ms[len(step_ms) // 2])
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device="cuda")
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = n * ws / (ms_max / 1e3)
    phases = {k_: v / args.steps for k_, v in phases.items()}
    launches = int(phases.pop("launches"))
    passes_run = int(phases.pop("passes_run"))

    # ---- end to end through the same C-ABI with host (pinned) buffers
    kh = keys.cpu().pin_memory()
    nh = nxt.cpu().pin_memory()
    oh = torch.empty_like(nh).pin_memory()
    pbit.sort_list(kh, nh, head, out_next=oh, digit_bits=K)
    barrier()
    torch.cuda.synchronize()
    e_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        pbit.sort_list(kh, nh, head, out_next=oh, digit_bits=K)
    e2e_s = (time.perf_counter() - t0) / e_steps
    e2e_t = torch.tensor([e2e_s], device="cuda")
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = n * ws / float(e2e_t.item())
    pipelined = e2e_pipelined(pbit, kh, nh, oh, head, K, n, e_steps, ws, args.e2e_threads) if args.e2e_threads > 1 else None
    # the PCIe bound of a synchronous host-buffer call: the same bytes copied alone (pinned
    # H2D of keys + next, D2H of out_next), measured here with plain device copies
    dk, dn = torch.empty_like(keys), torch.empty_like(nxt)
    torch.cuda.synchronize()
    c0 = time.perf_counter()
    for _ in range(3):
        dk.copy_(kh, non_blocking=True)
        dn.copy_(nh, non_blocking=True)
        torch.cuda.synchronize()
    h2d_s = (time.perf_counter() - c0) / 3
    c0 = time.perf_counter()
    for _ in range(3):
        oh.copy_(dn, non_blocking=True)
        torch.cuda.synchronize()
    d2h_s = (time.perf_counter() - c0) / 3
    del dk, dn
    pcie = {"h2d_gbs": round(n * (kb // 8 + 4) / h2d_s / 1e9, 1), "d2h_gbs": round(n * 4 / d2h_s / 1e9, 1),
            "copies_alone_ms": round((h2d_s + d2h_s) * 1e3, 2),
            "bound_nodes_per_s": n / (h2d_s + d2h_s + ms_max / 1e3),
            "note": "copies alone + the device-timed call: what a synchronous call moving these bytes "
                    "over PCIe can reach without overlap; the call overlaps the pack and the apply"}

    # ---- roofline of the dominant kernel
    bpn = phase_bytes_per_node(kb)
    pass_ms = [(k_, v) for k_, v in phases.items() if k_.startswith("pass")]
    cand = {k_: v for k_, v in phases.items() if not k_.startswith("pass")}
    for i, (k_, v) in enumerate(pass_ms):
        cand[k_] = v
    dom = max(cand, key=cand.get)
    if dom.startswith("pass"):
        last_idx = len(pass_ms) - 1
        b = bpn["pass_last"] if dom == pass_ms[last_idx][0] else bpn["pass"]
    else:
        b = bpn[dom]
    peak, peak_src = load_peaks()
    dom_ms = cand[dom]
    achieved = b * n / (dom_ms / 1e3) / 1e9
    traffic = None
    tr = load_traffic(args.config)
    if tr and dom in tr:
        traffic = tr[dom]
    total_alg = sum(bpn["pass"] if k_.startswith("pass") else bpn.get(k_, 0) for k_ in cand)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "kernel_ms": round(dom_ms, 4), "alg_bytes_per_node": b, "peak_source": peak_src,
                "phase_ms": {k_: round(v, 4) for k_, v in phases.items()},
                "whole_call_impl_bytes_per_node": total_alg,
                # the method's one-read-one-write bound (read key + next, write
                # out_next) over the dominant kernel's time and over the whole call
                "method_bytes_per_node": method_bytes_per_node(kb),
                "frac_at_method_bytes": round(method_bytes_per_node(kb) * n / (dom_ms / 1e3) / 1e9 / peak, 4),
                "whole_call_method_frac": round(method_bytes_per_node(kb) * n / (ms / 1e3) / 1e9 / peak, 4)}
    if dom == "walk":
        # the walk visits every node once in list order = one random 128 B line per node
        # (tools/micro/randread.cu); its ceiling is the measured random-line rate
        roofline["walk_random_lines_per_s"] = round(n / (dom_ms / 1e3) / 1e9, 2)
        roofline["walk_random_line_ceiling_per_s"] = WALK_LINE_CEILING_G
        roofline["walk_frac_of_random_line_ceiling"] = round(n / (dom_ms / 1e3) / 1e9 / WALK_LINE_CEILING_G, 4)
    whole = None
    if tr:
        # SURVEY Q16 reading of the north star's HBM gate: DRAM bytes of one whole call
        # (ncu, summed over its launches) / device time of the call
        dram = sum(v for k_, v in tr.items() if not k_.startswith("_"))
        whole = {"dram_bytes_per_call": dram, "ms": round(ms, 4), "gbs": round(dram / (ms / 1e3) / 1e9, 1),
                 "frac_of_peak": round(dram / (ms / 1e3) / 1e9 / peak, 4),
                 "frac_of_nominal_8tbs": round(dram / (ms / 1e3) / 1e9 / 8000.0, 4),
                 # DRAM bytes / time rises with wasted traffic: read it with the amplification
                 # over the method's bound and the work-normalised fraction beside it
                 "amplification_over_method_bytes": round(dram / (method_bytes_per_node(kb) * n), 2),
                 "work_normalised_frac": round(method_bytes_per_node(kb) * n / (ms / 1e3) / 1e9 / peak, 4),
                 "source": tr.get("_source")}

    # ---- the paper's tables-versus-lists comparison on this GPU: the same
    # keys sorted as an ARRAY (pbit_sort_array: the radix passes without ranking/relink)
    idx = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        pbit.sort_array(keys, key_bits=kb, digit_bits=K, out_index=idx)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(st)
    for _ in range(args.steps):
        pbit.sort_array(keys, key_bits=kb, digit_bits=K, out_index=idx)
    a1.record(st)
    torch.cuda.synchronize()
    arr_ms = a0.elapsed_time(a1) / args.steps
    array_ctx = {"what": "same keys sorted as an array (pbit_sort_array -> sorted index), P:1118-1177",
                 "ms": round(arr_ms, 4), "keys_per_s": n / (arr_ms / 1e3), "list_over_array_time": round(ms / arr_ms, 3)}
    del idx

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, min(n, args.cpu_sample), args.cpu_reps)

    clocks = clk.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "ms_per_step_median": round(ms_median, 4),
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32" if kb <= 32 else "u64", "data": "synthetic",
                "config": bench_config(args.config, n, K),
                "passes_run": passes_run,
                "hbm_gbs_method": round(method_bytes_per_node(kb) * n * ws / (ms_max / 1e3) / 1e9, 1),
                "roofline": roofline, "whole_call_dram": whole, "array_sort": array_ctx, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * (kb // 8 + 4),
                        "d2h_bytes_per_step": n * 4 + 4, "pcie": pcie, "pipelined": pipelined},
                "gpu_launches": launches * args.steps, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=None, help="override n (default: the config's)")
    ap.add_argument("--digit-bits", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=1 << 24)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-threads", type=int, default=2, help="host threads of the pipelined e2e (<= 1: off)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[0] > 1:
        run_mg(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
