#!/usr/bin/env python
"""tools/make_goldens.py -- golden results of the BASELINE.json configs, from the ORACLE only.

For each config the list is generated on the host by workloads.py (the same generator
the GPU tests run on the device; the input hash is stored so the GPU side proves it sorted
the same list) and sorted by the paper-literal oracle (oracle.pbit_sort, K = 4: the
listing P:346-361 with the ascending loops P:379-380).  Stored per config in
tests/golden/config_<name>.json:

  n, key_bits, seed        the workload (workloads.CONFIGS / the extra cases below)
  input_sha256             sha256(keys bytes || next bytes || head as u32 LE)
  out_head                 the oracle's head of the sorted list
  out_next_sha256          sha256 of the oracle's out_next (u32 LE, node-indexed)
  payload_seq_sha256       (keys with a payload, C4) sha256 of payload[v_0], payload[v_1], ...
                           along the oracle's sorted list (reading Q11: the payload
                           follows its node)
  oracle_s, cpu            wall time of the oracle call and the CPU it ran on

No value here comes from the CUDA path: this script imports only oracle/ and workloads.py.

  python tools/make_goldens.py C1 C2 X26 C3 C4 C5 C3:float C4:signed:desc
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# Extra oracle-compared cases beyond C1..C5: sizes that are not powers of two and reach
# the plan classes of the full configs (ruler spacing 64 from 2^26 nodes).
EXTRA = {
    "X26": dict(n=(1 << 26) + 4099, key_bits=32, keys="zipf", links="random", seed=2626, digit_bits=8,
                desc="n=2^26+4099, u32 Zipf(1.1), random links (plan class s=64, ragged tail)"),
    "X26u64": dict(n=(1 << 26) - 777, key_bits=64, keys="runs4096", links="random", seed=2664, digit_bits=8,
                   desc="n=2^26-777, u64 runs4096 + payload, random links"),
}


def make(name: str):
    if name in workloads.CONFIGS:
        c = workloads.CONFIGS[name]
        return workloads.make_config(name), c
    c = EXTRA[name]
    li = workloads.make_list(c["n"], c["key_bits"], c["seed"], keys=c["keys"], links=c["links"])
    li.name = name
    return li, c


def input_sha256(keys: np.ndarray, nxt: np.ndarray, head: int) -> str:
    h = hashlib.sha256()
    h.update(memoryview(np.ascontiguousarray(keys)).cast("B"))
    h.update(memoryview(np.ascontiguousarray(nxt)).cast("B"))
    h.update(np.array([head & 0xFFFFFFFF], np.uint32).tobytes())
    return h.hexdigest()


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def main(names):
    for spec in names:
        # "<config>[:<kind>[:desc]]" -- key kinds and the descending order (N1) at full size
        parts = spec.split(":")
        name, kind, desc = parts[0], parts[1] if len(parts) > 1 else "unsigned", len(parts) > 2 and parts[2] == "desc"
        t0 = time.time()
        li, c = make(name)
        keys = workloads.keys_numpy(li)
        nxt = workloads.next_numpy(li)
        head = li.head
        payload = li.payload.numpy() if li.payload is not None else None
        del li
        t_gen = time.time() - t0
        ih = input_sha256(keys, nxt, head)
        t1 = time.time()
        oh, on = oracle.pbit_sort(keys, nxt, head, c["key_bits"], 4, descending=desc, kind=kind)
        t_or = time.time() - t1
        rec = {"n": int(nxt.shape[0]), "key_bits": c["key_bits"], "seed": c["seed"], "desc": c["desc"],
               "input_sha256": ih, "out_head": int(oh), "out_next_sha256": hashlib.sha256(on.tobytes()).hexdigest(),
               "oracle_K": 4, "oracle_s": round(t_or, 2), "gen_s": round(t_gen, 2),
               "cpu": f"{cpu_model()}, 1 thread (nproc {os.cpu_count()})"}
        if payload is not None:
            order = oracle.list_order(on, oh)
            rec["payload_seq_sha256"] = hashlib.sha256(payload[order].tobytes()).hexdigest()
            del order
        del on, keys, nxt, payload
        gname = name if (kind == "unsigned" and not desc) else f"{name}_{kind}{'_desc' if desc else ''}"
        rec.update(name=gname, config=name, kind=kind, descending=desc)
        print(gname, json.dumps(rec), flush=True)
        out = os.path.join(GOLDEN_DIR, f"config_{gname}.json")
        with open(out + ".tmp", "w") as f:
            json.dump(rec, f, indent=1, sort_keys=True)
            f.write("\n")
        os.replace(out + ".tmp", out)


if __name__ == "__main__":
    oracle.build()
    main(sys.argv[1:] or ["C1", "C2"])
