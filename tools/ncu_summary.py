"""Summarise the ncu evidence captured by tools/profile_round.sh into profiles/.

  python tools/ncu_summary.py gpurun_out/<tag> <config> [--out profiles]

Writes profiles/<tag>_launches.md (every launch of one pbit_sort_list call: device time,
share, DRAM bytes), profiles/<tag>_kernels.md (the `--set full` metrics of the hot
kernels) and profiles/traffic_<config>.json (DRAM bytes per launch by phase, read by
bench.py for the roofline `traffic` field).
"""
from __future__ import annotations

import argparse
import csv
import json
import os
from collections import OrderedDict


def phase_of(name: str, onesweep_idx: int, key_passes: int) -> str:
    if "k_pack" in name:
        return "pack"
    if "k_rank" in name:
        return "rank"
    if "k_walk" in name:
        return "walk"
    if "k_gather" in name or "k_plan" in name:
        return "gather"
    if "k_onesweep" in name:
        # every k_onesweep launch of a list sort is a key pass (u64 keys: up to 8); the
        # relink has kernels of its own
        return f"pass{onesweep_idx}"
    if "k_relink" in name:
        return "relink"
    if "k_selftest" in name:
        return "selftest"
    return "other"


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hi]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit")
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[ni] == "gpu__time_duration.sum":
            d["ms"] = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                       "second": 1e3, "s": 1e3}.get(unit, 1e-6) * v
        else:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[r[ni]] = v * scale
    return list(launches.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("config")
    ap.add_argument("--out", default="profiles")
    ap.add_argument("--key-passes", type=int, default=4)
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    tag = os.path.basename(a.dir.rstrip("/"))
    os.makedirs(a.out, exist_ok=True)
    L = read_launches(os.path.join(a.dir, "launches.csv"))
    # pbit kernels only (drop torch's generator kernels); the timed call is the last one
    L = [x for x in L if "pbit::" in x["name"] or x["name"].startswith(("k_", "void k_", "void pbit"))]
    starts = [i for i, x in enumerate(L) if "k_pack" in x["name"]]
    call = L[starts[-1]:] if starts else L
    tot = sum(x.get("ms", 0) for x in call)
    k_os = 0
    by_phase = OrderedDict()
    lines = [f"# ncu launch list -- {tag} ({a.config}), one pbit_sort_list call",
             "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` (serialised, cold-cache launches: compare shares, not absolutes).",
             "",
             "| # | kernel | phase | ms | share | DRAM read GB | DRAM write GB |",
             "|---|---|---|---|---|---|---|"]
    for i, x in enumerate(call):
        name = x["name"].split("(")[0].replace("void ", "")
        ph = phase_of(name, k_os, a.key_passes)
        if "k_onesweep" in name:
            k_os += 1
        r, w = x.get("dram__bytes_read.sum", 0), x.get("dram__bytes_write.sum", 0)
        p = by_phase.setdefault(ph, {"ms": 0.0, "read": 0.0, "write": 0.0, "launches": 0})
        p["ms"] += x.get("ms", 0)
        p["read"] += r
        p["write"] += w
        p["launches"] += 1
        lines.append(f"| {i} | `{name[:60]}` | {ph} | {x.get('ms', 0):.4f} | {100 * x.get('ms', 0) / tot:.1f}% | "
                     f"{r / 1e9:.3f} | {w / 1e9:.3f} |")
    lines += ["", f"Total device time of the call: {tot:.3f} ms", "", "## By phase", "",
              "| phase | launches | ms | share | DRAM GB (r+w) | DRAM GB/s |", "|---|---|---|---|---|---|"]
    for ph, p in by_phase.items():
        gb = (p["read"] + p["write"]) / 1e9
        lines.append(f"| {ph} | {p['launches']} | {p['ms']:.3f} | {100 * p['ms'] / tot:.1f}% | {gb:.3f} | "
                     f"{gb / (p['ms'] / 1e3) if p['ms'] else 0:.0f} |")
    open(os.path.join(a.out, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    traffic = {ph: p["read"] + p["write"] for ph, p in by_phase.items()}
    traffic["_source"] = f"profiles/{tag}_launches.md (ncu dram__bytes_read.sum + dram__bytes_write.sum per phase)"
    json.dump(traffic, open(os.path.join(a.out, f"traffic_{a.config}.json"), "w"), indent=1)

    # full-set metrics of the hot kernels
    raw = os.path.join(a.dir, "full_raw.csv")
    if os.path.exists(raw):
        rows = list(csv.reader(open(raw)))
        h = rows[0]
        want = [("gpu__time_duration.sum", "duration ms"), ("dram__bytes_read.sum", "DRAM read"),
                ("dram__bytes_write.sum", "DRAM write"),
                ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
                ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
                ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
                ("launch__registers_per_thread", "regs/thread"),
                ("launch__occupancy_limit_registers", "CTA limit (regs)"),
                ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
                ("smsp__inst_executed.sum", "warp instructions"),
                ("lts__t_sector_hit_rate.pct", "L2 hit %")]
        idx = [(h.index(k), lab) for k, lab in want if k in h]
        units = rows[1]
        out = [f"# ncu --set full -- {tag} ({a.config}): hot kernels", "",
               "| kernel | " + " | ".join(lab for _, lab in idx) + " |",
               "|---|" + "---|" * len(idx)]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:48]
            cells = []
            for i, _ in idx:
                u = units[i]
                cells.append(f"{r[i]} {u}".strip())
            out.append(f"| `{name}` | " + " | ".join(cells) + " |")
        open(os.path.join(a.out, f"{tag}_kernels.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(lines[-(len(by_phase) + 2):]))


if __name__ == "__main__":
    main()
