"""Print an ncu --csv --metrics log as one row per launch: python tools/ncu_table.py <csv>"""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    key = (r["ID"], r["Kernel Name"][:60])
    rows.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
names = []
for v in rows.values():
    for m in v:
        if m not in names:
            names.append(m)
short = [m.replace("gpu__time_duration.sum", "time").replace("dram__bytes_", "dram_").replace(".sum", "")
         .replace("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%").replace("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%") for m in names]
print("| id | kernel | " + " | ".join(short) + " |")
for (i, k), v in rows.items():
    print(f"| {i} | {k} | " + " | ".join(f"{v[m][0]} {v[m][1]}" if m in v else "" for m in names) + " |")
