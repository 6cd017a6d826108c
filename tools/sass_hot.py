"""Summarise `ncu --page source --print-source sass --csv` output: hottest instructions
by warp-stall samples and by instructions executed."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot_s = sum(f(r[si]) for r in data)
tot_i = sum(f(r[ie]) for r in data)
print(f"instructions {len(data)} samples {tot_s:.0f} warp-inst {tot_i:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(data)), key=lambda i: -f(data[i][si]))[:n]
for i in sorted(top):
    r = data[i]
    print(f"{i:5d} {f(r[si]) / tot_s * 100:5.1f}%  {f(r[ie]):12.0f}  {r[1][:90]}")
