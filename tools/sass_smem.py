import csv, sys
lines = open(sys.argv[1]).read().splitlines()
hi = next(i for i,l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(lines[hi:]))
hdr = rows[0]; H = {h:i for i,h in enumerate(hdr)}
def f(r,k):
    try: return float(r[H[k]].replace(',',''))
    except: return 0.0
data = rows[1:]
half = len(data)//2
if half and all(data[i][1] == data[i+half][1] for i in range(0, min(50, half))): data = data[:half]
acc = {}
for r in data:
    w = f(r,'L1 Wavefronts Shared')
    if w == 0: continue
    op = r[1].split()
    op = op[1] if op[0].startswith('@') else op[0]
    a = acc.setdefault(op, [0, 0])
    a[0] += w; a[1] += f(r,'Instructions Executed')
print(lines[0][:100])
for k, (w, i) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:20s} wf={w/1e6:7.2f}M inst={i/1e6:6.2f}M wf/inst={w/max(i,1):5.2f}")
