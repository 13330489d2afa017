"""Summarise an ncu --csv launch list: last N launches, per-kernel totals."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum':
            out.append((int(d['ID']), d['Kernel Name'], float(d['Metric Value'].replace(',', ''))))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tail = out[-n:]
tot = sum(t for _, _, t in tail)
agg = collections.defaultdict(float)
for i, k, t in tail:
    agg[k.split('(')[0][-60:]] += t
for k, t in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{t/1e3:9.1f} us {100*t/tot:5.1f}%  {k}")
print(f"total {tot/1e3:.1f} us over {len(tail)} launches")
if len(sys.argv) > 3:
    for i, k, t in tail: print(i, f"{t/1e3:8.1f}", k[:90])
