"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ inst]) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in data:
    n = d['Kernel Name'].split('(')[0][:64]
    if d['Metric Name'] == 'gpu__time_duration.sum':
        agg[n][0] += 1
        agg[n][1] += float(d['Metric Value']) / 1e3
    else:
        agg[n][2] += float(d['Metric Value'])
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for n, (c, t, ins) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t:9.1f} us {100*t/tot:5.1f}% n={c:3d} avg={t/max(c,1):7.1f} warp-inst/launch={ins/max(c,1)/1e6:7.2f}M  {n}")
