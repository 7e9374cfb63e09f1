"""Print an ncu --csv launch list (gpu__time_duration.sum [+ inst, grid]) one line per launch:
    python tools/launch_table.py gpurun_out/.../launch.csv"""
import csv
import sys
from collections import OrderedDict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
    d = OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[ii], {'name': r[ki]})[r[mi]] = r[vi]
    tot = 0.0
    for k, v in d.items():
        t = float(v.get('gpu__time_duration.sum', 0)) / 1000
        tot += t
        print(f"{k:>4} {t:8.2f} us grid {v.get('launch__grid_size', ''):>6} inst {v.get('smsp__inst_executed.sum', ''):>10}  {v['name'][:80]}")
    print(f"total {tot:.1f} us over {len(d)} launches")
