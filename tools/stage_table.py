"""Compact table of tools/stage_probe.py outputs: python tools/stage_table.py file..."""
import json
import sys

for f in sys.argv[1:]:
    print(f)
    tot = 0.0
    n = 0
    for l in open(f):
        if '{' not in l:
            continue
        st, js = l.split(' ', 1)
        d = json.loads(js)
        tot += d['step_ms']
        n += 1
        print(f"  {st:4s} step {d['step_ms']:.4f} k {d['kernels']:3d} fwd {d['dag_forward']:.4f} sf {d['scoring_forward']:.4f} "
              f"sb {d['scoring_backward']:.4f} bwd {d['dag_backward']:.4f} sp {d['sparse_adam']:.4f} dn {d['dense_adam']:.4f}")
    if n:
        print(f"  mean step {tot / n:.4f} ms")
