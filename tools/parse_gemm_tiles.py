"""Pair tools/gemm_tiles.py's log lines with the ncu launch list (GEMM + its split-K reduce)."""
import csv
import sys

csvf, logf = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(csvf)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
seq = []
for r in rows[hdr + 1:]:
    d = dict(zip(rows[hdr], r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    n = d["Kernel Name"]
    if "gemm_tf32x3" in n or "gemm_reduce" in n:
        seq.append(("R" if "reduce" in n else "G", d["Grid Size"], float(d["Metric Value"].replace(",", "")) / 1e3))
calls, i = [], 0
while i < len(seq):
    t, g = seq[i][2], seq[i][1]
    i += 1
    if i < len(seq) and seq[i][0] == "R":
        t += seq[i][2]
        i += 1
    calls.append((t, g))
logs = [l.strip() for l in open(logf) if l.startswith("M=")]
for j, l in enumerate(logs):
    c = calls[3 * j:3 * j + 3]
    print(f"{l.split(': relerr')[0]:55s} {min(x[0] for x in c):7.1f} us grid={c[0][1]}  {l.split(': ')[-1]}")
