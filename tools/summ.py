"""Summaries of bench JSON lines and ncu CSVs in gpurun_out/ (tools/summ.py FILE...)."""
import collections
import csv
import json
import sys

for f in sys.argv[1:]:
    if f.endswith(".json"):
        for line in open(f):
            if line.startswith("{"):
                d = json.loads(line)
                r = d.get("roofline", {})
                print(f, d.get("value"), (d.get("e2e") or {}).get("value"), d.get("ms_per_step"), r.get("kernel"),
                      r.get("frac"), r.get("stage_ms"), r.get("all"), d.get("ms_per_step_by_structure"))
    elif f.endswith(".csv"):
        hdr, data = None, collections.defaultdict(lambda: collections.defaultdict(list))
        for r in csv.reader(open(f)):
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr is None or len(r) < len(hdr):
                continue
            d = dict(zip(hdr, r))
            data[d["Kernel Name"].split("(")[0][:60]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
        print(f)
        for k, v in data.items():
            t, rd, wr = v["gpu__time_duration.sum"], v["dram__bytes_read.sum"], v["dram__bytes_write.sum"]
            n = len(t)
            if n:
                print(f"  {k:60s} n={n} t={sum(t) / n / 1e3:.2f}us rd={sum(rd) / n / 1e6:.2f}MB "
                      f"wr={sum(wr) / n / 1e6:.2f}MB  -> {(sum(rd) + sum(wr)) / sum(t):.0f} GB/s")
