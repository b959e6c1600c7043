"""Mean per-launch duration by kernel from an ncu --csv launch list:
    python tools/kry_launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0][:60]].append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print(f"{k:60s} n={len(v):4d} mean_us={sum(v) / len(v) / 1e3:9.1f}")
