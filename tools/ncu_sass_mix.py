"""Instruction mix and stall hot spots of one kernel from an ncu report:
    python tools/ncu_sass_mix.py report.ncu-rep [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
mix = defaultdict(int)
samp = defaultdict(int)
tot_i = tot_s = 0
for r in body:
    op = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", op).split(" ")[0]
    base = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    mix[base] += n
    samp[base] += s
    tot_i += n
    tot_s += s
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for k in sorted(mix, key=lambda k: -mix[k])[:top]:
    print(f"  {k:10s} {mix[k]:12d} {mix[k] / tot_i:6.1%}   samples {samp[k] / max(tot_s, 1):6.1%}")
print("hottest instructions (stall samples):")
for r in sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f"  {r[ix['Address']][-5:]} {int(r[ix['Warp Stall Sampling (All Samples)']]):6d}  {r[ix['Source']].strip()[:90]}")
