"""Stall samples per CUDA source line of a kernel in an ncu report:
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = []
tot = 0
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0]:
        continue
    try:
        samp = int(r[4])
        inst = int(r[7] or 0)
    except ValueError:
        continue
    agg.append((samp, inst, fname, r[0], r[1].strip()))
    tot += samp
agg.sort(reverse=True)
print(f"total samples {tot}")
for samp, inst, f, ln, src in agg[:top]:
    print(f"{samp / tot:6.1%} {inst:11d}  {f}:{ln:5s} {src[:90]}")
