"""Per-source-line stall-reason breakdown of an ncu report (needs -lineinfo):
    python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg, tot = None, None, [], 0
totals = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    col = {h: i for i, h in enumerate(hdr)}
    try:
        samp = int(r[col["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    st = {}
    for h, i in col.items():
        if h.startswith("stall_"):
            try:
                v = int(r[i])
            except ValueError:
                continue
            if v:
                st[h[6:]] = v
                totals[h[6:]] = totals.get(h[6:], 0) + v
    agg.append((samp, fname, r[0], r[1].strip(), st))
    tot += samp
agg.sort(key=lambda a: -a[0])
print(f"total samples {tot}; by reason: " + ", ".join(f"{k} {v / tot:.1%}" for k, v in sorted(totals.items(), key=lambda kv: -kv[1])[:8]))
for samp, f, ln, src, st in agg[:top]:
    top3 = ", ".join(f"{k} {v / samp:.0%}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{samp / tot:6.1%}  {f}:{ln:5s} {src[:70]:70s} [{top3}]")
