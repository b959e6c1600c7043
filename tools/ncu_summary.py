"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("<unnamed>::", "")
        name = re.sub(r"<.*", "", name)
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    unit = "ns"
    s = sum(tot.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:28s} {cnt[k]:8d} {tot[k] / 1e6:10.2f} {tot[k] / s:7.3f} {tot[k] / cnt[k] / 1e3:9.1f}")
    print(f"{'total':28s} {sum(cnt.values()):8d} {s / 1e6:10.2f}   ({unit} per launch, cold-cache serialised)")


if __name__ == "__main__":
    main(sys.argv[1])
