"""Summarise one-kernel `ncu --set full` captures (.ncu-rep) into a short
table: duration, DRAM traffic and throughput, L2 hit rate, occupancy limits,
registers and the top warp-stall reasons.

    python tools/ncu_full_summary.py gpurun_out/full_*.ncu-rep > profiles/rNN_ncu_full_summary.txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes_read.sum.per_second", "dram read rate"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "blocks/SM (regs)"),
    ("launch__occupancy_limit_shared_mem", "blocks/SM (smem)"),
    ("launch__occupancy_limit_warps", "blocks/SM (warps)"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def summarise(path):
    for hdr, units, r in raw(path):
        col = {h: i for i, h in enumerate(hdr)}
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "")
        print(f"== {name}  [{path.split('/')[-1]}]")
        for key, label in KEYS:
            if key in col:
                print(f"   {label:24s} {r[col[key]]:>14s} {units[col[key]]}")
        stalls = []
        for h, i in col.items():
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", h)
            if m and r[i]:
                try:
                    stalls.append((float(r[i].replace(",", "")), m.group(1)))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarise(p)
